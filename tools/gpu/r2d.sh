python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/r2d_pytest.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/r2d_pytest.log
python tools/ref_suite/run_ref_suite.py --mode boundary --out gpurun_out/r2d_refsuite_boundary.json > gpurun_out/r2d_refsuite.log 2>&1
python tools/ref_suite/run_ref_suite.py --mode full --out gpurun_out/r2d_refsuite_full.json >> gpurun_out/r2d_refsuite.log 2>&1
grep '^{' gpurun_out/r2d_refsuite.log
timeout 600 python bench.py --T 65536 --window 16384 --steps 2 --warmup 1 --no-cpu-baseline --e2e-T 1024 > gpurun_out/r2d_bench.json 2> gpurun_out/r2d_bench.err; echo "bench rc=$?"
