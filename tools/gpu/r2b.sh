python -m pytest tests/test_gpu_ts.py tests/test_gpu_bench_path.py -x -q -m gpu -p no:cacheprovider > gpurun_out/r2b_pytest.log 2>&1; echo "pytest rc=$?"
tail -5 gpurun_out/r2b_pytest.log
timeout 600 python bench.py --T 65536 --window 16384 --steps 2 --warmup 1 --no-cpu-baseline --e2e-T 1024 > gpurun_out/r2b_bench.json 2> gpurun_out/r2b_bench.err; echo "bench rc=$?"
tail -3 gpurun_out/r2b_bench.err
python tools/ref_suite/run_ref_suite.py --mode boundary --out gpurun_out/r2b_refsuite_boundary.json > gpurun_out/r2b_refsuite.log 2>&1; echo "ref suite rc=$?"
tail -3 gpurun_out/r2b_refsuite.log
python tools/ref_suite/run_ref_suite.py --mode full --out gpurun_out/r2b_refsuite_full.json >> gpurun_out/r2b_refsuite.log 2>&1
tail -1 gpurun_out/r2b_refsuite.log
