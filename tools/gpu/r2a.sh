# round-2 GPU check: full -m gpu suite + a short bench (scratch script for gpurun)
python -m pytest tests -x -q -m gpu -p no:cacheprovider > gpurun_out/r2a_pytest.log 2>&1; echo "pytest rc=$?"
tail -5 gpurun_out/r2a_pytest.log
timeout 600 python bench.py --T 65536 --window 16384 --steps 2 --warmup 1 --no-cpu-baseline --e2e-T 1024 > gpurun_out/r2a_bench.json 2> gpurun_out/r2a_bench.err; echo "bench rc=$?"
tail -3 gpurun_out/r2a_bench.err
