# round-2 re-entry check: full -m gpu suite, smoke, default bench (scratch script for gpurun)
python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/r2g_pytest.log 2>&1; echo "pytest rc=$?"
tail -5 gpurun_out/r2g_pytest.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2g_smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/r2g_smoke.log
timeout 900 python bench.py > gpurun_out/r2g_bench.json 2> gpurun_out/r2g_bench.err; echo "bench rc=$?"
tail -3 gpurun_out/r2g_bench.err; cut -c1-600 gpurun_out/r2g_bench.json
