# checkpoint: full -m gpu suite + reference suite (both modes)
timeout 1500 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/r2u_pytest.log 2>&1; echo "pytest rc=$?"
tail -4 gpurun_out/r2u_pytest.log
timeout 900 python tools/ref_suite/run_ref_suite.py --mode boundary --out gpurun_out/r2u_refsuite_boundary.json > gpurun_out/r2u_refsuite.log 2>&1
timeout 900 python tools/ref_suite/run_ref_suite.py --mode full --out gpurun_out/r2u_refsuite_full.json >> gpurun_out/r2u_refsuite.log 2>&1
grep '^{' gpurun_out/r2u_refsuite.log | cut -c1-300
