python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/r2f_pytest.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/r2f_pytest.log
python tools/ref_suite/run_ref_suite.py --mode boundary --out gpurun_out/r2f_refsuite_boundary.json > gpurun_out/r2f_refsuite.log 2>&1
python tools/ref_suite/run_ref_suite.py --mode full --out gpurun_out/r2f_refsuite_full.json >> gpurun_out/r2f_refsuite.log 2>&1
grep '^{' gpurun_out/r2f_refsuite.log | cut -c1-200
