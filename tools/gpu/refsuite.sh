mkdir -p gpurun_out
python tools/ref_suite/run_ref_suite.py --mode boundary --out gpurun_out/r2x_refsuite_boundary.json > gpurun_out/r2x_refsuite.log 2>&1; echo "boundary rc=$?" >> gpurun_out/r2x_refsuite.log
python tools/ref_suite/run_ref_suite.py --mode full --out gpurun_out/r2x_refsuite_full.json >> gpurun_out/r2x_refsuite.log 2>&1; echo "full rc=$?" >> gpurun_out/r2x_refsuite.log
