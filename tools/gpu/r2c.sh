python tools/reanchor_diag.py 65536 16384 128 32768 > gpurun_out/r2c_diag1.json 2>&1
python tools/reanchor_diag.py 65536 16384 64 32768 > gpurun_out/r2c_diag2.json 2>&1
python tools/reanchor_diag.py 65536 16384 128 30000 > gpurun_out/r2c_diag3.json 2>&1
python -m pytest tests/test_gpu_harness.py -x -q -m gpu -p no:cacheprovider -k sharded > gpurun_out/r2c_pytest.log 2>&1; tail -3 gpurun_out/r2c_pytest.log
