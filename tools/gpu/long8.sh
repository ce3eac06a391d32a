mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_scan_long.py -q -x > gpurun_out/long8_pytest.log 2>&1; echo "rc $?" >> gpurun_out/long8_pytest.log
timeout 600 python tools/small_d_bench.py --ds 8,16 --engines long --reps 3 --cpu-sample 64 > gpurun_out/long8_bench.jsonl 2> gpurun_out/long8_bench.err
GOOM_LONG_FAST=0 timeout 600 python tools/small_d_bench.py --ds 8 --engines long --reps 3 --cpu-sample 64 >> gpurun_out/long8_bench.jsonl 2>> gpurun_out/long8_bench.err
