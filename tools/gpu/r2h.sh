# SSM contractive test, small-d long-chain HBM figure, config 4 full-length sites
python -m pytest tests/test_gpu_ssm.py -q -m gpu -p no:cacheprovider -k contractive 2>&1 | tail -3
timeout 900 python tools/small_d_bench.py > gpurun_out/r2h_small_d.jsonl 2> gpurun_out/r2h_small_d.err; echo "small_d rc=$?"; cut -c1-400 gpurun_out/r2h_small_d.jsonl; tail -2 gpurun_out/r2h_small_d.err
timeout 1500 python tools/config4_lyapunov.py > gpurun_out/r2h_config4.json 2> gpurun_out/r2h_config4.err; echo "config4 rc=$?"; cat gpurun_out/r2h_config4.json; tail -2 gpurun_out/r2h_config4.err
