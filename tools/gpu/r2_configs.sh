mkdir -p gpurun_out
timeout 900 python tools/config1_chain.py > gpurun_out/r2_config1.json 2> gpurun_out/r2_config1.err
timeout 1200 python tools/config4_lyapunov.py > gpurun_out/r2_config4.json 2> gpurun_out/r2_config4.err
timeout 900 python tools/config5_ssm.py > gpurun_out/r2_config5.json 2> gpurun_out/r2_config5.err
