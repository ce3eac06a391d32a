mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_core.py -q -x -k "fused_scales" > gpurun_out/c2_pytest.log 2>&1; echo "rc $?" >> gpurun_out/c2_pytest.log
timeout 300 ncu --set full --clock-control none --import-source on -k regex:lmme_tc_kernel -s 1 -c 1 -o gpurun_out/c2_tc128_fused -f python tools/lmme_prof2.py 128 1024 2 > gpurun_out/c2_ncu.log 2>&1
GOOM_TC_FUSE=0 timeout 300 ncu --set full --clock-control none --import-source on -k regex:lmme_tc_kernel -s 1 -c 1 -o gpurun_out/c2_tc128_prepass -f python tools/lmme_prof2.py 128 1024 2 >> gpurun_out/c2_ncu.log 2>&1
