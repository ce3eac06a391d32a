mkdir -p gpurun_out
rm -f gpurun_out/c2_ab.txt
timeout 600 python -m pytest tests/test_gpu_core.py -q -x -k "fused_scales or lmme" > gpurun_out/c2_pytest.log 2>&1; echo "rc $?" >> gpurun_out/c2_pytest.log
for v in "GOOM_TC_DEBUG=0" "GOOM_TC_DEBUG=32" "GOOM_TC_DEBUG=7" "GOOM_TC_DEBUG=39" "GOOM_TC_PREFETCH=1" "GOOM_TC_FUSE=0"; do env $v timeout 120 python tools/lmme_prof2.py 128 1024 15 >> gpurun_out/c2_ab.txt 2>&1; echo "  $v" >> gpurun_out/c2_ab.txt; done
timeout 200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum --clock-control none -k regex:lmme_tc_kernel -s 2 -c 1 python tools/lmme_prof2.py 128 1024 3 2>&1 | grep -E "duration|bytes" >> gpurun_out/c2_ab.txt
