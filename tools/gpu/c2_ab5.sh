mkdir -p gpurun_out
rm -f gpurun_out/c2_ab5.txt
timeout 600 python -m pytest tests/test_gpu_core.py -q -x -k "fused_scales or lmme" > gpurun_out/c2_pytest.log 2>&1; echo "rc $?" >> gpurun_out/c2_pytest.log
for v in "GOOM_TC_FUSE=1" "GOOM_TC_FUSE=0"; do
env $v timeout 120 python tools/lmme_prof2.py 64 1024 9 >> gpurun_out/c2_ab5.txt 2>&1; echo "  $v" >> gpurun_out/c2_ab5.txt
done
timeout 200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:lmme_tc -s 1 -c 1 python tools/lmme_prof2.py 64 1024 2 2>&1 | grep -E "duration|bytes" >> gpurun_out/c2_ab5.txt
