mkdir -p gpurun_out
rm -f gpurun_out/c2_ab4.txt
timeout 600 python -m pytest tests/test_gpu_core.py -q -x -k "fused_scales" > gpurun_out/c2_pytest.log 2>&1; echo "rc $?" >> gpurun_out/c2_pytest.log
GOOM_TC_DEBUG=64 timeout 600 python -m pytest tests/test_gpu_core.py -q -x -k "fused_scales" >> gpurun_out/c2_pytest.log 2>&1; echo "rc $?" >> gpurun_out/c2_pytest.log
for d in 256; do for v in 0 64; do
GOOM_TC_DEBUG=$v timeout 120 python tools/lmme_prof2.py $d 1024 9 >> gpurun_out/c2_ab4.txt 2>&1; echo "  dbg $v" >> gpurun_out/c2_ab4.txt
done; done
