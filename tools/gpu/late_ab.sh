mkdir -p gpurun_out
GOOM_TC_LATE=4 GOOM_TC1_LATE=4 timeout 600 python -m pytest tests/test_gpu_core.py -q -x -k "fused_scales" > gpurun_out/late_pytest.log 2>&1; echo "rc $?" >> gpurun_out/late_pytest.log
GOOM_TC_LATE=8 GOOM_TC1_LATE=8 timeout 600 python -m pytest tests/test_gpu_core.py -q -x -k "fused_scales" >> gpurun_out/late_pytest.log 2>&1; echo "rc $?" >> gpurun_out/late_pytest.log
: > gpurun_out/late_ab.txt
for rep in 1 2; do
for lf in 1 2 4 8 16; do
  echo -n "d256 lf=$lf " >> gpurun_out/late_ab.txt
  GOOM_TC_LATE=$lf timeout 300 python tools/lmme_prof2.py 256 1024 15 >> gpurun_out/late_ab.txt 2>&1
done
for lf in 1 2 4 8; do
  echo -n "d128 lf=$lf " >> gpurun_out/late_ab.txt
  GOOM_TC1_LATE=$lf timeout 300 python tools/lmme_prof2.py 128 1024 15 >> gpurun_out/late_ab.txt 2>&1
done
done
