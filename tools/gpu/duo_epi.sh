mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_core.py -q -x -k "fused_scales or lmme" > gpurun_out/duo_epi_pytest.log 2>&1; echo "rc $?" >> gpurun_out/duo_epi_pytest.log
: > gpurun_out/duo_epi.txt
for b in 1024 1024 256 2048 4096; do
  timeout 300 python tools/lmme_prof2.py 64 $b 20 >> gpurun_out/duo_epi.txt 2>&1
done
GOOM_TC_DEBUG=7 timeout 300 python tools/lmme_prof2.py 64 1024 20 >> gpurun_out/duo_epi.txt 2>&1
