mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
GOOM_TC_DUO=1 timeout 600 python -m pytest tests/test_gpu_core.py -q -x -k "fused_scales or lmme" > gpurun_out/duo_pytest.log 2>&1; echo "rc $?" >> gpurun_out/duo_pytest.log
: > gpurun_out/duo_ab.txt
for mode in 0 1 0 1; do
  echo "mode $mode" >> gpurun_out/duo_ab.txt
  GOOM_TC_DUO=$mode timeout 300 python tools/lmme_prof2.py 64 1024 20 >> gpurun_out/duo_ab.txt 2>&1
done
GOOM_TC_DUO=1 timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/duo_launches.csv python tools/lmme_prof2.py 64 1024 2 > /dev/null 2>&1
