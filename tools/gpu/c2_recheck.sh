mkdir -p gpurun_out
timeout 600 python tools/config2_lmme_sweep.py > gpurun_out/r2y_config2_sweep.json 2> gpurun_out/r2y_config2_sweep.err
bash tools/gpu/c2_batch_scaling.sh
cp gpurun_out/c2_batch_scaling.txt gpurun_out/r2y_c2_batch_scaling.txt
: > gpurun_out/r2y_late_ab.txt
for lf in 1 2 4 8; do
  echo -n "d256 lf=$lf " >> gpurun_out/r2y_late_ab.txt
  GOOM_TC_LATE=$lf timeout 300 python tools/lmme_prof2.py 256 1024 15 >> gpurun_out/r2y_late_ab.txt 2>&1
  echo -n "d128 lf=$lf " >> gpurun_out/r2y_late_ab.txt
  GOOM_TC1_LATE=$lf timeout 300 python tools/lmme_prof2.py 128 1024 15 >> gpurun_out/r2y_late_ab.txt 2>&1
done
