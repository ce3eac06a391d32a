mkdir -p gpurun_out
: > gpurun_out/duo_dbg.txt
for dbg in 0 7 8 0; do
  echo "debug $dbg" >> gpurun_out/duo_dbg.txt
  GOOM_TC_DEBUG=$dbg timeout 300 python tools/lmme_prof2.py 64 1024 20 >> gpurun_out/duo_dbg.txt 2>&1
  GOOM_TC_DUO=1 GOOM_TC_DEBUG=$dbg timeout 300 python tools/lmme_prof2.py 64 1024 20 >> gpurun_out/duo_dbg.txt 2>&1
done
for b in 256 512 2048 4096; do
  echo "batch $b" >> gpurun_out/duo_dbg.txt
  timeout 300 python tools/lmme_prof2.py 64 $b 20 >> gpurun_out/duo_dbg.txt 2>&1
done
