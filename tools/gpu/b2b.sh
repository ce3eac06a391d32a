mkdir -p gpurun_out
: > gpurun_out/b2b.txt
for d in 64 128 256; do
  timeout 300 python tools/lmme_b2b.py $d 1024 20 >> gpurun_out/b2b.txt 2>&1
  timeout 300 python tools/lmme_prof2.py $d 1024 20 >> gpurun_out/b2b.txt 2>&1
done
