mkdir -p gpurun_out
: > gpurun_out/c2_batch_scaling.txt
for cfg in "128 512" "128 1024" "128 2048" "128 4096" "256 256" "256 512" "256 1024" "256 2048" "512 256" "512 512" "512 1024" "512 2048" "1024 256" "1024 512" "1024 1024"; do
  set -- $cfg
  timeout 300 python tools/lmme_prof2.py $1 $2 7 >> gpurun_out/c2_batch_scaling.txt 2>&1
done
