mkdir -p gpurun_out
timeout 600 python tools/config2_lmme_sweep.py > gpurun_out/r2_config2_sweep.json 2> gpurun_out/r2_config2_sweep.err
timeout 900 python tools/small_d_bench.py --ds 8,16,32,64 --reps 3 --cpu-sample 256 > gpurun_out/r2_small_d.jsonl 2> gpurun_out/r2_small_d.err
for d in 64 128; do
  timeout 300 ncu --set full --clock-control none --import-source on -k regex:lmme_tc_kernel -s 1 -c 1 -o gpurun_out/r2_c2_d${d} -f python tools/lmme_prof2.py $d 1024 2 > gpurun_out/r2_c2_d${d}.log 2>&1
done
timeout 300 ncu --set full --clock-control none --import-source on -k regex:lmme_tc2_kernel -s 1 -c 1 -o gpurun_out/r2_c2_d256 -f python tools/lmme_prof2.py 256 1024 2 > gpurun_out/r2_c2_d256.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:long_fold_tc -s 0 -c 1 -o gpurun_out/r2_l64 -f python tools/ncu_long_tc.py 64 > gpurun_out/r2_l64.log 2>&1
