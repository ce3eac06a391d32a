mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__inst_issued.avg.pct_of_peak_sustained_active,sm__warps_active.avg.pct_of_peak_sustained_active --clock-control none --csv --log-file gpurun_out/long8_launches.csv python tools/small_d_bench.py --ds 8 --reps 1 --cpu-sample 8 --engines long > gpurun_out/long8_launches.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:long_fold_kernel -s 0 -c 1 -o gpurun_out/long8_r -f python tools/small_d_bench.py --ds 8 --reps 1 --cpu-sample 8 --engines long > gpurun_out/long8_r.log 2>&1
ncu -i gpurun_out/long8_r.ncu-rep --page raw --csv > gpurun_out/long8_r_raw.csv 2>&1
rm -f gpurun_out/long8_r.ncu-rep
