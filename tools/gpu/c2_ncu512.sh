mkdir -p gpurun_out
timeout 400 ncu --set full --clock-control none --import-source on -k regex:lmme_tc2_kernel -s 1 -c 1 -o gpurun_out/r2_c2_d512 -f python tools/lmme_prof2.py 512 1024 2 > gpurun_out/r2_c2_d512.log 2>&1
ncu -i gpurun_out/r2_c2_d512.ncu-rep --page raw --csv > gpurun_out/r2_c2_d512_raw.csv 2>&1
ncu -i gpurun_out/r2_c2_d512.ncu-rep --page details --csv > gpurun_out/r2_c2_d512_details.csv 2>&1
