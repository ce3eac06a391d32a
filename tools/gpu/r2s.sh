ncu --set full --import-source on --clock-control none -k regex:lmme_tc_kernel --launch-skip 2 --launch-count 1 -o gpurun_out/r2s_tc128 python tools/lmme_prof2.py 128 > /dev/null 2>&1
