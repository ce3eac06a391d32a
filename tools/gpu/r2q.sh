python tools/lmme_prof2.py 256; GOOM_TC_DEBUG=64 python tools/lmme_prof2.py 256; GOOM_TC2_FUSE=0 python tools/lmme_prof2.py 256
ncu --set full --import-source on --clock-control none -k regex:lmme_tc2 --launch-skip 2 --launch-count 1 -o gpurun_out/r2q_fused python tools/lmme_prof2.py 256 > /dev/null 2>&1
GOOM_TC2_FUSE=0 ncu --set full --import-source on --clock-control none -k regex:lmme_tc2 --launch-skip 2 --launch-count 1 -o gpurun_out/r2q_prepass python tools/lmme_prof2.py 256 > /dev/null 2>&1
