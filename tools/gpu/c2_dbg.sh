mkdir -p gpurun_out
rm -f gpurun_out/c2_dbg.txt
run() { echo "== $*" >> gpurun_out/c2_dbg.txt; env "$@" timeout 200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,lts__t_bytes.sum --clock-control none -k regex:lmme_tc_kernel -s 2 -c 1 python tools/lmme_prof2.py 128 1024 3 2>&1 | grep -E "duration|bytes" >> gpurun_out/c2_dbg.txt; }
run GOOM_TC_FUSE=1
run GOOM_TC_FUSE=0
run GOOM_TC_FUSE=0 GOOM_TC_DEBUG=5
run GOOM_TC_FUSE=0 GOOM_TC_DEBUG=6
run GOOM_TC_FUSE=0 GOOM_TC_DEBUG=1
run GOOM_TC_FUSE=0 GOOM_TC_DEBUG=2
run GOOM_TC_FUSE=0 GOOM_TC_DEBUG=7
run GOOM_TC_FUSE=0 GOOM_TC_DEBUG=4
run GOOM_TC_FUSE=1 GOOM_TC_DEBUG=7
run GOOM_TC_FUSE=1 GOOM_TC_DEBUG=6
