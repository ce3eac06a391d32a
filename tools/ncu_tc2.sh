#!/bin/bash
# ncu --set full of the pair kernel under several GOOM_TC_DEBUG modes (d=512, batch 256)
for dbg in ${DBGS:-0 7 9}; do
  GOOM_TC2=1 GOOM_TC_DEBUG=$dbg timeout 300 ncu --set full --clock-control none --import-source on \
    -k regex:lmme_tc2 -s 1 -c 1 -o gpurun_out/tc2_dbg${dbg} -f python tools/ncu_one.py 512 256 \
    > gpurun_out/tc2_dbg${dbg}.log 2>&1
done
