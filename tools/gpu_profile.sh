#!/bin/bash
# ncu evidence for the bench's dominant kernel and the launch list of a short bench.
TAG=${TAG:-prof}
mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/${TAG}_launches.csv python bench.py --T 16384 --steps 1 --warmup 1 \
  --no-cpu-baseline --e2e-T 256 > gpurun_out/${TAG}_ncu_bench.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:lmme_ts -s 2 -c 1 \
  -o gpurun_out/${TAG}_phase3 -f python tools/ncu_ts.py 2 8192 > gpurun_out/${TAG}_phase3.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:lmme_ts -s 2 -c 1 \
  -o gpurun_out/${TAG}_phase1 -f python tools/ncu_ts.py 1 128 > gpurun_out/${TAG}_phase1.log 2>&1
