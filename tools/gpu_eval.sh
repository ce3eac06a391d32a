#!/bin/bash
# One gpurun call: GPU tests, the default bench, the ncu launch list of a short bench,
# and one ncu --set full capture of the phase-3 LMME kernel. Outputs under gpurun_out/.
set -x
mkdir -p gpurun_out
TAG=${TAG:-eval}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/${TAG}_smi.txt 2>&1
if [ "${SKIP_TESTS:-0}" != 1 ]; then
  timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/${TAG}_pytest.log 2>&1
  echo "pytest exit $?" >> gpurun_out/${TAG}_pytest.log
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1
fi
timeout 900 python bench.py ${BENCH_ARGS} > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err
if [ "${SKIP_NCU:-0}" != 1 ]; then
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/${TAG}_launches.csv python bench.py --T 16384 --steps 1 --warmup 1 \
    --no-cpu-baseline --e2e-T 512 > gpurun_out/${TAG}_ncu_bench.log 2>&1
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:lmme_tc -s 2 -c 1 \
    -o gpurun_out/${TAG}_lmme_full -f python tools/ncu_one.py 512 512 > gpurun_out/${TAG}_ncu_full.log 2>&1
fi
ls -la gpurun_out
