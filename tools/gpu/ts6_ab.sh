mkdir -p gpurun_out
GOOM_TS_STAGES=2 timeout 900 python -m pytest tests/test_gpu_ts.py tests/test_gpu_bench_path.py -q -x > gpurun_out/ts6_test.log 2>&1; echo "rc $?" >> gpurun_out/ts6_test.log
: > gpurun_out/ts6_ab.txt
for i in 1 2; do
for st in 0 2; do
  GOOM_TS_STAGES=$st timeout 600 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-reanchor --e2e-T 512 --e2e-goom-T 512 > gpurun_out/ts6_$st.json 2> gpurun_out/ts6_$st.err
  python -c "
import json
d=json.loads(open('gpurun_out/ts6_$st.json').read().strip().splitlines()[-1])
ph=d['roofline']['phases']
print('stages $st', round(d['value']), d['clocks']['sm_mhz'], {k:(round(v['share_of_step'],3), round(v['frac'],3)) for k,v in ph.items()})" >> gpurun_out/ts6_ab.txt 2>&1
done
done
