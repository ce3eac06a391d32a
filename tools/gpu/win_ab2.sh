mkdir -p gpurun_out
: > gpurun_out/win_ab2.txt
for cfg in "32768 128" "49152 128" "40960 128" "32768 128" "49152 128"; do
  set -- $cfg
  timeout 600 python bench.py --steps 2 --warmup 3 --window $1 --block $2 --no-cpu-baseline --no-reanchor --e2e-T 512 --e2e-goom-T 512 > gpurun_out/win2_$1_$2.json 2> gpurun_out/win2_$1_$2.err
  python -c "
import json
d=json.loads(open('gpurun_out/win2_$1_$2.json').read().strip().splitlines()[-1])
ph=d['roofline']['phases']
print('window $1 block $2', round(d['value']), d['clocks']['sm_mhz'], {k:(round(v['share_of_step'],3), round(v['frac'],3)) for k,v in ph.items()})" >> gpurun_out/win_ab2.txt 2>&1 || tail -2 gpurun_out/win2_$1_$2.err >> gpurun_out/win_ab2.txt
done
