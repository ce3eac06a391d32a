mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests/test_gpu_scan_long.py -q -x > gpurun_out/upper_pytest.log 2>&1; echo "rc $?" >> gpurun_out/upper_pytest.log
: > gpurun_out/upper_ab.txt
for cfg in "16 32" "4 4" "8 8" "4 8" "2 4" "16 32" "4 4"; do
  set -- $cfg
  GOOM_LONG_S=$1 GOOM_LONG_TOP=$2 timeout 300 python tools/small_d_bench.py --ds 8,16,32,64 --reps 5 --cpu-sample 8 --engines long > gpurun_out/upper_ab_$1_$2.jsonl 2>>gpurun_out/upper_ab.err
  python -c "import sys,json; print('s=$1 top=$2', ' '.join('d%d %.4f' % (json.loads(l)['d'], json.loads(l)['ms']) for l in open('gpurun_out/upper_ab_$1_$2.jsonl')))" >> gpurun_out/upper_ab.txt
done
