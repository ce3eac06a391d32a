for i in 1 2; do
timeout 600 python bench.py --T 65536 --window 16384 --steps 3 --warmup 1 --no-cpu-baseline --e2e-T 1024 > gpurun_out/r2e_bench_a$i.json 2> gpurun_out/r2e_bench_a$i.err
timeout 600 python bench.py --T 65536 --window 16384 --steps 3 --warmup 1 --no-cpu-baseline --e2e-T 1024 --no-reanchor > gpurun_out/r2e_bench_b$i.json 2> gpurun_out/r2e_bench_b$i.err
done
python - <<'PY'
import json
for f in ("a1","b1","a2","b2"):
    d=json.load(open(f"gpurun_out/r2e_bench_{f}.json")); print(f, d["value"], d["ms_per_step"], d["clocks"]["sm_mhz"])
PY
python -m pytest tests/test_gpu_scan.py tests/test_gpu_bench_path.py -q -m gpu -p no:cacheprovider -k "cta or snapshots" 2>&1 | tail -3
