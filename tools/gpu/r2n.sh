# PDL A/B on the headline bench + correctness of the tile-scaled path with PDL on
python -m pytest tests/test_gpu_ts.py tests/test_gpu_bench_path.py -q -m gpu -p no:cacheprovider -x 2>&1 | tail -2
for i in 1 2; do
for p in 1 0; do
GOOM_TS_PDL=$p timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-T 1024 > gpurun_out/r2n_bench_pdl${p}_$i.json 2> gpurun_out/r2n_bench_pdl${p}_$i.err
python - <<PY
import json
d=json.load(open("gpurun_out/r2n_bench_pdl${p}_$i.json")); ph=d["roofline"]["phases"]
print("pdl=$p run $i", round(d["value"]), d["clocks"]["sm_mhz"], {k: round(v["frac"],3) for k,v in ph.items()}, round(d["roofline"]["whole_step"]["frac"],3))
PY
done; done
