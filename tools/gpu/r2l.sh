python -m pytest tests/test_gpu_scan_long.py -q -m gpu -p no:cacheprovider -x 2>&1 | tail -3
timeout 600 python tools/small_d_bench.py --engines long > gpurun_out/r2l_small_d.jsonl 2> gpurun_out/r2l_small_d.err; echo "small_d rc=$?"
python - <<'PY'
import json
for l in open("gpurun_out/r2l_small_d.jsonl"):
    r=json.loads(l); print(r["d"], r["engine"][:10], round(r["ms"],3), round(r["achieved_gbs"],1), round(r["frac_hbm"],3), round(r["moved_gbs"],1))
PY
for d in 8 32; do
ncu --set full --import-source on --clock-control none -k regex:long_fold --launch-skip 0 --launch-count 1 -o gpurun_out/r2l_long_R0_d$d python tools/long_prof.py $d > /dev/null 2>&1
done
