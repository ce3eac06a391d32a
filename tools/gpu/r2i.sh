# long-chain small-d engine: parity tests + HBM figure
python -m pytest tests/test_gpu_scan_long.py -q -m gpu -p no:cacheprovider -x 2>&1 | tail -15
timeout 600 python tools/small_d_bench.py --engines long > gpurun_out/r2i_small_d.jsonl 2> gpurun_out/r2i_small_d.err; echo "small_d rc=$?"
python - <<'PY'
import json
for l in open("gpurun_out/r2i_small_d.jsonl"):
    r=json.loads(l); print(r["d"], r["engine"][:10], round(r["ms"],3), round(r["achieved_gbs"],1), round(r["frac_hbm"],3), round(r["moved_gbs"],1))
PY
tail -3 gpurun_out/r2i_small_d.err
