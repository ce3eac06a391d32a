#!/bin/bash
# Time the TC kernel with stages disabled (GOOM_TC_DEBUG) to find the bottleneck.
for dbg in ${DBGS:-0 1 2 3 4}; do
  echo "GOOM_TC_DEBUG=$dbg"
  GOOM_TC_DEBUG=$dbg timeout 120 python - <<'PY'
import sys, torch
sys.path.insert(0, ".")
import paper_2510_03426_b200 as g
for d, batch in ((512, 512), (1024, 128)):
    A = torch.complex(torch.randn(batch, d, d, device="cuda"), torch.zeros(batch, d, d, device="cuda"))
    B = torch.complex(torch.randn(batch, d, d, device="cuda"), torch.zeros(batch, d, d, device="cuda"))
    for _ in range(2): torch.ops.goom.lmme(A, B)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(5): torch.ops.goom.lmme(A, B)
    e.record(); torch.cuda.synchronize()
    ms = s.elapsed_time(e) / 5
    print(f"  d={d} batch={batch}: {ms:.3f} ms  {2*d**3*batch/ms/1e9:.1f} TF/s", flush=True)
PY
done
