"""Time the batched complex64 LMME (batch 1024) at d in argv under the current
GOOM_TC_DEBUG profiling mode (0 = normal, 1 = no transform, 2 = no MMA, 3 = no loads,
6 = B as one box): median of 20 event-timed launches after an L2 flush each."""
import json
import os
import sys

import torch

sys.path.insert(0, ".")
import paper_2510_03426_b200 as g  # noqa: E402,F401

dev = torch.device("cuda")
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
out = {"mode": os.environ.get("GOOM_TC_DEBUG", "0")}
for d in map(int, sys.argv[1:] or ["128", "256"]):
    A = torch.ops.goom.from_real(torch.randn(1024, d, d, device=dev), float("-inf"), False)
    B = torch.ops.goom.from_real(torch.randn(1024, d, d, device=dev), float("-inf"), False)
    ts = []
    for i in range(23):
        flush.add_(1)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        torch.ops.goom.lmme(A, B)
        b.record()
        torch.cuda.synchronize()
        if i >= 3:
            ts.append(a.elapsed_time(b) * 1e3)
    ts.sort()
    out[d] = round(ts[len(ts) // 2], 1)
    del A, B
print(json.dumps(out))
