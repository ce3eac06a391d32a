"""Profiling aid: kernel-by-kernel CUDA time of one d = 64 long-chain scan (T = 2^20 by
default) through torch.profiler (CUPTI records, no replay)."""
import sys

import torch
from torch.profiler import ProfilerActivity, profile

sys.path.insert(0, ".")
import paper_2510_03426_b200 as g  # noqa: E402
from paper_2510_03426_b200 import harness  # noqa: E402

T = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 20
d = int(sys.argv[2]) if len(sys.argv) > 2 else 64
g._lib.load()
A = harness.random_chain(T, d, seed=d)
out = torch.ops.goom.scan_chain_long(A, None)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    out = torch.ops.goom.scan_chain_long(A, None)
    torch.cuda.synchronize()
tot = 0.0
for e in prof.events():
    if e.device_type.name == "CUDA":
        print(f"{e.device_time_total / 1e3:9.3f} ms  {e.name[:90]}")
        tot += e.device_time_total / 1e3
print(f"total {tot:.3f} ms")
