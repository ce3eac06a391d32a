"""Kernel-level breakdown of one tile-scaled chain_ts window via torch.profiler (CUPTI
activity records, no replay): groups kernels by name + grid and reports time per group."""
import sys
from collections import defaultdict

import torch
from torch.profiler import ProfilerActivity, profile

sys.path.insert(0, ".")
from paper_2510_03426_b200 import ops  # noqa: E402

d = 512
T = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
blocks = [int(x) for x in sys.argv[2].split(",")] if len(sys.argv) > 2 else [128]
dev = torch.device("cuda")
L = ops.ts_random_normal(T, d, 1, 0, dev)
for s in blocks:
    ops.chain_ts(L, s, None, digests=True, carry_out=True)
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        ops.chain_ts(L, s, None, digests=True, carry_out=True)
        b.record()
        torch.cuda.synchronize()
    wall = a.elapsed_time(b)
    groups = defaultdict(lambda: [0, 0.0])
    first, last = None, None
    for e in prof.events():
        if e.device_type.name != "CUDA":
            continue
        key = e.name[:60]
        groups[key][0] += 1
        groups[key][1] += e.device_time_total / 1e3 if hasattr(e, "device_time_total") else 0
    tot = sum(v[1] for v in groups.values())
    print(f"T={T} block={s}: event wall {wall:.2f} ms, kernel sum {tot:.2f} ms, gaps {wall - tot:.2f} ms")
    for k, (n, t) in sorted(groups.items(), key=lambda kv: -kv[1][1]):
        print(f"   {t:8.2f} ms  n={n:5d}  avg {t / n * 1e3:8.1f} us  {k}")
