"""Kernel breakdown (torch.profiler / CUPTI) of one batched complex64 LMME call per d."""
import sys
from collections import defaultdict

import torch
from torch.profiler import ProfilerActivity, profile

sys.path.insert(0, ".")
import paper_2510_03426_b200 as g  # noqa: E402,F401

dev = torch.device("cuda")
for d in [int(x) for x in (sys.argv[1].split(",") if len(sys.argv) > 1 else ["64", "256", "512"])]:
    batch = 1024
    A = torch.ops.goom.from_real(torch.randn(batch, d, d, device=dev), float("-inf"), False)
    B = torch.ops.goom.from_real(torch.randn(batch, d, d, device=dev), float("-inf"), False)
    for _ in range(3):
        torch.ops.goom.lmme(A, B)
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        torch.ops.goom.lmme(A, B)
        torch.cuda.synchronize()
    groups = defaultdict(lambda: [0, 0.0])
    for e in prof.events():
        if e.device_type.name == "CUDA":
            groups[e.name[:80]][0] += 1
            groups[e.name[:80]][1] += e.device_time_total
    print(f"d={d}:")
    for k, (n, t) in sorted(groups.items(), key=lambda kv: -kv[1][1]):
        print(f"   {t:9.1f} us  n={n}  {k}")
