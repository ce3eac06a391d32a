"""Kernel breakdown (torch.profiler / CUPTI) of config 5's head-batched SSM forward and
backward (16 heads x 32 sequences x T = 4096, d = 64)."""
import sys
from collections import defaultdict

import numpy as np
import torch
from torch.profiler import ProfilerActivity, profile

sys.path.insert(0, ".")
from paper_2510_03426_b200 import ssm  # noqa: E402

rng = np.random.default_rng(5)
H, S, T, d = 16, 32, 4096, 64
dev = torch.device("cuda")
A = rng.standard_normal((H, d, d))
for h in range(H):
    A[h] *= 1.2 / np.max(np.abs(np.linalg.eigvals(A[h])))
B, C, D = (rng.standard_normal((H, r, d)) for r in (d, 2 * d, 2 * d))
A, B, C, D = (torch.as_tensor(x, device=dev) for x in (A, B, C, D))
x0 = torch.randn(H, S, d, dtype=torch.float64, device=dev)
u = torch.randn(H, S, T, d, dtype=torch.float64, device=dev)
gy = torch.randn(H, S, T, 2 * d, dtype=torch.float64, device=dev)
for _ in range(2):
    sl, ss, c, y = ssm.ssm_forward_heads(A, B, C, D, x0, u)
    ssm.ssm_backward_heads(A, B, C, D, x0, u, sl, ss, c, gy)
torch.cuda.synchronize()
for name, fn in (("forward", lambda: ssm.ssm_forward_heads(A, B, C, D, x0, u)),
                 ("backward", lambda: ssm.ssm_backward_heads(A, B, C, D, x0, u, sl, ss, c, gy))):
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
    groups = defaultdict(lambda: [0, 0.0])
    for e in prof.events():
        if e.device_type.name == "CUDA":
            groups[e.name[:70]][0] += 1
            groups[e.name[:70]][1] += e.device_time_total / 1e3
    tot = sum(v[1] for v in groups.values())
    print(f"{name}: wall {a.elapsed_time(b):.2f} ms, kernels {tot:.2f} ms")
    for k, (n, t) in sorted(groups.items(), key=lambda kv: -kv[1][1])[:12]:
        print(f"   {t:8.2f} ms  n={n:5d}  avg {t / n * 1e3:8.1f} us  {k}")
    big = sorted(((e.device_time_total, e.name[:40]) for e in prof.events()
                  if e.device_type.name == "CUDA" and e.device_time_total > 300), reverse=True)
    print("   launches > 300 us:", ", ".join(f"{t / 1e3:.2f} ms {n}" for t, n in big[:14]))
