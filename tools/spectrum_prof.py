"""Kernel breakdown (torch.profiler / CUPTI) of config 4's full spectrum_parallel
(Lorenz-96 d = 64, T leaves; stages (a) selective scan, (b) unit-column QR bases,
(c) J_t Q_{t-1}, (d) batched QR |diag R|)."""
import os
import sys
from collections import defaultdict

import torch
from torch.profiler import ProfilerActivity, profile

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import systems_port as S  # noqa: E402
import paper_2510_03426_b200 as g  # noqa: E402

T = int(sys.argv[1]) if len(sys.argv) > 1 else 24000
f, df, x0, dt = S.lorenz96(64)
mats = S.integrate_chain(f, df, x0, dt, burn_in=1000, T=T, seed=0)
chain = g.JacobianChain(dt=dt, mats=mats)
g.spectrum_parallel(g.JacobianChain(dt=dt, mats=mats[:256]))
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    spec = g.spectrum_parallel(chain)
    torch.cuda.synchronize()
groups = defaultdict(lambda: [0, 0.0])
for e in prof.events():
    if e.device_type.name == "CUDA":
        groups[e.name[:70]][0] += 1
        groups[e.name[:70]][1] += e.device_time_total / 1e3
print(f"T={T}: spectrum wall {spec.wall_seconds * 1e3:.1f} ms, kernels {sum(v[1] for v in groups.values()):.1f} ms")
for k, (n, t) in sorted(groups.items(), key=lambda kv: -kv[1][1])[:10]:
    print(f"   {t:8.2f} ms  n={n:5d}  avg {t / n * 1e3:9.1f} us  {k}")
