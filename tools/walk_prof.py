"""Kernel breakdown (torch.profiler / CUPTI, no replay) of the config-4 selective chain
(Lorenz-96 d=64, colinearity(0.99, 12, 1e-9)) on a T-leaf prefix."""
import os
import sys
from collections import defaultdict

import torch
from torch.profiler import ProfilerActivity, profile

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import gooms_port as G  # noqa: E402
from oracle import systems_port as S  # noqa: E402
import paper_2510_03426_b200 as g  # noqa: E402

T = int(sys.argv[1]) if len(sys.argv) > 1 else 24000
f, df, x0, dt = S.lorenz96(64)
mats = S.integrate_chain(f, df, x0, dt, burn_in=1000, T=T, seed=0)
al, as_ = G.log_sign(S.spectrum_leaves(mats))
A = g.join(al, as_, torch.complex128)
pol = g.colinearity_policy(0.99, 12, 1e-9)
for _ in range(2):
    V, sites = g._selective_chain_core(A, pol, 256)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    V, sites = g._selective_chain_core(A, pol, 256)
    e.record()
    torch.cuda.synchronize()
wall = s.elapsed_time(e)
groups = defaultdict(lambda: [0, 0.0])
for ev in prof.events():
    if ev.device_type.name != "CUDA":
        continue
    groups[ev.name[:70]][0] += 1
    groups[ev.name[:70]][1] += ev.device_time_total / 1e3
tot = sum(v[1] for v in groups.values())
print(f"T={T}: wall {wall:.2f} ms ({T / wall * 1e3:.0f} mat/s), {len(sites)} resets, kernels {tot:.2f} ms")
for k, (n, t) in sorted(groups.items(), key=lambda kv: -kv[1][1]):
    print(f"   {t:8.2f} ms  n={n:5d}  avg {t / n * 1e3:9.1f} us  {k}")
