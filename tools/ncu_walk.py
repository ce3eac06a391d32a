"""Config-4 selective walk (Lorenz-96 d=64) on a T-leaf prefix, for ncu -k selective_walk."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import gooms_port as G  # noqa: E402
from oracle import systems_port as S  # noqa: E402
import paper_2510_03426_b200 as g  # noqa: E402

T = int(sys.argv[1]) if len(sys.argv) > 1 else 6000
f, df, x0, dt = S.lorenz96(64)
mats = S.integrate_chain(f, df, x0, dt, burn_in=1000, T=T, seed=0)
al, as_ = G.log_sign(S.spectrum_leaves(mats))
A = g.join(al, as_, torch.complex128)
pol = g.colinearity_policy(0.99, 12, 1e-9)
for _ in range(2):
    V, sites = g._selective_chain_core(A, pol, 256)
torch.cuda.synchronize()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record()
V, sites = g._selective_chain_core(A, pol, 256)
e.record()
torch.cuda.synchronize()
print(f"T={T}: {s.elapsed_time(e):.1f} ms, {len(sites)} resets, {T / s.elapsed_time(e) * 1e3:.0f} mat/s")
