"""Layout diagnostic for lmme_ts: products with identity / permutation operands."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2510_03426_b200 as g  # noqa: E402
from paper_2510_03426_b200 import ops  # noqa: E402

d = 256
rng = np.random.default_rng(0)
R = rng.standard_normal((1, d, d)).astype(np.float32)
I = np.eye(d, dtype=np.float32)[None]


def goom(x):
    return g.join(np.log(np.abs(x)), np.where(x < 0, -1.0, 1.0))


def real(z):
    z = z.cpu()
    return np.exp(z.real.double().numpy()) * np.where(np.cos(z.imag.double().numpy()) < 0, -1, 1)


for name, A, B in (("R*I", R, I), ("I*R", I, R), ("R*R", R, R)):
    C = real(ops.lmme_ts(ops.ts_from_goom(goom(A)), ops.ts_from_goom(goom(B)), 0))[0]
    W = (A[0].astype(np.float64) @ B[0].astype(np.float64))
    err = np.abs(C - W)
    bad = np.argwhere(err > 1e-3 * np.abs(W).max())
    print(f"{name}: max err {err.max():.3e}, bad {len(bad)} / {d*d}", flush=True)
    if len(bad):
        print("  first bad (i,j):", bad[:8].tolist(), flush=True)
        # for I*R: which column of R landed at (i, j)?
        if name == "I*R":
            for (i, j) in bad[:6]:
                cand = np.argwhere(np.abs(R[0] - C[i, j]) < 1e-5)
                print(f"   C[{i},{j}]={C[i,j]:.4f} want {W[i,j]:.4f}; equals R at {cand[:3].tolist()}")
        if name == "R*I":
            for (i, j) in bad[:6]:
                cand = np.argwhere(np.abs(R[0] - C[i, j]) < 1e-5)
                print(f"   C[{i},{j}]={C[i,j]:.4f} want {W[i,j]:.4f}; equals R at {cand[:3].tolist()}")
