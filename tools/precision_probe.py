"""Median / max error of each LMME backend vs the float64 oracle (numpy)."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2510_03426_b200 as g  # noqa: E402
from oracle import gooms_port as G  # noqa: E402

rng = np.random.default_rng(5)
for (n, k, m) in ((256, 1024, 256), (512, 512, 512), (128, 4096, 128)):
    a = rng.standard_normal((n, k)).astype(np.float32)
    b = rng.standard_normal((k, m)).astype(np.float32)
    al, as_ = G.log_sign(a)
    bl, bs = G.log_sign(b)
    want = a.astype(np.float64) @ b.astype(np.float64)
    kappa = np.abs(want) / (np.abs(a).astype(np.float64) @ np.abs(b).astype(np.float64))
    for be, name in ((1, "simt"), (2, "tc")):
        g._lib.set_backend(be)
        out = torch.ops.goom.lmme(g.join(al, as_), g.join(bl, bs))
        l = out.real.double().cpu().numpy()
        s = np.where(np.cos(out.imag.double().cpu().numpy()) < 0, -1, 1)
        got = s * np.exp(l)
        rel = np.abs(got - want) / (np.abs(a).astype(np.float64) @ np.abs(b).astype(np.float64))
        fro = np.linalg.norm(got - want) / np.linalg.norm(want)
        print(f"{name} n={n} k={k} m={m}: err/sum|ab| median={np.median(rel):.2e} max={rel.max():.2e} "
              f"frob={fro:.2e} flips(kappa>1e-4)={int(np.sum((np.sign(got)!=np.sign(want)) & (kappa>1e-4)))}", flush=True)
