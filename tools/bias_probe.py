"""Signed relative error of single tile-scaled LMMEs vs float64 (bias probe). GOOM_TS_DEBUG
bits: 16 small plane rounded to TF32 (RN), 32 big*big first, 64 plain TF32."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2510_03426_b200 as g  # noqa: E402
from paper_2510_03426_b200 import ops  # noqa: E402

rng = np.random.default_rng(1)
for d in (256, 512):
    A = rng.standard_normal((8, d, d)).astype(np.float32)
    B = rng.standard_normal((8, d, d)).astype(np.float32)
    C = A.astype(np.float64) @ B.astype(np.float64)
    tA = ops.ts_from_goom(g.join(*[torch.tensor(x) for x in (np.log(np.abs(A)), np.sign(A))]))
    tB = ops.ts_from_goom(g.join(*[torch.tensor(x) for x in (np.log(np.abs(B)), np.sign(B))]))
    out = ops.lmme_ts(tA, tB, 0).cpu()
    got = np.exp(out.real.double().numpy()) * np.where(np.cos(out.imag.double().numpy()) < 0, -1, 1)
    rms = np.sqrt((C ** 2).mean())
    m = np.abs(C) > 0.5 * rms
    rel = (np.abs(got) - np.abs(C))[m] / np.abs(C)[m]
    C32 = (A @ B).astype(np.float64)
    rel32 = (np.abs(C32) - np.abs(C))[m] / np.abs(C)[m]
    print(f"dbg={os.environ.get('GOOM_TS_DEBUG','0')} d={d}: gpu mean {rel.mean():+.3e} std {rel.std():.3e} | "
          f"numpy f32 mean {rel32.mean():+.3e} std {rel32.std():.3e}", flush=True)
