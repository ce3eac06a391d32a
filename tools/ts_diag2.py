import os, sys
import numpy as np
import torch
sys.path.insert(0, ".")
import paper_2510_03426_b200 as g
from paper_2510_03426_b200 import ops
d = 256
rng = np.random.default_rng(0)
R = rng.standard_normal((1, d, d)).astype(np.float32)
def goom(x):
    return g.join(np.log(np.abs(x)), np.where(x < 0, -1.0, 1.0))
ta = ops.ts_from_goom(goom(R)); tb = ops.ts_from_goom(goom(R))
print("dbg", os.environ.get("GOOM_TS_DEBUG"), "q sample", ta.q[0, :4].tolist(), "G", ta.G[0].tolist(), "U max", ta.U.abs().max().item())
out = ops.lmme_ts(ta, tb, 1)
print(" out U[0,:4,:4]", out.U[0, :4, :4].tolist())
print(" out q[0,:4]", out.q[0, :4].tolist(), "nonzero U", (out.U != 0).sum().item())
C = ops.lmme_ts(ta, tb, 0)
print(" goom C[0,0,:4]", C[0, 0, :4].tolist())
W = R[0].astype(np.float64) @ R[0].astype(np.float64)
print(" want", W[0, :4].tolist())
