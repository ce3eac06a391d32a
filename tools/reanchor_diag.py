"""Diagnose re-anchored sign flips on the bench path (config 3 harness, d = 512):
where the GPU's P_{t0+W} disagrees in sign with the float64 oracle recomputed from the GPU's
own P_{t0}, print the flipped entries' structure (rows / columns / blocks), their
cancellation ratio, magnitude relative to the row and column maxima, and the float64
oracle's value next to the GPU's."""
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2510_03426_b200 as goom  # noqa: E402
from paper_2510_03426_b200 import harness, ops  # noqa: E402
from oracle import gooms_port as G  # noqa: E402
from oracle import reanchor as R  # noqa: E402

T = int(sys.argv[1]) if len(sys.argv) > 1 else 65536
window = int(sys.argv[2]) if len(sys.argv) > 2 else 16384
block = int(sys.argv[3]) if len(sys.argv) > 3 else 128
t0 = int(sys.argv[4]) if len(sys.argv) > 4 else T // 2
W, d, seed = 64, 512, 2510
goom._lib.load()
run = harness.run_chain(T, d, seed=seed, window=window, block=block,
                        snapshots=(t0, t0 + W - 1, t0 + W))
al, as_ = (x[0].cpu().numpy() for x in ops.ts_log_sign(run.snapshots_ts[t0]))
pl, ps = (x[0].cpu().numpy() for x in ops.ts_log_sign(run.snapshots_ts[t0 + W - 1]))
fl, fs = (x[0].cpu().numpy() for x in ops.ts_log_sign(run.snapshots_ts[t0 + W]))
leaves = ops.ts_random_normal(W, d, seed, t0 + 1, torch.device("cuda")).U.cpu().numpy()
l64, s64 = G.log_sign(leaves.astype(np.float64))
_, (ol, os_), (ql, qs), _ = R.fold(al, as_, l64, s64)
kap = G.cancellation(l64[-1], s64[-1], ql, qs)
flip = (fs != os_) & (kap >= 1e-4)
ii, jj = np.nonzero(flip)
out = {"T": T, "window": window, "block": block, "t0": t0, "flips": int(flip.sum()),
       "rows": sorted(set(ii.tolist()))[:20], "n_rows": len(set(ii.tolist())),
       "cols": sorted(set(jj.tolist()))[:20], "n_cols": len(set(jj.tolist()))}
# GPU's own one-step continuation from its P_{t0+W-1}: is the flip already in the GPU's
# state one step earlier (i.e. the direction differs), or made by the last product?
_, (gl1, gs1), _, _ = R.fold(pl, ps, l64[-1:], s64[-1:])
out["flips_vs_gpu_prev_step_continued"] = int(((fs != gs1) & (kap >= 1e-4)).sum())
# the oracle's P_{t0+W-1} vs the GPU's
kprev = G.cancellation(l64[-2], s64[-2], *R.fold(al, as_, l64[:-2], s64[:-2])[1]) if W > 2 else None
out["prev_step_flips"] = int(((ps != qs) & (kprev >= 1e-4)).sum()) if kprev is not None else None
ent = []
for i, j in list(zip(ii, jj))[:12]:
    ent.append({"i": int(i), "j": int(j), "kappa": float(kap[i, j]), "gpu": float(fl[i, j]),
                "oracle": float(ol[i, j]), "row_max_minus": float(ol[i].max() - ol[i, j]),
                "col_max_minus": float(ol[:, j].max() - ol[i, j])})
out["entries"] = ent
out["row_kappa_spread"] = [float(kap[i].min()) for i in sorted(set(ii.tolist()))[:5]]
print(json.dumps(out, indent=1))
