"""Debug aid: config 1 seed 1 (d = 8, T = 1000, block 32) — the position where the scaled-real
error of the GPU chain exceeds the reference float32 runs', and the entry responsible."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
sys.path.insert(0, "tests")
import paper_2510_03426_b200 as g  # noqa: E402
from goom_testlib import chain_kappa, scaled_real_err, to_np  # noqa: E402
from oracle import gooms_port as G  # noqa: E402

seed = int(sys.argv[1]) if len(sys.argv) > 1 else 1
T, d = 1000, 8
mats = np.random.default_rng(seed).standard_normal((T, d, d))
al, as_ = G.log_sign(mats)
A = g.join(al, as_)
for name, blk in (("block32", 32), ("fold", T)):
    gl, gs = to_np(torch.ops.goom.scan_chain(A, blk, None))
    wl, ws = G.chain_blocked(al, as_, T)
    l32, s32 = G.log_sign(mats.astype(np.float32))
    r32 = [G.chain_blocked(l32, s32, T), G.chain_blocked(l32, s32, 32)]
    e = scaled_real_err(gl, gs, wl, ws)
    er = np.max([scaled_real_err(r[0], r[1], wl, ws) for r in r32], axis=0)
    t = int(np.argmax(e / np.maximum(4 * er, 1e-4)))
    kap = chain_kappa(al, as_, wl, ws)
    c = wl[t].max()
    dif = np.abs(gs[t] * np.exp(gl[t] - c) - ws[t] * np.exp(wl[t] - c))
    i, j = np.unravel_index(np.argmax(dif), dif.shape)
    print(f"{name}: worst t={t} gpu {e[t]:.3e} ref32 {er[t]:.3e}; entry ({i},{j}) rel mag "
          f"{np.exp(wl[t][i, j] - c):.3e} kappa {kap[t][i, j]:.2e} sign gpu {gs[t][i, j]} want "
          f"{ws[t][i, j]} ref32 {[r[1][t][i, j] for r in r32]}; log gpu {gl[t][i, j]:.6f} want "
          f"{wl[t][i, j]:.6f}")
