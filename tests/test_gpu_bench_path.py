"""Parity of the exact config-3 bench path (harness.run_chain on the tile-scaled engine:
generated tile-scaled leaves, phase 1 batched launches, Kogge-Stone tree of block totals,
phase 3 with the digest epilogue, window carries) against the float64 oracle.

* T = 512: every digest compared with the oracle's sequential fold of the same leaves
  (the reference's scan_sequential / _scan_affine_stack with block >= T), calibrated by
  the reference's own float32 run; full prefixes at several t via snapshots.
* T = 4096, window 1024, block 128 (the bench's block, 8 blocks per window, 4 windows):
  re-anchored windows — the oracle recomputes 64 steps from GPU snapshots
  P_{t0} deep in the chain and compares P_{t0+64} entry by entry (rel-log within 4x the
  float32 reference's error or 1e-4, signs exact where kappa >= 1e-4) and every digest of
  the stretch.
"""

import numpy as np
import pytest
import torch

from goom_testlib import to_np
from oracle import gooms_port as G
from oracle import reanchor as R

pytestmark = pytest.mark.gpu

D = 512


@pytest.fixture(scope="module")
def h():
    import paper_2510_03426_b200 as goom
    from paper_2510_03426_b200 import harness

    goom._lib.load()
    return harness


def leaves_real(T, d, seed, t0):
    from paper_2510_03426_b200 import ops

    return ops.ts_random_normal(T, d, seed, t0, torch.device("cuda")).U.cpu().numpy()


def test_bench_path_every_digest_vs_oracle(h):
    T, seed = 512, 21
    snaps = (0, 100, 255, 256, 511)
    run = h.run_chain(T, D, seed=seed, window=128, block=16, snapshots=snaps)
    dg = run.digests.double().cpu().numpy()
    assert (dg[:, 2] == 1).all()
    x = leaves_real(T, D, seed, 0)
    al, as_ = G.log_sign(x.astype(np.float64))
    p0 = (al[0], as_[0])
    keep = tuple(t for t in snaps if t > 0)
    dg_o, _, _, kept = R.fold(p0[0], p0[1], al[1:], as_[1:], keep=keep)
    l32, s32 = G.log_sign(x)
    dg_r, _, _, kept32 = R.fold(l32[0], s32[0], l32[1:], s32[1:], keep=keep)
    # P_0 = A_0: digest of the leaf itself
    t0d = R._digest1(al[0])
    dg_o = np.vstack([np.array(t0d)[None], dg_o])
    dg_r = np.vstack([np.array(R._digest1(l32[0].astype(np.float64)))[None], dg_r])
    for col in (0, 1):
        e_gpu = np.abs(dg[:, col] - dg_o[:, col]) / np.maximum(1.0, np.abs(dg_o[:, col]))
        e_ref = np.abs(dg_r[:, col] - dg_o[:, col]) / np.maximum(1.0, np.abs(dg_o[:, col]))
        ulp2 = 2 * np.spacing(np.abs(dg_o[:, col]).astype(np.float32)).astype(np.float64)
        bound = np.maximum(np.maximum(4 * e_ref, 1e-4), ulp2 / np.maximum(1.0, np.abs(dg_o[:, col])))
        assert np.all(e_gpu <= bound), (col, np.flatnonzero(e_gpu > bound)[:10], e_gpu.max())
    # full prefixes: entrywise rel-log (kappa-masked), signs exact where kappa >= 1e-4
    for t in keep:
        gl, gs = to_np(run.snapshots[t][None])
        ol, os_ = kept[t]
        rl, rs = kept32[t]
        e_gpu = R._rel(gl[0], ol)
        e_ref = R._rel(rl, ol)
        assert e_gpu.max() <= max(4 * e_ref.max(), 1e-4), (t, e_gpu.max(), e_ref.max())
        assert np.mean(gs[0] == os_) > 0.999, t
    gl, gs = to_np(run.snapshots[0][None])
    assert R._rel(gl[0], al[0]).max() < 1e-6 and np.all(gs[0] == as_[0])


@pytest.mark.parametrize("t0", [768, 2048, 4096 - 128])
def test_bench_path_reanchored_windows(h, t0):
    """Block starts t0 (block 128): the oracle folds A_t0 .. A_t0+63 onto the block carry the
    engine applied there (its own P_{t0-1}, exact to the engine's precision) and compares
    P_{t0+63} and every digest of the stretch; window 1024 puts t0 = 2048 on a window
    boundary (the carry is the previous window's carry-out)."""
    from paper_2510_03426_b200 import ops

    T, seed, W = 4096, 2510, 64
    run = h.run_chain(T, D, seed=seed, window=1024, block=128, snapshots=(t0 + W - 1,),
                      anchors=(t0,))
    assert bool((run.digests[:, 2] == 1).all())
    al, as_ = (x[0].cpu().numpy() for x in ops.ts_log_sign(run.anchors_ts[t0]))
    fl, fs = (x[0].cpu().numpy() for x in ops.ts_log_sign(run.snapshots_ts[t0 + W - 1]))
    leaves = leaves_real(W, D, seed, t0)
    dg = run.digests[t0:t0 + W, :2].cpu().numpy()
    r = R.check_window(al, as_, leaves, fl, fs, dg)
    assert r["ok"], r
    assert r["sign_flips"] == 0 and r["sign_checked"] > 0.99 * D * D
    # the complex64 snapshot is the same prefix rounded to float32 logs
    zl, zs = to_np(run.snapshots[t0 + W - 1][None])
    assert np.abs(zl[0] - fl).max() <= 2 * np.spacing(np.float32(np.abs(fl).max()))
    assert np.array_equal(zs[0], fs)
    with pytest.raises(ValueError):
        h.run_chain(256, D, seed=seed, window=128, block=64, anchors=(65,))


def test_harness_snapshots_equal_full_window_output(h):
    """Snapshots recomputed from the workspace (L_t (x) block carry) are the prefixes the
    full phase-3 output writes for the same window (same product; the snapshot leaves through
    the tile-scaled epilogue, so logs agree to float32 rounding and signs exactly)."""
    from paper_2510_03426_b200 import ops

    d, T, block = 256, 96, 16
    L = ops.ts_random_normal(T, d, 5, 0, torch.device("cuda"))
    P, _, _ = ops.chain_ts(L, block, None, out=True, digests=False, carry_out=False)
    _, _, _, S, _ = ops.chain_ts(L, block, None, digests=True, carry_out=False,
                                 snapshots=[0, 15, 16, 95])
    S64 = ops.ts_to_goom(S)
    for j, t in enumerate([0, 15, 16, 95]):
        # the same product through the tile-scaled epilogue, exported: equal to the complex64
        # epilogue's output within float32 rounding of the log (q + log|U| vs log|S| + a + b)
        gl, gs = to_np(S64[j:j + 1])
        wl, ws = to_np(P[t:t + 1])
        assert np.array_equal(gs, ws), t
        assert np.abs(gl - wl).max() <= 4 * np.spacing(np.float32(np.abs(wl).max())), t
