"""Re-anchored window check for chains too long for the CPU (TEST ORACLE ONLY).

SURVEY §8c(5): a GPU run of a 2^20-long d = 512 chain cannot be recomputed on the
host, but any W <= 64-step stretch of it can, starting from a prefix the GPU
provides. Given the GPU snapshot P_{t0} (complex64: float32 log + sign), the real
leaves A_{t0+1} .. A_{t0+W} (regenerated from the counter-based RNG) and the GPU's
own results for that stretch (the digests of P_{t0+1..t0+W} and the snapshot
P_{t0+W}), this module

  * recomputes the stretch with the reference's sequential fold
    (`P_t = A_t (x) P_{t-1}`, scan.py:181-214 with block >= T; products accumulate on
    the left, combine_affine scan.py:92-103) in float64 — the oracle;
  * recomputes it again in float32 from the same float32 anchor — the reference's own
    float32 run, which calibrates the tolerance (a fixed 1e-4 is not met
    by float32 itself);
  * compares the GPU's P_{t0+W} with the oracle entry by entry, and the GPU digests
    (max log, log Frobenius norm) with the oracle's at every step.

Two frames are reported:
  * the reference's `_rel_log_diff` (pkg/tests/test_scan.py:209-213: |x - y| /
    max(1, |y|)) on the absolute logs, which at t0 ~ 2^19 (|log| ~ 1.6e6) is a weak
    bound (1e-4 of 1.6e6 = 160 nats);
  * the anchored frame: every log shifted by the anchor's max log c0, so values are
    O(W * 3.1) nats and the same relative criterion bounds the error in nats. Complex64
    logs at 1.6e6 are quantised at 0.125 nats (float32 ulp), which the float32 reference
    run shares; hence the bound max(4 x the reference float32's error, 1e-4) per step.

Signs must match the oracle exactly wherever the cancellation ratio of the last LMME is
kappa >= 1e-4 (the float32 reference's flips there are reported beside: it starts from the
anchor rounded to float32 logs, which at |log| ~ 1e5 is 0.4% noise per entry).
"""

from __future__ import annotations

import numpy as np

from . import gooms_port as G

NEG_INF = float("-inf")


def _digest1(log):
    """(max log, log Frobenius norm) of one float64 log matrix."""
    top = float(log.max())
    if top == NEG_INF:
        return top, top
    with np.errstate(invalid="ignore", over="ignore"):
        return top, top + 0.5 * float(np.log(np.exp(2.0 * (log - top)).sum()))


def fold(p_log, p_sign, a_log, a_sign, keep=()):
    """Sequential fold from the anchor: P_w = A_w (x) P_{w-1}, w = 1..W, streamed.
    Returns (digests (W, 2) float64, P_W, P_{W-1}, {w: P_w for w in keep}) with each P a
    (log, sign) pair in the inputs' dtype (1-based w: keep=(W,) is the last state)."""
    W = a_log.shape[0]
    dg = np.empty((W, 2), dtype=np.float64)
    kept = {}
    prev = (p_log, p_sign)
    for w in range(W):
        prev = (p_log, p_sign)
        p_log, p_sign = G.lmme(a_log[w], a_sign[w], p_log, p_sign)
        dg[w] = _digest1(p_log.astype(np.float64))
        if w + 1 in keep:
            kept[w + 1] = (p_log.copy(), p_sign.copy())
    return dg, (p_log, p_sign), prev, kept


def _rel(x, y, shift=0.0):
    x = np.asarray(x, dtype=np.float64) - shift
    y = np.asarray(y, dtype=np.float64) - shift
    both = (x == NEG_INF) & (y == NEG_INF)
    with np.errstate(invalid="ignore"):
        d = np.where(both, 0.0, np.abs(x - y) / np.maximum(1.0, np.abs(y)))
    return np.where(np.isnan(d), np.inf, d)


def fold_block(p_log, p_sign, a_log, a_sign):
    """The chain engine's tree for a stretch that starts a block: local products
    L_w = A_w (x) L_{w-1} (L_0 = A_0) within the block, each prefix L_w (x) P (the block
    carry on the right; scan.py:196-213). Returns (digests (W, 2), P_{W-1}) like fold."""
    W = a_log.shape[0]
    dg = np.empty((W, 2), dtype=np.float64)
    L = (a_log[0], a_sign[0])
    for w in range(W):
        if w:
            L = G.lmme(a_log[w], a_sign[w], L[0], L[1])
        out = G.lmme(L[0], L[1], p_log, p_sign)
        dg[w] = _digest1(out[0].astype(np.float64))
    return dg, out


def check_window(anchor_log, anchor_sign, leaves, gpu_final_log, gpu_final_sign,
                 gpu_digests, factor=4.0, floor=1e-4, kappa_min=1e-2, sign_kappa=1e-4):
    """Re-anchored check of one stretch.

    anchor_log/sign: the matrix the GPU applied on the right of the stretch (d, d) — the
    engine's block carry, its own P_{t0-1} (float64 log of the tile-scaled state,
    ops.ts_log_sign) — and +-1 sign. leaves: real A_{t0..t0+W-1} (W, d, d), float32 values
    (the chain's leaves exactly). gpu_final_log/sign: the GPU's P_{t0+W-1} (d, d).
    gpu_digests: (W, >=2) GPU digests of P_{t0..t0+W-1} (max log, log Frobenius).

    The float64 oracle folds the leaves sequentially onto the anchor; the tolerance is
    calibrated by the reference's own float32 runs from the same anchor (rounded to float32
    logs, as a float32 user holds it) along both trees — the sequential fold and the
    engine's block tree L_w (x) anchor — taking the larger error, as the §8c chain criterion
    does over block sizes. Returns a dict of metrics; `ok` is the verdict."""
    anchor_log = np.asarray(anchor_log, dtype=np.float64)
    anchor_sign = np.asarray(anchor_sign, dtype=np.float64)
    leaves = np.asarray(leaves, dtype=np.float32)
    W = leaves.shape[0]
    c0 = float(anchor_log.max())
    # oracle: float64 from the anchor as the engine holds it
    al64, as64 = G.log_sign(leaves.astype(np.float64))
    dg_o, (o_l, o_s), (q_l, q_s), _ = fold(anchor_log, anchor_sign, al64, as64)
    # the reference's own float32 runs from the same anchor: sequential fold and block tree
    al32, as32 = G.log_sign(leaves)
    a32 = (anchor_log.astype(np.float32), anchor_sign.astype(np.float32))
    dg_r1, (r1_l, r1_s), _, _ = fold(a32[0], a32[1], al32, as32)
    dg_r2, (r2_l, r2_s) = fold_block(a32[0], a32[1], al32, as32)
    # last-step cancellation ratio (signs are only defined where the sum does not cancel)
    kap = G.cancellation(al64[-1], as64[-1], q_l, q_s)
    mask = kap >= kappa_min
    gl = np.asarray(gpu_final_log, dtype=np.float64)
    gs = np.asarray(gpu_final_sign, dtype=np.float64)

    def err(x, shift=0.0):
        return float(np.max(np.where(mask, _rel(x, o_l, shift), 0.0)))

    fin = mask & np.isfinite(o_l)

    def nats(x):
        with np.errstate(invalid="ignore"):
            return float(np.max(np.where(fin, np.abs(np.asarray(x, np.float64) - o_l), 0.0)))

    e_gpu_abs, e_gpu = err(gl), err(gl, c0)
    e_ref_abs = max(err(r1_l), err(r2_l))
    e_ref = max(err(r1_l, c0), err(r2_l, c0))
    smask = kap >= sign_kappa
    flips = int(np.sum((gs != o_s) & smask))
    flips_ref32 = [int(np.sum((r != o_s) & smask)) for r in (r1_s, r2_s)]
    # digests at every step of the stretch, anchored frame
    dg = np.asarray(gpu_digests, dtype=np.float64)

    def derr(d):
        return np.maximum(_rel(d[:, 0], dg_o[:, 0], c0), _rel(d[:, 1], dg_o[:, 1], c0))

    de_gpu = derr(dg)
    de_ref = np.maximum(derr(dg_r1), derr(dg_r2))
    # a float32 digest cannot resolve less than its own ulp at |log| ~ c0 (0.125 nats at 2^21):
    # two ulps are allowed on top of the calibrated bound (one digest is two numbers per step,
    # so a float32 run's error there can be zero by luck)
    ulp2 = 2.0 * float(np.spacing(np.float32(abs(c0) + 4.0 * W)))
    quant = ulp2 / np.maximum(1.0, np.abs(dg_o[:, 1] - c0))
    dbound = np.maximum(np.maximum(factor * de_ref, floor), quant)
    ok = (e_gpu <= max(factor * e_ref, floor) and e_gpu_abs <= max(factor * e_ref_abs, floor)
          and flips == 0 and bool(np.all(de_gpu <= dbound)))
    return dict(ok=bool(ok), W=W, c0=c0, kappa_masked_frac=float(mask.mean()),
                rel_log_abs_gpu=e_gpu_abs, rel_log_abs_ref32=e_ref_abs,
                rel_log_anchored_gpu=e_gpu, rel_log_anchored_ref32=e_ref,
                max_abs_nats_gpu=nats(gl), max_abs_nats_ref32=max(nats(r1_l), nats(r2_l)),
                sign_flips=flips, sign_flips_ref32=flips_ref32, sign_checked=int(smask.sum()),
                digest_rel_anchored_gpu_max=float(de_gpu.max()),
                digest_rel_anchored_ref32_max=float(de_ref.max()),
                digest_steps_over_bound=int(np.sum(de_gpu > dbound)))
