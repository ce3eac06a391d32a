"""GPU parity of the tile-scaled chain engine (lmme_ts.cu, chain_ts.cu; d % 256 == 0)
against the float64 oracle, with the SURVEY §8c criteria: per-LMME rel-log error <= 1e-4
where the cancellation ratio kappa >= 1e-2 and signs exact where kappa >= 1e-4; chains
within 4x the reference's own float32 error (or 2e-4); digests consistent with the
complex64 digest of the same prefixes; edge cases the reference tests (zero rows,
magnitudes beyond float64, non-canonical phases, broadcast carries)."""

import math

import numpy as np
import pytest
import torch

from goom_testlib import (chain_kappa, chain_parity, lmme_parity, scaled_real_err,
                          TC_CHAIN_FLOOR, tc_chain_scaled_floor, to_np)
from oracle import gooms_port as G

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def g():
    import paper_2510_03426_b200 as goom

    goom._lib.load()
    return goom


@pytest.fixture(scope="module")
def ops():
    from paper_2510_03426_b200 import ops

    return ops


def cz(log, sign):
    import paper_2510_03426_b200 as goom

    return goom.join(log, sign)


def rand_ls(rng, *shape):
    return G.log_sign(rng.standard_normal(shape).astype(np.float32))


@pytest.mark.parametrize("d,batch", [(256, 3), (512, 3), (1024, 1)])
def test_lmme_ts_all_epilogues_match_oracle(g, ops, d, batch):
    rng = np.random.default_rng(d)
    al, as_ = rand_ls(rng, batch, d, d)
    bl, bs = rand_ls(rng, batch, d, d)
    ta, tb = ops.ts_from_goom(cz(al, as_)), ops.ts_from_goom(cz(bl, bs))
    for kind in (0, 1):
        out = ops.lmme_ts(ta, tb, kind)
        if kind == 1:
            out = ops.ts_to_goom(out)
        err, flips = lmme_parity(to_np(out), al, as_, bl, bs)
        assert err < 1e-4 and flips == 0, (kind, err, flips)
    # digest epilogue == digest of the oracle product
    dg = ops.lmme_ts(ta, tb, 2).double().cpu().numpy()
    wl, _ = G.lmme(al.astype(np.float64), as_.astype(np.float64), bl.astype(np.float64),
                   bs.astype(np.float64))
    top = wl.reshape(batch, -1).max(axis=1)
    lfro = top + 0.5 * np.log(np.exp(2 * (wl.reshape(batch, -1) - top[:, None])).sum(axis=1))
    assert np.abs(dg[:, 0] - top).max() < 1e-4 * max(1, np.abs(top).max())
    assert np.abs(dg[:, 1] - lfro).max() < 1e-4 * max(1, np.abs(lfro).max())
    assert (dg[:, 2] == 1).all()


def test_lmme_ts_broadcast_and_block_carry(g, ops):
    """Phase-3 shape: every product b uses B[b // div] (stride-0 / div addressing)."""
    d = 256
    rng = np.random.default_rng(7)
    al, as_ = rand_ls(rng, 6, d, d)
    bl, bs = rand_ls(rng, 2, d, d)
    ta, tb = ops.ts_from_goom(cz(al, as_)), ops.ts_from_goom(cz(bl, bs))
    out = ops.lmme_ts(ta, tb, 0, b_div=3)
    err, flips = lmme_parity(to_np(out), al, as_, np.repeat(bl, 3, 0), np.repeat(bs, 3, 0))
    assert err < 1e-4 and flips == 0
    one = ops.lmme_ts(ta, tb[0:1], 0)
    err, flips = lmme_parity(to_np(one), al, as_, np.repeat(bl[:1], 6, 0), np.repeat(bs[:1], 6, 0))
    assert err < 1e-4 and flips == 0


def test_lmme_ts_edge_cases(g, ops):
    """Zero rows / columns (-inf logs), magnitudes beyond float64 (logs ~1e4), a zero
    matrix, non-canonical phases (2 pi, 3 pi, -pi) — core.py:93-113, test_core.py:84-90,
    220-227."""
    d = 256
    rng = np.random.default_rng(11)
    al, as_ = rand_ls(rng, 4, d, d)
    bl, bs = rand_ls(rng, 4, d, d)
    al[0, 5, :] = -np.inf            # zero row of A -> zero row of C
    bl[0, :, 7] = -np.inf            # zero column of B -> zero column of C
    al[1] += 5000.0                  # |x| ~ e^5000: beyond float64
    bl[1] -= 3000.0
    al[2, :, :] = -np.inf            # zero matrix
    A = cz(al, as_)
    B = cz(bl, bs)
    # phases congruent to 0 / pi mod 2 pi
    ph = torch.where(A.imag[3] != 0, torch.tensor(3 * math.pi, device=A.device),
                     torch.tensor(2 * math.pi, device=A.device))
    A[3] = torch.complex(A.real[3], ph)
    out = ops.lmme_ts(ops.ts_from_goom(A), ops.ts_from_goom(B), 0)
    gl, gs = to_np(out)
    wl, ws = G.lmme(al.astype(np.float64), as_.astype(np.float64), bl.astype(np.float64),
                    bs.astype(np.float64))
    assert np.all(gl[0, 5, :] == -np.inf) and np.all(gs[0, 5, :] == 1)
    assert np.all(gl[0, :, 7] == -np.inf)
    assert np.all(gl[2] == -np.inf) and np.all(gs[2] == 1)
    for b in (0, 1, 3):
        m = np.isfinite(wl[b])
        err, flips = lmme_parity((np.where(m, gl[b], wl[b])[None], gs[b][None]), al[b:b + 1],
                                 as_[b:b + 1], bl[b:b + 1], bs[b:b + 1])
        assert err < 1e-4 and flips == 0, (b, err, flips)
    # b = 1: the reference's clamped scales (core.py:252-253: b = max(colmax(B), 0) = 0 for
    # a B of logs ~ -3000) underflow its exp(B - b) to zero, so it returns -inf everywhere;
    # the tile-scaled engine keeps Eq. 11's clamp by default and does the same
    assert np.all(wl[1] == -np.inf)
    assert np.all(gl[1] == -np.inf) and np.all(gs[1] == 1)


def test_lmme_ts_truemax_opt_in(g, ops):
    """GOOM_TS_SCALES=truemax (opt-in, read once per process): true-max scales return the
    finite product where the clamp underflows (checked against the oracle on the shifted
    operands plus the shift)."""
    import os
    import subprocess
    import sys

    d = 256
    rng = np.random.default_rng(11)
    al, as_ = rand_ls(rng, 1, d, d)
    bl, bs = rand_ls(rng, 1, d, d)
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    path = os.path.join(root, "gpurun_out", "_truemax.npz")
    os.makedirs(os.path.dirname(path), exist_ok=True)
    np.savez(path, al=al + 5000.0, as_=as_, bl=bl - 3000.0, bs=bs)
    code = (
        "import sys, numpy as np, torch; sys.path.insert(0, '.');"
        "import paper_2510_03426_b200 as goom; from paper_2510_03426_b200 import ops;"
        "z = np.load(sys.argv[1]);"
        "A = goom.join(z['al'], z['as_']); B = goom.join(z['bl'], z['bs']);"
        "out = ops.lmme_ts(ops.ts_from_goom(A), ops.ts_from_goom(B), 0).cpu();"
        "np.savez(sys.argv[1] + '.out.npz', l=out.real.double().numpy(),"
        " s=np.where(np.cos(out.imag.double().numpy()) < 0, -1.0, 1.0))")
    env = dict(os.environ, GOOM_TS_SCALES="truemax")
    subprocess.run([sys.executable, "-c", code, path], cwd=root, env=env, check=True, timeout=300)
    with np.load(path + ".out.npz") as z:
        gl, gs = z["l"], z["s"]
    os.remove(path)
    os.remove(path + ".out.npz")
    sl, ss = G.lmme(al.astype(np.float64), as_.astype(np.float64), bl.astype(np.float64),
                    bs.astype(np.float64))
    assert np.isfinite(gl).all()
    kap = G.cancellation(al.astype(np.float64), as_.astype(np.float64), bl.astype(np.float64),
                         bs.astype(np.float64))[0]
    rel = np.abs(gl[0] - (sl[0] + 2000.0)) / np.abs(sl[0] + 2000.0)
    assert np.max(np.where(kap >= 1e-2, rel, 0.0)) < 1e-4
    assert np.all((gs[0] == ss[0]) | (kap < 1e-4))


def _engine(lib, e):
    return lib.set_chain_engine(e)


@pytest.mark.parametrize("kind", ["shrinking_identity", "gauss_rho_half"])
def test_ts_clamp_underflows_like_the_reference(g, ops, kind):
    """Eq. 11's clamp on shrinking chains: 0.55 I and a spectral-radius
    ~0.5 Gaussian chain, T = 300, d = 256 / 512, next to the d = 128 path. The exact
    complex64 engine (the public default) and the tile-scaled engine (opt-in) both follow
    the float64 oracle where its logs are above `hi`, and both return -inf below `lo` — the
    reference's float32 exp flushes there (its scales are clamped at 0, so the operands'
    exps underflow; core.py:252-253). 0.55 I is exact in every engine (powers of one scalar,
    the float32 flush at e^-87.3 falls between steps), so its band is narrow and its -inf
    pattern is the same for every d and engine."""
    T, block = 300, 16
    hi, lo = (-85.0, -105.0) if kind == "shrinking_identity" else (-70.0, -120.0)
    pats = {}
    for d in (128, 256, 512):
        rng = np.random.default_rng(d)
        if kind == "shrinking_identity":
            mats = np.broadcast_to(0.55 * np.eye(d), (T, d, d)).copy()
        else:
            mats = rng.standard_normal((T, d, d)) * (0.5 / np.sqrt(d))
        al, as_ = G.log_sign(mats)
        A = cz(al, as_)
        want, wsign = G.chain_blocked(al, as_, block)
        kap = chain_kappa(al, as_, want, wsign)  # entries that are not cancellation noise
        engines = (0, 1) if d % 256 == 0 else (0,)
        for e in engines:
            prev = _engine(g._lib, e)
            try:
                gl, gs = to_np(g.scan_chain(A, block_size=block))
            finally:
                _engine(g._lib, prev)
            up = want > hi
            assert np.isfinite(gl[up]).all(), (d, e)
            up &= kap >= 1e-2
            rel = np.abs(gl[up] - want[up]) / np.maximum(1.0, np.abs(want[up]))
            assert rel.max() < 2e-3, (d, e, rel.max())
            down = want < lo
            assert down.any()
            assert np.all(gl[down] == -np.inf), (d, e, int(np.sum(gl[down] != -np.inf)))
            if kind == "shrinking_identity":
                pats[(d, e)] = np.isfinite(np.diagonal(gl, axis1=1, axis2=2)).all(axis=1)
    if kind == "shrinking_identity":
        ref = pats[(128, 0)]
        assert 0 < ref.sum() < T
        for k, v in pats.items():
            assert np.array_equal(v, ref), (k, np.flatnonzero(v != ref)[:5])


def test_ts_engine_block_flush_is_the_documented_limit(g, ops):
    """A right-operand column far below the largest entry of its 256-column block while its
    own column maximum is >= 0 (P_t = diag(e^{3t}, e^{t}, ...)): the reference keeps it (its
    column scales are per column), the public scan (exact complex64 engine) matches the
    oracle, and the opt-in tile-scaled engine flushes it once the spread passes ~e^87 —
    the format limit documented in lmme_ts.cu / DESIGN.md."""
    d, T, block = 256, 64, 8
    diag = np.ones(d)
    diag[0] = np.e ** 3
    diag[1:] = np.e
    mats = np.broadcast_to(np.diag(diag), (T, d, d)).copy()
    al, as_ = G.log_sign(mats)
    A = cz(al, as_)
    want, _ = G.chain_blocked(al, as_, block)
    prev = _engine(g._lib, 0)
    try:
        gl, _ = to_np(g.scan_chain(A, block_size=block))
        _engine(g._lib, 1)
        tl, _ = to_np(g.scan_chain(A, block_size=block))
    finally:
        _engine(g._lib, prev)
    d1 = np.arange(T)
    w11 = want[:, 1, 1]
    assert np.allclose(gl[:, 1, 1], w11, rtol=1e-5)           # exact engine: kept
    spread = want[:, 0, 0] - want[:, 1, 1]                     # 2 (t + 1) nats
    assert np.allclose(tl[spread < 60, 1, 1], w11[spread < 60], rtol=1e-5)
    assert np.all(tl[spread > 110, 1, 1] == -np.inf)           # tile-scaled: flushed
    assert d1.size == T


@pytest.mark.parametrize("engine", [0, 1])
@pytest.mark.parametrize("d,T,block", [(256, 64, 8), (256, 33, 64), (512, 24, 5), (1024, 6, 2),
                                       (256, 1, 4)])
def test_chain_ts_matches_float64_oracle(g, ops, d, T, block, engine):
    """The public chain scan for d % 256 == 0 on both engines (0: exact complex64 kernels,
    the default; 1: tile-scaled) vs the float64 oracle, calibrated by the reference's own
    float32 runs (SURVEY §8c chain criterion)."""
    rng = np.random.default_rng(d * T + block)
    mats = rng.standard_normal((T, d, d))
    al, as_ = G.log_sign(mats)
    prev = g._lib.set_chain_engine(engine)
    try:
        out = g.scan_chain(cz(al, as_), block_size=block)
    finally:
        g._lib.set_chain_engine(prev)
    gl, gs = to_np(out)
    want = G.chain_blocked(al, as_, T)
    l32, s32 = G.log_sign(mats.astype(np.float32))
    refs = [G.chain_blocked(l32, s32, block), G.chain_blocked(l32, s32, T)]
    r = chain_parity(gl, gs, al, as_, want, refs, scaled_floor=tc_chain_scaled_floor(d, T),
                     floor=TC_CHAIN_FLOOR)
    assert r["ok"], (r["bad"], r["flips"], r["scaled_bad"])


def test_chain_ts_carry_digests_and_windows(g, ops):
    """Carry-in / carry-out and digests of chain_ts: two windows with the carry threaded
    through equal one window (within float32 noise), digests equal the complex64 digest of
    the same prefixes, and the carry-out is the last prefix."""
    d, T, block = 256, 48, 8
    rng = np.random.default_rng(5)
    al, as_ = rand_ls(rng, T, d, d)
    leaves = ops.ts_from_goom(cz(al, as_))
    P, dg, c = ops.chain_ts(leaves, block, None, out=True, digests=True, carry_out=True)
    dref = torch.ops.goom.digest(P)
    assert torch.allclose(dg[:, :3], dref[:, :3], rtol=1e-5, atol=1e-4)
    cl, cs = to_np(ops.ts_to_goom(c))
    pl, ps = to_np(P[-1:])
    # same product, tile-scaled vs complex64 epilogue: q = rowmax + G + e ln 2 rounds at
    # ulp(|log|) ~ 1.5e-5 for the logs ~130 reached here
    assert scaled_real_err(cl, cs, pl, ps).max() < 1e-4
    P1, _, c1 = ops.chain_ts(leaves[0:20], block, None, out=True, digests=False, carry_out=True)
    P2, _, _ = ops.chain_ts(leaves[20:48], block, c1, out=True, digests=False, carry_out=False)
    got = torch.cat([P1, P2])
    gl, gs = to_np(got)
    wl, ws = to_np(P)
    assert scaled_real_err(gl, gs, wl, ws).max() < 1e-3
    # the public scan with a complex64 carry equals the tile-scaled carry path
    carry = ops.ts_to_goom(c1)[0]
    pub = g.scan_chain(cz(al[20:], as_[20:]), block, carry)
    ql, qs = to_np(pub)
    pl2, ps2 = to_np(P2)
    assert scaled_real_err(ql, qs, pl2, ps2).max() < 1e-4


def test_random_normal_ts_is_the_same_chain(g, ops):
    from paper_2510_03426_b200 import harness

    d = 256
    a = harness.random_chain(6, d, seed=4, t0=3)
    t = ops.ts_random_normal(6, d, seed=4, t0=3, device=a.device)
    x = torch.ops.goom.to_real(a, True).float()
    assert torch.allclose(t.U, x, rtol=2e-6, atol=1e-6)
    assert (t.q == 0).all()


def test_random_normal_ts_is_counter_based(g, ops):
    """Leaf t is a function of (seed, t) only: one call over 7 leaves equals two calls over
    3 + 4 (different grid-stride partitions of the counters, the two-counter main loop and
    its single-counter tail), bit for bit; and different seeds differ."""
    d, dev = 256, torch.device("cuda")
    whole = ops.ts_random_normal(7, d, 9, 5, dev).U
    parts = torch.cat([ops.ts_random_normal(3, d, 9, 5, dev).U,
                       ops.ts_random_normal(4, d, 9, 8, dev).U])
    assert torch.equal(whole, parts)
    assert not torch.equal(whole, ops.ts_random_normal(7, d, 10, 5, dev).U)
    z = whole.double()
    assert abs(float(z.mean())) < 0.01 and abs(float(z.std()) - 1.0) < 0.01


def test_harness_ts_growth_and_digest_parity(g, ops):
    """Config 3 machinery at d = 512 on the tile-scaled engine: per-prefix digests equal
    the complex64 digests of the same chain, and log||P_t|| grows at (ln 2 + psi(d/2)) / 2."""
    from paper_2510_03426_b200 import harness

    d, T = 512, 300
    run = harness.run_chain(T, d, seed=3, window=128, block=16)
    P = g.scan_chain(harness.random_chain(T, d, seed=3), 16)
    ref = torch.ops.goom.digest(P).double().cpu().numpy()
    dg = run.digests.double().cpu().numpy()
    assert (dg[:, 2] == 1).all()
    assert np.max(np.abs(dg[:, 1] - ref[:, 1]) / np.maximum(1, np.abs(ref[:, 1]))) < 1e-4
    gl, gs = to_np(run.final[None])
    rl, rs = to_np(P[-1:])
    assert scaled_real_err(gl, gs, rl, rs).max() < 1e-2
    rate = harness.growth_rate(run.digests)
    psi = math.log(d / 2) - 1 / d - 1 / (12 * (d / 2) ** 2)
    assert abs(rate - 0.5 * (math.log(2) + psi)) < 0.02


def test_harness_streams_real_host_leaves(g, ops):
    """run_chain with real float32 leaves in pinned host memory (copied window by window on a
    copy stream) equals the run on the same chain generated on the device."""
    from paper_2510_03426_b200 import harness

    d, T = 256, 96
    gen = harness.run_chain(T, d, seed=11, window=32, block=8)
    host = ops.ts_random_normal(T, d, 11, 0, torch.device("cuda")).U.cpu().pin_memory()
    got = harness.run_chain(T, d, window=32, block=8, leaves=host)
    assert torch.equal(got.digests, gen.digests)
    dev_real = harness.run_chain(T, d, window=32, block=8, leaves=host.cuda())
    assert torch.equal(dev_real.digests, gen.digests)
    with pytest.raises(ValueError):
        harness.run_chain(T, d, window=32, block=8, leaves=host.double())


def test_chain_ts_persistent_phase1_matches_launches(g, ops):
    """The opt-in persistent phase 1 (GOOM_CHAIN_PERSISTENT=1: one launch, step-major tiles,
    release / acquire counters) gives the same digests as the per-step launches: same
    products in the same order, so bitwise-equal."""
    import os
    import subprocess
    import sys

    code = (
        "import sys, torch; sys.path.insert(0, '.');"
        "from paper_2510_03426_b200 import ops;"
        "L = ops.ts_random_normal(4096, 512, 7, 0, torch.device('cuda'));"
        "_, dg, c = ops.chain_ts(L, 64, None, digests=True, carry_out=True);"
        "torch.save((dg.cpu(), ops.ts_to_goom(c).cpu()), sys.argv[1])")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    outs = []
    for flag in ("0", "1"):
        path = os.path.join(root, "gpurun_out", f"_persist_{flag}.pt")
        os.makedirs(os.path.dirname(path), exist_ok=True)
        env = dict(os.environ, GOOM_CHAIN_PERSISTENT=flag)
        subprocess.run([sys.executable, "-c", code, path], cwd=root, env=env, check=True,
                       timeout=300)
        outs.append(torch.load(path))
        os.remove(path)
    assert torch.equal(outs[0][0], outs[1][0])
    assert torch.equal(outs[0][1], outs[1][1])
