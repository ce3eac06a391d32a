"""GPU parity of the scan engines against the oracle and the reference's golden scans.

Mirrors pkg/tests/test_scan.py (TestScanParallel, TestSelectiveScan,
TestGoldenThreeStep) plus the SURVEY §8c chain criterion: per position,
err(GPU complex64 vs float64 oracle) <= max(4 * err(reference float32 vs
float64 oracle), 1e-4) in _rel_log_diff, signs exact where |x| is not near 0.
"""

import numpy as np
import pytest
import torch

from goom_testlib import (NEG_INF, chain_parity, load_golden, rel_log_diff_per, scaled_real_err,
                          to_np)
from oracle import gooms_port as G

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def g():
    import paper_2510_03426_b200 as goom

    goom._lib.load()
    return goom


def cz(log, sign):
    import paper_2510_03426_b200 as goom

    return goom.join(log, sign)


def calibrated_ok(got_log, want64, ref32, floor=1e-4, factor=4.0):
    e_gpu = rel_log_diff_per(got_log, want64)
    e_ref = rel_log_diff_per(ref32, want64)
    bound = np.maximum(factor * e_ref, floor)
    bad = np.flatnonzero(e_gpu > bound)
    return bad, e_gpu, e_ref


# ---------------------------------------------------------------------------
# product chains / affine scans


@pytest.mark.parametrize("block", [1, 16, 32, 64, 1000])
def test_config1_chain_d8_T1000(g, block):
    """Config 1: 1,000 random-normal 8x8 leaves, all prefixes (golden from the reference),
    against the float64 sequential oracle, calibrated by the reference's own float32 runs."""
    z = load_golden("config1_chain")
    al, as_ = G.log_sign(z["mats"])
    out = g.scan_chain(cz(al, as_), block_size=block)
    gl, gs = to_np(out)
    want = (z["seq_f64"][0], z["seq_f64"][1])
    refs = [z["seq_f32"], z["par32_f32"]]
    r = chain_parity(gl, gs, al, as_, want, refs)
    assert r["ok"], (r["bad"], r["e_gpu"][r["bad"]], r["e_ref"][r["bad"]], r["flips"],
                     r["scaled_bad"])


@pytest.mark.parametrize("block", [1, 32, 1000])
def test_config1_chain_complex128_matches_float64_reference(g, block):
    """complex128 GOOMs reproduce the reference's own float64 run to its float64
    tolerance (test_scan.py:227-237 uses 1e-10 across block sizes)."""
    z = load_golden("config1_chain")
    al, as_ = G.log_sign(z["mats"])
    out = g.scan_chain(g.join(al, as_, torch.complex128), block_size=block)
    gl, gs = to_np(out)
    want = z["seq_f64"] if block >= 1000 else (z["par32_f64"] if block == 32 else z["seq_f64"])
    assert G.rel_log_diff(gl, want[0]) < 1e-9
    assert np.array_equal(gs, want[1])


def test_block_ge_T_is_sequential_fold_bitwise(g):
    """scan.py:217-225: block >= T degenerates to the sequential fold (same combines)."""
    rng = np.random.default_rng(38)
    A = cz(*G.log_sign(rng.standard_normal((7, 3, 3))))
    B = cz(*G.log_sign(rng.standard_normal((7, 3, 3))))
    st = g._Stack(A, B)
    par = g._scan_affine_stack(st, 7)
    seq = g._Stack(A.clone(), B.clone())
    for t in range(1, 7):
        seq.A[t] = torch.ops.goom.lmme(A[t], seq.A[t - 1])
        seq.B[t] = torch.ops.goom.lmme_gadd(A[t], seq.B[t - 1], B[t])
    assert torch.equal(par.A, seq.A) and torch.equal(par.B, seq.B)


def test_affine_golden_T64_d4(g):
    z = load_golden("affine_T64_d4")
    st = g._Stack(cz(z["alog"], z["asign"]), cz(z["blog"], z["bsign"]))
    for block, key in ((64, "seq"), (8, "par8")):
        out = g._scan_affine_stack(st, block)
        gl, gs = to_np(out.A)
        bl, bs = to_np(out.B)
        ref = z[key]
        assert G.rel_log_diff(gl, ref[0]) < 1e-4
        assert G.rel_log_diff(bl, ref[2]) < 1e-4
        assert np.mean(gs == ref[1]) > 0.999 and np.mean(bs == ref[3]) > 0.999


def test_1024_leaves_across_block_sizes(g):
    """test_scan.py:227-237 at complex64: blocks {4,16,64} vs the f64 sequential oracle."""
    rng = np.random.default_rng(39)
    T, d = 1024, 8
    st64 = G.random_stack(rng, T, d, biases=True)
    seq = G.scan_sequential(st64)
    st32 = G.Stack(*(x.astype(np.float32) for x in (st64.alog, st64.asign, st64.blog, st64.bsign)),
                   st64.flags.copy())
    st = g._Stack(cz(st64.alog, st64.asign), cz(st64.blog, st64.bsign))
    st128 = g._Stack.from_arrays(st64.alog, st64.asign, st64.blog, st64.bsign)
    # the reference's own float32 noise at each position: worst over its block sizes
    refs = [G.scan_affine_blocked(st32, b) for b in (4, 16, 64, T)]
    ref_a = np.max([scaled_real_err(r.alog, r.asign, seq.alog, seq.asign) for r in refs], axis=0)
    ref_b = np.max([scaled_real_err(r.blog, r.bsign, seq.blog, seq.bsign) for r in refs], axis=0)
    for bs in (4, 16, 64):
        out = g._scan_affine_stack(st, bs)
        for slot, wl, ws, err_ref in ((out.A, seq.alog, seq.asign, ref_a),
                                      (out.B, seq.blog, seq.bsign, ref_b)):
            gl, gs = to_np(slot)
            err = scaled_real_err(gl, gs, wl, ws)
            bad = np.flatnonzero(err > np.maximum(4 * err_ref, 1e-4))
            assert bad.size == 0, (bs, bad[:5], err[bad[:5]], err_ref[bad[:5]])
        # complex128: the reference's float64 tolerance (1e-10, sign-exact)
        o128 = g._scan_affine_stack(st128, bs)
        ref64 = G.scan_affine_blocked(st64, bs)
        gl, gs = to_np(o128.A)
        assert G.rel_log_diff(gl, ref64.alog) < 1e-10 and np.array_equal(gs, ref64.asign)
        gl, gs = to_np(o128.B)
        assert G.rel_log_diff(gl, ref64.blog) < 1e-10 and np.array_equal(gs, ref64.bsign)


def test_zero_bias_affine_is_product_chain(g):
    """test_scan.py:328-337: zero biases -> pure product chain; bias slot stays zero."""
    rng = np.random.default_rng(48)
    mats = rng.standard_normal((12, 3, 3))
    leaves = [g.ScanPair(g.GoomMatrix.from_real(m), g.GoomMatrix.zeros(3, 3)) for m in mats]
    out = g.scan_parallel(leaves, g.combine_affine, block_size=4)
    prod = np.eye(3)
    for m, pair in zip(mats, out):
        prod = m @ prod
        np.testing.assert_allclose(pair.A.to_real(), prod, rtol=1e-5, atol=1e-6)
        assert bool((pair.B.log_mag == NEG_INF).all())


def test_chain_with_carry_in(g):
    rng = np.random.default_rng(9)
    T, d = 40, 6
    al, as_ = G.log_sign(rng.standard_normal((T, d, d)))
    cl, cs = G.log_sign(rng.standard_normal((d, d)))
    out = g.scan_chain(cz(al, as_), block_size=8, carry=cz(cl, cs))
    # oracle: prefix products times the carry on the right
    st = G.Stack(np.concatenate([cl[None], al]), np.concatenate([cs[None], as_]),
                 np.full((T + 1, d, d), NEG_INF), np.ones((T + 1, d, d)), np.zeros(T + 1, bool))
    want = G.scan_sequential(st)
    gl, gs = to_np(out)
    assert scaled_real_err(gl, gs, want.alog[1:], want.asign[1:]).max() < 1e-5


def test_pairs_api_and_sequential(g):
    rng = np.random.default_rng(37)
    mats = [rng.standard_normal((3, 3)) for _ in range(16)]
    bias = [rng.standard_normal((3, 3)) for _ in range(16)]
    leaves = [g.ScanPair(g.GoomMatrix.from_real(a), g.GoomMatrix.from_real(b))
              for a, b in zip(mats, bias)]
    out = g.scan_sequential(leaves, g.combine_affine)
    x = np.eye(3)
    for a, b, pair in zip(mats, bias, out):
        x = a @ x + b
        got = pair.A.to_real() + pair.B.to_real()
        np.testing.assert_allclose(got, x, rtol=1e-4, atol=1e-5)
    with pytest.raises(ValueError):
        g.scan_parallel(leaves, g.combine_affine, block_size=0)


# ---------------------------------------------------------------------------
# selective scans


def _chain_states(V):
    return to_np(V)


def test_selective_norm_threshold_sites_golden(g):
    z = load_golden("sel_norm_T300_d4")
    A = cz(z["alog"], z["asign"])
    want_sites = list(z["sites"])
    for block in (2, 4, 7, 32):
        V, sites = g._selective_chain_core(A, g.norm_threshold_policy(12.0), block)
        assert sites == want_sites
        gl, gs = _chain_states(V)
        assert scaled_real_err(gl, gs, *z["seq_state"]).max() < 1e-4
    # pair API: flags monotone from the first site (test_scan.py:306-314)
    leaves = [g.ScanPair(g.GoomMatrix(z["alog"][i], z["asign"][i]),
                         g.GoomMatrix.zeros(4, 4)) for i in range(len(z["alog"]))]
    states, sites = g.scan_selective(leaves, g.norm_threshold_policy(12.0), block_size=8)
    flags = np.array([s.reset_applied for s in states])
    assert sites == want_sites
    assert np.array_equal(flags, np.arange(len(flags)) >= sites[0])
    np.testing.assert_array_equal(flags, z["seq_flags"])


def test_selective_interval_8(g):
    z = load_golden("sel_norm_interval8")
    V, sites = g._selective_chain_core(cz(z["alog"], z["asign"]),
                                       g.norm_threshold_policy(5.0, interval=8), 16)
    assert sites == list(z["sites"])
    assert all(s % 8 == 0 for s in sites)
    gl, gs = _chain_states(V)
    assert scaled_real_err(gl, gs, *z["seq_state"]).max() < 1e-4


def test_selective_with_biases_rounds(g):
    z = load_golden("sel_norm_bias")
    st = g._Stack(cz(z["alog"], z["asign"]), cz(z["blog"], z["bsign"]))
    for block in (4, 16, 64):
        out, sites = g.scan_selective(st, g.norm_threshold_policy(12.0), block_size=block)
        assert sites == list(z["sites"])
        np.testing.assert_array_equal(out.flags.cpu().numpy(), z["seq_flags"])
        gl, gs = to_np(out.states())
        assert scaled_real_err(gl, gs, *z["seq_state"]).max() < 1e-4


def test_colinearity_lorenz_sites(g):
    """spectrum_parallel stage (a) on a Lorenz chain: sites identical to the reference."""
    z = load_golden("sel_colin_lorenz")
    # the reference's array-level call (lyapunov.py:341): float64 arrays -> complex128 chain
    Vl, Vs, sites = g._selective_chain_core(z["alog"], z["asign"], g.colinearity_policy(0.99, 12),
                                            256)
    assert sites == list(z["sites"])
    assert G.rel_log_diff(Vl, z["Vlog"]) < 1e-9
    assert scaled_real_err(Vl, Vs, z["Vlog"], z["Vsign"]).max() < 1e-10
    w = load_golden("sel_colin_lorenz_walk")
    V1, S1, s1 = g._selective_chain_core(z["alog"][:600], z["asign"][:600],
                                         g.colinearity_policy(0.99, 1), 64)
    assert s1 == list(w["sites"])
    assert scaled_real_err(V1, S1, w["Vlog"], w["Vsign"]).max() < 1e-10


def test_colinearity_lorenz96_d64_sites(g):
    """SURVEY §8d config 4 at reduced T: Lorenz-96 d=64 Jacobians (oracle/systems_port,
    pinned by the lorenz96_d16 golden), colinearity(0.99, 12) — sites identical to the
    reference algorithm, states within f64 tolerance."""
    from oracle import systems_port as S

    f, df, x0, dt = S.lorenz96(64)
    leaves = S.spectrum_leaves(S.integrate_chain(f, df, x0, dt, burn_in=200, T=1200, seed=0))
    al, asg = G.log_sign(leaves)
    Vc, Sc, sites_ref = G.selective_chain(al, asg, G.colinearity_policy(0.99, 12), 256)
    assert sites_ref, "the workload must exercise resets"
    Vl, Vs, sites = g._selective_chain_core(al, asg, g.colinearity_policy(0.99, 12), 256)
    assert sites == sites_ref
    assert scaled_real_err(Vl, Vs, Vc, Sc).max() < 1e-9


def test_colinearity_predicate_and_reset_kats(g):
    """pkg/tests/test_lyapunov.py:164-215 on the device policy."""
    import math

    m = g.GoomMatrix.from_real(np.eye(3))
    assert g.colinearity_select(m, 0.1) is False
    assert g.colinearity_select(g.GoomMatrix.from_real(np.array([[1.0, 1.0], [2.0, 2.0]])), 0.999)
    th = math.radians(0.5)
    m = g.GoomMatrix.from_real(np.array([[1.0, math.cos(th)], [0.0, math.sin(th)]]))
    assert g.colinearity_select(m, 0.99) is True
    assert g.colinearity_select(m, 0.99999) is False
    assert g.colinearity_select(g.GoomMatrix.from_real(np.array([[1.0, 0.0], [0.0, 0.0]])), 0.5)
    assert g.colinearity_select(g.GoomMatrix.from_real(np.array([[1.0, -2.0], [1.0, -2.0]])), 0.99)
    z = load_golden("orthonormal_reset")
    out = g.orthonormal_reset(g.GoomMatrix(z["qlog"], z["qsign"])).to_real()
    want = G.to_real(z["rlog"], z["rsign"])
    np.testing.assert_allclose(out, want, atol=1e-6)
    np.testing.assert_allclose(out.T @ out, np.eye(4), atol=1e-5)
    huge = g.orthonormal_reset(g.GoomMatrix(z["hlog"], np.ones((2, 2)))).to_real()
    assert bool(np.isfinite(huge).all())
    with pytest.raises(ValueError):
        g.orthonormal_reset(g.GoomMatrix.from_real(np.array([[1.0, 1.0], [1.0, 1.0]])))


def test_appendix_c_callable_policy(g):
    """Appendix C worked example (test_scan.py:142-178) with host-callable select/reset."""
    z = load_golden("appendix_c")
    target = z["a1"] @ z["x0"]

    def select(m):
        real = m.to_real()
        return real.shape == target.shape and np.allclose(real, target, rtol=1e-5)

    def reset(m):
        x = m.to_real()
        return g.GoomMatrix.from_real(x / (1.0 + np.linalg.norm(x)))

    pol = g.ResetPolicy(select=select, reset=reset)
    leaves = [g.ScanPair(g.GoomMatrix.from_real(x), g.GoomMatrix.zeros(3, 3))
              for x in (z["x0"], z["a1"], z["a2"], z["a3"])]
    for block in (None, 1, 2, 3, 4):
        states, sites = g.scan_selective(leaves, pol, block_size=block)
        assert sites == [2]
        for i, key in ((1, "want1"), (2, "want2"), (3, "want3")):
            np.testing.assert_allclose(states[i].state.to_real(), z[key],
                                       rtol=1e-5, atol=1e-6)
        assert [s.reset_applied for s in states] == [False, False, True, True]


def test_never_firing_equals_affine(g):
    """test_scan.py:255-265: a never-firing selective scan equals the affine scan."""
    rng = np.random.default_rng(42)
    T, d = 200, 3
    A = cz(*G.log_sign(rng.standard_normal((T, d, d))))
    st = g._Stack(A, torch.full_like(A, complex(NEG_INF, 0.0)))
    aff = g._scan_affine_stack(st, 16)
    V, sites = g._selective_chain_core(A, g.never_policy(16), 16)
    assert sites == []
    assert torch.equal(V, aff.A)


def test_parenthesizations_length_six(g):
    rng = np.random.default_rng(47)
    mats = []
    for _ in range(6):
        q, _ = np.linalg.qr(rng.standard_normal((2, 2)))
        mats.append(np.exp(rng.normal(1.0, 0.2)) * q)
    al, as_ = G.log_sign(np.array(mats))
    want_states, want_sites = G.selective_sequential(
        G.Stack(al, as_, np.full_like(al, NEG_INF), np.ones_like(as_), np.zeros(6, bool)),
        G.norm_threshold_policy(1.0))
    for block in range(1, 7):
        V, sites = g._selective_chain_core(cz(al, as_), g.norm_threshold_policy(1.0), block)
        assert sites == want_sites
        gl, gs = to_np(V[-1:])
        wl, ws = want_states.state(5)
        assert scaled_real_err(gl, gs, wl[None], ws[None]).max() < 1e-5


@pytest.mark.parametrize("d,T,block", [(128, 100, 8), (256, 40, 16), (128, 33, 64)])
def test_chain_fused_scales_match_prepass_path(g, d, T, block):
    """The tcgen05 chain with scales emitted by the producing epilogues equals the same
    chain scanned with the pre-pass (SIMT backend), within float32 noise; also with a carry."""
    rng = np.random.default_rng(d + T)
    A = cz(*G.log_sign(rng.standard_normal((T, d, d)).astype(np.float32)))
    carry = cz(*G.log_sign(rng.standard_normal((d, d)).astype(np.float32)))
    for c in (None, carry):
        fused = g.scan_chain(A, block, c)
        prev = g._lib.set_backend(1)
        try:
            ref = g.scan_chain(A, block, c)
        finally:
            g._lib.set_backend(prev)
        fl, fs = to_np(fused)
        rl, rs = to_np(ref)
        # 3xTF32 vs FP32 SIMT differ by ~1e-6 per step; over T steps that accumulates
        assert scaled_real_err(fl, fs, rl, rs).max() < 1e-3
        assert np.isfinite(fl).all()


@pytest.mark.parametrize("d,T,block", [(3, 50, 4), (8, 1000, 32), (16, 300, 17), (32, 200, 64),
                                       (8, 5, 8)])
@pytest.mark.parametrize("c128", [False, True])
def test_warp_resident_small_chain_is_bitwise_the_blocked_tree(g, d, T, block, c128):
    """d <= 32 chains run on the warp-resident kernels (scan_small.cu); their A slot must be
    bitwise the generic multi-launch blocked tree (the affine engine's A slot)."""
    rng = np.random.default_rng(d * T)
    dt = torch.complex128 if c128 else torch.complex64
    A = g.join(*G.log_sign(rng.standard_normal((T, d, d))), dt)
    Bz = g.join(*G.log_sign(rng.standard_normal((T, d, 1))), dt)
    flags = torch.zeros(T, dtype=torch.uint8, device=A.device)
    small = g.scan_chain(A, block)
    generic, _, _ = torch.ops.goom.scan_affine(A, Bz, flags, block)
    assert torch.equal(small, generic)
    carry = g.join(*G.log_sign(rng.standard_normal((d, d))), dt)
    with_carry = g.scan_chain(A, block, carry)
    cl, cs = to_np(carry[None])
    al, as_ = to_np(A)
    want = G.scan_sequential(G.Stack(np.concatenate([cl, al]), np.concatenate([cs, as_]),
                                     np.full((T + 1, d, d), -np.inf), np.ones((T + 1, d, d)),
                                     np.zeros(T + 1, bool)))
    wl, ws = to_np(with_carry)
    assert scaled_real_err(wl, ws, want.alog[1:], want.asign[1:]).max() < (1e-9 if c128 else 5e-3)


def test_parallel_beats_sequential_on_wide_chain(g):
    """test_scan.py:340-360: 2^15 leaves of 8x8 through the pair API, parallel (block 256)
    vs the sequential fold — same last state to 1e-10, and at least 2x faster."""
    import time

    rng = np.random.default_rng(49)
    T, d = 2 ** 15, 8
    alog = rng.uniform(-1, 1, (T, d, d))
    asign = rng.choice([-1.0, 1.0], (T, d, d))
    stack = g._Stack.from_arrays(alog, asign, np.full((T, d, d), -np.inf), np.ones((T, d, d)))
    g.scan_parallel(stack, g.combine_affine, block_size=256)  # warm
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    seq = g._scan_affine_stack(stack, T)  # block >= T: the sequential fold (scan.py:217-225)
    torch.cuda.synchronize()
    t_seq = time.perf_counter() - t0
    t0 = time.perf_counter()
    par = g.scan_parallel(stack, g.combine_affine, block_size=256)
    torch.cuda.synchronize()
    t_par = time.perf_counter() - t0
    pl = par.A[-1].real.cpu().numpy()
    sl = seq.A[-1].real.cpu().numpy()
    assert G.rel_log_diff(pl, sl) < 1e-10
    assert t_seq / t_par >= 2.0, (t_seq, t_par)


# ---------------------------------------------------------------------------
# CTA-resident chain scan, 32 < d <= 64 (scan_cta.cu)


@pytest.mark.parametrize("d,T,block", [(64, 300, 16), (48, 97, 10), (33, 64, 64), (64, 1, 4),
                                       (40, 130, 128)])
def test_chain_cta_matches_float64_oracle(g, d, T, block):
    """The CTA-resident walks (phase 1 and the carry fold in shared memory, the carry
    applied once per block) vs the float64 oracle of the same tree, calibrated by the
    reference's own float32 runs (SURVEY §8c chain criterion)."""
    rng = np.random.default_rng(d * 1000 + T)
    mats = rng.standard_normal((T, d, d))
    al, as_ = G.log_sign(mats)
    out = g.scan_chain(cz(al, as_), block_size=block)
    gl, gs = to_np(out)
    want = G.chain_blocked(al, as_, block)
    l32, s32 = G.log_sign(mats.astype(np.float32))
    refs = [G.chain_blocked(l32, s32, block), G.chain_blocked(l32, s32, T)]
    r = chain_parity(gl, gs, al, as_, want, refs)
    assert r["ok"], (r["bad"], r["flips"], r["scaled_bad"])


def test_chain_cta_complex128_and_carry(g):
    """complex128 (FP64) walks vs the float64 oracle at 1e-10, with and without a carry."""
    d, T, block = 64, 80, 8
    rng = np.random.default_rng(77)
    al, as_ = G.log_sign(rng.standard_normal((T, d, d)))
    cl, cs = G.log_sign(rng.standard_normal((d, d)))
    A = g.join(al, as_, np.float64)
    out = torch.ops.goom.scan_chain(A, block, None)
    gl = out.real.cpu().numpy()
    want, wsign = G.chain_blocked(al, as_, block)
    assert G.rel_log_diff(gl, want) < 1e-10
    outc = torch.ops.goom.scan_chain(A, block, g.join(cl, cs, np.float64))
    wl, _ = G.lmme(want, wsign, np.broadcast_to(cl, want.shape), np.broadcast_to(cs, want.shape))
    assert G.rel_log_diff(outc.real.cpu().numpy(), wl) < 1e-9


def test_chain_cta_bitwise_equals_batched_launches(g):
    """Same products, same arithmetic (lmme_whole_kernel's): the CTA-resident engine is
    bitwise equal to the batched per-step launches (GOOM_CHAIN_CTA=0), complex64 and
    complex128, with and without a carry."""
    import os
    import subprocess
    import sys

    code = (
        "import sys, numpy as np, torch; sys.path.insert(0, '.');"
        "import paper_2510_03426_b200 as g;"
        "rng = np.random.default_rng(5); outs = [];\n"
        "for d, T, blk, dt in ((64, 200, 16, np.float32), (48, 77, 9, np.float32),"
        " (64, 50, 8, np.float64)):\n"
        "    x = rng.standard_normal((T, d, d)); c = rng.standard_normal((d, d))\n"
        "    A = torch.ops.goom.from_real(torch.tensor(x).cuda(), float('-inf'), dt == np.float64)\n"
        "    C = torch.ops.goom.from_real(torch.tensor(c).cuda(), float('-inf'), dt == np.float64)\n"
        "    outs += [torch.view_as_real(torch.ops.goom.scan_chain(A, blk, None)).cpu(),"
        " torch.view_as_real(torch.ops.goom.scan_chain(A, blk, C)).cpu()]\n"
        "torch.save(outs, sys.argv[1])")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    res = []
    for flag in ("0", "1"):
        path = os.path.join(root, "gpurun_out", f"_cta_{flag}.pt")
        os.makedirs(os.path.dirname(path), exist_ok=True)
        env = dict(os.environ, GOOM_CHAIN_CTA=flag)
        subprocess.run([sys.executable, "-c", code, path], cwd=root, env=env, check=True,
                       timeout=300)
        res.append(torch.load(path))
        os.remove(path)
    for a, b in zip(*res):
        assert torch.equal(a, b)
