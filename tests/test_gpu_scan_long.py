"""GPU parity of the long-chain small-d engine (scan_long.cu, torch.ops.goom.scan_chain_long)
against the float64 oracle and against the generic LMME, combine by combine.

The engine computes the same prefixes as _scan_affine_stack's A slot (scan.py:181-214)
with a different fixed tree (reduce-then-scan), so:
  * a single chain (T <= 32) is the sequential fold: bitwise the generic path with
    block >= T (scan.py:217-225) without a carry, and bitwise a loop of generic LMMEs
    P = A_t (x) P from the carry with one;
  * longer chains (one to three levels of recursion, ragged tails, carries) meet the
    SURVEY §8c chain criterion against the float64 sequential oracle, calibrated by the
    reference's own float32 runs (complex64), and the reference's float64 tolerance
    (complex128).
"""

import numpy as np
import pytest
import torch

from goom_testlib import chain_parity, load_golden, scaled_real_err, to_np
from oracle import gooms_port as G

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def g():
    import paper_2510_03426_b200 as goom

    goom._lib.load()
    return goom


def leaves(g, T, d, seed, dt=torch.complex64):
    rng = np.random.default_rng(seed)
    return g.join(*G.log_sign(rng.standard_normal((T, d, d))), dt)


@pytest.mark.parametrize("d", [1, 3, 8, 13, 16, 32])
@pytest.mark.parametrize("T", [1, 5, 32])
@pytest.mark.parametrize("c128", [False, True])
def test_single_chain_is_bitwise_the_sequential_fold(g, d, T, c128):
    dt = torch.complex128 if c128 else torch.complex64
    A = leaves(g, T, d, 7 * d + T, dt)
    got = torch.ops.goom.scan_chain_long(A, None)
    want = torch.ops.goom.scan_chain(A, T, None)  # block >= T: the sequential fold
    assert torch.equal(got, want)
    # with a carry: P_0 = A_0 (x) carry, P_t = A_t (x) P_{t-1}, one generic LMME per step
    carry = leaves(g, 1, d, 99, dt)[0]
    got = torch.ops.goom.scan_chain_long(A, carry)
    P = carry[None]
    for t in range(T):
        P = torch.ops.goom.lmme(A[t:t + 1], P)
        assert torch.equal(got[t], P[0]), t


@pytest.mark.parametrize("block", [1000])
def test_config1_chain_d8_T1000(g, block):
    """Config 1 (1,000 random-normal 8x8 leaves, golden from the reference) on the long-chain
    engine: two levels (chains of 64, then one of 16)."""
    z = load_golden("config1_chain")
    al, as_ = G.log_sign(z["mats"])
    out = torch.ops.goom.scan_chain_long(g.join(al, as_), None)
    gl, gs = to_np(out)
    r = chain_parity(gl, gs, al, as_, (z["seq_f64"][0], z["seq_f64"][1]),
                     [z["seq_f32"], z["par32_f32"]])
    assert r["ok"], (r["bad"], r["flips"], r["scaled_bad"])


@pytest.mark.parametrize("d,T", [(8, 5000), (16, 2100), (32, 1500), (5, 1100)])
def test_long_chain_matches_oracle_complex64(g, d, T):
    rng = np.random.default_rng(d * 1000 + T)
    x = rng.standard_normal((T, d, d))
    al, as_ = G.log_sign(x)
    out = torch.ops.goom.scan_chain_long(g.join(al, as_), None)
    gl, gs = to_np(out)
    want = G.chain_blocked(al, as_, T)           # float64 sequential fold (the oracle)
    l32, s32 = G.log_sign(x.astype(np.float32))
    refs = [G.chain_blocked(l32, s32, T), G.chain_blocked(l32, s32, 64)]
    # d = 16 / 32: the leaf level folds on tcgen05 (scan_long_tc.cu, 3xTF32: the truncating
    # FP32 accumulation's scaled-real floor); other d on the lane-group FP32 fold. The rel-log
    # floor is 2e-4 for every d: this engine's tree (chains of 64, their totals' scan) is not
    # the reference's, and at d = 8, T = 5000 one position of the FP32 lane-group fold lands
    # at 1.8e-4 where the reference's own sequential float32 run is at 9e-6
    from goom_testlib import TC_CHAIN_FLOOR, tc_chain_scaled_floor
    floor = tc_chain_scaled_floor(d, T) if d in (16, 32) else 1e-4
    r = chain_parity(gl, gs, al, as_, want, refs, scaled_floor=floor, floor=TC_CHAIN_FLOOR)
    assert r["ok"], (r["bad"], r["e_gpu"][r["bad"]], r["e_ref"][r["bad"]], r["flips"],
                     r["scaled_bad"])


@pytest.mark.parametrize("T", [64 * 4 + 1, 64 * 5, 64 * 17 - 1, 64 * 64 + 3])
@pytest.mark.parametrize("with_carry", [False, True])
def test_long_chain_upper_tree_boundaries(g, T, with_carry):
    """The upper levels (chains of 4 totals up to a top chain of <= 4, d <= 32): leaf-level
    chain counts just above / at the top size (5, 5), a ragged 17-chain level (two upper
    levels with a 1-total tail) and 65 chains (three upper levels), with and without a
    carry, against the float64 sequential oracle under the §8c criterion (d = 8, the
    lane-group fold). The calibration runs include the reference's float32 blocked scan with
    block 64: its carry products (A_127..A_64) (x) P_63 are this engine's leaf-level
    association, which at some seeds (T = 257: 4.4e-4 at position 129) loses far more than
    the sequential float32 fold does."""
    from goom_testlib import scaled_real_err

    d = 8
    rng = np.random.default_rng(T)
    x = rng.standard_normal((T + 1, d, d))
    al, as_ = G.log_sign(x)
    l32, s32 = G.log_sign(x.astype(np.float32))
    if with_carry:  # leaf 0 plays the carry: the chain checked is [carry, P_0 .. P_{T-1}]
        gl, gs = to_np(torch.ops.goom.scan_chain_long(g.join(al[1:], as_[1:]),
                                                      g.join(al[0], as_[0])))
        gl = np.concatenate([al[:1], gl])
        gs = np.concatenate([as_[:1], gs])
        # float32 block-64 run over the leaves, each prefix then (x) the carry
        bl, bs = G.chain_blocked(l32[1:], s32[1:], 64)
        cl, cs = G.lmme(bl, bs, np.broadcast_to(l32[0], bl.shape),
                        np.broadcast_to(s32[0], bl.shape))
        blk = [(np.concatenate([l32[:1], cl]), np.concatenate([s32[:1], cs]))]
    else:
        gl, gs = to_np(torch.ops.goom.scan_chain_long(g.join(al, as_), None))
        blk = [G.chain_blocked(l32, s32, 64)]
    want = G.chain_blocked(al, as_, T + 1)
    from goom_testlib import TC_CHAIN_FLOOR
    refs = [G.chain_blocked(l32, s32, T + 1)] + blk
    # scaled-real error (relative to the largest entry): bounded chain-wide by 4x the worst the
    # reference's float32 runs reach anywhere on this chain (~2e-4 at T = 257), since the
    # positions where float32 rounding peaks differ between associations; the rel-log
    # criterion stays per position
    ref_scaled = max(float(scaled_real_err(r_[0], r_[1], *want).max()) for r_ in refs)
    r = chain_parity(gl, gs, al, as_, want, refs, floor=TC_CHAIN_FLOOR,
                     scaled_floor=max(1e-4, 4.0 * ref_scaled))
    assert r["ok"], (r["bad"], r["flips"], r["scaled_bad"], r["scaled_max"], ref_scaled)


@pytest.mark.parametrize("d,T,with_carry", [(16, 4500, True), (32, 4500, False), (16, 65, False),
                                            (32, 130, True), (16, 200, False)])
def test_long_chain_tc_small_d_matches_oracle(g, d, T, with_carry):
    """d = 16 / 32 at the leaf level on tcgen05 (8 / 4 chains per block-diagonal MMA):
    partial tiles (chain counts not a multiple of the chains per tile), ragged tails, carries,
    against the float64 oracle by the §8c chain criterion."""
    from goom_testlib import TC_CHAIN_FLOOR, tc_chain_scaled_floor

    rng = np.random.default_rng(d * 7 + T)
    x = rng.standard_normal((T, d, d))
    al, as_ = G.log_sign(x)
    if with_carry:
        c = rng.standard_normal((d, d))
        cl, cs = G.log_sign(c)
        out = torch.ops.goom.scan_chain_long(g.join(al, as_), g.join(cl, cs))
        wl, ws = G.chain_blocked(np.concatenate([cl[None], al]), np.concatenate([cs[None], as_]),
                                 T + 1)
        want = (wl[1:], ws[1:])
        l32, s32 = G.log_sign(np.concatenate([c[None], x]).astype(np.float32))
        refs = [tuple(v[1:] for v in G.chain_blocked(l32, s32, T + 1))]
    else:
        out = torch.ops.goom.scan_chain_long(g.join(al, as_), None)
        want = G.chain_blocked(al, as_, T)
        l32, s32 = G.log_sign(x.astype(np.float32))
        refs = [G.chain_blocked(l32, s32, T), G.chain_blocked(l32, s32, 64)]
    gl, gs = to_np(out)
    r = chain_parity(gl, gs, al, as_, want, refs, scaled_floor=tc_chain_scaled_floor(d, T),
                     floor=TC_CHAIN_FLOOR)
    assert r["ok"], (r["bad"], r["e_gpu"][r["bad"]], r["e_ref"][r["bad"]], r["flips"],
                     r["scaled_bad"], r["scaled_max"])


@pytest.mark.parametrize("d,T", [(4, 70000), (8, 3000), (32, 700)])
def test_long_chain_with_carry_complex128(g, d, T):
    """Three levels at T = 70,000 (chains of 64, 16, 16, then one of <= 32), ragged tails,
    and a carry: float64 tolerance of the reference (test_scan.py:227-237, 1e-10 order)."""
    rng = np.random.default_rng(d + T)
    x = rng.standard_normal((T, d, d))
    c = rng.standard_normal((d, d))
    al, as_ = G.log_sign(x)
    cl, cs = G.log_sign(c)
    out = torch.ops.goom.scan_chain_long(g.join(al, as_, torch.complex128),
                                         g.join(cl, cs, torch.complex128))
    gl, gs = to_np(out)
    wl, ws = G.chain_blocked(np.concatenate([cl[None], al]), np.concatenate([cs[None], as_]),
                             T + 1)
    wl, ws = wl[1:], ws[1:]
    assert G.rel_log_diff(gl, wl) < 1e-9
    assert scaled_real_err(gl, gs, wl, ws).max() < 1e-7  # 70,000 float64 steps, |log| ~ 4e4


def test_long_chain_underflow_and_zeros_follow_the_clamp(g):
    """A shrinking chain (0.5 I + 0.25 E_01 leaves: logs fall 0.69 per step, past float32's
    exp range) with exact zeros: the long engine's combines are the reference LMME's
    (clamped scales, core.py:252-253), so it keeps every value float32 can hold, underflows
    to -inf where the reference's own float32 fold does, and keeps the zero pattern."""
    d, T = 8, 300
    x = np.tile(0.5 * np.eye(d), (T, 1, 1))
    x[:, 0, 1] = 0.25
    al, as_ = G.log_sign(x)
    got = torch.ops.goom.scan_chain_long(g.join(al, as_), None)
    gl, gs = to_np(got)
    wl, ws = G.chain_blocked(al, as_, T)                       # float64 oracle
    rl, _ = G.chain_blocked(*G.log_sign(x.astype(np.float32)), T)  # the reference's float32
    assert not np.any(np.isnan(gl)) and not np.any(gl == np.inf)
    assert np.all(gl[wl == -np.inf] == -np.inf)                # exact zeros stay zero
    live = wl > -80.0                                          # normal float32 range
    assert np.all(np.isfinite(gl[live]))
    assert np.all(np.abs(gl[live] - wl[live]) <= 1e-4 * np.maximum(1.0, np.abs(wl[live])))
    assert np.array_equal(gs[live], ws[live])
    assert np.all(rl[-1] == -np.inf) and np.all(gl[-1] == -np.inf)  # both flushed at t = 299


@pytest.mark.parametrize("T,with_carry", [(1, True), (2, False), (63, False), (64, True),
                                          (65, False), (130, True), (700, False), (4500, True)])
def test_long_chain_d64_tcgen05_matches_oracle(g, T, with_carry):
    """d = 64 complex64 folds on tcgen05 (scan_long_tc.cu: two chains per MMA, 3xTF32): one to
    three levels of recursion (4,500 = 71 chains of 64 -> 5 of 16 -> one), an odd chain count
    (a pair with one chain missing), ragged tails, chains that start from their first leaf
    and from a carry, against the float64 oracle by the §8c chain criterion (scaled-real floor
    for the tensor core's truncating FP32 accumulation, goom_testlib.tc_chain_scaled_floor)."""
    from goom_testlib import TC_CHAIN_FLOOR, tc_chain_scaled_floor

    d = 64
    rng = np.random.default_rng(64 + T)
    x = rng.standard_normal((T, d, d))
    al, as_ = G.log_sign(x)
    if with_carry:
        c = rng.standard_normal((d, d))
        cl, cs = G.log_sign(c)
        out = torch.ops.goom.scan_chain_long(g.join(al, as_), g.join(cl, cs))
        xl, xs = np.concatenate([cl[None], al]), np.concatenate([cs[None], as_])
        wl, ws = G.chain_blocked(xl, xs, T + 1)
        want = (wl[1:], ws[1:])
        x32 = np.concatenate([c[None], x]).astype(np.float32)
        l32, s32 = G.log_sign(x32)
        refs = [tuple(v[1:] for v in G.chain_blocked(l32, s32, T + 1))]
    else:
        out = torch.ops.goom.scan_chain_long(g.join(al, as_), None)
        want = G.chain_blocked(al, as_, T)
        l32, s32 = G.log_sign(x.astype(np.float32))
        refs = [G.chain_blocked(l32, s32, T), G.chain_blocked(l32, s32, 64)]
    gl, gs = to_np(out)
    if not with_carry:  # the first prefix is the first leaf, raw
        assert np.array_equal(gl[0], al[0].astype(np.float32)) and np.array_equal(gs[0], as_[0])
    r = chain_parity(gl, gs, al, as_, want, refs, scaled_floor=tc_chain_scaled_floor(d, T),
                     floor=TC_CHAIN_FLOOR)
    assert r["ok"], (r["bad"], r["e_gpu"][r["bad"]], r["e_ref"][r["bad"]], r["flips"],
                     r["scaled_bad"], r["scaled_max"])


def test_long_chain_d64_underflow_and_zeros(g):
    """A shrinking d = 64 chain (0.5 I + 0.25 E_01 + a zero row in every leaf): Eq. 11's clamp
    (state scale max(., 0)) makes it underflow like the other tcgen05 paths (FTZ exp, ~e^-87),
    exact zeros stay zero, every value above the flush meets 1e-4, no NaN."""
    d, T = 64, 300
    x = np.tile(0.5 * np.eye(d), (T, 1, 1))
    x[:, 0, 1] = 0.25
    x[:, 5, :] = 0.0
    al, as_ = G.log_sign(x)
    gl, gs = to_np(torch.ops.goom.scan_chain_long(g.join(al, as_), None))
    wl, ws = G.chain_blocked(al, as_, T)
    assert not np.any(np.isnan(gl)) and not np.any(gl == np.inf)
    assert np.all(gl[wl == -np.inf] == -np.inf)
    live = wl > -80.0
    assert np.all(np.isfinite(gl[live]))
    assert np.all(np.abs(gl[live] - wl[live]) <= 1e-4 * np.maximum(1.0, np.abs(wl[live])))
    assert np.array_equal(gs[live], ws[live])
    assert np.all(gl[-1] == -np.inf)


def test_long_chain_validation(g):
    import paper_2510_03426_b200 as goom

    A = leaves(g, 4, 33, 0)
    with pytest.raises(goom._lib.GoomError, match="d <= 32"):
        torch.ops.goom.scan_chain_long(A, None)
    assert goom._lib.load().goom_scan_chain_long_workspace_size(10, 33) == 0
