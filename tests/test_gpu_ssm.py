"""GPU parity of the SSM forward pass against golden vectors the
reference produced (tests/golden/make_golden_ssm.py) and the reference's own test cases
(pkg/tests/test_ssm.py)."""

import math

import numpy as np
import pytest

from goom_testlib import load_golden

pytestmark = pytest.mark.gpu
NEG_INF = float("-inf")


@pytest.fixture(scope="module")
def s():
    import paper_2510_03426_b200 as goom
    from paper_2510_03426_b200 import ssm

    goom._lib.load()
    return ssm


def rel_log(x, y):
    both = (x == NEG_INF) & (y == NEG_INF)
    with np.errstate(invalid="ignore"):
        d = np.where(both, 0.0, np.abs(x - y) / np.maximum(1.0, np.abs(y)))
    return float(np.max(d))


@pytest.mark.parametrize("name", ["ssm_random_d4", "ssm_growing_d8", "ssm_explode_d8"])
def test_ssm_parallel_matches_reference(s, name):
    z = load_golden(name)
    p = s.SsmParams(z["A"], z["B"], z["C"], z["D"])
    run = s.ssm_forward_parallel(p, z["x0"], z["u"])
    assert rel_log(run.state_log, z["state_log"]) < 1e-10
    np.testing.assert_array_equal(run.state_sign, z["state_sign"])
    np.testing.assert_allclose(run.scales, z["scales"], rtol=1e-10, atol=0)
    np.testing.assert_allclose(run.y, z["y"], rtol=1e-7, atol=1e-9)
    assert np.isfinite(run.state_log).all() and np.isfinite(run.y).all()


def test_ssm_sequential_matches_parallel_and_reference(s):
    z = load_golden("ssm_random_d4")
    p = s.SsmParams(z["A"], z["B"], z["C"], z["D"])
    seq = s.ssm_forward_sequential(p, z["x0"], z["u"])
    par = s.ssm_forward_parallel(p, z["x0"], z["u"])
    assert rel_log(seq.state_log, z["seq_state_log"]) < 1e-10
    assert rel_log(par.state_log, seq.state_log) < 1e-8      # test_ssm.py:88-99
    np.testing.assert_array_equal(par.state_sign, seq.state_sign)
    np.testing.assert_allclose(par.y, seq.y, rtol=1e-7, atol=1e-9)


def test_ssm_small_systems(s):
    """test_ssm.py:41-84: memoryless, counter, zero-input systems; shape checks."""
    d = 3
    rng = np.random.default_rng(61)
    c = np.vstack([np.eye(d), np.zeros((d, d))])
    p = s.SsmParams(np.zeros((d, d)), np.eye(d), c, np.zeros((2 * d, d)))
    u = rng.standard_normal((16, d))
    run = s.ssm_forward_parallel(p, np.zeros(d), u)
    scaled = run.scaled_states()
    np.testing.assert_allclose(scaled * np.exp(run.scales[:, None] - 2.0), u, rtol=1e-12)
    np.testing.assert_allclose(run.y[:, :d], scaled, rtol=1e-12)
    p = s.SsmParams(np.eye(2), np.eye(2), np.vstack([np.eye(2), np.zeros((2, 2))]),
                    np.zeros((4, 2)))
    run = s.ssm_forward_sequential(p, np.zeros(2), np.tile([1.0, 0.0], (50, 1)))
    np.testing.assert_allclose(run.state_log[:, 0], np.log(np.arange(1, 51)), rtol=1e-12)
    assert np.all(run.state_log[:, 1] == NEG_INF)
    p = s.SsmParams(rng.standard_normal((3, 3)), rng.standard_normal((3, 3)),
                    rng.standard_normal((6, 3)), rng.standard_normal((6, 3)))
    run = s.ssm_forward_parallel(p, np.zeros(3), np.zeros((8, 3)))
    assert np.all(run.state_log == NEG_INF)
    np.testing.assert_array_equal(run.scales, np.zeros(8))
    np.testing.assert_array_equal(run.y, np.zeros((8, 6)))
    with pytest.raises(ValueError):
        s.SsmParams(np.eye(3), np.eye(2), np.ones((6, 3)), np.ones((6, 3)))
    with pytest.raises(ValueError):
        s.ssm_forward_parallel(p, np.zeros(2), np.zeros((4, 3)))
    with pytest.raises(ValueError):
        s.ssm_forward_parallel(p, np.zeros(3), np.zeros((0, 3)))


def test_ssm_batched_equals_per_sequence(s):
    """Sequences concatenated into one scan (each led by its (0, x0) leaf) give the same
    states as scanning them one by one."""
    rng = np.random.default_rng(5)
    d, T, S = 8, 100, 5
    p = s.SsmParams(rng.standard_normal((d, d)) * 0.4, rng.standard_normal((d, d)),
                    rng.standard_normal((2 * d, d)), rng.standard_normal((2 * d, d)))
    x0s = rng.standard_normal((S, d))
    us = rng.standard_normal((S, T, d))
    sl, ss, c, y = (t.cpu().numpy() for t in s.ssm_forward_batched(p, x0s, us, block_size=32,
                                                                    chunk=0))
    cl, cs, cc, cy = (t.cpu().numpy() for t in s.ssm_forward_batched(p, x0s, us, chunk=16))
    assert rel_log(cl, sl) < 1e-10
    np.testing.assert_array_equal(cs, ss)
    np.testing.assert_allclose(cy, y, rtol=1e-9, atol=1e-12)
    for i in range(S):
        one = s.ssm_forward_parallel(p, x0s[i], us[i], block_size=32)
        assert rel_log(sl[i], one.state_log) < 1e-10
        np.testing.assert_array_equal(ss[i], one.state_sign)
        np.testing.assert_allclose(y[i], one.y, rtol=1e-9, atol=1e-12)


def test_ssm_chunked_matches_reference_growth(s):
    """The chunked evaluation on the reference's growing-spectral-radius fixture (T = 512
    not a multiple of the chunk: padded steps)."""
    z = load_golden("ssm_growing_d8")
    p = s.SsmParams(z["A"], z["B"], z["C"], z["D"])
    sl, ss, c, y = (t.cpu().numpy() for t in s.ssm_forward_batched(p, z["x0"][None],
                                                                    z["u"][None], chunk=48))
    assert rel_log(sl[0], z["state_log"]) < 1e-10
    np.testing.assert_array_equal(ss[0], z["state_sign"])
    np.testing.assert_allclose(y[0], z["y"], rtol=1e-7, atol=1e-9)


def _rel_max(x, y):
    return float(np.max(np.abs(x - y)) / max(1e-300, float(np.max(np.abs(y)))))


@pytest.mark.parametrize("name", ["ssm_bwd_d4", "ssm_bwd_d8", "ssm_bwd_growing_d8"])
@pytest.mark.parametrize("chunk", [16, 64])
def test_ssm_backward_matches_autograd(s, name, chunk):
    """GPU adjoint vs torch float64 autograd of the reference's forward (golden)."""
    z = load_golden(name)
    p = s.SsmParams(z["A"], z["B"], z["C"], z["D"])
    run = s.ssm_forward_parallel(p, z["x0"], z["u"])
    g = s.ssm_backward(p, run, z["gy"], chunk=chunk)
    for k in ("A", "B", "C", "D", "x0", "u"):
        assert _rel_max(getattr(g, k), z["d" + k]) < 1e-9, k


def test_ssm_backward_past_float64_range_matches_oracle(s):
    """States beyond e^{800}: the adjoint lives below float64 range; GPU vs the oracle's
    log-domain restatement."""
    from oracle import gooms_port as G

    rng = np.random.default_rng(9)
    d, T = 8, 2100
    a = rng.standard_normal((d, d))
    a *= 1.5 / np.max(np.abs(np.linalg.eigvals(a)))
    p = s.SsmParams(a, rng.standard_normal((d, d)), rng.standard_normal((2 * d, d)),
                    rng.standard_normal((2 * d, d)))
    x0, u = rng.standard_normal(d), rng.standard_normal((T, d))
    gy = rng.standard_normal((T, 2 * d))
    run = s.ssm_forward_parallel(p, x0, u)
    assert run.scales.max() > 800.0
    g = s.ssm_backward(p, run, gy)
    r = G.ssm_backward(p.A, p.B, p.C, p.D, x0, u, run.state_log, run.state_sign, run.scales, gy)
    for k in ("A", "B", "C", "D", "x0", "u"):
        assert np.isfinite(getattr(g, k)).all(), k
        assert _rel_max(getattr(g, k), r[k]) < 1e-8, k


def test_ssm_heads_forward_backward_match_per_head(s):
    """Head-batched forward/backward (every launch covers all heads) equals the per-head
    single-sequence path; the autograd layer returns the same gradients."""
    import torch

    rng = np.random.default_rng(12)
    H, S, T, d = 3, 2, 70, 8
    A = rng.standard_normal((H, d, d)) * 0.4
    B, C, D = (rng.standard_normal((H, r, d)) for r in (d, 2 * d, 2 * d))
    x0s, us = rng.standard_normal((H, S, d)), rng.standard_normal((H, S, T, d))
    gy = rng.standard_normal((H, S, T, 2 * d))
    sl, ss, c, y = (t.cpu().numpy() for t in s.ssm_forward_heads(A, B, C, D, x0s, us, chunk=16))
    grads = [t.cpu().numpy() for t in s.ssm_backward_heads(A, B, C, D, x0s, us, sl, ss, c, gy,
                                                           chunk=16)]
    dA, dB, dC, dD, dx0, du = grads
    for h in range(H):
        p = s.SsmParams(A[h], B[h], C[h], D[h])
        acc = {k: 0.0 for k in "ABCD"}
        for i in range(S):
            run = s.ssm_forward_parallel(p, x0s[h, i], us[h, i], block_size=32)
            assert rel_log(sl[h, i], run.state_log) < 1e-10
            np.testing.assert_allclose(y[h, i], run.y, rtol=1e-9, atol=1e-12)
            g = s.ssm_backward(p, run, gy[h, i], chunk=32)
            for k in "ABCD":
                acc[k] = acc[k] + getattr(g, k)
            assert _rel_max(dx0[h, i], g.x0) < 1e-9
            assert _rel_max(du[h, i], g.u) < 1e-9
        for k, got in zip("ABCD", (dA, dB, dC, dD)):
            assert _rel_max(got[h], acc[k]) < 1e-9, k
    dev = torch.device("cuda")
    ts = [torch.tensor(v, dtype=torch.float64, device=dev, requires_grad=True)
          for v in (A, B, C, D, x0s, us)]
    out = s.ssm_layer(*ts, chunk=16)
    (out * torch.tensor(gy, device=dev)).sum().backward()
    for t, ref in zip(ts, grads):
        assert _rel_max(t.grad.cpu().numpy(), ref) < 1e-12


def test_ssm_matches_50_digit_recurrence_despite_growth(s):
    """test_ssm.py:114-131: spectral radius 1.5, T = 512: the scaled states match a 50-digit
    affine recurrence to 1e-9 at several steps while the states grow like 1.5^t."""
    mpmath = pytest.importorskip("mpmath")
    rng = np.random.default_rng(66)
    d, T = 8, 512
    a = rng.standard_normal((d, d))
    a *= 1.5 / np.max(np.abs(np.linalg.eigvals(a)))
    p = s.SsmParams(a, rng.standard_normal((d, d)), rng.standard_normal((2 * d, d)),
                    rng.standard_normal((2 * d, d)))
    x0 = rng.standard_normal(d)
    u = rng.standard_normal((T, d))
    run = s.ssm_forward_parallel(p, x0, u)
    with mpmath.workdps(50):
        A = [[mpmath.mpf(float(v)) for v in row] for row in p.A]
        bu = (p.B @ u.T).T
        x = [mpmath.mpf(float(v)) for v in x0]
        checks = {0, 1, 63, 255, 511}
        for t in range(T):
            x = [mpmath.fsum(A[i][k] * x[k] for k in range(d)) + mpmath.mpf(float(bu[t][i]))
                 for i in range(d)]
            if t in checks:
                ours = run.state_sign[t] * np.exp(run.state_log[t] - run.scales[t])
                sc = mpmath.exp(-mpmath.mpf(float(run.scales[t])))
                want = np.array([float(v * sc) for v in x])
                np.testing.assert_allclose(ours, want, rtol=1e-9)
    assert run.state_log[-1].max() > 512 * np.log(1.5) * 0.8


def test_ssm_scaled_state_bound(s):
    """test_ssm.py:155-163: every scaled state entry is at most e^2 and each state's max is e^2."""
    rng = np.random.default_rng(68)
    d = 4
    a = rng.standard_normal((d, d))
    a *= 1.8 / np.max(np.abs(np.linalg.eigvals(a)))
    p = s.SsmParams(a, rng.standard_normal((d, d)), rng.standard_normal((2 * d, d)),
                    rng.standard_normal((2 * d, d)))
    run = s.ssm_forward_parallel(p, rng.standard_normal(d), rng.standard_normal((300, d)))
    scaled = run.scaled_states()
    e2 = np.exp(2.0)
    assert np.all(np.abs(scaled) <= e2 * (1 + 1e-12))
    np.testing.assert_allclose(np.max(np.abs(scaled), axis=1), e2)


@pytest.mark.parametrize("T", [1, 2])
def test_ssm_backward_shortest_chains(s, T):
    """T = 1 / 2: the x_{-1} = x0 term of dA alone / with one more step, vs the oracle."""
    from oracle import gooms_port as G

    rng = np.random.default_rng(70 + T)
    d = 4
    p = s.SsmParams(rng.standard_normal((d, d)), rng.standard_normal((d, d)),
                    rng.standard_normal((2 * d, d)), rng.standard_normal((2 * d, d)))
    x0, u = rng.standard_normal(d), rng.standard_normal((T, d))
    gy = rng.standard_normal((T, 2 * d))
    run = s.ssm_forward_parallel(p, x0, u)
    g = s.ssm_backward(p, run, gy, chunk=16)
    r = G.ssm_backward(p.A, p.B, p.C, p.D, x0, u, run.state_log, run.state_sign, run.scales, gy)
    for k in ("A", "B", "C", "D", "x0", "u"):
        assert _rel_max(getattr(g, k), r[k]) < 1e-10, k


def test_ssm_bu_panel_layout_bitwise_equals_permuted_path(s):
    """T % chunk == 0: B u is produced straight in the chunked scan's panel layout
    (_bu_panels, one LMME of batch H L, bias read at its batch stride); the states are
    bitwise those of the (H, S, T, d) B u permuted into panels."""
    import torch

    rng = np.random.default_rng(21)
    H, S, T, d, L = 3, 5, 96, 8, 16
    dev = torch.device("cuda")
    A = torch.tensor(rng.standard_normal((H, d, d)) * 0.5, device=dev)
    B = torch.tensor(rng.standard_normal((H, d, d)), device=dev)
    x0 = torch.tensor(rng.standard_normal((H, S, d)), device=dev)
    u = torch.tensor(rng.standard_normal((H, S, T, d)), device=dev)
    bi = s._bu_panels(B, u, L)
    bu = s._bu_heads(B, u)
    ref_bi = bu.reshape(H, S, T // L, L, d).permute(3, 0, 4, 1, 2).reshape(L, H, d, S * T // L)
    assert torch.equal(torch.view_as_real(bi), torch.view_as_real(ref_bi))
    got = s._chunked_scan(s._goom(A), u.new_empty(()).expand(H, S, T, d), s._goom(x0), L, bi=bi)
    ref = s._chunked_scan(s._goom(A), bu, s._goom(x0), L)
    assert torch.equal(torch.view_as_real(got), torch.view_as_real(ref))
    Cm, Dm = rng.standard_normal((H, 2 * d, d)), rng.standard_normal((H, 2 * d, d))
    sl, ss, c, y = s.ssm_forward_heads(A.cpu().numpy(), B.cpu().numpy(), Cm, Dm,
                                       x0.cpu().numpy(), u.cpu().numpy(), chunk=L)
    # the fused export (goom_ssm_export_c128) against the permuted states through torch
    rss = s._sign_of(ref)
    rc = s._scales(ref.real)
    rz = rss * torch.exp(ref.real - rc[..., None] + 2.0)
    assert torch.equal(sl, ref.real) and torch.equal(ss, rss) and torch.equal(c, rc)
    Ct, Dt = torch.tensor(Cm, device=dev), torch.tensor(Dm, device=dev)
    ry = (torch.bmm(rz.reshape(H, S * T, d), Ct.transpose(1, 2)) +
          torch.bmm(u.reshape(H, S * T, d), Dt.transpose(1, 2))).reshape(H, S, T, 2 * d)
    assert torch.equal(y, ry)


def test_ssm_adjoint_panels_export_bitwise(s):
    """The backward's panel kernels (goom_ssm_panels_c128 in, reversed goom_ssm_export_c128
    out) against the flipped / permuted torch path they replace: bitwise equal adjoints."""
    import torch
    from paper_2510_03426_b200 import ops

    rng = np.random.default_rng(23)
    H, S, T, d, L = 2, 3, 48, 8, 16
    dev = torch.device("cuda")
    h = torch.tensor(rng.standard_normal((H, S, T, d)), device=dev)
    h[0, 1, 5] = 0.0
    c = torch.tensor(rng.standard_normal((H, S, T)) * 40, device=dev)
    K = c.max(dim=-1).values
    At = s._goom(torch.tensor(rng.standard_normal((H, d, d)) * 0.4, device=dev))
    zero = torch.full((H, S, d), complex(float("-inf"), 0.0), dtype=torch.complex128, device=dev)
    g = s._goom(h)
    g = torch.complex(g.real + (K[..., None] - c)[..., None], g.imag)
    ref_bi = g.flip(2).reshape(H, S, T // L, L, d).permute(3, 0, 4, 1, 2).reshape(L, H, d, -1)
    bi = ops.ssm_panels(h, L, K, c, reverse=True)
    assert torch.equal(torch.view_as_real(bi), torch.view_as_real(ref_bi))
    lam = s._chunked_scan(At, g.flip(2), zero, L).flip(2)
    X, L2, nC = s._chunked_scan(At, h.new_empty(()).expand(H, S, T, d), zero, L, bi=bi,
                                panels=True)
    ll, ls = ops.ssm_export(X, H, L2, S, nC, T, full=False, reverse=True, kshift=K)
    assert torch.equal(ll, lam.real - K[..., None, None])
    assert torch.equal(ls, s._sign_of(lam))


def test_ssm_chunked_contractive_powers_keep_the_carry(s):
    """the Hillis-Steele chunk carry squares A^L up to A^(L nC / 2). With a
    contractive A (spectral radius ~0.6) those powers fall below e^-745 long before the
    states do when x0 is large and the inputs are zero: x_t = A^t x0 stays representable
    (e^{690 - 0.51 t} at t ~ 2048), and the chunked evaluation must keep the
    A^(L off) (x) s term (max-normalised powers) — compared with the per-step sequential
    recurrence (ssm.py:99-108)."""
    rng = np.random.default_rng(31)
    H, S, T, d, L = 1, 2, 4096, 8, 64
    A = rng.standard_normal((d, d))
    A *= 0.6 / np.max(np.abs(np.linalg.eigvals(A)))
    B, C, D = rng.standard_normal((d, d)), rng.standard_normal((2 * d, d)), rng.standard_normal(
        (2 * d, d))
    x0s = rng.standard_normal((H, S, d)) * 1e300
    us = np.zeros((H, S, T, d))
    sl, ss, c, y = (t.cpu().numpy() for t in s.ssm_forward_heads(A[None], B[None], C[None],
                                                                    D[None], x0s, us, chunk=L))
    p = s.SsmParams(A, B, C, D)
    for i in range(S):
        seq = s.ssm_forward_sequential(p, x0s[0, i], us[0, i])
        # states the reference's float64 interior holds as normal numbers: below e^-708 its
        # exp() of the right operand is subnormal (precision lost digit by digit, flushed at
        # e^-745) and any evaluation order — its own parallel scan included — differs there
        normal = seq.state_log > -700.0
        assert normal[2000:].any()  # the states after chunk 31 are representable
        assert np.all(np.isfinite(sl[0, i][normal]))
        assert rel_log(np.where(normal, sl[0, i], 0.0), np.where(normal, seq.state_log, 0.0)) < 1e-9


def test_ssm_heads_past_grid_y_limit(s):
    """H * L > 65535 (head, step) rows: the panel / export kernels launch in grid.y slices
     instead of refusing; heads on both sides of the slice boundary match the
    per-head single-sequence path, forward and backward."""
    rng = np.random.default_rng(65536)
    H, S, T, d, L = 2100, 1, 64, 2, 32  # H * L = 67200
    A = rng.standard_normal((H, d, d)) * 0.5
    B, C, D = (rng.standard_normal((H, r, d)) for r in (d, 2 * d, 2 * d))
    x0s, us = rng.standard_normal((H, S, d)), rng.standard_normal((H, S, T, d))
    gy = rng.standard_normal((H, S, T, 2 * d))
    sl, ss, c, y = (t.cpu().numpy() for t in s.ssm_forward_heads(A, B, C, D, x0s, us, chunk=L))
    grads = [t.cpu().numpy() for t in s.ssm_backward_heads(A, B, C, D, x0s, us, sl, ss, c, gy,
                                                           chunk=L)]
    for h in (0, 2047, 2048, H - 1):  # rows h L + i on both sides of 65535
        p = s.SsmParams(A[h], B[h], C[h], D[h])
        run = s.ssm_forward_parallel(p, x0s[h, 0], us[h, 0], block_size=32)
        assert rel_log(sl[h, 0], run.state_log) < 1e-10
        np.testing.assert_allclose(y[h, 0], run.y, rtol=1e-9, atol=1e-12)
        g = s.ssm_backward(p, run, gy[h, 0], chunk=32)
        for k, got in zip("ABCD", grads[:4]):
            assert _rel_max(got[h], getattr(g, k)) < 1e-9, (h, k)
        assert _rel_max(grads[5][h, 0], g.u) < 1e-9


def test_ssm_adjoint_source_kernel_matches_torch_reference(s):
    """goom_ssm_adjoint_source_f64 against the torch formulation it replaces (ssm.py:84-98's
    export, differentiated): z = ss e^{sl - c + 2}, h = e^2 gz minus ss[i*] sum(gz z) at the
    first argmax i*; with an all-zero state (sl = -inf: no correction), ties for the maximum
    (the first index takes it) and d < 32 / d = 64."""
    import torch

    from paper_2510_03426_b200 import ops

    for d in (7, 64):
        torch.manual_seed(d)
        n = 1000
        sl = torch.randn(n, d, dtype=torch.float64, device="cuda") * 5
        ss = torch.where(torch.rand(n, d, device="cuda") < 0.5, -1.0, 1.0).to(torch.float64)
        gz = torch.randn(n, d, dtype=torch.float64, device="cuda")
        sl[3] = float("-inf")
        sl[5, 1] = sl[5, 4] = sl[5].max() + 1.0  # a tie: index 1 wins
        c = sl.max(dim=-1).values
        c = torch.where(c == float("-inf"), torch.zeros_like(c), c)
        h, z = ops.ssm_adjoint_source(sl, ss, c, gz)
        zr = ss * torch.exp(sl - c[:, None] + 2.0)
        hr = math.exp(2.0) * gz
        live = sl.max(dim=-1).values != float("-inf")
        istar = sl.argmax(dim=-1, keepdim=True)
        corr = torch.gather(ss, -1, istar) * (gz * zr).sum(-1, keepdim=True)
        hr = hr.scatter_add(-1, istar, -corr * live[:, None].to(hr.dtype))
        assert torch.equal(z, zr)
        torch.testing.assert_close(h, hr, rtol=1e-13, atol=1e-13)
        assert torch.equal(h[3], math.exp(2.0) * gz[3])
        assert h[5, 1] != math.exp(2.0) * gz[5, 1] and h[5, 4] == math.exp(2.0) * gz[5, 4]
