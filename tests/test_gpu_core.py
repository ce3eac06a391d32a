"""GPU parity of the goom-core kernels against the oracle and reference golden vectors.

Mirrors pkg/tests/test_core.py (TestLmme, TestColumnNormalization,
TestToRealScaled, TestRandomizedProperties) at complex64 tolerances: the
reference pins float64 to 1e-12; the B200 path computes in float32 (complex64
GOOMs, as the north star specifies), pinned to the §8c criterion instead.
"""

import math

import numpy as np
import pytest
import torch

from goom_testlib import NEG_INF, lmme_parity, load_golden, to_np
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


@pytest.fixture(params=[0, 1, 2], ids=["auto", "simt", "tc"])
def backend(request, g):
    prev = g._lib.set_backend(request.param)
    yield request.param
    g._lib.set_backend(prev)


# ---------------------------------------------------------------------------
# LMME


def test_lmme_two_by_two(g):
    z = load_golden("lmme_2x2")
    out = torch.ops.goom.lmme(cz(z["alog"], z["asign"]), cz(z["blog"], z["bsign"]))
    real = torch.ops.goom.to_real(out, True).cpu().numpy()
    np.testing.assert_allclose(real, [[19, 22], [43, 50]], rtol=2e-6)


@pytest.mark.parametrize("tag", ["f64", "f32"])
def test_lmme_64_against_golden(g, tag):
    z = load_golden(f"lmme_64_{tag}")
    out = torch.ops.goom.lmme(cz(z["alog"], z["asign"]), cz(z["blog"], z["bsign"]))
    gl, gs = to_np(out)
    err, flips = lmme_parity((gl, gs), z["alog"].astype(np.float32), z["asign"],
                             z["blog"].astype(np.float32), z["bsign"])
    assert err < 1e-4 and flips == 0
    # normalized Frobenius error of the real product (test_core.py:196-203, f32 bound of :238-249)
    want = G.to_real(z["olog"].astype(np.float64), z["osign"])
    got = gs * np.exp(gl)
    assert np.linalg.norm(got - want) / np.linalg.norm(want) < 1e-5


def test_lmme_batched_rectangular_edge_cases(g):
    z = load_golden("lmme_batched_f32")
    out = torch.ops.goom.lmme(cz(z["alog"], z["asign"]), cz(z["blog"], z["bsign"]))
    gl, gs = to_np(out)
    wl, ws = z["olog"].astype(np.float64), z["osign"]
    # all-zero row / column -> (-inf, +1) exactly (test_core.py:220-227)
    assert np.all(gl[0, 1] == NEG_INF) and np.all(gs[0, 1] == 1.0)
    assert np.all(gl[2, :, 0] == NEG_INF)
    # the clamp regime (scales max(., 0)) reproduces the reference's float32 values
    assert np.array_equal(gl == NEG_INF, wl == NEG_INF)
    finite = wl != NEG_INF
    assert np.max(np.abs(gl[finite] - wl[finite]) / np.maximum(1, np.abs(wl[finite]))) < 1e-4
    # vs the float64 oracle where float32 does not underflow (item 4 is the clamp regime)
    keep = [i for i in range(gl.shape[0]) if i != 4]
    err, flips = lmme_parity((gl[keep], gs[keep]), z["alog"][keep], z["asign"][keep],
                             z["blog"][keep], z["bsign"][keep])
    assert err < 1e-4 and flips == 0


@pytest.mark.parametrize("d", [3, 8, 16, 32, 33, 64, 100, 128, 256, 512])
def test_lmme_square_sweep(g, d, backend):
    if backend == 2 and d % 128 and d > 32:
        pytest.skip("tcgen05 path tiles d % 128 == 0")
    rng = np.random.default_rng(1000 + d)
    batch = 6
    a = rng.standard_normal((batch, d, d)).astype(np.float32)
    b = rng.standard_normal((batch, d, d)).astype(np.float32)
    al, as_ = G.log_sign(a)
    bl, bs = G.log_sign(b)
    out = torch.ops.goom.lmme(cz(al, as_), cz(bl, bs))
    err, flips = lmme_parity(to_np(out), al, as_, bl, bs)
    assert err < 1e-4, err
    assert flips == 0


@pytest.mark.parametrize("n,k,m", [(5, 7, 3), (64, 64, 1), (128, 128, 1), (40, 70, 90),
                                   (256, 512, 128), (1, 33, 1)])
def test_lmme_rectangular(g, n, k, m):
    rng = np.random.default_rng(n * 7 + k * 3 + m)
    al, as_ = G.log_sign(rng.standard_normal((3, n, k)).astype(np.float32))
    bl, bs = G.log_sign(rng.standard_normal((3, k, m)).astype(np.float32))
    out = torch.ops.goom.lmme(cz(al, as_), cz(bl, bs))
    assert tuple(out.shape) == (3, n, m)
    err, flips = lmme_parity(to_np(out), al, as_, bl, bs)
    assert err < 1e-4 and flips == 0


def test_lmme_broadcast_and_huge_logs(g):
    rng = np.random.default_rng(5)
    al = rng.uniform(-20, 20, (4, 16, 16)).astype(np.float32) + np.float32(1e6)
    as_ = rng.choice([-1.0, 1.0], al.shape).astype(np.float32)
    bl = rng.uniform(-20, 20, (16, 16)).astype(np.float32)
    bs = rng.choice([-1.0, 1.0], bl.shape).astype(np.float32)
    out = torch.ops.goom.lmme(cz(al, as_), cz(bl, bs))
    gl, gs = to_np(out)
    for i in range(4):
        err, flips = lmme_parity((gl[i], gs[i]), al[i], as_[i], bl, bs)
        assert err < 1e-4 and flips == 0
    assert np.all(np.isfinite(gl))


def test_lmme_identity_and_row_scaling(g):
    """test_core.py:175-182 / 350-382: identity left operand, row scaling invariance."""
    rng = np.random.default_rng(24)
    batch, d = 10000, 3  # the reference's 10^4-case sweep (test_core.py:350-382)
    # |log| <= 40 keeps every shifted exponential in float32's normal range
    logs = rng.uniform(-40, 40, (batch, d, d)).astype(np.float32)
    signs = rng.choice([-1.0, 1.0], (batch, d, d)).astype(np.float32)
    eye_l, eye_s = G.identity(d, np.float32)
    out = torch.ops.goom.lmme(cz(eye_l, eye_s), cz(logs, signs))
    gl, gs = to_np(out)
    # float32: (x - b) rounds at ulp(80)/2 ~ 4e-6 before the exp/log round trip
    assert np.max(np.abs(gl - logs) / np.maximum(1, np.abs(logs))) < 1e-5
    assert np.array_equal(gs, signs)
    shift = rng.uniform(0, 100, (batch, 1)).astype(np.float32)
    shifted = logs.copy()
    shifted[:, 0, :] += shift
    base = to_np(torch.ops.goom.lmme(cz(logs, signs), cz(logs, signs)))
    other = to_np(torch.ops.goom.lmme(cz(shifted, signs), cz(logs, signs)))
    ol = other[0].copy()
    ol[:, 0, :] -= shift
    mask = np.isfinite(base[0])
    assert np.max(np.abs(ol - base[0])[mask] / np.maximum(1, np.abs(base[0][mask]))) < 1e-4


def test_lmme_bitwise_repeatable(g, backend):
    rng = np.random.default_rng(12)
    d = 128
    a = cz(*G.log_sign(rng.standard_normal((4, d, d)).astype(np.float32)))
    b = cz(*G.log_sign(rng.standard_normal((4, d, d)).astype(np.float32)))
    o1 = torch.ops.goom.lmme(a, b)
    o2 = torch.ops.goom.lmme(a, b)
    assert torch.equal(o1, o2)


def test_lmme_dimension_mismatch(g):
    a = torch.zeros(2, 3, dtype=torch.complex64, device="cuda")
    b = torch.zeros(2, 2, dtype=torch.complex64, device="cuda")
    with pytest.raises(ValueError):
        torch.ops.goom.lmme(a, b)
    with pytest.raises(ValueError):
        g.lmme(g.GoomMatrix(a), g.GoomMatrix(b))


def test_lmme_gadd_fused(g):
    rng = np.random.default_rng(3)
    al, as_ = G.log_sign(rng.standard_normal((5, 8, 8)).astype(np.float32))
    bl, bs = G.log_sign(rng.standard_normal((5, 8, 2)).astype(np.float32))
    dl, ds = G.log_sign(rng.standard_normal((5, 8, 2)).astype(np.float32))
    fused = torch.ops.goom.lmme_gadd(cz(al, as_), cz(bl, bs), cz(dl, ds))
    two = torch.ops.goom.gadd(torch.ops.goom.lmme(cz(al, as_), cz(bl, bs)), cz(dl, ds))
    assert torch.equal(fused, two)


# ---------------------------------------------------------------------------
# gadd, conversions


@pytest.mark.parametrize("tag", ["f32", "f64"])
def test_gadd_golden_commutative_cancellation(g, tag):
    z = load_golden(f"gadd_{tag}")
    a = cz(z["alog"], z["asign"])
    b = cz(z["blog"], z["bsign"])
    ab = torch.ops.goom.gadd(a, b)
    ba = torch.ops.goom.gadd(b, a)
    assert torch.equal(ab, ba)  # bitwise commutative (test_core.py:327-338)
    gl, gs = to_np(ab)
    assert np.all(gl[:256] == NEG_INF) and np.all(gs[:256] == 1.0)  # exact cancellation
    wl, ws = z["olog"].astype(np.float64), z["osign"]
    fin = np.isfinite(wl)
    assert np.array_equal(np.isfinite(gl), fin)
    assert np.max(np.abs(gl[fin] - wl[fin]) / np.maximum(1, np.abs(wl[fin]))) < 1e-5
    assert np.array_equal(gs[fin], ws[fin])


@pytest.mark.parametrize("tag", ["f32", "f64"])
def test_from_real_golden(g, tag):
    z = load_golden(f"from_real_{tag}")
    x = torch.as_tensor(z["x"]).cuda()
    out = torch.ops.goom.from_real(x, NEG_INF, False)
    gl, gs = to_np(out)
    fin = np.isfinite(z["olog"])
    assert np.max(np.abs(gl[fin] - z["olog"][fin]) / np.maximum(1, np.abs(z["olog"][fin]))) < 1e-6
    assert np.array_equal(gs, z["osign"])
    assert np.all(gl[~fin] == NEG_INF)


def test_round_trip_and_overflow(g):
    rng = np.random.default_rng(20)
    xs = (rng.standard_normal(10_000) * np.exp(rng.uniform(-30, 30, 10_000))).astype(np.float32)
    xs[xs == 0] = 1.0
    m = g.GoomMatrix.from_real(xs.reshape(100, -1))
    back = m.to_real().ravel()
    # a complex64 GOOM holds log|x| to ulp(32)/2 ~ 1e-6 absolute -> ~1e-6 relative in x
    assert np.all(np.abs(back / xs - 1.0) < 5e-6)
    big = g.GoomMatrix(np.array([[800.0, 800.0]]), np.array([[1.0, -1.0]]))
    r = big.to_real()
    assert r[0, 0] == np.inf and r[0, 1] == -np.inf
    with pytest.raises(ValueError):
        g.GoomMatrix.from_real(np.array([[np.nan]]))
    with pytest.raises(ValueError):
        g.GoomMatrix.from_real(np.array([[np.inf]]))


def test_to_real_scaled_golden(g):
    z = load_golden("to_real_scaled")
    e2 = math.exp(2.0)
    for i in range(z["log"].shape[0]):
        m = g.GoomMatrix(z["log"][i].astype(np.float32), z["sign"][i])
        out, c = g.to_real_scaled(m)
        assert abs(c - z["c"][i]) <= 1e-3 * max(1.0, abs(z["c"][i]))
        assert np.max(np.abs(out)) <= e2 * (1 + 1e-6)
        np.testing.assert_allclose(out, z["out"][i], rtol=1e-3, atol=1e-6)
    zero = g.GoomMatrix.zeros(2, 2)
    out, c = g.to_real_scaled(zero)
    assert c == 0.0 and float(np.abs(out).max()) == 0.0


def test_column_normalization(g):
    z = load_golden("col_log_norms")
    out = g._col_log_norms(z["log"].astype(np.float32))
    np.testing.assert_allclose(out, z["out"], rtol=1e-6, atol=1e-4)
    m = g.GoomMatrix.from_real(np.array([[3.0], [4.0]]))
    out, nu = g.log_unit_norm_columns(m)
    np.testing.assert_allclose(out.to_real().ravel(), [0.6, 0.8], rtol=1e-6)
    assert abs(nu[0] - math.log(5.0)) < 1e-6
    with pytest.raises(ValueError):
        g.log_unit_norm_columns(g.GoomMatrix.zeros(2, 2))


def test_array_level_entry_points(g):
    """The private array entry points the reference's callers use."""
    rng = np.random.default_rng(7)
    al, as_ = G.log_sign(rng.standard_normal((4, 6, 6)))
    bl, bs = G.log_sign(rng.standard_normal((4, 6, 6)))
    ol, os_ = g._lmme_arrays(al, as_, bl, bs)
    assert isinstance(ol, np.ndarray) and ol.shape == (4, 6, 6)
    wl, ws = G.lmme(al, as_, bl, bs)
    assert G.rel_log_diff(ol, wl) < 1e-5
    gl, gs = g._gadd_arrays(al, as_, bl, bs)
    wl, ws = G.gadd(al, as_, bl, bs)
    assert G.rel_log_diff(gl, wl) < 1e-5
    x = rng.standard_normal((3, 3))
    ll, ls = g._log_sign_arrays(x)
    np.testing.assert_allclose(ll, np.log(np.abs(x)), rtol=1e-6)


# ---------------------------------------------------------------------------
# complex128 GOOMs: the reference's float64 tolerances


def test_lmme_complex128_reference_tolerances(g):
    """test_core.py:184-203 at float64 backing: 2x2 KAT rtol 1e-14, 64x64 vs the 50-digit
    oracle's float64 image <= 1e-12 normalized Frobenius error."""
    z = load_golden("lmme_2x2")
    c128 = torch.complex128
    out = torch.ops.goom.lmme(g.join(z["alog"], z["asign"], c128), g.join(z["blog"], z["bsign"], c128))
    np.testing.assert_allclose(torch.ops.goom.to_real(out, True).cpu().numpy(),
                               [[19, 22], [43, 50]], rtol=1e-14)
    z = load_golden("lmme_64_f64")
    out = torch.ops.goom.lmme(g.join(z["alog"], z["asign"], c128), g.join(z["blog"], z["bsign"], c128))
    gl, gs = to_np(out)
    want = G.to_real(z["olog"], z["osign"])
    got = gs * np.exp(gl)
    assert np.linalg.norm(got - want) / np.linalg.norm(want) < 1e-12
    assert G.rel_log_diff(gl, z["olog"]) < 1e-10


def test_gadd_and_conversions_complex128(g):
    z = load_golden("gadd_f64")
    a = g.join(z["alog"], z["asign"], torch.complex128)
    b = g.join(z["blog"], z["bsign"], torch.complex128)
    ab = torch.ops.goom.gadd(a, b)
    assert torch.equal(ab, torch.ops.goom.gadd(b, a))
    gl, gs = to_np(ab)
    fin = np.isfinite(z["olog"])
    assert np.array_equal(np.isfinite(gl), fin)
    assert np.max(np.abs(gl[fin] - z["olog"][fin]) / np.maximum(1, np.abs(z["olog"][fin]))) < 1e-14
    z = load_golden("from_real_f64")
    m = torch.ops.goom.from_real(torch.as_tensor(z["x"]).cuda(), NEG_INF, True)
    gl, gs = to_np(m)
    fin = np.isfinite(z["olog"])
    np.testing.assert_allclose(gl[fin], z["olog"][fin], rtol=1e-15, atol=1e-15)
    assert np.array_equal(gs, z["osign"])
    back = torch.ops.goom.to_real(m, True).cpu().numpy()
    nz = z["x"] != 0
    assert np.all(np.abs(back[nz] / z["x"][nz] - 1.0) < 1e-12)  # test_core.py:312-317


@pytest.mark.parametrize("d", [3, 16, 33, 64])
def test_lmme_complex128_sweep(g, d):
    rng = np.random.default_rng(77 + d)
    al, as_ = G.log_sign(rng.standard_normal((5, d, d)))
    bl, bs = G.log_sign(rng.standard_normal((5, d, d)))
    out = torch.ops.goom.lmme(g.join(al, as_, torch.complex128), g.join(bl, bs, torch.complex128))
    err, flips = lmme_parity(to_np(out), al, as_, bl, bs, tol=1e-12, kappa_min=1e-3)
    assert err < 1e-12 and flips == 0


@pytest.mark.parametrize("n,k,m", [(128, 32, 128), (256, 1024, 128), (128, 96, 384), (1024, 1024, 1024)])
def test_lmme_tcgen05_shapes(g, n, k, m):
    """The tcgen05 3xTF32 kernel on its tile grid, incl. K not a multiple of 128 and d = 1024
    (the error budget case of SURVEY §8a: 3xTF32 must match FP32, no sign flips)."""
    prev = g._lib.set_backend(2)
    try:
        rng = np.random.default_rng(n + 3 * k + 7 * m)
        batch = 2 if n * m * k <= 2 ** 24 else 1
        al, as_ = G.log_sign(rng.standard_normal((batch, n, k)).astype(np.float32))
        bl, bs = G.log_sign(rng.standard_normal((batch, k, m)).astype(np.float32))
        out = torch.ops.goom.lmme(cz(al, as_), cz(bl, bs))
        err, flips = lmme_parity(to_np(out), al, as_, bl, bs)
        assert err < 1e-4 and flips == 0
        # the single-LMME error budget of SURVEY §8a: normalised Frobenius error of the real
        # product vs float64 <= 1e-5 (pkg/tests/test_core.py:238-249's float32 bound)
        gl, gs = to_np(out)
        want = a64 = None
        for i in range(batch):
            want = al[i].astype(np.float64), as_[i], bl[i].astype(np.float64), bs[i]
            a64 = G.to_real(want[0], want[1]) @ G.to_real(want[2], want[3])
            got = gs[i] * np.exp(gl[i])
            assert np.linalg.norm(got - a64) / np.linalg.norm(a64) < 1e-5
    finally:
        g._lib.set_backend(prev)


def test_lmme_tcgen05_fused_gadd_and_broadcast(g):
    prev = g._lib.set_backend(2)
    try:
        rng = np.random.default_rng(11)
        al, as_ = G.log_sign(rng.standard_normal((3, 128, 128)).astype(np.float32))
        bl, bs = G.log_sign(rng.standard_normal((128, 256)).astype(np.float32))
        dl, ds = G.log_sign(rng.standard_normal((3, 128, 256)).astype(np.float32))
        fused = torch.ops.goom.lmme_gadd(cz(al, as_), cz(bl, bs), cz(dl, ds))
        plain = torch.ops.goom.lmme(cz(al, as_), cz(bl, bs))
        two = torch.ops.goom.gadd(plain, cz(dl, ds))
        assert torch.equal(fused, two)
        for i in range(3):
            err, flips = lmme_parity(to_np(plain[i]), al[i], as_[i], bl, bs)
            assert err < 1e-4 and flips == 0
    finally:
        g._lib.set_backend(prev)


@pytest.mark.parametrize("n,k,m", [(64, 64, 64), (48, 40, 56), (33, 64, 7)])
def test_lmme_whole_kernel_bitwise_equals_prepass_path(g, n, k, m):
    """n, k, m <= 64 take the one-CTA-per-product kernel with the row / column maxima fused;
    it must be bitwise equal to the pre-pass + tiled path (goom_lmme_scaled_c64 with the
    clamped maxima computed here), which the golden tests pin against the reference."""
    import ctypes

    torch.manual_seed(n * 10000 + k * 100 + m)
    batch = 37
    A = torch.ops.goom.from_real(torch.randn(batch, n, k, device="cuda") * 3, float("-inf"), False)
    B = torch.ops.goom.from_real(torch.randn(batch, k, m, device="cuda") * 3, float("-inf"), False)
    A[0, 1, :] = torch.complex(torch.tensor(float("-inf")), torch.tensor(0.0))  # a zero row
    lib = g._lib.load()
    lib.goom_set_lmme_backend(1)  # the SIMT kernel (n = m = k = 64 otherwise runs on tcgen05)
    try:
        got = torch.ops.goom.lmme(A, B)
    finally:
        lib.goom_set_lmme_backend(0)
    ra = A.real.amax(dim=2).clamp_min(0).contiguous()
    cb = B.real.amax(dim=1).clamp_min(0).contiguous()
    ref = torch.empty_like(got)
    lib = g._lib.load()
    g._lib.check(lib.goom_lmme_scaled_c64(
        g._lib.goom_operand(A.data_ptr(), n * k, 1), ra.data_ptr(), n,
        g._lib.goom_operand(B.data_ptr(), k * m, 1), cb.data_ptr(), m, ref.data_ptr(), n * m,
        batch, n, k, m, ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)))
    torch.cuda.synchronize()
    assert torch.equal(torch.view_as_real(got), torch.view_as_real(ref))


def test_lmme_64_vector_kernel_gadd_and_unaligned(g):
    """The 16-byte-vector d = 64 kernel (aligned operands) against the generic whole kernel
    (the same products read from storage shifted by one complex64, which is not 16-byte
    aligned): bitwise equal, with and without the fused bias gadd, and with a broadcast
    (stride 0) right operand."""
    torch.manual_seed(64)
    batch = 41
    A = torch.ops.goom.from_real(torch.randn(batch, 64, 64, device="cuda") * 3, float("-inf"), False)
    B = torch.ops.goom.from_real(torch.randn(batch, 64, 64, device="cuda") * 3, float("-inf"), False)
    D = torch.ops.goom.from_real(torch.randn(batch, 64, 64, device="cuda") * 50, float("-inf"), False)
    A[3, :, 5] = torch.complex(torch.tensor(float("-inf")), torch.tensor(0.0))

    def shifted(x):
        buf = torch.empty(x.numel() + 1, dtype=x.dtype, device=x.device)
        v = buf[1:].view(x.shape)
        v.copy_(x)
        assert v.data_ptr() % 16 == 8
        return v

    As, Bs, Ds = shifted(A), shifted(B), shifted(D)
    eq = lambda x, y: torch.equal(torch.view_as_real(x), torch.view_as_real(y))
    lib = g._lib.load()
    lib.goom_set_lmme_backend(1)  # the SIMT kernels (aligned d = 64 otherwise runs on tcgen05)
    try:
        assert eq(torch.ops.goom.lmme(A, B), torch.ops.goom.lmme(As, Bs))
        assert eq(torch.ops.goom.lmme_gadd(A, B, D), torch.ops.goom.lmme_gadd(As, Bs, Ds))
        assert eq(torch.ops.goom.lmme_gadd(A, B, D),
                  torch.ops.goom.gadd(torch.ops.goom.lmme(A, B), D))
        b0 = B[:1].expand(batch, 64, 64)
        assert eq(torch.ops.goom.lmme(A, b0),
                  torch.ops.goom.lmme(As, shifted(B[:1]).expand(batch, 64, 64)))
    finally:
        lib.goom_set_lmme_backend(0)


def test_lmme_64x64_against_50_digit_reference(g):
    """test_core.py:196-203 with its 50-digit oracle (mpmath): complex128 LMME of two
    64x64 N(0,1) matrices, Frobenius relative error < 1e-12; complex64 (3xTF32) < 1e-6."""
    mpmath = pytest.importorskip("mpmath")
    rng = np.random.default_rng(8)
    a = rng.standard_normal((64, 64))
    b = rng.standard_normal((64, 64))
    with mpmath.workdps(50):
        A = [[mpmath.mpf(float(x)) for x in row] for row in a]
        B = [[mpmath.mpf(float(x)) for x in row] for row in b]
        want = np.array([[float(mpmath.fsum(A[i][k] * B[k][j] for k in range(64)))
                          for j in range(64)] for i in range(64)])
    for dt, tol in ((torch.complex128, 1e-12), (torch.complex64, 1e-6)):
        al, as_ = G.log_sign(a)
        bl, bs = G.log_sign(b)
        out = torch.ops.goom.lmme(g.join(al, as_, dt), g.join(bl, bs, dt))
        gl, gs = to_np(out)
        got = gs * np.exp(gl.astype(np.float64))
        err = np.linalg.norm(got - want) / np.linalg.norm(want)
        assert err < tol, (dt, err)


def test_column_norms_and_scaled_export_reference_cases(g):
    """test_core.py:258-311 (log_unit_norm_columns, to_real_scaled) and the 10^4 float64
    round trip (test_core.py:318-323), on float64-backed GoomMatrix (the reference's default
    backing, complex128 here too)."""
    m = g.GoomMatrix.from_real(np.array([[1.0], [0.0]]), dtype=np.float64)
    out, nu = g.log_unit_norm_columns(m)
    assert abs(nu[0]) < 1e-14
    np.testing.assert_allclose(out.to_real().ravel(), [1.0, 0.0])
    m = g.GoomMatrix(np.full((2, 1), 1000.0), np.ones((2, 1)), dtype=np.float64)
    out, _ = g.log_unit_norm_columns(m)
    np.testing.assert_allclose(out.to_real().ravel(), [0.70710678, 0.70710678],
                               rtol=1e-7)
    rng = np.random.default_rng(14)
    m = g.GoomMatrix(rng.uniform(-500, 500, (6, 6)), rng.choice([-1.0, 1.0], (6, 6)),
                     dtype=np.float64)
    out, _ = g.log_unit_norm_columns(m)
    norms = np.log(np.linalg.norm(out.to_real(), axis=0))
    assert np.max(np.abs(norms)) < 1e-10
    out, c = g.to_real_scaled(g.GoomMatrix(np.full((3, 3), 1e6), np.ones((3, 3)),
                                           dtype=np.float64))
    assert c == 1e6
    np.testing.assert_array_equal(out, np.full((3, 3), np.exp(2.0)))
    out, c = g.to_real_scaled(g.GoomMatrix.from_real(np.array([[1.0]]), dtype=np.float64))
    assert c == 0.0 and float(out[0, 0]) == np.exp(2.0)
    rng = np.random.default_rng(15)
    m = g.GoomMatrix(rng.uniform(-1e8, 1e8, (4, 4)), rng.choice([-1.0, 1.0], (4, 4)),
                     dtype=np.float64)
    out, c = g.to_real_scaled(m)
    o = np.abs(out)
    assert o.max() == np.exp(2.0) and np.all(o <= np.exp(2.0))
    rng = np.random.default_rng(20)
    xs = rng.standard_normal(10_000) * np.exp(rng.uniform(-200, 200, 10_000))
    xs = np.where(xs == 0, 1.0, xs)
    back = g.GoomMatrix.from_real(xs.reshape(100, -1), dtype=np.float64).to_real()
    back = back.ravel()
    assert np.all(np.abs(back / xs - 1.0) < 1e-12)


@pytest.mark.parametrize("shape,bcast,bias", [
    ((256, 256, 256), False, False), ((256, 256, 256), True, False),
    ((128, 128, 128), False, False), ((128, 128, 128), True, False),
    ((128, 64, 128), False, True), ((128, 512, 128), False, False),
    ((128, 128, 128), False, True),
    ((64, 64, 64), False, False), ((64, 64, 64), True, False), ((64, 128, 64), False, True)])
def test_lmme_fused_scales_bitwise_equals_scaled_path(g, shape, bcast, bias):
    """The config-2 HBM-bound shapes reduce Eq. 11's clamped row / column maxima in-kernel (no
    pre-pass): n = m = 256 in the pair kernel (lmme_tc2.cu kFuse), n = m = 128 through the
    one-SM kernel's scale pass (lmme_tc.cu kFuse: every K-block read once ahead for the
    maxima, once for the main loop). Bitwise equal to the same shape fed precomputed clamped
    maxima (goom_lmme_scaled_c64), over enough products that every CTA cycles through its 4
    scale-table slots, with all-negative rows (clamp), zero rows and columns, rows near 1e5,
    non-canonical phases (2 pi, -pi) in some products, a broadcast right operand, and the
    fused bias gadd (the scaled entry has no bias: it is added by the same gadd kernel).
    n = m = 64 packs two products per tcgen05 tile (lmme_tc.cu kDuo); an odd batch leaves the
    last tile half empty. The scaled reference at n = 64 is the SIMT kernel (bitwise the same
    clamped-scale arithmetic is NOT expected there), so 64 is checked against the float64
    oracle on every edge-case product instead."""
    import ctypes

    n, k, m = shape
    torch.manual_seed(n + k + bcast + 7 * bias)
    batch = 701 if n == 64 else 700
    A = torch.ops.goom.from_real(torch.randn(batch, n, k, device="cuda") * 3, float("-inf"), False)
    B = torch.ops.goom.from_real(torch.randn(1 if bcast else batch, k, m, device="cuda") * 3,
                                 float("-inf"), False)
    A.real[5, 7, :] -= 200.0                                     # row entirely below 0: a = 0
    A[9, 3, :] = torch.complex(torch.tensor(float("-inf")), torch.tensor(0.0))   # zero row
    B[0, :, 11] = torch.complex(torch.tensor(float("-inf")), torch.tensor(0.0))  # zero column
    A.real[17, 100:120, :] += 1e5                                # huge logs
    A.imag[40] = torch.where(A.imag[40] != 0, torch.full_like(A.imag[40], -math.pi),
                             torch.full_like(A.imag[40], 2 * math.pi))  # non-canonical phases
    Bx = B.expand(batch, k, m) if bcast else B
    ra = A.real.amax(dim=2).clamp_min(0).contiguous()
    cb = B.real.amax(dim=1).clamp_min(0).contiguous()
    ref = torch.empty(batch, n, m, dtype=A.dtype, device="cuda")
    lib = g._lib.load()
    g._lib.check(lib.goom_lmme_scaled_c64(
        g._lib.goom_operand(A.data_ptr(), n * k, 1), ra.data_ptr(), n,
        g._lib.goom_operand(B.data_ptr(), 0 if bcast else k * m, 1), cb.data_ptr(),
        0 if bcast else m, ref.data_ptr(), n * m, batch, n, k, m,
        ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)))
    if bias:
        D = torch.ops.goom.from_real(torch.randn(batch, n, m, device="cuda") * 40, float("-inf"),
                                     False)
        got = torch.ops.goom.lmme_gadd(A, Bx, D)
        ref = torch.ops.goom.gadd(ref, D)
    else:
        got = torch.ops.goom.lmme(A, Bx)
    torch.cuda.synchronize()
    if n != 64:
        assert torch.equal(torch.view_as_real(got), torch.view_as_real(ref))
    else:  # the zero / underflow pattern equals the SIMT kernel's (same clamped scales)
        lib.goom_set_lmme_backend(1)
        try:
            simt = torch.ops.goom.lmme_gadd(A, Bx, D) if bias else torch.ops.goom.lmme(A, Bx)
        finally:
            lib.goom_set_lmme_backend(0)
        assert torch.equal(got.real == float("-inf"), simt.real == float("-inf"))
    # parity with the float64 oracle on a few products, including the edge cases (product 5's
    # row 7 is the clamp case: it underflows exactly like the reference float32 run, which the
    # float64 oracle does not, so it is pinned by the bitwise check above only)
    if bias and n != 64:
        return
    if bias:  # the fused bias on the duo path equals gadd of the unfused product
        plain = torch.ops.goom.lmme(A, Bx)
        assert torch.equal(torch.view_as_real(got), torch.view_as_real(torch.ops.goom.gadd(plain, D)))
        return
    for i in (9, 17, 40, batch - 2, batch - 1):
        al, as_ = to_np(A[i:i + 1])
        bl, bs = to_np(B[0 if bcast else i:(0 if bcast else i) + 1])
        err, flips = lmme_parity(to_np(got[i:i + 1]), al, as_, bl, bs)
        assert err < 1e-4 and flips == 0, (i, err, flips)
