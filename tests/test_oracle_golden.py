"""Pin the numpy oracle (oracle/gooms_port.py) against vectors the reference produced.

The fixtures come from tests/golden/make_golden.py, which runs the unmodified
reference (`/root/reference/pkg/src/gooms`). Where the oracle follows the
reference's ufunc order exactly the check is bitwise.
"""

import numpy as np
import pytest

from oracle import gooms_port as G
from goom_testlib import load_golden

NEG_INF = float("-inf")


def eq(a, b):
    np.testing.assert_array_equal(np.asarray(a), np.asarray(b))


@pytest.mark.parametrize("name", ["lmme_2x2", "lmme_64_f64", "lmme_64_f32", "lmme_batched_f32"])
def test_lmme_bitwise(name):
    z = load_golden(name)
    ol, os_ = G.lmme(z["alog"], z["asign"], z["blog"], z["bsign"])
    assert ol.dtype == z["olog"].dtype
    eq(ol, z["olog"])
    eq(os_, z["osign"])


def test_lmme_2x2_value():
    z = load_golden("lmme_2x2")
    np.testing.assert_allclose(G.to_real(z["olog"], z["osign"]), [[19, 22], [43, 50]], rtol=1e-14)


def test_lmme_rowscale():
    z = load_golden("lmme_rowscale")
    for key, src in (("0", z["a"]), ("1", z["s"])):
        al, as_ = G.log_sign(src)
        bl, bs = G.log_sign(z["b"])
        ol, os_ = G.lmme(al, as_, bl, bs)
        eq(ol, z["olog" + key])
        eq(os_, z["osign" + key])


@pytest.mark.parametrize("tag", ["f64", "f32"])
def test_gadd_bitwise_and_commutative(tag):
    z = load_golden(f"gadd_{tag}")
    ol, os_ = G.gadd(z["alog"], z["asign"], z["blog"], z["bsign"])
    eq(ol, z["olog"])
    eq(os_, z["osign"])
    ol2, os2 = G.gadd(z["blog"], z["bsign"], z["alog"], z["asign"])
    eq(ol2, ol)
    eq(os2, os_)
    assert np.all(ol[:256] == NEG_INF) and np.all(os_[:256] == 1.0)


@pytest.mark.parametrize("tag", ["f64", "f32"])
def test_from_real(tag):
    z = load_golden(f"from_real_{tag}")
    ml, ms = G.log_sign(z["x"])
    eq(ml, z["olog"])
    eq(ms, z["osign"])


def test_to_real_scaled_and_col_norms():
    z = load_golden("to_real_scaled")
    for i in range(z["log"].shape[0]):
        o, c = G.to_real_scaled(z["log"][i], z["sign"][i])
        eq(o, z["out"][i])
        assert c == z["c"][i]
    z = load_golden("col_log_norms")
    eq(G.col_log_norms(z["log"]), z["out"])


def _stack(z, prefix=""):
    return G.Stack(z["alog"].copy(), z["asign"].copy(), z["blog"].copy(), z["bsign"].copy(),
                   z["flags"].copy())


def test_affine_scans():
    z = load_golden("affine_T64_d4")
    st = _stack(z)
    seq = G.scan_sequential(st)
    eq(np.array([seq.alog, seq.asign, seq.blog, seq.bsign]), z["seq"])
    par = G.scan_affine_blocked(st, 8)
    eq(np.array([par.alog, par.asign, par.blog, par.bsign]), z["par8"])


@pytest.mark.parametrize("tag,dt", [("f64", np.float64), ("f32", np.float32)])
def test_config1_chain(tag, dt):
    z = load_golden("config1_chain")
    al, as_ = G.log_sign(z["mats"].astype(dt))
    T = len(al)
    bl = np.full_like(al, NEG_INF)
    st = G.Stack(al, as_, bl, np.ones_like(as_), np.zeros(T, dtype=bool))
    seq = G.scan_sequential(st)
    eq(np.array([seq.alog, seq.asign]), z[f"seq_{tag}"])
    L, S = G.chain_blocked(al, as_, 32)
    eq(np.array([L, S]), z[f"par32_{tag}"])


def _chain_stack(al, as_):
    T = len(al)
    return G.Stack(al.copy(), as_.copy(), np.full_like(al, NEG_INF), np.ones_like(as_),
                   np.zeros(T, dtype=bool))


def test_selective_norm_threshold():
    z = load_golden("sel_norm_T300_d4")
    st = _chain_stack(z["alog"], z["asign"])
    pol = G.norm_threshold_policy(12.0)
    out, sites = G.scan_selective(st, pol, None)
    assert sites == list(z["sites"])
    eq(np.array([[out.state(i)[0] for i in range(len(out))],
                 [out.state(i)[1] for i in range(len(out))]]), z["seq_state"])
    eq(out.flags, z["seq_flags"])
    out7, sites7 = G.scan_selective(st, pol, 7)
    assert sites7 == list(z["sites"])
    eq(np.array([[out7.state(i)[0] for i in range(len(out7))],
                 [out7.state(i)[1] for i in range(len(out7))]]), z["par_state"])


def test_selective_interval8():
    z = load_golden("sel_norm_interval8")
    st = _chain_stack(z["alog"], z["asign"])
    out, sites = G.scan_selective(st, G.norm_threshold_policy(5.0, interval=8), None)
    assert sites == list(z["sites"])
    eq(np.array([[out.state(i)[0] for i in range(len(out))],
                 [out.state(i)[1] for i in range(len(out))]]), z["seq_state"])


def test_selective_with_biases_rounds():
    z = load_golden("sel_norm_bias")
    T = len(z["alog"])
    st = G.Stack(z["alog"].copy(), z["asign"].copy(), z["blog"].copy(), z["bsign"].copy(),
                 np.zeros(T, dtype=bool))
    pol = G.norm_threshold_policy(12.0)
    out, sites = G.scan_selective(st, pol, None)
    assert sites == list(z["sites"])
    eq(out.flags, z["seq_flags"])
    out16, sites16 = G.scan_selective(st, pol, 16)
    assert sites16 == list(z["sites"])
    got = np.array([out16.state(i)[0] for i in range(T)])
    assert G.rel_log_diff(got, z["seq_state"][0]) < 1e-10


def test_colinearity_chain_lorenz():
    z = load_golden("sel_colin_lorenz")
    V, Vs, sites = G.selective_chain(z["alog"], z["asign"], G.colinearity_policy(0.99, 12), 256)
    assert sites == list(z["sites"])
    eq(V, z["Vlog"])
    eq(Vs, z["Vsign"])
    w = load_golden("sel_colin_lorenz_walk")
    V1, Vs1, s1 = G.selective_chain(z["alog"][:600], z["asign"][:600], G.colinearity_policy(0.99, 1), 64)
    assert s1 == list(w["sites"])
    eq(V1, w["Vlog"])
    eq(Vs1, w["Vsign"])


def test_orthonormal_reset_kat():
    z = load_golden("orthonormal_reset")
    rl, rs = G.orthonormal_reset(z["qlog"], z["qsign"])
    eq(rl, z["rlog"])
    eq(rs, z["rsign"])
    hl, hs = G.orthonormal_reset(z["hlog"], np.ones((2, 2)))
    eq(hl, z["hrlog"])
    eq(hs, z["hrsign"])


def test_appendix_c_with_callable_policy():
    z = load_golden("appendix_c")
    target = z["a1"] @ z["x0"]

    def select(l, s):
        return np.allclose(G.to_real(l, s), target, rtol=1e-9)

    def reset(l, s):
        x = G.to_real(l, s)
        return G.log_sign(x / (1.0 + np.linalg.norm(x)))

    mats = [z["x0"], z["a1"], z["a2"], z["a3"]]
    al, as_ = G.log_sign(np.array(mats))
    st = _chain_stack(al, as_)
    pol = G.Policy(select=select, reset=reset)
    for block in (None, 1, 2, 3, 4):
        out, sites = G.scan_selective(st, pol, block)
        assert sites == [2]
        for i, key in ((1, "want1"), (2, "want2"), (3, "want3")):
            np.testing.assert_allclose(G.to_real(*out.state(i)), z[key], rtol=1e-12)
        assert list(out.flags) == [False, False, True, True]


def test_complex_adapters_round_trip():
    rng = np.random.default_rng(0)
    log = rng.uniform(-50, 50, (7, 9)).astype(np.float32)
    sign = rng.choice([-1.0, 1.0], (7, 9)).astype(np.float32)
    z = G.join_complex(log, sign)
    assert z.dtype == np.complex64
    l2, s2 = G.split_complex(z, np.float32)
    eq(l2, log)
    eq(s2, sign)
    # non-canonical phases: 2*pi is positive, 3*pi negative
    w = np.array([1 + 2j * np.pi, 1 + 3j * np.pi], dtype=np.complex64)
    assert list(G.split_complex(w)[1]) == [1.0, -1.0]


def test_lorenz96_jacobians_match_reference_machinery():
    """oracle/systems_port.py vs the reference's systems._flow_system (golden, d=16)."""
    from oracle import systems_port as S

    z = load_golden("lorenz96_d16")
    f, df, x0, dt = S.lorenz96(16)
    mats = S.integrate_chain(f, df, x0, dt, burn_in=200, T=40, seed=0)
    np.testing.assert_allclose(mats, z["mats"], rtol=1e-12, atol=1e-12)


# ---- Lyapunov stages (b)-(d) and the LLE (tests/golden/make_golden_lyap.py) ----------


def test_oracle_qr_batched_matches_reference():
    z = load_golden("qr_batched")
    q, r = G.qr_factor_batched(z["ms"])
    np.testing.assert_array_equal(q, z["q"])
    np.testing.assert_array_equal(r, z["r"])


@pytest.mark.parametrize("name,interval", [("spectrum_lorenz", 8), ("spectrum_l96_d16", 12)])
def test_oracle_spectrum_parallel_matches_reference(name, interval):
    z = load_golden(name)
    lam, resets = G.spectrum_parallel(z["mats"], float(z["dt"]), check_interval=interval)
    assert resets == int(z["resets"])
    np.testing.assert_allclose(lam, z["lambdas"], rtol=0, atol=1e-12)


def test_oracle_lle_parallel_matches_reference():
    z = load_golden("lle_random")
    for i in range(len(z["par"])):
        got = G.lle_parallel(z["mats"][i], z["u0"][i], 0.5)
        assert abs(got - z["par"][i]) <= 1e-12
        assert abs(got - z["seq"][i]) <= 1e-8


@pytest.mark.parametrize("name", ["ssm_random_d4", "ssm_growing_d8", "ssm_explode_d8"])
def test_oracle_ssm_forward_matches_reference(name):
    z = load_golden(name)
    sl, ss, c, y = G.ssm_forward_parallel(z["A"], z["B"], z["C"], z["D"], z["x0"], z["u"])
    np.testing.assert_array_equal(sl, z["state_log"])
    np.testing.assert_array_equal(ss, z["state_sign"])
    np.testing.assert_array_equal(c, z["scales"])
    np.testing.assert_array_equal(y, z["y"])


def _rel_max(x, y):
    return float(np.max(np.abs(x - y)) / max(1e-300, float(np.max(np.abs(y)))))


@pytest.mark.parametrize("name", ["ssm_bwd_d4", "ssm_bwd_d8", "ssm_bwd_growing_d8"])
def test_oracle_ssm_backward_matches_autograd(name):
    """The log-domain adjoint restatement against torch float64 autograd of the reference's
    forward (tests/golden/make_golden_ssm_bwd.py; the forward states are the reference's)."""
    z = load_golden(name)
    r = G.ssm_backward(z["A"], z["B"], z["C"], z["D"], z["x0"], z["u"], z["state_log"],
                       z["state_sign"], z["scales"], z["gy"])
    for k in ("A", "B", "C", "D", "x0", "u"):
        assert _rel_max(r[k], z["d" + k]) < 1e-12, k


def test_oracle_ssm_backward_past_float64_range():
    """c_t beyond 745 (states e^{800+}): the adjoint e^{-c_t} is below float64 range; the
    shifted recurrence still gives finite, non-zero parameter gradients."""
    rng = np.random.default_rng(9)
    d, T = 4, 2100
    a = rng.standard_normal((d, d))
    a *= 1.5 / np.max(np.abs(np.linalg.eigvals(a)))
    B, C, D = rng.standard_normal((d, d)), rng.standard_normal((2 * d, d)), rng.standard_normal((2 * d, d))
    x0, u = rng.standard_normal(d), rng.standard_normal((T, d))
    gy = rng.standard_normal((T, 2 * d))
    sl, ss, c, y = G.ssm_forward_parallel(a, B, C, D, x0, u)
    assert c.max() > 800.0
    r = G.ssm_backward(a, B, C, D, x0, u, sl, ss, c, gy)
    for k in ("A", "B", "C", "x0"):
        assert np.isfinite(r[k]).all() and np.abs(r[k]).max() > 0, k
    assert np.isfinite(r["u"]).all()
