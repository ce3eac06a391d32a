"""GPU parity of the Lyapunov stages (b)-(d) and the LLE against
golden vectors the reference produced (tests/golden/make_golden_lyap.py) and the reference's
own test cases (pkg/tests/test_lyapunov.py:218-290)."""

import math

import numpy as np
import pytest

from goom_testlib import load_golden

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def g():
    import paper_2510_03426_b200 as goom

    goom._lib.load()
    return goom


def test_qr_factor_batched_matches_reference(g):
    """Full-rank stacks: Q (unique with diag R > 0) and |diag R| equal the reference's. The
    rank-deficient matrix (index 3: two equal columns) has a non-unique Q beyond its rank:
    only its leading columns, orthonormality and |diag R| are compared; the zero matrix
    (index 4) gives Q = I, R = 0 in both."""
    z = load_golden("qr_batched")
    q, r = g.qr_factor_batched(z["ms"])  # the reference's return: (Q, R) numpy
    want_diag = np.abs(np.diagonal(z["r"], axis1=1, axis2=2))
    got_diag = np.diagonal(r, axis1=1, axis2=2)
    assert np.all(got_diag >= 0)
    for b in (0, 1, 2, 4, 5):
        np.testing.assert_allclose(r[b], z["r"][b], rtol=0, atol=1e-12)
    for b in (0, 1, 2, 4, 5):
        np.testing.assert_allclose(got_diag[b], want_diag[b], rtol=0, atol=1e-12)
    np.testing.assert_allclose(got_diag[3][:3], want_diag[3][:3], rtol=0, atol=1e-12)
    for b in (0, 1, 2, 4, 5):
        np.testing.assert_allclose(q[b], z["q"][b], rtol=0, atol=1e-12)
    np.testing.assert_allclose(q[3][:, :2], z["q"][3][:, :2], rtol=0, atol=1e-12)
    np.testing.assert_allclose(q[3].T @ q[3], np.eye(5), atol=1e-12)


@pytest.mark.parametrize("name,interval", [("spectrum_lorenz", 8), ("spectrum_l96_d16", 12)])
def test_spectrum_parallel_matches_reference(g, name, interval):
    z = load_golden(name)
    chain = g.JacobianChain(dt=float(z["dt"]), mats=z["mats"])
    res = g.spectrum_parallel(chain, check_interval=interval)
    assert res.resets == int(z["resets"])
    np.testing.assert_allclose(res.lambdas, z["lambdas"], rtol=0, atol=1e-9)
    assert np.max(np.abs(res.lambdas - z["seq"])) <= 0.05  # test_lyapunov.py:240-248


def test_spectrum_identity_and_benign_chains(g):
    """test_lyapunov.py:219-237: scalar identity chain exact; benign chain without resets."""
    chain = g.JacobianChain(dt=1.0, mats=np.tile(2.5 * np.eye(3), (64, 1, 1)))
    seq = g.spectrum_sequential(chain)
    par = g.spectrum_parallel(chain)
    assert par.resets == 0
    np.testing.assert_allclose(par.lambdas, seq.lambdas, atol=1e-12)
    np.testing.assert_allclose(par.lambdas, [math.log(2.5)] * 3, atol=1e-12)
    rng = np.random.default_rng(57)
    qs = [np.linalg.qr(rng.standard_normal((3, 3)))[0] for _ in range(50)]
    chain = g.JacobianChain(dt=1.0, mats=np.array([1.5 * q for q in qs]))
    seq = g.spectrum_sequential(chain)
    par = g.spectrum_parallel(chain, colinearity_threshold=0.999999, check_interval=4)
    assert par.resets == 0
    np.testing.assert_allclose(par.lambdas, seq.lambdas, atol=1e-6)
    with pytest.raises(ValueError):
        g.spectrum_parallel(chain, s0=2.0 * np.eye(3))


def test_lle_matches_reference(g):
    z = load_golden("lle_random")
    for i in range(len(z["par"])):
        chain = g.JacobianChain(dt=0.5, mats=z["mats"][i])
        got = g.lle_parallel(chain, z["u0"][i])
        assert abs(got - z["par"][i]) <= 1e-10
        assert abs(got - g.lle_sequential(chain, z["u0"][i])) <= 1e-8
    ident = g.JacobianChain(dt=1.0, mats=np.tile(np.eye(3), (32, 1, 1)))
    assert abs(g.lle_parallel(ident, np.array([1.0, 0.0, 0.0]))) < 1e-14
    dbl = g.JacobianChain(dt=1.0, mats=np.tile(2.0 * np.eye(3), (32, 1, 1)))
    assert abs(g.lle_parallel(dbl, np.array([0.0, 1.0, 0.0])) - math.log(2.0)) < 1e-12
    with pytest.raises(ValueError):
        g.lle_parallel(ident, np.array([0.0, 0.0, 0.0]))


def test_spectrum_sequential_and_parallel_properties(g):
    """test_lyapunov.py:135-162 on both GPU estimators: c I gives log(c)/dt, scaling every
    Jacobian by 4 shifts every exponent by log(4)/dt, the exponents sum to the mean log|det|
    (sequential; the parallel one within its reset tolerance), invalid S0 raises."""
    import math

    chain = g.JacobianChain(dt=0.5, mats=np.tile(1.7 * np.eye(3), (50, 1, 1)))
    for est in (g.spectrum_sequential, g.spectrum_parallel):
        np.testing.assert_allclose(est(chain).lambdas, math.log(1.7) / 0.5, rtol=1e-12)
    rng = np.random.default_rng(54)
    mats = rng.standard_normal((64, 3, 3))
    for est, tol in ((g.spectrum_sequential, 1e-9), (g.spectrum_parallel, 1e-6)):
        base = est(g.JacobianChain(dt=0.1, mats=mats)).lambdas
        scaled = est(g.JacobianChain(dt=0.1, mats=4.0 * mats)).lambdas
        np.testing.assert_allclose(scaled - base, math.log(4.0) / 0.1, rtol=tol)
    rng = np.random.default_rng(55)
    mats = rng.standard_normal((200, 3, 3))
    want = np.mean([math.log(abs(np.linalg.det(m))) for m in mats]) / 0.25
    res = g.spectrum_sequential(g.JacobianChain(dt=0.25, mats=mats))
    assert abs(res.lambdas.sum() - want) / abs(want) < 1e-6
    with pytest.raises(ValueError):
        g.spectrum_sequential(g.JacobianChain(dt=1.0, mats=np.tile(np.eye(2), (4, 1, 1))),
                              s0=np.array([[2.0, 0.0], [0.0, 1.0]]))
