"""The reference's scalar GOOM API (core.py:33-144: Goom, ZeroPolicy, from_real, to_real,
gmul, gadd, lse_reduce) as host Python — the cases of pkg/tests/test_core.py
TestScalarMapping / TestScalarArithmetic / TestLseReduce (no GPU needed)."""

import math

import numpy as np
import pytest

mpmath = pytest.importorskip("mpmath")
mpmath.mp.dps = 50


@pytest.fixture(scope="module")
def g():
    import paper_2510_03426_b200 as goom

    return goom


NEG_INF = float("-inf")


def test_scalar_mapping(g):
    x = g.from_real(20.0855)
    assert abs(x.log_mag - 3.0) < 1e-5 and x.sign == 1
    assert g.from_real(-1.0) == g.Goom(0.0, -1)
    z = g.from_real(0.0)
    assert z.log_mag == NEG_INF and z.sign == 1
    f32 = g.from_real(0.0, g.ZeroPolicy.finite_floor(32))
    assert abs(f32.log_mag - (-174.673)) < 0.01
    assert float(np.exp(np.float32(f32.log_mag))) == 0.0
    assert abs(g.ZeroPolicy.finite_floor(64).floor_value - (-1416.79)) < 0.01
    for bad in (float("nan"), float("inf")):
        with pytest.raises(ValueError):
            g.from_real(bad)
    assert abs(g.to_real(g.Goom(3.0, 1)) - 20.0855) < 1e-3
    assert g.to_real(g.Goom(NEG_INF, 1)) == 0.0 and g.to_real(g.Goom(0.0, -1)) == -1.0
    assert g.to_real(g.Goom(800.0, 1)) == math.inf and g.to_real(g.Goom(800.0, -1)) == -math.inf
    rng = np.random.default_rng(11)
    xs = rng.standard_normal(1000) * np.exp(rng.uniform(-100, 100, 1000))
    for v in xs[xs != 0][:100]:
        assert abs(g.to_real(g.from_real(v)) / v - 1.0) < 1e-12


def test_scalar_arithmetic(g):
    G_ = g.Goom
    assert g.gmul(G_(3.0, 1), G_(2.0, -1)) == G_(5.0, -1)
    assert g.gmul(G_(7.0, -1), G_(NEG_INF, 1)) == G_(NEG_INF, 1)
    big = g.gmul(g.from_real(1e200), g.from_real(1e200))
    assert abs(big.log_mag - float(2 * mpmath.log(mpmath.mpf("1e200")))) < 1e-9
    assert big.sign == 1 and g.to_real(big) == math.inf
    two = g.gadd(G_(0.0, 1), G_(0.0, 1))
    assert abs(two.log_mag - math.log(2.0)) < 1e-15 and two.sign == 1
    assert g.gadd(G_(0.0, 1), G_(0.0, -1)) == G_(NEG_INF, 1)
    ls = g.gadd(G_(100.0, 1), G_(0.0, -1))
    assert abs(ls.log_mag - float(mpmath.log(mpmath.exp(100) - 1))) < 1e-12 and ls.sign == 1
    rng = np.random.default_rng(3)
    logs = rng.uniform(-100, 100, (10_000, 2))
    signs = rng.choice([-1, 1], (10_000, 2))
    for i in range(0, 10_000, 997):
        a, b = G_(logs[i, 0], int(signs[i, 0])), G_(logs[i, 1], int(signs[i, 1]))
        assert g.gadd(a, b) == g.gadd(b, a)
    rng = np.random.default_rng(4)
    for _ in range(200):
        gs = [G_(float(rng.uniform(-100, 100)), int(rng.choice([-1, 1]))) for _ in range(3)]
        left = g.gadd(g.gadd(gs[0], gs[1]), gs[2])
        right = g.gadd(gs[0], g.gadd(gs[1], gs[2]))
        if left.log_mag == NEG_INF or right.log_mag == NEG_INF:
            continue
        assert abs(left.log_mag - right.log_mag) / max(1.0, abs(left.log_mag)) < 1e-10


def test_lse_reduce(g):
    G_ = g.Goom
    assert g.lse_reduce([G_(0.0, 1)]) == G_(0.0, 1)
    assert abs(g.lse_reduce([G_(0.0, 1)] * 4).log_mag - math.log(4.0)) < 1e-15
    with pytest.raises(ValueError):
        g.lse_reduce([])
    rng = np.random.default_rng(5)
    xs = rng.standard_normal(1000)
    got = g.lse_reduce([g.from_real(x) for x in xs])
    total = mpmath.fsum([mpmath.mpf(float(x)) for x in xs])
    assert got.sign == (1 if total >= 0 else -1)
    assert abs(got.log_mag - float(mpmath.log(abs(total)))) < 1e-12
    rng = np.random.default_rng(6)
    gs = [G_(float(rng.uniform(-50, 50)), int(rng.choice([-1, 1]))) for _ in range(64)]
    folded = gs[0]
    for x in gs[1:]:
        folded = g.gadd(folded, x)
    red = g.lse_reduce(gs)
    assert abs(folded.log_mag - red.log_mag) / max(1.0, abs(folded.log_mag)) < 1e-12
