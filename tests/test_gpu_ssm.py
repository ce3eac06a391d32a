"""GPU parity of the SSM forward pass against golden vectors the
reference produced (tests/golden/make_golden_ssm.py) and the reference's own test cases
(pkg/tests/test_ssm.py)."""

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
