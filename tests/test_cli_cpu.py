"""CPU tests of the command-line front end and the host-side input generation
(SPEC.md:457-510 cli, SPEC.md:414-440 oracle_eval; systems.py of the reference).

No GPU: usage errors (exit 2), the 50-digit oracle's known answers, and the systems'
Jacobian chains against the oracle's restatement of the reference's RK4 / variational RK4
(oracle/systems_port.py, lyapunov.py:106-130)."""

import math

import numpy as np
import pytest

from oracle import systems_port as SP


def run_cli(argv, capsys):
    from paper_2510_03426_b200 import cli

    rc = cli.main(argv)
    out = capsys.readouterr()
    return rc, out.out, out.err


@pytest.mark.parametrize("argv", [
    [],                                              # no subcommand
    ["chain", "--steps", "5"],                       # missing --d
    ["chain", "--d", "x"],                           # not an int
    ["chain", "--d", "8", "--backend", "real16"],    # bad choice
    ["errbench", "--op", "tan"],                     # unknown op
    ["lyapunov", "spectrum", "--system", "duffing", "--steps", "10"],  # unknown system
    ["scanselftest", "--blocks", "4,x"],             # bad block list
    ["scanselftest", "--blocks", "0"],               # block < 1
])
def test_usage_errors_exit_2(argv, capsys):
    rc, out, err = run_cli(argv, capsys)
    assert rc == 2
    assert out == ""
    assert "error" in err or "unknown" in err


def test_oracle_known_answers():
    import mpmath

    from paper_2510_03426_b200.harness import oracle_eval

    with mpmath.workdps(60):
        e = oracle_eval("exp", 1.0)
        assert abs(e - mpmath.e) < mpmath.mpf(10) ** -49        # 50 digits, computed not typed
    assert oracle_eval("matmul", [[1, 2], [3, 4]], [[5, 6], [7, 8]]) == [[19, 22], [43, 50]]
    assert abs(float(oracle_eval("log", 2.0)) - math.log(2.0)) < 1e-15
    assert oracle_eval("identity", 0.1) == mpmath.mpf(0.1)     # float inputs are exact
    with pytest.raises(ValueError):
        oracle_eval("log", -1.0)
    with pytest.raises(ValueError):
        oracle_eval("tan", 1.0)


def test_errbench_validation():
    from paper_2510_03426_b200.harness import errbench

    with pytest.raises(ValueError):
        errbench("square", 1e6, 1e-6, 10)          # empty range
    with pytest.raises(ValueError):
        errbench("square", -1.0, 1.0, 10)          # log spacing needs positive bounds
    with pytest.raises(ValueError):
        errbench("square", 1e-6, 1e6, 10, backing=16)


def test_lorenz96_chain_matches_reference_rk4():
    """Our tangent-propagating RK4 step Jacobians == the reference's variational RK4
    (systems.py:33-45) on the same trajectory, jitter from the same Philox stream."""
    from paper_2510_03426_b200 import lyapunov, systems

    d = 12
    f, df, x0, dt = SP.lorenz96(d)
    want = SP.integrate_chain(f, df, x0, dt, burn_in=50, T=40, seed=3)
    got = lyapunov.integrate_chain(systems.lorenz96(d), burn_in=50, T=40, seed=3)
    assert got.dt == dt
    np.testing.assert_allclose(got.mats, want, rtol=1e-12, atol=1e-12)
    # tr J of the flow is -d: det of the step Jacobian ~ exp(-d dt)
    assert abs(np.log(abs(np.linalg.det(got.mats[0]))) + d * dt) < 1e-3


def test_builtin_systems_shape_and_determinism():
    from paper_2510_03426_b200 import lyapunov, systems

    for name, make in systems.BUILTIN_SYSTEMS.items():
        s = make()
        a = lyapunov.integrate_chain(s, burn_in=10, T=5, seed=1)
        b = lyapunov.integrate_chain(s, burn_in=10, T=5, seed=1)
        assert a.mats.shape == (5, s.dim, s.dim)
        assert np.array_equal(a.mats, b.mats)
    h = systems.henon()
    x = np.array([0.3, -0.2])
    np.testing.assert_array_equal(h.jacobian(x), [[-2 * 1.4 * 0.3, 1.0], [0.3, 0.0]])
    # Lorenz: finite-difference check of the step Jacobian
    lz = systems.lorenz()
    x = np.array([1.0, 2.0, 20.0])
    J = lz.jacobian(x)
    eps = 1e-6
    fd = np.stack([(lz.step(x + eps * e) - lz.step(x - eps * e)) / (2 * eps) for e in np.eye(3)], 1)
    np.testing.assert_allclose(J, fd, rtol=1e-6, atol=1e-7)
    with pytest.raises(ValueError):
        lyapunov.integrate_chain(lz, T=0)


def test_worker_count_and_rng(monkeypatch):
    from paper_2510_03426_b200 import systems

    monkeypatch.setenv("GOOM_WORKERS", "3")
    assert systems.worker_count() == 3
    assert systems.worker_count(5) == 5
    with pytest.raises(ValueError):
        systems.worker_count(0)
    a = systems.make_rng(7, 1).standard_normal(4)
    b = SP.make_rng(7, 1).standard_normal(4)
    assert np.array_equal(a, b)
