"""Jacobian-chain inputs for the selective (Lyapunov) configs — TEST / BENCH INPUT ONLY.

Restates the reference's RK4 step and variational-RK4 step Jacobian
(systems.py:25-56) and its trajectory integrator (lyapunov.py:106-130), plus the
Lorenz-96 system SURVEY §8d config 4 names (built with the same machinery;
the reference ships no Lorenz-96). Pinned against the golden fixture
`tests/golden/lorenz96_d16.npz`, produced with the reference's own
`systems._flow_system` (tests/golden/make_golden.py).
"""

from __future__ import annotations

import numpy as np


def rk4_step(f, x, dt):
    """systems.py:25-30."""
    k1 = f(x)
    k2 = f(x + 0.5 * dt * k1)
    k3 = f(x + 0.5 * dt * k2)
    k4 = f(x + dt * k3)
    return x + (dt / 6.0) * (k1 + 2 * k2 + 2 * k3 + k4)


def rk4_jacobian(f, df, x, dt):
    """Variational RK4 Jacobian of one step, systems.py:33-45."""
    eye = np.eye(len(x))
    k1 = f(x)
    l1 = df(x)
    x2 = x + 0.5 * dt * k1
    k2 = f(x2)
    l2 = df(x2) @ (eye + 0.5 * dt * l1)
    x3 = x + 0.5 * dt * k2
    k3 = f(x3)
    l3 = df(x3) @ (eye + 0.5 * dt * l2)
    x4 = x + dt * k3
    l4 = df(x4) @ (eye + dt * l3)
    return eye + (dt / 6.0) * (l1 + 2 * l2 + 2 * l3 + l4)


def lorenz96(d, F=8.0, dt=0.01):
    """Lorenz-96 x_i' = (x_{i+1} - x_{i-2}) x_{i-1} - x_i + F; returns (f, df, x0, dt)."""
    idx = np.arange(d)
    ip1, im1, im2 = (idx + 1) % d, (idx - 1) % d, (idx - 2) % d

    def f(x):
        return (x[ip1] - x[im2]) * x[im1] - x + F

    def df(x):
        J = -np.eye(d)
        J[idx, ip1] += x[im1]
        J[idx, im2] -= x[im1]
        J[idx, im1] += x[ip1] - x[im2]
        return J

    x0 = np.full(d, F)
    x0[0] += 0.01
    return f, df, x0, dt


def make_rng(seed, stream=0):
    """util.py:23-26: numpy Philox keyed (seed, stream)."""
    key = np.array([np.uint64(seed), np.uint64(stream)], dtype=np.uint64)
    return np.random.Generator(np.random.Philox(key=key))


def integrate_chain(f, df, x0, dt, burn_in=0, T=1, seed=0):
    """lyapunov.py:106-130 with the default-state jitter of the reference."""
    rng = make_rng(seed)
    x = x0 + 1e-3 * rng.standard_normal(len(x0))
    for _ in range(burn_in):
        x = rk4_step(f, x, dt)
    mats = np.empty((T, len(x0), len(x0)))
    for t in range(T):
        mats[t] = rk4_jacobian(f, df, x, dt)
        x = rk4_step(f, x, dt)
        if not np.isfinite(x).all():
            raise ValueError(f"non-finite state at step {burn_in + t}")
    return mats


def spectrum_leaves(mats):
    """spectrum_parallel stage (a) leaves [S0 = I, J_0 .. J_{T-2}] (lyapunov.py:335-340)."""
    T, d = mats.shape[0], mats.shape[1]
    leaves = np.empty_like(mats)
    leaves[0] = np.eye(d)
    leaves[1:] = mats[: T - 1]
    return leaves
