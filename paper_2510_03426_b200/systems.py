"""Built-in dynamical systems for the Lyapunov front end (host-side input generation).

The names and constructors follow the reference's `gooms.systems` (systems.py:14-131:
DynamicalSystem, lorenz, rossler, henon, identity_system, BUILTIN_SYSTEMS) so a caller's
`integrate_chain(lorenz(), ...)` keeps working; `lorenz96` is added for config 4
(SURVEY §8d). Flows advance with classical RK4 and carry their tangent map through the
same four stages, so each recorded Jacobian is the exact derivative of the discrete step
(up to float64 rounding). This is numpy on the host: the Jacobian chain it produces is
the input of the GPU scan, not part of it.
"""

from __future__ import annotations

import os
from dataclasses import dataclass, field
from typing import Callable

import numpy as np

# the reference's named counter-based generator (util.py:8, 23-26): manifests carry the name
RNG_NAME = "philox4x64"


def make_rng(seed, stream=0) -> np.random.Generator:
    """numpy Philox keyed by (seed, stream): the same draws on any machine or scheduler."""
    return np.random.Generator(np.random.Philox(key=np.array([seed, stream], dtype=np.uint64)))


def worker_count(explicit=None) -> int:
    """Explicit value, else GOOM_WORKERS, else the CPU count (util.py:11-20)."""
    raw = explicit if explicit is not None else (os.environ.get("GOOM_WORKERS") or os.cpu_count() or 1)
    n = int(raw)
    if n < 1:
        raise ValueError("worker count must be >= 1")
    return n


@dataclass(frozen=True)
class DynamicalSystem:
    """A discrete-time map x -> step(x) with its Jacobian at x."""

    name: str
    dim: int
    dt: float
    step: Callable[[np.ndarray], np.ndarray]
    jacobian: Callable[[np.ndarray], np.ndarray]
    default_state: np.ndarray = field(repr=False, default=None)


def _rk4_with_tangent(f, df, x, dt, want_tangent):
    """One RK4 step of x' = f(x); with want_tangent, also d(step)/dx by pushing the
    identity through the four stages (stage i's tangent K_i = Df(x_i) (I + c_i dt K_{i-1}))."""
    half = 0.5 * dt
    stages = (0.0, half, half, dt)
    xs, ks, tangents = x, [], []
    eye = np.eye(x.shape[0])
    prev_k = None
    prev_t = None
    for c in stages:
        xi = x if prev_k is None else x + c * prev_k
        ki = f(xi)
        if want_tangent:
            ji = df(xi)
            ti = ji if prev_t is None else ji @ (eye + c * prev_t)
            tangents.append(ti)
            prev_t = ti
        ks.append(ki)
        prev_k = ki
    weights = (1.0, 2.0, 2.0, 1.0)
    if want_tangent:
        acc = sum(w * t for w, t in zip(weights, tangents))
        return eye + (dt / 6.0) * acc
    return xs + (dt / 6.0) * sum(w * k for w, k in zip(weights, ks))


def _flow(name, dim, dt, f, df, x0) -> DynamicalSystem:
    return DynamicalSystem(name=name, dim=dim, dt=dt,
                           step=lambda x: _rk4_with_tangent(f, df, x, dt, False),
                           jacobian=lambda x: _rk4_with_tangent(f, df, x, dt, True),
                           default_state=np.asarray(x0, dtype=np.float64))


def lorenz(sigma=10.0, rho=28.0, beta=8.0 / 3.0, dt=0.01) -> DynamicalSystem:
    """Lorenz-63; spectrum sum = -(sigma + 1 + beta) = -13.667 for the defaults."""
    def f(x):
        return np.array([sigma * (x[1] - x[0]), x[0] * (rho - x[2]) - x[1], x[0] * x[1] - beta * x[2]])

    def df(x):
        return np.array([[-sigma, sigma, 0.0], [rho - x[2], -1.0, -x[0]], [x[1], x[0], -beta]])

    return _flow("lorenz", 3, dt, f, df, [1.0, 1.0, 1.0])


def rossler(a=0.2, b=0.2, c=5.7, dt=0.05) -> DynamicalSystem:
    def f(x):
        return np.array([-x[1] - x[2], x[0] + a * x[1], b + x[2] * (x[0] - c)])

    def df(x):
        return np.array([[0.0, -1.0, -1.0], [1.0, a, 0.0], [x[2], 0.0, x[0] - c]])

    return _flow("rossler", 3, dt, f, df, [0.1, 0.0, 0.1])


def lorenz96(d=64, forcing=8.0, dt=0.01) -> DynamicalSystem:
    """Lorenz-96 (config 4): x_i' = (x_{i+1} - x_{i-2}) x_{i-1} - x_i + F; tr Df = -d."""
    idx = np.arange(d)
    ip1, im1, im2 = (idx + 1) % d, (idx - 1) % d, (idx - 2) % d

    def f(x):
        return (x[ip1] - x[im2]) * x[im1] - x + forcing

    def df(x):
        j = -np.eye(d)
        j[idx, ip1] += x[im1]
        j[idx, im2] -= x[im1]
        j[idx, im1] += x[ip1] - x[im2]
        return j

    x0 = np.full(d, forcing)
    x0[0] += 0.01
    return _flow("lorenz96", d, dt, f, df, x0)


def henon(a=1.4, b=0.3) -> DynamicalSystem:
    """The Henon map; lambda_1 + lambda_2 = log b."""
    return DynamicalSystem(name="henon", dim=2, dt=1.0,
                           step=lambda x: np.array([1.0 - a * x[0] * x[0] + x[1], b * x[0]]),
                           jacobian=lambda x: np.array([[-2.0 * a * x[0], 1.0], [b, 0.0]]),
                           default_state=np.array([0.1, 0.1]))


def identity_system(dim=3, dt=1.0) -> DynamicalSystem:
    """Every step is the identity map (its Jacobian chain is I, I, ...)."""
    return DynamicalSystem(name="identity", dim=dim, dt=dt, step=lambda x: x,
                           jacobian=lambda x: np.eye(dim), default_state=np.zeros(dim))


BUILTIN_SYSTEMS = {"lorenz": lorenz, "rossler": rossler, "henon": henon}
