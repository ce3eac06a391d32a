"""Lyapunov estimators on the selective scan — drop-in for `gooms.lyapunov`'s
policy (lyapunov.py:137-278), parallel spectrum (lyapunov.py:311-356) and largest
exponent (lyapunov.py:383-429).

`colinearity_policy` returns a built-in device policy: the predicate
(max off-diagonal |cos| of the log-unit-normalised columns > threshold, or
log|det| < log(volume_floor), or an all-zero column) and the CGS2 orthonormal
reset run inside the scan on the GPU in FP64.

`spectrum_parallel` runs all four stages on the GPU in FP64/complex128 (the
reference's precision for this path, lyapunov.py:336): (a) the fused selective
scan, (b) log-unit-normalised states -> orthonormal bases (one CTA per state:
column log-norms and Householder QR fused, `goom_unit_qr_batched_c128`),
(c) J_t Q_{t-1} as one batched FP64 GEMM, (d) the batched QR's |diag R|
(`goom_qr_batched_f64`) averaged in the log domain. `lle_parallel` is one affine
scan with a d x 1 bias and a final log-sum-exp.
"""

from __future__ import annotations

import math
import time
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .core import GoomMatrix
from .scan import ResetPolicy, _selective_chain_core, builtin_policy
from .systems import make_rng, worker_count  # noqa: F401  (the reference's lyapunov namespace)


def colinearity_policy(threshold=0.99, check_interval=12, volume_floor=1e-9) -> ResetPolicy:
    """lyapunov.colinearity_policy (lyapunov.py:239-278): consume_leaf False."""
    if not (0.0 < threshold < 1.0):
        raise ValueError("threshold must be in (0, 1)")
    return builtin_policy(_lib.POLICY_COLINEARITY, threshold=float(threshold),
                          log_volume_floor=math.log(volume_floor),
                          check_interval=check_interval, consume_leaf=False)


def colinearity_select(m: GoomMatrix, threshold) -> bool:
    """True when a column pair has |cos| > threshold (lyapunov.py:146-155).

    Pure cosine test: the volume floor is disabled (log floor = -inf).
    """
    if not (0.0 < threshold < 1.0):
        raise ValueError("threshold must be in (0, 1)")
    fire = torch.ops.goom.policy_select(m.data, _lib.POLICY_COLINEARITY, float(threshold),
                                        float("-inf"))
    return bool(fire.item())


def orthonormal_reset(m: GoomMatrix) -> GoomMatrix:
    """CGS2 orthonormal basis of the column span (lyapunov.py:197-219)."""
    if m.rows != m.cols:
        raise ValueError("expected a square matrix")
    return GoomMatrix._wrap(torch.ops.goom.policy_reset(m.data, _lib.POLICY_COLINEARITY))


# ---------------------------------------------------------------------------
# chains, QR, the spectrum and the largest exponent


@dataclass
class JacobianChain:
    """A sequence of step-map Jacobians along one trajectory (lyapunov.py:22-40)."""

    dt: float
    mats: np.ndarray  # (T, d, d)

    def __post_init__(self):
        self.mats = np.asarray(self.mats, dtype=np.float64)
        if self.mats.ndim != 3 or self.mats.shape[1] != self.mats.shape[2]:
            raise ValueError("mats must be a (T, d, d) array")

    @property
    def T(self):
        return self.mats.shape[0]

    @property
    def dim(self):
        return self.mats.shape[1]


def integrate_chain(system, x0=None, burn_in=0, T=1, seed=0) -> JacobianChain:
    """Step Jacobians J(x_0), J(x_1), ... along a trajectory of `system` after `burn_in`
    discarded steps (lyapunov.py:106-130). Without x0 the start is the system's default
    state jittered by 1e-3 N(0, 1) from the (seed, 0) Philox stream, as the reference does."""
    from .systems import make_rng

    if T < 1:
        raise ValueError("T must be >= 1")
    x = (system.default_state + 1e-3 * make_rng(seed).standard_normal(system.dim)
         if x0 is None else np.array(x0, dtype=np.float64))
    for i in range(burn_in):
        x = system.step(x)
        if not np.all(np.isfinite(x)):
            raise ValueError(f"non-finite state at burn-in step {i}")
    mats = np.empty((T, system.dim, system.dim))
    for t in range(T):
        mats[t] = system.jacobian(x)
        x = system.step(x)
        if not np.all(np.isfinite(x)):
            raise ValueError(f"non-finite state at step {burn_in + t}")
    return JacobianChain(dt=system.dt, mats=mats)


@dataclass
class SpectrumResult:
    lambdas: np.ndarray  # descending, units 1/time
    wall_seconds: float
    method: str  # "sequential" | "parallel"
    resets: int = 0


def _dev():
    if not torch.cuda.is_available():
        raise RuntimeError("the Lyapunov estimators run on the GPU (no CPU path)")
    return torch.device("cuda", torch.cuda.current_device())


def _stream():
    import ctypes

    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def qr_factor_batched(ms):
    """Householder QR over a stack with diag(R) >= 0 (lyapunov.py:79-99), the reference's
    return: (Q, R) float64 numpy stacks. Q and |diag R| come from the batched GPU kernel
    (goom_qr_batched_f64, d <= 64); R = triu(Q^T M) by one batched FP64 product."""
    m = torch.as_tensor(np.asarray(ms, dtype=np.float64), device=_dev()).contiguous()
    q, _ = _qr_device(m)
    r = torch.triu(torch.bmm(q.transpose(1, 2), m))
    return q.cpu().numpy(), r.cpu().numpy()


def qr_factor(m):
    """Householder QR of one square matrix with R[i, i] >= 0 (lyapunov.py:54-76)."""
    a = np.array(m, dtype=np.float64)
    if a.ndim != 2 or a.shape[0] != a.shape[1]:
        raise ValueError("expected a square matrix")
    if not np.isfinite(a).all():
        raise ValueError("non-finite entries")
    q, r = qr_factor_batched(a[None])
    return q[0], r[0]


def _qr_device(ms):
    """Householder QR over a stack with diag(R) >= 0 (lyapunov.py:79-99) on the GPU:
    returns (Q, |diag R|) as float64 CUDA tensors (d <= 64)."""
    m = torch.as_tensor(ms, dtype=torch.float64, device=_dev()).contiguous()
    if m.dim() != 3 or m.shape[1] != m.shape[2]:
        raise ValueError("expected a (N, d, d) stack")
    N, d = m.shape[0], m.shape[1]
    q = torch.empty_like(m)
    diag = torch.empty((N, d), dtype=torch.float64, device=m.device)
    _lib.call("goom_qr_batched_f64", m.data_ptr(), q.data_ptr(), diag.data_ptr(), N, d, _stream())
    return q, diag


def _validate_s0(chain, s0):
    d = chain.dim
    if s0 is None:
        return np.eye(d)
    s0 = np.asarray(s0, dtype=np.float64)
    if s0.shape != (d, d):
        raise ValueError("S0 shape must match the chain dimension")
    if np.max(np.abs(np.linalg.norm(s0, axis=0) - 1.0)) > 1e-8:
        raise ValueError("S0 must have unit-norm columns")
    return s0


def spectrum_parallel(chain, s0=None, colinearity_threshold=0.99, check_interval=12,
                      block_size=256, workers=None) -> SpectrumResult:
    """Parallel Lyapunov spectrum (lyapunov.py:311-356), all stages on the GPU.
    `workers` is accepted for signature compatibility (the reference's thread pool)."""
    s0 = _validate_s0(chain, s0)
    start = time.perf_counter()
    T, d = chain.T, chain.dim
    dev = _dev()
    mats = torch.as_tensor(chain.mats, dtype=torch.float64, device=dev)
    policy = colinearity_policy(colinearity_threshold, check_interval)
    # (a) states S_0 .. S_{T-1} from S0 and all Jacobians but the last
    leaves = torch.empty((T, d, d), dtype=torch.float64, device=dev)
    leaves[0] = torch.as_tensor(s0, dtype=torch.float64, device=dev)
    if T > 1:
        leaves[1:] = mats[: T - 1]
    A = torch.ops.goom.from_real(leaves, float("-inf"), True)
    V, sites = _selective_chain_core(A, policy, block_size)
    # (b) per-state orthonormal input bases
    bases = torch.empty((T, d, d), dtype=torch.float64, device=dev)
    _lib.call("goom_unit_qr_batched_c128", V.data_ptr(), bases.data_ptr(), T, d, _stream())
    # (c) output states J_t Q_{t-1}
    outputs = torch.bmm(mats, bases)
    # (d) exponents from the triangular factors
    _, diag = _qr_device(outputs)
    if bool((diag == 0.0).any()):
        raise ValueError("degenerate Jacobian chain")
    lam = (torch.log(diag).mean(dim=0) / chain.dt).cpu().numpy()
    return SpectrumResult(np.sort(lam)[::-1].copy(), time.perf_counter() - start, "parallel",
                          resets=len(sites))


def spectrum_sequential(chain, s0=None) -> SpectrumResult:
    """Classical estimator (lyapunov.py:290-308): per-step QR of the propagated basis, on
    the GPU one step at a time (the reference's sequential baseline, not a fast path)."""
    s0 = _validate_s0(chain, s0)
    start = time.perf_counter()
    dev = _dev()
    mats = torch.as_tensor(chain.mats, dtype=torch.float64, device=dev)
    q, _ = _qr_device(torch.as_tensor(s0, device=dev)[None])
    acc = torch.zeros(chain.dim, dtype=torch.float64, device=dev)
    for t in range(chain.T):
        q, diag = _qr_device((mats[t] @ q[0])[None])
        if bool((diag == 0.0).any()):
            raise ValueError(f"degenerate Jacobian chain at step {t}")
        acc += torch.log(diag[0])
    lam = (acc / (chain.dt * chain.T)).cpu().numpy()
    return SpectrumResult(np.sort(lam)[::-1].copy(), time.perf_counter() - start, "sequential")


def lle_parallel(chain, u0, block_size=256) -> float:
    """Largest exponent from one log-domain affine scan, no renormalisation
    (lyapunov.py:403-429): leaves (J_t, 0) after (0, u0); the final bias slot's squared
    norm is a log-sum-exp of doubled log magnitudes."""
    u = np.asarray(u0, dtype=np.float64)
    if abs(np.linalg.norm(u) - 1.0) > 1e-10:
        raise ValueError("u0 must have unit norm")
    T, d = chain.T, chain.dim
    dev = _dev()
    real = torch.zeros((T + 1, d, d), dtype=torch.float64, device=dev)
    real[1:] = torch.as_tensor(chain.mats, dtype=torch.float64, device=dev)
    A = torch.ops.goom.from_real(real, float("-inf"), True)
    bias = torch.zeros((T + 1, d, 1), dtype=torch.float64, device=dev)
    bias[0, :, 0] = torch.as_tensor(u, device=dev)
    B = torch.ops.goom.from_real(bias, float("-inf"), True)
    flags = torch.zeros(T + 1, dtype=torch.uint8, device=dev)
    _, ob, _ = torch.ops.goom.scan_affine(A, B, flags, int(block_size))
    final = ob[-1, :, 0].real
    m = float(final.max())
    if m == float("-inf"):
        raise ValueError("deviation vector vanished")
    lse = 2.0 * m + math.log(float(torch.exp(2.0 * (final - m)).sum()))
    return lse / (2.0 * chain.dt * T)


def lle_sequential(chain, u0) -> float:
    """Norm-growth estimator with per-step renormalisation (lyapunov.py:383-400)."""
    u = np.asarray(u0, dtype=np.float64)
    if abs(np.linalg.norm(u) - 1.0) > 1e-10:
        raise ValueError("u0 must have unit norm")
    dev = _dev()
    mats = torch.as_tensor(chain.mats, dtype=torch.float64, device=dev)
    v = torch.as_tensor(u, device=dev).clone()
    acc = 0.0
    for t in range(chain.T):
        sv = mats[t] @ v
        ns = float(torch.linalg.vector_norm(sv))
        if ns == 0.0:
            raise ValueError(f"deviation vector vanished at step {t}")
        acc += math.log(ns)
        v = sv / ns
    return acc / (chain.dt * chain.T)


# ---------------------------------------------------------------------------
# goomjac v1: the Jacobian-chain text format (lyapunov.py:433-476; host I/O)


def save_jacobian_chain(chain, path):
    """`goomjac v1 d=<d> T=<T> dt=<repr>` then T*d rows of d repr() floats."""
    with open(path, "w") as fh:
        fh.write(f"goomjac v1 d={chain.dim} T={chain.T} dt={float(chain.dt)!r}\n")
        for mat in chain.mats:
            for row in mat:
                fh.write(" ".join(repr(float(v)) for v in row) + "\n")


def load_jacobian_chain(path) -> JacobianChain:
    """Strict parser: bad header / field / row count / width / non-finite -> ValueError."""
    with open(path) as fh:
        lines = fh.read().split("\n")
    if lines and lines[-1] == "":
        lines.pop()
    if not lines:
        raise ValueError("empty jacobian chain file")
    head = lines[0].split()
    if len(head) != 5 or head[:2] != ["goomjac", "v1"]:
        raise ValueError(f"bad header: {lines[0]!r}")
    try:
        kv = dict(item.split("=", 1) for item in head[2:])
        d, T, dt = int(kv["d"]), int(kv["T"]), float(kv["dt"])
    except (KeyError, ValueError) as exc:
        raise ValueError(f"bad header: {lines[0]!r}") from exc
    if d < 1 or T < 1 or not dt > 0:
        raise ValueError("header fields out of range")
    rows = lines[1:]
    if len(rows) != T * d:
        raise ValueError(f"expected {T * d} matrix rows, found {len(rows)}")
    mats = np.empty((T * d, d))
    for i, line in enumerate(rows):
        vals = line.split()
        if len(vals) != d:
            raise ValueError(f"row {i + 2}: expected {d} values, found {len(vals)}")
        mats[i] = [float(v) for v in vals]
    if not np.isfinite(mats).all():
        raise ValueError("non-finite matrix entries")
    return JacobianChain(dt=dt, mats=mats.reshape(T, d, d))
