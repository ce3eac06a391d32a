"""Non-diagonal linear state-space recurrence in the log domain — drop-in for
`gooms.ssm` (ssm.py:1-137) on the GPU.

x_t = A x_{t-1} + B u_t runs on complex128 GOOMs (the reference computes this path in
float64, ssm.py:132-138) as one affine prefix scan (`goom_scan_affine_c128`): leaves
(A, B u_t) after a leading (0, x0), so every prefix's bias column is the state x_t;
the output map y_t = C (s e^{log x_t - c_t + 2}) + D u_t runs in FP64 on the GPU.
`ssm_forward_batched` runs many sequences that share one parameter set (config 5: 16
heads x 32 sequences) with the powers of A shared over fixed-length chunks (O(T d^2)
matrix-vector work, `_chunked_states`), or as ONE affine scan over the concatenated
sequences (each leading (0, x0) leaf zeroes the carry of the previous sequence).
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np
import torch

NEG_INF = float("-inf")


@dataclass(frozen=True)
class SsmParams:
    """Transition A (d x d), input B (d x d), output C (2d x d), feedthrough D (2d x d)."""

    A: np.ndarray
    B: np.ndarray
    C: np.ndarray
    D: np.ndarray

    def __post_init__(self):
        a, b, c, d = (np.asarray(m, dtype=np.float64) for m in (self.A, self.B, self.C, self.D))
        n = a.shape[0]
        if a.shape != (n, n) or b.shape != (n, n):
            raise ValueError("A and B must be square with matching dimension")
        if c.shape != (2 * n, n) or d.shape != (2 * n, n):
            raise ValueError("C and D must be (2d, d) for the gated output width")
        for m in (a, b, c, d):
            if not np.isfinite(m).all():
                raise ValueError("parameters must be finite")
        object.__setattr__(self, "A", a)
        object.__setattr__(self, "B", b)
        object.__setattr__(self, "C", c)
        object.__setattr__(self, "D", d)

    @property
    def dim(self):
        return self.A.shape[0]


@dataclass(frozen=True)
class SsmRun:
    """States in the log domain plus the rescaled outputs (ssm.py:47-72): numpy arrays,
    state_log / state_sign (T, d), scales c_t, outputs y (T, 2d)."""

    x0: np.ndarray
    u: np.ndarray
    y: np.ndarray
    scales: np.ndarray
    state_log: np.ndarray
    state_sign: np.ndarray

    def scaled_states(self):
        return self.state_sign * np.exp(self.state_log - self.scales[:, None] + 2.0)

    def __post_init__(self):
        if len(self.y) != len(self.u):
            raise ValueError("output length must match input length")


def _dev():
    if not torch.cuda.is_available():
        raise RuntimeError("the SSM runs on the GPU (no CPU path)")
    return torch.device("cuda", torch.cuda.current_device())


def _check_inputs(params, x0, u):
    x0 = np.asarray(x0, dtype=np.float64)
    u = np.asarray(u, dtype=np.float64)
    d = params.dim
    if x0.shape[-1:] != (d,):
        raise ValueError("x0 dimension mismatch")
    if u.ndim < 2 or u.shape[-1] != d:
        raise ValueError("u must be (T, d)")
    if u.shape[-2] < 1:
        raise ValueError("need at least one input step")
    return x0, u


def _goom(x: torch.Tensor) -> torch.Tensor:
    return torch.ops.goom.from_real(x, NEG_INF, True)


def _finish(params, x0, u, state: torch.Tensor, to_host: bool = True):
    """ssm.py:84-98 on the GPU: per-state max-log scale, shifted export, FP64 output map.
    to_host=False keeps the results as CUDA tensors (no device->host copy)."""
    sl, ph = state.real, state.imag
    ss = torch.where(torch.cos(ph) < 0, -1.0, 1.0).to(torch.float64)
    c = sl.max(dim=-1).values
    c = torch.where(c == NEG_INF, torch.zeros_like(c), c)
    scaled = ss * torch.exp(sl - c[..., None] + 2.0)
    dev = state.device
    ut = torch.as_tensor(u, device=dev)
    y = scaled @ torch.as_tensor(params.C.T, device=dev) + ut @ torch.as_tensor(params.D.T,
                                                                                  device=dev)
    if not to_host:
        return sl, ss, c, y
    return sl.cpu().numpy(), ss.cpu().numpy(), c.cpu().numpy(), y.cpu().numpy()


def _bu(params, u_t: torch.Tensor) -> torch.Tensor:
    """B u_t for every step as GOOMs (ssm.py:107-109: LMME of log B with log u; B is one
    broadcast operand, stride 0)."""
    d = params.dim
    Bg = _goom(torch.as_tensor(params.B, device=u_t.device))
    ug = _goom(u_t.reshape(-1, d, 1))
    return torch.ops.goom.lmme(Bg[None], ug)


def _scan_states(params, x0s: np.ndarray, us: np.ndarray, block_size: int) -> torch.Tensor:
    """States of S sequences (x0s (S, d), us (S, T, d)) sharing `params`: one affine scan
    over S (T + 1) leaves; returns complex128 (S, T, d)."""
    dev = _dev()
    S, T, d = us.shape
    u_t = torch.as_tensor(us, dtype=torch.float64, device=dev)
    bu = _bu(params, u_t).reshape(S, T, d, 1)
    n = T + 1
    A = torch.empty((S, n, d, d), dtype=torch.complex128, device=dev)
    A[:, 0] = torch.complex(torch.full((d, d), NEG_INF, dtype=torch.float64, device=dev),
                            torch.zeros((d, d), dtype=torch.float64, device=dev))
    A[:, 1:] = _goom(torch.as_tensor(params.A, device=dev))
    Bb = torch.empty((S, n, d, 1), dtype=torch.complex128, device=dev)
    Bb[:, 0] = _goom(torch.as_tensor(x0s, dtype=torch.float64, device=dev).reshape(S, d, 1))
    Bb[:, 1:] = bu
    flags = torch.zeros(S * n, dtype=torch.uint8, device=dev)
    _, ob, _ = torch.ops.goom.scan_affine(A.reshape(S * n, d, d), Bb.reshape(S * n, d, 1), flags,
                                          int(block_size))
    return ob.reshape(S, n, d)[:, 1:]


def ssm_forward_parallel(params, x0, u, block_size=256) -> SsmRun:
    """Scan evaluation (ssm.py:110-137): the recurrence as an affine prefix scan."""
    x0, u = _check_inputs(params, x0, u)
    state = _scan_states(params, x0[None], u[None], block_size)[0]
    sl, ss, c, y = _finish(params, x0, u, state)
    return SsmRun(x0=x0, u=u, y=y, scales=c, state_log=sl, state_sign=ss)


def ssm_forward_sequential(params, x0, u) -> SsmRun:
    """Reference evaluation (ssm.py:99-108): one log-domain update per step, each an LMME
    with the gadd of B u_t fused into its epilogue (T dependent launches)."""
    x0, u = _check_inputs(params, x0, u)
    dev = _dev()
    T, d = u.shape
    bu = _bu(params, torch.as_tensor(u, device=dev))
    Ag = _goom(torch.as_tensor(params.A, device=dev))[None]
    x = _goom(torch.as_tensor(x0, device=dev).reshape(1, d, 1))
    states = torch.empty((T, d), dtype=torch.complex128, device=dev)
    for t in range(T):
        x = torch.ops.goom.lmme_gadd(Ag, x, bu[t:t + 1])
        states[t] = x[0, :, 0]
    sl, ss, c, y = _finish(params, x0, u, states)
    return SsmRun(x0=x0, u=u, y=y, scales=c, state_log=sl, state_sign=ss)


def _chunked_states(params, x0s: np.ndarray, us: np.ndarray, chunk: int) -> torch.Tensor:
    """States of S sequences sharing A by chunks of L = `chunk` steps with the powers of A
    shared by every chunk — O(T d^2) matrix-vector work instead of the affine scan's
    O(T d^3) matrix-matrix work on a constant A slot:
      local   y_{c,i} = A (x) y_{c,i-1} (+) b_{cL+i}   (L-1 launches, all chunks at once)
      entry   s_{c+1} = A^L (x) s_c (+) y_{c,L-1}     (nC launches, s_0 = x0)
      state   x_{cL+i} = A^{i+1} (x) s_c (+) y_{c,i}   (L launches)
    Every launch is one LMME of a d x d power with a d x (S nC) panel of column vectors.
    Same states as the reference's scan up to float64 rounding (a different tree)."""
    dev = _dev()
    S, T, d = us.shape
    L = max(1, min(chunk, T))
    nC = (T + L - 1) // L
    Tp = nC * L
    u_t = torch.zeros((S, Tp, d), dtype=torch.float64, device=dev)
    u_t[:, :T] = torch.as_tensor(us, dtype=torch.float64, device=dev)
    b = _bu(params, u_t).reshape(S, nC, L, d)                    # b_t, padded steps = 0 (-inf)
    Ag = _goom(torch.as_tensor(params.A, device=dev))
    # panel layout: column index = s * nC + c
    bi = b.permute(2, 3, 0, 1).reshape(L, d, S * nC)             # [i] -> (d, S nC)
    Y = torch.empty((L, d, S * nC), dtype=torch.complex128, device=dev)
    Y[0] = bi[0]
    for i in range(1, L):
        Y[i] = torch.ops.goom.lmme_gadd(Ag[None], Y[i - 1][None], bi[i][None])[0]
    P = torch.empty((L, d, d), dtype=torch.complex128, device=dev)  # P[i] = A^{i+1}
    P[0] = Ag
    for i in range(1, L):
        P[i] = torch.ops.goom.lmme(Ag[None], P[i - 1][None])[0]
    s = torch.empty((nC, d, S), dtype=torch.complex128, device=dev)  # chunk-entry states
    s[0] = _goom(torch.as_tensor(x0s, dtype=torch.float64, device=dev).T.contiguous())
    Yl = Y[L - 1].reshape(d, S, nC)
    for c in range(1, nC):
        s[c] = torch.ops.goom.lmme_gadd(P[L - 1][None], s[c - 1][None],
                                        Yl[:, :, c - 1].contiguous()[None])[0]
    S_all = s.permute(1, 2, 0).reshape(d, S * nC)                # (d, S nC) like the panels
    X = torch.ops.goom.lmme_gadd(P, S_all.expand(L, d, S * nC).contiguous(), Y)  # (L, d, S nC)
    X = X.reshape(L, d, S, nC).permute(2, 3, 0, 1).reshape(S, Tp, d)
    return X[:, :T]


def ssm_forward_batched(params, x0s, us, block_size=256, chunk=64):
    """Many sequences with one parameter set (config 5's batch per head): x0s (S, d),
    us (S, T, d) -> (state_log, state_sign, scales, y) as float64 CUDA tensors with a
    leading S (a model keeps them on the device; the single-sequence functions return the
    reference's numpy SsmRun).
    chunk > 0: the shared-powers chunked evaluation (_chunked_states); chunk = 0: one
    affine scan over the concatenated sequences (the reference's tree per block)."""
    x0s, us = _check_inputs(params, x0s, us)
    if us.ndim != 3 or x0s.shape != (us.shape[0], params.dim):
        raise ValueError("x0s must be (S, d) and us (S, T, d)")
    if chunk:
        state = _chunked_states(params, x0s, us, chunk)
    else:
        state = _scan_states(params, x0s, us, block_size)
    return _finish(params, x0s, us, state, to_host=False)
