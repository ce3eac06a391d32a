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
from typing import Optional

import numpy as np
import torch

from . import ops

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


def _bu_heads(B: torch.Tensor, u: torch.Tensor) -> torch.Tensor:
    """B_h u_t for every head and step as GOOMs: one LMME of each head's d x d B with its
    d x (S T) panel of inputs (ssm.py:107-109). B (H, d, d) real, u (H, S, T, d) real ->
    (H, S, T, d) complex128."""
    H, S, T, d = u.shape
    ug = _goom(u.reshape(H, S * T, d).transpose(1, 2))
    bu = torch.ops.goom.lmme(_goom(B), ug)                               # (H, d, S T)
    return bu.transpose(1, 2).reshape(H, S, T, d)


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


def _bu_panels(B: torch.Tensor, u: torch.Tensor, L: int) -> torch.Tensor:
    """_bu_heads produced directly in _chunked_scan's panel layout (T % L == 0): one LMME
    of batch H L — head h's B against step i's panel of its d x (S nC) inputs, column
    s nC + c = step c L + i of sequence s — so bi[i] (H, d, S nC) is a slice of the
    (H, L, d, S nC) result instead of a 2 GB permuted copy of (H, S, T, d) GOOMs. Every
    element is the same LMME as _bu_heads (same operands, scales and k order): bitwise equal."""
    H, S, T, d = u.shape
    nC = T // L
    N = S * nC
    ug = _goom(u.reshape(H, S, nC, L, d).permute(0, 3, 4, 1, 2).reshape(H * L, d, N))
    out = ops.lmme_indexed(_goom(B), L, ug, 1, H * L)                   # (H L, d, N)
    return out.view(H, L, d, N).transpose(0, 1)                         # (L, H, d, N)


def _max_normalised(M: torch.Tensor, shift: torch.Tensor):
    """(M - m, shift + m) per leading index with m = max finite log of M (0 for an
    all-zero matrix): the same GOOM matrices with their largest entry at log 0."""
    m = M.real.amax(dim=(-2, -1))
    m = torch.where(torch.isfinite(m), m, torch.zeros_like(m))
    out = M.clone()
    out.real.sub_(m.view(-1, 1, 1))
    return out, shift + m


def _chunked_scan(Ag: torch.Tensor, b: torch.Tensor, s0: torch.Tensor, chunk: int,
                  bi: Optional[torch.Tensor] = None, panels: bool = False):
    """x_t = A (x) x_{t-1} (+) b_t for H heads x S sequences with the powers of A shared by
    every chunk of L = `chunk` steps — O(T d^2) matrix-vector work instead of the affine
    scan's O(T d^3) matrix-matrix work on a constant A slot. Ag (H, d, d), b (H, S, T, d),
    s0 (H, S, d) complex128 GOOMs -> states (H, S, T, d):
      local   y_{c,i} = A (x) y_{c,i-1} (+) b_{cL+i}   (L-1 launches, all heads and chunks)
      powers  P_i = A^{i+1}                            (L-1 launches, all heads)
      entry   s_{c+1} = A^L (x) s_c (+) y_{c,L-1}     (log2 nC launches, s_0 = the initial state)
      state   x_{cL+i} = A^{i+1} (x) s_c (+) y_{c,i}   (one launch: every (head, i) pair, the
                                                      head's entry panel shared via div = L)
    Every launch is an LMME of d x d matrices with d x (S nC) panels of column vectors.
    The same states as the reference's scan up to float64 rounding (a different tree)."""
    H, S, T, d = b.shape
    dev = b.device
    L = max(1, min(chunk, T))
    nC = (T + L - 1) // L
    Tp = nC * L
    if bi is not None:  # b only carries the shape: the steps come laid out (_bu_panels)
        pass
    elif Tp != T:
        zero = torch.complex(torch.tensor(NEG_INF, dtype=torch.float64),
                             torch.tensor(0.0, dtype=torch.float64))
        bp = torch.full((H, S, Tp, d), zero, dtype=torch.complex128, device=dev)
        bp[:, :, :T] = b
        b = bp
    N = S * nC
    # panels: column index = s * nC + c; bi[i] (H, d, N)
    if bi is None:
        bi = b.reshape(H, S, nC, L, d).permute(3, 0, 4, 1, 2).contiguous().reshape(L, H, d, N)
    Ag = Ag.contiguous()
    # every step's LMME writes straight into its slot of the stacked buffers (no copies)
    Y = torch.empty((L, H, d, N), dtype=torch.complex128, device=dev)
    Y[0] = bi[0]
    for i in range(1, L):
        ops.lmme_indexed(Ag, 1, Y[i - 1], 1, H, bi[i], out=Y[i])
    P = torch.empty((H, L, d, d), dtype=torch.complex128, device=dev)  # P[h, i] = A_h^{i+1}
    P[:, 0] = Ag
    k = 1
    while k < L:  # doubling: A^{k+j+1} = A^k (x) A^{j+1}, j < k — log2 L launches, not L - 1
        m = min(k, L - k)
        blk = ops.lmme_indexed(P[:, k - 1], m, P[:, :m].reshape(H * m, d, d), 1, H * m)
        P[:, k:k + m] = blk.view(H, m, d, d)
        k += m
    # chunk-entry states s_c = A^L (x) s_{c-1} (+) y_{c-1, L-1} by a Hillis-Steele scan over
    # the chunks (log2 nC rounds of one batched LMME each, with A^L, A^2L, A^4L, ...) instead
    # of nC - 1 sequential launches of H products. The powers A^(L 2^j) are kept max-
    # normalised with their log shift carried per head: squaring a contractive A^L under the
    # LMME's 0-clamped scales (core.py:252-253) would otherwise underflow to all -inf once
    # ||A^(L 2^j)|| < e^-745 and silently drop the A^(L off) (x) s term, which the
    # sequential recurrence keeps whenever the product itself is representable.
    cur = torch.empty((H, nC, d, S), dtype=torch.complex128, device=dev)
    cur[:, 0] = s0.transpose(1, 2)
    cur[:, 1:] = Y[L - 1].reshape(H, d, S, nC).permute(0, 3, 1, 2)[:, :nC - 1]
    Mp, shift = _max_normalised(P[:, L - 1].contiguous(), torch.zeros(H, dtype=torch.float64,
                                                                       device=dev))
    off = 1
    while off < nC:
        n = nC - off
        t = ops.lmme_indexed(Mp, n, cur[:, :n].reshape(H * n, d, S), 1, H * n).view(H, n, d, S)
        t.real.add_(shift.view(H, 1, 1, 1))
        nxt = torch.ops.goom.gadd(t, cur[:, off:])
        cur[:, off:] = nxt  # stream-ordered after the reads above
        off *= 2
        if off < nC:
            Mp, shift = _max_normalised(ops.lmme_indexed(Mp, 1, Mp, 1, H), 2.0 * shift)
    S_all = cur.permute(0, 2, 3, 1).reshape(H, d, N)                    # (H, d, S nC)
    Yh = Y.permute(1, 0, 2, 3).reshape(H * L, d, N)                     # batch index h L + i
    X = ops.lmme_indexed(P.reshape(H * L, d, d), 1, S_all, L, H * L, Yh)
    if panels:  # (H L, d, S nC): state (h, s, cc L + i) is column s nC + cc of matrix h L + i
        return X, L, nC
    X = X.reshape(H, L, d, S, nC).permute(0, 3, 4, 1, 2).reshape(H, S, Tp, d)
    return X[:, :, :T]


def _chunked_states(params, x0s: np.ndarray, us: np.ndarray, chunk: int) -> torch.Tensor:
    """One head (S sequences) through _chunked_scan; returns complex128 (S, T, d)."""
    dev = _dev()
    u_t = torch.as_tensor(us, dtype=torch.float64, device=dev)
    Ag = _goom(torch.as_tensor(params.A, device=dev))[None]
    bu = _bu_heads(torch.as_tensor(params.B, device=dev)[None], u_t[None])
    s0 = _goom(torch.as_tensor(x0s, dtype=torch.float64, device=dev))[None]
    return _chunked_scan(Ag, bu, s0, chunk)[0]


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


# ---------------------------------------------------------------------------
# many heads, forward + backward (config 5: 16 heads x 32 sequences, d = 64, T = 4096)

_E2 = math.exp(2.0)


def _heads_args(A, B, C, D, x0s, us):
    dev = _dev()
    t = [torch.as_tensor(v, dtype=torch.float64, device=dev) for v in (A, B, C, D, x0s, us)]
    A, B, C, D, x0s, us = t
    if A.dim() != 3 or A.shape[1] != A.shape[2]:
        raise ValueError("A must be (H, d, d)")
    H, d = A.shape[0], A.shape[1]
    if B.shape != (H, d, d) or C.shape != (H, 2 * d, d) or D.shape != (H, 2 * d, d):
        raise ValueError("B (H, d, d), C and D (H, 2d, d) must match A")
    if us.dim() != 4 or us.shape[0] != H or us.shape[-1] != d or us.shape[2] < 1:
        raise ValueError("us must be (H, S, T, d) with T >= 1")
    if x0s.shape != (H, us.shape[1], d):
        raise ValueError("x0s must be (H, S, d)")
    for m in (A, B, C, D, x0s, us):
        if not bool(torch.isfinite(m).all()):
            raise ValueError("inputs must be finite")
    return A, B, C, D, x0s, us


def _sign_of(z: torch.Tensor) -> torch.Tensor:
    return torch.where(torch.cos(z.imag) < 0, -1.0, 1.0).to(torch.float64)


def _scales(sl: torch.Tensor) -> torch.Tensor:
    c = sl.max(dim=-1).values
    return torch.where(c == NEG_INF, torch.zeros_like(c), c)


def ssm_forward_heads(A, B, C, D, x0s, us, chunk=64):
    """H heads, each with its own (A, B, C, D) and S sequences: x0s (H, S, d), us
    (H, S, T, d) -> (state_log, state_sign, scales, y) float64 CUDA tensors with leading
    (H, S). Every launch covers all heads (the per-head loop of ssm_forward_batched folded
    into the LMME batch); the recurrence and output map are ssm.py:84-98, 110-137."""
    A, B, C, D, x0s, us = _heads_args(A, B, C, D, x0s, us)
    H, S, T, d = us.shape
    L = max(1, min(chunk, T))
    if T % L == 0:
        shape_only = us.new_empty(()).expand(H, S, T, d)  # no storage: bi carries the steps
        bu, bi = shape_only, _bu_panels(B, us, L)
    else:
        bu, bi = _bu_heads(B, us), None
    if d <= 64:  # the export reads the scan's panels directly (goom_ssm_export_c128)
        X, L, nC = _chunked_scan(_goom(A), bu, _goom(x0s), chunk, bi=bi, panels=True)
        sl, ss, c, z = ops.ssm_export(X, H, L, S, nC, T)
        del X
    else:
        state = _chunked_scan(_goom(A), bu, _goom(x0s), chunk, bi=bi)
        sl, ss = state.real, _sign_of(state)
        c = _scales(sl)
        z = ss * torch.exp(sl - c[..., None] + 2.0)
    y = (torch.bmm(z.reshape(H, S * T, d), C.transpose(1, 2)) +
         torch.bmm(us.reshape(H, S * T, d), D.transpose(1, 2))).reshape(H, S, T, 2 * d)
    return sl, ss, c, y


def _bmm_tn(a: torch.Tensor, b: torch.Tensor) -> torch.Tensor:
    """a^T b per head for a (H, K, d), b (H, K, d') with K = all (sequence, step) pairs. A
    long K is split into P slabs batched next to the heads and summed after: as one GEMM
    per head the d x d' output is a handful of tiles, so the whole 10^5-long reduction ran
    on a few SMs (1.3 ms per call at config 5)."""
    H, K, d = a.shape
    P = 32
    if K % P == 0 and K >= 512 * P:
        pa, pb = a.reshape(H * P, K // P, d), b.reshape(H * P, K // P, b.shape[-1])
        return torch.bmm(pa.transpose(1, 2), pb).reshape(H, P, d, -1).sum(dim=1)
    return torch.bmm(a.transpose(1, 2), b)


def _scaled_outer(alog, asign, b, heads_shape):
    """sum over (S, T) of a_t b_t^T with a = asign e^{alog} in float64 without underflow
    of the common scale: a per-head shift m, e^m (a e^{-m})^T b. alog/asign (H, S, T, d),
    b (H, S, T, d') real -> (H, d, d')."""
    H = heads_shape
    m = alog.reshape(H, -1).max(dim=1).values                          # (H,)
    mf = torch.where(torch.isfinite(m), m, torch.zeros_like(m))
    a = asign * torch.exp(alog - mf[:, None, None, None])
    d, d2 = alog.shape[-1], b.shape[-1]
    out = _bmm_tn(a.reshape(H, -1, d), b.reshape(H, -1, d2))
    out = out * torch.exp(mf)[:, None, None]
    return torch.where(torch.isfinite(m)[:, None, None], out, torch.zeros_like(out))


def _factored_outer(za, ea, b, heads_shape):
    """sum over (S, T) of a_t b_t^T for a_t = za_t e^{ea_t} (za (H, S, T, d) bounded, ea
    (H, S, T) one log factor per step), b (H, S, T, d') real -> (H, d, d'): the factors,
    shifted by their per-head maximum, scale b; the maximum comes back once at the end."""
    H = heads_shape
    mh = ea.reshape(H, -1).max(dim=1).values                           # (H,)
    w = torch.exp(ea - mh[:, None, None])
    d, d2 = za.shape[-1], b.shape[-1]
    out = _bmm_tn(za.reshape(H, -1, d), (b * w[..., None]).reshape(H, -1, d2))
    return out * torch.exp(mh)[:, None, None]


def _factored_rows(za, ea, M):
    """a_t M per step for a_t = za_t e^{ea_t} (za (H, S, T, d), ea (H, S, T), M (H, d, d'))."""
    H, S, T, d = za.shape
    out = torch.bmm(za.reshape(H, S * T, d), M).reshape(H, S, T, M.shape[-1])
    return out * torch.exp(ea)[..., None]


def _rowwise(alog, asign, M):
    """a_t M per step (a = asign e^{alog} (H, S, T, d), M (H, d, d')) with a per-step shift,
    so a step whose adjoint is below float64 range rounds to zero instead of to garbage."""
    m = alog.max(dim=-1).values
    mf = torch.where(torch.isfinite(m), m, torch.zeros_like(m))
    a = asign * torch.exp(alog - mf[..., None])
    H, S, T, d = alog.shape
    out = torch.bmm(a.reshape(H, S * T, d), M).reshape(H, S, T, M.shape[-1])
    return torch.where(torch.isfinite(m)[..., None], out * torch.exp(mf)[..., None],
                       torch.zeros_like(out))


def ssm_backward_heads(A, B, C, D, x0s, us, state_log, state_sign, scales, gy, chunk=64):
    """Gradients of sum(gy * y) for ssm_forward_heads: (dA, dB, dC, dD, dx0s, dus), the
    parameter gradients summed over each head's S sequences. The reference has no autodiff
    (SURVEY §8d config 5); this is the adjoint recurrence, pinned against torch float64
    autograd (tests/golden/make_golden_ssm_bwd.py) and the oracle's log-domain restatement
    (oracle/gooms_port.ssm_backward):
      z_t = s_t e^{l_t - c_t + 2}, c_t = l_{t,i*} (i* the first argmax; constant for an
      all-zero state), gz_t = C^T gy_t,
      dL/dx_t (direct) = e^{-c_t} h_t,  h_t = e^2 gz_t - e_{i*} s_{t,i*} (gz_t . z_t),
      lam_t = A^T (x) lam_{t+1} (+) e^{-c_t} h_t  — a reverse GOOM scan (_chunked_scan on
      A^T, run on lam e^{K}, K = max_t c_t), so the adjoint stays exact while e^{-c_t} is far
      below float64 range,
      dA = sum lam_t x_{t-1}^T (x_{-1} = x0), dB = sum lam_t u_t^T, du_t = B^T lam_t + D^T gy_t,
      dx0 = A^T lam_0, dC = sum gy_t z_t^T, dD = sum gy_t u_t^T."""
    A, B, C, D, x0s, us = _heads_args(A, B, C, D, x0s, us)
    dev = A.device
    sl = torch.as_tensor(state_log, dtype=torch.float64, device=dev)
    ss = torch.as_tensor(state_sign, dtype=torch.float64, device=dev)
    c = torch.as_tensor(scales, dtype=torch.float64, device=dev)
    gy = torch.as_tensor(gy, dtype=torch.float64, device=dev)
    H, S, T, d = us.shape
    if gy.shape != (H, S, T, 2 * d) or sl.shape != (H, S, T, d) or c.shape != (H, S, T):
        raise ValueError("forward results / gy shapes do not match the inputs")
    gz = torch.bmm(gy.reshape(H, S * T, 2 * d), C).reshape(H, S, T, d)
    # direct gradient through z_t = x_t e^{2 - c(x_t)}: h = e^2 gz minus the max's share
    if d <= 64:  # one fused pass (goom_ssm_adjoint_source_f64)
        h, z = ops.ssm_adjoint_source(sl, ss, c, gz)
    else:
        z = ss * torch.exp(sl - c[..., None] + 2.0)
        h = _E2 * gz
        live = sl.max(dim=-1).values != NEG_INF
        istar = sl.argmax(dim=-1, keepdim=True)
        corr = torch.gather(ss, -1, istar) * (gz * z).sum(-1, keepdim=True)
        h = h.scatter_add(-1, istar, -corr * live[..., None].to(h.dtype))
    # adjoint: reverse-time scan with A^T from a zero adjoint, run on lam e^{K} with K the
    # sequence's largest scale: the reference LMME clamps its scales at 0 (core.py:250-251),
    # so adjoints ~ e^{-c_t} below float64 range would vanish, while lam e^{K} >~ 1
    K = c.max(dim=-1).values                                           # (H, S)
    zero = torch.full((H, S, d), complex(NEG_INF, 0.0), dtype=torch.complex128, device=dev)
    At = _goom(A.transpose(1, 2).contiguous())
    L = max(1, min(chunk, T))
    if T % L == 0 and d <= 64:
        # reversed, shifted GOOMs straight into the panel layout and the adjoints straight out
        # of it (goom_ssm_panels_c128 / goom_ssm_export_c128): no flipped or permuted copies.
        # The export's per-step scale gives every adjoint as lam_t = zl_t e^{e_t} with
        # zl = sign e^{log + K - cl + 2} (|zl| <= e^2) and e_t = cl_t - K - 2 one number per
        # step, so the parameter gradients need no per-element max / exp over (S, T, d)
        bi = ops.ssm_panels(h, L, K, c, reverse=True)
        X, L, nC = _chunked_scan(At, h.new_empty(()).expand(H, S, T, d), zero, chunk, bi=bi,
                                 panels=True)
        del bi
        _, _, cl, zl = ops.ssm_export(X, H, L, S, nC, T, full=True, reverse=True, kshift=K)
        del X
        e = cl - K[..., None] - 2.0                                      # (H, S, T)
        x0g = _goom(x0s)
        c0 = _scales(x0g.real)
        x0n = _sign_of(x0g) * torch.exp(x0g.real - c0[..., None])
        dA = _factored_outer(zl[:, :, :1], e[:, :, :1] + c0[..., None], x0n[:, :, None], H)
        if T > 1:  # x_{t-1} = z_{t-1} e^{c_{t-1} - 2}
            dA = dA + _factored_outer(zl[:, :, 1:], e[:, :, 1:] + c[:, :, :-1] - 2.0,
                                      z[:, :, :-1], H)
        dB = _factored_outer(zl, e, us, H)
        dus = _factored_rows(zl, e, B) + torch.bmm(gy.reshape(H, S * T, 2 * d), D).reshape(
            H, S, T, d)
        dx0s = _factored_rows(zl[:, :, :1], e[:, :, :1], A)[:, :, 0]
        dC = _bmm_tn(gy.reshape(H, S * T, 2 * d), z.reshape(H, S * T, d))
        dD = _bmm_tn(gy.reshape(H, S * T, 2 * d), us.reshape(H, S * T, d))
        return dA, dB, dC, dD, dx0s, dus
    else:
        g = _goom(h)
        g = torch.complex(g.real + (K[..., None] - c)[..., None], g.imag)
        lam = _chunked_scan(At, g.flip(2), zero, chunk).flip(2)
        ll, ls = lam.real - K[..., None, None], _sign_of(lam)
    # dA = sum_t lam_t x_{t-1}^T as (lam_t e^{c_{t-1}}) (x_{t-1} e^{-c_{t-1}})^T: for t >= 1
    # x_{t-1} e^{-c_{t-1}} = z_{t-1} e^{-2} (already exported); t = 0 takes x_{-1} = x0
    x0g = _goom(x0s)
    c0 = _scales(x0g.real)
    x0n = _sign_of(x0g) * torch.exp(x0g.real - c0[..., None])
    dA = _scaled_outer(ll[:, :, :1] + c0[:, :, None, None], ls[:, :, :1], x0n[:, :, None], H)
    if T > 1:
        dA = dA + _scaled_outer(ll[:, :, 1:] + c[:, :, :-1, None], ls[:, :, 1:],
                                z[:, :, :-1] * math.exp(-2.0), H)
    dB = _scaled_outer(ll, ls, us, H)
    dus = _rowwise(ll, ls, B) + torch.bmm(gy.reshape(H, S * T, 2 * d), D).reshape(H, S, T, d)
    dx0s = _rowwise(ll[:, :, :1], ls[:, :, :1], A)[:, :, 0]
    dC = _bmm_tn(gy.reshape(H, S * T, 2 * d), z.reshape(H, S * T, d))
    dD = _bmm_tn(gy.reshape(H, S * T, 2 * d), us.reshape(H, S * T, d))
    return dA, dB, dC, dD, dx0s, dus


@dataclass(frozen=True)
class SsmGrads:
    """Gradients of sum(dy * y) for one sequence (numpy float64)."""

    A: np.ndarray
    B: np.ndarray
    C: np.ndarray
    D: np.ndarray
    x0: np.ndarray
    u: np.ndarray


def ssm_backward(params, run: SsmRun, dy, chunk=64) -> SsmGrads:
    """Adjoint of ssm_forward_parallel / ssm_forward_sequential for one sequence: the
    gradients of sum(dy * run.y) with respect to A, B, C, D, x0 and u (see
    ssm_backward_heads for the recurrence)."""
    dy = np.asarray(dy, dtype=np.float64)
    if dy.shape != run.y.shape:
        raise ValueError("dy must match the output shape (T, 2d)")
    p = params
    r = ssm_backward_heads(p.A[None], p.B[None], p.C[None], p.D[None], run.x0[None, None],
                           run.u[None, None], run.state_log[None, None],
                           run.state_sign[None, None], run.scales[None, None], dy[None, None],
                           chunk)
    dA, dB, dC, dD, dx0, du = (t.cpu().numpy() for t in r)
    return SsmGrads(A=dA[0], B=dB[0], C=dC[0], D=dD[0], x0=dx0[0, 0], u=du[0, 0])


class SsmFunction(torch.autograd.Function):
    """y = SSM(A, B, C, D, x0s, us) for H heads x S sequences as a differentiable layer:
    forward = ssm_forward_heads, backward = ssm_backward_heads (a deep RNN stacks these)."""

    @staticmethod
    def forward(ctx, A, B, C, D, x0s, us, chunk):
        sl, ss, c, y = ssm_forward_heads(A, B, C, D, x0s, us, chunk)
        ctx.save_for_backward(A, B, C, D, x0s, us, sl, ss, c)
        ctx.chunk = chunk
        return y

    @staticmethod
    def backward(ctx, gy):
        A, B, C, D, x0s, us, sl, ss, c = ctx.saved_tensors
        grads = ssm_backward_heads(A, B, C, D, x0s, us, sl, ss, c, gy.contiguous(), ctx.chunk)
        return (*grads, None)


def ssm_layer(A, B, C, D, x0s, us, chunk=64):
    """Differentiable multi-head GOOM SSM (float64 CUDA tensors, shapes as in
    ssm_forward_heads); returns y (H, S, T, 2d)."""
    return SsmFunction.apply(A, B, C, D, x0s, us, chunk)
