"""PyTorch custom ops (`torch.ops.goom.*`) over the C ABI.

Each op takes / returns complex64 or complex128 CUDA tensors (GOOMs), calls
exactly one ABI entry point on the current CUDA stream (the _c64 or _c128
twin, by dtype), and allocates outputs and workspace through the caching
allocator. No op has a CPU implementation: a CPU tensor or a missing library
raises.
"""

from __future__ import annotations

import ctypes
import math
from typing import NamedTuple, Optional, Tuple

import torch

from . import _lib

NEG_INF = float("-inf")
_CPLX = (torch.complex64, torch.complex128)


_LIB = torch.library.Library("goom", "DEF")  # noqa: TOR901 (operators defined below)


def _op(name: str):
    """Register `fn` as torch.ops.goom.<name> with a CUDA kernel only (a CPU tensor raises in
    the dispatcher). A plain Library definition: the dispatcher calls straight into `fn`
    (torch.library.custom_op measured ~17 us of Python wrapping per call, the whole
    boundary's host cost ~50 us -> ~25 us; tools/host_overhead.py)."""
    def deco(fn):
        _LIB.define(name + torch.library.infer_schema(fn, mutates_args=()))
        _LIB.impl(name, fn, "CUDA")
        return fn
    return deco


_raw_stream = getattr(torch._C, "_cuda_getCurrentRawStream", None)


def _stream():
    if _raw_stream is not None:  # the current stream's handle without a Stream object
        return ctypes.c_void_p(_raw_stream(torch.cuda.current_device()))
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def _need_cuda(*ts):
    for t in ts:
        if t is not None and not t.is_cuda:
            raise ValueError("goom ops take CUDA tensors (there is no CPU path)")


def _need_goom(*ts):
    for t in ts:
        if t is not None and t.dtype not in _CPLX:
            raise ValueError("GOOM tensors are complex64 or complex128")


def _real_of(dtype):
    return torch.float64 if dtype == torch.complex128 else torch.float32


def _ws(nbytes: int, device):
    if nbytes == 0:
        return None, 0
    return torch.empty(int(nbytes), dtype=torch.uint8, device=device), int(nbytes)


def _ptr(t):
    return None if t is None else t.data_ptr()


def _size(base: str, dtype, *args) -> int:
    name = base if dtype == torch.complex64 else base + "_c128"
    return int(getattr(_lib.load(), name)(*args))


# ---------------------------------------------------------------------------
# conversions


@_op("from_real")
def from_real(x: torch.Tensor, zero_log: float, double: bool) -> torch.Tensor:
    """real -> GOOM (complex128 if `double`, else complex64)."""
    _need_cuda(x)
    if x.dtype not in (torch.float32, torch.float64):
        raise ValueError("from_real expects float32 or float64 values")
    if double:
        x = x.to(torch.float64).contiguous()
        out = torch.empty(x.shape, dtype=torch.complex128, device=x.device)
        _lib.call("goom_from_real_c128", x.data_ptr(), out.data_ptr(), x.numel(), zero_log,
                  _stream())
        return out
    x = x.contiguous()
    out = torch.empty(x.shape, dtype=torch.complex64, device=x.device)
    name = "goom_from_real_f64" if x.dtype == torch.float64 else "goom_from_real_f32"
    _lib.call(name, x.data_ptr(), out.data_ptr(), x.numel(), zero_log, _stream())
    return out


@_op("to_real")
def to_real(z: torch.Tensor, double: bool) -> torch.Tensor:
    _need_cuda(z)
    _need_goom(z)
    z = z.contiguous()
    if z.dtype == torch.complex128:
        out = torch.empty(z.shape, dtype=torch.float64, device=z.device)
        _lib.call("goom_to_real_c128", z.data_ptr(), out.data_ptr(), z.numel(), _stream())
        return out
    dt = torch.float64 if double else torch.float32
    out = torch.empty(z.shape, dtype=dt, device=z.device)
    fn = "goom_to_real_f64" if double else "goom_to_real_f32"
    _lib.call(fn, z.data_ptr(), out.data_ptr(), z.numel(), _stream())
    return out


@_op("to_real_scaled")
def to_real_scaled(z: torch.Tensor) -> Tuple[torch.Tensor, torch.Tensor]:
    """Per-matrix (last two dims) Eq. 29 export; returns (values, c)."""
    _need_cuda(z)
    _need_goom(z)
    z = z.contiguous()
    n = z.shape[-1] * z.shape[-2] if z.dim() >= 2 else z.numel()
    batch = z.numel() // max(n, 1) if n else 0
    rt = _real_of(z.dtype)
    out = torch.empty(z.shape, dtype=rt, device=z.device)
    c = torch.empty(z.shape[:-2] if z.dim() >= 2 else (), dtype=rt, device=z.device)
    name = "goom_to_real_scaled_f32" if z.dtype == torch.complex64 else "goom_to_real_scaled_c128"
    _lib.call(name, z.data_ptr(), out.data_ptr(), c.data_ptr(), batch, n, _stream())
    return out, c


@_op("gadd")
def gadd(a: torch.Tensor, b: torch.Tensor) -> torch.Tensor:
    _need_cuda(a, b)
    _need_goom(a, b)
    if a.dtype != b.dtype:
        raise ValueError("gadd operands must share a dtype")
    a, b = torch.broadcast_tensors(a, b)
    a = a.contiguous()
    b = b.contiguous()
    out = torch.empty(a.shape, dtype=a.dtype, device=a.device)
    _lib.call(_lib.fn("goom_gadd", a.dtype), a.data_ptr(), b.data_ptr(), out.data_ptr(),
              a.numel(), _stream())
    return out


@_op("col_log_norms")
def col_log_norms(z: torch.Tensor) -> torch.Tensor:
    _need_cuda(z)
    _need_goom(z)
    z = z.contiguous()
    rows, cols = z.shape[-2], z.shape[-1]
    batch = z.numel() // (rows * cols)
    out = torch.empty(z.shape[:-2] + (cols,), dtype=_real_of(z.dtype), device=z.device)
    _lib.call(_lib.fn("goom_col_log_norms", z.dtype), z.data_ptr(), out.data_ptr(), batch, rows,
              cols, _stream())
    return out


# ---------------------------------------------------------------------------
# LMME


def _bcast_operands(a: torch.Tensor, b: torch.Tensor):
    """np.matmul broadcasting over leading dims -> (a, b, batch_shape, batch, strideA, strideB)."""
    ab, bb = a.shape[:-2], b.shape[:-2]
    if ab == bb and a.is_contiguous() and b.is_contiguous():  # the common case: no broadcast
        batch = math.prod(ab)
        mat_a, mat_b = a.shape[-1] * a.shape[-2], b.shape[-1] * b.shape[-2]
        return a, b, ab, batch, (mat_a if batch != 1 else 0), (mat_b if batch != 1 else 0)
    batch_shape = torch.broadcast_shapes(ab, bb)
    batch = math.prod(batch_shape)

    def prep(t, tb):
        mat = t.shape[-1] * t.shape[-2]
        if math.prod(tb) == 1:
            return t.reshape(t.shape[-2:]).contiguous(), 0
        if tuple(tb) == tuple(batch_shape):
            return t.contiguous(), mat
        return t.expand(batch_shape + t.shape[-2:]).contiguous(), mat

    a2, sa = prep(a, ab)
    b2, sb = prep(b, bb)
    return a2, b2, batch_shape, batch, sa, sb


def _lmme_impl(a, b, d):
    _need_cuda(a, b, d)
    _need_goom(a, b, d)
    if a.dtype != b.dtype or (d is not None and d.dtype != a.dtype):
        raise ValueError("operands must share a backing dtype")
    if a.dim() < 2 or b.dim() < 2:
        raise ValueError("lmme operands must be at least 2-D")
    n, k = a.shape[-2], a.shape[-1]
    k2, m = b.shape[-2], b.shape[-1]
    if k != k2:
        raise ValueError(f"dimension mismatch: {tuple(a.shape)} x {tuple(b.shape)}")
    a2, b2, batch_shape, batch, sa, sb = _bcast_operands(a, b)
    out = torch.empty(batch_shape + (n, m), dtype=a.dtype, device=a.device)
    if batch == 0:
        return out
    ws, nws = _ws(_size("goom_lmme_workspace_size", a.dtype, batch, n, k, m), a.device)
    if d is None:
        _lib.call(_lib.fn("goom_lmme", a.dtype), _lib.goom_operand(a2.data_ptr(), sa, 1),
                  _lib.goom_operand(b2.data_ptr(), sb, 1), out.data_ptr(), n * m, batch, n, k, m,
                  _ptr(ws), nws, _stream())
    else:
        d2 = d.expand(batch_shape + (n, m)).contiguous()
        _lib.call(_lib.fn("goom_lmme_gadd", a.dtype), _lib.goom_operand(a2.data_ptr(), sa, 1),
                  _lib.goom_operand(b2.data_ptr(), sb, 1),
                  _lib.goom_operand(d2.data_ptr(), n * m, 1), out.data_ptr(), n * m, batch, n, k,
                  m, _ptr(ws), nws, _stream())
    return out


@_op("lmme")
def lmme(a: torch.Tensor, b: torch.Tensor) -> torch.Tensor:
    """log(exp(a) @ exp(b)) over GOOMs, np.matmul broadcasting (core.py:242-285)."""
    return _lmme_impl(a, b, None)


@_op("lmme_gadd")
def lmme_gadd(a: torch.Tensor, b: torch.Tensor, d: torch.Tensor) -> torch.Tensor:
    """lmme(a, b) (+) d — the fused bias-slot combine (scan.py:176-177)."""
    return _lmme_impl(a, b, d)


def lmme_indexed(a: torch.Tensor, a_div: int, b: torch.Tensor, b_div: int, batch: int,
                 d: Optional[torch.Tensor] = None, out: Optional[torch.Tensor] = None
                 ) -> torch.Tensor:
    """C[i] = A[i // a_div] (x) B[i // b_div] (+ D[i]) for i < batch, one launch.
    a (Na, n, k) and b (Nb, k, m) are stacks (N = 1 broadcasts); d, when given, is
    (batch, n, m), any batch stride. Shares operands across a batch without materialising the broadcast
    (e.g. one chunk-entry panel per head against every power of A). `out` may be any
    (batch, n, m) view whose matrices are row-major (e.g. a strided slice of a larger
    buffer): the kernel writes there directly, no copy."""
    _need_cuda(a, b, d)
    _need_goom(a, b, d)
    if a.dim() != 3 or b.dim() != 3 or a.shape[2] != b.shape[1]:
        raise ValueError("lmme_indexed takes (N, n, k) and (N, k, m) stacks")
    n, k, m = a.shape[1], a.shape[2], b.shape[2]
    for t, div in ((a, a_div), (b, b_div)):
        if t.shape[0] != 1 and (batch - 1) // div >= t.shape[0]:
            raise ValueError("operand stack too short for batch / div")
    a, b = a.contiguous(), b.contiguous()
    if out is None:
        out = torch.empty((batch, n, m), dtype=a.dtype, device=a.device)
    elif (out.shape != (batch, n, m) or out.dtype != a.dtype or out.stride(-1) != 1 or
          (n > 1 and out.stride(-2) != m)):
        raise ValueError("out must be a (batch, n, m) view with row-major matrices")
    strideC = out.stride(0) if batch > 1 else n * m
    if batch == 0:
        return out
    sa = 0 if a.shape[0] == 1 else n * k
    sb = 0 if b.shape[0] == 1 else k * m
    ws, nws = _ws(_size("goom_lmme_workspace_size", a.dtype, batch, n, k, m), a.device)
    oa = _lib.goom_operand(a.data_ptr(), sa, max(1, a_div))
    ob = _lib.goom_operand(b.data_ptr(), sb, max(1, b_div))
    if d is None:
        _lib.call(_lib.fn("goom_lmme", a.dtype), oa, ob, out.data_ptr(), strideC, batch, n, k, m,
                  _ptr(ws), nws, _stream())
    else:
        if d.shape != (batch, n, m) or d.dtype != a.dtype:
            raise ValueError("bias must be (batch, n, m) of the operands' dtype")
        if d.stride(-1) != 1 or (n > 1 and d.stride(-2) != m):
            d = d.contiguous()  # row-major matrices at any batch stride are read in place
        sd = d.stride(0) if batch > 1 else n * m
        _lib.call(_lib.fn("goom_lmme_gadd", a.dtype), oa, ob, _lib.goom_operand(d.data_ptr(), sd, 1),
                  out.data_ptr(), strideC, batch, n, k, m, _ptr(ws), nws, _stream())
    return out


def ssm_export(X: torch.Tensor, H: int, L: int, S: int, nC: int, T: int, full: bool = True,
               reverse: bool = False, kshift: Optional[torch.Tensor] = None):
    """(state_log, state_sign, scales, z) of the SSM from the chunked scan's state-assembly
    panels X (H L, d, S nC) complex128 (goom_ssm_export_c128): the same values as the
    permuted states through ssm.py:84-98's max / shifted export, in one pass. full=False
    returns (log - kshift[h, s], sign) only; reverse=True flips time (the adjoint scan)."""
    _need_cuda(X)
    d = X.shape[1]
    if X.dtype != torch.complex128 or X.shape != (H * L, d, S * nC) or not X.is_contiguous():
        raise ValueError("X must be a contiguous (H*L, d, S*nC) complex128 tensor")
    if kshift is not None:
        kshift = kshift.to(torch.float64).contiguous()
        if kshift.shape != (H, S):
            raise ValueError("kshift must be (H, S)")
    opts = dict(dtype=torch.float64, device=X.device)
    sl, ss = (torch.empty((H, S, T, d), **opts) for _ in range(2))
    z = torch.empty((H, S, T, d), **opts) if full else None
    c = torch.empty((H, S, T), **opts) if full else None
    _lib.call("goom_ssm_export_c128", X.data_ptr(), H, L, d, S, nC, T, sl.data_ptr(),
              ss.data_ptr(), _ptr(c), _ptr(z), int(reverse), _ptr(kshift), _stream())
    return (sl, ss, c, z) if full else (sl, ss)


def ssm_adjoint_source(sl: torch.Tensor, ss: torch.Tensor, c: torch.Tensor,
                       gz: torch.Tensor) -> Tuple[torch.Tensor, torch.Tensor]:
    """(h, z) of the SSM backward (goom_ssm_adjoint_source_f64): z = ss e^{sl - c + 2} and
    h = e^2 gz minus the export max's gradient at each state's first argmax. sl, ss, gz
    (..., d) and c (...) float64 CUDA tensors, d <= 64."""
    _need_cuda(sl, ss, c, gz)
    d = sl.shape[-1]
    if not (sl.shape == ss.shape == gz.shape and c.shape == sl.shape[:-1]):
        raise ValueError("sl, ss, gz (..., d) and c (...) must match")
    sl, ss, c, gz = (t.to(torch.float64).contiguous() for t in (sl, ss, c, gz))
    h = torch.empty_like(sl)
    z = torch.empty_like(sl)
    _lib.call("goom_ssm_adjoint_source_f64", sl.data_ptr(), ss.data_ptr(), c.data_ptr(),
              gz.data_ptr(), c.numel(), d, h.data_ptr(), z.data_ptr(), _stream())
    return h, z


def ssm_panels(h: torch.Tensor, L: int, K: Optional[torch.Tensor] = None,
               c: Optional[torch.Tensor] = None, reverse: bool = False) -> torch.Tensor:
    """Real h (H, S, T, d) float64 -> complex128 GOOM panels (L, H, d, S T / L) in the
    chunked scan's layout (goom_ssm_panels_c128), the log part shifted by K[h, s] -
    c[h, s, t] when K is given, time reversed when `reverse`."""
    _need_cuda(h)
    H, S, T, d = h.shape
    if h.dtype != torch.float64 or T % L:
        raise ValueError("h must be float64 with T a multiple of L")
    h = h.contiguous()
    if K is not None:
        K, c = K.to(torch.float64).contiguous(), c.to(torch.float64).contiguous()
    nC = T // L
    out = torch.empty((L, H, d, S * nC), dtype=torch.complex128, device=h.device)
    _lib.call("goom_ssm_panels_c128", h.data_ptr(), _ptr(K), _ptr(c), H, L, d, S, nC, T,
              int(reverse), out.data_ptr(), _stream())
    return out


# ---------------------------------------------------------------------------
# scans


@_op("scan_chain")
def scan_chain(a: torch.Tensor, block: int, carry: Optional[torch.Tensor]) -> torch.Tensor:
    """Inclusive left-accumulating product chain (A slot of _scan_affine_stack)."""
    _need_cuda(a, carry)
    _need_goom(a, carry)
    a = a.contiguous()
    T, d = a.shape[0], a.shape[-1]
    out = torch.empty_like(a)
    ws, nws = _ws(_size("goom_scan_chain_workspace_size", a.dtype, T, d, block), a.device)
    c = None if carry is None else carry.to(a.dtype).contiguous()
    _lib.call(_lib.fn("goom_scan_chain", a.dtype), a.data_ptr(), out.data_ptr(), T, d, block,
              _ptr(c), _ptr(ws), nws, _stream())
    return out


@_op("scan_chain_long")
def scan_chain_long(a: torch.Tensor, carry: Optional[torch.Tensor]) -> torch.Tensor:
    """The same inclusive product chain for d <= 32 (and complex64 d = 16 / 32 / 64 folded on tcgen05 at the leaf level:
    scan_long_tc.cu) on the long-chain engine (scan_long.cu: reduce-then-scan, a fixed tree of
    depth O(s log_s T) instead of the block tree's s + T/s)."""
    _need_cuda(a, carry)
    _need_goom(a, carry)
    a = a.contiguous()
    T, d = a.shape[0], a.shape[-1]
    out = torch.empty_like(a)
    ws, nws = _ws(_size("goom_scan_chain_long_workspace_size", a.dtype, T, d), a.device)
    c = None if carry is None else carry.to(a.dtype).contiguous()
    _lib.call(_lib.fn("goom_scan_chain_long", a.dtype), a.data_ptr(), out.data_ptr(), T, d,
              _ptr(c), _ptr(ws), nws, _stream())
    return out


@_op("scan_affine")
def scan_affine(a: torch.Tensor, b: torch.Tensor, flags: torch.Tensor,
                block: int) -> Tuple[torch.Tensor, torch.Tensor, torch.Tensor]:
    """Inclusive affine scan under combine_affine (scan.py:181-214)."""
    _need_cuda(a, b, flags)
    _need_goom(a, b)
    a = a.contiguous()
    b = b.to(a.dtype).contiguous()
    flags = flags.to(torch.uint8).contiguous()
    T, d, m = a.shape[0], a.shape[-1], b.shape[-1]
    oa = torch.empty_like(a)
    ob = torch.empty_like(b)
    of = torch.empty_like(flags)
    ws, nws = _ws(_size("goom_scan_affine_workspace_size", a.dtype, T, d, m, block), a.device)
    _lib.call(_lib.fn("goom_scan_affine", a.dtype), a.data_ptr(), b.data_ptr(), flags.data_ptr(),
              oa.data_ptr(), ob.data_ptr(), of.data_ptr(), T, d, m, block, _ptr(ws), nws,
              _stream())
    return oa, ob, of


def policy_struct(kind: int, interval: int, consume: bool, threshold: float,
                  log_floor: float) -> _lib.goom_reset_policy:
    return _lib.goom_reset_policy(int(kind), int(interval), int(bool(consume)), 0,
                                  float(threshold), float(log_floor))


@_op("scan_selective_chain")
def scan_selective_chain(a: torch.Tensor, kind: int, interval: int, consume: bool,
                         threshold: float, log_floor: float,
                         block: int) -> Tuple[torch.Tensor, torch.Tensor]:
    """Selective-reset product chain with a built-in policy (scan.py:342-484).
    Returns (states, sites) with sites an int64 CUDA tensor."""
    _need_cuda(a)
    _need_goom(a)
    a = a.contiguous()
    T, d = a.shape[0], a.shape[-1]
    pol = policy_struct(kind, interval, consume, threshold, log_floor)
    out = torch.empty_like(a)
    sites = torch.empty(T + 1, dtype=torch.int64, device=a.device)
    nbytes = _size("goom_scan_selective_chain_workspace_size", a.dtype, T, d, ctypes.byref(pol),
                   block)
    ws, nws = _ws(nbytes, a.device)
    _lib.call(_lib.fn("goom_scan_selective_chain", a.dtype), a.data_ptr(), out.data_ptr(), T, d,
              ctypes.byref(pol), block, sites.data_ptr(), sites[T:].data_ptr(), _ptr(ws), nws,
              _stream())
    n = int(sites[T].item())
    return out, sites[:n].clone()


@_op("policy_select")
def policy_select(x: torch.Tensor, kind: int, threshold: float, log_floor: float) -> torch.Tensor:
    _need_cuda(x)
    _need_goom(x)
    x = x.contiguous()
    d = x.shape[-1]
    batch = x.numel() // (d * d)
    pol = policy_struct(kind, 1, False, threshold, log_floor)
    fire = torch.empty(x.shape[:-2], dtype=torch.uint8, device=x.device)
    _lib.call(_lib.fn("goom_policy_select", x.dtype), x.data_ptr(), batch, d, ctypes.byref(pol),
              fire.data_ptr(), _stream())
    return fire.bool()


@_op("policy_reset")
def policy_reset(x: torch.Tensor, kind: int) -> torch.Tensor:
    _need_cuda(x)
    _need_goom(x)
    x = x.contiguous()
    d = x.shape[-1]
    batch = x.numel() // (d * d)
    pol = policy_struct(kind, 1, False, 0.5, 0.0)
    out = torch.empty_like(x)
    _lib.call(_lib.fn("goom_policy_reset", x.dtype), x.data_ptr(), out.data_ptr(), batch, d,
              ctypes.byref(pol), _stream())
    return out


# ---------------------------------------------------------------------------
# long-chain harness


@_op("random_normal")
def random_normal(like: torch.Tensor, T: int, d: int, seed: int, t0: int) -> torch.Tensor:
    """(T, d, d) complex64 GOOMs of N(0,1) reals; leaf t is keyed (seed, (t0 + t) * d * d)
    so any window / shard regenerates the same chain. `like` only fixes the device."""
    out = torch.empty((T, d, d), dtype=torch.complex64, device=like.device)
    _lib.call("goom_random_normal_c64", out.data_ptr(), out.numel(), int(seed),
              int(t0) * d * d, _stream())
    return out


@_op("digest")
def digest(x: torch.Tensor) -> torch.Tensor:
    """Per matrix: (max log|x|, log Frobenius norm, finite flag, 0) as float32 (batch, 4)."""
    _need_cuda(x)
    if x.dtype != torch.complex64:
        raise ValueError("digest takes complex64 GOOMs")
    x = x.contiguous()
    n = x.shape[-1] * x.shape[-2]
    batch = x.numel() // n
    out = torch.empty((batch, 4), dtype=torch.float32, device=x.device)
    _lib.call("goom_digest_c64", x.data_ptr(), batch, n, out.data_ptr(), _stream())
    return out


def kernel_launches() -> int:
    """libgoom kernel launches so far in this process."""
    return int(_lib.load().goom_kernel_launches())


# ---------------------------------------------------------------------------
# tile-scaled fp32 chain engine (include/goom.h; d % 256 == 0)


class TsMats(NamedTuple):
    """T tile-scaled d x d matrices: X_ij = U_ij exp(q[i][j // 256]); G[J] = max_i q[i][J]
    as order-preserving uint bits stored in int32 (0 = unset)."""
    U: torch.Tensor  # (T, d, d) float32
    q: torch.Tensor  # (T, d, d // 256) float32
    G: torch.Tensor  # (T, d // 256) int32

    @property
    def T(self) -> int:
        return self.U.shape[0]

    def __getitem__(self, i):  # slice of matrices
        return TsMats(self.U[i], self.q[i], self.G[i])


def ts_eligible(d: int) -> bool:
    return d >= 256 and d % 256 == 0


def ts_empty(T: int, d: int, device) -> TsMats:
    if not ts_eligible(d):
        raise ValueError(f"tile-scaled matrices need d % 256 == 0, got {d}")
    return TsMats(torch.empty((T, d, d), dtype=torch.float32, device=device),
                  torch.empty((T, d, d // 256), dtype=torch.float32, device=device),
                  torch.zeros((T, d // 256), dtype=torch.int32, device=device))


def ts_random_normal(T: int, d: int, seed: int, t0: int, device) -> TsMats:
    """Leaves t0 .. t0+T-1 of the random_normal chain, tile-scaled (same values)."""
    m = ts_empty(T, d, device)
    _lib.call("goom_random_normal_ts", m.U.data_ptr(), m.q.data_ptr(), m.G.data_ptr(), T, d,
              int(seed), int(t0), _stream())
    return m


def ts_from_goom(x: torch.Tensor) -> TsMats:
    _need_cuda(x)
    if x.dtype != torch.complex64:
        raise ValueError("tile-scaled import takes complex64 GOOMs")
    x = x.contiguous()
    d = x.shape[-1]
    if x.shape[-2] != d:
        raise ValueError("square matrices expected")
    xb = x.reshape(-1, d, d)
    m = ts_empty(xb.shape[0], d, x.device)
    _lib.call("goom_ts_from_c64", xb.data_ptr(), xb.shape[0], d, d, m.U.data_ptr(), m.q.data_ptr(),
              m.G.data_ptr(), _stream())
    return m


def ts_to_goom(m: TsMats) -> torch.Tensor:
    T, d = m.U.shape[0], m.U.shape[-1]
    out = torch.empty((T, d, d), dtype=torch.complex64, device=m.U.device)
    _lib.call("goom_ts_to_c64", m.U.data_ptr(), m.q.data_ptr(), T, d, d, out.data_ptr(), _stream())
    return out


def lmme_ts(a: TsMats, b: TsMats, kind: int = 0, b_div: int = 1):
    """C[i] = a[i] (x) b[i // b_div] on tile-scaled operands (a single-matrix operand
    broadcasts). kind 0 -> complex64 (T, d, d); 1 -> TsMats; 2 -> digests (T, 4)."""
    d = a.U.shape[-1]
    batch = max(a.T, b.T * b_div if b.T > 1 else a.T)
    dev = a.U.device
    a_stride = 1 if a.T > 1 else 0
    b_stride = 1 if b.T > 1 else 0
    C = oU = oq = oG = dg = parts = None
    if kind == 0:
        C = torch.empty((batch, d, d), dtype=torch.complex64, device=dev)
    elif kind == 1:
        res = ts_empty(batch, d, dev)
        oU, oq, oG = res.U, res.q, res.G
    else:
        dg = torch.empty((batch, 4), dtype=torch.float32, device=dev)
        parts = torch.empty((batch * (d // 32) * (d // 256), 4), dtype=torch.float32, device=dev)

    def p(t):
        return None if t is None else t.data_ptr()

    _lib.call("goom_lmme_ts", a.U.data_ptr(), a.q.data_ptr(), a.G.data_ptr(), a_stride, 1,
              b.U.data_ptr(), b.q.data_ptr(), b.G.data_ptr(), b_stride, int(b_div), int(kind),
              p(C), p(oU), p(oq), p(oG), p(dg), p(parts), batch, d, d, d, _stream())
    if kind == 0:
        return C
    if kind == 1:
        return res
    return dg


def _ts_extras(T: int, d: int, block: int, snapshots, carries, ws: torch.Tensor,
               nws: int) -> Tuple["TsMats", "TsMats"]:
    """From the window just scanned in `ws`: the prefixes at window-local indices
    `snapshots` (goom_chain_ts_snapshots) and the block carries of the blocks `carries`
    (goom_chain_ts_carries), both tile-scaled — the engine's own precision (ts_log_sign)."""
    res = []
    for name, idx in (("goom_chain_ts_snapshots", snapshots), ("goom_chain_ts_carries", carries)):
        idx = [int(i) for i in (idx or ())]
        out = ts_empty(len(idx), d, ws.device)
        if idx:
            arr = ctypes.cast((ctypes.c_int64 * len(idx))(*idx), ctypes.c_void_p)
            extra = (None,) if name == "goom_chain_ts_snapshots" else ()
            _lib.call(name, T, d, int(block), arr, len(idx), *extra, out.U.data_ptr(),
                      out.q.data_ptr(), out.G.data_ptr(), ws.data_ptr(), nws, _stream())
        res.append(out)
    return res[0], res[1]


def ts_log_sign(m: TsMats) -> Tuple[torch.Tensor, torch.Tensor]:
    """Tile-scaled matrices as float64 (log|x|, sign): log = q[i][j // 256] + log|U_ij|
    evaluated in float64, so the value is exactly what the engine holds (a complex64 export
    rounds the log to float32: 0.125 nats at |log| ~ 1e6)."""
    d = m.U.shape[-1]
    q = m.q.double().repeat_interleave(256, dim=-1)
    u = m.U.double()
    log = torch.where(u == 0, torch.full_like(u, NEG_INF), torch.log(u.abs()) + q)
    return log, torch.where(u < 0, -1.0, 1.0).to(torch.float64)


def chain_ts(leaves: TsMats, block: int, carry: Optional[TsMats] = None, out: bool = False,
             digests: bool = True, carry_out: bool = True, snapshots=None, carries=None):
    """One window of the long-chain scan on tile-scaled leaves: returns
    (prefixes complex64 or None, digests (T, 4) or None, last prefix TsMats or None), plus —
    when `snapshots` (window-local prefix indices) or `carries` (block indices) is given —
    the tile-scaled snapshots and block carries as a 4th and 5th element."""
    T, d = leaves.U.shape[0], leaves.U.shape[-1]
    dev = leaves.U.device
    ws, nws = _ws(int(_lib.load().goom_chain_ts_workspace_size(T, d, int(block))), dev)
    P = torch.empty((T, d, d), dtype=torch.complex64, device=dev) if out else None
    dg = torch.empty((T, 4), dtype=torch.float32, device=dev) if digests else None
    co = ts_empty(1, d, dev) if carry_out else None

    def p(t):
        return None if t is None else t.data_ptr()

    _lib.call("goom_chain_ts", leaves.U.data_ptr(), leaves.q.data_ptr(), leaves.G.data_ptr(), T, d,
              int(block), p(carry.U if carry else None), p(carry.q if carry else None),
              p(carry.G if carry else None), p(P), p(dg), p(co.U if co else None),
              p(co.q if co else None), p(co.G if co else None), ws.data_ptr(), nws, _stream())
    if snapshots is not None or carries is not None:
        return (P, dg, co) + _ts_extras(T, d, block, snapshots, carries, ws, nws)
    return P, dg, co


class ChainWindow(NamedTuple):
    """A window's carry-independent state kept between chain_ts_local and chain_ts_finish."""
    ws: torch.Tensor
    nbytes: int
    T: int
    d: int
    block: int


def chain_ts_local(leaves: TsMats, block: int):
    """Phases 1-2 of a window with no carry: returns (ChainWindow, window total TsMats)."""
    T, d = leaves.U.shape[0], leaves.U.shape[-1]
    dev = leaves.U.device
    ws, nws = _ws(int(_lib.load().goom_chain_ts_workspace_size(T, d, int(block))), dev)
    tot = ts_empty(1, d, dev)
    _lib.call("goom_chain_ts_local", leaves.U.data_ptr(), leaves.q.data_ptr(),
              leaves.G.data_ptr(), T, d, int(block), tot.U.data_ptr(), tot.q.data_ptr(),
              tot.G.data_ptr(), ws.data_ptr(), nws, _stream())
    return ChainWindow(ws, nws, T, d, int(block)), tot


def chain_ts_finish(win: ChainWindow, carry: Optional[TsMats], out: bool = False,
                    digests: bool = True, carry_out: bool = True, snapshots=None,
                    carries=None):
    """Phase 3 of a window prepared by chain_ts_local, with a right carry (or none);
    `snapshots` / `carries` as in chain_ts (the carries then include the right carry)."""
    dev = win.ws.device
    P = torch.empty((win.T, win.d, win.d), dtype=torch.complex64, device=dev) if out else None
    dg = torch.empty((win.T, 4), dtype=torch.float32, device=dev) if digests else None
    co = ts_empty(1, win.d, dev) if carry_out else None

    def p(t):
        return None if t is None else t.data_ptr()

    _lib.call("goom_chain_ts_finish", win.T, win.d, win.block, p(carry.U if carry else None),
              p(carry.q if carry else None), p(carry.G if carry else None), p(P), p(dg),
              p(co.U if co else None), p(co.q if co else None), p(co.G if co else None),
              win.ws.data_ptr(), win.nbytes, _stream())
    if snapshots is not None or carries is not None:
        return (P, dg, co) + _ts_extras(win.T, win.d, win.block, snapshots, carries, win.ws,
                                        win.nbytes)
    return P, dg, co
