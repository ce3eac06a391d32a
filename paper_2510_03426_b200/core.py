"""GOOM representation and log-domain arithmetic — drop-in for `gooms.core`.

A matrix of GOOMs is ONE complex64 CUDA tensor: real part log|x|, imaginary
part 0 or pi (the paper's Complex64 GOOM). The reference
stores the same information as two same-dtype arrays (log_mag, sign)
(core.py:148-170); `GoomMatrix.log_mag` / `.sign` expose that view.

Array work (conversions, LMME, gadd, column norms, scaled export) runs in the
sm_100a library through `torch.ops.goom.*`. The scalar helpers (`Goom`,
`gmul`, `gadd`, `lse_reduce`, scalar `from_real` / `to_real`) are host-side
scalar API kept for drop-in completeness (reference core.py:16-145); they are
not on the data-parallel path.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np
import torch

from . import ops

NEG_INF = float("-inf")
PI32 = float(np.float32(np.pi))
BACKINGS = {32: np.float32, 64: np.float64}


def _device():
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2510_03426_b200 needs a CUDA (sm_100a) device; there is no CPU path")
    return torch.device("cuda", torch.cuda.current_device())


# ---------------------------------------------------------------------------
# scalar API (host side; core.py:21-145)


def floor_for(bits):
    """log(SNN^2) of a backing format (core.py:21-30)."""
    dtype = BACKINGS[bits]
    return 2.0 * math.log(float(np.finfo(dtype).tiny))


@dataclass(frozen=True)
class ZeroPolicy:
    """Encoding of the real zero: -inf sentinel or a finite floor (core.py:33-56)."""

    mode: str = "sentinel"
    floor_value: float = NEG_INF

    def __post_init__(self):
        if self.mode not in ("sentinel", "finite_floor"):
            raise ValueError(f"unknown zero-policy mode {self.mode!r}")
        if self.mode == "finite_floor" and not math.isfinite(self.floor_value):
            raise ValueError("finite_floor policy needs a finite floor_value")

    @staticmethod
    def sentinel():
        return ZeroPolicy("sentinel", NEG_INF)

    @staticmethod
    def finite_floor(bits=64):
        return ZeroPolicy("finite_floor", floor_for(bits))

    @property
    def zero_log(self):
        return self.floor_value if self.mode == "finite_floor" else NEG_INF


SENTINEL = ZeroPolicy.sentinel()


@dataclass(frozen=True, eq=False)
class Goom:
    """One real as (log|x|, sign); zeros compare equal regardless of sign."""

    log_mag: float
    sign: int

    def __post_init__(self):
        if self.sign not in (1, -1):
            raise ValueError("sign must be +1 or -1")
        if math.isnan(self.log_mag):
            raise ValueError("log_mag must not be NaN")

    def __eq__(self, other):
        if not isinstance(other, Goom):
            return NotImplemented
        if self.log_mag == NEG_INF and other.log_mag == NEG_INF:
            return True
        return self.log_mag == other.log_mag and self.sign == other.sign

    def __hash__(self):
        return hash((NEG_INF, 1)) if self.log_mag == NEG_INF else hash((self.log_mag, self.sign))

    def as_complex(self) -> complex:
        return complex(self.log_mag, math.pi if self.sign < 0 else 0.0)


def from_real(x, policy=SENTINEL):
    x = float(x)
    if math.isnan(x):
        raise ValueError("cannot represent NaN")
    if math.isinf(x):
        raise ValueError("cannot represent an infinite value")
    if x == 0.0:
        return Goom(policy.zero_log, 1)
    return Goom(math.log(abs(x)), -1 if x < 0.0 else 1)


def to_real(g):
    if g.log_mag == NEG_INF:
        return 0.0
    try:
        mag = math.exp(g.log_mag)
    except OverflowError:
        mag = math.inf
    return g.sign * mag


def gmul(a, b):
    if a.log_mag == NEG_INF or b.log_mag == NEG_INF:
        return Goom(NEG_INF, 1)
    return Goom(a.log_mag + b.log_mag, a.sign * b.sign)


def gadd(a, b, policy=SENTINEL):
    top = max(a.log_mag, b.log_mag)
    if top == NEG_INF:
        return Goom(policy.zero_log, 1)
    t = a.sign * math.exp(a.log_mag - top) + b.sign * math.exp(b.log_mag - top)
    if t == 0.0:
        return Goom(policy.zero_log, 1)
    return Goom(top + math.log(abs(t)), -1 if t < 0.0 else 1)


def lse_reduce(gooms, policy=SENTINEL):
    gooms = list(gooms)
    if not gooms:
        raise ValueError("lse_reduce needs at least one element")
    top = max(g.log_mag for g in gooms)
    if top == NEG_INF:
        return Goom(policy.zero_log, 1)
    t = math.fsum(g.sign * math.exp(g.log_mag - top) for g in gooms)
    if t == 0.0:
        return Goom(policy.zero_log, 1)
    return Goom(top + math.log(abs(t)), -1 if t < 0.0 else 1)


# ---------------------------------------------------------------------------
# tensor helpers


def _to_tensor(x, dtype=None):
    if isinstance(x, torch.Tensor):
        t = x
    else:
        t = torch.as_tensor(np.asarray(x))
    if dtype is not None:
        t = t.to(dtype)
    return t.to(_device())


def complex_dtype(dtype=None, like=None):
    """GOOM dtype: complex64 by default (the paper's Complex64 GOOM); complex128
    for float64 / complex128 requests (the reference's float64 backing)."""
    if dtype is None and like is not None:
        dtype = like
    if dtype is None:
        return torch.complex64
    if isinstance(dtype, torch.dtype):
        if dtype in (torch.float64, torch.complex128):
            return torch.complex128
        return torch.complex64
    return torch.complex128 if np.dtype(dtype) in (np.float64, np.complex128) else torch.complex64


def join(log_mag, sign, dtype=None) -> torch.Tensor:
    """(log, sign) arrays -> GOOM tensor on the GPU (complex64 unless dtype says 128)."""
    cd = complex_dtype(dtype)
    rt = torch.float64 if cd == torch.complex128 else torch.float32
    log_t = _to_tensor(log_mag)
    if log_t.is_complex():
        raise ValueError("log_mag must be real")
    sign_t = _to_tensor(sign, log_t.dtype)
    if log_t.shape != sign_t.shape:
        raise ValueError("log_mag and sign shapes differ")
    pi = math.pi if rt == torch.float64 else PI32
    im = torch.where(sign_t < 0, torch.tensor(pi, device=log_t.device, dtype=rt),
                     torch.tensor(0.0, device=log_t.device, dtype=rt))
    return torch.complex(log_t.to(rt), im)


def split(z: torch.Tensor):
    """GOOM tensor -> (log_mag, sign in {+1,-1}) in the matching real dtype."""
    sign = torch.where(torch.cos(z.imag) < 0, -1.0, 1.0).to(z.real.dtype)
    return z.real, sign


def _dtype_of_arrays(x):
    """Array-level entry points keep the reference's dtype: float64 -> complex128."""
    dt = x.dtype if isinstance(x, (np.ndarray, torch.Tensor)) else np.asarray(x).dtype
    return complex_dtype(dt)


def _like_input(t: torch.Tensor, ref):
    if isinstance(ref, np.ndarray):
        return t.detach().cpu().numpy()
    return t


# ---------------------------------------------------------------------------
# GoomMatrix (core.py:148-226)


class GoomMatrix:
    """Dense 2-D GOOM matrix (core.py:148-226), backed on the GPU by ONE complex tensor
    (`.data`: complex64 for a float32 backing, complex128 for float64 — the reference's
    default). The reference's host-side view is kept as its API has it: `.log_mag` and
    `.sign` are numpy arrays of the backing dtype, `.dtype` is that numpy dtype and
    `to_real()` returns a numpy array; they are materialised from the device on first use
    (instances are immutable, core.py:153-154, so the copy is cached)."""

    __slots__ = ("data", "_host")

    def __init__(self, log_mag, sign=None, dtype=None):
        if sign is None:
            z = log_mag if isinstance(log_mag, torch.Tensor) else _to_tensor(log_mag)
            if not z.is_complex():
                raise ValueError("single-argument GoomMatrix takes a complex GOOM tensor")
            z = z.to(device=_device(), dtype=complex_dtype(dtype, z.dtype))
        else:
            if dtype is None:  # the backing is the dtype of log_mag (core.py:158-170)
                lm = log_mag if isinstance(log_mag, torch.Tensor) else np.asarray(log_mag)
                if isinstance(lm, torch.Tensor):
                    dtype = lm.dtype
                elif lm.dtype in (np.float32, np.float64):
                    dtype = lm.dtype
                else:
                    raise ValueError("backing dtype must be float32 or float64")
            z = join(log_mag, sign, dtype)
        if z.dim() != 2:
            raise ValueError("GoomMatrix is 2-D")
        if bool(torch.isnan(z.real).any()):
            raise ValueError("log_mag must not contain NaN")
        self.data = z
        self._host = None

    @classmethod
    def _wrap(cls, z: torch.Tensor) -> "GoomMatrix":
        obj = object.__new__(cls)
        obj.data = z
        obj._host = None
        return obj

    def _host_view(self):
        if self._host is None:
            rt = np.float64 if self.data.dtype == torch.complex128 else np.float32
            l, s = split(self.data)
            self._host = (l.cpu().numpy().astype(rt, copy=False),
                          s.cpu().numpy().astype(rt, copy=False))
        return self._host

    @property
    def rows(self):
        return self.data.shape[0]

    @property
    def cols(self):
        return self.data.shape[1]

    @property
    def shape(self):
        return tuple(self.data.shape)

    @property
    def dtype(self):
        """The backing float dtype (numpy), as the reference's `log_mag.dtype`."""
        return np.dtype(np.float64 if self.data.dtype == torch.complex128 else np.float32)

    @property
    def backing(self) -> torch.dtype:
        """The device tensor's dtype (torch.complex64 / torch.complex128)."""
        return self.data.dtype

    @property
    def log_mag(self) -> np.ndarray:
        return self._host_view()[0]

    @property
    def sign(self) -> np.ndarray:
        return self._host_view()[1]

    def numpy(self):
        """(log_mag, sign) as float64 numpy arrays."""
        l, s = self._host_view()
        return l.astype(np.float64), s.astype(np.float64)

    @classmethod
    def from_real(cls, values, policy=SENTINEL, dtype=np.float64):
        """Elementwise real -> GOOM on the GPU (core.py:188-199); float64 backing by default
        as in the reference, float32 -> complex64."""
        if dtype is None:
            dtype = np.float64
        v = _to_tensor(values)
        if v.dtype not in (torch.float32, torch.float64):
            v = v.to(torch.float64)
        v = v.to(torch.float32 if np.dtype(dtype) == np.float32 else torch.float64)
        if v.dim() != 2:
            raise ValueError("expected a 2-D array")
        if bool(torch.isnan(v).any()):
            raise ValueError("cannot represent NaN")
        if bool(torch.isinf(v).any()):
            raise ValueError("cannot represent an infinite value")
        double = complex_dtype(dtype) == torch.complex128
        return cls._wrap(torch.ops.goom.from_real(v, float(policy.zero_log), double))

    @classmethod
    def zeros(cls, rows, cols, policy=SENTINEL, dtype=np.float64):
        z = torch.full((rows, cols), complex(policy.zero_log, 0.0),
                       dtype=complex_dtype(np.float64 if dtype is None else dtype),
                       device=_device())
        return cls._wrap(z)

    @classmethod
    def identity(cls, n, policy=SENTINEL, dtype=np.float64):
        z = torch.full((n, n), complex(policy.zero_log, 0.0),
                       dtype=complex_dtype(np.float64 if dtype is None else dtype),
                       device=_device())
        z.diagonal().real.zero_()
        return cls._wrap(z)

    def to_real(self):
        """sign * exp(log) in the backing dtype, overflow -> +-inf (core.py:213-216): a numpy
        array, as the reference returns (computed on the GPU, copied to the host)."""
        return self.to_real_device().cpu().numpy()

    def to_real_device(self, double=False):
        """sign * exp(log) as a CUDA tensor (float64 for a complex128 backing or `double`)."""
        return torch.ops.goom.to_real(self.data, bool(double))

    def __getitem__(self, idx):
        i, j = idx
        z = complex(self.data[i, j].item())
        if z.real == NEG_INF:
            return Goom(NEG_INF, 1)
        return Goom(z.real, -1 if math.cos(z.imag) < 0 else 1)

    def __repr__(self):
        return f"GoomMatrix({self.rows}x{self.cols}, dtype={self.dtype}, {self.data.dtype} on " \
               f"{self.data.device})"


# ---------------------------------------------------------------------------
# array-level kernels (core.py:229-323)



class _StackedGoom(GoomMatrix):
    """Element i of a stacked GOOM tensor, sliced only when `.data` is first read: a scan
    over a long host list hands back T pairs, and most callers read a few of them
    (creating T tensor views up front cost ~6 us per pair)."""

    __slots__ = ("_base", "_i")

    @property
    def data(self):
        return self._base[self._i]

    @classmethod
    def _of(cls, base: torch.Tensor, i: int) -> "GoomMatrix":
        obj = object.__new__(cls)
        obj._base, obj._i, obj._host = base, i, None
        return obj


def _log_sign_arrays(values, policy=SENTINEL):
    """real -> (log|v|, sign) with the zero encoding (core.py:229-239)."""
    v = _to_tensor(values)
    if v.dtype not in (torch.float32, torch.float64):
        v = v.to(torch.float64)
    z = torch.ops.goom.from_real(v.contiguous(), float(policy.zero_log), v.dtype == torch.float64)
    l, s = split(z)
    return _like_input(l, values), _like_input(s, values)


def log_matmul_exp(x: torch.Tensor, y: torch.Tensor) -> torch.Tensor:
    """LMME on complex64 GOOM tensors with np.matmul broadcasting (Eq. 9-12)."""
    return torch.ops.goom.lmme(x, y)


def _lmme_arrays(alog, asign, blog, bsign):
    """Array-level LMME (core.py:242-261); returns (log, sign) like the inputs."""
    dt = _dtype_of_arrays(alog)
    z = torch.ops.goom.lmme(join(alog, asign, dt), join(blog, bsign, dt))
    l, s = split(z)
    return _like_input(l, alog), _like_input(s, alog)


def _gadd_arrays(alog, asign, blog, bsign):
    """Elementwise signed LSE (core.py:264-275)."""
    dt = _dtype_of_arrays(alog)
    z = torch.ops.goom.gadd(join(alog, asign, dt), join(blog, bsign, dt))
    l, s = split(z)
    return _like_input(l, alog), _like_input(s, alog)


def lmme(a: GoomMatrix, b: GoomMatrix) -> GoomMatrix:
    """Log-domain matrix product exp(a) @ exp(b) (core.py:278-285)."""
    if a.cols != b.rows:
        raise ValueError(f"dimension mismatch: {a.shape} x {b.shape}")
    if a.dtype != b.dtype:
        raise ValueError("operands must share a backing dtype")
    return GoomMatrix._wrap(torch.ops.goom.lmme(a.data, b.data))


def _col_log_norms(log_mag):
    """Per-column log Euclidean norms over axis -2 (core.py:288-296)."""
    l = _to_tensor(log_mag)
    rt = torch.float64 if l.dtype == torch.float64 else torch.float32
    z = torch.complex(l.to(rt), torch.zeros_like(l, dtype=rt))
    out = torch.ops.goom.col_log_norms(z).unsqueeze(-2)
    return _like_input(out, log_mag)


def log_unit_norm_columns(m: GoomMatrix):
    """Shift columns to log-unit Euclidean norm; returns (matrix, shifts) (core.py:299-310)."""
    nu = torch.ops.goom.col_log_norms(m.data)
    if bool((nu == NEG_INF).any()):
        raise ValueError("cannot normalize an all-zero column")
    re = m.data.real
    out_log = torch.where(re == NEG_INF, re, re - nu.unsqueeze(0))
    z = torch.complex(out_log, m.data.imag)
    return GoomMatrix._wrap(z), nu.double().cpu().numpy()


def to_real_scaled(m: GoomMatrix):
    """Eq. 29: sign*exp(log - c + 2) with c the max log (core.py:313-323); returns
    (numpy array in the backing dtype, c) as the reference does."""
    out, c = torch.ops.goom.to_real_scaled(m.data)
    return out.cpu().numpy(), float(c.item())
