"""ctypes binding of the C ABI in include/goom.h (libgoom.so, built in-tree).

This is the only place the Python package touches native code. There is no
CPU fallback: if the library or a CUDA device is missing, every op raises.
"""

from __future__ import annotations

import ctypes
import os
import threading

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libgoom.so")

GOOM_OK = 0
_STATUS = {
    1: "EINVAL",
    2: "ESHAPE",
    3: "EDTYPE",
    4: "ECUDA",
    5: "EUNSUPPORTED",
    6: "EWORKSPACE",
    7: "ERANK",
}

POLICY_NEVER = 0
POLICY_COLINEARITY = 1
POLICY_NORM_THRESHOLD = 2


class GoomError(RuntimeError):
    """A CUDA / library failure (status ECUDA, EUNSUPPORTED, EWORKSPACE)."""


class goom_operand(ctypes.Structure):
    _fields_ = [("ptr", ctypes.c_void_p), ("stride", ctypes.c_int64), ("div", ctypes.c_int64)]


class goom_reset_policy(ctypes.Structure):
    _fields_ = [
        ("kind", ctypes.c_int32),
        ("check_interval", ctypes.c_int32),
        ("consume_leaf", ctypes.c_int32),
        ("reserved", ctypes.c_int32),
        ("threshold", ctypes.c_double),
        ("log_volume_floor", ctypes.c_double),
    ]


_P = ctypes.c_void_p
_I64 = ctypes.c_int64
_I = ctypes.c_int
_SZ = ctypes.c_size_t

# name -> (restype, argtypes); mirrors include/goom.h one to one
SIGNATURES = {
    "goom_last_error": (ctypes.c_char_p, []),
    "goom_version": (ctypes.c_char_p, []),
    "goom_device_supported": (_I, [_I]),
    "goom_from_real_f32": (_I, [_P, _P, _I64, ctypes.c_float, _P]),
    "goom_from_real_f64": (_I, [_P, _P, _I64, ctypes.c_double, _P]),
    "goom_to_real_f32": (_I, [_P, _P, _I64, _P]),
    "goom_to_real_f64": (_I, [_P, _P, _I64, _P]),
    "goom_to_real_scaled_f32": (_I, [_P, _P, _P, _I64, _I64, _P]),
    "goom_gadd_c64": (_I, [_P, _P, _P, _I64, _P]),
    "goom_col_log_norms_c64": (_I, [_P, _P, _I64, _I, _I, _P]),
    "goom_lmme_workspace_size": (_SZ, [_I64, _I, _I, _I]),
    "goom_lmme_c64": (_I, [goom_operand, goom_operand, _P, _I64, _I64, _I, _I, _I, _P, _SZ, _P]),
    "goom_lmme_gadd_c64": (
        _I,
        [goom_operand, goom_operand, goom_operand, _P, _I64, _I64, _I, _I, _I, _P, _SZ, _P],
    ),
    "goom_set_lmme_backend": (_I, [_I]),
    "goom_set_chain_engine": (_I, [_I]),
    "goom_lmme_scaled_c64": (
        _I,
        [goom_operand, _P, _I64, goom_operand, _P, _I64, _P, _I64, _I64, _I, _I, _I, _P],
    ),
    "goom_scan_chain_workspace_size": (_SZ, [_I64, _I, _I]),
    "goom_scan_chain_c64": (_I, [_P, _P, _I64, _I, _I, _P, _P, _SZ, _P]),
    "goom_scan_chain_long_workspace_size": (_SZ, [_I64, _I]),
    "goom_scan_chain_long_c64": (_I, [_P, _P, _I64, _I, _P, _P, _SZ, _P]),
    "goom_scan_affine_workspace_size": (_SZ, [_I64, _I, _I, _I]),
    "goom_scan_affine_c64": (_I, [_P, _P, _P, _P, _P, _P, _I64, _I, _I, _I, _P, _SZ, _P]),
    "goom_scan_selective_chain_workspace_size": (
        _SZ,
        [_I64, _I, ctypes.POINTER(goom_reset_policy), _I],
    ),
    "goom_scan_selective_chain_c64": (
        _I,
        [_P, _P, _I64, _I, ctypes.POINTER(goom_reset_policy), _I, _P, _P, _P, _SZ, _P],
    ),
    "goom_policy_select_c64": (_I, [_P, _I64, _I, ctypes.POINTER(goom_reset_policy), _P, _P]),
    "goom_policy_reset_c64": (_I, [_P, _P, _I64, _I, ctypes.POINTER(goom_reset_policy), _P]),
    # complex128 (FP64) twins
    "goom_from_real_c128": (_I, [_P, _P, _I64, ctypes.c_double, _P]),
    "goom_to_real_c128": (_I, [_P, _P, _I64, _P]),
    "goom_to_real_scaled_c128": (_I, [_P, _P, _P, _I64, _I64, _P]),
    "goom_ssm_export_c128": (_I, [_P, _I64, _I64, _I, _I64, _I64, _I64, _P, _P, _P, _P, _I, _P,
                                  _P]),
    "goom_ssm_panels_c128": (_I, [_P, _P, _P, _I64, _I64, _I, _I64, _I64, _I64, _I, _P, _P]),
    "goom_ssm_adjoint_source_f64": (_I, [_P, _P, _P, _P, _I64, _I, _P, _P, _P]),
    "goom_gadd_c128": (_I, [_P, _P, _P, _I64, _P]),
    "goom_col_log_norms_c128": (_I, [_P, _P, _I64, _I, _I, _P]),
    "goom_lmme_workspace_size_c128": (_SZ, [_I64, _I, _I, _I]),
    "goom_lmme_c128": (_I, [goom_operand, goom_operand, _P, _I64, _I64, _I, _I, _I, _P, _SZ, _P]),
    "goom_lmme_gadd_c128": (
        _I,
        [goom_operand, goom_operand, goom_operand, _P, _I64, _I64, _I, _I, _I, _P, _SZ, _P],
    ),
    "goom_scan_chain_workspace_size_c128": (_SZ, [_I64, _I, _I]),
    "goom_scan_chain_c128": (_I, [_P, _P, _I64, _I, _I, _P, _P, _SZ, _P]),
    "goom_scan_chain_long_workspace_size_c128": (_SZ, [_I64, _I]),
    "goom_scan_chain_long_c128": (_I, [_P, _P, _I64, _I, _P, _P, _SZ, _P]),
    "goom_scan_affine_workspace_size_c128": (_SZ, [_I64, _I, _I, _I]),
    "goom_scan_affine_c128": (_I, [_P, _P, _P, _P, _P, _P, _I64, _I, _I, _I, _P, _SZ, _P]),
    "goom_scan_selective_chain_workspace_size_c128": (
        _SZ,
        [_I64, _I, ctypes.POINTER(goom_reset_policy), _I],
    ),
    "goom_scan_selective_chain_c128": (
        _I,
        [_P, _P, _I64, _I, ctypes.POINTER(goom_reset_policy), _I, _P, _P, _P, _SZ, _P],
    ),
    "goom_policy_select_c128": (_I, [_P, _I64, _I, ctypes.POINTER(goom_reset_policy), _P, _P]),
    "goom_policy_reset_c128": (_I, [_P, _P, _I64, _I, ctypes.POINTER(goom_reset_policy), _P]),
    # long-chain harness
    "goom_random_normal_c64": (_I, [_P, _I64, ctypes.c_uint64, ctypes.c_uint64, _P]),
    "goom_digest_c64": (_I, [_P, _I64, _I64, _P, _P]),
    "goom_kernel_launches": (ctypes.c_longlong, []),
    # Lyapunov stages (b)-(d)
    "goom_qr_batched_f64": (_I, [_P, _P, _P, _I64, _I, _P]),
    "goom_unit_qr_batched_c128": (_I, [_P, _P, _I64, _I, _P]),
    # tile-scaled fp32 chain engine
    "goom_random_normal_ts": (_I, [_P, _P, _P, _I64, _I, ctypes.c_uint64, ctypes.c_uint64, _P]),
    "goom_ts_from_c64": (_I, [_P, _I64, _I, _I, _P, _P, _P, _P]),
    "goom_ts_to_c64": (_I, [_P, _P, _I64, _I, _I, _P, _P]),
    "goom_lmme_ts": (
        _I,
        [_P, _P, _P, _I64, _I64, _P, _P, _P, _I64, _I64, _I, _P, _P, _P, _P, _P, _P, _I64, _I,
         _I, _I, _P],
    ),
    "goom_chain_ts_workspace_size": (_SZ, [_I64, _I, _I]),
    "goom_chain_ts_local": (_I, [_P, _P, _P, _I64, _I, _I, _P, _P, _P, _P, _SZ, _P]),
    "goom_chain_ts_finish": (
        _I,
        [_I64, _I, _I, _P, _P, _P, _P, _P, _P, _P, _P, _P, _SZ, _P],
    ),
    "goom_chain_ts_snapshots": (_I, [_I64, _I, _I, _P, _I, _P, _P, _P, _P, _P, _SZ, _P]),
    "goom_chain_ts_carries": (_I, [_I64, _I, _I, _P, _I, _P, _P, _P, _P, _SZ, _P]),
    "goom_chain_ts_phase3_timing": (None, [_I]),
    "goom_chain_ts_phase3_stats": (_I, [_P, _P, _P]),
    "goom_chain_ts_phase_stats": (_I, [_I, _P, _P, _P]),
    "goom_scan_chain_sharded_workspace_size": (_SZ, [_I64, _I, _I, _I]),
    "goom_scan_chain_sharded_c64": (_I, [_P, _P, _I64, _I, _I, _P, _P, _SZ, _P]),
    "goom_scan_chain_sharded_digest_workspace_size": (_SZ, [_I64, _I, _I, _I]),
    "goom_scan_chain_sharded_digest_c64": (_I, [_P, _P, _I64, _I, _I, _P, _P, _SZ, _P]),
    "goom_chain_ts": (
        _I,
        [_P, _P, _P, _I64, _I, _I, _P, _P, _P, _P, _P, _P, _P, _P, _P, _SZ, _P],
    ),
}


def fn(base: str, dtype) -> str:
    """ABI name for a complex dtype: base_c64 / base_c128 (torch.complex64/128)."""
    import torch

    if dtype == torch.complex64:
        return base + "_c64"
    if dtype == torch.complex128:
        return base + "_c128"
    raise ValueError(f"GOOM tensors are complex64 or complex128, got {dtype}")

_lib = None
_lock = threading.Lock()


def load(path: str = LIB_PATH):
    """Load libgoom.so and declare every ABI signature (no GPU needed)."""
    global _lib
    if _lib is not None:  # loaded: no lock on the per-call path
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(path):
            raise GoomError(
                f"libgoom.so not found at {path}; build it with "
                "`python -c 'import __graft_entry__ as g; g.build()'` (nvcc, sm_100a)"
            )
        lib = ctypes.CDLL(path)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
        return lib


def check(rc: int) -> None:
    """Map a goom_status to the reference's exception types."""
    if rc == GOOM_OK:
        return
    msg = load().goom_last_error().decode(errors="replace")
    tag = _STATUS.get(rc, str(rc))
    if tag in ("EINVAL", "ESHAPE", "EDTYPE", "ERANK"):
        raise ValueError(f"{msg} [{tag}]")
    raise GoomError(f"{msg} [{tag}]")


def call(name: str, *args) -> None:
    check(getattr(load(), name)(*args))


def operand(t, stride=None, div=1):
    """goom_operand for a complex64 CUDA tensor of stacked matrices."""
    if stride is None:
        stride = t.shape[-1] * t.shape[-2] if t.dim() >= 3 and t.shape[0] > 1 else 0
    return goom_operand(t.data_ptr(), int(stride), int(div))


def null_operand():
    return goom_operand(None, 0, 1)


def set_chain_engine(engine: int) -> int:
    """Complex64 chain-scan engine for d % 256 == 0: 0 exact complex64 kernels (default),
    1 tile-scaled. Returns the previous setting (-1 queries)."""
    return int(load().goom_set_chain_engine(int(engine)))


def set_backend(backend: int) -> int:
    """0 auto, 1 SIMT FP32, 2 tcgen05 3xTF32. Returns the previous setting."""
    return int(load().goom_set_lmme_backend(int(backend)))
