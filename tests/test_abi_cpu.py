"""CPU-side checks of the drop-in boundary: libgoom.so loads, exports every
symbol include/goom.h declares, validates arguments before touching the GPU,
and the Python layer raises the reference's errors (no compute without a GPU)."""

import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "goom.h")
LIB = os.path.join(ROOT, "paper_2510_03426_b200", "libgoom.so")


def declared_functions():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    names = re.findall(r"\b(goom_[a-z0-9_]+)\s*\(", text)
    return sorted(set(names))


@pytest.fixture(scope="module")
def lib():
    if not os.path.exists(LIB):
        pytest.skip("libgoom.so not built (run __graft_entry__.build())")
    return ctypes.CDLL(LIB)


def test_header_declares_the_path():
    names = declared_functions()
    for must in ("goom_lmme_c64", "goom_gadd_c64", "goom_from_real_f32", "goom_to_real_f32",
                 "goom_to_real_scaled_f32", "goom_scan_chain_c64", "goom_scan_affine_c64",
                 "goom_scan_selective_chain_c64", "goom_last_error"):
        assert must in names


def test_every_declared_symbol_is_exported(lib):
    missing = [n for n in declared_functions() if not hasattr(lib, n)]
    assert not missing, missing


def test_python_binding_matches_header():
    from paper_2510_03426_b200 import _lib

    assert set(_lib.SIGNATURES) == set(declared_functions())
    _lib.load()


def test_argument_errors_without_gpu(lib):
    from paper_2510_03426_b200 import _lib

    L = _lib.load()
    # empty scan / bad block: validated before any CUDA call (scan.py:518-519, 539-540)
    rc = L.goom_scan_chain_c64(None, None, 0, 8, 4, None, None, 0, None)
    assert rc == 1 and b"empty" in L.goom_last_error()
    rc = L.goom_scan_chain_c64(None, None, 10, 8, 0, None, None, 0, None)
    assert rc == 1 and b"block_size" in L.goom_last_error()
    rc = L.goom_scan_affine_c64(None, None, None, None, None, None, 0, 4, 4, 2, None, 0, None)
    assert rc == 1
    pol = _lib.goom_reset_policy(1, 0, 0, 0, 0.99, -20.0)
    rc = L.goom_scan_selective_chain_c64(None, None, 5, 4, ctypes.byref(pol), 4, None, None, None,
                                         0, None)
    assert rc == 1  # null pointers / interval < 1
    a = _lib.goom_operand(None, 0, 1)
    rc = L.goom_lmme_c64(a, a, None, 0, 1, 0, 4, 4, None, 0, None)
    assert rc == 2  # ESHAPE
    # SSM panel kernels: shapes validated before any launch (d <= 64, T <= nC L / == nC L)
    rc = L.goom_ssm_export_c128(None, 2, 16, 65, 3, 4, 64, None, None, None, None, 0, None, None)
    assert rc == 2 and b"d <= 64" in L.goom_last_error()
    rc = L.goom_ssm_export_c128(None, 2, 16, 8, 3, 4, 65, None, None, None, None, 0, None, None)
    assert rc == 2
    rc = L.goom_ssm_export_c128(None, 0, 16, 8, 3, 4, 64, None, None, None, None, 0, None, None)
    assert rc == 0  # nothing to export
    rc = L.goom_ssm_panels_c128(None, None, None, 2, 16, 8, 3, 4, 63, 1, None, None)
    assert rc == 2 and b"T == nC * L" in L.goom_last_error()
    rc = L.goom_ssm_panels_c128(None, None, None, 2, 16, 8, 3, 4, 64, 1, None, None)
    assert rc == 1  # null pointers
    with pytest.raises(ValueError):
        _lib.check(1)
    with pytest.raises(_lib.GoomError):
        _lib.check(4)


def test_workspace_queries(lib):
    from paper_2510_03426_b200 import _lib

    L = _lib.load()
    assert L.goom_scan_chain_workspace_size(1000, 8, 32) >= 1000 * 64 * 8
    assert L.goom_scan_affine_workspace_size(100, 4, 1, 8) > 0
    pol = _lib.goom_reset_policy(1, 12, 0, 0, 0.99, -20.7)
    assert L.goom_scan_selective_chain_workspace_size(1000, 64, ctypes.byref(pol), 256) > 0
    assert L.goom_lmme_workspace_size(16, 8, 8, 8) == 0  # small kernel: in-kernel scales
    assert L.goom_lmme_workspace_size(16, 64, 64, 64) == 0  # one CTA per product, fused scales
    assert L.goom_lmme_workspace_size(16, 128, 128, 128) >= 2 * 16 * 128 * 4


def test_public_api_names():
    import paper_2510_03426_b200 as g

    for name in ("from_real", "to_real", "gmul", "gadd", "lse_reduce", "lmme", "log_matmul_exp",
                 "log_unit_norm_columns", "to_real_scaled", "GoomMatrix", "Goom", "ZeroPolicy",
                 "ScanPair", "ResetPolicy", "combine_affine", "combine_selective",
                 "scan_sequential", "scan_parallel", "scan_selective", "colinearity_policy",
                 "_lmme_arrays", "_gadd_arrays", "_log_sign_arrays", "_col_log_norms", "_Stack",
                 "_scan_affine_stack", "_selective_chain_core"):
        assert hasattr(g, name), name


def test_scalar_api_matches_reference_semantics():
    """Host-side scalar helpers (reference core.py:93-145; test_core.py:26-161)."""
    import math

    import paper_2510_03426_b200 as g

    assert abs(g.from_real(20.0855).log_mag - 3.0) < 1e-5
    assert g.from_real(-1.0) == g.Goom(0.0, -1)
    assert g.from_real(0.0).log_mag == -math.inf
    assert abs(g.ZeroPolicy.finite_floor(64).floor_value + 1416.79) < 0.01
    assert g.gadd(g.Goom(0.0, 1), g.Goom(0.0, -1)) == g.Goom(-math.inf, 1)
    assert g.to_real(g.Goom(800.0, -1)) == -math.inf
    with pytest.raises(ValueError):
        g.from_real(float("nan"))
    with pytest.raises(ValueError):
        g.lse_reduce([])


def test_empty_scans_raise_without_gpu():
    import paper_2510_03426_b200 as g

    with pytest.raises(ValueError):
        g.scan_sequential([], g.combine_affine)
    with pytest.raises(ValueError):
        g.scan_parallel([], g.combine_affine, 4)
    with pytest.raises(ValueError):
        g.scan_selective([], g.never_policy(), 4)


def test_ops_refuse_cpu_tensors():
    import torch

    import paper_2510_03426_b200  # noqa: F401

    x = torch.zeros(2, 2, dtype=torch.complex64)
    with pytest.raises(Exception):
        torch.ops.goom.lmme(x, x)


def test_lmme_broadcast_fast_path_matches_general():
    """ops._bcast_operands: the no-broadcast fast path (same leading dims, contiguous) returns
    what np.matmul broadcasting gives (batch shape, batch, per-operand matrix strides) — the
    general path is kept for broadcasts and non-contiguous operands. Shape logic only: CPU
    tensors, no GPU."""
    import math

    import torch

    from paper_2510_03426_b200 import ops

    def general(a, b):
        batch_shape = torch.broadcast_shapes(a.shape[:-2], b.shape[:-2])
        batch = 1
        for s in batch_shape:
            batch *= s
        # the reference's operand of one matrix is shared (stride 0), else one matrix per index
        sa = 0 if math.prod(a.shape[:-2]) == 1 else a.shape[-1] * a.shape[-2]
        sb = 0 if math.prod(b.shape[:-2]) == 1 else b.shape[-1] * b.shape[-2]
        return tuple(batch_shape), batch, sa, sb

    z = torch.complex64
    cases = [((5, 3, 4), (5, 4, 2)), ((1, 3, 4), (1, 4, 2)), ((3, 4), (4, 2)),
             ((2, 3, 3, 4), (2, 3, 4, 2)), ((0, 3, 4), (0, 4, 2)),
             ((5, 3, 4), (1, 4, 2)), ((5, 3, 4), (4, 2)), ((2, 1, 3, 4), (1, 6, 4, 2))]
    for sa_, sb_ in cases:
        a, b = torch.zeros(sa_, dtype=z), torch.zeros(sb_, dtype=z)
        a2, b2, batch_shape, batch, sa, sb = ops._bcast_operands(a, b)
        want = general(a, b)
        assert (tuple(batch_shape), batch, sa, sb) == want, (sa_, sb_)
        assert a2.is_contiguous() and b2.is_contiguous()
        mat = a.shape[-1] * a.shape[-2]
        assert a2.numel() in (a.numel(), batch * mat, mat)
    # a non-contiguous operand takes the general path and comes back contiguous
    a = torch.zeros(4, 5, 3, dtype=z).transpose(1, 2)
    b = torch.zeros(4, 5, 2, dtype=z)
    a2, b2, batch_shape, batch, sa, sb = ops._bcast_operands(a, b)
    assert a2.is_contiguous() and tuple(batch_shape) == (4,) and sa == 15 and sb == 10
