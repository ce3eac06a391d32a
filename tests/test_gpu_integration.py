"""INTEGRATION.md §2's ctypes binding, executed as documented: `_lmme_arrays` (core.py:242-261)
bound straight to goom_lmme_c128 — the binding a `gooms` maintainer would add — must give the
reference's 2x2 KAT (test_core.py:184-188) and match the oracle on a random batch."""

import ctypes
import os

import numpy as np
import pytest
import torch

from oracle import gooms_port as G

pytestmark = pytest.mark.gpu
LIB = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                   "paper_2510_03426_b200", "libgoom.so")


@pytest.fixture(scope="module")
def lmme_arrays():
    _lib = ctypes.CDLL(LIB)

    class goom_operand(ctypes.Structure):
        _fields_ = [("ptr", ctypes.c_void_p), ("stride", ctypes.c_int64), ("div", ctypes.c_int64)]

    _lib.goom_lmme_c128.argtypes = [goom_operand, goom_operand, ctypes.c_void_p, ctypes.c_int64,
                                    ctypes.c_int64, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                    ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p]
    _lib.goom_lmme_workspace_size_c128.restype = ctypes.c_size_t
    _lib.goom_last_error.restype = ctypes.c_char_p

    def _lmme_arrays(alog, asign, blog, bsign):
        to_goom = lambda l, s: torch.complex(torch.as_tensor(l, dtype=torch.float64),  # noqa: E731
                                             torch.where(torch.as_tensor(s) < 0, np.pi, 0.0)
                                             .double()).cuda().contiguous()
        A, B = to_goom(alog, asign), to_goom(blog, bsign)
        batch = int(np.prod(A.shape[:-2], dtype=np.int64))
        n, k, m = A.shape[-2], A.shape[-1], B.shape[-1]
        C = torch.empty(A.shape[:-2] + (n, m), dtype=torch.complex128, device="cuda")
        nws = _lib.goom_lmme_workspace_size_c128(batch, n, k, m)
        ws = torch.empty(nws, dtype=torch.uint8, device="cuda")
        rc = _lib.goom_lmme_c128(goom_operand(A.data_ptr(), n * k, 1),
                                 goom_operand(B.data_ptr(), k * m, 1), C.data_ptr(), n * m,
                                 batch, n, k, m, ws.data_ptr(), nws,
                                 torch.cuda.current_stream().cuda_stream)
        if rc:
            raise ValueError(_lib.goom_last_error().decode())
        out = C.cpu()
        return out.real.numpy(), np.where(np.cos(out.imag.numpy()) < 0, -1.0, 1.0)

    return _lmme_arrays


def test_documented_binding_kat_and_oracle(lmme_arrays):
    al, as_ = G.log_sign(np.array([[1.0, 2.0], [3.0, 4.0]]))
    bl, bs = G.log_sign(np.array([[5.0, 6.0], [7.0, 8.0]]))
    l, s = lmme_arrays(al, as_, bl, bs)
    np.testing.assert_allclose(s * np.exp(l), [[19.0, 22.0], [43.0, 50.0]], rtol=1e-13)
    rng = np.random.default_rng(3)
    al, as_ = G.log_sign(rng.standard_normal((5, 24, 40)))
    bl, bs = G.log_sign(rng.standard_normal((5, 40, 16)))
    l, s = lmme_arrays(al, as_, bl, bs)
    wl, ws = G.lmme(al, as_, bl, bs)
    assert G.rel_log_diff(l, wl) < 1e-10
    np.testing.assert_array_equal(s, ws)
