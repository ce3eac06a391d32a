"""A/B probe: the config-2 LMME from a second libgoom.so build (raw C-ABI call through ctypes)
against the loaded one (torch.ops.goom.lmme), bit for bit, at the given d (batch 1024)."""
import ctypes
import sys

import torch

sys.path.insert(0, ".")
from paper_2510_03426_b200 import _lib  # noqa: E402

_lib.load(sys.argv[1])
import paper_2510_03426_b200 as g  # noqa: E402,F401

other = ctypes.CDLL(sys.argv[2])
fn = other.goom_lmme_c64
fn.restype = ctypes.c_int
fn.argtypes = _lib.SIGNATURES["goom_lmme_c64"][1]
wsz = other.goom_lmme_workspace_size
wsz.restype = ctypes.c_size_t
wsz.argtypes = _lib.SIGNATURES["goom_lmme_workspace_size"][1]
for d in [int(x) for x in sys.argv[3].split(",")]:
    batch = 1024
    torch.manual_seed(d)
    A = torch.ops.goom.from_real(torch.randn(batch, d, d, device="cuda") * 3, float("-inf"), False)
    B = torch.ops.goom.from_real(torch.randn(batch, d, d, device="cuda") * 3, float("-inf"), False)
    ref = torch.ops.goom.lmme(A, B)
    out = torch.empty_like(ref)
    n = int(wsz(batch, d, d, d))
    ws = torch.empty(max(n, 1), dtype=torch.uint8, device="cuda")
    rc = fn(_lib.goom_operand(A.data_ptr(), d * d, 1), _lib.goom_operand(B.data_ptr(), d * d, 1),
            out.data_ptr(), d * d, batch, d, d, d, ws.data_ptr() if n else None, n,
            ctypes.c_void_p(torch.cuda.current_stream().cuda_stream))
    torch.cuda.synchronize()
    print(f"d={d} rc={rc} bitwise equal: {torch.equal(torch.view_as_real(out), torch.view_as_real(ref))}")
