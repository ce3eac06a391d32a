"""Probe: host time per call of the LMME boundary layers on a tiny problem (the GPU finishes
each call in a few microseconds, so the host is the bound): torch.ops.goom.lmme (custom-op
dispatch + _lmme_impl), ops._lmme_impl direct, the raw C-ABI call through ctypes, and the
drop-in core.lmme on GoomMatrix-backed tensors."""
import sys
import time

import torch

sys.path.insert(0, ".")
import paper_2510_03426_b200 as g  # noqa: E402
from paper_2510_03426_b200 import ops, _lib  # noqa: E402

lib = _lib.load()
for d, batch in ((8, 1), (64, 16)):
    A = torch.ops.goom.from_real(torch.randn(batch, d, d, device="cuda"), float("-inf"), False)
    B = torch.ops.goom.from_real(torch.randn(batch, d, d, device="cuda"), float("-inf"), False)
    C = torch.empty_like(A)
    nws = int(lib.goom_lmme_workspace_size(batch, d, d, d))
    ws = torch.empty(max(nws, 1), dtype=torch.uint8, device="cuda")
    stream = ops._stream()

    def raw():
        _lib.call("goom_lmme_c64", _lib.goom_operand(A.data_ptr(), d * d, 1),
                  _lib.goom_operand(B.data_ptr(), d * d, 1), C.data_ptr(), d * d, batch, d, d, d,
                  ws.data_ptr() if nws else None, nws, stream)

    for name, fn in (("torch.ops.goom.lmme", lambda: torch.ops.goom.lmme(A, B)),
                     ("ops.lmme (direct)", lambda: ops.lmme(A, B)),
                     ("ops._lmme_impl", lambda: ops._lmme_impl(A, B, None)),
                     ("C-ABI via ctypes", raw)):
        for _ in range(50):
            fn()
        torch.cuda.synchronize()
        n = 2000
        t0 = time.perf_counter()
        for _ in range(n):
            fn()
        t1 = time.perf_counter()
        torch.cuda.synchronize()
        t2 = time.perf_counter()
        print(f"d={d} batch={batch} {name:22s} host {1e6 * (t1 - t0) / n:7.1f} us/call, "
              f"host+device {1e6 * (t2 - t0) / n:7.1f} us/call")
