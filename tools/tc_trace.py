"""Profiling aid (not product): ring timeline of CTA 0 in the fused one-SM LMME (config 2,
d = 128) from the GOOM_TC_TRACE build (tools/tc_trace.sh -> tools/bin/libgoom_trace.so).
Rows: 0 loader issue, 1 transform warp 0 starts waiting, 2 data landed, 3 MMA issue,
4 transform done; per tile 5/6/7 epilogue wait start / accumulator full / done."""
import ctypes
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2510_03426_b200 as g  # noqa: E402

lib = g._lib.load(os.path.join(ROOT, "tools", "bin", "libgoom_trace.so"))
d = int(sys.argv[1]) if len(sys.argv) > 1 else 128
batch = int(sys.argv[2]) if len(sys.argv) > 2 else 1024
A = torch.ops.goom.from_real(torch.randn(batch, d, d, device="cuda"), float("-inf"), False)
B = torch.ops.goom.from_real(torch.randn(batch, d, d, device="cuda"), float("-inf"), False)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for _ in range(3):
    flush.add_(1)
    torch.ops.goom.lmme(A, B)
torch.cuda.synchronize()
buf = (ctypes.c_longlong * (8 * 256))()
lib.goom_tc_trace_read.restype = ctypes.c_int
assert lib.goom_tc_trace_read(buf) == 0
t = np.array(buf, dtype=np.int64).reshape(8, 256)
nk = d // 16
t0 = t[0, 0]
n = int((t[0] != 0).sum())
print(f"positions {n}, span {(t[4, n - 1] - t0)} clk")
print(" g type tile kb  issue  land-issue  wait->land  xform  mma-land")
for i in range(n):
    if i < nk:
        typ, tile, kb = "S", 0, i
    else:
        j = i - nk
        per = 2 * nk
        tile, r = divmod(j, per)
        kb, sub = divmod(r, 2)
        typ = "M" if sub == 0 else "S"
        if typ == "S":
            tile += 1
    mma = (t[3, i] - t[2, i]) if typ == "M" else 0
    print(f"{i:3d} {typ} {tile:3d} {kb:2d} {t[0, i] - t0:7d} {t[2, i] - t[0, i]:7d} "
          f"{t[2, i] - t[1, i]:7d} {t[4, i] - t[2, i]:6d} {mma:7d}")
for lt in range(8):
    if t[5, lt] == 0:
        break
    print(f"epi tile {lt}: wait {t[5, lt] - t0} full {t[6, lt] - t0} done {t[7, lt] - t0} "
          f"(busy {t[7, lt] - t[6, lt]})")
