"""Profiling aid (not product): step timeline of CTA 0 in the tile-resident long-chain fold (d = 16 / 32 / 64)
(scan_long_tc.cu) from the trace build (tools/tc_trace.sh -> tools/bin/libgoom_trace.so).
Rows: 0 MMA has the leaf, 1 MMA has B (issue), 2 epilogue has the accumulator, 3 row
maxima done, 4 chain maximum done, 5 B written; 6 transform has the leaf, 7 transform done."""
import ctypes
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2510_03426_b200 as g  # noqa: E402
from paper_2510_03426_b200 import harness  # noqa: E402

lib = g._lib.load(os.path.join(ROOT, "tools", "bin", "libgoom_trace.so"))
T = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 18
d = int(sys.argv[2]) if len(sys.argv) > 2 else 64
A = harness.random_chain(T, d, seed=1)
for _ in range(2):
    out = torch.ops.goom.scan_chain_long(A, None)
torch.cuda.synchronize()
buf = (ctypes.c_longlong * (8 * 256))()
lib.goom_l64_trace_read.restype = ctypes.c_int
assert lib.goom_l64_trace_read(buf) == 0
t = np.array(buf, dtype=np.int64).reshape(8, 256)
t0 = t[1, 0]
print(" g   mma_leaf mma_issue acc  rowmax chainmax bwritten | xf_leaf xf_done | step")
for i in range(1, 120):
    print(f"{i:3d} {t[0, i] - t0:8d} {t[1, i] - t0:8d} {t[2, i] - t[1, i]:5d} {t[3, i] - t[2, i]:5d}"
          f" {t[4, i] - t[3, i]:5d} {t[5, i] - t[4, i]:5d} | {t[6, i] - t0:8d} {t[7, i] - t[6, i]:5d}"
          f" | {t[1, i] - t[1, i - 1]:5d}")
