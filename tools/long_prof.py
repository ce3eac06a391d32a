"""Profiling driver for the long-chain small-d engine (scan_long.cu): T = 2^20 chain of
N(0,1) d x d complex64 leaves through torch.ops.goom.scan_chain_long, `reps` times.
Used under ncu (tools/gpu/*.sh); prints the CUDA-event time of the last rep."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2510_03426_b200 as g  # noqa: E402
from paper_2510_03426_b200 import harness  # noqa: E402

d = int(sys.argv[1]) if len(sys.argv) > 1 else 8
T = int(sys.argv[2]) if len(sys.argv) > 2 else 1 << 20
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 1
g._lib.load()
A = harness.random_chain(T, d, seed=d)
for _ in range(reps):
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    out = torch.ops.goom.scan_chain_long(A, None)
    e.record()
    torch.cuda.synchronize()
    del out
print(f"d={d} T={T} {s.elapsed_time(e):.3f} ms")
