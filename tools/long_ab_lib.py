"""A/B probe: the long-chain scan (T = 2^20, all prefixes) timed with libgoom.so loaded from a
given path, so two builds compare on one box (CUDA events, median of 5)."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2510_03426_b200 import _lib  # noqa: E402

_lib.load(sys.argv[1])
import paper_2510_03426_b200 as g  # noqa: E402,F401

for d in [int(x) for x in sys.argv[2].split(",")]:
    T = 1 << 20
    A = torch.ops.goom.random_normal(torch.empty(0, device="cuda"), T, d, 3, 0)
    torch.ops.goom.scan_chain_long(A, None)
    ts = []
    for _ in range(5):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        torch.ops.goom.scan_chain_long(A, None)
        e.record()
        torch.cuda.synchronize()
        ts.append(s.elapsed_time(e))
    ts.sort()
    print(f"{sys.argv[1].split('/')[-1]} d={d} median {ts[2]:.3f} ms")
