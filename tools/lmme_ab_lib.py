"""A/B probe: the config-2 LMME timed (tools/lmme_prof2.py's method) with libgoom.so loaded from
a given path (e.g. a build of an earlier commit), so two builds compare on the same box."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2510_03426_b200 import _lib  # noqa: E402

path = sys.argv[1]
_lib.load(path)  # cached: every op below calls this library
import paper_2510_03426_b200 as g  # noqa: E402,F401

for d in [int(x) for x in sys.argv[2].split(",")]:
    batch = 1024
    A = torch.ops.goom.from_real(torch.randn(batch, d, d, device="cuda"), float("-inf"), False)
    B = torch.ops.goom.from_real(torch.randn(batch, d, d, device="cuda"), float("-inf"), False)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    ts = []
    for _ in range(15):
        flush.add_(1)
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        torch.ops.goom.lmme(A, B)
        e.record()
        torch.cuda.synchronize()
        ts.append(s.elapsed_time(e))
    ts.sort()
    print(f"{path.split('/')[-1]} d={d} median {ts[len(ts) // 2] * 1e3:.1f} us")
