"""The SSM chunk-carry LMME shape (16 heads: 64 x 64 A^L times 64 x 32 entry states, fused
bias gadd) on the complex128 whole-product kernel, for ncu; prints the event-timed median."""
import sys

import torch

sys.path.insert(0, ".")
import paper_2510_03426_b200 as g  # noqa: E402,F401
from paper_2510_03426_b200 import ops  # noqa: E402

dev = torch.device("cuda")
H, d, S = 16, 64, 32
f = lambda *s: torch.ops.goom.from_real(torch.randn(*s, device=dev, dtype=torch.float64), float("-inf"), True)
A, X, Dm = f(H, d, d), f(H, d, S), f(H, d, S)
out = torch.empty_like(Dm)
for _ in range(3):
    ops.lmme_indexed(A, 1, X, 1, H, Dm, out=out)
ts = []
for _ in range(21):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    ops.lmme_indexed(A, 1, X, 1, H, Dm, out=out)
    b.record()
    torch.cuda.synchronize()
    ts.append(a.elapsed_time(b) * 1e3)
print(f"whole c128 {H} x ({d}x{d} @ {d}x{S}) + gadd: {sorted(ts)[10]:.1f} us")
