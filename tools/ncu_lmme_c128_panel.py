"""One warm + profiled complex128 LMME of config 5's shape (16 heads: 64 x 64 powers times
64 x 2048 panels) for ncu; prints the event-timed median of 20 launches."""
import sys

import torch

sys.path.insert(0, ".")
import paper_2510_03426_b200 as g  # noqa: E402,F401

dev = torch.device("cuda")
H, d, N = 16, 64, int(sys.argv[1]) if len(sys.argv) > 1 else 2048
A = torch.ops.goom.from_real(torch.randn(H, d, d, device=dev, dtype=torch.float64), float("-inf"), True)
B = torch.ops.goom.from_real(torch.randn(H, d, N, device=dev, dtype=torch.float64) * 30, float("-inf"), True)
for _ in range(3):
    torch.ops.goom.lmme(A, B)
ts = []
for _ in range(20):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    torch.ops.goom.lmme(A, B)
    b.record()
    torch.cuda.synchronize()
    ts.append(a.elapsed_time(b) * 1e3)
ts.sort()
print(f"c128 lmme {H}x{d}x{d} @ {d}x{N}: {ts[10]:.1f} us, GEMM {2 * H * d * d * N / ts[10] / 1e6:.2f} TF/s")
