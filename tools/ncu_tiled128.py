"""The SSM's complex128 panel LMME (16 heads: 64x64 powers (x) 64x2048 panels, fused gadd)
for ncu: one warm + one profiled launch."""
import sys

import torch

sys.path.insert(0, ".")
import paper_2510_03426_b200 as g  # noqa: E402,F401

dev = torch.device("cuda")
A = torch.ops.goom.from_real(torch.randn(16, 64, 64, dtype=torch.float64, device=dev), float("-inf"), True)
B = torch.ops.goom.from_real(torch.randn(16, 64, 2048, dtype=torch.float64, device=dev), float("-inf"), True)
D = torch.ops.goom.from_real(torch.randn(16, 64, 2048, dtype=torch.float64, device=dev), float("-inf"), True)
for _ in range(3):
    torch.ops.goom.lmme_gadd(A, B, D)
torch.cuda.synchronize()
