"""One warm + profiled batched complex64 LMME at d (default 64) for ncu."""
import sys

import torch

sys.path.insert(0, ".")
import paper_2510_03426_b200 as g  # noqa: E402,F401

d = int(sys.argv[1]) if len(sys.argv) > 1 else 64
dev = torch.device("cuda")
A = torch.ops.goom.from_real(torch.randn(1024, d, d, device=dev), float("-inf"), False)
B = torch.ops.goom.from_real(torch.randn(1024, d, d, device=dev), float("-inf"), False)
for _ in range(3):
    torch.ops.goom.lmme(A, B)
torch.cuda.synchronize()
