"""One warm + one profiled LMME launch (for ncu -k regex:lmme_tc)."""
import sys

import torch

sys.path.insert(0, ".")
import paper_2510_03426_b200 as g  # noqa: E402

d = int(sys.argv[1]) if len(sys.argv) > 1 else 512
batch = int(sys.argv[2]) if len(sys.argv) > 2 else 256
A = torch.complex(torch.randn(batch, d, d, device="cuda"), torch.zeros(batch, d, d, device="cuda"))
B = torch.complex(torch.randn(batch, d, d, device="cuda"), torch.zeros(batch, d, d, device="cuda"))
for _ in range(3):
    torch.ops.goom.lmme(A, B)
torch.cuda.synchronize()
