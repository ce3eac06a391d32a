"""One warm + profiled lmme_ts launch (phase-3 shape: digest epilogue, carry per 64)."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2510_03426_b200 import ops  # noqa: E402

kind = int(sys.argv[1]) if len(sys.argv) > 1 else 2
batch = int(sys.argv[2]) if len(sys.argv) > 2 else 1024
d = 512
dev = torch.device("cuda")
L = ops.ts_random_normal(batch, d, 1, 0, dev)
C = ops.ts_random_normal(batch // 64, d, 2, 0, dev)
for _ in range(3):
    ops.lmme_ts(L, C, kind, b_div=64)
torch.cuda.synchronize()
