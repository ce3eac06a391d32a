"""Time the device leaf generator (tile-scaled N(0,1) leaves, d = 512) alone: GB/s written."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2510_03426_b200 import ops  # noqa: E402

T, d = int(sys.argv[1]) if len(sys.argv) > 1 else 32768, 512
dev = torch.device("cuda")
L = ops.ts_random_normal(T, d, 1, 0, dev)
torch.cuda.synchronize()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record()
for i in range(5):
    L = ops.ts_random_normal(T, d, 1, i * T, dev)
e.record()
torch.cuda.synchronize()
ms = s.elapsed_time(e) / 5
print(f"T={T} d={d}: {ms:.2f} ms per window, {T * d * d * 4 / ms / 1e6:.0f} GB/s, "
      f"{T * d * d / ms / 1e6:.0f} M normals/ms; checksum {float(L.U[:4].double().sum()):.6f}")
