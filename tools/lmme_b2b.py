"""Probe: n back-to-back batched complex64 LMMEs (config 2's shape) between two CUDA events,
no L2 flush in between (each call moves 24 d^2 batch bytes; at d = 64, batch 1024: 100 MB, on
the order of the 126 MB L2). Prints the per-call average next to the single-call median of
tools/lmme_prof2.py's method, to separate launch-to-launch overhead from in-kernel time."""
import sys

import torch

sys.path.insert(0, ".")
import paper_2510_03426_b200 as g  # noqa: E402

d = int(sys.argv[1]) if len(sys.argv) > 1 else 64
batch = int(sys.argv[2]) if len(sys.argv) > 2 else 1024
n = int(sys.argv[3]) if len(sys.argv) > 3 else 20
g._lib.load()
As = [torch.ops.goom.from_real(torch.randn(batch, d, d, device="cuda"), float("-inf"), False)
      for _ in range(4)]
Bs = [torch.ops.goom.from_real(torch.randn(batch, d, d, device="cuda"), float("-inf"), False)
      for _ in range(4)]
for i in range(3):
    torch.ops.goom.lmme(As[i % 4], Bs[i % 4])
torch.cuda.synchronize()
res = []
for rep in range(5):
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for i in range(n):
        torch.ops.goom.lmme(As[i % 4], Bs[i % 4])  # 4 operand sets: 400 MB, beyond the L2
    e.record()
    torch.cuda.synchronize()
    res.append(s.elapsed_time(e) / n)
res.sort()
gbs = 24 * d * d * batch / (res[len(res) // 2] * 1e-3) / 1e9
print(f"d={d} batch={batch} back-to-back x{n}: {res[len(res) // 2] * 1e3:.1f} us per call ({gbs:.0f} GB/s)")
