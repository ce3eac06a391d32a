"""lmme_ts kernel time per epilogue kind at large batch (separates epilogue cost from the
phase-1 launch overhead)."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2510_03426_b200 import ops  # noqa: E402

d = 512
dev = torch.device("cuda")
L = ops.ts_random_normal(8192, d, 1, 0, dev)
C = ops.ts_random_normal(8192, d, 2, 0, dev)


def ev(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


for kind in (1, 2):
    for name, B, div in (("distinct B", C, 1), ("carry B", C[0:64], 128)):
        ms = ev(lambda: ops.lmme_ts(L, B, kind, b_div=div))
        print(f"kind {kind} {name} b8192: {ms:.2f} ms {2 * d**3 * 8192 / ms / 1e9:.0f} TF/s", flush=True)
for b in (128, 256, 512, 1024):
    ms = ev(lambda: ops.lmme_ts(L[0:b], C[0:b], 1), reps=10)
    print(f"kind 1 distinct b{b}: {ms * 1e3:.0f} us ({ms * 1e3 / b:.2f} us/product)", flush=True)
