"""CUDA-event breakdown of one d=512 harness window (T=8192, block 64) into its launches'
shapes: leaf generation, phase 1 (63 x batch 128, tile-scaled out), phase 2 (Kogge-Stone,
7 launches), phase 3 (batch 8192, digest epilogue). Approximate shapes via ops.lmme_ts."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2510_03426_b200 import ops  # noqa: E402

d, T, s = 512, int(sys.argv[1]) if len(sys.argv) > 1 else 8192, int(sys.argv[2]) if len(sys.argv) > 2 else 64
nb = T // s
dev = torch.device("cuda")


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


L = ops.ts_random_normal(T, d, 1, 0, dev)
C = ops.ts_random_normal(nb, d, 2, 0, dev)
A128, B128 = L[0:nb], C
t_rng = ev(lambda: ops.ts_random_normal(T, d, 3, 0, dev))
t_p1 = ev(lambda: ops.lmme_ts(A128, B128, 1)) * (s - 1)
t_p2 = sum(ev(lambda: ops.lmme_ts(L[0:nb - h], C[0:nb - h], 1)) for h in [1 << j for j in range(7) if (1 << j) < nb])
t_p3 = ev(lambda: ops.lmme_ts(L, C, 2, b_div=s))
full = ev(lambda: ops.chain_ts(L, s, None, digests=True, carry_out=True), reps=2)
tot = t_rng + t_p1 + t_p2 + t_p3
print(f"T={T} block={s}: rng {t_rng:.2f} ms | phase1 {t_p1:.2f} ms ({t_p1/(s-1)*1e3:.0f} us x {s-1}) | "
      f"phase2 tree {t_p2:.2f} ms | phase3 {t_p3:.2f} ms | sum {tot:.2f} ms -> {T/tot*1e3:.0f} mat/s | "
      f"chain_ts call {full:.2f} ms (+rng {T/(full+t_rng)*1e3:.0f} mat/s)")
