"""Probe: a small run of the kernels changed in round 2 (leaf generator, long-chain scan, fused
config-2 LMMEs) for compute-sanitizer --tool memcheck (0 errors, profiles/r2_memcheck.txt)."""
import sys, torch, numpy as np
sys.path.insert(0, ".")
import paper_2510_03426_b200 as g
from paper_2510_03426_b200 import ops
g._lib.load()
dev = torch.device("cuda")
for T in (1, 3, 7):
    L = ops.ts_random_normal(T, 256, 9, 5, dev)
rng = np.random.default_rng(0)
from oracle import gooms_port as G
for d, T in ((8, 300), (8, 1100), (16, 300), (5, 700)):
    A = g.join(*G.log_sign(rng.standard_normal((T, d, d))), torch.complex64)
    torch.ops.goom.scan_chain_long(A, A[0])
A = torch.ops.goom.from_real(torch.randn(6, 256, 256, device=dev), float("-inf"), False)
torch.ops.goom.lmme(A, A)
A = torch.ops.goom.from_real(torch.randn(5, 128, 128, device=dev), float("-inf"), False)
torch.ops.goom.lmme(A, A)
torch.cuda.synchronize()
print("done")
