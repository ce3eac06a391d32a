import sys, time
import numpy as np
import torch
sys.path.insert(0, ".")
import paper_2510_03426_b200 as g
from paper_2510_03426_b200 import scan as S
from paper_2510_03426_b200.core import GoomMatrix
g._lib.load()
rng = np.random.default_rng(49)
T, d = 2**15, 8
alog = rng.uniform(-1, 1, (T, d, d)); asign = rng.choice([-1.0, 1.0], (T, d, d))
leaves = [S.ScanPair(GoomMatrix(alog[t], asign[t]), GoomMatrix.zeros(d, d)) for t in range(T)]
for rep in range(2):
    torch.cuda.synchronize()
    t0 = time.perf_counter(); st = S._Stack.from_pairs(leaves); torch.cuda.synchronize(); t1 = time.perf_counter()
    out = S._scan_affine_stack(st, T); torch.cuda.synchronize(); t2 = time.perf_counter()
    outp = S._scan_affine_stack(st, 256); torch.cuda.synchronize(); t3 = time.perf_counter()
    pairs = outp.to_pairs(); t4 = time.perf_counter()
    lm = pairs[-1].A.log_mag; t5 = time.perf_counter()
    print(f"from_pairs {t1-t0:.3f} seqscan {t2-t1:.3f} parscan {t3-t2:.3f} to_pairs {t4-t3:.3f} log_mag {t5-t4:.4f}")
import cProfile, pstats
cProfile.run("S.scan_parallel(leaves, S.combine_affine, block_size=256, workers=4)", "/tmp/pp.out")
pstats.Stats("/tmp/pp.out").sort_stats("cumtime").print_stats(12)
t0 = time.perf_counter(); S.scan_sequential(leaves, S.combine_affine); t1 = time.perf_counter()
print(f"scan_sequential {t1 - t0:.3f} s")
cProfile.run("S.scan_sequential(leaves, S.combine_affine)", "/tmp/ps.out")
pstats.Stats("/tmp/ps.out").sort_stats("tottime").print_stats(10)
