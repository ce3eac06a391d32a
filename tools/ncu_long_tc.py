"""Profiling aid: one long-chain scan (T = 2^18) for ncu -k regex:long_fold_tc."""
import sys
import torch
sys.path.insert(0, ".")
import paper_2510_03426_b200 as g
from paper_2510_03426_b200 import harness
g._lib.load()
d = int(sys.argv[1])
A = harness.random_chain(1 << 18, d, seed=1)
out = torch.ops.goom.scan_chain_long(A, None)
torch.cuda.synchronize()
