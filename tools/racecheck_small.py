"""Probe: the lane-group long-chain fold (scan_long.cu, d = 5 / 8 / 16 / 32, several recursion
levels, a carry) under compute-sanitizer --tool racecheck (profiles/r2_racecheck.txt)."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2510_03426_b200 as g  # noqa: E402
from oracle import gooms_port as G  # noqa: E402

g._lib.load()
rng = np.random.default_rng(0)
for d, T in ((8, 300), (5, 140), (16, 40), (32, 40)):
    A = g.join(*G.log_sign(rng.standard_normal((T, d, d))), torch.complex64)
    torch.ops.goom.scan_chain_long(A, A[0])
torch.cuda.synchronize()
print("done")
