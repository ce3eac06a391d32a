"""Per-rank time of a time-sharded d = 512 chain (T = 2^20 over G ranks), measured on ONE
GPU: the resident two-pass shard (run_shard_resident, local products kept) and the
recompute path (shard_total + run_chain), with an identity exchange in place of the NCCL
all-gather (a 2 MiB all-gather is negligible next to either). Prints JSON lines."""
import json
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_2510_03426_b200 import harness, sharded  # noqa: E402

T, d, block = 1 << 20, 512, 128
for G in (8, 4, 2):
    n = T // G
    for mode in ("resident", "recompute"):
        if mode == "resident":
            w = 32768  # sharded.run_chain_sharded's choice: shrink only if all then fits
            while w > 8192 and not sharded.resident_fits(n, d, w):
                w //= 2
            if not sharded.resident_fits(n, d, w):
                w = 32768
            fn = lambda: sharded.run_shard_resident(n, d, 1, 0, w, block, lambda t: t)  # noqa: E731
        else:
            w = 32768
            fn = lambda: harness.run_chain(n, d, 1, w, block, carry=sharded.shard_total(  # noqa: E731
                n, d, 1, 0, w, block))
        fn()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        print(json.dumps({"G": G, "mode": mode, "window": w, "per_rank_s": dt,
                          "projected_matrices_per_s": T / dt}), flush=True)
        torch.cuda.empty_cache()
