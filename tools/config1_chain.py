"""chains of 1,000 random-normal 8x8 matrices (seeds 1..30), all
prefixes, sequential fold vs parallel blocked scan — the correctness configuration
(latency-bound: 1,000 x 512 B), so only times are reported.

GPU: `scan_chain` (the A slot of the affine scan, warp-resident kernels for d <= 32) on
complex64 and complex128 GOOMs, block 1000 (= the sequential fold, scan.py:217-225) and
block 16 / 32 / 64; and the full affine scan with zero d x d biases (`scan_affine`, both
slots). CUDA events, device-resident inputs, median of 30 chains (one per seed).
CPU: the oracle port (the reference algorithm) in float64, sequential fold and blocked
scan with block 32, on the same chains. Parity: every seed's complex64 prefixes against the
float64 oracle by the §8c chain criterion (goom_testlib.chain_parity, calibrated by the
reference's own float32 runs, sequential and block 32). Prints one JSON line."""
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
from goom_testlib import chain_parity  # noqa: E402
from oracle import gooms_port as G  # noqa: E402
import paper_2510_03426_b200 as g  # noqa: E402

T, d = 1000, 8
dev = torch.device("cuda")


def ev(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return float(np.median(ts))


gpu = {}
cpu = {"seq_f64_ms": [], "blocked32_f64_ms": []}
ok = 0
fails = []
for seed in range(1, 31):
    mats = np.random.default_rng(seed).standard_normal((T, d, d))
    al, as_ = G.log_sign(mats)
    A64 = g.join(al, as_, torch.complex64)
    A128 = g.join(al, as_, torch.complex128)
    Z64 = torch.full_like(A64, complex(float("-inf"), 0.0))
    flags = torch.zeros(T, dtype=torch.uint8, device=dev)
    for name, fn in (
            ("c64_fold", lambda: torch.ops.goom.scan_chain(A64, T, None)),
            ("c64_block16", lambda: torch.ops.goom.scan_chain(A64, 16, None)),
            ("c64_block32", lambda: torch.ops.goom.scan_chain(A64, 32, None)),
            ("c64_block64", lambda: torch.ops.goom.scan_chain(A64, 64, None)),
            ("c128_fold", lambda: torch.ops.goom.scan_chain(A128, T, None)),
            ("c128_block32", lambda: torch.ops.goom.scan_chain(A128, 32, None)),
            ("c64_affine_block32", lambda: torch.ops.goom.scan_affine(A64, Z64, flags, 32))):
        gpu.setdefault(name, []).append(ev(fn))
    out = torch.ops.goom.scan_chain(A64, 32, None).cpu().numpy()
    gl, gs = G.split_complex(out)
    t0 = time.perf_counter()
    want = G.chain_blocked(al, as_, T)
    cpu["seq_f64_ms"].append((time.perf_counter() - t0) * 1e3)
    t0 = time.perf_counter()
    G.chain_blocked(al, as_, 32)
    cpu["blocked32_f64_ms"].append((time.perf_counter() - t0) * 1e3)
    # the reference's own float32 runs: its float32 path converts the float32 matrices
    # (log_sign of x.astype(float32), as tests/golden/make_golden.py records), sequential
    # and block 32; the float64 logs rounded to float32 (the GPU's exact input) beside them
    l32, s32 = G.log_sign(mats.astype(np.float32))
    r32, q32 = al.astype(np.float32), as_.astype(np.float32)
    refs = [G.chain_blocked(l32, s32, T), G.chain_blocked(l32, s32, 32),
            G.chain_blocked(r32, q32, T), G.chain_blocked(r32, q32, 32)]
    r = chain_parity(gl, gs, al, as_, want, refs)
    ok += bool(r["ok"])
    if not r["ok"]:
        fails.append(dict(seed=seed, bad=len(r["bad"]), flips=r["flips"],
                          scaled_bad=len(r["scaled_bad"]), scaled_max=r["scaled_max"],
                          worst_ratio=float(np.max(r["e_gpu"] / np.maximum(4 * r["e_ref"], 2e-4)))))
print(json.dumps({
    "config": "chain_d8_T1000", "seeds": 30, "T": T, "d": d,
    "gpu_ms_median": {k: float(np.median(v)) for k, v in gpu.items()},
    "cpu_ms_median": {k: float(np.median(v)) for k, v in cpu.items()},
    "cpu": "oracle port (reference algorithm, float64 numpy), 1 host thread per chain",
    "parity_seeds_ok": ok, "parity_fails": fails,
    "parity": "complex64 block 32 vs float64 sequential oracle, §8c calibrated chain criterion "
              "(tests/goom_testlib.chain_parity)",
}))
