"""Quick CUDA-event timing of the batched LMME (config 2 sweep) and chain scan."""
import json
import sys
import time

import torch

sys.path.insert(0, ".")
import paper_2510_03426_b200 as g  # noqa: E402


def bench(fn, iters=5, warm=2):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(iters):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / iters


out = {}
for backend in [int(b) for b in (sys.argv[1].split(",") if len(sys.argv) > 1 else ["0"])]:
    g._lib.set_backend(backend)
    for d in (64, 128, 256, 512, 1024):
        batch = 1024 if d <= 512 else 256
        A = torch.complex(torch.randn(batch, d, d, device="cuda"), torch.zeros(batch, d, d, device="cuda"))
        B = torch.complex(torch.randn(batch, d, d, device="cuda"), torch.zeros(batch, d, d, device="cuda"))
        ms = bench(lambda: torch.ops.goom.lmme(A, B))
        tf = 2 * d**3 * batch / (ms * 1e-3) / 1e12
        gbs = 24 * d * d * batch / (ms * 1e-3) / 1e9
        out[f"b{backend}_lmme_d{d}"] = dict(ms=ms, per_s=batch / (ms * 1e-3), tflops=tf, gbs=gbs)
        print(f"backend {backend} d={d} batch={batch}: {ms:.3f} ms  {batch/(ms*1e-3):.0f} prod/s  {tf:.1f} TF/s  {gbs:.0f} GB/s", flush=True)
        del A, B
    for d, T, blk in ((8, 1000, 32), (64, 4096, 64), (512, 512, 32)):
        A = torch.complex(torch.randn(T, d, d, device="cuda"), torch.zeros(T, d, d, device="cuda"))
        ms = bench(lambda: g.scan_chain(A, blk), iters=3, warm=1)
        print(f"backend {backend} chain d={d} T={T} block={blk}: {ms:.3f} ms  {T/(ms*1e-3):.0f} mat/s", flush=True)
        out[f"b{backend}_chain_d{d}_T{T}"] = dict(ms=ms, per_s=T / (ms * 1e-3))
json.dump(out, open("gpurun_out/probe.json", "w"), indent=1)
