"""the batched LMME (torch.ops.goom.lmme, complex64 GOOMs in and out)
at d = 64 .. 1024, batch 1024 products of N(0,1) matrices, on 1 B200.

Per d: CUDA-event time of one batched call (an L2-sized buffer is rewritten before each
timed call, so operands come from HBM), products/s, algorithmic GB/s (24 d^2 B per product:
read A, B, write C as complex64) and TF/s (2 d^3), and the fraction of the bound
min(HBM, 3xTF32): bound time = max(bytes / HBM peak, flops / (bf16 dense / 6)), both peaks
from MEASURED_PEAKS.json (HBM copy GB/s; burst dense bf16 / 6). Parity: two products per d against the oracle
(float64 restatement of core.py:242-261) by the §8c metric. CPU baseline: the oracle port
in float32 (numpy / OpenBLAS, all host threads) on a 16-product sample at each d.
Prints one JSON line."""
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import gooms_port as G  # noqa: E402
import paper_2510_03426_b200 as g  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
HBM = peaks["hbm_gbs"] * 1e9
# an isolated batched call is a short burst: the BURST bf16 peak / 6 (3xTF32 at half the bf16
# rate, three MMAs per product) is its denominator, not the sustained one of a long step
TC = peaks["bf16_tflops"] * 1e12 / 6.0
dev = torch.device("cuda")
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)


def timed(fn, reps=5):
    ts = []
    for _ in range(reps):
        flush.add_(1)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) / 1e3)
    return float(np.median(ts))


rows = []
for d in (64, 128, 256, 512, 1024):
    batch = 1024
    gen = torch.Generator(device=dev).manual_seed(d)
    ra = torch.randn(batch, d, d, device=dev, generator=gen)
    rb = torch.randn(batch, d, d, device=dev, generator=gen)
    A = torch.ops.goom.from_real(ra, float("-inf"), False)
    B = torch.ops.goom.from_real(rb, float("-inf"), False)
    del ra, rb
    C = torch.ops.goom.lmme(A, B)
    torch.cuda.synchronize()
    t = timed(lambda: torch.ops.goom.lmme(A, B))
    # kernel breakdown of one call (CUPTI records via torch.profiler, no replay)
    from torch.profiler import ProfilerActivity, profile
    flush.add_(1)
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        torch.ops.goom.lmme(A, B)
        torch.cuda.synchronize()
    kern = {}
    for e in prof.events():
        if e.device_type.name == "CUDA":
            nm = e.name.replace("(anonymous namespace)::", "").replace("void ", "")
            nm = nm.split("(")[0].split("<")[0].split("::")[-1]
            kern[nm] = kern.get(nm, 0.0) + e.device_time_total / 1e3
    by, fl = 24.0 * d * d * batch, 2.0 * d ** 3 * batch
    bound = max(by / HBM, fl / TC)
    # parity on two products against the float64 oracle (sign exact where kappa >= 1e-4)
    err = 0.0
    flips = 0
    for i in (0, batch - 1):
        al, as_ = G.split_complex(A[i].cpu().numpy())
        bl, bs = G.split_complex(B[i].cpu().numpy())
        ol, os_ = G.lmme(al, as_, bl, bs)
        cl, cs = G.split_complex(C[i].cpu().numpy())
        kl, _ = G.lmme(al, np.ones_like(as_), bl, np.ones_like(bs))
        kappa = np.exp(ol - kl)
        m = kappa >= 1e-2
        err = max(err, float(np.max(np.abs(cl - ol)[m] / np.maximum(1.0, np.abs(ol[m])))))
        flips += int(np.sum((cs != os_) & (kappa >= 1e-4)))
    # CPU: oracle float32 on 16 products
    al32 = np.stack([G.split_complex(A[i].cpu().numpy(), np.float32)[0] for i in range(16)])
    as32 = np.stack([G.split_complex(A[i].cpu().numpy(), np.float32)[1] for i in range(16)])
    bl32 = np.stack([G.split_complex(B[i].cpu().numpy(), np.float32)[0] for i in range(16)])
    bs32 = np.stack([G.split_complex(B[i].cpu().numpy(), np.float32)[1] for i in range(16)])
    t0 = time.perf_counter()
    G.lmme(al32, as32, bl32, bs32)
    cpu = 16 / (time.perf_counter() - t0)
    rows.append(dict(d=d, batch=batch, ms=t * 1e3, products_per_s=batch / t,
                     gbs=by / t / 1e9, tflops=fl / t / 1e12,
                     bound="hbm" if by / HBM >= fl / TC else "tensor",
                     roofline_frac=bound / t, parity_rel_log=err, sign_flips=flips,
                     cpu_products_per_s=cpu, kernels_ms=kern))
    print(json.dumps(rows[-1]), file=sys.stderr, flush=True)
    del A, B, C
    torch.cuda.empty_cache()
print(json.dumps({"config": "lmme_sweep", "dtype": "complex64 (3xTF32 on tcgen05 for d >= 64)",
                  "hbm_peak_gbs": HBM / 1e9, "tensor_peak_tflops_3xtf32": TC / 1e12,
                  "peaks": "MEASURED_PEAKS.json (copy GB/s; burst dense bf16 / 6)",
                  "cpu": f"oracle port float32, numpy/OpenBLAS, {os.cpu_count()} host threads",
                  "rows": rows}))
