"""Tile-scaled engine checks vs the complex64 path + timing (GPU; run under timeout)."""
import os
import sys
import time

import torch

sys.path.insert(0, ".")
import paper_2510_03426_b200 as g  # noqa: E402
from paper_2510_03426_b200 import harness, ops  # noqa: E402


def rgoom(b, d, seed):
    gen = torch.Generator(device="cuda").manual_seed(seed)
    x = torch.randn(b, d, d, device="cuda", generator=gen)
    return torch.complex(x.abs().log(), torch.where(x < 0, torch.tensor(3.14159265, device="cuda"), 0.0))


def cmp(name, got, want):
    d = (got.real - want.real).abs() / want.real.abs().clamp_min(1)
    fin = torch.isfinite(d)
    sd = ((got.imag != 0) != (want.imag != 0)) & (want.real > want.real.amax(dim=(-1, -2), keepdim=True) - 10)
    print(f"{name}: max rel-log {d[fin].max().item():.3e} mean {d[fin].mean().item():.3e} "
          f"nonfinite {(~fin).sum().item()} sign diffs(|x| within e^10 of max) {sd.sum().item()}", flush=True)


def timeit(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / reps


torch.manual_seed(0)
for d in (256, 512, 1024):
    A, B = rgoom(8, d, 1), rgoom(8, d, 2)
    want = torch.ops.goom.lmme(A, B)
    ta, tb = ops.ts_from_goom(A), ops.ts_from_goom(B)
    cmp(f"d={d} ts->goom import/export", ops.ts_to_goom(ta), A)
    cmp(f"d={d} lmme_ts kind0", ops.lmme_ts(ta, tb, 0), want)
    cmp(f"d={d} lmme_ts kind1", ops.ts_to_goom(ops.lmme_ts(ta, tb, 1)), want)
    dg = ops.lmme_ts(ta, tb, 2)
    dw = torch.ops.goom.digest(want)
    print(f"d={d} digest max|diff| {(dg - dw).abs().max().item():.3e}  got {dg[0].tolist()} want {dw[0].tolist()}", flush=True)
    # broadcast B (phase-3 shape)
    want_b = torch.ops.goom.lmme(A, B[:1].expand(8, d, d).contiguous())
    cmp(f"d={d} lmme_ts broadcast B", ops.lmme_ts(ta, tb[0:1], 0), want_b)

# chain: TS engine vs complex64 engine (GOOM_CHAIN_TS read once per process -> compare to tc path)
for d, T, blk in ((512, 300, 64), (256, 100, 16)):
    A = rgoom(T, d, 5)
    out_ts = g.scan_chain(A, blk)
    leaves = ops.ts_from_goom(A)
    P, dg, c = ops.chain_ts(leaves, blk, None, out=True, digests=True, carry_out=True)
    cmp(f"chain d={d} T={T}: scan_chain(ts) vs chain_ts out", out_ts, P)
    cmp(f"chain d={d} T={T}: carry-out vs last prefix", ops.ts_to_goom(c)[0], P[-1])
    dw = torch.ops.goom.digest(P)
    print(f"chain digests max|diff| {(dg - dw).abs().max().item():.3e}", flush=True)
    # reference: sequential fold with the tc2 complex64 lmme
    seq = [A[0]]
    for t in range(1, T):
        seq.append(torch.ops.goom.lmme(A[t:t + 1], seq[-1][None])[0])
    cmp(f"chain d={d} T={T}: ts vs sequential complex64 fold", out_ts, torch.stack(seq))

# timing (d = 512, batch 1024): kernel only
d, b = 512, 1024
A, B = rgoom(b, d, 3), rgoom(b, d, 4)
ta, tb = ops.ts_from_goom(A), ops.ts_from_goom(B)
for kind in (0, 1, 2):
    ms = timeit(lambda: ops.lmme_ts(ta, tb, kind))
    print(f"lmme_ts kind{kind} d={d} batch={b}: {ms:.3f} ms  {2*d**3*b/ms/1e9:.1f} TF/s", flush=True)
ms = timeit(lambda: ops.lmme_ts(ta, tb[0:1], 2, b_div=b))
print(f"lmme_ts kind2 broadcast-B d={d} batch={b}: {ms:.3f} ms  {2*d**3*b/ms/1e9:.1f} TF/s", flush=True)
d, b = 1024, 256
A, B = rgoom(b, d, 3), rgoom(b, d, 4)
ta, tb = ops.ts_from_goom(A), ops.ts_from_goom(B)
for kind in (0, 1, 2):
    ms = timeit(lambda: ops.lmme_ts(ta, tb, kind))
    print(f"lmme_ts kind{kind} d={d} batch={b}: {ms:.3f} ms  {2*d**3*b/ms/1e9:.1f} TF/s", flush=True)
del A, B, ta, tb
torch.cuda.empty_cache()
# harness window
for T in (8192,):
    torch.cuda.synchronize()
    t0 = time.time()
    run = harness.run_chain(T, 512, seed=2510, window=8192, block=64)
    torch.cuda.synchronize()
    t1 = time.time()
    run = harness.run_chain(T, 512, seed=2510, window=8192, block=64)
    torch.cuda.synchronize()
    t2 = time.time()
    print(f"harness T={T} d=512: {(t2-t1)*1e3:.1f} ms  {T/(t2-t1):.0f} mat/s  growth {harness.growth_rate(run.digests):.5f} finite {bool((run.digests[:,2]==1).all())}", flush=True)
