#!/usr/bin/env python3
"""LMME prefix-scan benchmark (BASELINE.json metric, config 3).

Workload: a T = 2^20-long chain of 512 x 512 random-normal matrices held as
complex64 GOOMs; every prefix P_t = A_t ... A_0 is computed with the blocked
LMME scan (tcgen05 3xTF32 kernels) and digested on the device (max log-mag,
log Frobenius norm, finiteness). Leaves are generated on the device from a
counter-based RNG keyed (seed, t) inside the timed region (2 TiB of leaves
cannot be resident); every window (32 GiB) is far larger than L2, so no L2
flush is needed between iterations. One step = the whole chain.

  python bench.py [--gpus N --steps K --warmup W]          # b200 arm
  python bench.py --impl reference ...                      # reference CPU arm
  torchrun --nproc-per-node N bench.py --gpus N ...         # time-sharded, NCCL all-gather

Prints ONE JSON line on rank 0.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "LMME prefix-scan matrices/sec (d=512, T=1M)"
UNIT = "matrices/s"


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=3)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", default="b200", choices=["b200", "reference"])
    p.add_argument("--T", type=int, default=1 << 20)
    p.add_argument("--d", type=int, default=512)
    p.add_argument("--window", type=int, default=32768)
    p.add_argument("--block", type=int, default=128)
    p.add_argument("--seed", type=int, default=2510)
    p.add_argument("--cpu-sample", type=int, default=128, help="leaves in the CPU baseline sample")
    p.add_argument("--e2e-T", type=int, default=8192)
    p.add_argument("--e2e-goom-T", type=int, default=4096,
                   help="leaves of the drop-in-boundary e2e (complex64 GOOMs from pinned host)")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-reanchor", action="store_true", help="skip the re-anchored checks")
    return p.parse_args()


# ---------------------------------------------------------------------------
# CPU baseline: the reference algorithm (numpy restatement, oracle/gooms_port.py)


def cpu_chain_rate(d: int, T: int, seed: int, dtype="float32", stock=False):
    """Time the reference's blocked scan (scan.py:181-214) on T random-normal leaves.
    dtype "float32": the reference's own float32 path (dtype preserved end to end; the
    precision the GPU's complex64 computes at) — the fastest CPU variant, the headline
    baseline; "float64": its default backing. stock=False times the A slot only (the
    product chain, 2 LMMEs/element at the block tree); stock=True the stock
    _scan_affine_stack on (A, zero-bias) pairs as scan_parallel runs it, bias LMMEs
    included (scan.py:173-178)."""
    import numpy as np

    from oracle import gooms_port as G

    rng = np.random.default_rng(seed)
    al, as_ = G.log_sign(rng.standard_normal((T, d, d)).astype(dtype))

    def run(a, s, blk):
        if not stock:
            return G.chain_blocked(a, s, blk)
        st = G.Stack(a, s, np.full(a.shape, -np.inf, dtype=a.dtype), np.ones_like(s),
                     np.zeros(a.shape[0], dtype=bool))
        return G.scan_affine_blocked(st, blk)

    run(al[:4], as_[:4], 2)  # warm BLAS
    t0 = time.perf_counter()
    run(al, as_, 32)
    dt = time.perf_counter() - t0
    return T / dt, dt


def cpu_cores():
    return os.cpu_count() or 1


def cpu_info():
    """Host CPU model, core count and the BLAS numpy runs on."""
    import numpy as np

    model = "unknown"
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    blas = "unknown"
    try:
        cfg = np.show_config(mode="dicts")
        b = cfg.get("Build Dependencies", {}).get("blas", {})
        blas = f"{b.get('name', '?')} {b.get('version', '')}".strip()
    except Exception:  # pragma: no cover
        pass
    return {"nproc": cpu_cores(), "cpu_model": model, "blas": blas}


def cpu_variants(d: int, T: int, seed: int):
    """The CPU baseline beside its variants: float32 / float64, chain-only / stock."""
    out = {}
    for name, dt, stock in (("float32_chain", "float32", False), ("float64_chain", "float64", False),
                            ("float64_stock_affine", "float64", True)):
        r, s = cpu_chain_rate(d, T, seed, dt, stock)
        out[name] = {"matrices_per_s": r, "seconds": round(s, 2)}
    return out


# ---------------------------------------------------------------------------
# clocks during the timed region


class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index):
        self.gpu = gpu_index
        self.rows = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            threading.Thread(target=self._read, daemon=True).start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [x.strip() for x in line.split(",")]
            if len(parts) == 6:
                self.rows.append(parts)

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if r[2 + i] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons, "samples": len(self.rows)}


# ---------------------------------------------------------------------------


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            pk = json.load(f)
        return pk, "measured"
    except OSError:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}, "fallback"


def cublas_tf32_tflops(torch, n=8192, reps=10):
    """In-run cuBLAS TF32 GEMM (fp32 matmul with TF32 tensor cores), best of `reps`: the
    measured denominator for a kind::tf32 kernel (the driver's peaks are bf16)."""
    prev = torch.backends.cuda.matmul.allow_tf32
    torch.backends.cuda.matmul.allow_tf32 = True
    try:
        a = torch.randn(n, n, device="cuda")
        b = torch.randn(n, n, device="cuda")
        for _ in range(2):
            a @ b
        torch.cuda.synchronize()
        best = float("inf")
        for _ in range(reps):
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            a @ b
            e.record()
            torch.cuda.synchronize()
            best = min(best, s.elapsed_time(e))
        return 2.0 * n ** 3 / (best / 1e3) / 1e12
    finally:
        torch.backends.cuda.matmul.allow_tf32 = prev


def reference_arm(args):
    """--impl reference: the reference CPU algorithm on the host cores (oracle port)."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    T = args.cpu_sample
    if args.warmup > 0:
        cpu_chain_rate(args.d, 8, args.seed)
    rates = []
    for i in range(args.steps):
        r, dt = cpu_chain_rate(args.d, T, args.seed + i)
        rates.append(r)
    v = statistics.median(rates)
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": T / v * 1e3,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic N(0,1) leaves",
        "config": {"workload": f"chain d={args.d}, sample of T={T} leaves of the T={args.T} chain",
                   "d": args.d, "T": args.T, "sample_T": T, "block": 32},
        "cpu_baseline": {"value": v, "unit": UNIT, "cores": cpu_cores(), "kind": "port",
                         "sample": f"{T} leaves, the reference's float32 blocked chain "
                                   f"(scan.py:181-214, its fastest CPU variant and the GPU's "
                                   f"precision) via oracle/gooms_port.chain_blocked",
                         "host": cpu_info(), "variants": cpu_variants(args.d, T, args.seed)},
        "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }), flush=True)


def main():
    args = parse()
    if args.impl == "reference":
        reference_arm(args)
        return

    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # GOOM_BENCH_SHARE_GPU=1 (test aid): ranks share the visible GPUs round-robin and talk
    # over gloo, so the N > 1 path (all-gather of the shard totals, max-over-ranks timing)
    # can be exercised on a one-GPU box; numbers from such a run are not bench values
    share = os.environ.get("GOOM_BENCH_SHARE_GPU") == "1"
    if share:
        local = local % torch.cuda.device_count()
    torch.cuda.set_device(local)
    if world > 1:
        if share:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    import paper_2510_03426_b200 as goom
    from paper_2510_03426_b200 import harness, ops, sharded

    goom._lib.load()
    dev = torch.device("cuda", local)
    T, d = args.T, args.d

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    # re-anchored parity windows on the timed run itself: the block carries
    # applied at two block starts (~2^19 and the last block) and the prefix 63 steps later
    W = min(REANCHOR_W, args.block)
    anchors = sorted({(a // args.block) * args.block for a in (T // 2, T - W - 1)
                      if a >= args.block})
    anchors = [a for a in anchors if a + W <= T and not args.no_reanchor]
    snaps = sorted({a + W - 1 for a in anchors})

    def one_step():
        return sharded.run_chain_sharded(T, d, args.seed, args.window, args.block,
                                         snapshots=snaps, anchors=anchors)

    for _ in range(args.warmup):
        one_step()
    barrier()

    launches0 = ops.kernel_launches()
    times = []
    lib = goom._lib.load()
    lib.goom_chain_ts_phase3_timing(1)  # the dominant kernel, timed inside the timed region
    with ClockSampler(local) as clocks:
        for _ in range(args.steps):
            barrier()
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            t0, run = one_step()
            e.record()
            barrier()
            ms = s.elapsed_time(e)
            if world > 1:
                tt = torch.tensor([ms], device=dev)
                dist.all_reduce(tt, op=dist.ReduceOp.MAX)
                ms = float(tt.item())
            times.append(ms)
    launches = ops.kernel_launches() - launches0
    import ctypes
    phases = {}
    for ph in range(4):
        n_, ms_, u_ = ctypes.c_int64(0), ctypes.c_double(0.0), ctypes.c_int64(0)
        goom._lib.check(lib.goom_chain_ts_phase_stats(ph, ctypes.byref(n_), ctypes.byref(ms_),
                                                      ctypes.byref(u_)))
        phases[ph] = (n_.value, ms_.value, u_.value)
    lib.goom_chain_ts_phase3_timing(0)
    p3_n, p3_ms, p3_prod = (ctypes.c_int64(phases[3][0]), ctypes.c_double(phases[3][1]),
                            ctypes.c_int64(phases[3][2]))
    if world > 1:
        lt = torch.tensor([launches], device=dev, dtype=torch.float64)
        dist.all_reduce(lt)
        launches = int(lt.item())
    ms_step = statistics.median(times)
    value = T / (ms_step / 1e3)

    # sanity of the run itself: growth rate of log||P_t|| vs (ln 2 + psi(d/2)) / 2
    dg = run.digests
    own = getattr(run, "windows", None)  # relay time-sharding: this rank's windows only
    if own:
        dg = torch.cat([dg[w0:w0 + m] for w0, m in own])
        w0, m = max(own, key=lambda x: x[1])
        growth = harness.growth_rate(run.digests[w0:w0 + m]) if m > 2 else float("nan")
    else:
        growth = harness.growth_rate(dg) if dg.shape[0] > 2 else float("nan")
    finite = bool((dg[:, 2] == 1).all().item())
    reanchored = reanchor_checks(run, t0, anchors, W, d, args.seed, ops, world, dist)

    # ---- roofline of the dominant kernel: the phase-3 batched LMME of a window ----
    # out[b] = L[b] (x) Cx[b / block] with the digest epilogue: exactly the chain engine's
    # phase-3 launch (chain_ts.cu) on tile-scaled operands; algorithmic 2 d^3 flop/product
    pk, src = measured_peaks()
    nb = args.window
    if ops.ts_eligible(d):
        L = ops.ts_random_normal(nb, d, args.seed, 0, dev)
        C = ops.ts_random_normal(nb // args.block, d, args.seed + 1, 0, dev)

        def phase3():
            ops.lmme_ts(L, C, 2, b_div=args.block)
        kname = "lmme_ts_kernel<digest> (tcgen05 cta_group::2 3xTF32, tile-scaled fp32 operands)"
    else:
        L = harness.random_chain(nb, d, args.seed, 0, dev)
        C = harness.random_chain(nb // args.block, d, args.seed + 1, 0, dev)

        def phase3():
            torch.ops.goom.lmme(L, torch.repeat_interleave(C, args.block, 0))
        kname = "lmme (complex64 tcgen05)"
    strm = torch.cuda.current_stream()
    phase3()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 3
    s.record(strm)
    for _ in range(reps):
        phase3()
    e.record(strm)
    torch.cuda.synchronize()
    lmme_ms = s.elapsed_time(e) / reps
    standalone_tflops = 2.0 * d ** 3 * nb / (lmme_ms / 1e3) / 1e12
    burst_3xtf32 = pk["bf16_tflops"] / 2 / 3
    # the roofline line: the phase-3 launches of the timed steps themselves (events on the
    # engine's stream), against the SUSTAINED peak (a kernel timed inside a long step)
    if p3_n.value > 0 and p3_ms.value > 0:
        tflops = 2.0 * d ** 3 * p3_prod.value / (p3_ms.value / 1e3) / 1e12
        avg_launch_ms = p3_ms.value / p3_n.value
        peak_3xtf32 = pk.get("bf16_tflops_sustained", pk["bf16_tflops"]) / 2 / 3
        timing = (f"in-run: {p3_n.value} phase-3 launches of the timed steps, CUDA events on "
                  f"the engine's stream, {avg_launch_ms:.2f} ms/launch")
        peak_kind = "sustained"
    else:
        tflops, avg_launch_ms, peak_3xtf32 = standalone_tflops, lmme_ms, burst_3xtf32
        timing = f"standalone phase-3 shape, {lmme_ms:.2f} ms/launch"
        peak_kind = "burst"
    # every phase of the timed steps (CUDA events on the engine's stream), per GPU
    peak_s = pk.get("bf16_tflops_sustained", pk["bf16_tflops"]) / 2 / 3
    hbm = pk.get("hbm_gbs", 6650.0)
    phase_rows = {}
    names = {0: "leaf generation (random_normal_ts_kernel)",
             1: "phase 1 local products (lmme_ts_kernel<ts out>, s-1 launches per window)",
             2: "phase 2 block-carry Kogge-Stone tree (lmme_ts_kernel<ts out>)",
             3: "phase 3 carry apply + digest (lmme_ts_kernel<digest>)"}
    for ph, (n_, ms_, u_) in phases.items():
        if n_ == 0 or ms_ <= 0:
            continue
        row = {"kernel": names[ph], "windows": n_, "ms_per_step": ms_ / max(args.steps, 1),
               "share_of_step": ms_ / max(args.steps, 1) / ms_step}
        if ph == 0:
            gbs = u_ * d * d * 4 / (ms_ / 1e3) / 1e9
            row.update(bound="hbm", achieved=gbs, unit="GB/s", frac=gbs / hbm,
                       units="leaves (4 B/element written)")
        else:
            tf = 2.0 * d ** 3 * u_ / (ms_ / 1e3) / 1e12
            row.update(bound="tensor", achieved=tf, unit="TFLOP/s", frac=tf / peak_s,
                       units=f"{u_} products")
        phase_rows[["rng", "phase1", "phase2", "phase3"][ph]] = row
    step_tf = 4.0 * d ** 3 * T / world / (ms_step / 1e3) / 1e12
    tf32_cublas = cublas_tf32_tflops(torch)
    traffic = None
    tf = os.path.join(ROOT, "profiles", "roofline_traffic.json")
    if os.path.exists(tf) and ops.ts_eligible(d) and d == 512:
        with open(tf) as f:
            per = json.load(f).get("dram_bytes_per_product")
        traffic = per * nb if per else None  # ncu capture scaled to this launch's batch
    del L, C
    torch.cuda.empty_cache()

    # ---- e2e through the public API: host leaves -> H2D -> scan -> digests D2H ----
    # The chain experiment's inputs are real random-normal matrices; the
    # user hands them to harness.run_chain as pinned host float32, which streams each
    # window's H2D copy on a copy stream under the previous window's scan.
    Te = args.e2e_T
    we = max(1, min(args.window, Te // 4))
    t0e, ne = sharded.shard_range(Te, rank, world)
    if ops.ts_eligible(d):
        host = ops.ts_random_normal(ne, d, args.seed + 7, t0e, dev).U.cpu().pin_memory()
    else:
        host = torch.ops.goom.to_real(harness.random_chain(ne, d, args.seed + 7, t0e, dev),
                                      False).cpu().pin_memory()
    e2e_times = []
    for it in range(2):
        barrier()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        carry = None
        if world > 1:
            dl = host.to(dev, non_blocking=True)
            if ops.ts_eligible(d):
                _, _, ct = ops.chain_ts(harness.real_leaves_ts(dl), args.block, None, out=False,
                                        digests=False, carry_out=True)
                tot = ops.ts_to_goom(ct)[0]
            else:
                tot = harness.chain_total(torch.ops.goom.from_real(dl, float("-inf"), False))
            carry = sharded.exclusive_carry(tot, torch.ops.goom.lmme)
            del dl
        r = harness.run_chain(ne, d, window=we, block=args.block, carry=carry, leaves=host)
        out = r.digests.to("cpu", non_blocking=True)
        e.record()
        barrier()
        ms = s.elapsed_time(e)
        if world > 1:
            tt = torch.tensor([ms], device=dev)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            ms = float(tt.item())
        if it > 0:
            e2e_times.append(ms)
        del r, out
    e2e_value = Te / (statistics.median(e2e_times) / 1e3)
    # the link's own ceiling in this run: a plain pinned H2D copy of the same leaves
    dcopy = torch.empty(host.shape, dtype=host.dtype, device=dev)
    h2d_ms = []
    for _ in range(3):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        dcopy.copy_(host, non_blocking=True)
        e.record()
        torch.cuda.synchronize()
        h2d_ms.append(s.elapsed_time(e))
    h2d_gbs = host.numel() * host.element_size() / (min(h2d_ms) / 1e3) / 1e9
    del dcopy

    # ---- e2e at the drop-in boundary: complex64 GOOM leaves (the reference's own data
    # format: log|x| + sign, scan.py:138-170) in pinned host memory -> the public drop-in scan
    # (torch.ops.goom.scan_chain = goom_scan_chain_c64, the _scan_affine_stack path, exact
    # complex64 engine) window by window; the H2D copy of window w+1 runs on a copy stream
    # under the scan of window w; per-prefix digests D2H. Every leaf crosses PCIe at 8 B per
    # element (twice the real-float32 variant above), so this is the link-bound figure.
    Tg = max(args.e2e_goom_T // world, 1) * world
    t0g, ng = sharded.shard_range(Tg, rank, world)
    wg = max(1, min(512, ng))
    hostg = torch.empty((ng, d, d), dtype=torch.complex64).pin_memory()
    for w0 in range(0, ng, wg):
        n = min(wg, ng - w0)
        hostg[w0:w0 + n].copy_(harness.random_chain(n, d, args.seed + 11, t0g + w0, dev))
    copy_stream = torch.cuda.Stream()
    bufs = [torch.empty((wg, d, d), dtype=torch.complex64, device=dev) for _ in range(2)]
    free_ev = [torch.cuda.Event(), torch.cuda.Event()]
    goom_times = []
    nw = (ng + wg - 1) // wg
    for it in range(2):
        barrier()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        carry = None
        if world > 1:  # the shard's exclusive carry (one all-gather of the shard totals)
            dl = hostg.to(dev, non_blocking=True)
            carry = sharded.exclusive_carry(harness.chain_total(dl), torch.ops.goom.lmme)
            del dl
        dig = torch.empty((ng, 4), dtype=torch.float32, device=dev)
        cur = torch.cuda.current_stream()
        landed = []

        def issue(i):  # H2D of window i on the copy stream, into the buffer window i - 2 freed
            w0 = i * wg
            n = min(wg, ng - w0)
            with torch.cuda.stream(copy_stream):
                if i >= 2:
                    copy_stream.wait_event(free_ev[i % 2])
                bufs[i % 2][:n].copy_(hostg[w0:w0 + n], non_blocking=True)
                ev = torch.cuda.Event()
                ev.record(copy_stream)
                landed.append(ev)

        issue(0)
        for i in range(nw):
            if i + 1 < nw:
                issue(i + 1)
            w0 = i * wg
            n = min(wg, ng - w0)
            cur.wait_event(landed[i])
            P = torch.ops.goom.scan_chain(bufs[i % 2][:n], args.block, carry)
            dig[w0:w0 + n] = torch.ops.goom.digest(P)
            carry = P[n - 1].clone()
            free_ev[i % 2].record(cur)
            del P
        out = dig.to("cpu", non_blocking=True)
        e.record()
        barrier()
        ms = s.elapsed_time(e)
        if world > 1:
            tt = torch.tensor([ms], device=dev)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            ms = float(tt.item())
        if it > 0:
            goom_times.append(ms)
        del out, dig
    goom_value = Tg / (statistics.median(goom_times) / 1e3)
    del hostg, bufs

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        v, dt = cpu_chain_rate(d, args.cpu_sample, args.seed)
        cpu = {"value": v, "unit": UNIT, "cores": cpu_cores(), "kind": "port",
               "sample": f"{args.cpu_sample} leaves of {d}x{d}, the reference's float32 "
                         f"blocked chain (scan.py:181-214; its fastest CPU variant, the GPU's "
                         f"precision) via oracle/gooms_port, {dt:.1f} s",
               "host": cpu_info(), "variants": cpu_variants(d, args.cpu_sample, args.seed)}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "c64 (f32 log + sign; 3xTF32 GEMM)",
            "data": "synthetic N(0,1) leaves generated on device (Philox, keyed by leaf index)",
            "config": {"workload": f"chain T={T} of {d}x{d} GOOM leaves, all prefixes digested",
                       "T": T, "d": d, "window": args.window, "block": args.block,
                       "parallelism": (f"time-sharded x{world} ({sharded.shard_mode()}: "
                                       + ("windows round-robin, carry relayed rank to rank"
                                          if sharded.shard_mode() == "relay" else
                                          "contiguous shards, all-gather of the shard totals")
                                       + ")") if world > 1 else "single GPU",
                       "l2": "no flush: every window (>= 16 GiB) exceeds the 126 MB L2"},
            "roofline": {"bound": "tensor", "achieved": tflops, "peak": peak_3xtf32,
                         "unit": "TFLOP/s", "frac": tflops / peak_3xtf32, "traffic": traffic,
                         "kernel": f"{kname}, phase-3 launch of batch={nb} (carry per "
                                   f"{args.block}); {timing}; algorithmic 2*d^3 flop/product",
                         "peak_source": f"{src} bf16 ({peak_kind}) "
                                        f"{pk.get('bf16_tflops_sustained') if peak_kind == 'sustained' else pk['bf16_tflops']}"
                                        " TF/s / 2 (TF32) / 3 (3xTF32 split)",
                         "standalone_tflops": standalone_tflops,
                         "frac_standalone_vs_burst": standalone_tflops / burst_3xtf32,
                         "tf32_cublas_tflops_in_run": tf32_cublas,
                         "frac_vs_cublas_tf32_div3": tflops / (tf32_cublas / 3),
                         "phases": phase_rows,
                         "whole_step": {"tflops_4d3_per_element": step_tf,
                                        "frac": step_tf / peak_s,
                                        "note": "4 d^3 flop per chain element (2 LMMEs), "
                                                "per GPU, vs the sustained 3xTF32 peak"}},
            "e2e": {"value": goom_value, "unit": UNIT, "h2d_bytes_per_step": ng * d * d * 8,
                    "d2h_bytes_per_step": ng * 16,
                    "h2d_gbs_per_gpu": ng * d * d * 8 / (statistics.median(goom_times) / 1e3) / 1e9,
                    "h2d_gbs_plain_copy_in_run": h2d_gbs,
                    "workload": f"T={Tg} complex64 GOOM leaves (log|x| + sign, the reference's "
                                f"format) in pinned host memory -> the drop-in scan "
                                f"(torch.ops.goom.scan_chain / goom_scan_chain_c64, window {wg}, "
                                f"H2D of the next window overlapped), per-prefix digests D2H",
                    "real_f32_leaves": {
                        "value": e2e_value, "h2d_bytes_per_step": ne * d * d * 4,
                        "d2h_bytes_per_step": ne * 16,
                        "h2d_gbs_per_gpu": ne * d * d * 4 / (statistics.median(e2e_times) / 1e3) / 1e9,
                        "workload": f"T={Te} real float32 leaves in pinned host memory -> "
                                    f"harness.run_chain (window {we}, H2D overlapped), digests D2H "
                                    f"(the chain experiment's input, SPEC.md:391-455)"}},
            "gpu_launches": launches // max(args.steps, 1),
            "clocks": clocks.summary(),
            "check": {"finite": finite, "growth_per_step": growth,
                      "expected_growth": 0.5 * (math.log(2) + _digamma(d / 2)),
                      "reanchored": reanchored},
        }
        if cpu:
            line["cpu_baseline"] = cpu
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


REANCHOR_W = 64


def reanchor_checks(run, t0, anchors, W, d, seed, ops, world, dist):
    """SURVEY §8c(5) on the timed run itself: for each block start a in this rank's shard
    the float64 oracle (oracle/reanchor.py; the checker, not the thing measured) folds the
    regenerated leaves A_a .. A_{a+W-1} onto the block carry the engine applied there (its
    own P_{a-1}), and compares P_{a+W-1} entry by entry and every digest of the stretch.
    Runs after the timed region."""
    from oracle import reanchor as R

    out = []
    for a in anchors:
        if a not in run.anchors_ts or a + W - 1 not in run.snapshots_ts:
            continue
        l0, s0 = (x[0].cpu().numpy() for x in ops.ts_log_sign(run.anchors_ts[a]))
        l1, s1 = (x[0].cpu().numpy() for x in ops.ts_log_sign(run.snapshots_ts[a + W - 1]))
        leaves = ops.ts_random_normal(W, d, seed, a, run.digests.device).U.cpu().numpy()
        dg = run.digests[a - t0:a - t0 + W, :2].cpu().numpy()
        tt = time.perf_counter()
        r = R.check_window(l0, s0, leaves, l1, s1, dg)
        r["t0"] = a
        r["cpu_s"] = round(time.perf_counter() - tt, 1)
        out.append(r)
    if world > 1:
        allr = [None] * world
        dist.all_gather_object(allr, out)
        out = [r for part in allr for r in part]
    return sorted(out, key=lambda r: r["t0"])


def _digamma(x):
    # asymptotic series (x >= 6 here)
    r = 0.0
    while x < 6:
        r -= 1 / x
        x += 1
    f = 1 / (x * x)
    return r + math.log(x) - 0.5 / x - f * (1 / 12 - f * (1 / 120 - f / 252))


if __name__ == "__main__":
    main()
