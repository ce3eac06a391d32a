"""SURVEY §8 row N1 / north star item (2): long small-d chains on the warp- and CTA-resident
scan engines, reported against HBM.

For d in {8, 16, 32, 64}: a T = 2^20 chain of N(0,1) d x d leaves (complex64 GOOMs,
generated on the device), the public blocked chain scan with ALL T prefixes written
(torch.ops.goom.scan_chain -> goom_scan_chain_c64: d <= 32 scan_small.cu, 32 < d <= 64
scan_cta.cu), CUDA events around the scan only. Algorithmic bytes per element: read the
leaf and write the prefix, 16 d^2 B (complex64); the two-level tree moves 32 d^2 B
(phase 1 writes the local products, phase 3 reads them back). GB/s = 16 d^2 T / time,
against the measured HBM copy peak (MEASURED_PEAKS.json). A 1,024-leaf sample of the
reference's blocked chain (oracle/gooms_port.chain_blocked, float64) gives the CPU rate.
Prints one JSON line per d.
"""

import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--T", type=int, default=1 << 20)
    ap.add_argument("--ds", default="8,16,32,64")
    ap.add_argument("--block", type=int, default=1024)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--cpu-sample", type=int, default=1024)
    ap.add_argument("--engines", default="all", help="all, or a list of long,tree")
    args = ap.parse_args()
    import torch

    import paper_2510_03426_b200 as g
    from paper_2510_03426_b200 import harness
    from oracle import gooms_port as G

    g._lib.load()
    with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
        hbm = json.load(f)["hbm_gbs"]
    for d in [int(x) for x in args.ds.split(",")]:
        A = harness.random_chain(args.T, d, seed=d)
        engines = (["long", "tree"] if d <= 32 or d == 64 else ["tree"]) \
            if args.engines == "all" else args.engines.split(",")
        for eng in engines:
            if eng == "long" and d > 32 and d != 64:
                continue
            run = (lambda: torch.ops.goom.scan_chain_long(A, None)) if eng == "long" else \
                (lambda: torch.ops.goom.scan_chain(A, args.block, None))
            report(args, d, eng, A, run, hbm, G, np, torch)
        del A
        torch.cuda.empty_cache()


def report(args, d, eng, A, run, hbm, G, np, torch):
    if True:
        out = run()  # warm-up (and workspace)
        del out
        torch.cuda.synchronize()
        times = []
        for _ in range(args.reps):
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            out = run()
            e.record()
            torch.cuda.synchronize()
            times.append(s.elapsed_time(e))
            del out
        ms = float(np.median(times))
        gbs = 16.0 * d * d * args.T / (ms / 1e3) / 1e9
        # CPU: the reference's blocked chain on a sample, float64
        x = np.random.default_rng(d).standard_normal((args.cpu_sample, d, d))
        al, as_ = G.log_sign(x)
        t0 = time.perf_counter()
        G.chain_blocked(al, as_, min(args.block, args.cpu_sample))
        cpu_s = time.perf_counter() - t0
        if eng == "long" and d in (16, 32, 64):
            engine = ("scan_long + scan_long_tc (reduce-then-scan; each leaf-level fold step one "
                      f"tcgen05 3xTF32 MMA for {128 // d} chains, block-diagonal, state resident "
                      "in shared memory)")
            moved = 24 * d * d
        elif eng == "long":
            engine = ("scan_long (reduce-then-scan, group of d lanes per chain; a fixed tree "
                      "other than the reference's block tree)")
            moved = 24 * d * d
        else:
            engine = ("scan_small (warp per block, the reference's block tree)" if d <= 32 else
                      "scan_cta (CTA per block, the reference's block tree)")
            moved = 32 * d * d
        print(json.dumps({
            "config": "small_d_chain", "d": d, "T": args.T,
            "block": args.block if eng == "tree" else None,
            "engine": engine, "ms": ms, "matrices_per_s": args.T / (ms / 1e3),
            "algorithmic_bytes_per_element": 16 * d * d, "achieved_gbs": gbs,
            "hbm_peak_gbs": hbm, "frac_hbm": gbs / hbm,
            "moved_bytes_per_element": moved,
            "moved_gbs": moved / (16 * d * d) * gbs, "flops_per_element": 4 * d ** 3,
            "gflops": 4.0 * d ** 3 * args.T / (ms / 1e3) / 1e9,
            "cpu_matrices_per_s": args.cpu_sample / cpu_s, "cpu_cores": os.cpu_count(),
            "cpu_kind": "port (oracle/gooms_port.chain_blocked, float64)",
        }), flush=True)


if __name__ == "__main__":
    main()
