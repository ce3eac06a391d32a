"""Lyapunov-spectrum stage (a) on Lorenz-96 (d=64, T=100k).

Selective-reset scan with colinearity_policy(0.99, check_interval=12, volume_floor=1e-9)
over leaves [I, J_0 .. J_{T-2}] (lyapunov.py:335-341), complex128 (the reference runs this
path in float64). Reports the GPU time for the full chain, and on a T_cpu prefix the
reference algorithm's time on the host (oracle port) and whether the reset sites agree.
Prints one JSON line.
"""

import argparse
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from oracle import gooms_port as G  # noqa: E402
from oracle import systems_port as S  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--T", type=int, default=100_000)
    ap.add_argument("--d", type=int, default=64)
    ap.add_argument("--T-cpu", type=int, default=4000)
    args = ap.parse_args()
    import torch

    import paper_2510_03426_b200 as g

    t0 = time.perf_counter()
    f, df, x0, dt = S.lorenz96(args.d)
    mats = S.integrate_chain(f, df, x0, dt, burn_in=1000, T=args.T, seed=0)
    leaves = S.spectrum_leaves(mats)
    al, as_ = G.log_sign(leaves)
    gen_s = time.perf_counter() - t0

    pol = g.colinearity_policy(0.99, 12, 1e-9)
    A = g.join(al, as_, torch.complex128)
    g._selective_chain_core(A[:64], pol, 256)  # warm-up
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    V, sites = g._selective_chain_core(A, pol, 256)
    e.record()
    torch.cuda.synchronize()
    gpu_ms = s.elapsed_time(e)
    # every log-magnitude finite or -inf (exact zeros, e.g. the identity leaf's off-diagonal)
    finite = bool((torch.isfinite(V.real) | (V.real == float("-inf"))).all())

    # the full spectrum estimator (stages (a)-(d), lyapunov.py:311-356) on the GPU
    chain = g.JacobianChain(dt=dt, mats=mats)
    g.spectrum_parallel(g.JacobianChain(dt=dt, mats=mats[:256]))  # warm-up
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    spec = g.spectrum_parallel(chain)
    torch.cuda.synchronize()
    spec_s = time.perf_counter() - t2
    lam_sum = float(np.sum(spec.lambdas))

    # parity + CPU baseline on a prefix
    Tc = min(args.T_cpu, args.T)
    t1 = time.perf_counter()
    Vc, Sc, sites_cpu = G.selective_chain(al[:Tc], as_[:Tc], G.colinearity_policy(0.99, 12), 256)
    cpu_s = time.perf_counter() - t1
    Vp, sites_pref = g._selective_chain_core(A[:Tc], pol, 256)
    vl = Vp.real.cpu().numpy()
    vs = np.where(np.cos(Vp.imag.cpu().numpy()) < 0, -1.0, 1.0)
    c = Vc.max(axis=(1, 2), keepdims=True)
    err = np.abs(vs * np.exp(vl - c) - Sc * np.exp(Vc - c)).max()
    print(json.dumps({
        "config": "lyapunov_lorenz96_selective", "d": args.d, "T": args.T,
        "policy": "colinearity(0.99, interval 12, volume 1e-9), consume_leaf=False",
        "gpu_ms": gpu_ms, "gpu_matrices_per_s": args.T / (gpu_ms / 1e3), "resets": len(sites),
        "spectrum_parallel_s": spec_s, "spectrum_matrices_per_s": args.T / spec_s,
        "lambda_max": float(spec.lambdas[0]), "lambda_sum": lam_sum,
        "spectrum_resets": spec.resets,
        "finite": finite, "input_generation_s": gen_s,
        "cpu_prefix_T": Tc, "cpu_s": cpu_s, "cpu_matrices_per_s": Tc / cpu_s,
        "cpu_cores": os.cpu_count(), "cpu_kind": "port (oracle/gooms_port.selective_chain, float64)",
        "sites_identical_on_prefix": sites_pref == sites_cpu, "prefix_resets": len(sites_cpu),
        "prefix_max_scaled_err": float(err),
    }), flush=True)


if __name__ == "__main__":
    main()
