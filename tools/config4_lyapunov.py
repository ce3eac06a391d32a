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
    ap.add_argument("--T-cpu", type=int, default=100_000, help="oracle prefix (default: all)")
    ap.add_argument("--sites-only", action="store_true",
                    help="print the GPU reset sites (JSON) and exit (direct-volume A/B)")
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
    if args.sites_only:
        _, sites = g._selective_chain_core(A, pol, 256)
        print(json.dumps({"sites": sites}))
        return
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
    margins = decision_margins(Vc, Sc, 12, 0.99, 1e-9)
    # the walk's volume test by determinant multiplicativity vs a direct factorisation of
    # every tested state (GOOM_WALK_DIRECT_VOLUME=1): same sites?
    import subprocess
    env = dict(os.environ, GOOM_WALK_DIRECT_VOLUME="1")
    out = subprocess.run([sys.executable, os.path.abspath(__file__), "--T", str(args.T), "--d",
                          str(args.d), "--sites-only"], env=env, capture_output=True, text=True,
                         timeout=1800)
    direct_sites = json.loads(out.stdout.strip().splitlines()[-1])["sites"]
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
        "sites_identical_full_length": sites == sites_cpu if Tc == args.T else None,
        "decision_margins": margins,
        "direct_volume_sites_identical": direct_sites == sites,
    }), flush=True)


def decision_margins(V, Sg, interval, threshold, volume_floor):
    """For every tested state of the oracle's run (positions p with (p+1) % interval == 0,
    lyapunov.py:255-269): the distance of max |cos| to the threshold and of log|det| of the
    unit-column state to log(volume_floor) — how close the reference's own decisions are to
    flipping (a GPU decision can only differ from the reference's inside rounding of these)."""
    T = V.shape[0]
    tested = np.array([p for p in range(T - 1) if (p + 1) % interval == 0])
    cos_m, vol_m = [], []
    fired = []
    for i in range(0, len(tested), 512):
        idx = tested[i:i + 512]
        lg, sg = V[idx], Sg[idx]
        top = lg.max(axis=1, keepdims=True)
        nu = top + 0.5 * np.log(np.sum(np.exp(2.0 * (lg - top)), axis=1, keepdims=True))
        real = sg * np.exp(lg - nu)
        gram = np.einsum("nki,nkj->nij", real, real)
        iu, ju = np.triu_indices(gram.shape[1], k=1)
        mx = np.abs(gram[:, iu, ju]).max(axis=1)
        sgn, ld = np.linalg.slogdet(real)
        cos_m.append(mx - threshold)
        vol_m.append(ld - np.log(volume_floor))
        fired.append((mx > threshold) | (sgn == 0) | (ld < np.log(volume_floor)))
    cos_m, vol_m, fired = np.concatenate(cos_m), np.concatenate(vol_m), np.concatenate(fired)
    return {"tested": int(len(tested)), "fired": int(fired.sum()),
            "min_abs_cos_margin": float(np.abs(cos_m).min()),
            "min_abs_logvol_margin": float(np.abs(vol_m).min()),
            "fired_by_cos": int((cos_m > 0).sum()), "fired_by_volume": int((vol_m < 0).sum()),
            "within_1e-6_cos": int((np.abs(cos_m) < 1e-6).sum()),
            "within_1e-6_logvol": int((np.abs(vol_m) < 1e-6).sum())}


if __name__ == "__main__":
    main()
