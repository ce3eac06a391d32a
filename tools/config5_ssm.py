"""non-diagonal GOOM recurrence, d_state = 64, 16 heads, batch 32,
T = 4096 — 512 sequences, forward + backward (ssm.ssm_forward_heads /
ssm_backward_heads: every launch covers all 16 heads; complex128 log-domain recurrence,
the reference's float64). Times are device-resident inputs, CUDA events around
forward and forward+backward; the host->device upload of the float64 inputs is reported
separately. Parity: head 0 sequence 0 against the oracle port's forward and its
log-domain adjoint (oracle/gooms_port.ssm_backward).
CPU baseline: the oracle port (forward scan + adjoint, float64) on one sequence, x 512.
Prints one JSON line."""

import argparse
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--d", type=int, default=64)
    ap.add_argument("--heads", type=int, default=16)
    ap.add_argument("--batch", type=int, default=32)
    ap.add_argument("--T", type=int, default=4096)
    ap.add_argument("--chunk", type=int, default=64)
    ap.add_argument("--reps", type=int, default=3)
    args = ap.parse_args()
    import torch

    from oracle import gooms_port as G
    from paper_2510_03426_b200 import ssm

    rng = np.random.default_rng(5)
    d, H, S, T = args.d, args.heads, args.batch, args.T
    A = rng.standard_normal((H, d, d))
    for h in range(H):
        A[h] *= rng.uniform(1.0, 1.5) / np.max(np.abs(np.linalg.eigvals(A[h])))
    B, C, D = (rng.standard_normal((H, r, d)) for r in (d, 2 * d, 2 * d))
    x0 = rng.standard_normal((H, S, d))
    u = rng.standard_normal((H, S, T, d))
    gy = rng.standard_normal((H, S, T, 2 * d))
    dev = torch.device("cuda")
    t0 = time.perf_counter()
    dA_, dB_, dC_, dD_, dx0_, du_, dgy_ = (torch.as_tensor(v, device=dev) for v in (A, B, C, D, x0, u, gy))
    torch.cuda.synchronize()
    upload_s = time.perf_counter() - t0

    def fwd():
        return ssm.ssm_forward_heads(dA_, dB_, dC_, dD_, dx0_, du_, chunk=args.chunk)

    def fwd_bwd():
        sl, ss, c, y = fwd()
        return (sl, ss, c, y), ssm.ssm_backward_heads(dA_, dB_, dC_, dD_, dx0_, du_, sl, ss, c,
                                                      dgy_, chunk=args.chunk)

    # warm-up on a slice
    ssm.ssm_forward_heads(dA_, dB_, dC_, dD_, dx0_[:, :2], du_[:, :2, :256], chunk=args.chunk)
    fwd_bwd()
    torch.cuda.synchronize()

    def timed(fn):
        ts = []
        for _ in range(args.reps):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            a.record()
            r = fn()
            b.record()
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b) / 1e3)
        return float(np.median(ts)), r

    f_s, (sl, ss, c, y) = timed(fwd)
    fb_s, (_, grads) = timed(fwd_bwd)
    b_s, _ = timed(lambda: ssm.ssm_backward_heads(dA_, dB_, dC_, dD_, dx0_, du_, sl, ss, c, dgy_,
                                                  chunk=args.chunk))
    finite = bool(torch.isfinite(sl).all() and torch.isfinite(y).all() and
                  all(bool(torch.isfinite(g).all()) for g in grads))
    # parity: head 0, sequence 0 vs the oracle
    osl, oss, oc, oy = G.ssm_forward_parallel(A[0], B[0], C[0], D[0], x0[0, 0], u[0, 0])
    sl0 = sl[0, 0].cpu().numpy()
    err = float(np.max(np.abs(sl0 - osl) / np.maximum(1.0, np.abs(osl))))
    t1 = time.perf_counter()
    ob = G.ssm_backward(A[0], B[0], C[0], D[0], x0[0, 0], u[0, 0], osl, oss, oc, gy[0, 0])
    cpu_bwd_s = time.perf_counter() - t1
    one = ssm.ssm_backward_heads(dA_[:1], dB_[:1], dC_[:1], dD_[:1], dx0_[:1, :1], du_[:1, :1],
                                 sl[:1, :1], ss[:1, :1], c[:1, :1], dgy_[:1, :1], chunk=args.chunk)
    gerr = {k: float(np.max(np.abs(g[0].cpu().numpy() - ob[k])) / np.max(np.abs(ob[k])))
            for k, g in zip(("A", "B", "C", "D"), one[:4])}
    gerr["u"] = float(np.max(np.abs(one[5][0, 0].cpu().numpy() - ob["u"])) / np.max(np.abs(ob["u"])))
    t1 = time.perf_counter()
    G.ssm_forward_parallel(A[1], B[1], C[1], D[1], x0[1, 0], u[1, 0])
    cpu_fwd_s = time.perf_counter() - t1
    steps = H * S * T
    print(json.dumps({
        "config": "ssm_forward_backward", "d": d, "heads": H, "batch": S, "T": T,
        "chunk": args.chunk, "gpu_forward_s": f_s, "gpu_forward_backward_s": fb_s,
        "gpu_backward_s": b_s,
        "gpu_steps_per_s_fwd": steps / f_s, "gpu_steps_per_s_fwd_bwd": steps / fb_s,
        "upload_s": upload_s, "finite": finite, "max_scale": float(c.max()),
        "gpu_timing": "CUDA events, float64 inputs resident on the device; outputs and "
                      "gradients left on the device",
        "parity_fwd_rel_log_vs_oracle": err,
        "sign_mismatch": int(np.sum(ss[0, 0].cpu().numpy() != oss)),
        "parity_bwd_rel_vs_oracle": gerr,
        "cpu_one_sequence_fwd_s": cpu_fwd_s, "cpu_one_sequence_bwd_s": cpu_bwd_s,
        "cpu_extrapolated_fwd_bwd_s": (cpu_fwd_s + cpu_bwd_s) * H * S,
        "cpu_kind": "port (oracle/gooms_port.ssm_forward_parallel + ssm_backward, float64, "
                    "one sequence x 512)", "cpu_cores": 1,
    }), flush=True)


if __name__ == "__main__":
    main()
