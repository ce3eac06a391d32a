"""non-diagonal GOOM recurrence, d_state = 64, 16 heads,
batch 32, T = 4096 — 512 sequences, each head's 32 sequences one affine scan on the GPU
(ssm.ssm_forward_batched, complex128). Backward: the reference has no autodiff, so there
is nothing to be parity-tested against ("parity unpinned"); not measured.
CPU baseline: the reference algorithm (oracle port, float64) on one sequence, x 512.
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
    args = ap.parse_args()
    import torch

    from oracle import gooms_port as G
    from paper_2510_03426_b200 import ssm

    rng = np.random.default_rng(5)
    d, H, S, T = args.d, args.heads, args.batch, args.T
    params = []
    for _ in range(H):
        a = rng.standard_normal((d, d))
        a *= rng.uniform(1.0, 1.5) / np.max(np.abs(np.linalg.eigvals(a)))
        params.append(ssm.SsmParams(a, rng.standard_normal((d, d)), rng.standard_normal((2 * d, d)),
                                    rng.standard_normal((2 * d, d))))
    x0 = rng.standard_normal((H, S, d))
    u = rng.standard_normal((H, S, T, d)).astype(np.float64)
    ssm.ssm_forward_batched(params[0], x0[0, :2], u[0, :2, :256])  # warm-up
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    finite = True
    for h in range(H):
        sl, ss, c, y = ssm.ssm_forward_batched(params[h], x0[h], u[h])
        finite &= bool(torch.isfinite(sl).all() and torch.isfinite(y).all())
    torch.cuda.synchronize()
    gpu_s = time.perf_counter() - t0
    # parity spot check: head 0, sequence 0 vs the oracle port
    osl, oss, oc, oy = G.ssm_forward_parallel(params[0].A, params[0].B, params[0].C, params[0].D,
                                              x0[0, 0], u[0, 0])
    sl, ss, c, y = (t.cpu().numpy() for t in ssm.ssm_forward_batched(params[0], x0[0, :1],
                                                                       u[0, :1]))
    err = float(np.max(np.abs(sl[0] - osl) / np.maximum(1.0, np.abs(osl))))
    t1 = time.perf_counter()
    G.ssm_forward_parallel(params[1].A, params[1].B, params[1].C, params[1].D, x0[1, 0], u[1, 0])
    cpu_seq_s = time.perf_counter() - t1
    print(json.dumps({
        "config": "ssm_forward", "d": d, "heads": H, "batch": S, "T": T,
        "gpu_s": gpu_s, "gpu_steps_per_s": H * S * T / gpu_s, "finite": finite,
        "gpu_timing": "host float64 inputs -> device, states + outputs left on the device",
        "parity_rel_log_vs_oracle": err, "sign_mismatch": int(np.sum(ss[0] != oss)),
        "cpu_one_sequence_s": cpu_seq_s, "cpu_extrapolated_s": cpu_seq_s * H * S,
        "cpu_kind": "port (oracle/gooms_port.ssm_forward_parallel, float64, one sequence x 512)",
        "cpu_cores": os.cpu_count(), "backward": "not measured (no reference autodiff)",
    }), flush=True)


if __name__ == "__main__":
    main()
