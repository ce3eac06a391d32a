"""Long-chain driver: the SPEC harness's chain experiment (SPEC.md:391-455,
PAPER.md:364-386) on top of the blocked chain scan.

A chain of T random-normal d x d leaves (generated on the device, keyed by
(seed, t)) is scanned in windows of W leaves: each window is one
`goom_scan_chain_c64` call whose carry-in is the previous window's last prefix,
so every prefix P_t = A_t ... A_0 is produced exactly once. Prefixes are not
kept (a 1M x 512 x 512 chain is 2 TiB): each window is digested per prefix
(max log-magnitude, log Frobenius norm, finiteness), and full prefixes are
kept at a stride.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Dict, Optional

import torch

from . import ops  # registers torch.ops.goom.*


@dataclass
class ChainRun:
    digests: torch.Tensor             # (T, 4) float32: max log, log ||P_t||_F, finite, 0
    final: torch.Tensor               # P_{T-1} (d, d) complex64
    snapshots: Dict[int, torch.Tensor]


def random_chain(T: int, d: int, seed: int = 0, t0: int = 0, device=None) -> torch.Tensor:
    dev = torch.device("cuda", torch.cuda.current_device()) if device is None else device
    return torch.ops.goom.random_normal(torch.empty(0, device=dev), T, d, seed, t0)


def run_chain(T: int, d: int, seed: int = 0, window: int = 4096, block: int = 64,
              t0: int = 0, carry: Optional[torch.Tensor] = None, snapshot_every: int = 0,
              leaves: Optional[torch.Tensor] = None) -> ChainRun:
    """Scan leaves t0 .. t0+T-1 (generated, or the given `leaves` tensor) with an
    optional right carry; returns per-prefix digests, the final prefix, snapshots.

    d % 256 == 0 runs on the tile-scaled engine (ops.chain_ts): leaves are generated
    (or imported) tile-scaled, prefixes are digested inside the phase-3 LMME epilogue
    and the carry between windows stays tile-scaled. Other d use the complex64 scan +
    digest kernels."""
    if ops.ts_eligible(d):
        return _run_chain_ts(T, d, seed, window, block, t0, carry, snapshot_every, leaves)
    dev = torch.device("cuda", torch.cuda.current_device())
    digests = torch.empty((T, 4), dtype=torch.float32, device=dev)
    snaps: Dict[int, torch.Tensor] = {}
    for w0 in range(0, T, window):
        n = min(window, T - w0)
        A = leaves[w0:w0 + n] if leaves is not None else random_chain(n, d, seed, t0 + w0, dev)
        P = torch.ops.goom.scan_chain(A, block, carry)
        digests[w0:w0 + n] = torch.ops.goom.digest(P)
        if snapshot_every:
            for t in range(w0, w0 + n):
                if (t0 + t) % snapshot_every == 0:
                    snaps[t0 + t] = P[t - w0].clone()
        carry = P[n - 1].clone()
        del P, A
    return ChainRun(digests, carry, snaps)


def _run_chain_ts(T, d, seed, window, block, t0, carry, snapshot_every, leaves) -> ChainRun:
    dev = torch.device("cuda", torch.cuda.current_device())
    digests = torch.empty((T, 4), dtype=torch.float32, device=dev)
    snaps: Dict[int, torch.Tensor] = {}
    c = ops.ts_from_goom(carry.reshape(1, d, d)) if carry is not None else None
    for w0 in range(0, T, window):
        n = min(window, T - w0)
        if leaves is not None:
            A = ops.ts_from_goom(leaves[w0:w0 + n])
        else:
            A = ops.ts_random_normal(n, d, seed, t0 + w0, dev)
        want = bool(snapshot_every) and any((t0 + t) % snapshot_every == 0
                                            for t in range(w0, w0 + n))
        P, dg, c = ops.chain_ts(A, block, c, out=want, digests=True, carry_out=True)
        digests[w0:w0 + n] = dg
        if want:
            for t in range(w0, w0 + n):
                if (t0 + t) % snapshot_every == 0:
                    snaps[t0 + t] = P[t - w0].clone()
        del P, A
    return ChainRun(digests, ops.ts_to_goom(c)[0], snaps)


def chain_total(A: torch.Tensor) -> torch.Tensor:
    """P = A_{T-1} ... A_0 by a balanced pairwise tree of batched LMMEs (log2 T launches)."""
    X = A
    while X.shape[0] > 1:
        n = X.shape[0]
        paired = torch.ops.goom.lmme(X[1:n - n % 2:2], X[0:n - n % 2:2])  # later (x) earlier
        X = torch.cat([paired, X[n - 1:]]) if n % 2 else paired
    return X[0]


def growth_rate(digests: torch.Tensor) -> float:
    """Per-step growth of log ||P_t||_F: ~ (ln 2 + psi(d/2)) / 2 for Gaussian leaves
    (the top Lyapunov exponent of random N(0,1) products)."""
    lf = digests[:, 1].double()
    T = lf.shape[0]
    if T < 3:
        return float("nan")
    h = T // 2
    return float((lf[-1] - lf[h]) / (T - 1 - h))
