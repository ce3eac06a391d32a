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

import math
from dataclasses import dataclass, field
from typing import Dict, Optional, Sequence

import numpy as np
import torch

from . import ops  # registers torch.ops.goom.*


@dataclass
class ChainRun:
    digests: torch.Tensor             # (T, 4) float32: max log, log ||P_t||_F, finite, 0
    final: torch.Tensor               # P_{T-1} (d, d) complex64
    snapshots: Dict[int, torch.Tensor]
    # tile-scaled engine only: the same snapshots at the engine's own precision
    # (ops.ts_log_sign gives exact float64 logs; the complex64 ones round to float32)
    snapshots_ts: Dict[int, "ops.TsMats"] = field(default_factory=dict)
    # tile-scaled engine only: for each requested block start t, the block carry the engine
    # applies to prefixes t .. t + block - 1 (its own P_{t-1}; ops.chain_ts `carries`)
    anchors_ts: Dict[int, "ops.TsMats"] = field(default_factory=dict)


def random_chain(T: int, d: int, seed: int = 0, t0: int = 0, device=None) -> torch.Tensor:
    dev = torch.device("cuda", torch.cuda.current_device()) if device is None else device
    return torch.ops.goom.random_normal(torch.empty(0, device=dev), T, d, seed, t0)


def _snapshot_set(T: int, t0: int, snapshot_every: int, snapshots: Sequence[int]):
    """Absolute prefix indices in [t0, t0 + T) to keep as full complex64 matrices."""
    want = {int(t) for t in snapshots if t0 <= int(t) < t0 + T}
    if snapshot_every:
        first = -(-t0 // snapshot_every) * snapshot_every
        want.update(range(first, t0 + T, snapshot_every))
    return want


def long_chain_eligible(d: int, dtype) -> bool:
    """The long-chain engine (ops.scan_chain_long) takes d <= 32, and d = 64 in complex64."""
    return d <= 32 or (d == 64 and dtype == torch.complex64)


def run_chain(T: int, d: int, seed: int = 0, window: int = 4096, block: int = 64,
              t0: int = 0, carry: Optional[torch.Tensor] = None, snapshot_every: int = 0,
              leaves: Optional[torch.Tensor] = None, snapshots: Sequence[int] = (),
              anchors: Sequence[int] = ()) -> ChainRun:
    """Scan leaves t0 .. t0+T-1 (generated, or the given `leaves` tensor) with an
    optional right carry; returns per-prefix digests, the final prefix, snapshots.

    Snapshots: the full prefixes P_t for every absolute t in `snapshots` (and every multiple
    of `snapshot_every`) inside the run, keyed by t. On the tile-scaled engine each one is
    recomputed from the window's workspace (L_t (x) its block carry, one product), so
    keeping them costs no full-window output. Anchors (tile-scaled engine): absolute block
    starts t (multiples of `block` from a window start; windows are multiples of `block`)
    whose block carry — the engine's own P_{t-1}, applied on the right of every local
    product of that block — is returned in `anchors_ts[t]` (re-anchored parity checks).

    `leaves` may be complex64 GOOMs on the device, or real float32 matrices — on the
    device, or in pinned host memory, in which case each window's host->device copy
    runs on a copy stream overlapped with the previous window's scan (tile-scaled path).

    d % 256 == 0 runs on the tile-scaled engine (ops.chain_ts): leaves are generated
    (or imported) tile-scaled, prefixes are digested inside the phase-3 LMME epilogue
    and the carry between windows stays tile-scaled. d <= 32 and d = 64 run the long-chain engine
    (ops.scan_chain_long); other d the complex64 block-tree scan. Both + digest kernels."""
    want = _snapshot_set(T, t0, snapshot_every, snapshots)
    if ops.ts_eligible(d):
        return _run_chain_ts(T, d, seed, window, block, t0, carry, want, leaves, anchors)
    dev = torch.device("cuda", torch.cuda.current_device())
    if leaves is not None and leaves.dtype == torch.float32:  # real matrices -> GOOMs
        leaves = torch.ops.goom.from_real(leaves.to(dev), float("-inf"), False)
    digests = torch.empty((T, 4), dtype=torch.float32, device=dev)
    snaps: Dict[int, torch.Tensor] = {}
    for w0 in range(0, T, window):
        n = min(window, T - w0)
        A = leaves[w0:w0 + n] if leaves is not None else random_chain(n, d, seed, t0 + w0, dev)
        # d <= 32: the long-chain engine (scan_long.cu; a fixed reduce-then-scan tree, the
        # block size only shapes the reference tree the other engines keep)
        P = (torch.ops.goom.scan_chain_long(A, carry) if long_chain_eligible(d, A.dtype) else
             torch.ops.goom.scan_chain(A, block, carry))
        digests[w0:w0 + n] = torch.ops.goom.digest(P)
        for t in range(w0, w0 + n):
            if t0 + t in want:
                snaps[t0 + t] = P[t - w0].clone()
        carry = P[n - 1].clone()
        del P, A
    return ChainRun(digests, carry, snaps)


_ORDERED_ZERO = -2147483648  # float_to_ordered(0.0f) = 0x80000000 as int32


def real_leaves_ts(x: torch.Tensor) -> "ops.TsMats":
    """Real float32 leaves (device) as tile-scaled matrices without a copy: U = x, q = 0,
    G = bits(0) (a real matrix is its own tile-scaled form with unit scales)."""
    T, d = x.shape[0], x.shape[-1]
    q = torch.zeros((T, d, d // 256), dtype=torch.float32, device=x.device)
    G = torch.full((T, d // 256), _ORDERED_ZERO, dtype=torch.int32, device=x.device)
    return ops.TsMats(x, q, G)


def _window_anchor_blocks(anchors, a0: int, n: int, block: int):
    """Block indices of a window starting at absolute index a0 (n leaves) for the anchors
    that fall inside it."""
    ks = []
    for t in anchors:
        if a0 <= t < a0 + n:
            if (t - a0) % block:
                raise ValueError(f"anchor {t} is not a block start (block {block})")
            ks.append((t - a0) // block)
    return sorted(ks)


def _run_chain_ts(T, d, seed, window, block, t0, carry, want, leaves, anchors=()) -> ChainRun:
    dev = torch.device("cuda", torch.cuda.current_device())
    digests = torch.empty((T, 4), dtype=torch.float32, device=dev)
    snaps: Dict[int, torch.Tensor] = {}
    snaps_ts: Dict[int, ops.TsMats] = {}
    anch: Dict[int, ops.TsMats] = {}
    if anchors and window % block:
        raise ValueError("anchors need window to be a multiple of block")
    c = ops.ts_from_goom(carry.reshape(1, d, d)) if carry is not None else None
    streamed = leaves is not None and not leaves.is_cuda
    if streamed:
        if leaves.dtype != torch.float32:
            raise ValueError("host leaves are streamed as real float32 matrices")
        main = torch.cuda.current_stream()
        copy = torch.cuda.Stream(device=dev)
        bufs = [torch.empty((min(window, T), d, d), dtype=torch.float32, device=dev)
                for _ in range(2)]
        ready = [torch.cuda.Event(), torch.cuda.Event()]
        free = [torch.cuda.Event(), torch.cuda.Event()]

        def h2d(i, w0):
            n = min(window, T - w0)
            copy.wait_event(free[i % 2])
            with torch.cuda.stream(copy):
                bufs[i % 2][:n].copy_(leaves[w0:w0 + n], non_blocking=True)
                ready[i % 2].record(copy)
        for e in free:
            e.record(main)
        h2d(0, 0)
    starts = list(range(0, T, window))
    for i, w0 in enumerate(starts):
        n = min(window, T - w0)
        if streamed:
            main.wait_event(ready[i % 2])
            if i + 1 < len(starts):
                h2d(i + 1, starts[i + 1])
            A = real_leaves_ts(bufs[i % 2][:n])
        elif leaves is not None:
            x = leaves[w0:w0 + n]
            A = real_leaves_ts(x.contiguous()) if x.dtype == torch.float32 else ops.ts_from_goom(x)
        else:
            A = ops.ts_random_normal(n, d, seed, t0 + w0, dev)
        local = sorted(t - t0 - w0 for t in want if t0 + w0 <= t < t0 + w0 + n)
        ks = _window_anchor_blocks(anchors, t0 + w0, n, block)
        _, dg, c, S, K = ops.chain_ts(A, block, c, digests=True, carry_out=True,
                                      snapshots=local, carries=ks)
        digests[w0:w0 + n] = dg
        for j, k in enumerate(ks):
            anch[t0 + w0 + k * block] = K[j:j + 1]
        if streamed:
            free[i % 2].record(main)
        if local:
            S64 = ops.ts_to_goom(S)
            for j, t in enumerate(local):
                snaps[t0 + w0 + t] = S64[j]
                snaps_ts[t0 + w0 + t] = S[j:j + 1]
        del A, S, K
    return ChainRun(digests, ops.ts_to_goom(c)[0], snaps, snaps_ts, anch)


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


# ---------------------------------------------------------------------------
# the chain-survival experiment (SPEC.md:391-455 run_chain; paper Fig. 1, Eq. 13-14)

BACKENDS = ("real64", "real32", "goom64", "goom32")


@dataclass(frozen=True)
class ChainConfig:
    """d x d random-normal chains of up to T_max steps, `trials` of them (SPEC ChainConfig)."""

    d: int
    T_max: int
    backend: str
    seed: int = 0
    trials: int = 1

    def __post_init__(self):
        if self.d < 1 or self.T_max < 1 or self.trials < 1:
            raise ValueError("d, T_max and trials must be >= 1")
        if self.backend not in BACKENDS:
            raise ValueError(f"backend must be one of {BACKENDS}")


@dataclass
class ChainResult:
    """Per trial: steps survived (<= T_max), whether the chain completed, and the first
    failure ('overflow', 'underflow', 'nan' or None)."""

    survived_steps: list
    completed: list
    failure_mode: list


def _first_failure(bad: torch.Tensor):
    """Index of the first True along dim 0 per column (T_max when none)."""
    T = bad.shape[0]
    idx = torch.arange(T, device=bad.device)[:, None].expand_as(bad)
    return torch.where(bad, idx, torch.full_like(idx, T)).min(dim=0).values


def chain_survival(cfg: ChainConfig) -> ChainResult:
    """Iterate S_t = A_t S_{t-1} (S_0 = A_0) over random-normal leaves (device RNG keyed by
    (seed + trial, t)) until T_max or the first non-finite state. Real backends multiply
    plainly in float64 / float32 (torch on the GPU, one batched product per step over the
    trials); GOOM backends run the chain scan on complex128 / complex64 GOOMs, all T_max
    prefixes, and a state fails when any log-magnitude is non-finite (NaN or +inf) — which
    for GOOMs is the representable range of the float64 / float32 log itself."""
    dev = torch.device("cuda", torch.cuda.current_device())
    d, T, n = cfg.d, cfg.T_max, cfg.trials
    leaves = [random_chain(T, d, cfg.seed + i, 0, dev) for i in range(n)]
    steps, modes = [], []
    if cfg.backend.startswith("real"):
        rt = torch.float64 if cfg.backend == "real64" else torch.float32
        A = torch.stack([torch.ops.goom.to_real(L, True) for L in leaves], dim=1).to(rt)  # (T, n, d, d)
        S = A[0].clone()
        alive = torch.ones(n, dtype=torch.bool, device=dev)
        surv = torch.full((n,), T, dtype=torch.int64, device=dev)
        mode = torch.zeros(n, dtype=torch.int8, device=dev)  # 0 none, 1 overflow, 2 underflow, 3 nan
        for t in range(T):
            if t:
                S = torch.bmm(A[t], S)
            flat = S.reshape(n, -1)
            nan = torch.isnan(flat).any(dim=1)
            inf = torch.isinf(flat).any(dim=1)
            zero = (flat == 0).all(dim=1)
            fail = alive & (nan | inf | zero)
            surv = torch.where(fail, torch.full_like(surv, t), surv)
            mode = torch.where(fail, torch.where(nan, 3, torch.where(inf, 1, 2)).to(torch.int8), mode)
            alive &= ~fail
            if t % 256 == 255 and not bool(alive.any()):
                break
        steps = surv.tolist()
        names = {0: None, 1: "overflow", 2: "underflow", 3: "nan"}
        modes = [names[int(m)] for m in mode.tolist()]
    else:
        ct = torch.complex128 if cfg.backend == "goom64" else torch.complex64
        for L in leaves:
            L = L.to(ct)
            P = torch.ops.goom.scan_chain_long(L, None) if long_chain_eligible(d, L.dtype) else \
                torch.ops.goom.scan_chain(L, 64, None)
            lg = P.real.reshape(T, -1)
            bad = torch.isnan(lg).any(dim=1) | torch.isposinf(lg).any(dim=1)
            first = int(_first_failure(bad[:, None])[0])
            steps.append(first)
            modes.append(None if first == T else
                         ("nan" if bool(torch.isnan(lg[first]).any()) else "overflow"))
    return ChainResult(survived_steps=steps, completed=[s == T for s in steps],
                       failure_mode=modes)


# ---------------------------------------------------------------------------
# error benchmarking against a 50-digit reference (Appendix D)

ERRBENCH_OPS = ("identity", "reciprocal", "sqrt", "square", "log", "exp", "add", "mul", "matmul")
ORACLE_DIGITS = 50


@dataclass
class ErrorStats:
    """SPEC ErrorStats plus the paper's Appendix D figures.

    abs_log10_error per sample = |log10|y| - log10|y_ref||: the error of the result's
    decimal order of magnitude (relative error / ln 10 for small errors). error_digits per
    sample = log10|y - y_ref|, the paper's "number of decimal digits of error" (exact
    results are left out of its statistics). matmul reports the Frobenius error normalised
    by ||C_ref||_F in max / mean (one sample). `direct_*` is the same operation evaluated in
    the backing float format itself, for comparison."""

    op_name: str
    input_range: tuple
    max_abs_log10_error: float
    mean_abs_log10_error: float
    samples: int
    backing: int
    max_error_digits: float
    mean_error_digits: float
    direct_max_abs_log10_error: float
    direct_mean_abs_log10_error: float


def oracle_eval(op: str, *args):
    """The operation in >= 50-digit software arithmetic (mpmath): scalars for the scalar
    ops (args are Python floats, converted exactly), a list of lists for matmul (args are
    two 2-D float arrays). Domain violations (log or sqrt of a negative) raise ValueError."""
    import mpmath

    with mpmath.workdps(ORACLE_DIGITS):
        if op == "matmul":
            a, b = args
            n, k, m = len(a), len(b), len(b[0])
            A = [[mpmath.mpf(float(a[i][j])) for j in range(k)] for i in range(n)]
            B = [[mpmath.mpf(float(b[i][j])) for j in range(m)] for i in range(k)]
            return [[mpmath.fsum(A[i][q] * B[q][j] for q in range(k)) for j in range(m)]
                    for i in range(n)]
        x = [mpmath.mpf(float(v)) for v in args]
        if op in ("log", "sqrt") and x[0] < 0:
            raise ValueError(f"{op} of a negative value in real arithmetic")
        table = {
            "identity": lambda: x[0],
            "reciprocal": lambda: 1 / x[0],
            "sqrt": lambda: mpmath.sqrt(x[0]),
            "square": lambda: x[0] * x[0],
            "log": lambda: mpmath.log(x[0]),
            "exp": lambda: mpmath.exp(x[0]),
            "add": lambda: x[0] + x[1],
            "mul": lambda: x[0] * x[1],
        }
        if op not in table:
            raise ValueError(f"unknown op {op!r}; one of {ERRBENCH_OPS}")
        return table[op]()


def _goom_eval(op: str, xs, ys, backing: int):
    """op over GOOMs on the GPU: inputs mapped by from_real, computed in the log domain
    (the library's kernels for add = gadd and matmul = LMME), mapped back by to_real."""
    dev = torch.device("cuda", torch.cuda.current_device())
    double = backing == 64
    rt = torch.float64 if double else torch.float32

    def goom(v):
        return torch.ops.goom.from_real(torch.as_tensor(v, dtype=rt, device=dev), float("-inf"),
                                        double)

    def real(z):
        return torch.ops.goom.to_real(z, double).cpu().numpy().astype(np.float64)

    gx = goom(xs)
    if op == "identity":
        return real(gx)
    if op == "reciprocal":
        return real(torch.complex(-gx.real, gx.imag))
    if op == "sqrt":
        return real(torch.complex(0.5 * gx.real, gx.imag))
    if op == "square":
        return real(torch.complex(2.0 * gx.real, torch.zeros_like(gx.imag)))
    if op == "log":   # the log-magnitude is the GOOM's real part (x > 0)
        return real(goom(gx.real))
    if op == "exp":   # e^x as a GOOM is (x, 0)
        return real(torch.complex(torch.as_tensor(xs, dtype=rt, device=dev),
                                  torch.zeros(len(xs), dtype=rt, device=dev)))
    gy = goom(ys)
    if op == "add":
        return real(torch.ops.goom.gadd(gx, gy))
    if op == "mul":
        return real(torch.complex(gx.real + gy.real, gx.imag + gy.imag))
    if op == "matmul":
        return real(torch.ops.goom.lmme(gx, gy))
    raise ValueError(f"unknown op {op!r}; one of {ERRBENCH_OPS}")


def _direct_eval(op: str, xs, ys, backing: int):
    dt = np.float64 if backing == 64 else np.float32
    x = np.asarray(xs, dtype=dt)
    y = None if ys is None else np.asarray(ys, dtype=dt)
    with np.errstate(all="ignore"):
        out = {"identity": lambda: x, "reciprocal": lambda: dt(1) / x, "sqrt": lambda: np.sqrt(x),
               "square": lambda: x * x, "log": lambda: np.log(x), "exp": lambda: np.exp(x),
               "add": lambda: x + y, "mul": lambda: x * y, "matmul": lambda: x @ y}[op]()
    return np.asarray(out, dtype=np.float64)


def errbench(op: str, range_low: float = 1e-6, range_high: float = 1e6, samples: int = 10_000,
             backing: int = 32, seed: int = 0) -> ErrorStats:
    """Errors of `op` evaluated over GOOMs against the 50-digit reference (SPEC errbench,
    PAPER.md:880). One-argument ops: `samples` inputs equally spaced in decimal digits over
    [range_low, range_high]; two-argument ops: a ceil(sqrt(samples))^2 grid of such pairs;
    matmul: two `samples` x `samples` N(0,1) matrices (the range does not apply), error
    normalised by the product's Frobenius norm. backing 32 / 64: complex64 / complex128."""
    import mpmath

    if op not in ERRBENCH_OPS:
        raise ValueError(f"unknown op {op!r}; one of {ERRBENCH_OPS}")
    if backing not in (32, 64):
        raise ValueError("backing must be 32 or 64")
    if samples < 1:
        raise ValueError("samples must be >= 1")
    dt = np.float64 if backing == 64 else np.float32
    if op == "matmul":
        rng = np.random.default_rng(seed)
        a = rng.standard_normal((samples, samples)).astype(dt)
        b = rng.standard_normal((samples, samples)).astype(dt)
        ref = oracle_eval("matmul", a.tolist(), b.tolist())
        got = _goom_eval(op, a, b, backing)
        direct = _direct_eval(op, a, b, backing)
        with mpmath.workdps(ORACLE_DIGITS):
            fro = mpmath.sqrt(mpmath.fsum(v * v for row in ref for v in row))

            def nerr(c):
                return float(mpmath.sqrt(mpmath.fsum((mpmath.mpf(float(c[i][j])) - ref[i][j]) ** 2
                                                     for i in range(samples)
                                                     for j in range(samples))) / fro)
            e, e_dir = nerr(got), nerr(direct)
        return ErrorStats(op, (samples, samples), e, e, 1, backing, math.log10(e) if e else
                          float("-inf"), math.log10(e) if e else float("-inf"), e_dir, e_dir)
    if not (0.0 < range_low < range_high) and op != "exp":
        raise ValueError("need 0 < range_low < range_high (log-spaced sampling)")
    if op == "exp" and not range_low < range_high:
        raise ValueError("need range_low < range_high")
    lo, hi = (math.log10(range_low), math.log10(range_high)) if range_low > 0 else (None, None)
    if op in ("add", "mul"):
        n = int(math.ceil(math.sqrt(samples)))
        grid = np.logspace(lo, hi, n).astype(dt)
        xs, ys = np.repeat(grid, n), np.tile(grid, n)
    else:
        xs = (np.logspace(lo, hi, samples) if lo is not None else
              np.linspace(range_low, range_high, samples)).astype(dt)
        ys = None
    got = _goom_eval(op, xs, ys, backing)
    direct = _direct_eval(op, xs, ys, backing)
    errs, digits, errs_dir = [], [], []
    with mpmath.workdps(ORACLE_DIGITS):
        for i in range(len(xs)):
            r = oracle_eval(op, xs[i]) if ys is None else oracle_eval(op, xs[i], ys[i])
            if r == 0:
                continue
            lr = mpmath.log10(abs(r))
            for val, sink in ((got[i], errs), (direct[i], errs_dir)):
                v = mpmath.mpf(float(val))
                sink.append(float(abs(mpmath.log10(abs(v)) - lr)) if v != 0 and
                            (v > 0) == (r > 0) else float("inf"))
            diff = abs(mpmath.mpf(float(got[i])) - r)
            if diff != 0:
                digits.append(float(mpmath.log10(diff)))
    e = np.asarray(errs)
    ed = np.asarray(errs_dir)
    dg = np.asarray(digits) if digits else np.asarray([float("-inf")])
    return ErrorStats(op, (float(range_low), float(range_high)), float(e.max()), float(e.mean()),
                      len(xs), backing, float(dg.max()), float(dg.mean()), float(ed.max()),
                      float(ed.mean()))
