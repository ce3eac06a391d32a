"""Command-line front end (the reference's pyproject names `gooms.cli:main`
but ships no cli.py). Every subcommand writes CSV to stdout (or --out) whose first lines
are the `#`-prefixed run manifest; the CSV body depends only on the command line (same
seed, same body). Exit codes: 0 success, 1 runtime / numerical failure, 2 usage error.

  python -m paper_2510_03426_b200 chain --d 8 --steps 100000 --backend goom64 --trials 30
  python -m paper_2510_03426_b200 lyapunov spectrum --system lorenz --steps 100000 --method par
  python -m paper_2510_03426_b200 lyapunov lle --system henon --steps 100000 --method par
  python -m paper_2510_03426_b200 ssm --d 8 --T 512 --rho 1.5 --check
  python -m paper_2510_03426_b200 errbench --op square --low 1e-6 --high 1e6 --samples 10000 --backing 32
  python -m paper_2510_03426_b200 scanselftest --len 1024 --d 8 --blocks 4,16,64

Every computation runs through the library's GPU kernels; the host only generates inputs
(systems, random matrices) and evaluates the 50-digit references of `errbench` / `ssm --check`.
"""

from __future__ import annotations

import argparse
import io
import math
import shlex
import sys
import time

import numpy as np

VERSION = "goom-b200 0.1.0"


class UsageError(Exception):
    pass


class _Parser(argparse.ArgumentParser):
    def error(self, message):  # argparse's own exit(2) with usage, raised so main() controls it
        raise UsageError(f"{self.prog}: error: {message}\n{self.format_usage()}")


def _parser() -> argparse.ArgumentParser:
    p = _Parser(prog="goom", description="GOOM LMME scans on B200 (arXiv 2510.03426)")
    p.add_argument("--out", help="CSV file (default: stdout)")
    p.add_argument("--workers", type=int, help="host worker count (GOOM_WORKERS fallback)")
    sub = p.add_subparsers(dest="cmd", required=True, parser_class=_Parser)

    c = sub.add_parser("chain", help="chain survival (paper Fig. 1, SPEC run_chain)")
    c.add_argument("--d", type=int, required=True)
    c.add_argument("--steps", type=int, default=100_000)
    c.add_argument("--backend", default="goom64", choices=["real64", "real32", "goom64", "goom32"])
    c.add_argument("--trials", type=int, default=1)
    c.add_argument("--seed", type=int, default=0)

    ly = sub.add_parser("lyapunov", help="Lyapunov spectrum / largest exponent")
    ly.add_argument("what", choices=["spectrum", "lle"])
    ly.add_argument("--system", required=True, help="lorenz | rossler | henon | file:<path>")
    ly.add_argument("--steps", type=int, default=100_000)
    ly.add_argument("--method", default="par", choices=["seq", "par"])
    ly.add_argument("--seed", type=int, default=0)
    ly.add_argument("--burn-in", type=int, default=10_000)
    ly.add_argument("--threshold", type=float, default=0.99)
    ly.add_argument("--check-interval", type=int, default=12)

    s = sub.add_parser("ssm", help="stabilisation-free SSM forward pass")
    s.add_argument("--d", type=int, required=True)
    s.add_argument("--T", type=int, default=512)
    s.add_argument("--rho", type=float, default=1.5, help="spectral radius of A")
    s.add_argument("--seed", type=int, default=0)
    s.add_argument("--check", action="store_true", help="compare with a 50-digit recurrence")

    e = sub.add_parser("errbench", help="errors vs a 50-digit reference (Appendix D)")
    e.add_argument("--op", required=True)
    e.add_argument("--low", type=float, default=1e-6)
    e.add_argument("--high", type=float, default=1e6)
    e.add_argument("--samples", type=int, default=10_000)
    e.add_argument("--backing", type=int, default=32, choices=[32, 64])
    e.add_argument("--seed", type=int, default=0)

    t = sub.add_parser("scanselftest", help="parallel vs sequential scan equivalence")
    t.add_argument("--len", type=int, default=1024)
    t.add_argument("--d", type=int, default=8)
    t.add_argument("--blocks", default="4,16,64")
    t.add_argument("--seed", type=int, default=0)
    t.add_argument("--tol", type=float, default=1e-10)
    return p


def _manifest(argv, args, backing, elapsed) -> str:
    from .systems import RNG_NAME, worker_count

    lines = [f"command: goom {shlex.join(argv)}", f"seed: {getattr(args, 'seed', 0)}",
             f"backing: {backing}", f"workers: {worker_count(args.workers)}",
             f"rng: {RNG_NAME} (host inputs); philox4x32-10 (device leaves, keyed by index)",
             f"version: {VERSION}", f"wall_clock_s: {elapsed:.3f}"]
    return "".join(f"# {x}\n" for x in lines)


def _csv(header, rows) -> str:
    out = io.StringIO()
    out.write(",".join(header) + "\n")
    for r in rows:
        out.write(",".join(_fmt(v) for v in r) + "\n")
    return out.getvalue()


def _fmt(v) -> str:
    if v is None:
        return "none"
    if isinstance(v, float):
        return repr(v)
    return str(v)


# ---------------------------------------------------------------------------


def cmd_chain(args):
    from .harness import ChainConfig, chain_survival

    r = chain_survival(ChainConfig(args.d, args.steps, args.backend, args.seed, args.trials))
    rows = [(args.d, i, args.backend, s, m) for i, (s, m) in
            enumerate(zip(r.survived_steps, r.failure_mode))]
    return _csv(("d", "trial", "backend", "survived_steps", "failure_mode"), rows), args.backend, []


def _chain_for(args):
    from . import lyapunov, systems

    if args.system.startswith("file:"):
        return lyapunov.load_jacobian_chain(args.system[5:])
    if args.system not in systems.BUILTIN_SYSTEMS:
        raise UsageError(f"unknown system {args.system!r}: lorenz, rossler, henon or file:<path>")
    sysm = systems.BUILTIN_SYSTEMS[args.system]()
    return lyapunov.integrate_chain(sysm, burn_in=args.burn_in, T=args.steps, seed=args.seed)


def cmd_lyapunov(args):
    from . import lyapunov, systems

    chain = _chain_for(args)
    if args.what == "spectrum":
        if args.method == "par":
            res = lyapunov.spectrum_parallel(chain, colinearity_threshold=args.threshold,
                                             check_interval=args.check_interval)
        else:
            res = lyapunov.spectrum_sequential(chain)
        rows = [(i, float(l), res.method, res.wall_seconds, res.resets)
                for i, l in enumerate(res.lambdas)]
    else:
        u0 = systems.make_rng(args.seed, 1).standard_normal(chain.dim)
        u0 /= np.linalg.norm(u0)
        t0 = time.perf_counter()
        lam = (lyapunov.lle_parallel(chain, u0) if args.method == "par" else
               lyapunov.lle_sequential(chain, u0))
        rows = [(0, float(lam), "parallel" if args.method == "par" else "sequential",
                 time.perf_counter() - t0, 0)]
    return (_csv(("exponent_index", "lambda", "method", "wall_seconds", "resets"), rows),
            "complex128", [])


def _ssm_case(d, T, rho, seed):
    from .systems import make_rng

    rng = make_rng(seed, 2)
    A = rng.standard_normal((d, d))
    A *= rho / np.max(np.abs(np.linalg.eigvals(A)))
    B = rng.standard_normal((d, d)) / math.sqrt(d)
    C = rng.standard_normal((2 * d, d)) / math.sqrt(d)
    D = rng.standard_normal((2 * d, d)) / math.sqrt(d)
    return A, B, C, D, rng.standard_normal(d), rng.standard_normal((T, d))


def ssm_oracle_states(A, B, x0, u, digits=50):
    """x_t = A x_{t-1} + B u_t in `digits`-digit arithmetic (mpmath), returned as
    (log|x_t|, sign) float64 arrays: the high-precision recurrence of SPEC acceptance 8."""
    import mpmath

    with mpmath.workdps(digits):
        d = len(x0)
        Am = [[mpmath.mpf(float(v)) for v in row] for row in A]
        Bu = [[mpmath.fsum(mpmath.mpf(float(B[i][k])) * mpmath.mpf(float(ut[k])) for k in range(d))
               for i in range(d)] for ut in u]
        x = [mpmath.mpf(float(v)) for v in x0]
        logs = np.empty((len(u), d))
        signs = np.empty((len(u), d))
        for t in range(len(u)):
            x = [mpmath.fsum(Am[i][k] * x[k] for k in range(d)) + Bu[t][i] for i in range(d)]
            for i, v in enumerate(x):
                logs[t, i] = float(mpmath.log(abs(v))) if v != 0 else -math.inf
                signs[t, i] = -1.0 if v < 0 else 1.0
    return logs, signs


def cmd_ssm(args):
    from . import ssm

    A, B, C, D, x0, u = _ssm_case(args.d, args.T, args.rho, args.seed)
    p = ssm.SsmParams(A, B, C, D)
    par = ssm.ssm_forward_parallel(p, x0, u)
    rows = [(t, float(par.state_log[t].max()), float(par.scales[t]), float(par.y[t, 0]))
            for t in range(args.T)]
    notes = []
    ok = True
    if args.check:
        seq = ssm.ssm_forward_sequential(p, x0, u)
        ol, os_ = ssm_oracle_states(A, B, x0, u)
        # shared rescaling: every state divided by its own largest magnitude (Eq. 29)
        c = ol.max(axis=1, keepdims=True)
        got = par.state_sign * np.exp(par.state_log - c)
        want = os_ * np.exp(ol - c)
        err = float(np.max(np.abs(got - want)))
        seq_par = float(np.max(np.abs(par.state_log - seq.state_log) /
                               np.maximum(1.0, np.abs(seq.state_log))))
        with np.errstate(all="ignore"):
            xr = np.array(x0, dtype=np.float64)
            direct_finite = True
            for t in range(args.T):
                xr = A @ xr + B @ u[t]
                direct_finite &= bool(np.all(np.isfinite(xr)))
        ok = err <= 1e-9 and seq_par <= 1e-8
        notes = [f"check: max_scaled_err_vs_50digit={err:.3e} (<= 1e-9)",
                 f"check: parallel_vs_sequential_rel_log={seq_par:.3e} (<= 1e-8)",
                 f"check: direct_binary64_recurrence_finite={direct_finite}",
                 f"check: {'ok' if ok else 'FAILED'}"]
    return (_csv(("t", "max_state_log", "scale", "y0"), rows), "complex128", notes,
            0 if ok else 1)


def cmd_errbench(args):
    from .harness import ERRBENCH_OPS, errbench

    if args.op not in ERRBENCH_OPS:
        raise UsageError(f"unknown op {args.op!r}; one of {', '.join(ERRBENCH_OPS)}")
    st = errbench(args.op, args.low, args.high, args.samples, args.backing, args.seed)
    row = (st.op_name, st.input_range[0], st.input_range[1], st.samples, st.backing,
           st.max_abs_log10_error, st.mean_abs_log10_error, st.max_error_digits,
           st.mean_error_digits, st.direct_max_abs_log10_error, st.direct_mean_abs_log10_error)
    hdr = ("op", "range_low", "range_high", "samples", "backing", "max_abs_log10_error",
           "mean_abs_log10_error", "max_error_digits", "mean_error_digits",
           "direct_max_abs_log10_error", "direct_mean_abs_log10_error")
    return _csv(hdr, [row]), f"binary{args.backing}", []


def cmd_scanselftest(args):
    from . import scan
    from .core import _log_sign_arrays

    try:
        blocks = [int(b) for b in args.blocks.split(",") if b]
    except ValueError:
        raise UsageError("--blocks takes a comma-separated list of integers")
    if not blocks or min(blocks) < 1 or args.len < 1 or args.d < 1:
        raise UsageError("--len, --d and every block must be >= 1")
    from .systems import make_rng

    rng = make_rng(args.seed, 3)
    T, d = args.len, args.d
    al, as_ = _log_sign_arrays(rng.standard_normal((T, d, d)))
    bl, bs = _log_sign_arrays(rng.standard_normal((T, d, d)))

    def stack():  # the reference's array form: derived stacks hand back numpy
        return scan._Stack(al, as_, bl, bs, np.zeros(T, dtype=bool))

    def host(x):  # a list of ScanPairs (the sequential selective scan) as a host stack
        if isinstance(x, scan._Stack):
            return x
        st = scan._Stack.from_pairs(x)
        st.host = True
        return st

    seq = scan.scan_parallel(stack(), scan.combine_affine, T)  # block >= T: the left fold
    rows, ok = [], True
    for b in blocks:
        par = scan.scan_parallel(stack(), scan.combine_affine, b)
        e = max(_rel_log(par.alog, seq.alog), _rel_log(par.blog, seq.blog))
        flips = int(np.sum(par.asign != seq.asign) + np.sum(par.bsign != seq.bsign))
        good = e <= args.tol and flips == 0
        ok &= good
        rows.append(("affine", b, e, flips, None, good))  # max rel-log over every element
    # selective resets (norm threshold, consume_leaf): sites exact, states within tol
    pol = scan.norm_threshold_policy(threshold=12.0, interval=1)
    # SPEC acceptance 3: sites exact, the final compound state (B after a reset, else A)
    # within tol as values (scaled by its largest magnitude; Q factors of resets hold entries
    # near cancellation whose per-element log is ill-conditioned)
    want, wsites = scan.scan_selective(stack(), pol)
    wl, ws = _states(host(want))
    for b in blocks:
        got, sites = scan.scan_selective(stack(), pol, b)
        gl, gs = _states(host(got))
        top = wl[-1].max()
        with np.errstate(invalid="ignore", over="ignore"):
            e = float(np.max(np.abs(gs[-1] * np.exp(gl[-1] - top) - ws[-1] * np.exp(wl[-1] - top))))
        flips = int(np.sum((gs[-1] != ws[-1]) & (wl[-1] > top - 20.0)))
        good = sites == wsites and len(wsites) >= 3 and e <= args.tol and flips == 0
        ok &= good
        rows.append(("selective", b, e, flips, len(sites), good))
    return (_csv(("scan", "block", "max_err", "sign_mismatches", "resets", "ok"), rows),
            "complex128", [f"selftest: {'ok' if ok else 'FAILED'}"], 0 if ok else 1)


def _states(st):
    f = np.asarray(st.flags, dtype=bool)[:, None, None]
    return np.where(f, st.blog, st.alog), np.where(f, st.bsign, st.asign)


def _rel_log(x, y) -> float:
    x, y = np.asarray(x), np.asarray(y)
    both = (x == -np.inf) & (y == -np.inf)
    with np.errstate(invalid="ignore"):
        d = np.where(both, 0.0, np.abs(x - y) / np.maximum(1.0, np.abs(y)))
    return float(np.nanmax(np.where(np.isnan(d), np.inf, d))) if d.size else 0.0


COMMANDS = {"chain": cmd_chain, "lyapunov": cmd_lyapunov, "ssm": cmd_ssm,
            "errbench": cmd_errbench, "scanselftest": cmd_scanselftest}


def main(argv=None) -> int:
    argv = list(sys.argv[1:] if argv is None else argv)
    try:
        args = _parser().parse_args(argv)
        t0 = time.perf_counter()
        res = COMMANDS[args.cmd](args)
    except UsageError as e:
        msg = str(e) if str(e).startswith("goom") else f"goom: error: {e}"
        sys.stderr.write(msg + ("\n" if not msg.endswith("\n") else ""))
        return 2
    except (ValueError, RuntimeError, ArithmeticError, OSError) as e:
        sys.stderr.write(f"goom {argv[0] if argv else ''}: {type(e).__name__}: {e}\n")
        return 1
    body, backing, notes = res[0], res[1], res[2]
    rc = res[3] if len(res) > 3 else 0
    text = _manifest(argv, args, backing, time.perf_counter() - t0) + body + \
        "".join(f"# {n}\n" for n in notes)
    if args.out:
        with open(args.out, "w") as f:
            f.write(text)
    else:
        sys.stdout.write(text)
    return rc


if __name__ == "__main__":
    sys.exit(main())
