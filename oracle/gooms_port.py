"""numpy restatement of the reference's LMME prefix-scan path (TEST ORACLE ONLY).

Every function below restates one reference routine of
`/root/reference/pkg/src/gooms/` (cited as file:line) on raw
(log-magnitude, sign) arrays, the reference's storage, plus the adapters to
the complex64 GOOM layout the B200 build uses at its boundary:

    log_mag = z.real ;  sign = -1 if cos(z.imag) < 0 else +1
    z       = log_mag + 1j * pi * [sign < 0]

The arithmetic order of each restated routine follows the reference (same
numpy ufunc sequence), so on float64 inputs the port reproduces the reference
bit for bit; `tests/test_oracle_golden.py` checks that against vectors the
reference itself produced.

This module is the checker and the CPU baseline. The product package never
imports it.
"""

from __future__ import annotations

import math
from dataclasses import dataclass
from typing import Callable, Optional

import numpy as np

NEG_INF = float("-inf")
PI32 = np.float32(np.pi)


# ---------------------------------------------------------------------------
# boundary adapters: complex GOOM  <->  (log_mag, sign) parity storage


def split_complex(z, dtype=np.float64):
    """complex GOOM -> (log_mag, sign) in `dtype` (SURVEY §0 adapter)."""
    z = np.asarray(z)
    log = z.real.astype(dtype)
    sign = np.where(np.cos(z.imag.astype(np.float64)) < 0, -1.0, 1.0).astype(dtype)
    return log, sign


def join_complex(log, sign, dtype=np.complex64):
    """(log_mag, sign) -> canonical complex GOOM: imag 0 or pi."""
    log = np.asarray(log)
    sign = np.asarray(sign)
    ft = np.float32 if dtype == np.complex64 else np.float64
    out = np.empty(log.shape, dtype=dtype)
    out.real = log.astype(ft)
    out.imag = np.where(sign < 0, ft(np.pi), ft(0.0))
    return out


# ---------------------------------------------------------------------------
# goom-core array kernels


def log_sign(values, zero_log=NEG_INF):
    """real -> (log|v|, sign v); zeros -> (zero_log, +1).  core.py:229-239."""
    values = np.asarray(values)
    dt = values.dtype.type
    with np.errstate(divide="ignore"):
        mag = np.log(np.abs(values))
    sgn = np.where(values < 0, dt(-1.0), dt(1.0))
    is_zero = values == 0
    if is_zero.any():
        mag = np.where(is_zero, dt(zero_log), mag)
        sgn = np.where(is_zero, dt(1.0), sgn)
    return mag.astype(values.dtype, copy=False), sgn


def lmme(alog, asign, blog, bsign):
    """Eq. 10-12 log-matmul-exp with max(.,0)-clamped scales.  core.py:242-261.

    Row scales of A (`max_j`, clamped at 0) and column scales of B shift the
    operands so every exponential is <= 1; the real product is taken in the
    operand dtype; the scales are added back as (log|I| + a) + b.
    """
    dt = alog.dtype.type
    row_scale = np.maximum(alog.max(axis=-1, keepdims=True), dt(0.0))
    col_scale = np.maximum(blog.max(axis=-2, keepdims=True), dt(0.0))
    with np.errstate(invalid="ignore"):
        lhs = asign * np.exp(alog - row_scale)
        rhs = bsign * np.exp(blog - col_scale)
    interior = np.matmul(lhs, rhs)
    with np.errstate(divide="ignore"):
        out_log = np.log(np.abs(interior)) + row_scale + col_scale
    out_sign = np.where(interior < 0, dt(-1.0), dt(1.0))
    return out_log, out_sign


def gadd(alog, asign, blog, bsign):
    """Elementwise signed log-sum-exp; both -inf -> (-inf, +1).  core.py:264-275."""
    dt = alog.dtype.type
    top = np.maximum(alog, blog)
    live = top != NEG_INF
    shift = np.where(live, top, dt(0.0))
    with np.errstate(invalid="ignore"):
        total = asign * np.exp(alog - shift) + bsign * np.exp(blog - shift)
    with np.errstate(divide="ignore"):
        out_log = np.where(live, shift + np.log(np.abs(total)), dt(NEG_INF))
    out_sign = np.where(live & (total < 0), dt(-1.0), dt(1.0))
    return out_log, out_sign


def col_log_norms(log):
    """log Euclidean norm of each column (axis -2).  core.py:288-296."""
    dt = log.dtype.type
    top = log.max(axis=-2, keepdims=True)
    live = top != NEG_INF
    shift = np.where(live, top, dt(0.0))
    acc = np.sum(np.exp(2.0 * (log - shift)), axis=-2, keepdims=True)
    with np.errstate(divide="ignore"):
        return np.where(live, shift + 0.5 * np.log(acc), dt(NEG_INF))


def to_real_scaled(log, sign):
    """Eq. 29 export sign*exp(log - c + 2), c = max log (0 if all zero).  core.py:313-323."""
    c = float(log.max()) if log.size else 0.0
    if c == NEG_INF:
        c = 0.0
    dt = log.dtype.type
    return sign * np.exp(log - dt(c) + dt(2.0)), c


def to_real(log, sign):
    """sign * exp(log), overflow -> signed inf.  core.py:213-216."""
    with np.errstate(over="ignore"):
        return sign * np.exp(log)


def identity(d, dtype=np.float64):
    log = np.full((d, d), NEG_INF, dtype=dtype)
    np.fill_diagonal(log, 0.0)
    return log, np.ones((d, d), dtype=dtype)


# ---------------------------------------------------------------------------
# pscan: affine pairs (A, B, flag) stacked along axis 0


@dataclass
class Stack:
    """Stacked scan elements (scan.py:138-170): A (T,d,d), B (T,d,m), flags (T,)."""

    alog: np.ndarray
    asign: np.ndarray
    blog: np.ndarray
    bsign: np.ndarray
    flags: np.ndarray

    def __len__(self):
        return len(self.flags)

    def copy(self):
        return Stack(self.alog.copy(), self.asign.copy(), self.blog.copy(),
                     self.bsign.copy(), self.flags.copy())

    def state(self, i):
        """ScanPair.state (scan.py:45-48): B after a reset, else A."""
        if self.flags[i]:
            return self.blog[i], self.bsign[i]
        return self.alog[i], self.asign[i]


def combine(pAl, pAs, pBl, pBs, cAl, cAs, cBl, cBs):
    """(prev, curr) -> (curr.A (x) prev.A, (curr.A (x) prev.B) (+) curr.B).  scan.py:173-178."""
    oAl, oAs = lmme(cAl, cAs, pAl, pAs)
    tl, ts = lmme(cAl, cAs, pBl, pBs)
    oBl, oBs = gadd(tl, ts, cBl, cBs)
    return oAl, oAs, oBl, oBs


def scan_sequential(st: Stack) -> Stack:
    """Left fold under combine_affine (scan.py:515-526 with scan.py:92-103)."""
    out = st.copy()
    for t in range(1, len(st)):
        (out.alog[t], out.asign[t], out.blog[t], out.bsign[t]) = combine(
            out.alog[t - 1], out.asign[t - 1], out.blog[t - 1], out.bsign[t - 1],
            st.alog[t], st.asign[t], st.blog[t], st.bsign[t])
        out.flags[t] = st.flags[t] or out.flags[t - 1]
    return out


def scan_affine_blocked(st: Stack, block: int) -> Stack:
    """Two-level blocked inclusive scan.  scan.py:181-214.

    Level 1: position i of every block is combined with position i-1 of the
    same block, batched across blocks, for i = 1..b-1.  Level 2: block k is
    combined, left to right, with the (already final) last element of block
    k-1.
    """
    n = len(st)
    b = min(block, n)
    o = st.copy()
    for i in range(1, b):
        cur = np.arange(i, n, b)
        if cur.size == 0:
            break
        prv = cur - 1
        o.alog[cur], o.asign[cur], o.blog[cur], o.bsign[cur] = combine(
            o.alog[prv], o.asign[prv], o.blog[prv], o.bsign[prv],
            o.alog[cur], o.asign[cur], o.blog[cur], o.bsign[cur])
        o.flags[cur] |= o.flags[prv]
    for lo in range(b, n, b):
        sl = slice(lo, min(lo + b, n))
        c = lo - 1
        o.alog[sl], o.asign[sl], o.blog[sl], o.bsign[sl] = combine(
            o.alog[c], o.asign[c], o.blog[c], o.bsign[c],
            o.alog[sl], o.asign[sl], o.blog[sl], o.bsign[sl])
        o.flags[sl] |= o.flags[c]
    return o


def chain_blocked(alog, asign, block):
    """A-slot of `scan_affine_blocked` for an all-zero-bias chain (the bias
    slot stays all -inf: lmme(A, zero) is zero and zero (+) zero is zero)."""
    n = len(alog)
    b = min(block, n)
    L = alog.copy()
    S = asign.copy()
    for i in range(1, b):
        cur = np.arange(i, n, b)
        if cur.size == 0:
            break
        L[cur], S[cur] = lmme(L[cur], S[cur], L[cur - 1], S[cur - 1])
    for lo in range(b, n, b):
        sl = slice(lo, min(lo + b, n))
        L[sl], S[sl] = lmme(L[sl], S[sl], L[lo - 1], S[lo - 1])
    return L, S


# ---------------------------------------------------------------------------
# selective resets


@dataclass
class Policy:
    """ResetPolicy (scan.py:51-89) over raw arrays."""

    select: Callable
    reset: Callable
    check_interval: int = 1
    consume_leaf: bool = True


def is_tested(p, interval):
    """scan.py:221-223: 0-based position p is tested when (p+1) % interval == 0."""
    return (p + 1) % interval == 0


def _unit_columns(log, sign):
    """Shared normalisation of lyapunov.py:211-215 / 259-263 (None on a zero column)."""
    with np.errstate(divide="ignore"):
        top = log.max(axis=0)
        if (top == NEG_INF).any():
            return None
        nu = top + 0.5 * np.log(np.sum(np.exp(2.0 * (log - top)), axis=0))
        return sign * np.exp(log - nu)


def colinearity_select(log, sign, threshold=0.99, volume_floor=1e-9):
    """colinearity_policy.select_raw.  lyapunov.py:255-269."""
    real = _unit_columns(log, sign)
    if real is None:
        return True
    gram = real.T @ real
    iu, ju = np.triu_indices(gram.shape[0], k=1)
    if np.max(np.abs(gram[iu, ju])) > threshold:
        return True
    det_sign, logdet = np.linalg.slogdet(real)
    return bool(det_sign == 0.0 or logdet < math.log(volume_floor))


def cgs2(a):
    """Two-pass Gram-Schmidt, column by column.  lyapunov.py:175-194."""
    n = a.shape[0]
    q = np.array(a, dtype=np.float64)
    tiny = 64.0 * np.finfo(np.float64).eps
    for j in range(n):
        v = q[:, j]
        for _ in range(2):
            for i in range(j):
                v -= (q[:, i] @ v) * q[:, i]
        nv = np.sqrt(v @ v)
        if nv < tiny:
            raise ValueError("rank-deficient state cannot be orthonormalized")
        q[:, j] = v / nv
    return q


def orthonormal_reset(log, sign):
    """lyapunov.py:209-219: log-unit columns, CGS2, back to (log, sign)."""
    real = _unit_columns(log, sign)
    if real is None:
        raise ValueError("cannot orthonormalize a state with an all-zero column")
    q = cgs2(real)
    with np.errstate(divide="ignore"):
        out_log = np.log(np.abs(q))
    return out_log, np.where(q < 0, -1.0, 1.0)


def colinearity_policy(threshold=0.99, check_interval=12, volume_floor=1e-9):
    """lyapunov.py:239-278 (consume_leaf False)."""
    return Policy(
        select=lambda l, s: colinearity_select(l, s, threshold, volume_floor),
        reset=orthonormal_reset,
        check_interval=check_interval,
        consume_leaf=False,
    )


def norm_threshold_policy(threshold, interval=1):
    """The reference's scan-test policy (pkg/tests/test_scan.py:60-75):
    fire when a column's log Euclidean norm exceeds `threshold`; reset to the
    LAPACK (numpy.linalg.qr) Q of the log-unit-norm-scaled state."""

    def select(log, sign):
        return bool(np.max(col_log_norms(log)) > threshold)

    def reset(log, sign):
        nu = col_log_norms(log)
        if (nu == NEG_INF).any():
            raise ValueError("cannot normalize an all-zero column")
        scaled = np.where(log == NEG_INF, log.dtype.type(NEG_INF), log - nu)
        q, _ = np.linalg.qr(sign * np.exp(scaled))
        return log_sign(q.astype(log.dtype))

    return Policy(select=select, reset=reset, check_interval=interval, consume_leaf=True)


def never_policy(interval=1):
    return Policy(select=lambda l, s: False, reset=lambda l, s: (l, s), check_interval=interval)


def selective_sequential(st: Stack, policy: Policy):
    """Reference selective left fold.  scan.py:226-246."""
    n = len(st)
    o = st.copy()
    sites = []
    d = st.alog.shape[-1]
    for t in range(1, n):
        if is_tested(t - 1, policy.check_interval):
            tl, ts = o.state(t - 1)
            if policy.select(tl, ts):
                rl, rs = policy.reset(tl, ts)
                zl = np.full((d, d), NEG_INF, dtype=st.alog.dtype)
                zs = np.ones((d, d), dtype=st.alog.dtype)
                if policy.consume_leaf:
                    o.alog[t], o.asign[t] = zl, zs
                    o.blog[t], o.bsign[t] = rl, rs
                else:
                    (o.alog[t], o.asign[t], o.blog[t], o.bsign[t]) = combine(
                        zl, zs, rl, rs, st.alog[t], st.asign[t], st.blog[t], st.bsign[t])
                o.flags[t] = True
                sites.append(t)
                continue
        (o.alog[t], o.asign[t], o.blog[t], o.bsign[t]) = combine(
            o.alog[t - 1], o.asign[t - 1], o.blog[t - 1], o.bsign[t - 1],
            st.alog[t], st.asign[t], st.blog[t], st.bsign[t])
        o.flags[t] = st.flags[t] or o.flags[t - 1]
    return o, sites


def local_products(alog, asign, s, skip_first):
    """Per-tile inclusive products, batched across tiles.  scan.py:317-339."""
    n = len(alog)
    L = alog.copy()
    S = asign.copy()
    if skip_first:
        eye_l, eye_s = identity(alog.shape[-1], alog.dtype)
        L[::s] = eye_l
        S[::s] = eye_s
    for i in range(1, s):
        cur = np.arange(i, n, s)
        if cur.size == 0:
            break
        L[cur], S[cur] = lmme(L[cur], S[cur], L[cur - 1], S[cur - 1])
    return L, S


def selective_chain_strided(alog, asign, policy: Policy):
    """Tile-total walk + batched materialisation.  scan.py:356-428."""
    n = len(alog)
    s = min(policy.check_interval, n)
    ntiles = (n + s - 1) // s
    d = alog.shape[-1]
    l0, s0 = local_products(alog, asign, s, skip_first=False)
    l1 = s1 = None
    carry_l = np.empty((ntiles, d, d), dtype=alog.dtype)
    carry_s = np.empty((ntiles, d, d), dtype=asign.dtype)
    mode = np.zeros(ntiles, dtype=np.int8)  # 0 none, 1 carry, 2 carry after consuming reset
    sites = []
    cl = cs = None
    consumed = False
    with np.errstate(divide="ignore", invalid="ignore"):
        for k in range(ntiles):
            lo = k * s
            p = min(lo + s, n) - 1
            if cl is None:
                el, es = l0[p], s0[p]
            elif consumed:
                mode[k] = 2
                carry_l[k], carry_s[k] = cl, cs
                if l1 is None:
                    l1, s1 = local_products(alog, asign, s, skip_first=True)
                el, es = (cl, cs) if p == lo else lmme(l1[p], s1[p], cl, cs)
            else:
                mode[k] = 1
                carry_l[k], carry_s[k] = cl, cs
                el, es = lmme(l0[p], s0[p], cl, cs)
            consumed = False
            if p % s == s - 1 and p <= n - 2 and policy.select(el, es):
                rl, rs = policy.reset(el, es)
                sites.append(p + 1)
                cl, cs = np.asarray(rl), np.asarray(rs)
                consumed = policy.consume_leaf
            else:
                cl, cs = el, es
    if mode[0] == 0:
        carry_l[0], carry_s[0] = identity(d, alog.dtype)
    reps = np.full(ntiles, s)
    reps[-1] = n - (ntiles - 1) * s
    ll, ls = l0, s0
    if (mode == 2).any():
        pm = np.repeat(mode, reps)[:, None, None] == 2
        ll = np.where(pm, l1, l0)
        ls = np.where(pm, s1, s0)
    V, Vs = lmme(ll, ls, np.repeat(carry_l, reps, axis=0), np.repeat(carry_s, reps, axis=0))
    if mode[0] == 0:
        first = min(s, n)
        V[:first], Vs[:first] = l0[:first], s0[:first]
    for k in np.flatnonzero(mode == 2):
        V[k * s], Vs[k * s] = carry_l[k], carry_s[k]
    return V, Vs, sites


def selective_chain_walk(alog, asign, policy: Policy, block):
    """Every-position tile walk (check_interval 1).  scan.py:431-484."""
    n = len(alog)
    s = min(block, n)
    V = np.empty_like(alog)
    Vs = np.empty_like(asign)
    l0, s0 = local_products(alog, asign, s, skip_first=False)
    l1 = s1 = None
    sites = []
    carry = None
    consumed = False
    for lo in range(0, n, s):
        hi = min(lo + s, n)
        sl = slice(lo, hi)
        if consumed:
            if l1 is None:
                l1, s1 = local_products(alog, asign, s, skip_first=True)
            V[sl], Vs[sl] = lmme(l1[sl], s1[sl], carry[0], carry[1])
            V[lo], Vs[lo] = carry
        elif carry is None:
            V[sl], Vs[sl] = l0[sl], s0[sl]
        else:
            V[sl], Vs[sl] = lmme(l0[sl], s0[sl], carry[0], carry[1])
        consumed = False
        crossed = False
        p = lo
        while p <= min(hi - 1, n - 2):
            if policy.select(V[p], Vs[p]):
                rl, rs = policy.reset(V[p], Vs[p])
                q = p + 1
                sites.append(q)
                if q >= hi:
                    carry = (np.asarray(rl), np.asarray(rs))
                    consumed = policy.consume_leaf
                    crossed = True
                    break
                if policy.consume_leaf:
                    V[q], Vs[q] = rl, rs
                else:
                    V[q], Vs[q] = lmme(alog[q], asign[q], np.asarray(rl), np.asarray(rs))
                for r in range(q + 1, hi):
                    V[r], Vs[r] = lmme(alog[r], asign[r], V[r - 1], Vs[r - 1])
                p = q
            else:
                p += 1
        if not crossed:
            carry = (V[hi - 1], Vs[hi - 1])
    return V, Vs, sites


def selective_chain(alog, asign, policy: Policy, block):
    """scan.py:342-353 dispatch."""
    if policy.check_interval > 1:
        return selective_chain_strided(alog, asign, policy)
    return selective_chain_walk(alog, asign, policy, block)


def selective_tiled(st: Stack, policy: Policy, block):
    """Pair-level view of the chain fast path.  scan.py:487-504."""
    V, Vs, sites = selective_chain(st.alog, st.asign, policy, block)
    n = len(st)
    out = Stack(V.copy(), Vs.copy(), np.full_like(V, NEG_INF), np.ones_like(Vs),
                np.zeros(n, dtype=bool))
    if sites:
        f = sites[0]
        out.flags[f:] = True
        out.alog[f:] = NEG_INF
        out.asign[f:] = 1.0
        out.blog[f:] = V[f:]
        out.bsign[f:] = Vs[f:]
    return out, sites


def selective_rounds(st: Stack, policy: Policy, block):
    """General-bias selective scan by repeated affine rounds.  scan.py:255-314."""
    n = len(st)
    out = scan_affine_blocked(st, block)
    sites = []
    start = 0
    d = st.alog.shape[-1]
    while True:
        fired = None
        for p in range(start, n - 1):
            if is_tested(p, policy.check_interval) and policy.select(*out.state(p)):
                fired = p
                break
        if fired is None:
            break
        q = fired + 1
        rl, rs = policy.reset(*out.state(fired))
        sites.append(q)
        if policy.consume_leaf:
            out.alog[q] = NEG_INF
            out.asign[q] = 1.0
            out.blog[q], out.bsign[q] = rl, rs
        else:
            zl = np.full_like(out.alog[q], NEG_INF)
            (out.alog[q], out.asign[q], out.blog[q], out.bsign[q]) = combine(
                zl, np.ones_like(zl), rl, rs, st.alog[q], st.asign[q], st.blog[q], st.bsign[q])
        out.flags[q:] = True
        if q == n - 1:
            break
        suffix = Stack(
            np.concatenate([out.alog[q:q + 1], st.alog[q + 1:]]),
            np.concatenate([out.asign[q:q + 1], st.asign[q + 1:]]),
            np.concatenate([out.blog[q:q + 1], st.blog[q + 1:]]),
            np.concatenate([out.bsign[q:q + 1], st.bsign[q + 1:]]),
            out.flags[q:].copy())
        sc = scan_affine_blocked(suffix, block)
        out.alog[q:], out.asign[q:] = sc.alog, sc.asign
        out.blog[q:], out.bsign[q:] = sc.blog, sc.bsign
        start = q
    return out, sites


def scan_selective(st: Stack, policy: Policy, block: Optional[int]):
    """scan.py:550-570 dispatch (None -> sequential reference)."""
    if block is None:
        return selective_sequential(st, policy)
    zero_bias = (not st.flags.any()) and bool(np.all(st.blog == NEG_INF))
    if zero_bias:
        return selective_tiled(st, policy, block)
    return selective_rounds(st, policy, block)


# ---------------------------------------------------------------------------
# Lyapunov stages (b)-(d) and the largest exponent


def qr_factor_batched(ms):
    """Householder QR over a stack, R diagonal made non-negative.  lyapunov.py:79-99.
    Reflector v = x + sign(x0) ||x|| e0 (sign(0) = +), beta = 2 / v.v (0 when v = 0),
    R <- R - beta v (v^T R), Q <- Q - beta (Q v) v^T, then column flips by sign(R_jj)."""
    r = np.array(ms, dtype=np.float64)
    N, n, _ = r.shape
    q = np.broadcast_to(np.eye(n), (N, n, n)).copy()
    for j in range(n):
        x = r[:, j:, j]
        norm_x = np.sqrt(np.einsum("nk,nk->n", x, x))
        v = x.copy()
        v[:, 0] += np.where(x[:, 0] >= 0, norm_x, -norm_x)
        vv = np.einsum("nk,nk->n", v, v)
        beta = np.where(vv > 0, 2.0 / np.where(vv > 0, vv, 1.0), 0.0)
        w = np.einsum("nk,nkm->nm", v, r[:, j:, :])
        r[:, j:, :] -= beta[:, None, None] * v[:, :, None] * w[:, None, :]
        u = np.einsum("nmk,nk->nm", q[:, :, j:], v)
        q[:, :, j:] -= beta[:, None, None] * u[:, :, None] * v[:, None, :]
    flip = np.where(np.diagonal(r, axis1=1, axis2=2) < 0, -1.0, 1.0)
    r *= flip[:, :, None]
    q *= flip[:, None, :]
    return q, r


def spectrum_parallel(mats, dt, colinearity_threshold=0.99, check_interval=12, block=256):
    """Parallel Lyapunov spectrum.  lyapunov.py:311-356: (a) selective colinearity scan of
    [S0 = I, J_0 .. J_{T-2}], (b) log-unit-normalised states -> batched QR bases,
    (c) J_t Q_{t-1}, (d) mean log |diag R| of the batched QR of (c), sorted descending."""
    T, d = mats.shape[0], mats.shape[-1]
    alog = np.empty((T, d, d))
    asign = np.empty((T, d, d))
    alog[0], asign[0] = log_sign(np.eye(d))
    if T > 1:
        alog[1:], asign[1:] = log_sign(mats[:T - 1])
    pol = colinearity_policy(colinearity_threshold, check_interval)
    V, Vs, sites = selective_chain(alog, asign, pol, block)
    nu = col_log_norms(V)
    if (nu == NEG_INF).any():
        raise ValueError("a scan state lost a whole column; cannot orthonormalize")
    bases = qr_factor_batched(Vs * np.exp(V - nu))[0]
    _, r = qr_factor_batched(np.matmul(mats, bases))
    diag = np.abs(np.diagonal(r, axis1=1, axis2=2))
    if np.any(diag == 0.0):
        raise ValueError("degenerate Jacobian chain")
    return np.sort(np.mean(np.log(diag), axis=0) / dt)[::-1], len(sites)


def lle_parallel(mats, u0, dt, block=256):
    """Largest exponent from one affine scan with a d x 1 bias.  lyapunov.py:403-429."""
    T, d = mats.shape[0], mats.shape[-1]
    alog = np.empty((T + 1, d, d))
    asign = np.empty((T + 1, d, d))
    alog[0] = NEG_INF
    asign[0] = 1.0
    alog[1:], asign[1:] = log_sign(mats)
    blog = np.full((T + 1, d, 1), NEG_INF)
    bsign = np.ones((T + 1, d, 1))
    blog[0], bsign[0] = log_sign(np.asarray(u0, dtype=np.float64).reshape(d, 1))
    out = scan_affine_blocked(Stack(alog, asign, blog, bsign, np.zeros(T + 1, bool)), block)
    final = out.blog[-1].ravel()
    m = final.max()
    lse = 2.0 * m + math.log(np.sum(np.exp(2.0 * (final - m))))
    return lse / (2.0 * dt * T)


def ssm_forward_parallel(A, B, C, D, x0, u, block=256):
    """Non-diagonal SSM as an affine scan (ssm.py:110-137): leaves (A, B u_t) after the
    leading (0, x0); states = the prefixes' bias columns; then _finish (ssm.py:84-98):
    c_t = max log x_t (0 for an all-zero state), y = (s e^{log - c + 2}) C^T + u D^T."""
    T, d = u.shape
    a_log, a_sign = log_sign(np.asarray(A, dtype=np.float64))
    b_log, b_sign = log_sign(np.asarray(B, dtype=np.float64))
    u_log, u_sign = log_sign(u.reshape(T, d, 1))
    bu_log, bu_sign = lmme(b_log, b_sign, u_log, u_sign)
    alog = np.empty((T + 1, d, d))
    asign = np.ones((T + 1, d, d))
    alog[0] = NEG_INF
    alog[1:] = a_log
    asign[1:] = a_sign
    blog = np.empty((T + 1, d, 1))
    bsign = np.empty((T + 1, d, 1))
    blog[0], bsign[0] = log_sign(np.asarray(x0, dtype=np.float64).reshape(d, 1))
    blog[1:] = bu_log
    bsign[1:] = bu_sign
    out = scan_affine_blocked(Stack(alog, asign, blog, bsign, np.zeros(T + 1, bool)), block)
    sl, ss = out.blog[1:, :, 0], out.bsign[1:, :, 0]
    c = sl.max(axis=1)
    c = np.where(c == NEG_INF, 0.0, c)
    y = (ss * np.exp(sl - c[:, None] + 2.0)) @ np.asarray(C).T + u @ np.asarray(D).T
    return sl, ss, c, y


def _signed_lse(logs, signs, axis):
    """log-domain signed sum along axis: (log|sum|, sign); an all -inf / cancelled sum -> (-inf, +1)."""
    m = np.max(logs, axis=axis, keepdims=True)
    mf = np.where(np.isfinite(m), m, 0.0)
    with np.errstate(under="ignore"):
        tot = np.sum(signs * np.exp(logs - mf), axis=axis, keepdims=True)
    with np.errstate(divide="ignore"):
        out = np.where(tot == 0.0, NEG_INF, np.log(np.abs(tot)) + mf)
    return np.squeeze(out, axis), np.squeeze(np.where(tot < 0, -1.0, 1.0), axis)


def _real_of_log(log, sign):
    with np.errstate(over="ignore", under="ignore"):
        return sign * np.exp(log)


def ssm_backward(A, B, C, D, x0, u, sl, ss, c, gy):
    """Gradients of sum(gy * y) for ssm_forward_parallel's outputs (sl, ss, c). The
    reference has no autodiff; this restates the adjoint of its
    forward (ssm.py:84-98, 99-137) in the log domain, one reverse step at a time with this
    module's lmme / gadd, and is pinned against torch float64 autograd on chains without
    overflow (tests/golden/make_golden_ssm_bwd.py):
      z_t = s_t e^{l_t - c_t + 2}; gz_t = C^T gy_t; i* = first argmax_i l_t,i;
      h_t = e^2 gz_t - e_{i*} s_{t,i*} (gz_t . z_t)   (no c-term for an all-zero state);
      lam_{T-1} = e^{-c} h_{T-1};  lam_t = A^T (x) lam_{t+1} (+) e^{-c_t} h_t (run on
      lam e^{K}, K = max_t c_t);
      dA = sum_t lam_t x_{t-1}^T (x_{-1} = x0), dB = sum_t lam_t u_t^T (signed log-sum-exp
      over t, then exp); du_t = B^T lam_t + D^T gy_t; dx0 = A^T lam_0;
      dC = sum gy_t z_t^T; dD = sum gy_t u_t^T.  Returns a dict of float64 arrays."""
    A, B, C, D = (np.asarray(m, dtype=np.float64) for m in (A, B, C, D))
    x0 = np.asarray(x0, dtype=np.float64)
    u = np.asarray(u, dtype=np.float64)
    gy = np.asarray(gy, dtype=np.float64)
    T, d = u.shape
    z = ss * np.exp(sl - c[:, None] + 2.0)
    gz = gy @ C
    h = math.exp(2.0) * gz
    live = np.max(sl, axis=1) != NEG_INF
    istar = np.argmax(sl, axis=1)
    dot = np.sum(gz * z, axis=1)
    rows = np.arange(T)
    h[rows, istar] -= np.where(live, ss[rows, istar] * dot, 0.0)
    hl, hs = log_sign(h)
    # the recurrence runs on lam e^{K}, K = max_t c_t: this module's lmme clamps its scales
    # at 0 like the reference, so an adjoint below e^{-745} would otherwise vanish
    K = float(np.max(c))
    gl = hl + (K - c)[:, None]
    at_l, at_s = log_sign(A.T.copy())
    lam_l = np.empty((T, d))
    lam_s = np.empty((T, d))
    cur_l, cur_s = gl[T - 1].reshape(d, 1), hs[T - 1].reshape(d, 1)
    lam_l[T - 1], lam_s[T - 1] = cur_l[:, 0], cur_s[:, 0]
    for t in range(T - 2, -1, -1):
        pl, ps = lmme(at_l, at_s, cur_l, cur_s)
        cur_l, cur_s = gadd(pl, ps, gl[t].reshape(d, 1), hs[t].reshape(d, 1))
        lam_l[t], lam_s[t] = cur_l[:, 0], cur_s[:, 0]
    lam_l = lam_l - K
    x0l, x0s = log_sign(x0)
    prev_l = np.concatenate([x0l[None], sl[:-1]])
    prev_s = np.concatenate([x0s[None], ss[:-1]])
    ul, us = log_sign(u)
    dA = _real_of_log(*_signed_lse(lam_l[:, :, None] + prev_l[:, None, :],
                                   lam_s[:, :, None] * prev_s[:, None, :], 0))
    dB = _real_of_log(*_signed_lse(lam_l[:, :, None] + ul[:, None, :],
                                   lam_s[:, :, None] * us[:, None, :], 0))
    bt_l, bt_s = log_sign(B.T.copy())
    bl, bs = lmme(np.broadcast_to(bt_l, (T, d, d)), np.broadcast_to(bt_s, (T, d, d)),
                  lam_l[:, :, None], lam_s[:, :, None])
    du = _real_of_log(bl[:, :, 0], bs[:, :, 0]) + gy @ D
    xl, xs = lmme(at_l, at_s, lam_l[0].reshape(d, 1), lam_s[0].reshape(d, 1))
    dx0 = _real_of_log(xl[:, 0], xs[:, 0])
    return {"A": dA, "B": dB, "C": gy.T @ z, "D": gy.T @ u, "x0": dx0, "u": du,
            "lam_log": lam_l, "lam_sign": lam_s}


# ---------------------------------------------------------------------------
# parity metrics


def rel_log_diff(x, y):
    """max |x-y| / max(1,|y|), -inf == -inf.  pkg/tests/test_scan.py:209-213."""
    x = np.asarray(x, dtype=np.float64)
    y = np.asarray(y, dtype=np.float64)
    denom = np.maximum(1.0, np.abs(y))
    both = (x == NEG_INF) & (y == NEG_INF)
    with np.errstate(invalid="ignore"):
        diff = np.where(both, 0.0, np.abs(x - y) / denom)
    diff = np.where(np.isnan(diff), np.inf, diff)
    return float(np.max(diff)) if diff.size else 0.0


def cancellation(alog, asign, blog, bsign):
    """kappa = |sum a b| / sum |a||b| per LMME output entry, in the log domain
    (SURVEY §8c): LMME(A,B) - LMME(|A|,|B|)."""
    sl, _ = lmme(alog, asign, blog, bsign)
    al, _ = lmme(alog, np.ones_like(asign), blog, np.ones_like(bsign))
    with np.errstate(invalid="ignore"):
        k = np.exp(sl - al)
    return np.where(np.isnan(k), 0.0, k)


def random_stack(rng, T, d, m=None, biases=False, dtype=np.float64):
    """Leaves A_t ~ N(0,1) (and optional B_t ~ N(0,1)) as a Stack."""
    m = d if m is None else m
    a = rng.standard_normal((T, d, d)).astype(dtype)
    al, as_ = log_sign(a)
    if biases:
        bl, bs = log_sign(rng.standard_normal((T, d, m)).astype(dtype))
    else:
        bl = np.full((T, d, m), NEG_INF, dtype=dtype)
        bs = np.ones((T, d, m), dtype=dtype)
    return Stack(al, as_, bl, bs, np.zeros(T, dtype=bool))
