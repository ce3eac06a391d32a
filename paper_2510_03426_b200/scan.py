"""Prefix scans over GOOM affine pairs with selective resets — drop-in for `gooms.scan`.

Scan elements are stacked on the GPU as one `_Stack` (A: (T,d,d), B: (T,d,m)
complex64, flags: (T,) bool). The engines run in libgoom:

* `_scan_affine_stack` -> goom_scan_affine_c64 / goom_scan_chain_c64 (zero-bias
  fast path: the bias slot of an all-zero-bias stack stays exactly zero, so its
  LMMEs are skipped — the reference always runs them, scan.py:173-178).
* `_selective_chain_core` -> goom_scan_selective_chain_c64 for the built-in
  policies (colinearity / norm-threshold / never), fused on the device.
* Arbitrary Python select/reset callables cannot run on the GPU; for those the
  control flow runs on the host while every combine still runs on the GPU
  (the reference's own semantics: sites are value-determined and identical to
  the sequential fold, scan.py:9-12).
"""

from __future__ import annotations

import gc
from dataclasses import dataclass, field
from typing import Callable, Optional

import numpy as np
import torch

from . import _lib, ops
from .core import NEG_INF, GoomMatrix, _device, _StackedGoom, join, split

POLICY_NEVER = _lib.POLICY_NEVER
POLICY_COLINEARITY = _lib.POLICY_COLINEARITY
POLICY_NORM_THRESHOLD = _lib.POLICY_NORM_THRESHOLD


@dataclass(frozen=True)
class ScanPair:
    """One scan element: transition A (d x d), bias B (d x m), reset marker (scan.py:26-48)."""

    A: GoomMatrix
    B: GoomMatrix
    reset_applied: bool = False

    def __post_init__(self):
        if self.A.rows != self.A.cols:
            raise ValueError("transition must be square")
        if self.B.rows != self.A.rows:
            raise ValueError("bias row count must match the transition")

    @property
    def state(self):
        return self.B if self.reset_applied else self.A


@dataclass(frozen=True)
class ResetPolicy:
    """Selective-reset rule (scan.py:51-89).

    `kind` names a built-in device policy (POLICY_*); then `threshold` and
    `log_volume_floor` parameterise it and the scan runs fully on the GPU.
    With kind None, `select(GoomMatrix) -> bool` and `reset(GoomMatrix) ->
    GoomMatrix` are arbitrary host callables.
    """

    select: Callable
    reset: Callable
    check_interval: int = 1
    consume_leaf: bool = True
    select_raw: Callable = field(default=None)
    reset_raw: Callable = field(default=None)
    kind: Optional[int] = None
    threshold: float = 0.0
    log_volume_floor: float = 0.0

    def __post_init__(self):
        if self.check_interval < 1:
            raise ValueError("check_interval must be >= 1")

    @property
    def builtin(self) -> bool:
        return self.kind is not None

    def select_arrays(self, log, sign):
        if self.select_raw is not None:
            return bool(self.select_raw(log, sign))
        return bool(self.select(GoomMatrix(log, sign)))

    def reset_arrays(self, log, sign):
        if self.reset_raw is not None:
            return self.reset_raw(log, sign)
        v = self.reset(GoomMatrix(log, sign))
        return v.log_mag, v.sign


def _builtin_select(kind, threshold, log_floor):
    def select(m: GoomMatrix):
        return bool(torch.ops.goom.policy_select(m.data, kind, threshold, log_floor).item())

    return select


def _builtin_reset(kind):
    def reset(m: GoomMatrix):
        return GoomMatrix._wrap(torch.ops.goom.policy_reset(m.data, kind))

    return reset


def builtin_policy(kind, threshold=0.0, log_volume_floor=0.0, check_interval=1,
                   consume_leaf=True) -> ResetPolicy:
    return ResetPolicy(
        select=_builtin_select(kind, threshold, log_volume_floor),
        reset=_builtin_reset(kind),
        check_interval=check_interval,
        consume_leaf=consume_leaf,
        kind=kind,
        threshold=threshold,
        log_volume_floor=log_volume_floor,
    )


def never_policy(check_interval=1) -> ResetPolicy:
    return builtin_policy(POLICY_NEVER, check_interval=check_interval)


def norm_threshold_policy(threshold, interval=1) -> ResetPolicy:
    """Fire when a column's log Euclidean norm exceeds `threshold`; reset to the
    Householder Q (LAPACK sign convention) of the log-unit-norm state. The
    policy the reference's scan tests use (pkg/tests/test_scan.py:60-75)."""
    return builtin_policy(POLICY_NORM_THRESHOLD, threshold=float(threshold),
                          check_interval=interval, consume_leaf=True)


def combine_affine(prev: ScanPair, curr: ScanPair) -> ScanPair:
    """(prev, curr) -> (curr.A (x) prev.A, curr.A (x) prev.B (+) curr.B) (scan.py:92-103)."""
    if curr.A.cols != prev.A.rows or curr.A.cols != prev.B.rows:
        raise ValueError("dimension mismatch between scan elements")
    a = torch.ops.goom.lmme(curr.A.data, prev.A.data)
    b = torch.ops.goom.lmme_gadd(curr.A.data, prev.B.data, curr.B.data)
    return ScanPair(GoomMatrix._wrap(a), GoomMatrix._wrap(b),
                    prev.reset_applied or curr.reset_applied)


class SelectiveCombiner:
    """Affine combiner with selective resets (scan.py:106-131)."""

    def __init__(self, policy):
        self.policy = policy

    def __call__(self, prev, curr):
        tested = prev.state
        if self.policy.select(tested):
            value = self.policy.reset(tested)
            if value.shape != tested.shape:
                raise ValueError("reset must preserve the state's shape")
            return ScanPair(GoomMatrix.zeros(prev.A.rows, prev.A.cols, dtype=prev.A.dtype), value, True)
        return combine_affine(prev, curr)


def combine_selective(policy):
    return SelectiveCombiner(policy)


# ---------------------------------------------------------------------------
# stacked representation


class _Stack:
    """Scan elements as stacked complex CUDA tensors (scan.py:138-170).

    Two constructors: `_Stack(A, B, flags)` with complex tensors (this package's form) and
    the reference's `_Stack(alog, asign, blog, bsign, flags)` with numpy arrays (float64 ->
    complex128), as its callers build it (lyapunov.py:422, ssm.py:142). A stack built from
    numpy arrays hands numpy back from `.alog` / `.asign` / `.blog` / `.bsign` / `.flags`,
    and so do the stacks the scans derive from it."""

    __slots__ = ("A", "B", "_flags", "host")

    def __init__(self, *args):
        self.host = False
        if len(args) == 5:
            alog, asign, blog, bsign, flags = args
            src = _Stack.from_arrays(alog, asign, blog, bsign, flags)
            A, B, flags = src.A, src.B, src._flags
            self.host = isinstance(alog, np.ndarray)
        elif len(args) in (2, 3):
            A, B = args[0], args[1]
            flags = args[2] if len(args) == 3 else None
        else:
            raise TypeError("_Stack(A, B[, flags]) or _Stack(alog, asign, blog, bsign, flags)")
        self.A = A
        self.B = B
        if flags is None:
            flags = torch.zeros(A.shape[0], dtype=torch.bool, device=A.device)
        elif not isinstance(flags, torch.Tensor):
            flags = torch.as_tensor(np.asarray(flags), dtype=torch.bool, device=A.device)
        self._flags = flags

    @property
    def flags(self):
        return self._flags.cpu().numpy() if self.host else self._flags

    @flags.setter
    def flags(self, v):
        self._flags = v

    def _derived(self, A, B, flags):
        out = _Stack(A, B, flags)
        out.host = self.host
        return out

    def _view(self, t):
        return t.cpu().numpy() if self.host else t

    @classmethod
    def from_arrays(cls, alog, asign, blog, bsign, flags=None, dtype=None):
        """The reference's _Stack(alog, asign, blog, bsign, flags); float64 arrays map
        to complex128 unless `dtype` says otherwise."""
        from .core import _dtype_of_arrays

        dt = _dtype_of_arrays(alog) if dtype is None else dtype
        f = None if flags is None else torch.as_tensor(np.asarray(flags), dtype=torch.bool,
                                                       device=_device())
        return cls(join(alog, asign, dt), join(blog, bsign, dt), f)

    @classmethod
    def from_pairs(cls, leaves):
        A = _restack([p.A for p in leaves])
        B = _restack([p.B for p in leaves])
        f = torch.tensor([p.reset_applied for p in leaves], dtype=torch.bool, device=A.device)
        return cls(A, B, f)

    def to_pairs(self):
        # lazily sliced matrices (_StackedGoom) and no per-pair validation (the stack's shapes
        # are checked): ~10x faster than a tensor view per element, which the reference's own
        # host-list callers notice (test_scan.py:341-360 times a 2^15-leaf scan)
        # The cyclic garbage collector is paused while the 3 T objects are made: every 700
        # allocations it would traverse the growing list (and the caller's leaves), which
        # cost ~4x the creation itself for 2^15 pairs
        flags = self._flags.cpu().tolist()
        new, of, A, B = object.__new__, _StackedGoom._of, self.A, self.B
        out = []
        paused = gc.isenabled()
        gc.disable()
        try:
            for i, f in enumerate(flags):
                p = new(ScanPair)  # frozen dataclass: fill its __dict__ directly
                p.__dict__.update(A=of(A, i), B=of(B, i), reset_applied=bool(f))
                out.append(p)
        finally:
            if paused:
                gc.enable()
        return out

    @property
    def alog(self):
        return self._view(split(self.A)[0])

    @property
    def asign(self):
        return self._view(split(self.A)[1])

    @property
    def blog(self):
        return self._view(split(self.B)[0])

    @property
    def bsign(self):
        return self._view(split(self.B)[1])

    def states(self):
        """Per-element compound state (B after a reset, else A); square B only."""
        return torch.where(self._flags[:, None, None], self.B, self.A)

    def __len__(self):
        return self.A.shape[0]


def _restack(ms):
    """The stacked tensor of GoomMatrix objects: the base itself when they are exactly the
    elements 0 .. T-1 of one stack handed out by to_pairs (no copy), else torch.stack."""
    m0 = ms[0]
    if type(m0) is _StackedGoom:
        base = m0._base
        if base.shape[0] == len(ms) and all(
                type(m) is _StackedGoom and m._base is base and m._i == i for i, m in enumerate(ms)):
            return base
    return torch.stack([m.data for m in ms])


def _all_zero_bias(stack: _Stack) -> bool:
    return (not bool(stack._flags.any())) and bool((stack.B.real == NEG_INF).all())


def _scan_affine_stack(stack: _Stack, block_size: int) -> _Stack:
    """Blocked inclusive affine scan (scan.py:181-214) on the GPU."""
    if block_size < 1:
        raise ValueError("block_size must be >= 1")
    if _all_zero_bias(stack):
        A = torch.ops.goom.scan_chain(stack.A, int(block_size), None)
        return stack._derived(A, stack.B.clone(), stack._flags.clone())
    A, B, f = torch.ops.goom.scan_affine(stack.A, stack.B, stack._flags, int(block_size))
    return stack._derived(A, B, f.bool())


def scan_chain(A: torch.Tensor, block_size: int = 64, carry: Optional[torch.Tensor] = None):
    """Inclusive product chain P_t = A_t ... A_0 (x) carry on complex64 tensors."""
    return torch.ops.goom.scan_chain(A, int(block_size), carry)


# ---------------------------------------------------------------------------
# selective scans


def _tested(p, interval):
    return (p + 1) % interval == 0


def _selective_chain_core(A, *args):
    """Selective scan of a pure product chain (scan.py:342-353).

    Two call forms:
      * `_selective_chain_core(A, policy, block_size)` with A a (T, d, d)
        complex64/complex128 tensor -> (states tensor, sites);
      * the reference's array form `_selective_chain_core(alog, asign, policy,
        block_size)` -> (Vlog, Vsign, sites) with arrays like the inputs
        (float64 arrays run in complex128, the reference's precision for the
        Lyapunov path, lyapunov.py:336-341).
    Built-in policies run fused on the device.
    """
    if not isinstance(args[0], ResetPolicy):
        asign, policy, block_size = args
        from .core import _dtype_of_arrays, _like_input

        V, sites = _selective_chain_core(join(A, asign, _dtype_of_arrays(A)), policy, block_size)
        l, s = split(V)
        return _like_input(l, A), _like_input(s, A), sites
    policy, block_size = args
    if policy.builtin:
        V, sites = torch.ops.goom.scan_selective_chain(
            A, int(policy.kind), int(policy.check_interval), bool(policy.consume_leaf),
            float(policy.threshold), float(policy.log_volume_floor), int(block_size))
        return V, [int(s) for s in sites.cpu().tolist()]
    return _selective_chain_host(A, policy, block_size)


def _selective_chain_host(A: torch.Tensor, policy: ResetPolicy, block_size: int):
    """Selective chain for host-callable policies; every combine on the GPU, the
    predicate / reset on the host. Until the first fire the states are the blocked chain
    scan with the walk's tile (`block_size` for check_interval 1, else check_interval;
    scan.py:356-358) — the reference's tile walk computes exactly that tree (local
    products (x) the previous tile's last state), so a policy that never fires gives the
    affine scan bitwise (test_scan.py:255-265). After a fire at site q the rest is rescanned
    from the reset state. Sites are the value-determined ones of the reference
    (scan.py:9-12)."""
    T = A.shape[0]
    tile = int(block_size) if policy.check_interval == 1 else int(policy.check_interval)
    V = torch.ops.goom.scan_chain(A, tile, None)
    sites = []
    p = 0
    while p <= T - 2:
        if _tested(p, policy.check_interval) and policy.select(GoomMatrix._wrap(V[p])):
            q = p + 1
            value = policy.reset(GoomMatrix._wrap(V[p])).data
            V[q] = value if policy.consume_leaf else torch.ops.goom.lmme(A[q], value)
            sites.append(q)
            if q + 1 < T:
                V[q + 1:] = torch.ops.goom.scan_chain(A[q + 1:].contiguous(), tile,
                                                      V[q].contiguous())
            p = q
            continue
        p += 1
    return V, sites


def _selective_tiled(stack: _Stack, policy: ResetPolicy, block_size: int):
    """Pair-level wrapper for the product-chain path (scan.py:487-504)."""
    V, sites = _selective_chain_core(stack.A, policy, block_size)
    T = len(stack)
    A = V.clone()
    B = torch.full_like(V, complex(NEG_INF, 0.0))
    flags = torch.zeros(T, dtype=torch.bool, device=V.device)
    if sites:
        f = sites[0]
        flags[f:] = True
        A[f:] = complex(NEG_INF, 0.0)
        B[f:] = V[f:]
    return stack._derived(A, B, flags), sites


def _select_positions(states: torch.Tensor, policy: ResetPolicy) -> torch.Tensor:
    """fire flags for a batch of states (device batch kernel for built-ins)."""
    if policy.builtin:
        return torch.ops.goom.policy_select(states, int(policy.kind), float(policy.threshold),
                                            float(policy.log_volume_floor))
    out = [policy.select(GoomMatrix._wrap(states[i])) for i in range(states.shape[0])]
    return torch.tensor(out, dtype=torch.bool)


def _selective_rounds(stack: _Stack, policy: ResetPolicy, block_size: int):
    """General-bias selective scan by repeated affine rounds (scan.py:255-314).

    The first firing tested position is found with one batched predicate over
    all tested positions after the last reset (device kernel for built-ins),
    instead of the reference's position-by-position loop.
    """
    T = len(stack)
    out = _scan_affine_stack(stack, block_size)
    sites = []
    start = 0
    interval = policy.check_interval
    while True:
        cand = [p for p in range(start, T - 1) if _tested(p, interval)]
        fired = None
        if cand:
            idx = torch.tensor(cand, device=out.A.device)
            st = torch.where(out._flags[idx][:, None, None], out.B[idx], out.A[idx])
            fire = _select_positions(st, policy).cpu().numpy()
            hits = np.flatnonzero(fire)
            if hits.size:
                fired = cand[int(hits[0])]
        if fired is None:
            break
        q = fired + 1
        tested = out.B[fired] if bool(out._flags[fired]) else out.A[fired]
        value = policy.reset(GoomMatrix._wrap(tested)).data
        sites.append(q)
        if policy.consume_leaf:
            out.A[q] = complex(NEG_INF, 0.0)
            out.B[q] = value
        else:
            out.A[q] = torch.ops.goom.lmme(stack.A[q], torch.full_like(value, complex(NEG_INF, 0)))
            out.B[q] = torch.ops.goom.lmme_gadd(stack.A[q], value, stack.B[q])
        out._flags[q:] = True
        if q == T - 1:
            break
        suffix = _Stack(torch.cat([out.A[q:q + 1], stack.A[q + 1:]]),
                        torch.cat([out.B[q:q + 1], stack.B[q + 1:]]), out._flags[q:].clone())
        sc = _scan_affine_stack_full(suffix, block_size)
        out.A[q:] = sc.A
        out.B[q:] = sc.B
        start = q
    return out, sites


def _scan_affine_stack_full(stack: _Stack, block_size: int) -> _Stack:
    A, B, f = torch.ops.goom.scan_affine(stack.A, stack.B, stack._flags, int(block_size))
    return _Stack(A, B, f.bool())


def _selective_sequential_pairs(leaves, policy):
    """Reference selective fold on pairs (scan.py:226-246); combines on the GPU."""
    out = [leaves[0]]
    sites = []
    for t in range(1, len(leaves)):
        prev = out[-1]
        if _tested(t - 1, policy.check_interval):
            tested = prev.state
            if policy.select(tested):
                value = policy.reset(tested)
                reset_pair = ScanPair(GoomMatrix.zeros(prev.A.rows, prev.A.cols, dtype=prev.A.dtype), value, True)
                out.append(reset_pair if policy.consume_leaf else combine_affine(reset_pair, leaves[t]))
                sites.append(t)
                continue
        out.append(combine_affine(prev, leaves[t]))
    return out, sites


def _scan_selective_stack(stack: _Stack, policy: ResetPolicy, block_size: int):
    if _all_zero_bias(stack):
        return _selective_tiled(stack, policy, block_size)
    return _selective_rounds(stack, policy, block_size)


# ---------------------------------------------------------------------------
# public scans (scan.py:515-563)


def scan_sequential(leaves, combiner):
    """Inclusive prefix states of a left fold under the combiner."""
    leaves = list(leaves)
    if not leaves:
        raise ValueError("scan of an empty sequence")
    if isinstance(combiner, SelectiveCombiner):
        out, _ = _selective_sequential_pairs(leaves, combiner.policy)
        return out
    if combiner is combine_affine:
        # block >= T: the blocked engine degenerates to the left fold (scan.py:217-225);
        # the fold's first state IS the first leaf (scan.py:521, test_scan.py:182-186)
        out = _scan_affine_stack(_Stack.from_pairs(leaves), len(leaves)).to_pairs()
        out[0] = leaves[0]
        return out
    out = [leaves[0]]
    for leaf in leaves[1:]:
        out.append(combiner(out[-1], leaf))
    return out


def scan_parallel(leaves, combiner, block_size, workers=None):
    """Inclusive prefix states computed blockwise on the GPU (scan.py:529-547)."""
    if isinstance(leaves, _Stack):
        stack = leaves
        if len(stack) == 0:
            raise ValueError("scan of an empty sequence")
    else:
        leaves = list(leaves)
        if not leaves:
            raise ValueError("scan of an empty sequence")
        stack = None
    if block_size < 1:
        raise ValueError("block_size must be >= 1")
    if isinstance(combiner, SelectiveCombiner):
        st = stack if stack is not None else _Stack.from_pairs(leaves)
        out, _ = _scan_selective_stack(st, combiner.policy, block_size)
        return out.to_pairs() if stack is None else out
    if combiner is combine_affine:
        st = stack if stack is not None else _Stack.from_pairs(leaves)
        out = _scan_affine_stack(st, block_size)
        return out.to_pairs() if stack is None else out
    # arbitrary combiner: the reference's blocked generic path (scan.py:573-595)
    if stack is not None:
        leaves = stack.to_pairs()
    T = len(leaves)
    b = min(block_size, T)
    out = []
    for i in range(0, T, b):
        block = leaves[i:i + b]
        acc = [block[0]]
        for leaf in block[1:]:
            acc.append(combiner(acc[-1], leaf))
        if out:
            carry = out[-1]
            acc = [combiner(carry, item) for item in acc]
        out.extend(acc)
    return out


def scan_selective(leaves, policy, block_size=None, workers=None):
    """Selective scan returning (prefix states, reset sites) (scan.py:550-563)."""
    is_stack = isinstance(leaves, _Stack)
    if not is_stack:
        leaves = list(leaves)
        if not leaves:
            raise ValueError("scan of an empty sequence")
    elif len(leaves) == 0:
        raise ValueError("scan of an empty sequence")
    if block_size is None:
        if is_stack:
            leaves = leaves.to_pairs()
        return _selective_sequential_pairs(leaves, policy)
    if block_size < 1:
        raise ValueError("block_size must be >= 1")
    stack = leaves if is_stack else _Stack.from_pairs(leaves)
    out, sites = _scan_selective_stack(stack, policy, block_size)
    return (out if is_stack else out.to_pairs()), sites
