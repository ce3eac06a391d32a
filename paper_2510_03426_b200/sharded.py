"""Time-sharded LMME chain scan over the GPUs of one node.

Rank g owns leaves [g*T/G, (g+1)*T/G). The only exchange is one all-gather of
the G chunk totals (d x d GOOMs, 2 MiB each at d = 512):

  1. local total  tot_g = A_{end-1} ... A_{start}   (pairwise tree of batched LMMEs)
  2. all-gather   tot_0 .. tot_{G-1}                (NCCL over NVLink; gloo in CPU tests)
  3. carry        C_g = tot_{g-1} ... tot_0         (products accumulate on the LEFT,
                                                     so the carry multiplies on the right)
  4. local scan   P_t = (A_t ... A_start) (x) C_g   (the chain engine's carry-in)

Results are deterministic for a fixed (G, window, block) but not bitwise equal
across G (different trees). The orchestration takes the LMME / scan / total
functions as arguments so the same code runs in the gloo CPU tests with the
numpy oracle standing in for the GPU.
"""

from __future__ import annotations

from typing import Callable, Optional, Tuple

import torch
import torch.distributed as dist


def shard_range(T: int, rank: int, world: int) -> Tuple[int, int]:
    """(first leaf, count) of `rank`'s contiguous shard; earlier ranks take the remainder."""
    base, rem = divmod(T, world)
    start = rank * base + min(rank, rem)
    return start, base + (1 if rank < rem else 0)


def fold_carry(totals, rank: int, lmme: Callable) -> Optional[torch.Tensor]:
    """C_rank = tot_{rank-1} (x) ... (x) tot_0 (None for rank 0): later chunks on the left."""
    carry = None
    for r in range(rank):
        carry = totals[r] if carry is None else lmme(totals[r], carry)
    return carry


def exclusive_carry(local_total: torch.Tensor, lmme: Callable, group=None) -> Optional[torch.Tensor]:
    """All-gather the chunk totals and fold the ones before this rank (None on rank 0)."""
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    real = torch.view_as_real(local_total.contiguous())
    gathered = [torch.empty_like(real) for _ in range(world)]
    dist.all_gather(gathered, real, group=group)
    return fold_carry([torch.view_as_complex(g) for g in gathered], rank, lmme)


def shard_total(n: int, d: int, seed: int, t0: int, window: int, block: int) -> torch.Tensor:
    """A_{t0+n-1} ... A_{t0} of this rank's shard, window by window (complex64 d x d).

    d % 256 == 0: the tile-scaled engine's phases 1 + 2 only (ops.chain_ts with no prefix
    output: its carry-out is the window total, phase 3 is skipped); otherwise a pairwise
    tree of batched complex64 LMMEs (harness.chain_total)."""
    from . import ops
    from .harness import chain_total, random_chain

    dev = torch.device("cuda", torch.cuda.current_device())
    total = None
    for w0 in range(0, n, window):
        m = min(window, n - w0)
        if ops.ts_eligible(d):
            _, _, c = ops.chain_ts(ops.ts_random_normal(m, d, seed, t0 + w0, dev), block, None,
                                   out=False, digests=False, carry_out=True)
            wt = ops.ts_to_goom(c)[0]
        else:
            wt = chain_total(random_chain(m, d, seed, t0 + w0))
        total = wt if total is None else torch.ops.goom.lmme(wt[None], total[None])[0]
    return total


def run_shard_resident(n: int, d: int, seed: int, t0: int, window: int, block: int,
                       exchange: Callable, max_resident: Optional[int] = None):
    """This rank's shard with its local products kept on the device (d % 256 == 0).

    Pass 1 runs the carry-independent phases 1-2 of every window (ops.chain_ts_local) and
    folds the window totals into the shard total, keeping the first `max_resident` windows'
    local products (default: as many as fit in free device memory); `exchange(total)`
    (all-gather + fold, or a test double) returns the shard's exclusive carry; pass 2 runs
    only phase 3 for the resident windows (ops.chain_ts_finish) and the whole window for the
    others. A fully resident rank does ~2 n products (the single-GPU work); one that keeps
    nothing does ~3 n (the totals recomputed, as shard_total + run_chain)."""
    from . import ops
    from .harness import ChainRun

    dev = torch.device("cuda", torch.cuda.current_device())
    if max_resident is None:
        per = min(window, n) * d * d * 4 * 1.08
        max_resident = max(0, int((0.92 * _free_bytes() - per) // per))
    wins, total = [], None
    for w0 in range(0, n, window):
        m = min(window, n - w0)
        leaves = ops.ts_random_normal(m, d, seed, t0 + w0, dev)
        win, wt = ops.chain_ts_local(leaves, block)
        del leaves
        keep = sum(1 for x in wins if x[2] is not None) < max_resident
        wins.append((w0, m, win if keep else None))
        del win
        total = wt if total is None else ops.lmme_ts(wt, total, 1)  # later windows on the left
    carry = exchange(ops.ts_to_goom(total)[0])
    c = ops.ts_from_goom(carry.reshape(1, d, d)) if carry is not None else None
    digests = torch.empty((n, 4), dtype=torch.float32, device=dev)
    for i, (w0, m, win) in enumerate(wins):
        if win is not None:
            _, dg, c = ops.chain_ts_finish(win, c, digests=True, carry_out=True)
        else:
            _, dg, c = ops.chain_ts(ops.ts_random_normal(m, d, seed, t0 + w0, dev), block, c,
                                    digests=True, carry_out=True)
        digests[w0:w0 + m] = dg
        wins[i] = None  # release the window's workspace
    return ChainRun(digests, ops.ts_to_goom(c)[0], {})


def _free_bytes() -> int:
    """Device memory available to new tensors: free on the device plus what the caching
    allocator holds but does not use."""
    free, _ = torch.cuda.mem_get_info()
    return free + torch.cuda.memory_reserved() - torch.cuda.memory_allocated()


def resident_fits(n: int, d: int, window: int) -> bool:
    """Whether every window's local products of an n-leaf shard fit in free device memory
    (tile-scaled: 4 B per element, plus one window of leaves being generated)."""
    need = (n + min(window, n)) * d * d * 4 * 1.08
    return need < 0.92 * _free_bytes()


def run_chain_sharded(T: int, d: int, seed: int = 0, window: int = 4096, block: int = 64,
                      group=None, snapshot_every: int = 0):
    """Rank-local part of a time-sharded chain run; returns (t0, ChainRun)."""
    from . import ops
    from .harness import run_chain

    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    t0, n = shard_range(T, rank, world)
    if world > 1 and ops.ts_eligible(d) and not snapshot_every:
        # a smaller window only pays when it lets the WHOLE shard stay resident (the engine's
        # launches lose efficiency below ~8k products); otherwise keep the window and let
        # run_shard_resident keep as many windows as fit
        w = window
        while w > 8192 and not resident_fits(n, d, w):
            w //= 2
        if not resident_fits(n, d, w):
            w = window
        # keeps as many windows' local products as fit; recomputes only the rest
        return t0, run_shard_resident(
            n, d, seed, t0, w, block,
            lambda tot: exclusive_carry(tot, torch.ops.goom.lmme, group))
    carry = None
    if world > 1:
        total = shard_total(n, d, seed, t0, window, block)
        carry = exclusive_carry(total, torch.ops.goom.lmme, group)
    return t0, run_chain(n, d, seed, window, block, t0=t0, carry=carry,
                         snapshot_every=snapshot_every)


def scan_chain_nccl(A_local: torch.Tensor, block: int = 64, group=None,
                    comm: Optional[int] = None) -> torch.Tensor:
    """Global prefixes of this rank's contiguous chunk of a chain split across ranks, in ONE
    C-ABI call (goom_scan_chain_sharded_c64: local scan, ncclAllGather of the chunk totals,
    exclusive carry, one batched LMME). A_local: complex64 (T_local, d, d) on this rank's
    GPU; ranks hold consecutive chunks in rank order. `comm` is a raw ncclComm_t; by default
    the NCCL communicator of `group` (torch's ProcessGroupNCCL)."""
    import ctypes

    from . import _lib

    if A_local.dtype != torch.complex64 or not A_local.is_cuda or A_local.dim() != 3:
        raise ValueError("A_local must be a complex64 CUDA tensor (T_local, d, d)")
    if comm is None:
        pg = group if group is not None else dist.distributed_c10d._get_default_group()
        comm = pg._get_backend(A_local.device)._comm_ptr()
    A_local = A_local.contiguous()
    T, d = A_local.shape[0], A_local.shape[1]
    lib = _lib.load()
    nranks = dist.get_world_size(group) if dist.is_initialized() else 1
    nws = int(lib.goom_scan_chain_sharded_workspace_size(T, d, int(block), nranks))
    ws = torch.empty(nws, dtype=torch.uint8, device=A_local.device)
    out = torch.empty_like(A_local)
    _lib.call("goom_scan_chain_sharded_c64", A_local.data_ptr(), out.data_ptr(), T, d, int(block),
              ctypes.c_void_p(comm), ws.data_ptr(), nws,
              ctypes.c_void_p(torch.cuda.current_stream().cuda_stream))
    return out
