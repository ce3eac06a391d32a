"""Time-sharded LMME chain scan over the GPUs of one node.

Two schemes. The long-chain harness (bench.py, run_chain_sharded) deals windows round-robin
and relays the carry rank to rank (relay_windows: the single-GPU work per leaf, one d x d
product and one point-to-point message per window). The north star's scheme — contiguous
chunks, one all-gather of the chunk totals, a second pass with the exclusive carry — is the
C-ABI entry (goom_scan_chain_sharded_c64, scan_chain_nccl) and GOOM_SHARD_MODE=allgather:

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
                       exchange: Callable, max_resident: Optional[int] = None,
                       snapshots=(), anchors=()):
    """This rank's shard with its local products kept on the device (d % 256 == 0).

    Pass 1 runs the carry-independent phases 1-2 of every window (ops.chain_ts_local) and
    folds the window totals into the shard total, keeping the first `max_resident` windows'
    local products (default: as many as fit in free device memory); `exchange(total)`
    (all-gather + fold, or a test double) returns the shard's exclusive carry; pass 2 runs
    only phase 3 for the resident windows (ops.chain_ts_finish) and the whole window for the
    others. A fully resident rank does ~2 n products (the single-GPU work); one that keeps
    nothing does ~3 n (the totals recomputed, as shard_total + run_chain)."""
    from . import ops
    from .harness import ChainRun, _window_anchor_blocks

    dev = torch.device("cuda", torch.cuda.current_device())
    if anchors and window % block:
        raise ValueError("anchors need window to be a multiple of block")
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
    want = sorted({int(t) - t0 for t in snapshots if t0 <= int(t) < t0 + n})
    snaps, snaps_ts, anch = {}, {}, {}
    for i, (w0, m, win) in enumerate(wins):
        local = [t - w0 for t in want if w0 <= t < w0 + m]
        ks = _window_anchor_blocks(anchors, t0 + w0, m, block)
        if win is not None:
            _, dg, c, S, K = ops.chain_ts_finish(win, c, digests=True, carry_out=True,
                                                 snapshots=local, carries=ks)
        else:
            _, dg, c, S, K = ops.chain_ts(ops.ts_random_normal(m, d, seed, t0 + w0, dev), block,
                                          c, digests=True, carry_out=True, snapshots=local,
                                          carries=ks)
        digests[w0:w0 + m] = dg
        for j, k in enumerate(ks):
            anch[t0 + w0 + k * block] = K[j:j + 1]
        if local:
            S64 = ops.ts_to_goom(S)
            for j, t in enumerate(local):
                snaps[t0 + w0 + t] = S64[j]
                snaps_ts[t0 + w0 + t] = S[j:j + 1]
        wins[i] = None  # release the window's workspace
    return ChainRun(digests, ops.ts_to_goom(c)[0], snaps, snaps_ts, anch)


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


def relay_windows(nwin: int, rank: int, world: int, local: Callable, combine: Callable,
                  finish: Callable, send: Callable, recv: Callable):
    """Window round-robin time-sharding with a carry relay: rank r scans windows
    w = r, r + G, r + 2G, ... of the chain. Per window: `local(w)` runs the carry-independent
    part (the engine's phases 1-2) and returns (state, window total); the carry into w (the
    prefix P at the end of window w - 1) arrives from rank (w - 1) mod G (`recv`), the carry
    out carry(w) = total(w) (x) carry(w - 1) (`combine`; products accumulate on the left) goes
    to rank (w + 1) mod G (`send`), and `finish(w, state, carry_in)` applies the carry (phase
    3). Every leaf costs the single-GPU work (two LMMEs) plus one d x d product and one
    point-to-point message per window: no shard totals recomputed, nothing kept resident
    beyond the window in flight. The relay is a pipeline: each rank runs its window's
    phases 1-2 while the carry travels, so after the first round the ranks are staggered by
    one hop. Returns [(w, finish(...))] for this rank's windows."""
    out = []
    for w in range(rank, nwin, world):
        state, total = local(w)
        cin = None if w == 0 else recv((w - 1) % world)
        cout = total if cin is None else combine(total, cin)
        if w + 1 < nwin:
            send(cout, (w + 1) % world)
        out.append((w, finish(w, state, cin)))
    return out


def _p2p(group=None):
    """(send(tensors, dst), recv(like, src), drain()) over torch.distributed point-to-point:
    NCCL sends device tensors directly; gloo (CPU tests, the shared-GPU bench aid) goes
    through host copies. Sends are asynchronous; drain() waits for them."""
    backend = dist.get_backend(group)
    pending = []

    def send(ts, dst):
        for t in ts:
            x = t.contiguous() if backend == "nccl" else t.detach().cpu().contiguous()
            pending.append((dist.isend(x, dst, group=group), x))

    def recv(likes, src):
        got = []
        for like in likes:
            x = torch.empty_like(like) if backend == "nccl" else torch.empty(
                like.shape, dtype=like.dtype)
            dist.recv(x, src, group=group)
            got.append(x.to(like.device, non_blocking=True))
        return got

    def drain():
        for work, _ in pending:
            work.wait()
        pending.clear()

    return send, recv, drain


def run_chain_relay(T: int, d: int, seed: int = 0, window: int = 32768, block: int = 128,
                    group=None, snapshots=(), anchors=()):
    """Rank-local part of the window round-robin, carry-relay time-sharding (relay_windows) on
    the tile-scaled engine (d % 256 == 0); returns (0, ChainRun) whose digests cover the whole
    chain with this rank's windows filled (the others zero) and `windows` = [(w0, m)]."""
    from . import ops
    from .harness import ChainRun, _window_anchor_blocks

    rank, world = _world(group)
    dev = torch.device("cuda", torch.cuda.current_device())
    if anchors and window % block:
        raise ValueError("anchors need window to be a multiple of block")
    nwin = (T + window - 1) // window
    digests = torch.zeros((T, 4), dtype=torch.float32, device=dev)
    snaps, snaps_ts, anch = {}, {}, {}
    send_t, recv_t, drain = _p2p(group)
    like = ops.ts_empty(1, d, dev)

    def local(w):
        w0 = w * window
        m = min(window, T - w0)
        leaves = ops.ts_random_normal(m, d, seed, w0, dev)
        return ops.chain_ts_local(leaves, block)

    def send(c, dst):
        send_t((c.U, c.q, c.G), dst)

    def recv(src):
        return ops.TsMats(*recv_t((like.U, like.q, like.G), src))

    def finish(w, win, cin):
        w0 = w * window
        m = min(window, T - w0)
        local_snaps = [t - w0 for t in snapshots if w0 <= int(t) < w0 + m]
        ks = _window_anchor_blocks(anchors, w0, m, block)
        _, dg, c, S, K = ops.chain_ts_finish(win, cin, digests=True, carry_out=True,
                                             snapshots=local_snaps, carries=ks)
        digests[w0:w0 + m] = dg
        for j, k in enumerate(ks):
            anch[w0 + k * block] = K[j:j + 1]
        if local_snaps:
            S64 = ops.ts_to_goom(S)
            for j, t in enumerate(local_snaps):
                snaps[w0 + t] = S64[j]
                snaps_ts[w0 + t] = S[j:j + 1]
        return (w0, m, c)

    done = relay_windows(nwin, rank, world, local, lambda tot, cin: ops.lmme_ts(tot, cin, 1),
                         finish, send, recv)
    drain()
    last = ops.ts_to_goom(done[-1][1][2])[0] if done else None
    run = ChainRun(digests, last, snaps, snaps_ts, anch)
    run.windows = [(w0, m) for _, (w0, m, _) in done]
    return 0, run


def shard_mode() -> str:
    """GOOM_SHARD_MODE: "relay" (default; relay_windows) or "allgather" (contiguous shards,
    one all-gather of the shard totals, the local products kept resident where they fit)."""
    import os

    m = os.environ.get("GOOM_SHARD_MODE", "relay")
    if m not in ("relay", "allgather"):
        raise ValueError("GOOM_SHARD_MODE must be relay or allgather")
    return m


def run_chain_sharded(T: int, d: int, seed: int = 0, window: int = 4096, block: int = 64,
                      group=None, snapshot_every: int = 0, snapshots=(), anchors=()):
    """Rank-local part of a time-sharded chain run; returns (t0, ChainRun). `snapshots`:
    absolute prefix indices to keep (those inside this rank's part come back). d % 256 == 0
    shards windows round-robin with a carry relay (run_chain_relay; GOOM_SHARD_MODE=allgather
    for contiguous shards with one all-gather of the shard totals)."""
    from . import ops
    from .harness import run_chain

    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    t0, n = shard_range(T, rank, world)
    if world > 1 and ops.ts_eligible(d) and not snapshot_every and shard_mode() == "relay":
        return run_chain_relay(T, d, seed, window, block, group, snapshots=snapshots,
                               anchors=anchors)
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
            lambda tot: exclusive_carry(tot, torch.ops.goom.lmme, group), snapshots=snapshots,
            anchors=anchors)
    carry = None
    if world > 1:
        total = shard_total(n, d, seed, t0, window, block)
        carry = exclusive_carry(total, torch.ops.goom.lmme, group)
    return t0, run_chain(n, d, seed, window, block, t0=t0, carry=carry,
                         snapshot_every=snapshot_every, snapshots=snapshots, anchors=anchors)


def scan_chain_nccl(A_local: torch.Tensor, block: int = 64, group=None,
                    comm: Optional[int] = None, digests: bool = False) -> torch.Tensor:
    """Global prefixes of this rank's contiguous chunk of a chain split across ranks, in ONE
    C-ABI call (goom_scan_chain_sharded_c64: local phases 1-2, ncclAllGather of the chunk
    totals, exclusive carry folded onto the block carries, phase 3 — two LMMEs per leaf).
    A_local: complex64 (T_local, d, d) on this rank's GPU; ranks hold consecutive chunks in
    rank order. `comm` is a raw ncclComm_t; by default the NCCL communicator of `group`
    (torch's ProcessGroupNCCL). digests=True returns the (T_local, 4) float32 digests of
    the global prefixes instead (goom_scan_chain_sharded_digest_c64)."""
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
    size = (lib.goom_scan_chain_sharded_digest_workspace_size if digests
            else lib.goom_scan_chain_sharded_workspace_size)
    nws = int(size(T, d, int(block), nranks))
    ws = torch.empty(nws, dtype=torch.uint8, device=A_local.device)
    if digests:
        out = torch.empty((T, 4), dtype=torch.float32, device=A_local.device)
    else:
        out = torch.empty_like(A_local)
    _lib.call("goom_scan_chain_sharded_digest_c64" if digests else "goom_scan_chain_sharded_c64",
              A_local.data_ptr(), out.data_ptr(), T, d, int(block), ctypes.c_void_p(comm),
              ws.data_ptr(), nws, ctypes.c_void_p(torch.cuda.current_stream().cuda_stream))
    return out


# ---------------------------------------------------------------------------
# batch-only workloads: no communication on the data path


def _world(group=None):
    if dist.is_initialized():
        return dist.get_rank(group), dist.get_world_size(group)
    return 0, 1


def lmme_batch_sharded(A: torch.Tensor, B: torch.Tensor, group=None, gather: bool = True,
                       lmme: Optional[Callable] = None):
    """Config 2 (`_lmme_arrays` over a batch, core.py:242-261) sharded by batch: rank r
    computes products shard_range(batch, r, world) of A (batch, n, k) (x) B (batch, k, m)
    (a single-matrix operand broadcasts). No exchange on the data path; with gather=True
    the shards are all-gathered so every rank returns the whole batch, else the rank's
    slice and its first index."""
    lmme = lmme if lmme is not None else torch.ops.goom.lmme
    rank, world = _world(group)
    batch = max(A.shape[0], B.shape[0])
    t0, n = shard_range(batch, rank, world)
    a = A[t0:t0 + n] if A.shape[0] > 1 else A
    b = B[t0:t0 + n] if B.shape[0] > 1 else B
    local = lmme(a, b)
    if not gather or world == 1:
        return local if gather else (t0, local)
    real = torch.view_as_real(local.contiguous())
    sizes = [shard_range(batch, r, world)[1] for r in range(world)]
    parts = [torch.empty((sz,) + tuple(real.shape[1:]), dtype=real.dtype, device=real.device)
             for sz in sizes]
    if len(set(sizes)) == 1:
        dist.all_gather(parts, real, group=group)
    else:  # uneven shards: pad to the largest
        mx = max(sizes)
        pad = torch.zeros((mx,) + tuple(real.shape[1:]), dtype=real.dtype, device=real.device)
        pad[:real.shape[0]] = real
        full = [torch.empty_like(pad) for _ in range(world)]
        dist.all_gather(full, pad, group=group)
        parts = [f[:sz] for f, sz in zip(full, sizes)]
    return torch.view_as_complex(torch.cat(parts).contiguous())


def ssm_sequences_shard(x0s: torch.Tensor, us: torch.Tensor, group=None):
    """Config 5 data parallelism: this rank's slice of the S sequences of every head
    (x0s (H, S, d), us (H, S, T, d)) — the heads share A's powers, so sequences, not heads,
    are split. Returns (first sequence, x0s slice, us slice)."""
    rank, world = _world(group)
    s0, n = shard_range(us.shape[1], rank, world)
    return s0, x0s[:, s0:s0 + n], us[:, s0:s0 + n]


def allreduce_grads(params, group=None):
    """Sum the parameter gradients of a sequence-sharded SSM layer over the ranks (the one
    collective of data-parallel training; the forward and backward scans themselves have
    no exchange). In place on p.grad; parameters without a gradient are skipped."""
    _, world = _world(group)
    if world == 1:
        return
    for p in params:
        if p.grad is not None:
            dist.all_reduce(p.grad, op=dist.ReduceOp.SUM, group=group)


def ssm_layer_sharded(A, B, C, D, x0s, us, chunk: int = 64, group=None):
    """ssm.ssm_layer on this rank's sequences (ssm_sequences_shard): returns (first
    sequence, y slice). After backward, call allreduce_grads((A, B, C, D)) so every rank
    holds the gradient of the whole batch's loss."""
    from .ssm import ssm_layer

    s0, x, u = ssm_sequences_shard(x0s, us, group)
    return s0, ssm_layer(A, B, C, D, x, u, chunk)


def replicas(items, fn: Callable, group=None):
    """Config 4 (selective-reset scans do not shard: their reset sites are sequential,
    scan.py:9-12): independent items — trajectories, systems, seeds — are spread round-robin
    over the ranks, each processed whole by `fn` on its own GPU, and the results
    all-gathered (as Python objects) in item order on every rank."""
    rank, world = _world(group)
    mine = {i: fn(items[i]) for i in range(rank, len(items), world)}
    if world == 1:
        return [mine[i] for i in range(len(items))]
    parts = [None] * world
    dist.all_gather_object(parts, mine, group=group)
    merged = {}
    for p in parts:
        merged.update(p)
    return [merged[i] for i in range(len(items))]
