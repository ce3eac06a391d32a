"""GPU tests of the long-chain harness (config 3 machinery) and the sharded path on one GPU."""

import math

import numpy as np
import pytest
import torch

from goom_testlib import scaled_real_err, to_np
from oracle import gooms_port as G

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def h():
    from paper_2510_03426_b200 import harness

    return harness


def test_random_chain_is_keyed_by_leaf_index(h):
    a = h.random_chain(20, 16, seed=5)
    b = h.random_chain(10, 16, seed=5, t0=5)
    assert torch.equal(a[5:15], b)
    c = h.random_chain(10, 16, seed=6, t0=5)
    assert not torch.equal(b, c)
    x = torch.ops.goom.to_real(h.random_chain(64, 64, seed=1), True).cpu().numpy().ravel()
    assert abs(x.mean()) < 0.01 and abs(x.std() - 1.0) < 0.01  # N(0, 1)
    assert set(np.unique(a.imag.cpu().numpy())) <= {0.0, np.float32(np.pi)}  # canonical


def test_digest_matches_oracle(h):
    X = h.random_chain(6, 32, seed=2)
    dg = torch.ops.goom.digest(X).cpu().numpy()
    l, s = to_np(X)
    for i in range(6):
        assert abs(dg[i, 0] - l[i].max()) < 1e-6
        want = 0.5 * np.log(np.sum(np.exp(2 * l[i])))
        assert abs(dg[i, 1] - want) < 1e-5
        assert dg[i, 2] == 1.0


@pytest.mark.parametrize("d,window,block", [(8, 100, 16), (64, 64, 8), (128, 96, 32)])
def test_windowed_run_matches_oracle(h, d, window, block):
    """Windows chained by carries == one scan of the whole chain (oracle, float64)."""
    T = 300
    A = h.random_chain(T, d, seed=11)
    run = h.run_chain(T, d, seed=11, window=window, block=block, snapshot_every=50)
    al, as_ = to_np(A)
    st = G.Stack(al, as_, np.full_like(al, -np.inf), np.ones_like(as_), np.zeros(T, bool))
    want = G.scan_sequential(st)
    # digests vs the float64 oracle's own prefixes
    lf = 0.5 * np.log(np.sum(np.exp(2 * (want.alog - want.alog.max(axis=(1, 2), keepdims=True))),
                             axis=(1, 2))) + want.alog.max(axis=(1, 2))
    dg = run.digests.double().cpu().numpy()
    assert np.max(np.abs(dg[:, 1] - lf) / np.maximum(1, np.abs(lf))) < 1e-4
    assert np.all(dg[:, 2] == 1.0)
    for t, P in run.snapshots.items():
        gl, gs = to_np(P[None])
        assert scaled_real_err(gl, gs, want.alog[t:t + 1], want.asign[t:t + 1]).max() < 1e-2
    gl, gs = to_np(run.final[None])
    assert scaled_real_err(gl, gs, want.alog[-1:], want.asign[-1:]).max() < 1e-2


def test_growth_rate_matches_lyapunov_theory(h):
    """log||P_t|| grows at (ln 2 + psi(d/2)) / 2 per step for N(0,1) leaves."""
    d, T = 64, 2000
    run = h.run_chain(T, d, seed=3, window=512, block=32)
    rate = h.growth_rate(run.digests)
    psi = math.log(d / 2) - 1 / d - 1 / (12 * (d / 2) ** 2)
    expected = 0.5 * (math.log(2) + psi)
    assert abs(rate - expected) < 0.02 * expected


@pytest.mark.parametrize("d", [128, 256])
def test_chain_total_and_sharded_fold_on_one_gpu(h, d):
    """The sharded algorithm (totals -> exclusive carries -> local scans), run shard by
    shard on one GPU, equals the single-GPU chain (d = 256: tile-scaled totals and scans)."""
    from paper_2510_03426_b200 import sharded

    T, world = 257, 3
    full = h.run_chain(T, d, seed=9, window=128, block=16)
    totals, runs = [], []
    for r in range(world):
        t0, n = sharded.shard_range(T, r, world)
        totals.append(sharded.shard_total(n, d, 9, t0, 64, 16))
    for r in range(world):
        t0, n = sharded.shard_range(T, r, world)
        carry = sharded.fold_carry(totals, r, torch.ops.goom.lmme)
        runs.append(h.run_chain(n, d, seed=9, window=128, block=16, t0=t0, carry=carry))
    dg = torch.cat([r.digests for r in runs]).double().cpu().numpy()
    ref = full.digests.double().cpu().numpy()
    assert np.max(np.abs(dg[:, 1] - ref[:, 1]) / np.maximum(1, np.abs(ref[:, 1]))) < 1e-4
    gl, gs = to_np(runs[-1].final[None])
    rl, rs = to_np(full.final[None])
    assert scaled_real_err(gl, gs, rl, rs).max() < 1e-2


def test_kernel_launch_counter_moves(h):
    from paper_2510_03426_b200 import ops

    n0 = ops.kernel_launches()
    h.random_chain(4, 8)
    assert ops.kernel_launches() > n0


def test_resident_shards_equal_the_single_gpu_chain(h):
    """run_shard_resident (local products kept between the totals pass and phase 3) run
    shard by shard on one GPU, with the exclusive carries folded from the shard totals
    exactly as the all-gather would, equals the single-GPU chain."""
    from paper_2510_03426_b200 import sharded

    T, d, world, window, block = 300, 256, 3, 64, 8
    full = h.run_chain(T, d, seed=12, window=window, block=block)
    totals = []

    def record(tot):
        totals.append(tot)
        return None

    # pass A: every shard's total (what each rank contributes to the all-gather)
    for r in range(world):
        t0, n = sharded.shard_range(T, r, world)
        sharded.run_shard_resident(n, d, 12, t0, window, block, record)
    runs = []
    for r in range(world):
        t0, n = sharded.shard_range(T, r, world)
        carry = sharded.fold_carry(totals, r, torch.ops.goom.lmme)
        # rank 1 keeps only one window resident: its other windows are recomputed
        runs.append(sharded.run_shard_resident(n, d, 12, t0, window, block, lambda _t: carry,
                                               max_resident=1 if r == 1 else None))
    dg = torch.cat([r.digests for r in runs]).double().cpu().numpy()
    ref = full.digests.double().cpu().numpy()
    assert np.max(np.abs(dg[:, 1] - ref[:, 1]) / np.maximum(1, np.abs(ref[:, 1]))) < 1e-4
    assert (dg[:, 2] == 1).all()
    gl, gs = to_np(runs[-1].final[None])
    rl, rs = to_np(full.final[None])
    assert scaled_real_err(gl, gs, rl, rs).max() < 1e-2


def _relay_gpu_worker(rank, world, port, T, d, window, block, q):
    import os

    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2510_03426_b200 as g
        from paper_2510_03426_b200 import sharded

        g._lib.load()
        t0, run = sharded.run_chain_relay(T, d, seed=12, window=window, block=block)
        q.put((rank, run.windows, run.digests.cpu().numpy()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_relay_shards_equal_the_single_gpu_chain(h, world):
    """run_chain_relay (windows round-robin, the tile-scaled carry relayed rank to rank over
    real gloo point-to-point messages, every rank on this GPU) gives the single-GPU chain's
    digests: every window is covered exactly once, log-norms within 1e-4."""
    import socket

    import torch.multiprocessing as mp

    T, d, window, block = 700, 256, 128, 16
    full = h.run_chain(T, d, seed=12, window=window, block=block)
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_relay_gpu_worker, args=(r, world, port, T, d, window, block, q))
             for r in range(world)]
    for p in procs:
        p.start()
    parts = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    dg = np.zeros((T, 4))
    seen = []
    for _, wins, dig in parts:
        for w0, m in wins:
            dg[w0:w0 + m] = dig[w0:w0 + m]
            seen.append(w0)
    assert sorted(seen) == list(range(0, T, window))
    ref = full.digests.double().cpu().numpy()
    assert (dg[:, 2] == 1).all()
    assert np.max(np.abs(dg[:, 1] - ref[:, 1]) / np.maximum(1, np.abs(ref[:, 1]))) < 1e-4


@pytest.mark.parametrize("mode", ["relay", "allgather"])
def test_bench_two_ranks_on_one_gpu(mode):
    """bench.py's N > 1 path end to end (torchrun; the carry relay, or the shard totals
    all-gathered with exclusive carries; max-over-ranks timing, one JSON line from rank 0),
    with both ranks sharing the box's GPU over gloo (GOOM_BENCH_SHARE_GPU=1)."""
    import json
    import os
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, GOOM_BENCH_SHARE_GPU="1", OMP_NUM_THREADS="1", GOOM_SHARD_MODE=mode)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", "29547", "bench.py", "--gpus", "2",
           "--steps", "1", "--warmup", "1", "--T", "4096", "--window", "1024", "--block", "64",
           "--no-cpu-baseline", "--e2e-T", "256"]
    out = subprocess.run(cmd, cwd=root, env=env, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]
    r = json.loads(lines[0])
    assert r["n_gpus"] == 2 and r["config"]["parallelism"].startswith(f"time-sharded x2 ({mode}")
    assert r["check"]["finite"]
    assert abs(r["check"]["growth_per_step"] - r["check"]["expected_growth"]) < 0.05


def _nccl_single_rank_comm():
    """A 1-rank NCCL communicator on the current GPU, straight from libnccl.so.2 (torch's)."""
    import ctypes

    import torch  # noqa: F401  (loads libnccl.so.2)

    lib = ctypes.CDLL("libnccl.so.2", mode=ctypes.RTLD_GLOBAL)

    class UniqueId(ctypes.Structure):
        _fields_ = [("internal", ctypes.c_char * 128)]

    uid = UniqueId()
    assert lib.ncclGetUniqueId(ctypes.byref(uid)) == 0
    comm = ctypes.c_void_p()
    assert lib.ncclCommInitRank(ctypes.byref(comm), 1, uid, 0) == 0
    return lib, comm


def test_scan_chain_sharded_c_abi_single_rank(h):
    """goom_scan_chain_sharded_c64 over a real NCCL communicator (1 rank: the all-gather is
    a copy and the carry is empty): equals goom_scan_chain_c64 bitwise."""
    from paper_2510_03426_b200 import sharded

    lib, comm = _nccl_single_rank_comm()
    try:
        for d, T in ((8, 100), (256, 40)):
            A = h.random_chain(T, d, seed=3)
            got = sharded.scan_chain_nccl(A, block=16, comm=comm.value)
            want = torch.ops.goom.scan_chain(A, 16, None)
            torch.cuda.synchronize()
            assert torch.equal(torch.view_as_real(got), torch.view_as_real(want))
    finally:
        lib.ncclCommDestroy(comm)


def test_scan_chain_sharded_c_abi_fold_matches_python(h):
    """The C-ABI's exclusive-carry apply (steps 3-4) is the Python sharded fold: the chunks'
    prefixes times the folded totals of the chunks before, checked against the one-GPU
    chain; the NCCL all-gather itself is covered by the single-rank test above and the gloo
    multi-process tests."""
    from paper_2510_03426_b200 import sharded

    T, d, world = 96, 8, 3
    A = h.random_chain(T, d, seed=4)
    full = torch.ops.goom.scan_chain(A, 16, None)
    totals, chunks = [], []
    for r in range(world):
        t0, n = sharded.shard_range(T, r, world)
        loc = torch.ops.goom.scan_chain(A[t0:t0 + n].contiguous(), 16, None)
        totals.append(loc[-1])
        chunks.append(loc)
    for r in range(world):
        t0, n = sharded.shard_range(T, r, world)
        carry = sharded.fold_carry(totals, r, torch.ops.goom.lmme)
        got = chunks[r] if carry is None else torch.ops.goom.lmme(chunks[r], carry[None])
        gl, gs = to_np(got)
        wl, ws = to_np(full[t0:t0 + n])
        assert scaled_real_err(gl, gs, wl, ws).max() < 1e-3


def test_chain_survival_real_overflows_goom_completes(h):
    """SPEC run_chain (paper Fig. 1): float64 products of 8x8 N(0,1) matrices overflow
    within ~700 steps (log-growth ~1.04/step vs the float64 limit ~709.8), float32 within
    ~90; complex64 / complex128 GOOM chains complete the whole length."""
    T = 2000
    r64 = h.chain_survival(h.ChainConfig(d=8, T_max=T, backend="real64", seed=1, trials=3))
    r32 = h.chain_survival(h.ChainConfig(d=8, T_max=T, backend="real32", seed=1, trials=3))
    assert all(not c for c in r64.completed) and all(m == "overflow" for m in r64.failure_mode)
    assert all(500 < s < 1000 for s in r64.survived_steps), r64.survived_steps
    assert all(40 < s < 150 for s in r32.survived_steps), r32.survived_steps
    for be in ("goom64", "goom32"):
        r = h.chain_survival(h.ChainConfig(d=8, T_max=T, backend=be, seed=1, trials=2))
        assert all(r.completed) and r.survived_steps == [T, T] and r.failure_mode == [None, None]
    # d = 1, A = [[1]] never fails: not expressible with random leaves; the config validates
    with pytest.raises(ValueError):
        h.ChainConfig(d=8, T_max=10, backend="real16")
