"""The fused cross-GPU reduction (``collective="p2p"``): the reduction kernel's
last CTA exchanges accumulators with every rank through peer-memory
mailboxes and folds them in rank order.

On the one-GPU box the protocol is exercised three ways: emulated ranks in
one process (one mailbox and one stream per rank, kernels running
concurrently on the device), world size 1 through ``sharded_reduce``, and two
processes sharing the GPU with CUDA IPC-mapped mailboxes.  The expected value
is always the all-gather semantics: per-rank accumulators folded in
ascending rank order (``parallel.ordered_fold``), bit for bit."""

import os
import socket

import numpy as np
import pytest

from paper_0911_3456_b200 import parallel as par

pytestmark = pytest.mark.gpu


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _rank_accumulators(kernel, shards):
    """Each rank's own accumulator (local reduction, no exchange)."""
    accs = []
    for args, base in shards:
        s = kernel.launch(*args, base=base)
        accs.append(kernel._read(s.result, kernel.spec.acc_dtype))
    return accs


def _emulate(kernel, shards, group, rounds=1):
    """Launch every emulated rank on its own stream; returns per-rank outs."""
    from paper_0911_3456_b200 import _runtime as rt, ndarray as nd
    pool = nd.default_pool()
    streams = [rt.Stream() for _ in shards]
    outs = [[pool.alloc_uninitialized(kernel.spec.acc_dtype, ()) for _ in shards]
            for _ in range(rounds)]
    for k in range(rounds):
        for r, ((args, base), st) in enumerate(zip(shards, streams)):
            with rt.use_stream(st.handle):
                s = kernel.launch(*args, base=base, peers=group[r])
                rt.memcpy_dtod(outs[k][r].address, s.result, kernel.spec.acc_dtype.size)
    for st in streams:
        st.synchronize()
    return [[o.get()[()] for o in row] for row in outs]


def _shard(pool, dtype, host_arrays, world):
    from paper_0911_3456_b200 import ndarray as nd
    n = host_arrays[0].size
    shards = []
    for r in range(world):
        lo, hi = par.shard_range(n, r, world)
        shards.append(([nd.from_host(pool, dtype, h[lo:hi]) for h in host_arrays], lo))
    return shards


@pytest.mark.parametrize("world", [1, 2, 3, 8])
def test_emulated_ranks_fold_like_allgather(pool, world):
    from paper_0911_3456_b200 import ndarray as nd, reduction as rd
    rng = np.random.default_rng(world)
    n = 4_000_037
    x = rng.uniform(-1, 1, n).astype(np.float32)
    y = rng.uniform(-1, 1, n).astype(np.float32)
    dot = rd.dot_kernel(nd.float32)
    shards = _shard(pool, nd.float32, [x, y], world)
    want = par.ordered_fold(lambda a, b: a + b, 0.0, _rank_accumulators(dot, shards))
    group = par.PeerMailbox.local_group(world)
    rounds = _emulate(dot, shards, group, rounds=4)   # four epochs back to back
    for row in rounds:
        assert all(float(v) == float(want) for v in row), (row, want)
    for m in group:
        m.close()


def test_emulated_ranks_integer_max_and_empty_shard(pool):
    """int64 wrapping sum and a custom max, with one rank holding nothing."""
    from paper_0911_3456_b200 import ndarray as nd, reduction as rd
    rng = np.random.default_rng(9)
    x = rng.integers(-(1 << 62), 1 << 62, 1_000_003, dtype=np.int64)
    world = 3
    parts = [x[:600_000], x[600_000:600_000], x[600_000:]]      # rank 1 is empty
    shards = [([nd.from_host(pool, nd.int64, p)], lo) for p, lo in zip(parts, (0, 600_000,
                                                                             600_000))]
    group = par.PeerMailbox.local_group(world)
    total = rd.sum_kernel(nd.int64)
    got = _emulate(total, shards, group)[0]
    want = int(np.sum(x))   # numpy int64 sum wraps like the kernel
    assert all(int(v) == want for v in got)
    mx = rd.make_reduction("int64_t *x", nd.int64, "INT64_MIN", "a > b ? a : b",
                           "x[i] ^ (x[i] >> 7)")
    got = _emulate(mx, shards, group)[0]
    assert all(int(v) == int(np.max(x ^ (x >> 7))) for v in got)
    for m in group:
        m.close()


def test_emulated_ranks_tma_and_general_paths(pool):
    from paper_0911_3456_b200 import elementwise as ew, ndarray as nd, reduction as rd
    rng = np.random.default_rng(3)
    x = rng.uniform(-2, 2, 2_000_003)
    world = 4
    shards = _shard(pool, nd.float64, [x], world)
    for variant, mapped in ((ew.VariantParams(cache="tma"), "x[i] * x[i]"),
                            (ew.VariantParams(), "x[i] * (double) (i % 3)")):   # uses i: general
        k = rd.make_reduction("double *x", nd.float64, "0", "a + b", mapped, "sq",
                              variant)
        want = par.ordered_fold(lambda a, b: a + b, 0.0, _rank_accumulators(k, shards))
        group = par.PeerMailbox.local_group(world)
        assert all(float(v) == float(want) for v in _emulate(k, shards, group)[0])
        for m in group:
            m.close()


@pytest.fixture()
def nccl_world1():
    torch = pytest.importorskip("torch")
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(_free_port()))
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    yield
    dist.destroy_process_group()


def test_world_one_p2p_through_sharded_reduce(nccl_world1, pool):
    from paper_0911_3456_b200 import ndarray as nd, reduction as rd
    n = (1 << 22) + 5
    host = np.random.default_rng(2).uniform(-1, 1, n).astype(np.float32)
    sx = par.scatter_from_host(host, nd.float32, n, 0, 1, pool)
    k = rd.sum_kernel(nd.float32)
    assert par.p2p_capable()
    got = [float(par.sharded_reduce(k, sx, collective=c)) for c in ("p2p", "allgather", "auto")]
    assert got[0] == got[1] == got[2] == float(k(sx.local))
    dev = par.sharded_reduce(k, sx, collective="p2p", return_device=True)
    assert float(dev.get()) == got[0]


def _ipc_rank(rank, world, port, cache_dir, queue):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RTCG_CACHE_DIR=cache_dir)
    from paper_0911_3456_b200 import _runtime, ndarray as nd, reduction as rd
    _runtime.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        n = 2_000_003
        host = np.random.default_rng(13).integers(-(1 << 40), 1 << 40, n, dtype=np.int64)
        pool = nd.MemoryPool(device=0)
        sx = par.scatter_from_host(host, nd.int64, n, rank, world, pool)
        mb = par.PeerMailbox.create()
        k = rd.sum_kernel(nd.int64)
        out = pool.alloc_uninitialized(nd.int64, ())
        got = []
        for _ in range(3):
            k.launch(sx.local, base=sx.base, out=out, peers=mb)
            got.append(int(out.get()[()]))
        dist.barrier()
        mb.close()
        queue.put((rank, got))
    finally:
        dist.destroy_process_group()


def test_two_processes_exchange_through_ipc_mailboxes(tmp_path):
    """Two processes on the one GPU, mailboxes mapped with CUDA IPC: the same
    protocol as NVLink peers (contexts time-slice, so this is slow but exact)."""
    import multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_ipc_rank, args=(r, 2, port, str(tmp_path / "c"), q))
             for r in range(2)]
    for p in procs:
        p.start()
    results = dict(q.get(timeout=240) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    n = 2_000_003
    host = np.random.default_rng(13).integers(-(1 << 40), 1 << 40, n, dtype=np.int64)
    assert results[0] == results[1] == [int(host.sum())] * 3


def test_emulated_ranks_survive_skew_over_many_epochs(pool):
    """Random per-rank delays before each reduction (a busy kernel of random
    length on the rank's stream) make ranks run ahead into the next epoch
    while others still fold: every rank must still get the exact ordered
    fold, round after round (parity banks + monotone epochs)."""
    from paper_0911_3456_b200 import _runtime as rt, elementwise as ew, ndarray as nd
    from paper_0911_3456_b200 import reduction as rd
    world, rounds = 4, 60
    rng = np.random.default_rng(21)
    x = rng.integers(-1000, 1000, 200_003).astype(np.int64)
    shards = _shard(pool, nd.int64, [x], world)
    k = rd.sum_kernel(nd.int64)
    want = int(x.sum())
    spin = ew.ElementwiseKernel("long iters, float *w",
                                "float a = w[i]; for (long t = 0; t < iters; ++t) "
                                "a = a * 0.999f + 0.001f; w[i] = a", "spin")
    busy = [pool.alloc(nd.float32, (4096,)) for _ in range(world)]
    group = par.PeerMailbox.local_group(world)
    streams = [rt.Stream() for _ in range(world)]
    outs = [[pool.alloc_uninitialized(nd.int64, ()) for _ in range(world)] for _ in range(rounds)]
    for j in range(rounds):
        for r in rng.permutation(world):
            with rt.use_stream(streams[r].handle):
                spin(int(rng.integers(0, 20000)), busy[r])
                s = k.launch(*shards[r][0], base=shards[r][1], peers=group[r])
                rt.memcpy_dtod(outs[j][r].address, s.result, 8)
    for st in streams:
        st.synchronize()
    got = [[int(o.get()[()]) for o in row] for row in outs]
    assert got == [[want] * world] * rounds
    for m in group:
        m.close()


def test_missing_peer_times_out_softly(pool):
    """A rank whose peer never arrives gives up after the mailbox timeout,
    records the epoch in its error word and poisons result/out (all bits
    set: -1 for int64, NaN for floats) so a device-side consumer cannot take
    the local value for the global one; check() raises PeerTimeout once,
    clears the word, and the context stays usable."""
    import time
    from paper_0911_3456_b200 import ndarray as nd, reduction as rd
    group = par.PeerMailbox.local_group(2, timeout_s=2.0)
    x = nd.from_host(pool, nd.int64, np.arange(1000, dtype=np.int64))
    k = rd.sum_kernel(nd.int64)
    out = pool.alloc_uninitialized(nd.int64, ())
    t0 = time.perf_counter()
    s = k.launch(x, peers=group[0], out=out)          # rank 1 never launches
    with pytest.raises(par.PeerTimeout):
        group[0].check()
    assert 1.5 < time.perf_counter() - t0 < 30
    assert int(k._read(s.result, nd.int64)) == -1     # poisoned, not the local sum
    assert int(out.get()[()]) == -1
    group[0].check()                                  # reported once, then clean
    assert int(k(x)) == int(np.arange(1000).sum())    # context alive
    # floats: NaN
    xf = nd.from_host(pool, nd.float32, np.ones(100, np.float32))
    kf = rd.sum_kernel(nd.float32)
    g2 = par.PeerMailbox.local_group(2, timeout_s=0.5)
    of = pool.alloc_uninitialized(nd.float32, ())
    kf.launch(xf, peers=g2[1], out=of)
    with pytest.raises(par.PeerTimeout):
        g2[1].check()
    assert np.isnan(of.get()[()])
    for m in group + g2:
        m.close()


def test_mailbox_timeout_validated():
    with pytest.raises(ValueError):
        par.PeerMailbox.local_group(2, timeout_s=0)


def test_overlapped_launches_with_the_peer_exchange(pool):
    """Emulated ranks launching back-to-back overlapped reductions: each
    rank's next reduction streams while its previous one exchanges.

    Emulated ranks share one GPU's SMs: an overlapped grid that launched
    early holds its CTAs while it waits, so many queued grids of several
    ranks could starve a rank that has not exchanged yet.  With one GPU per
    rank that cannot happen (a rank's waiting grid only waits on its own
    predecessor, resident by construction); here the grids are pinned to 2
    CTAs so every queued grid fits on the device at once."""
    from paper_0911_3456_b200 import elementwise as ew, ndarray as nd, reduction as rd
    rng = np.random.default_rng(61)
    x = rng.uniform(-1, 1, 2_000_011).astype(np.float32)
    y = rng.uniform(-1, 1, 2_000_011).astype(np.float32)
    world = 3
    dot = rd.dot_kernel(nd.float32, ew.VariantParams(workers=2))
    shards = _shard(pool, nd.float32, [x, y], world)
    want = par.ordered_fold(lambda a, b: a + b, 0.0, _rank_accumulators(dot, shards))
    from paper_0911_3456_b200 import _runtime as rt
    group = par.PeerMailbox.local_group(world)
    streams = [rt.Stream() for _ in range(world)]
    outs = [[pool.alloc_uninitialized(nd.float64, ()) for _ in range(world)] for _ in range(8)]
    for j in range(8):
        for r in range(world):
            with rt.use_stream(streams[r].handle):
                s = dot.launch(*shards[r][0], base=shards[r][1], peers=group[r],
                               overlap_previous=True)
                rt.memcpy_dtod(outs[j][r].address, s.result, 8)
    for st in streams:
        st.synchronize()
    assert all(float(o.get()) == float(want) for row in outs for o in row)
    for m in group:
        m.close()


def test_emulated_ranks_with_dynamic_chunks(pool):
    """VariantParams.chunk under the in-kernel exchange: each rank's chunk
    partials fold in chunk order, then the ranks' accumulators in rank
    order -- every rank ends with the ordered fold of the local results,
    over four epochs (the chunk counters re-armed between them)."""
    from paper_0911_3456_b200 import elementwise as ew, ndarray as nd, reduction as rd
    rng = np.random.default_rng(12)
    n, world = 8_000_000, 4                       # shard starts stay 16-byte aligned
    x = rng.uniform(-1, 1, n).astype(np.float32)
    y = rng.uniform(-1, 1, n).astype(np.float32)
    dot = rd.dot_kernel(nd.float32, ew.VariantParams(unroll=2, chunk=4096))
    shards = _shard(pool, nd.float32, [x, y], world)
    assert dot.launch_config(*shards[1][0])["entry"] == dot.name     # the vector entry
    want = par.ordered_fold(lambda a, b: a + b, 0.0, _rank_accumulators(dot, shards))
    group = par.PeerMailbox.local_group(world)
    for row in _emulate(dot, shards, group, rounds=4):
        assert all(float(v) == float(want) for v in row), (row, want)
    for m in group:
        m.close()
