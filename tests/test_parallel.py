"""Multi-process sharding logic.

CPU: world-size-2 ``gloo`` process groups exercise the host side -- shard
ranges (the reference's worker formula), the rank-ordered all-gather of
per-rank accumulators, and the ordered fold -- with per-rank partials
computed by the CPU oracle.  GPU: the same driver end to end on one B200 with
an NCCL group of size 1 (the only GPU count available to the test box).
"""

import os
import socket

import numpy as np
import pytest
from hypothesis import given
from hypothesis import strategies as st

from paper_0911_3456_b200 import parallel as par


@given(st.integers(0, 10**7), st.integers(1, 16))
def test_shard_ranges_partition(n, world):
    ranges = [par.shard_range(n, r, world) for r in range(world)]
    assert ranges[0][0] == 0 and ranges[-1][1] == n
    for (lo, hi), (lo2, _) in zip(ranges, ranges[1:]):
        assert lo <= hi == lo2
    sizes = [hi - lo for lo, hi in ranges]
    assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        par.shard_range(n, world, world)


def test_nccl_op_only_when_exact():
    from paper_0911_3456_b200 import ndarray as nd, reduction as rd
    spec = lambda t, red: rd.ReductionSpec(f"{t.cname} *x", t, "0", red)  # noqa: E731
    assert par.nccl_op(spec(nd.int64, "a + b")) == "sum"
    assert par.nccl_op(spec(nd.int32, " b+a ")) == "sum"
    assert par.nccl_op(spec(nd.float32, "a + b")) is None        # float sum: ordered fold
    assert par.nccl_op(spec(nd.float64, "a > b ? a : b")) == "max"
    assert par.nccl_op(spec(nd.int8, "a < b ? a : b")) == "min"
    assert par.nccl_op(spec(nd.int16, "a + b")) is None           # no ncclInt16
    assert par.nccl_op(spec(nd.int64, "a * b")) is None


def test_ordered_fold_is_left_fold():
    assert par.ordered_fold(lambda a, b: a * 10 + b, 0, [1, 2, 3]) == 123


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, n, queue):
    import torch
    import torch.distributed as dist
    from oracle import cport
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        rng = np.random.default_rng(42)
        x = rng.integers(-(1 << 62), 1 << 62, size=n, dtype=np.int64)
        f = rng.uniform(-1, 1, n).astype(np.float32)
        lo, hi = par.shard_range(n, rank, world)
        s64 = cport.Reduction("int64_t *x", "int64", "0", "a + b")
        mx = cport.Reduction("float *x", "float32", "-INFINITY", "a > b ? a : b")
        local = torch.tensor([int(s64.fold_partials(s64.partials(x[lo:hi])))], dtype=torch.int64)
        gathered = par.gather_partials(local)
        total = par.ordered_fold(lambda a, b: (a + b + (1 << 63)) % (1 << 64) - (1 << 63), 0,
                                 [int(v) for v in gathered])
        lmax = torch.tensor([float(mx(f[lo:hi]))], dtype=torch.float64)
        gmax = max(float(v) for v in par.gather_partials(lmax))
        order = par.gather_partials(torch.tensor([rank * 10 + 1], dtype=torch.int64))
        queue.put((rank, total, gmax, [int(v) for v in order],
                   int(cport.Reduction("int64_t *x", "int64", "0", "a + b")(x)), float(f.max())))
    finally:
        dist.destroy_process_group()


def test_two_rank_gloo_partials_combine_like_single_process():
    import multiprocessing as mp
    ctx = mp.get_context("spawn")
    queue = ctx.Queue()
    port, n, world = _free_port(), 100_003, 2
    procs = [ctx.Process(target=_worker, args=(r, world, port, n, queue)) for r in range(world)]
    for p in procs:
        p.start()
    results = [queue.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, total, gmax, order, single, fmax in results:
        assert order == [1, 11]              # ascending rank order
        assert total == single               # wrapping int64 sum: exact
        assert gmax == fmax


# --- GPU: the real driver on one device ------------------------------------------------------


@pytest.fixture()
def nccl_world1():
    torch = pytest.importorskip("torch")
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(_free_port()))
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    yield
    dist.destroy_process_group()


@pytest.mark.gpu
def test_sharded_reduce_and_elementwise_single_rank(nccl_world1, pool):
    from oracle import cport
    from paper_0911_3456_b200 import elementwise as ew, ndarray as nd, reduction as rd
    n = (1 << 22) + 7
    rng = np.random.default_rng(5)
    host = rng.integers(-(1 << 62), 1 << 62, size=n, dtype=np.int64)
    sx = par.scatter_from_host(host, nd.int64, n, 0, 1, pool)
    got = par.sharded_reduce(rd.sum_kernel(nd.int64), sx)
    assert int(got) == int(cport.Reduction("int64_t *x", "int64", "0", "a + b")(host))
    dev = par.sharded_reduce(rd.sum_kernel(nd.int64), sx, return_device=True)
    assert int(dev.get()) == int(got)
    for collective in ("allreduce", "allgather"):
        assert int(par.sharded_reduce(rd.sum_kernel(nd.int64), sx, collective=collective)) == \
            int(got)
    mx = par.sharded_reduce(rd.max_kernel(nd.int64), sx, collective="allreduce")
    assert int(mx) == int(host.max())
    fx = par.scatter_from_host(host.astype(np.float32) * 1e-18, nd.float32, n, 0, 1, pool)
    with pytest.raises(ValueError):
        par.sharded_reduce(rd.sum_kernel(nd.float32), fx, collective="allreduce")
    assert float(par.sharded_reduce(rd.sum_kernel(nd.float32), fx)) == \
        float(rd.sum_kernel(nd.float32)(fx.local))
    out = par.ShardedArray(pool.alloc(nd.int64, (n,)), sx.base, n, 0, 1)
    par.sharded_elementwise(ew.ElementwiseKernel("long *x, long *z", "z[i] = x[i] ^ i", "xi"),
                            sx, out)
    assert np.array_equal(out.local.get(), host ^ np.arange(n, dtype=np.int64))


@pytest.mark.gpu
def test_shard_slices_keep_global_index(pool):
    """Two shards of one array processed separately give the unsharded result."""
    from paper_0911_3456_b200 import elementwise as ew, ndarray as nd, reduction as rd
    n = 1_000_003
    host = np.random.default_rng(1).uniform(-1, 1, n)
    k = ew.ElementwiseKernel("double *x, double *z", "z[i] = x[i] * (double) i", "xtimesi")
    whole = np.zeros(n)
    parts = []
    for r in range(3):
        s = par.scatter_from_host(host, nd.float64, n, r, 3, pool)
        z = pool.alloc(nd.float64, (s.local.size,))
        k(s.local, z, base=s.base)
        parts.append(z.get())
    whole = np.concatenate(parts)
    assert np.array_equal(whole, host * np.arange(n, dtype=np.float64))
    mx = rd.max_kernel(nd.float64)
    per_rank = [mx.launch(par.scatter_from_host(host, nd.float64, n, r, 3, pool).local) and
                mx._read(mx.scratch(0).out, nd.float64) for r in range(3)]
    assert max(per_rank) == host.max()


def _gpu_rank(rank, world, port, cache_dir, queue):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RTCG_CACHE_DIR=cache_dir)
    from paper_0911_3456_b200 import _runtime, elementwise as ew, ndarray as nd, reduction as rd
    _runtime.set_device(0)
    import torch
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        n = 3_000_017
        rng = np.random.default_rng(77)
        hi = rng.integers(-(1 << 62), 1 << 62, size=n, dtype=np.int64)
        hf = rng.uniform(-1, 1, n).astype(np.float32)
        pool = nd.MemoryPool(device=0)
        si = par.scatter_from_host(hi, nd.int64, n, rank, world, pool)
        sf = par.scatter_from_host(hf, nd.float32, n, rank, world, pool)
        out = {
            "sum_i64_allreduce": int(par.sharded_reduce(rd.sum_kernel(nd.int64), si,
                                                        collective="allreduce")),
            "sum_i64_allgather": int(par.sharded_reduce(rd.sum_kernel(nd.int64), si,
                                                        collective="allgather")),
            "max_f32": float(par.sharded_reduce(rd.max_kernel(nd.float32), sf)),
            "sum_f32": float(par.sharded_reduce(rd.sum_kernel(nd.float32), sf)),
        }
        z = par.ShardedArray(pool.alloc(nd.int64, (si.local.size,)), si.base, n, rank, world)
        par.sharded_elementwise(ew.ElementwiseKernel("long *x, long *z", "z[i] = x[i] + i", "xpi"),
                                si, z)
        lo, hi_ = par.shard_range(n, rank, world)
        out["elementwise_ok"] = bool(np.array_equal(z.local.get(),
                                                     hi[lo:hi_] + np.arange(lo, hi_)))
        queue.put((rank, out))
    finally:
        dist.destroy_process_group()


@pytest.mark.gpu
def test_two_ranks_sharing_the_gpu_reduce_like_one(tmp_path):
    """World size 2 (gloo; both ranks on the one B200): the sharded reductions
    and elementwise kernels equal the single-process results."""
    import multiprocessing as mp
    from oracle import csem, cport
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gpu_rank, args=(r, 2, port, str(tmp_path / "c"), q))
             for r in range(2)]
    for p in procs:
        p.start()
    results = dict(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    n = 3_000_017
    rng = np.random.default_rng(77)
    hi = rng.integers(-(1 << 62), 1 << 62, size=n, dtype=np.int64)
    hf = rng.uniform(-1, 1, n).astype(np.float32)
    want_i = int(cport.Reduction("int64_t *x", "int64", "0", "a + b")(hi))
    for r in (0, 1):
        got = results[r]
        assert got["sum_i64_allreduce"] == want_i == got["sum_i64_allgather"]
        assert got["max_f32"] == float(hf.max())
        terms = hf.astype(np.float64)
        assert abs(got["sum_f32"] - csem.exact_sum(terms)) <= \
            csem.float_reduction_bound(terms, "float32")
        assert got["elementwise_ok"]
    assert results[0] == results[1]           # every rank holds the same answer


def test_peer_plan_uses_bus_ids_not_ordinals():
    """under per-rank CUDA_VISIBLE_DEVICES every rank calls its
    GPU device 0; distinct physical GPUs must still be recognised (and peers
    this process cannot see make the exchange impossible)."""
    a, b = "0000:1b:00.0", "0000:43:00.0"
    assert par.peer_plan([a, b], {a: 0, b: 1})
    assert not par.peer_plan([a, a], {a: 0})                 # two ranks, one GPU
    assert not par.peer_plan([a, b], {a: 0})                 # peer not visible here
    assert par.peer_plan([a], {a: 0})


def test_mailbox_descriptor_layout_matches_the_kernel_struct():
    # struct rtcg::xr {int rank, world; u64 mbox[64]; u64 timeout_ns;}
    assert par._XR.size == 8 + 8 * par.XR_MAX + 8
