"""PyCUDA-style GPUArray conveniences and the stream-ordered system allocator."""

import time

import numpy as np
import pytest

from paper_0911_3456_b200 import _runtime, gpuarray, ndarray as nd

pytestmark = pytest.mark.gpu


def test_fill_astype_copy(pool):
    a = pool.alloc(nd.int32, (1001,))
    a.fill(-7)
    assert np.all(a.get() == -7)
    h = np.random.default_rng(1).uniform(-3, 3, 1001)
    f = nd.from_host(pool, nd.float64, h)
    i = f.astype(np.int16)
    assert i.dtype is nd.int16 and np.array_equal(i.get(), h.astype(np.int16))  # C truncation
    c = f.copy()
    assert c.address != f.address and np.array_equal(c.get(), h)
    u = pool.alloc(nd.uint8, (5,)).fill(300)     # scalar conversion wraps like C
    assert list(u.get()) == [44] * 5


def test_module_reductions_return_device_scalars(pool):
    h = np.arange(1, 101, dtype=np.int64)
    x = nd.from_host(pool, nd.int64, h)
    s = gpuarray.sum(x)
    assert isinstance(s, nd.NdArray) and s.shape == () and int(s.get()) == 5050
    assert int(gpuarray.max(x).get()) == 100 and int(gpuarray.min(x).get()) == 1
    y = nd.from_host(pool, nd.float32, np.ones(100, np.float32))
    d = gpuarray.dot(x, y)                     # promoted to float64
    assert d.dtype is nd.float64 and float(d.get()) == 5050.0


def test_large_blocks_use_stream_ordered_allocation(pool):
    """Blocks above the 1 GiB top class bypass the size classes (reference
    semantics) but come from the stream-ordered allocator: allocate/free
    cycles do not stall and data is intact."""
    n = (1 << 28) + 1                       # 2 GiB of float64: bypass
    x = pool.alloc(nd.float64, (n,))
    x.fill(1.5)
    assert float(gpuarray.sum(x).get()) == 1.5 * n
    _runtime.synchronize()
    cycles = []
    for _ in range(20):
        t0 = time.perf_counter()
        t = pool.alloc_uninitialized(nd.float64, (n,))
        t.free()
        cycles.append(time.perf_counter() - t0)
    # the first cycle may grow the driver's pool; steady state must not stall
    assert sorted(cycles)[10] < 2e-3, cycles
    s = pool.stats()
    assert s["bytes_held"] + s["bytes_outstanding"] == s["bytes_from_system"]
    x.free()


def test_oom_trims_cached_pool_memory_and_retries(pool):
    """Fill the device with stream-ordered blocks, free them (they stay cached
    in the driver pool), then a synchronous allocation of most of the device
    must still succeed: out-of-memory triggers a trim and one retry."""
    free, total = _runtime.mem_get_info()
    chunk = 8 << 30
    held = []
    while True:
        try:
            held.append(_runtime.mem_alloc_async(chunk))
        except _runtime.DeviceOutOfMemory:
            break
        if len(held) * chunk > total:
            break
    assert held
    for p in held:
        _runtime.mem_free_async(p)
    _runtime.synchronize()
    big = _runtime.mem_alloc(len(held) * chunk - chunk)   # needs the cached memory back
    _runtime.mem_free(big)
