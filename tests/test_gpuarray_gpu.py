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


@pytest.mark.parametrize("nbytes", [1, 4097, (1 << 20) - 1, 1 << 20, (32 << 20) + 13,
                                    (100 << 20) + 5])
def test_staged_host_copies_roundtrip_exactly(pool, nbytes):
    """Pageable host buffers go through the pinned staging pipeline above
    1 MiB (chunks of 32 MiB over 3 stages, so the largest case wraps the
    stages); every size, odd host offsets included, round-trips bit-exactly."""
    rng = np.random.default_rng(nbytes)
    raw = rng.integers(0, 256, nbytes + 3, dtype=np.uint8)
    host = raw[3:]                             # misaligned host address
    g = pool.alloc_uninitialized(nd.uint8, (nbytes,))
    g.copy_from_host(host)
    back = np.empty(nbytes + 1, np.uint8)[1:]  # misaligned destination
    g.to_host(out=back)
    assert np.array_equal(back, host)
    stream = _runtime.Stream()
    with _runtime.use_stream(stream):
        h2 = host[::-1].copy()
        g.copy_from_host(h2, sync=False)
        h2[:] = 0                              # source reusable once the call returns
        assert np.array_equal(g.get(), host[::-1])
    stream.synchronize()


def test_pinned_and_pageable_paths_agree(pool):
    n = (48 << 20) // 8 + 3
    h = np.random.default_rng(3).integers(-(1 << 62), 1 << 62, n, dtype=np.int64)
    pin = nd.pinned_empty((n,), nd.int64)
    pin[:] = h
    a = nd.from_host(pool, nd.int64, h)
    b = nd.from_host(pool, nd.int64, pin)
    out_pin = nd.pinned_empty((n,), nd.int64)
    a.to_host(out=out_pin)
    assert np.array_equal(out_pin, h) and np.array_equal(b.get(), h)
    # an interior slice of a page-locked buffer is page-locked too (the
    # runtime asks cuPointerGetAttributes for the memory type of the range)
    assert _runtime.host_is_pinned(pin.ctypes.data)
    assert _runtime.host_is_pinned(pin[7:].ctypes.data)
    assert not _runtime.host_is_pinned(h.ctypes.data)
    c = nd.from_host(pool, nd.int64, pin[7:])
    out_view = out_pin[5:n - 2]
    c.to_host(out=out_view)
    assert np.array_equal(out_pin[5:n - 2], h[7:])


def test_roofline_helper_reports_hbm_fraction(pool):
    from paper_0911_3456_b200 import autotune as at, elementwise as ew, reduction as rd
    n = 1 << 26
    x = pool.alloc(nd.float32, (n,))
    y = pool.alloc(nd.float32, (n,))
    z = pool.alloc(nd.float32, (n,))
    axpy = ew.ElementwiseKernel("float a, float *x, float b, float *y, float *z",
                                "z[i] = a * x[i] + b * y[i]", "axpy_roof")
    r = at.roofline(axpy, 2.0, x, -3.0, y, z)
    assert r["bytes"] == 12 * n and r["GB/s"] > 3000 and 0.4 < r["frac"] < 1.3
    d = at.roofline(rd.dot_kernel(nd.float32), x, y)
    assert d["bytes"] == 8 * n and d["GB/s"] > 3000
