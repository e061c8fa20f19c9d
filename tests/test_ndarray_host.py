"""Dtypes, promotion and the pool's host-side logic (reference
tests/test_ndarray.py, tests/test_acceptance.py:233-268 and :442-472).  The
pool is exercised with injected host allocators so this runs without a GPU;
the device allocator itself is covered by the GPU tests."""

import ctypes
import threading

import numpy as np
import pytest
from hypothesis import given
from hypothesis import strategies as st

from paper_0911_3456_b200 import ndarray as nd

PROMOTION = {
    "int8": ("int8", "int16", "int32", "int64", "int16", "int32", "int64", "float64",
             "float32", "float64"),
    "int16": ("int16", "int16", "int32", "int64", "int16", "int32", "int64", "float64",
              "float32", "float64"),
    "int32": ("int32", "int32", "int32", "int64", "int32", "int32", "int64", "float64",
              "float64", "float64"),
    "int64": ("int64",) * 7 + ("float64", "float64", "float64"),
    "uint8": ("int16", "int16", "int32", "int64", "uint8", "uint16", "uint32", "uint64",
              "float32", "float64"),
    "uint16": ("int32", "int32", "int32", "int64", "uint16", "uint16", "uint32", "uint64",
               "float32", "float64"),
    "uint32": ("int64", "int64", "int64", "int64", "uint32", "uint32", "uint32", "uint64",
               "float64", "float64"),
    "uint64": ("float64",) * 4 + ("uint64",) * 4 + ("float64", "float64"),
    "float32": ("float32", "float32", "float64", "float64", "float32", "float32", "float64",
                "float64", "float32", "float64"),
    "float64": ("float64",) * 10,
}


def test_dtypes():
    assert {d.name for d in nd.DTYPES} == set(PROMOTION)
    for d in nd.DTYPES:
        assert d.np.itemsize == d.size == ctypes.sizeof(nd.ctype_for(d))
    assert nd.BY_NAME["float32"] is nd.float32 and nd.BY_CNAME["int64_t"] is nd.int64
    assert nd.dtype_of(np.float64) is nd.float64 and nd.dtype_of("int8") is nd.int8
    with pytest.raises(TypeError):
        nd.dtype_of(np.complex64)


def test_promotion_table_frozen_and_numpy_equal():
    for a in nd.DTYPES:
        for j, b in enumerate(nd.DTYPES):
            got = nd.promote(a, b)
            assert got.name == PROMOTION[a.name][j] == np.promote_types(a.name, b.name).name
            assert got is nd.promote(b, a)
        assert nd.promote(a, a) is a


def test_size_classes():
    assert nd.size_class(1) == 64 and nd.size_class(64) == 64 and nd.size_class(65) == 128
    assert nd.size_class(4000) == 4096 and nd.size_class(1 << 30) == 1 << 30
    assert nd.size_class((1 << 30) + 1) is None
    with pytest.raises(ValueError):
        nd.size_class(0)


@given(st.integers(1, 1 << 30))
def test_size_class_is_covering_power_of_two(nbytes):
    cls = nd.size_class(nbytes)
    assert cls >= max(nbytes, 64) and cls & (cls - 1) == 0
    assert cls == 64 or cls // 2 < max(nbytes, 65)


class HostDevice:
    """Stand-in allocator: ctypes buffers, zeroing with memset."""

    def __init__(self, fail_at=None):
        self.calls, self.fail_at, self.freed, self.zeroed = 0, fail_at, [], []

    def alloc(self, nbytes):
        self.calls += 1
        if self.fail_at is not None and self.calls == self.fail_at:
            raise MemoryError("injected")
        return ctypes.create_string_buffer(nbytes)

    def free(self, handle):
        self.freed.append(handle)

    def zero(self, address, nbytes):
        self.zeroed.append(nbytes)
        ctypes.memset(address, 0, nbytes)

    def pool(self):
        return nd.MemoryPool(self.alloc, system_free=self.free, zero_fill=self.zero)


def test_pool_hits_zeroing_and_counters():
    dev = HostDevice()
    pool = dev.pool()
    for _ in range(100):
        pool.free(pool.alloc(nd.float64, (1000,)))
    s = pool.stats()
    assert s["allocations_served"] == 100 and s["pool_hits"] == 99
    assert dev.zeroed == [8000] * 100  # zero on every allocation, also on reuse
    a = pool.alloc(nd.float32, (1024,))
    pool.free(a)
    b = pool.alloc(nd.float32, (1000,))
    assert pool.stats()["pool_hits"] == 100 and b.size == 1000
    u = pool.alloc_uninitialized(nd.float32, (1000,))
    assert dev.zeroed[-1] == 4000 and u.size == 1000  # the earlier alloc zeroed, not this one


def test_empty_and_zero_extent_arrays():
    pool = HostDevice().pool()
    a = pool.alloc(nd.float32, (0,))
    assert a.size == 0 and a.nbytes == 0 and a.address == 0
    assert pool.stats()["bytes_from_system"] == 0
    pool.free(a)
    b = pool.alloc(nd.float32, (4, 0, 2))
    assert b.size == 0 and b.shape == (4, 0, 2)
    with pytest.raises(nd.ShapeMismatch):
        pool.alloc(nd.float32, (-1,))


def test_free_semantics():
    dev = HostDevice()
    pool = dev.pool()
    a = pool.alloc(nd.float32, (256,))
    held = pool.stats()["bytes_from_system"]
    pool.free(a)
    s = pool.stats()
    assert s["bytes_from_system"] == held and s["bytes_held"] == held
    with pytest.raises(ValueError):
        pool.free(a)
    with pytest.raises(ValueError):
        a.address
    with pytest.raises(ValueError):
        pool.free(HostDevice().pool().alloc(nd.int8, (3,)))
    assert pool.release_free() > 0 and pool.stats()["bytes_from_system"] == 0
    assert len(dev.freed) == 1


def test_bypass_blocks_return_to_device():
    dev = HostDevice()
    pool = nd.MemoryPool(lambda n: 0x10000, system_free=dev.free, zero_fill=lambda a, n: None)
    big = pool.alloc(nd.uint8, ((1 << 30) + 1,))
    assert pool.stats()["bytes_outstanding"] == (1 << 30) + 1
    pool.free(big)
    assert pool.stats()["bytes_from_system"] == 0 and dev.freed == [0x10000]


def test_release_and_retry_on_allocator_failure():
    dev = HostDevice()
    pool = dev.pool()
    pool.free(pool.alloc(nd.float32, (100,)))
    assert pool.stats()["bytes_held"] > 0
    dev.fail_at = dev.calls + 1
    big = pool.alloc(nd.float32, (5000,))
    assert big.size == 5000 and pool.stats()["bytes_held"] == 0
    always = nd.MemoryPool(lambda n: (_ for _ in ()).throw(MemoryError("no")))
    with pytest.raises(nd.OutOfMemory):
        always.alloc(nd.float32, (100,))


def test_device_oom_is_a_memory_error():
    from paper_0911_3456_b200 import _runtime
    assert issubclass(_runtime.DeviceOutOfMemory, MemoryError)


@given(st.lists(st.tuples(st.booleans(), st.integers(1, 5000)), max_size=40))
def test_pool_conservation_under_random_traffic(actions):
    pool = HostDevice().pool()
    live = []
    for do_alloc, n in actions:
        if do_alloc or not live:
            live.append(pool.alloc(nd.uint8, (n,)))
        else:
            pool.free(live.pop(len(live) // 2))
    s = pool.stats()
    assert s["bytes_held"] + s["bytes_outstanding"] == s["bytes_from_system"]
    assert s["pool_hits"] <= s["allocations_served"]


def test_pool_thread_safety_smoke():
    pool = HostDevice().pool()

    def work():
        for _ in range(200):
            pool.free(pool.alloc(nd.int16, (128,)))
    threads = [threading.Thread(target=work) for _ in range(4)]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    s = pool.stats()
    assert s["allocations_served"] == 800 and s["bytes_outstanding"] == 0
    assert s["bytes_held"] + s["bytes_outstanding"] == s["bytes_from_system"]


def test_array_metadata_and_interface():
    pool = HostDevice().pool()
    a = pool.alloc(nd.int16, (3, 5))
    assert a.nbytes == 30 and a.size == 15 and a.ndim == 2 and len(a) == 3
    cai = a.__cuda_array_interface__
    assert cai["shape"] == (3, 5) and cai["typestr"] == "<i2" and cai["data"][0] == a.address
    assert nd.GPUArray is nd.NdArray and "GPUArray" in repr(a)


def test_dropped_arrays_return_to_the_pool():
    import gc
    dev = HostDevice()
    pool = dev.pool()
    a = pool.alloc(nd.float32, (1000,))
    held_before = pool.stats()["bytes_held"]
    del a
    gc.collect()
    s = pool.stats()
    assert s["bytes_held"] == held_before + 4096 and s["bytes_outstanding"] == 0
    b = pool.alloc(nd.float32, (1000,))
    assert pool.stats()["pool_hits"] == 1
    pool.free(b)           # an explicit free leaves nothing for the GC: no double return
    del b
    gc.collect()
    assert pool.stats()["bytes_held"] == 4096


def test_alloc_and_alloc_uninitialized_are_thread_safe():
    """Every alloc() zero-fills exactly once even while other threads call
    alloc_uninitialized() on the same pool (it used to swap the pool's zero
    function for the duration of the call)."""
    import ctypes
    import threading
    zeroed = []
    lock = threading.Lock()

    def zero(address, nbytes):
        with lock:
            zeroed.append(address)
    pool = nd.MemoryPool(lambda n: ctypes.create_string_buffer(n), zero_fill=zero)
    rounds = 2000

    def zeroing():
        for _ in range(rounds):
            pool.alloc(nd.float32, (16,)).free()

    def raw():
        for _ in range(rounds):
            pool.alloc_uninitialized(nd.float32, (16,)).free()
    threads = [threading.Thread(target=f) for f in (zeroing, raw, raw, zeroing)]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    assert len(zeroed) == 2 * rounds


def test_host_argument_handlers_and_views():
    import ctypes
    from paper_0911_3456_b200 import driver as drv
    a = np.arange(10, dtype=np.float32)
    assert drv.In(a).copy_in and not drv.In(a).copy_out
    assert drv.Out(a).copy_out and not drv.Out(a).copy_in
    assert drv.InOut(a).copy_in and drv.InOut(a).copy_out and drv.InOut(a).size == 10
    with pytest.raises(TypeError):
        drv.In([1, 2, 3])
    with pytest.raises(ValueError):
        drv.In(a[::2])
    ro = a.copy()
    ro.flags.writeable = False
    drv.In(ro)
    with pytest.raises(ValueError):
        drv.Out(ro)
    pool = nd.MemoryPool(lambda n: ctypes.create_string_buffer(n), zero_fill=lambda p, n: None)
    g = pool.alloc(nd.int32, (100,))
    v = g[10:20]
    assert v.size == 10 and v.address == g.address + 40 and v.pool is pool
    assert g[-5:].size == 5 and g[90:200].size == 10 and g[50:10].size == 0
    with pytest.raises(TypeError):
        g[::2]
    with pytest.raises(TypeError):
        g[3]
    with pytest.raises(ValueError):
        v.free()
    g.free()
    with pytest.raises(ValueError):
        g[0:1]


@pytest.mark.timeout(60)
def test_collection_inside_the_pool_lock_does_not_deadlock():
    """A cyclic garbage collection can run while the pool holds its lock (any
    allocation inside the locked section); an unreachable array in a cycle
    then returns its block from __del__ on the same thread."""
    import gc
    dev = HostDevice()
    pool = dev.pool()

    class Holder:
        pass
    h = Holder()
    h.me, h.arr = h, pool.alloc(nd.float32, (100,))
    del h                                   # now only reachable through its own cycle
    with pool._lock:
        gc.collect()                        # __del__ -> _give_back on this thread
    assert pool.stats()["bytes_outstanding"] == 0
