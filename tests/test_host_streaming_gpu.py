"""Streamed host calls (``driver.In`` / ``Out`` / ``InOut``): chunked
upload / kernel / download on two streams must give exactly the result of
the resident path, for pageable and page-locked host arrays, mixed with
GPUArray arguments, at chunk edges and with shard bases."""

import numpy as np
import pytest

from oracle import cport
from paper_0911_3456_b200 import driver as drv, elementwise as ew, ndarray as nd

pytestmark = pytest.mark.gpu

AXPY = ("float a, float *x, float b, float *y, float *z", "z[i] = a * x[i] + b * y[i]")


@pytest.mark.parametrize("pinned", [False, True])
@pytest.mark.parametrize("chunk", [None, 1 << 16, 99_999])
def test_axpy_host_in_out_equals_oracle(kernel_env, pinned, chunk):
    kwargs, pool = kernel_env
    n = 1_000_003
    rng = np.random.default_rng(3)
    if pinned:
        x, y, z = (nd.pinned_empty((n,), nd.float32) for _ in range(3))
        x[:] = rng.uniform(-1, 1, n)
        y[:] = rng.uniform(-1, 1, n)
    else:
        x = rng.uniform(-1, 1, n).astype(np.float32)
        y = rng.uniform(-1, 1, n).astype(np.float32)
        z = np.zeros(n, np.float32)
    k = ew.make_elementwise(*AXPY, "axpy_host", **kwargs)
    k._call_host((2.0, drv.In(x), -3.0, drv.In(y), drv.Out(z)), None, chunk=chunk) if chunk \
        else k(2.0, drv.In(x), -3.0, drv.In(y), drv.Out(z))
    want = np.zeros(n, np.float32)
    cport.Elementwise(*AXPY)(2.0, np.asarray(x), -3.0, np.asarray(y), want)
    assert np.array_equal(np.asarray(z), want)


def test_inout_mixed_with_device_arrays_and_global_index(kernel_env):
    kwargs, pool = kernel_env
    n = 300_001
    host = np.arange(n, dtype=np.int64)
    dev = nd.from_host(pool, nd.int64, np.full(n, 7, np.int64))
    k = ew.make_elementwise("long *h, long *d", "h[i] = h[i] * 2 + d[i] + i", "mix_host", **kwargs)
    k._call_host((drv.InOut(host), dev), None, chunk=65_536)
    assert np.array_equal(host, np.arange(n) * 3 + 7)


def test_explicit_n_and_errors(kernel_env):
    kwargs, pool = kernel_env
    k = ew.make_elementwise(*AXPY, "axpy_host_err", **kwargs)
    x = np.ones(1000, np.float32)
    z = np.zeros(1000, np.float32)
    k(1.0, drv.In(x), 1.0, drv.In(x), drv.Out(z), n=10)
    assert np.all(z[:10] == 2.0) and np.all(z[10:] == 0.0)
    with pytest.raises(ew.DtypeMismatch):
        k(1.0, drv.In(x.astype(np.float64)), 1.0, drv.In(x), drv.Out(z))
    with pytest.raises(ew.DtypeMismatch):
        k(drv.In(x), drv.In(x), 1.0, drv.In(x), drv.Out(z))
    with pytest.raises(nd.ShapeMismatch):
        k(1.0, drv.In(x), 1.0, drv.In(x[:5]), drv.Out(z))   # n = first vector's size
    with pytest.raises(ValueError):
        drv.Out(np.ones(4, np.float32)[::2])


def test_views_share_storage(kernel_env):
    kwargs, pool = kernel_env
    a = nd.from_host(pool, nd.int32, np.arange(100, dtype=np.int32))
    v = a[10:20]
    ew.make_elementwise("int *x", "x[i] = -x[i]", "neg_view", **kwargs)(v)
    got = a.get()
    assert np.array_equal(got[10:20], -np.arange(10, 20)) and got[9] == 9 and got[20] == 20
    assert np.array_equal((v + 1).get(), -np.arange(10, 20) + 1)
    with pytest.raises(ValueError):
        v.free()


def test_stream_objects_and_handles_are_accepted(kernel_env):
    from paper_0911_3456_b200 import _runtime, reduction as rd
    kwargs, pool = kernel_env
    st = _runtime.Stream()
    x = nd.from_host(pool, nd.float32, np.arange(1000, dtype=np.float32))
    z = pool.alloc(nd.float32, (1000,))
    k = ew.make_elementwise("float *x, float *z", "z[i] = x[i] + 1", "plus1_st", **kwargs)
    k(x, z, stream=st)
    k(x, z, stream=st.handle)
    st.synchronize()
    assert np.array_equal(z.get(), np.arange(1000) + 1)
    s = rd.sum_kernel(nd.float32, **kwargs)
    assert float(s(x, stream=st)) == float(np.arange(1000).sum())


@pytest.mark.parametrize("pinned", [False, True])
def test_reduction_over_host_inputs(kernel_env, pinned):
    """dot(driver.In(x), driver.In(y)): chunked uploads, one reduction per
    chunk, chunk accumulators folded in order -- within the fp64-accumulation
    bound of the resident result; integer sums exact."""
    from oracle import csem
    from paper_0911_3456_b200 import reduction as rd
    kwargs, pool = kernel_env
    n = 3_000_017
    rng = np.random.default_rng(9)
    if pinned:
        x, y = nd.pinned_empty((n,), nd.float32), nd.pinned_empty((n,), nd.float32)
        x[:] = rng.uniform(-1, 1, n)
        y[:] = rng.uniform(-1, 1, n)
    else:
        x = rng.uniform(-1, 1, n).astype(np.float32)
        y = rng.uniform(-1, 1, n).astype(np.float32)
    dot = rd.dot_kernel(nd.float32, **kwargs)
    got = float(dot(drv.In(x), drv.In(y)))
    terms = (np.asarray(x) * np.asarray(y)).astype(np.float64)
    assert abs(got - csem.exact_sum(terms)) <= csem.float_reduction_bound(terms, "float32")
    dev = dot(drv.In(x), drv.In(y), return_device=True)
    assert float(dev.get()) == got                       # deterministic chunk order
    ints = rng.integers(-(1 << 40), 1 << 40, n)
    s = rd.sum_kernel(nd.int64, **kwargs)
    assert int(s._call_host((drv.In(ints),), None, 0, False, chunk=123_457)) == int(ints.sum())
    assert int(s(drv.In(ints[:0]))) == 0                 # empty: the neutral
    with pytest.raises(ValueError):
        s(drv.Out(np.zeros(4, np.int64)))


def _slow_producer(kwargs):
    """Writes y[i] = i % 13 after a long dependent sinf chain per element, so
    the kernel is still running when the host call is issued."""
    return ew.make_elementwise(
        "float *y, int reps",
        "float v = 0.0f; for (int k = 0; k < reps; ++k) v = sinf(v + 1.0f); "
        "y[i] = (float) (i % 13) + (v > 10.0f ? 1.0f : 0.0f)", "slow_producer", **kwargs)


@pytest.mark.parametrize("user_stream", [False, True])
def test_streamed_call_waits_for_producer_on_callers_stream(kernel_env, user_stream):
    """the streamed call's private streams must start after the
    work already queued on the caller's stream (here: the kernel writing the
    device argument y)."""
    from paper_0911_3456_b200 import _runtime
    kwargs, pool = kernel_env
    n = 1 << 22
    x = np.arange(n, dtype=np.float32)
    z = np.zeros(n, np.float32)
    y = pool.alloc_uninitialized(nd.float32, (n,))
    prod = _slow_producer(kwargs)
    add = ew.make_elementwise("float *x, float *y, float *z", "z[i] = x[i] + y[i]",
                              "add_host", **kwargs)
    st = _runtime.Stream() if user_stream else None
    with _runtime.use_stream(st):
        prod(y, 3000)
        add(drv.In(x), y, drv.Out(z))
    want = x + (np.arange(n) % 13).astype(np.float32)
    assert np.array_equal(z, want)
    if st is not None:
        st.synchronize()
        st.close()
    y.free()


def test_streamed_reduction_waits_for_producer(kernel_env):
    from paper_0911_3456_b200 import _runtime
    from paper_0911_3456_b200 import reduction as rd
    kwargs, pool = kernel_env
    n = 1 << 22
    x = np.ones(n, np.int64)
    y = pool.alloc_uninitialized(nd.float32, (n,))
    prod = _slow_producer(kwargs)
    k = rd.make_reduction("int64_t *x, float *y", nd.int64, "0", "a + b",
                          "x[i] * (int64_t) y[i]", "dot_host_order", **kwargs)
    st = _runtime.Stream()
    with _runtime.use_stream(st):
        prod(y, 3000)
        got = k(drv.In(x), y)
    assert int(got) == int((np.arange(n) % 13).sum())
    st.close()
