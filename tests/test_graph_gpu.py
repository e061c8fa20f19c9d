"""CUDA-graph capture and replay of generated kernels."""

import numpy as np
import pytest

from paper_0911_3456_b200 import _runtime, elementwise as ew, fusion, graph
from paper_0911_3456_b200 import ndarray as nd, reduction as rd

pytestmark = pytest.mark.gpu


def test_captured_chain_replays_like_eager_calls(pool, shared_cache):
    n = 1 << 16
    rng = np.random.default_rng(4)
    hx = rng.uniform(-1, 1, n).astype(np.float32)
    hy = rng.uniform(-1, 1, n).astype(np.float32)
    x, y = nd.from_host(pool, nd.float32, hx), nd.from_host(pool, nd.float32, hy)
    z = pool.alloc(nd.float32, (n,))
    w = pool.alloc(nd.float32, (n,))
    out = pool.alloc(nd.float32, ())
    axpy = ew.ElementwiseKernel("float a, float *x, float b, float *y, float *z",
                                "z[i] = a * x[i] + b * y[i]", "axpy", cache=shared_cache)
    chain = fusion.fused(lambda p, q: (p * 2 + q) - p)
    dot = rd.dot_kernel(nd.float32, cache=shared_cache)
    g = graph.Graph()
    with _runtime.use_stream(g.stream):      # warm up on the graph's stream
        axpy(2.0, x, -3.0, y, z)
        chain(z, y, out=w)
        dot.launch(w, w, out=out)
        g.synchronize()
    with g.capture():
        axpy(2.0, x, -3.0, y, z)
        chain(z, y, out=w)
        dot.launch(w, w, out=out)
    z.copy_from_host(np.zeros(n, np.float32))
    for _ in range(50):
        g.launch()
    g.synchronize()
    zz = np.float32(2.0) * hx + np.float32(-3.0) * hy
    ww = (zz * np.float32(2) + hy) - zz
    assert np.array_equal(z.get(), zz) and np.array_equal(w.get(), ww)
    want = float(np.float32(np.sum((ww * ww).astype(np.float64))))
    assert abs(float(out.get()) - want) <= 1e-6 * abs(want)
    # replay is cheaper than three Python-issued launches
    import time
    t0 = time.perf_counter()
    for _ in range(200):
        g.launch()
    g.synchronize()
    replay = (time.perf_counter() - t0) / 200
    with _runtime.use_stream(g.stream):
        t0 = time.perf_counter()
        for _ in range(200):
            axpy(2.0, x, -3.0, y, z)
            chain(z, y, out=w)
            dot.launch(w, w, out=out)
        g.synchronize()
    eager = (time.perf_counter() - t0) / 200
    assert replay < eager
    g.close()


def test_capture_rejects_legacy_stream():
    with pytest.raises(ValueError):
        graph.Graph(_runtime.Stream(handle=0))


def test_captured_overlapped_reductions(pool, shared_cache):
    """Overlapped (programmatic dependent) reduction launches inside a CUDA
    graph: captured as programmatic edges, replays give the eager results."""
    n = 1 << 20
    rng = np.random.default_rng(9)
    hx = rng.uniform(-1, 1, n).astype(np.float32)
    x = nd.from_host(pool, nd.float32, hx)
    outs = [pool.alloc(nd.float32, ()) for _ in range(3)]
    dot = rd.dot_kernel(nd.float32, cache=shared_cache)
    sq = rd.make_reduction("float *x", nd.float32, "0", "a > b ? a : b", "x[i] * x[i]",
                           "mx_g", cache=shared_cache)
    want = (float(dot(x, x)), float(sq(x)))
    g = graph.Graph()
    with _runtime.use_stream(g.stream):
        dot.launch(x, x, out=outs[0])
        sq.launch(x, out=outs[1])
        g.synchronize()
    with g.capture():
        dot.launch(x, x, out=outs[0], overlap_previous=True)
        sq.launch(x, out=outs[1], overlap_previous=True)
        dot.launch(x, x, out=outs[2], overlap_previous=True)
    for o in outs:
        o.copy_from_host(np.zeros((), np.float32))
    for _ in range(20):
        g.launch()
    g.synchronize()
    assert [float(o.get()) for o in outs] == [want[0], want[1], want[0]]
