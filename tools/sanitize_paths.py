"""Exercise every kernel-template path once at small sizes (for compute-sanitizer).

Paths: elementwise vector / general (neighbour access, aliasing, misaligned),
head/tail splits, contiguous + strided partitions, full-grid and resident
waves; reductions vector / general / TMA / combine / empty span / multi-CTA
last-block fold; fused chains and fused chain+reduction; a captured graph;
elementwise TMA rings (read, read-write, mixed widths, tile edges); the
cross-rank peer exchange with emulated ranks on their own streams; views and
streamed host calls (driver.In/Out); per-thread cp.async rings.
"""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
from paper_0911_3456_b200 import _runtime as rt, elementwise as ew, fusion, graph
from paper_0911_3456_b200 import ndarray as nd, reduction as rd

rt.set_device(0)
pool = nd.MemoryPool(device=0)
rng = np.random.default_rng(0)
checks = 0
for n in (1, 5, 37, 1000, 65_539):
    hx = rng.uniform(-1, 1, n + 1).astype(np.float32)
    hy = rng.uniform(-1, 1, n + 1).astype(np.float32)
    x, y = nd.from_host(pool, nd.float32, hx), nd.from_host(pool, nd.float32, hy)
    z = pool.alloc(nd.float32, (n + 1,))
    for v in (ew.VariantParams(), ew.VariantParams(unroll=4, block=64, waves=1,
                                                  chunking="contiguous-blocks"),
              ew.VariantParams(unroll=16, block=1024, waves=2),
              ew.VariantParams(unroll=2, block=64, workers=3, prefetch=True)):
        ew.ElementwiseKernel("float a, float *x, float b, float *y, float *z",
                             "z[i] = a * x[i] + b * y[i]", "axpy", v)(2.0, x, -3.0, y, z, n=n)
        ew.ElementwiseKernel("float *x, float *z", "z[i] = x[i + 1] - x[i]", "nb", v)(x, z, n=n)
        ew.ElementwiseKernel("float *x, float *z", "if (x[i] > 0) z[i] = x[i]", "cw", v)(x, z, n=n)
        ew.ElementwiseKernel("float *x, float *z", "z[i] = 2 * x[i]", "al", v)(x, x, n=n)
        for cache in ("default", "tma"):
            rv = ew.VariantParams(unroll=v.unroll, block=max(64, v.block), waves=v.waves,
                                  chunking=v.chunking, cache=cache, workers=v.workers,
                                  prefetch=v.prefetch)
            float(rd.dot_kernel(nd.float32, rv)(x, y, n=n))
            float(rd.make_reduction("float *x", nd.float32, "0", "a + b", "x[i+1] - x[i]",
                                    name="tv", variant=rv)(x, n=n))
            checks += 2
    zm = pool.alloc(nd.float32, (n + 3,))         # misaligned views are not expressible;
    ew.ElementwiseKernel("float *z", "z[i] = (float) i", "iota")(zm, n=n, base=3)  # base offset
    fusion.fused(lambda p, q: (p * 2 + q) - p)(x, y)
    checks += 6
float(rd.sum_kernel(nd.float64)(pool.alloc(nd.float64, (0,))))     # empty span -> combine
# elementwise TMA rings
from paper_0911_3456_b200 import driver as drv, parallel as par  # noqa: E402
for n in (1, 37, 20_000, 100_003):
    a = nd.from_host(pool, nd.float64, rng.uniform(-2, 2, n))
    b8 = nd.from_host(pool, nd.int8, rng.integers(-9, 9, n).astype(np.int8))
    c = pool.alloc(nd.float64, (n,))
    for blk, wk in ((64, None), (256, None), (1024, None), (128, 2)):   # workers=2: ring wraps
        tv = ew.VariantParams(cache="tma", block=blk, workers=wk)
        ew.ElementwiseKernel("double *x, double *z", "z[i] = x[i] * 2 + sin(x[i])", "tps", tv)(a, c)
        ew.ElementwiseKernel("double *x, double *z", "z[i] += x[i]", "trw", tv)(a, c)
        ew.ElementwiseKernel("int8_t *b, double *x, double *z", "z[i] = b[i] * x[i]", "tmx",
                             tv)(b8, a, c)
        checks += 3
    fusion.reduce(fusion.lazy(a) * 2 - a, "sum").get()
    a[n // 3:n // 2 + 1] * 2.0
    checks += 2
# per-thread cp.async rings (stages): read-only, read-write, mixed widths,
# unaligned heads/tails, grids shorter than the ring, shard bases
for n in (1, 5, 37, 20_000, 100_003):
    a = nd.from_host(pool, nd.float64, rng.uniform(-2, 2, n + 3))
    f32 = nd.from_host(pool, nd.float32, rng.uniform(-1, 1, n + 3).astype(np.float32))
    c = nd.from_host(pool, nd.float64, rng.uniform(-1, 1, n + 3))
    for st, un, blk, wk in ((2, 1, 128, None), (3, 2, 256, None), (8, 4, 64, 2), (4, 1, 512, 1)):
        rv = ew.VariantParams(stages=st, unroll=un, block=blk, waves=1, workers=wk)
        ew.ElementwiseKernel("double a, double *x, double *z",
                             "z[i] = ((a*x[i] + 2.0)*x[i] - 1.5)*x[i] + sin(x[i])", "rps", rv)(
                                 0.5, a[1:], c[1:], base=5)
        ew.ElementwiseKernel("float *x, double *y, double *z", "z[i] += x[i] * y[i]", "rmx", rv)(
            f32, a, c, n=n)
        checks += 2
# peer exchange, 3 emulated ranks on their own streams (needs the ranks'
# kernels to run concurrently: initcheck serialises launches, so it skips this)
EXCHANGE = "--no-exchange" not in sys.argv
xs = rng.integers(-100, 100, 90_001).astype(np.int64)
group = par.PeerMailbox.local_group(3)
streams = [rt.Stream() for _ in range(3)] if EXCHANGE else []
ks = rd.sum_kernel(nd.int64)
parts = [nd.from_host(pool, nd.int64, xs[r * 30_000:(r + 1) * 30_000 + (r == 2)])
         for r in range(3)]
for _ in range(3 if EXCHANGE else 0):
    for r in range(3):
        with rt.use_stream(streams[r].handle):
            ks.launch(parts[r], base=r * 30_000, peers=group[r])
for st in streams:
    st.synchronize()
assert all(int(ks._read(ks.scratch(0, st.handle).result, nd.int64)) == int(xs.sum())
           for st in streams)
checks += 9 if EXCHANGE else 0
# a peer that never arrives: soft timeout, poisoned result, error word reported once
lone = par.PeerMailbox.local_group(2, timeout_s=0.2)
ks.launch(parts[0], peers=lone[0], out=pool.alloc(nd.int64, ()))
try:
    lone[0].check()
    raise AssertionError("the missing peer was not reported")
except par.PeerTimeout:
    pass
lone[0].check()
checks += 1
# overlapped (programmatic dependent) reductions back to back
ov = rd.dot_kernel(nd.float32)
oo = pool.alloc(nd.float32, ())
big_x = nd.from_host(pool, nd.float32, rng.uniform(-1, 1, 200_003).astype(np.float32))
for _ in range(6):
    ov.launch(big_x, big_x, out=oo, overlap_previous=True)
assert abs(float(oo.get()) - float(ov(big_x, big_x))) == 0
checks += 6
# streamed host call
hx = rng.uniform(-1, 1, 300_001).astype(np.float32)
hz = np.zeros_like(hx)
axs = ew.ElementwiseKernel("float *x, float *z", "z[i] = x[i] * 3", "hs")
axs._call_host((drv.In(hx), drv.Out(hz)), None, chunk=65_536)
assert np.array_equal(hz, hx * np.float32(3))
checks += 5
g = graph.Graph()
big = nd.from_host(pool, nd.int64, np.arange(1 << 20, dtype=np.int64))
o = pool.alloc(nd.int64, ())
k = rd.sum_kernel(nd.int64)
with rt.use_stream(g.stream):
    k.launch(big, out=o)
    g.synchronize()
with g.capture():
    k.launch(big, out=o)
g.launch()
g.synchronize()
assert int(o.get()) == (1 << 20) * ((1 << 20) - 1) // 2
# the prelude's sin / cos (coefficient-table loads, the out-of-line library
# call for |x| >= 2^31, inf and NaN) through vector, prefetch and ring entries
# and a reduction map
trig_x = np.concatenate([rng.uniform(-4, 4, 5001), [0.0, -0.0, 2.0**31, -1e300, np.inf, np.nan]])
tx = nd.from_host(pool, nd.float64, trig_x)
tz = pool.alloc(nd.float64, trig_x.shape)
for v in (ew.VariantParams(), ew.VariantParams(block=128, waves=4, prefetch=True),
          ew.VariantParams(block=256, unroll=2, waves=2, stages=2)):
    ew.ElementwiseKernel("double *x, double *z", "z[i] = sin(x[i]) + cos(x[i])", "trig", v)(tx, tz)
    checks += 1
want = np.sin(trig_x[:5001]) + np.cos(trig_x[:5001])
assert np.allclose(tz.get()[:5001], want, rtol=0, atol=1e-14)
rd.make_reduction("double *x", nd.float64, "0", "a + b", "sin(x[i])", "sum_sin")(tx[:5001])
checks += 1
# dynamic chunk scheduling (VariantParams.chunk): tiny / ragged spans, a
# base offset, overlapped launches alternating the slots' counters
for n in (1, 4099, 100_003, 1 << 20):
    hx = rng.uniform(-1, 1, n).astype(np.float32)
    gx = nd.from_host(pool, nd.float32, hx)
    for dv in (ew.VariantParams(chunk=1024), ew.VariantParams(unroll=4, block=128, chunk=4096,
                                                              workers=3)):
        dk = rd.dot_kernel(nd.float32, dv)
        want = float(dk(gx, gx))
        od = pool.alloc_uninitialized(nd.float32, ())
        for _ in range(3):
            dk.launch(gx, gx, out=od, overlap_previous=True)
        assert float(od.get()) == want
        checks += 4
xi = nd.from_host(pool, nd.int64, rng.integers(-(1 << 40), 1 << 40, 300_000, dtype=np.int64))
oi = pool.alloc_uninitialized(nd.int64, ())
rd.sum_kernel(nd.int64, ew.VariantParams(chunk=2048)).launch(xi[4096:], n=200_000, base=4096,
                                                              out=oi)
assert int(oi.get()) == int(xi.get()[4096:204_096].sum())
checks += 1
rt.synchronize()
print(f"sanitize paths ok ({checks} launches checked)")
