"""Quick end-to-end probe on a GPU box: correctness + rough bandwidth."""
import sys, time
import numpy as np
sys.path.insert(0, ".")
from paper_0911_3456_b200 import _runtime as rt, elementwise as ew, reduction as rd, ndarray as nd, jit

print("gpu", rt.have_gpu(), rt.device_info(0))
pool = nd.default_pool()
rng = np.random.default_rng(0)
for n in (0, 1, 7, 1000, 1 << 20):
    x = rng.uniform(-1, 1, n).astype(np.float32); y = rng.uniform(-1, 1, n).astype(np.float32)
    gx, gy = nd.from_host(pool, nd.float32, x), nd.from_host(pool, nd.float32, y)
    gz = pool.alloc(nd.float32, (n,))
    k = ew.make_elementwise("float a, float *x, float b, float *y, float *z", "z[i] = a*x[i] + b*y[i]", "axpy")
    k(2.0, gx, -3.0, gy, gz)
    ref = np.float32(2.0) * x + np.float32(-3.0) * y
    print("axpy", n, np.array_equal(gz.to_host(), ref), k.launch_config(2.0, gx, -3.0, gy, gz) if n else "")
    d = rd.dot_kernel(nd.float32)
    got = d(gx, gy)
    exact = np.float32(np.sum((x * y).astype(np.float64)))
    print("dot", n, got, exact, got == exact)
for dt in (nd.int8, nd.int32, nd.int64, nd.uint16, nd.float64):
    h = rng.integers(-100, 100, 10001).astype(dt.np) if dt.kind != "f" else rng.uniform(-1, 1, 10001)
    g = nd.from_host(pool, dt, h)
    print(dt.name, "sum", rd.sum_kernel(dt)(g), h.sum(dtype=h.dtype) if dt.kind != "f" else h.sum(), "max", rd.max_kernel(dt)(g), h.max(), "min", rd.min_kernel(dt)(g), h.min())

def bench(fn, reps=20):
    e0, e1 = rt.Event(), rt.Event()
    fn(); rt.synchronize()
    best = 1e9
    for _ in range(reps):
        e0.record(); fn(); e1.record(); e1.synchronize()
        best = min(best, e0.elapsed_ms(e1))
    return best

n = 1 << 28
gx = nd.from_host(pool, nd.float32, rng.uniform(-1, 1, n).astype(np.float32))
gy = nd.from_host(pool, nd.float32, rng.uniform(-1, 1, n).astype(np.float32))
gz = pool.alloc(nd.float32, (n,))
for u in (1, 2, 4, 8):
    for blk in (128, 256, 512):
        for ch in ("contiguous-blocks", "strided"):
            v = ew.VariantParams(unroll=u, block=blk, chunking=ch)
            k = ew.make_elementwise("float a, float *x, float b, float *y, float *z", "z[i] = a*x[i] + b*y[i]", "axpy", v)
            ms = bench(lambda: k(2.0, gx, -3.0, gy, gz))
            d = rd.dot_kernel(nd.float32, v)
            ms2 = bench(lambda: d(gx, gy, return_device=True))
            print(f"u={u} b={blk} {ch:18s} axpy {ms*1e3:7.1f} us {12*n/ms/1e6:7.0f} GB/s | dot {ms2*1e3:7.1f} us {8*n/ms2/1e6:7.0f} GB/s grid={k.launch_config(2.0, gx, -3.0, gy, gz)['grid']}")
