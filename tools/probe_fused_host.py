import sys, time, cProfile, pstats
sys.path.insert(0, '/root/repo')
import numpy as np
from paper_0911_3456_b200 import _runtime as rt, ndarray as nd, fusion, elementwise as ew
rt.set_device(0)
pool = nd.MemoryPool(device=0)
x = nd.from_host(pool, nd.float32, np.ones(1 << 16, np.float32))
y = nd.from_host(pool, nd.float32, np.ones(1 << 16, np.float32))
z = pool.alloc(nd.float32, (1 << 16,))
chain = fusion.fused(lambda p, q: (p * 2 + q) - p)
add = ew.ElementwiseKernel("float *x, float *y, float *z", "z[i] = x[i] + y[i]", "add")
def eager():
    t1 = x * 2
    t2 = t1 + y
    t3 = t2 - x
    for t in (t1, t2, t3):
        t.free()
def fused():
    chain(x, y).free()
def direct():
    add(x, y, z)
for name, fn in (("direct", direct), ("fused", fused), ("eager", eager)):
    for _ in range(300): fn()
    rt.synchronize()
    t0 = time.perf_counter()
    for _ in range(3000): fn()
    rt.synchronize()
    print(name, "host us per call", round((time.perf_counter() - t0) / 3000 * 1e6, 2), flush=True)
for name, fn in (("fused", fused), ("eager", eager)):
    pr = cProfile.Profile(); pr.enable()
    for _ in range(3000): fn()
    pr.disable(); rt.synchronize()
    print("=====", name)
    pstats.Stats(pr).sort_stats('tottime').print_stats(12)
