"""Why are f64 streams slower than int64 streams of the same bytes?"""
import sys, math
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
from paper_0911_3456_b200 import _runtime as rt, elementwise as ew, ndarray as nd, reduction as rd

def dev_ms(fn, reps=8):
    fn(); rt.synchronize()
    s, e = rt.Event(), rt.Event(); best = math.inf
    for _ in range(reps):
        s.record(); fn(); e.record(); e.synchronize(); best = min(best, s.elapsed_ms(e))
    return best

rt.set_device(0)
pool = nd.MemoryPool(device=0)
n = 1 << 28
rng = np.random.default_rng(0)
hx = rng.uniform(-1, 1, n)
for dname, host in (("float64", hx), ("int64", (hx * 1e6).astype(np.int64)), ("uint64", (np.abs(hx) * 1e6).astype(np.uint64))):
    d = nd.BY_NAME[dname]; c = d.cname
    x = nd.from_host(pool, d, host); y = nd.from_host(pool, d, host[::-1].copy()); z = pool.alloc_uninitialized(d, (n,))
    for op in ("z[i] = x[i]", "z[i] = x[i] + y[i]", "z[i] = x[i] * y[i]"):
        for v in (ew.VariantParams(), ew.VariantParams(unroll=1, block=1024), ew.VariantParams(unroll=8, block=128)):
            k = ew.ElementwiseKernel(f"{c} *x, {c} *y, {c} *z", op, "k_" + dname, v)
            ms = dev_ms(lambda: k(x, y, z))
            nb = (2 if op == "z[i] = x[i]" else 3) * 8 * n
            print(f"{dname:8s} {op:22s} u={v.unroll} b={v.block:4d} {ms*1e3:8.1f} us {nb/ms/1e6:7.0f} GB/s", flush=True)
    s = rd.sum_kernel(d); o = pool.alloc_uninitialized(d, ())
    print(dname, "sum", round(8*n/dev_ms(lambda: s.launch(x, out=o))/1e6), "GB/s")
    for a in (x, y, z): a.free()
