"""Partition policy sweep at 2^28: grid-stride vs contiguous CTA ranges
(the reference worker formula) for dot and axpy over unroll x block x waves."""
import itertools, sys
sys.path.insert(0, "/root/repo")
import numpy as np
from paper_0911_3456_b200 import _runtime as rt, elementwise as ew, ndarray as nd, reduction as rd
def mean_ms(fn, reps=30):
    fn(); rt.synchronize(); s, e = rt.Event(), rt.Event(); s.record()
    for _ in range(reps): fn()
    e.record(); e.synchronize(); return s.elapsed_ms(e) / reps
rt.set_device(0); pool = nd.MemoryPool(device=0); n = 1 << 28
rng = np.random.default_rng(0)
x = nd.from_host(pool, nd.float32, rng.uniform(-1, 1, n).astype(np.float32))
y = nd.from_host(pool, nd.float32, rng.uniform(-1, 1, n).astype(np.float32))
z = pool.alloc_uninitialized(nd.float32, (n,)); o = pool.alloc_uninitialized(nd.float32, ())
res = []
for ch, u, b, w in itertools.product(("strided", "contiguous-blocks"), (1, 2, 4, 8), (128, 256, 512), (1, 2, 4)):
    v = ew.VariantParams(chunking=ch, unroll=u, block=b, waves=w)
    dot = rd.dot_kernel(nd.float32, v)
    axpy = ew.ElementwiseKernel("float a, float *x, float b, float *y, float *z", "z[i] = a * x[i] + b * y[i]", "axpy", v)
    res.append((ch, u, b, w, round(8 * n / mean_ms(lambda: dot.launch(x, y, out=o)) / 1e6), round(12 * n / mean_ms(lambda: axpy(2.0, x, -3.0, y, z)) / 1e6)))
for ch in ("strided", "contiguous-blocks"):
    r = [t for t in res if t[0] == ch]
    print(ch, "best dot", max(r, key=lambda t: t[4]), "best axpy", max(r, key=lambda t: t[5]))
