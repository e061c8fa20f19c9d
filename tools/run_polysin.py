"""C3 kernel alone (for ncu): f64 z = ((a x + 2) x - 1.5) x + sin x at 2^28,
variant from argv (unroll block waves), 3 launches."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402
from paper_0911_3456_b200 import _runtime as rt, elementwise as ew, ndarray as nd  # noqa: E402

u, b, w = (int(v) for v in (sys.argv[1:4] if len(sys.argv) >= 4 else (1, 1024, 1)))
op = sys.argv[4] if len(sys.argv) > 4 else "z[i] = ((a*x[i] + 2.0)*x[i] - 1.5)*x[i] + sin(x[i])"
rt.set_device(0)
pool = nd.MemoryPool(device=0)
n = 1 << 28
x = nd.from_host(pool, nd.float64, np.random.default_rng(1).uniform(-2, 2, n))
z = pool.alloc_uninitialized(nd.float64, (n,))
k = ew.ElementwiseKernel("double a, double *x, double *z", op, "polysin",
                         ew.VariantParams(unroll=u, block=b, waves=w))
for _ in range(3):
    k(0.5, x, z)
rt.synchronize()
s, e = rt.Event(), rt.Event()
s.record()
for _ in range(10):
    k(0.5, x, z)
e.record()
e.synchronize()
ms = s.elapsed_ms(e) / 10
print(f"polysin u={u} b={b} w={w}: {ms * 1e3:.1f} us  {16 * n / ms / 1e6:.0f} GB/s")
