"""Load-policy sweep at 2^28 (dot f32, axpy f32, sum f32): default (LDG.128
.CONSTANT), no-l1, l2-256 (LDG.E.LTC256B: 256-byte L2 prefetch), l2-256-no-l1,
streaming, x unroll x block x waves; mean of 20 back-to-back launches."""
import itertools
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402
from paper_0911_3456_b200 import _runtime as rt, elementwise as ew, ndarray as nd  # noqa: E402
from paper_0911_3456_b200 import reduction as rd  # noqa: E402


def mean_ms(fn, reps=20):
    fn()
    rt.synchronize()
    s, e = rt.Event(), rt.Event()
    s.record()
    for _ in range(reps):
        fn()
    e.record()
    e.synchronize()
    return s.elapsed_ms(e) / reps


rt.set_device(0)
pool = nd.MemoryPool(device=0)
n = 1 << 28
rng = np.random.default_rng(0)
x = nd.from_host(pool, nd.float32, rng.uniform(-1, 1, n).astype(np.float32))
y = nd.from_host(pool, nd.float32, rng.uniform(-1, 1, n).astype(np.float32))
z = pool.alloc_uninitialized(nd.float32, (n,))
o = pool.alloc_uninitialized(nd.float32, ())
caches = ("default", "no-l1", "l2-256", "l2-256-no-l1", "streaming")
rows = []
for c, u, b, w in itertools.product(caches, (1, 2, 4, 8), (128, 256, 512), (0, 1, 2)):
    v = ew.VariantParams(cache=c, unroll=u, block=b, waves=w)
    dot = rd.dot_kernel(nd.float32, v)
    sm = rd.sum_kernel(nd.float32, v)
    axpy = ew.ElementwiseKernel("float a, float *x, float b, float *y, float *z",
                                "z[i] = a * x[i] + b * y[i]", "axpy", v)
    rows.append({"cache": c, "unroll": u, "block": b, "waves": w,
                 "dot": round(8 * n / mean_ms(lambda: dot.launch(x, y, out=o)) / 1e6),
                 "sum": round(4 * n / mean_ms(lambda: sm.launch(x, out=o)) / 1e6),
                 "axpy": round(12 * n / mean_ms(lambda: axpy(2.0, x, -3.0, y, z)) / 1e6)})
for k in ("dot", "sum", "axpy"):
    for c in caches:
        best = max((r for r in rows if r["cache"] == c), key=lambda r: r[k])
        print(k, c, best[k], {q: best[q] for q in ("unroll", "block", "waves")}, flush=True)
Path("gpurun_out").mkdir(exist_ok=True)
Path("gpurun_out/sweep_cache.json").write_text(json.dumps(rows, indent=1))
