"""Grid-policy sweep: waves x unroll x block for copy / axpy / dot / f64 add."""
import itertools, json, math, sys
from concurrent.futures import ThreadPoolExecutor
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
N = 1 << 28
rng = np.random.default_rng(0)
x = nd.from_host(pool, nd.float32, rng.uniform(-1, 1, N).astype(np.float32))
y = nd.from_host(pool, nd.float32, rng.uniform(-1, 1, N).astype(np.float32))
z = pool.alloc_uninitialized(nd.float32, (N,))
o = pool.alloc_uninitialized(nd.float32, ())
xd = nd.from_host(pool, nd.float64, rng.uniform(-1, 1, N))
yd = nd.from_host(pool, nd.float64, rng.uniform(-1, 1, N))
zd = pool.alloc_uninitialized(nd.float64, (N,))
cases = {
    "copy_f32": (lambda v: ew.ElementwiseKernel("float *x, float *z", "z[i] = x[i]", "cp32", v), lambda k: k(x, z), 8 * N),
    "axpy_f32": (lambda v: ew.ElementwiseKernel("float a, float *x, float b, float *y, float *z", "z[i] = a * x[i] + b * y[i]", "axpy", v), lambda k: k(2.0, x, -3.0, y, z), 12 * N),
    "add_f64": (lambda v: ew.ElementwiseKernel("double *x, double *y, double *z", "z[i] = x[i] + y[i]", "add64", v), lambda k: k(xd, yd, zd), 24 * N),
    "dot_f32": (lambda v: rd.dot_kernel(nd.float32, v), lambda k: k.launch(x, y, out=o), 8 * N),
}
out = {}
for name, (make, call, nbytes) in cases.items():
    combos = list(itertools.product((1, 2, 4, 8), (128, 256, 512, 1024)))
    with ThreadPoolExecutor(8) as ex:
        list(ex.map(lambda c: make(ew.VariantParams(unroll=c[0], block=c[1])), combos))
    rows = []
    for (u, b), w in itertools.product(combos, (0, 1, 2, 4)):
        k = make(ew.VariantParams(unroll=u, block=b, waves=w))
        ms = dev_ms(lambda: call(k))
        rows.append({"unroll": u, "block": b, "waves": w, "us": round(ms * 1e3, 1), "GB/s": round(nbytes / ms / 1e6)})
    rows.sort(key=lambda r: r["us"])
    out[name] = rows
    print(name, json.dumps(rows[:6]), flush=True)
    by_w = {w: max(r["GB/s"] for r in rows if r["waves"] == w) for w in (0, 1, 2, 4)}
    print("   best per waves:", by_w, flush=True)
Path("gpurun_out").mkdir(exist_ok=True)
Path("gpurun_out/sweep_waves.json").write_text(json.dumps(out, indent=1))
