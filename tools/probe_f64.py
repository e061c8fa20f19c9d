"""Why are some f64 streams slower than int64 streams of the same bytes?

Same kernels (copy / add / sum at 2^28 elements), same variant, different
data sources: host-uniform doubles, the C5 sweep's device fill pattern,
integers, random 64-bit patterns.  Timed two ways: best of 5 single launches
and the mean of 20 back-to-back launches."""
import json
import math
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402
from paper_0911_3456_b200 import _runtime as rt, elementwise as ew, ndarray as nd  # noqa: E402
from paper_0911_3456_b200 import reduction as rd  # noqa: E402


def best_ms(fn, reps=5):
    fn()
    rt.synchronize()
    s, e = rt.Event(), rt.Event()
    best = math.inf
    for _ in range(reps):
        s.record()
        fn()
        e.record()
        e.synchronize()
        best = min(best, s.elapsed_ms(e))
    return best


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
fill = {c: ew.ElementwiseKernel(f"long seed, {c} *x",
                                f"x[i] = ({c}) ((long) (((unsigned long) i * 2654435761UL + seed) % 2001)"
                                f" - 1000) / ({c}) {'1000.0' if c == 'double' else '1'}",
                                f"fill_{c}") for c in ("double", "long")}
hu = rng.uniform(-1, 1, n)
sources = {
    "f64_host_uniform": (nd.float64, lambda: hu, None),
    "f64_fill_pattern": (nd.float64, None, 1),
    "f64_zeros": (nd.float64, lambda: np.zeros(n), None),
    "f64_host_int_valued": (nd.float64, lambda: np.round(hu * 1000.0), None),
    "i64_fill_pattern": (nd.int64, None, 1),
    "i64_random_bits": (nd.int64, lambda: rng.integers(-2**62, 2**62, n), None),
    "i64_from_f64_bits": (nd.int64, lambda: hu.view(np.int64), None),
}
rows = []
for name, (d, host, seed) in sources.items():
    c = d.cname
    if host is not None:
        x = nd.from_host(pool, d, host())
        y = nd.from_host(pool, d, host()[::-1].copy())
    else:
        x = pool.alloc_uninitialized(d, (n,))
        y = pool.alloc_uninitialized(d, (n,))
        fill["double" if d.kind == "f" else "long"](seed, x)
        fill["double" if d.kind == "f" else "long"](seed + 6, y)
    z = pool.alloc_uninitialized(d, (n,))
    o = pool.alloc_uninitialized(d, ())
    cp = ew.ElementwiseKernel(f"{c} *x, {c} *z", "z[i] = x[i]", f"cp_{c}")
    add = ew.ElementwiseKernel(f"{c} *x, {c} *y, {c} *z", "z[i] = x[i] + y[i]", f"add_{c}")
    sm = rd.sum_kernel(d)
    row = {"data": name}
    for kname, fn, nb in (("copy", lambda: cp(x, z), 16 * n), ("add", lambda: add(x, y, z), 24 * n),
                          ("sum", lambda: sm.launch(x, out=o), 8 * n)):
        row[kname + "_best5"] = round(nb / best_ms(fn) / 1e6)
        row[kname + "_mean20"] = round(nb / mean_ms(fn) / 1e6)
    rows.append(row)
    print(json.dumps(row), flush=True)
    for a in (x, y, z, o):
        a.free()
    pool.release_free()
Path("gpurun_out").mkdir(exist_ok=True)
Path("gpurun_out/probe_f64.json").write_text(json.dumps(rows, indent=1))
