"""One-step-per-thread elementwise kernels (waves 0): device time of axpy f32
and x + y over dtypes at 2^28, several blocks/unrolls; 10-launch bursts,
best of 3.  Compare with the same variants at waves 1 (grid-stride)."""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402
from paper_0911_3456_b200 import _runtime as rt, elementwise as ew, ndarray as nd  # noqa: E402

rt.set_device(0)
pool = nd.MemoryPool(device=0)
N = 1 << 28


def best_ms(fn, burst=10, reps=3):
    fn()
    rt.synchronize()
    s, e = rt.Event(), rt.Event()
    best = float("inf")
    for _ in range(reps):
        s.record()
        for _ in range(burst):
            fn()
        e.record()
        e.synchronize()
        best = min(best, s.elapsed_ms(e) / burst)
    return best


rows = []
for dname in ("float32", "float64", "int32"):
    d = nd.BY_NAME[dname]
    c = d.cname
    x = pool.alloc(d, (N,))
    y = pool.alloc(d, (N,))
    z = pool.alloc_uninitialized(d, (N,))
    sig = f"{c} a, {c} *x, {c} b, {c} *y, {c} *z"
    for op_name, op in (("axpy", "z[i] = a * x[i] + b * y[i]"), ("add", "z[i] = x[i] + y[i]")):
        for block, unroll, waves in ((128, 1, 0), (256, 1, 0), (512, 2, 0), (128, 1, 1),
                                     (256, 2, 2)):
            k = ew.ElementwiseKernel(sig, op, f"{op_name}_{dname}",
                                     ew.VariantParams(block=block, unroll=unroll, waves=waves))
            ms = best_ms(lambda: k(2, x, 3, y, z))
            row = {"op": op_name, "dtype": dname, "block": block, "unroll": unroll,
                   "waves": waves, "GB/s": round(3 * d.size * N / ms / 1e6, 1)}
            rows.append(row)
            print(json.dumps(row), flush=True)
    for a in (x, y, z):
        a.free()
Path("gpurun_out").mkdir(exist_ok=True)
Path("gpurun_out/probe_one_step.json").write_text(json.dumps(rows, indent=1))
