"""Which untuned default variant is robust across dtypes and kernel kinds?"""
import itertools, json, math, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
from paper_0911_3456_b200 import _runtime as rt, elementwise as ew, ndarray as nd, reduction as rd

def dev_ms(fn, reps=6):
    fn(); rt.synchronize()
    s, e = rt.Event(), rt.Event(); best = math.inf
    for _ in range(reps):
        s.record(); fn(); e.record(); e.synchronize(); best = min(best, s.elapsed_ms(e))
    return best

rt.set_device(0)
pool = nd.MemoryPool(device=0)
N = 1 << 28
cands = [(1, 128), (1, 256), (1, 512), (2, 128), (2, 256), (4, 128), (4, 256)]
table = {}
for dname in ("float32", "float64", "int32", "int64", "int8", "int16"):
    d = nd.BY_NAME[dname]; c = d.cname
    fill = ew.ElementwiseKernel(f"{c} *x", f"x[i] = ({c}) (i % 100)", f"f_{dname}")
    x = pool.alloc_uninitialized(d, (N,)); y = pool.alloc_uninitialized(d, (N,)); z = pool.alloc_uninitialized(d, (N,))
    fill(x); fill(y)
    o = pool.alloc_uninitialized(d, ())
    for u, b in cands:
        v = ew.VariantParams(unroll=u, block=b)
        add = ew.ElementwiseKernel(f"{c} *x, {c} *y, {c} *z", "z[i] = x[i] + y[i]", f"a_{dname}", v)
        dot = rd.dot_kernel(d, v); sm = rd.sum_kernel(d, v)
        r = {"add": 3 * d.size * N / dev_ms(lambda: add(x, y, z)) / 1e6,
             "dot": 2 * d.size * N / dev_ms(lambda: dot.launch(x, y, out=o)) / 1e6,
             "sum": d.size * N / dev_ms(lambda: sm.launch(x, out=o)) / 1e6}
        table.setdefault(f"u{u}b{b}", {})[dname] = {k: round(vv) for k, vv in r.items()}
        print(dname, u, b, {k: round(vv) for k, vv in r.items()}, flush=True)
    for a in (x, y, z, o): a.free()
    pool.release_free()
worst = {k: min(min(vv.values()) for vv in v.values()) for k, v in table.items()}
mean = {k: sum(sum(vv.values()) for vv in v.values()) / (3 * len(v)) for k, v in table.items()}
print("worst-case GB/s per candidate:", json.dumps(worst))
print("mean GB/s per candidate:", json.dumps({k: round(v) for k, v in mean.items()}))
Path("gpurun_out/sweep_defaults.json").write_text(json.dumps(table, indent=1))
