"""One-read/one-write f64 streams at 2^28: copy, cubic polynomial, poly + sin,
over unroll x block x waves (LDG path) -- the ceiling a compute-heavy C3
expression should reach."""
import itertools
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402
from paper_0911_3456_b200 import _runtime as rt, elementwise as ew, ndarray as nd  # noqa: E402


def mean_ms(fn, reps=10):
    fn()
    rt.synchronize()
    s, e = rt.Event(), rt.Event()
    s.record()
    for _ in range(reps):
        fn()
    e.record()
    e.synchronize()
    return s.elapsed_ms(e) / reps


import os  # noqa: E402
from paper_0911_3456_b200 import _codegen as cg  # noqa: E402
if os.environ.get("TMA_STAGE_BYTES"):
    cg.TMA_STAGE_BYTES = int(os.environ["TMA_STAGE_BYTES"])
rt.set_device(0)
pool = nd.MemoryPool(device=0)
n = 1 << 28
x = nd.from_host(pool, nd.float64, np.random.default_rng(1).uniform(-2, 2, n))
z = pool.alloc_uninitialized(nd.float64, (n,))
ops = {"copy": "z[i] = x[i]", "poly": "z[i] = ((a*x[i] + 2.0)*x[i] - 1.5)*x[i]",
       "polysin": "z[i] = ((a*x[i] + 2.0)*x[i] - 1.5)*x[i] + sin(x[i])"}
only = [a for a in sys.argv[1:] if not a.startswith("--")] or list(ops)
caches = ("tma",) if "--tma-only" in sys.argv else \
    ("default", "tma") if "--tma" in sys.argv else ("default",)
rows = []
for name in [o for o in ops if o in only]:
    op = ops[name]
    prefetches = (False, True) if "--prefetch" in sys.argv else (False,)
    for u, b, w, c, pf in itertools.product((1, 2, 4), (128, 256, 512, 1024), (0, 1, 2, 4),
                                            caches, prefetches):
        if pf and w == 0:
            continue              # one step per thread: nothing to prefetch
        try:
            k = ew.ElementwiseKernel("double a, double *x, double *z", op, "k_" + name,
                                     ew.VariantParams(unroll=u, block=b, waves=w, cache=c,
                                                      prefetch=pf))
        except Exception as exc:  # noqa: BLE001
            print(name, u, b, w, c, "build failed", str(exc)[:200], file=sys.stderr)
            continue
        ms = mean_ms(lambda: k(0.5, x, z))
        rows.append({"op": name, "unroll": u, "block": b, "waves": w, "cache": c,
                     "prefetch": pf,
                     "GB/s": round(16 * n / ms / 1e6)})
    best = sorted((r for r in rows if r["op"] == name), key=lambda r: -r["GB/s"])[:5]
    for r in best:
        print(json.dumps(r), flush=True)
Path("gpurun_out").mkdir(exist_ok=True)
Path(f"gpurun_out/sweep_copylike{os.environ.get('TMA_STAGE_BYTES', '')}.json").write_text(json.dumps(rows, indent=1))
