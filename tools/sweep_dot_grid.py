"""Fine grid-size sweep for the headline dot (2^28 f32): waves 1..8 and explicit CTA counts."""
import itertools, json, math, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
from paper_0911_3456_b200 import _runtime as rt, elementwise as ew, ndarray as nd, reduction as rd

def dev_ms(fn, reps=30):
    fn(); rt.synchronize()
    evs = [rt.Event() for _ in range(reps + 1)]
    evs[0].record()
    for j in range(reps):
        fn(); evs[j + 1].record()
    evs[-1].synchronize()
    return evs[0].elapsed_ms(evs[-1]) / reps   # back-to-back mean, like bench.py

rt.set_device(0)
pool = nd.MemoryPool(device=0)
N = 1 << 28
rng = np.random.default_rng(0)
x = nd.from_host(pool, nd.float32, rng.uniform(-1, 1, N).astype(np.float32))
y = nd.from_host(pool, nd.float32, rng.uniform(-1, 1, N).astype(np.float32))
o = pool.alloc_uninitialized(nd.float32, ())
rows = []
for u, b in itertools.product((1, 2, 4, 8, 16), (128, 256, 512, 1024)):
    base = rd.dot_kernel(nd.float32, ew.VariantParams(unroll=u, block=b))
    for w in (1, 2, 4, 8):
        k = rd.dot_kernel(nd.float32, ew.VariantParams(unroll=u, block=b, waves=w))
        ms = dev_ms(lambda: k.launch(x, y, out=o))
        rows.append({"unroll": u, "block": b, "waves": w, "grid": k.launch_config(x, y)["grid"],
                     "us": round(ms * 1e3, 1), "GB/s": round(8 * N / ms / 1e6)})
    for g in (148, 296, 444, 592, 740, 888, 1184, 1776, 2368):
        k = rd.dot_kernel(nd.float32, ew.VariantParams(unroll=u, block=b, workers=g))
        ms = dev_ms(lambda: k.launch(x, y, out=o))
        rows.append({"unroll": u, "block": b, "workers": g, "us": round(ms * 1e3, 1),
                     "GB/s": round(8 * N / ms / 1e6)})
rows.sort(key=lambda r: r["us"])
for r in rows[:12]:
    print(json.dumps(r))
Path("gpurun_out/sweep_dot_grid.json").write_text(json.dumps(rows, indent=1))
