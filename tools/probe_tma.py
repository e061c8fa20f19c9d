"""TMA-staged reductions vs the LDG.128 vector path (dot f32, sum i64, max|x|)."""
import itertools, json, math, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
from paper_0911_3456_b200 import _runtime as rt, elementwise as ew, ndarray as nd, reduction as rd

def dev_ms(fn, reps=10):
    fn(); rt.synchronize()
    s, e = rt.Event(), rt.Event(); best = math.inf
    for _ in range(reps):
        s.record(); fn(); e.record(); e.synchronize(); best = min(best, s.elapsed_ms(e))
    return best

rt.set_device(0)
pool = nd.MemoryPool(device=0)
N = 1 << 28
rng = np.random.default_rng(0)
hx = rng.uniform(-1, 1, N).astype(np.float32); hy = rng.uniform(-1, 1, N).astype(np.float32)
x, y = nd.from_host(pool, nd.float32, hx), nd.from_host(pool, nd.float32, hy)
o = pool.alloc_uninitialized(nd.float32, ())
want = float(np.float32(np.dot(hx.astype(np.float64), hy.astype(np.float64))))
rows = []
for cache, block, waves in itertools.chain(
        itertools.product(["tma"], [128, 256, 512, 1024], [1, 2]),
        [("default", 512, 1), ("default", 128, 1), ("default", 256, 2)]):
    v = ew.VariantParams(cache=cache, block=block, waves=waves, unroll=8 if cache == "default" else 4)
    k = rd.dot_kernel(nd.float32, v)
    ms = dev_ms(lambda: k.launch(x, y, out=o))
    got = float(k(x, y))
    cfg = k.launch_config(x, y)
    rows.append({"cache": cache, "block": block, "waves": waves, "us": round(ms * 1e3, 1),
                 "GB/s": round(8 * N / ms / 1e6), "grid": cfg["grid"], "smem": cfg["smem"],
                 "rel_err": abs(got - want) / abs(want)})
    print(json.dumps(rows[-1]), flush=True)
Path("gpurun_out").mkdir(exist_ok=True)
Path("gpurun_out/probe_tma.json").write_text(json.dumps(rows, indent=1))
