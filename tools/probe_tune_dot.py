"""Tuner ranking vs long-loop truth for the headline dot (2^28 f32): the
tuner's top 8 variants re-timed over 200 back-to-back launches."""
import sys, json
sys.path.insert(0, "/root/repo")
import numpy as np
from paper_0911_3456_b200 import _runtime as rt, autotune as at, elementwise as ew, ndarray as nd, reduction as rd
rt.set_device(0)
pool = nd.MemoryPool(device=0)
n = 1 << 28
rng = np.random.default_rng([0, 0])
gx = nd.from_host(pool, nd.float32, rng.uniform(-1, 1, n).astype(np.float32))
gy = nd.from_host(pool, nd.float32, rng.uniform(-1, 1, n).astype(np.float32))
spec = rd.ReductionSpec("float *x, float *y", nd.float32, "0", "a + b", "x[i] * y[i]")
axes = dict(at.DEFAULT_AXES, waves=(0, 1, 2), cache=("default", "tma"))
t = at.tune_reduction(spec, "dot_k", n, axes, args=[gx, gy], constraints=(lambda a: a["cache"] != "tma" or a["unroll"] == 1,), protocol=at.MeasurementProtocol(warmup=1, repeats=3), burst=10)
ok = sorted([e for e in t.table if e.status == "ok"], key=lambda e: e.stat_seconds)
o = pool.alloc_uninitialized(nd.float32, ())
def mean_ms(fn, reps=200):
    fn(); rt.synchronize()
    s, e = rt.Event(), rt.Event(); s.record()
    for _ in range(reps): fn()
    e.record(); e.synchronize(); return s.elapsed_ms(e) / reps
for e in ok[:8]:
    a = e.as_dict()
    k = rd.ReductionKernel(spec, "dot_k", ew.VariantParams(**a))
    print(a, "tuner", round(8 * n / e.stat_seconds / 1e9), "200-step", round(8 * n / mean_ms(lambda: k.launch(gx, gy, out=o)) / 1e6), flush=True)
