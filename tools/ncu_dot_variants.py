"""Every variant of the bench's dot tuning space, launched twice each, for a
metrics-only ncu pass (DRAM bytes per launch by variant):

    ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
        --clock-control none -k regex:dot_k --csv --log-file gpurun_out/dot_variants.csv \
        python tools/ncu_dot_variants.py

Prints the launch order (variant per launch) as JSON on stdout."""
import itertools
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402
from paper_0911_3456_b200 import _runtime as rt, elementwise as ew, ndarray as nd  # noqa: E402
from paper_0911_3456_b200 import reduction as rd  # noqa: E402

rt.set_device(0)
pool = nd.MemoryPool(device=0)
n = 1 << 28
rng = np.random.default_rng(0)
x = nd.from_host(pool, nd.float32, rng.uniform(-1, 1, n).astype(np.float32))
y = nd.from_host(pool, nd.float32, rng.uniform(-1, 1, n).astype(np.float32))
o = pool.alloc_uninitialized(nd.float32, ())
spec = rd.ReductionSpec("float *x, float *y", nd.float32, "0", "a + b", "x[i] * y[i]")
order = []
for unroll, block, waves, cache in itertools.product((1, 2, 4, 8, 16), (128, 256, 512, 1024),
                                                     (0, 1, 2), ("default", "tma")):
    if cache == "tma" and unroll != 1:
        continue
    v = {"block": block, "cache": cache, "unroll": unroll, "waves": waves}
    k = rd.ReductionKernel(spec, "dot_k", ew.VariantParams(**v))
    for _ in range(2):
        k.launch(x, y, out=o)
        order.append(v)
rt.synchronize()
print(json.dumps(order))
