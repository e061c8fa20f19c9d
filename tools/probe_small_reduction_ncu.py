"""Launch a 2^16 / 2^20 float32 sum and x + y a few times each (serial
launches) for an ncu metrics pass: where a small reduction's device time
goes next to an elementwise kernel over the same bytes.

    ncu --metrics gpu__time_duration.sum,... python tools/probe_small_reduction_ncu.py
"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402
from paper_0911_3456_b200 import _runtime as rt, ndarray as nd, elementwise as ew  # noqa: E402
from paper_0911_3456_b200 import reduction as rd  # noqa: E402

rt.set_device(0)
pool = nd.MemoryPool(device=0)
add = ew.ElementwiseKernel("float *x, float *y, float *z", "z[i] = x[i] + y[i]", "add_small")
s = rd.sum_kernel(nd.float32)
for lg in (16, 20):
    n = 1 << lg
    x = nd.from_host(pool, nd.float32, np.ones(n, np.float32))
    y = nd.from_host(pool, nd.float32, np.ones(n, np.float32))
    z = pool.alloc(nd.float32, (n,))
    o = pool.alloc(nd.float32, ())
    for _ in range(5):
        add(x, y, z)
        s.launch(x, out=o)
    rt.synchronize()
    print(lg, s.launch_config(x), flush=True)
