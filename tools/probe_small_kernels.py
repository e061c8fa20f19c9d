import sys; sys.path.insert(0, '/root/repo')
import numpy as np
from paper_0911_3456_b200 import _runtime as rt, ndarray as nd, elementwise as ew, reduction as rd
rt.set_device(0)
pool = nd.MemoryPool(device=0)
for lg in (12, 16, 20):
    n = 1 << lg
    x = nd.from_host(pool, nd.float32, np.ones(n, np.float32))
    y = nd.from_host(pool, nd.float32, np.ones(n, np.float32))
    z = pool.alloc(nd.float32, (n,))
    o = pool.alloc(nd.float32, ())
    add = ew.ElementwiseKernel("float *x, float *y, float *z", "z[i] = x[i] + y[i]", f"add{lg}")
    s = rd.ReductionKernel(rd.ReductionSpec("float *x", nd.float32, "0", "a + b", None), f"sum{lg}")
    for _ in range(5):
        add(x, y, z); s.launch(x, out=o)
    rt.synchronize()
    print(lg, s.launch_config(x), add.launch_config(x, y, z) if hasattr(add, "launch_config") else "")
