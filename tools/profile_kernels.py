"""Launch the benchmark kernels with their tuned variants a few times each, for
ncu (``-k regex:<name>``).  Variants come from profiles/r01_bench_c4_2p32.json."""
import json, sys
from pathlib import Path
ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import numpy as np
from paper_0911_3456_b200 import _runtime as rt, elementwise as ew, ndarray as nd, reduction as rd

bench = json.loads((ROOT / "profiles" / "r01_bench_c4_2p32.json").read_text())
V = lambda a: ew.VariantParams(**a)  # noqa: E731
rt.set_device(0)
pool = nd.MemoryPool(device=0)
n = 1 << 28
rng = np.random.default_rng(0)
x = nd.from_host(pool, nd.float32, rng.uniform(-1, 1, n).astype(np.float32))
y = nd.from_host(pool, nd.float32, rng.uniform(-1, 1, n).astype(np.float32))
z = pool.alloc_uninitialized(nd.float32, (n,))
o = pool.alloc_uninitialized(nd.float32, ())
dot = rd.ReductionKernel(rd.ReductionSpec("float *x, float *y", nd.float32, "0", "a + b",
                                          "x[i] * y[i]"), "dot_k", V(bench["config"]["variant"]))
axpy = ew.ElementwiseKernel("float a, float *x, float b, float *y, float *z",
                            "z[i] = a * x[i] + b * y[i]", "axpy",
                            V(bench["workloads"]["axpy_f32_2p28"]["variant"]))
for _ in range(3):
    dot.launch(x, y, out=o)
    axpy(2.0, x, -3.0, y, z)
rt.synchronize()
print("dot", dot.launch_config(x, y), "axpy", axpy.launch_config(2.0, x, -3.0, y, z))
