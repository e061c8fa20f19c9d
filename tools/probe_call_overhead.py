"""Where does the host time of one ElementwiseKernel call go (on the GPU box)?"""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_0911_3456_b200 import _runtime as rt, elementwise as ew, ndarray as nd
from paper_0911_3456_b200 import _codegen as cg
rt.set_device(0)
pool = nd.MemoryPool(device=0)
x = pool.alloc(nd.float32, (1 << 16,)); z = pool.alloc(nd.float32, (1 << 16,))
k = ew.ElementwiseKernel("float a, float *x, float *z", "z[i] = a * x[i] + 1.0f", "lat")
k(2.0, x, z); rt.synchronize()
N = 5000
def clock(label, fn):
    t0 = time.perf_counter()
    for _ in range(N):
        fn()
    rt.synchronize()
    print(f"{label:28s} {(time.perf_counter() - t0) / N * 1e6:7.2f} us", flush=True)
clock("full call", lambda: k(2.0, x, z))
vals, ptrs, vectors, n = k._binder.bind((2.0, x, z), None, 0, "lat", ew._ERRORS)
fn = k.vectorized.function(0)
grid = cg.grid_for(fn, 0, 256, None, n, 4, 0)
k._binder.set_range(vals, 0, n)
clock("bind only", lambda: k._binder.bind((2.0, x, z), None, 0, "lat", ew._ERRORS))
clock("raw rt.launch", lambda: rt.launch(fn, grid, 256, ptrs, 0, None))
lib = rt.lib()
clock("raw ctypes rtcg_launch", lambda: lib.rtcg_launch(fn, grid, 256, 0, None, ptrs))
s = rt.Stream()
clock("raw ctypes, created stream", lambda: lib.rtcg_launch(fn, grid, 256, 0, s.handle, ptrs))
with rt.use_stream(s):
    clock("full call, created stream", lambda: k(2.0, x, z))
