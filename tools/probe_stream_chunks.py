"""Streamed host call (driver.In/Out) chunk-size sweep for the C3 kernel, and
the raw duplex pinned copy rate (H2D and D2H concurrently) as its ceiling."""
import sys, time
sys.path.insert(0, "/root/repo")
import numpy as np
from paper_0911_3456_b200 import _runtime as rt, elementwise as ew, ndarray as nd, driver as drv
rt.set_device(0)
n = 1 << 28
hx = nd.pinned_empty((n,), nd.float64); hx[:] = np.random.default_rng(0).uniform(-2, 2, n)
hz = nd.pinned_empty((n,), nd.float64)
k = ew.ElementwiseKernel("double a, double *x, double *z", "z[i] = ((a*x[i] + 2.0)*x[i] - 1.5)*x[i] + sin(x[i])", "ps", ew.VariantParams(block=256, waves=1, prefetch=True))
for mib in (8, 16, 32, 64, 128, 256):
    step = (mib << 20) // 16
    k._call_host((0.5, drv.In(hx), drv.Out(hz)), None, chunk=step)
    t0 = time.perf_counter()
    for _ in range(3): k._call_host((0.5, drv.In(hx), drv.Out(hz)), None, chunk=step)
    s = (time.perf_counter() - t0) / 3
    print(mib, "MiB chunks:", round(16 * n / s / 1e9, 1), "GB/s")
# pure duplex copy reference: async H2D and D2H on two streams
gx = nd.empty((n,), nd.float64); gz = nd.empty((n,), nd.float64)
s1, s2 = rt.Stream(), rt.Stream()
t0 = time.perf_counter()
for _ in range(3):
    rt.memcpy_htod(gx.address, hx.ctypes.data, 8 * n, s1.handle)
    rt.memcpy_dtoh(hz.ctypes.data, gz.address, 8 * n, s2.handle)
    s1.synchronize(); s2.synchronize()
print("duplex copy", round(16 * n * 3 / (time.perf_counter() - t0) / 1e9, 1), "GB/s")
