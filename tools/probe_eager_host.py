import sys, time, cProfile, pstats
sys.path.insert(0, '/root/repo')
import numpy as np
from paper_0911_3456_b200 import _runtime as rt, ndarray as nd
rt.set_device(0)
pool = nd.MemoryPool(device=0)
x = nd.from_host(pool, nd.float32, np.ones(1 << 16, np.float32))
y = nd.from_host(pool, nd.float32, np.ones(1 << 16, np.float32))
def eager():
    t1 = x * 2
    t2 = t1 + y
    t3 = t2 - x
    for t in (t1, t2, t3):
        t.free()
for _ in range(200): eager()
rt.synchronize()
t0 = time.perf_counter()
for _ in range(2000): eager()
rt.synchronize()
print("per chain us", (time.perf_counter() - t0) / 2000 * 1e6)
pr = cProfile.Profile(); pr.enable()
for _ in range(2000): eager()
pr.disable(); rt.synchronize()
pstats.Stats(pr).sort_stats('tottime').print_stats(14)
