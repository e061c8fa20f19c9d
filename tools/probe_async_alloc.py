"""Host cost of stream-ordered allocation (cuMemAllocAsync / cuMemFreeAsync)
of a 2 GiB block on the legacy and a created stream."""
import sys, time
sys.path.insert(0, "/root/repo")
from paper_0911_3456_b200 import _runtime as rt
rt.set_device(0)
n = (2 << 30) + 8
for label, stream in (("legacy", 0), ("created", rt.Stream().handle)):
    with rt.use_stream(stream):
        ts = []
        for k in range(6):
            t0 = time.perf_counter(); p = rt.mem_alloc_async(n); t1 = time.perf_counter(); rt.mem_free_async(p); t2 = time.perf_counter()
            ts.append((round((t1-t0)*1e3, 3), round((t2-t1)*1e3, 3)))
        rt.synchronize()
        print(label, ts, flush=True)
ts = []
for k in range(4):
    t0 = time.perf_counter(); p = rt.mem_alloc(n); t1 = time.perf_counter(); rt.mem_free(p); t2 = time.perf_counter()
    ts.append((round((t1-t0)*1e3, 3), round((t2-t1)*1e3, 3)))
print("sync", ts)
