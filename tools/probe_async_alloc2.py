"""Pool allocate/free cycle times for blocks above the pooled classes (the
stream-ordered allocator behind MemoryPool) and free/total device memory."""
import sys, time
sys.path.insert(0, "/root/repo")
from paper_0911_3456_b200 import _runtime as rt, ndarray as nd
rt.set_device(0)
pool = nd.MemoryPool(device=0)
def cycles(label, nbytes, k=6):
    ts = []
    for _ in range(k):
        t0 = time.perf_counter(); a = pool.alloc_uninitialized(nd.uint8, (nbytes,)); t1 = time.perf_counter(); a.free(); t2 = time.perf_counter()
        ts.append((round((t1 - t0) * 1e3, 2), round((t2 - t1) * 1e3, 2)))
    print(label, ts, "free/total GB", [round(v / 1e9, 1) for v in rt.mem_get_info()], flush=True)
cycles("2G fresh", 2 << 30)
big = pool.alloc_uninitialized(nd.uint8, (32 << 30,)); big.free()
cycles("2G after 32G freed", 2 << 30)
a = pool.alloc_uninitialized(nd.uint8, (16 << 30,)); b = pool.alloc_uninitialized(nd.uint8, (16 << 30,))
cycles("2G with 32G live", 2 << 30)
a.free(); b.free()
cycles("2G after all freed", 2 << 30)
hold = [rt.mem_alloc(1 << 30) for _ in range(100)]
cycles("2G with 100G sync-held", 2 << 30)
for h in hold: rt.mem_free(h)
cycles("2G after sync freed", 2 << 30)
