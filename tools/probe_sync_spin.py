"""Synchronous small reductions: what does waiting cost?  A 2^16 float32 sum
whose out slot is this thread's page-locked host slot; per call (best of
many): launch only; launch + cuStreamSynchronize (what ``kernel(x)`` does);
launch + a host spin on the slot until the value lands (the slot is preset
to a sentinel the result cannot equal).  Python-side perf_counter."""
import ctypes
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402
from paper_0911_3456_b200 import _runtime as rt, ndarray as nd, reduction as rd  # noqa: E402

rt.set_device(0)
pool = nd.MemoryPool(device=0)
x = nd.from_host(pool, nd.float32, np.ones(1 << 16, np.float32))
k = rd.sum_kernel(nd.float32)
slot = rd._host_slot()
cell = ctypes.c_float.from_address(slot)


def launch():
    k.launch(x, out_address=slot)


def with_sync():
    launch()
    rt.stream_synchronize(0)
    return cell.value


def with_spin():
    cell.value = -1.0
    launch()
    while cell.value == -1.0:
        pass
    return cell.value


res = {}
for name, fn in (("launch_only", launch), ("launch_sync", with_sync), ("launch_spin", with_spin)):
    for _ in range(200):
        fn()
    rt.synchronize()
    best, times = float("inf"), []
    for _ in range(2000):
        t0 = time.perf_counter()
        fn()
        dt = time.perf_counter() - t0
        times.append(dt)
        if name == "launch_only":
            rt.synchronize()
    res[name] = {"best_us": round(min(times) * 1e6, 2), "median_us": round(float(np.median(times)) * 1e6, 2)}
    rt.synchronize()
res["result"] = with_spin()
print(json.dumps(res))
