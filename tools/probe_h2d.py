"""Host<->device copy bandwidth: driver pageable path vs the runtime's pinned
staging pipeline (rtcg_copy_htod/dtoh) vs page-locked buffers, and the staging
pipeline's host-thread count (RTCG_COPY_THREADS, one subprocess each).

    python tools/probe_h2d.py            # full table
"""
import os
import subprocess
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402

N = 1 << 28          # 1 GiB of float32


def _bw(fn, reps=4):
    fn()
    t0 = time.perf_counter()
    for _ in range(reps):
        fn()
    return reps * N * 4 / (time.perf_counter() - t0) / 1e9


def one(label_only=False):
    from paper_0911_3456_b200 import _runtime as rt, ndarray as nd
    rt.set_device(0)
    pool = nd.MemoryPool(device=0)
    page = np.random.default_rng(0).uniform(-1, 1, N).astype(np.float32)
    out = np.empty_like(page)
    g = pool.alloc_uninitialized(nd.float32, (N,))
    rows = {}
    if not label_only:
        def drv_h2d():
            rt.memcpy_htod(g.address, page.ctypes.data, g.nbytes)
            rt.synchronize()

        def drv_d2h():
            rt.memcpy_dtoh(out.ctypes.data, g.address, g.nbytes)
            rt.synchronize()
        rows["pageable, driver"] = (_bw(drv_h2d), _bw(drv_d2h))
        pin = nd.pinned_empty((N,), nd.float32)
        pin[:] = page
        pout = nd.pinned_empty((N,), nd.float32)
        rows["pinned"] = (_bw(lambda: g.copy_from_host(pin)), _bw(lambda: g.to_host(out=pout)))
    rows["pageable, staged"] = (_bw(lambda: g.copy_from_host(page)), _bw(lambda: g.to_host(out=out)))
    assert np.array_equal(out, page)
    for k, (h, d) in rows.items():
        print(f"{k:22s} threads={os.environ.get('RTCG_COPY_THREADS', 'auto'):>4s} "
              f"HtoD {h:6.1f} GB/s  DtoH {d:6.1f} GB/s", flush=True)


if __name__ == "__main__":
    if "--child" in sys.argv:
        one(label_only=True)
        raise SystemExit(0)
    one()
    for t in (1, 2, 4, 8, 12, 16):
        subprocess.run([sys.executable, __file__, "--child"],
                       env={**os.environ, "RTCG_COPY_THREADS": str(t)}, check=True)
    print("without non-temporal stores:", flush=True)
    subprocess.run([sys.executable, __file__, "--child"],
                   env={**os.environ, "RTCG_COPY_NT": "0"}, check=True)
    print(f"host cores: {os.cpu_count()}")
