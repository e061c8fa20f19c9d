"""Variant sweep on the GPU: device-timed GB/s for the benchmark kernels.

    python tools/sweep.py [--out gpurun_out/sweep.json] [--only axpy,dot,...]
"""
import argparse
import itertools
import json
import math
import sys
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_0911_3456_b200 import _runtime as rt, autotune as at, elementwise as ew  # noqa: E402
from paper_0911_3456_b200 import jit, ndarray as nd, reduction as rd  # noqa: E402

PEAK = 6549.1
N = 1 << 28


def best_ms(fn, reps=10):
    fn()
    rt.synchronize()
    s, e = rt.Event(), rt.Event()
    best = math.inf
    for _ in range(reps):
        s.record()
        fn()
        e.record()
        e.synchronize()
        best = min(best, s.elapsed_ms(e))
    return best


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--out", default="gpurun_out/sweep.json")
    p.add_argument("--only", default="")
    a = p.parse_args()
    only = set(filter(None, a.only.split(",")))
    rt.set_device(0)
    pool = nd.MemoryPool(device=0)
    rng = np.random.default_rng(0)
    x = nd.from_host(pool, nd.float32, rng.uniform(-1, 1, N).astype(np.float32))
    y = nd.from_host(pool, nd.float32, rng.uniform(-1, 1, N).astype(np.float32))
    z = pool.alloc_uninitialized(nd.float32, (N,))
    o = pool.alloc_uninitialized(nd.float32, ())
    results = {}

    grid = list(itertools.product((1, 2, 4, 8, 16), (128, 256, 512, 1024),
                                  ("default", "streaming", "no-l1"), ("strided",)))
    grid += [(u, b, "default", "contiguous-blocks") for u in (2, 4, 8) for b in (256, 512)]

    def run(name, make, call, nbytes, variants):
        if only and name not in only:
            return
        with ThreadPoolExecutor(8) as ex:
            kernels = list(ex.map(lambda v: (v, make(v)), variants))
        rows = []
        for v, k in kernels:
            try:
                ms = best_ms(lambda: call(k))
            except Exception as exc:  # noqa: BLE001
                rows.append({"variant": str(v), "error": str(exc)[:200]})
                continue
            gbs = nbytes / ms / 1e6
            rows.append({"variant": v.__dict__ if hasattr(v, "__dict__") else str(v),
                         "ms": round(ms, 4), "GB/s": round(gbs, 1), "frac": round(gbs / PEAK, 4)})
        rows.sort(key=lambda r: r.get("ms", 1e9))
        results[name] = rows
        print(name, json.dumps(rows[:5]), flush=True)

    V = [ew.VariantParams(unroll=u, block=b, cache=c, chunking=ch) for u, b, c, ch in grid]
    run("axpy", lambda v: ew.ElementwiseKernel("float a, float *x, float b, float *y, float *z",
                                               "z[i] = a * x[i] + b * y[i]", "axpy", v),
        lambda k: k(2.0, x, -3.0, y, z), 12 * N, V)
    run("dot", lambda v: rd.ReductionKernel(rd.ReductionSpec(
        "float *x, float *y", nd.float32, "0", "a + b", "x[i] * y[i]"), "dot_k", v),
        lambda k: k.launch(x, y, out=o), 8 * N, V)
    run("maxabs", lambda v: rd.make_reduction("float *x", nd.float32, "0", "a > b ? a : b",
                                              "fabsf(x[i])", name="maxabs", variant=v),
        lambda k: k.launch(x, out=o), 4 * N, V)
    run("sumsq", lambda v: rd.make_reduction("float *x", nd.float32, "0", "a + b",
                                             "x[i] * x[i]", name="sumsq", variant=v),
        lambda k: k.launch(x, out=o), 4 * N, V)
    for arr in (x, y, z):
        arr.free()
    if not only or "polysin" in only or "sum_i64" in only:
        xd = nd.from_host(pool, nd.float64, rng.uniform(-2, 2, N))
        zd = pool.alloc_uninitialized(nd.float64, (N,))
        PV = [ew.VariantParams(unroll=u, block=b) for u in (1, 2, 4, 8) for b in (128, 256, 512)]
        run("polysin", lambda v: ew.ElementwiseKernel(
            "double a, double *x, double *z",
            "z[i] = ((a*x[i] + 2.0)*x[i] - 1.5)*x[i] + sin(x[i])", "polysin", v),
            lambda k: k(0.5, xd, zd), 16 * N, PV)
        fm = jit.ToolchainConfig().with_fmad(True)
        run("polysin_fmad", lambda v: ew.ElementwiseKernel(
            "double a, double *x, double *z",
            "z[i] = ((a*x[i] + 2.0)*x[i] - 1.5)*x[i] + sin(x[i])", "polysin", v, config=fm),
            lambda k: k(0.5, xd, zd), 16 * N, PV)
        o64 = pool.alloc_uninitialized(nd.int64, ())
        xi = nd.from_host(pool, nd.int64, rng.integers(-(1 << 62), 1 << 62, N, dtype=np.int64))
        run("sum_i64", lambda v: rd.sum_kernel(nd.int64, v), lambda k: k.launch(xi, out=o64),
            8 * N, V)
    Path(a.out).parent.mkdir(exist_ok=True)
    Path(a.out).write_text(json.dumps(results, indent=1))


if __name__ == "__main__":
    main()
