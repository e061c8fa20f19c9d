"""BASELINE config C5: GPUArray chains + reductions over n = 2^16..2^32 and
dtypes, plus compile/cache latency and an autotune campaign (1 GPU).

    python tools/c5_sweep.py [--max-log2 32] [--out gpurun_out/c5_sweep.json]

Inputs are synthesised on the device by a generated kernel (no host copies),
so 2^32-element arrays need no host RAM.  Times are CUDA-event device times,
best of 5 after a warm-up; GB/s uses algorithmic bytes.
"""
import argparse
import json
import math
import sys
import tempfile
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_0911_3456_b200 import _runtime as rt, autotune as at, elementwise as ew  # noqa: E402
from paper_0911_3456_b200 import fusion, jit, ndarray as nd, reduction as rd  # noqa: E402


def dev_ms(fn, reps=5):
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
    p.add_argument("--min-log2", type=int, default=16)
    p.add_argument("--max-log2", type=int, default=32)
    p.add_argument("--out", default="gpurun_out/c5_sweep.json")
    a = p.parse_args()
    rt.set_device(0)
    pool = nd.MemoryPool(device=0)
    report = {"sizes": {}, "latency": {}, "autotune": {}}

    # --- compile / cache latency -------------------------------------------------------
    cold_root = Path(tempfile.mkdtemp(prefix="rtcg-cold-"))
    sig, op = "float a, float *x, float *z", "z[i] = a * x[i] + 1.0f"
    t0 = time.perf_counter()
    ew.ElementwiseKernel(sig, op, "lat_probe", cache=jit.CacheStore(cold_root))
    cold = time.perf_counter() - t0
    warm = []
    for _ in range(20):
        t0 = time.perf_counter()
        ew.ElementwiseKernel(sig, op, "lat_probe", cache=jit.CacheStore(cold_root))
        warm.append(time.perf_counter() - t0)
    k = ew.ElementwiseKernel(sig, op, "lat_probe", cache=jit.CacheStore(cold_root))
    x = pool.alloc(nd.float32, (1 << 16,))
    z = pool.alloc(nd.float32, (1 << 16,))
    k(2.0, x, z)           # first launch: cuModuleLoadData
    rt.synchronize()
    t0 = time.perf_counter()
    for _ in range(1000):
        k(2.0, x, z)
    rt.synchronize()
    per_launch = (time.perf_counter() - t0) / 1000
    # the same call captured in a CUDA graph: host cost per replay
    from paper_0911_3456_b200 import graph as gr
    g = gr.Graph()
    with rt.use_stream(g.stream):
        k(2.0, x, z)
        g.synchronize()
    with g.capture():
        for _ in range(10):
            k(2.0, x, z)
    g.launch()
    g.synchronize()
    t0 = time.perf_counter()
    for _ in range(100):
        g.launch()
    g.synchronize()
    per_graph_kernel = (time.perf_counter() - t0) / 1000
    report["latency"] = {"cold_nvrtc_construct_ms": round(cold * 1e3, 2),
                         "graph_replay_us_per_kernel": round(per_graph_kernel * 1e6, 2),
                         "warm_cache_construct_ms_median": round(sorted(warm)[10] * 1e3, 3),
                         "cold_over_warm": round(cold / sorted(warm)[10], 1),
                         "host_call_us_back_to_back": round(per_launch * 1e6, 2)}
    print(json.dumps(report["latency"]), flush=True)

    # --- autotune campaign and store hit ----------------------------------------------------
    store = at.TuneStore(tempfile.mkdtemp(prefix="rtcg-tune-"))
    spec = rd.ReductionSpec("float *x, float *y", nd.float32, "0", "a + b", "x[i] * y[i]")
    t0 = time.perf_counter()
    r = at.tune_reduction(spec, "dot_c5", 1 << 26, at.DEFAULT_AXES, store=store, pool=pool)
    campaign = time.perf_counter() - t0
    t0 = time.perf_counter()
    r2 = at.tune_reduction(spec, "dot_c5", 1 << 26, at.DEFAULT_AXES, store=store, pool=pool)
    hit = time.perf_counter() - t0
    report["autotune"] = {"problem": "dot f32 n=2^26", "variants": len(r.table),
                          "campaign_s": round(campaign, 2), "store_hit_s": round(hit, 4),
                          "best": r.best_assignment, "best_us": round(r.best_seconds * 1e6, 1),
                          "store_hit_same_best": r2.best_assignment == r.best_assignment}
    print(json.dumps(report["autotune"]), flush=True)

    # --- size x dtype sweep -----------------------------------------------------------------
    kernels = {}
    for dname in ("float32", "float64", "int32", "int64"):
        d = nd.BY_NAME[dname]
        c = d.cname
        fill = ew.ElementwiseKernel(f"long seed, {c} *x",
                                    f"x[i] = ({c}) ((long) (((unsigned long) i * 2654435761UL + seed) % 2001) - 1000)"
                                    f" / ({c}) {'1000.0' if d.kind == 'f' else '1'}",
                                    f"fill_{dname}")
        add = ew.ElementwiseKernel(f"{c} *x, {c} *y, {c} *z", "z[i] = x[i] + y[i]", f"add_{dname}")
        sm = rd.sum_kernel(d)
        mx = rd.max_kernel(d)
        dot = rd.dot_kernel(d)
        kernels[dname] = (fill, add, sm, mx, dot)
    for lg in range(a.min_log2, a.max_log2 + 1, 2):
        n = 1 << lg
        row = {}
        for dname, (fill, add, sm, mx, dot) in kernels.items():
            d = nd.BY_NAME[dname]
            sz = d.size
            try:
                x = pool.alloc_uninitialized(d, (n,))
                y = pool.alloc_uninitialized(d, (n,))
                z = pool.alloc_uninitialized(d, (n,))
            except Exception as exc:  # noqa: BLE001
                row[dname] = {"error": f"alloc: {exc}"[:120]}
                continue
            fill(1, x)
            fill(7, y)
            o = pool.alloc_uninitialized(d, ())
            res = {}

            def rec(name, fn, nbytes):
                ms = dev_ms(fn)
                res[name] = {"us": round(ms * 1e3, 2), "GB/s": round(nbytes / ms / 1e6, 1)}
            rec("add", lambda: add(x, y, z), 3 * sz * n)
            if lg <= 30:  # eager chain needs 2 extra temporaries
                def eager():
                    t1 = x * 2
                    t2 = t1 + y
                    t3 = t2 - x
                    for t in (t1, t2, t3):
                        t.free()
                rec("chain_eager", eager, 3 * sz * n)   # algorithmic: read x, y; write z
            f = fusion.fused(lambda p, q: (p * 2 + q) - p)
            rec("chain_fused", lambda: f(x, y, out=z), 3 * sz * n)
            fr = fusion.fused(lambda p, q: (p * 2 + q) - p, reduce="sum")

            def chain_then_sum():
                f(x, y, out=z)
                sm.launch(z, out=o)
            # chain + reduction: algorithmic bytes = the two inputs
            rec("chain_sum_two_pass", chain_then_sum, 2 * sz * n)
            rec("chain_sum_fused", lambda: fr(x, y).free(), 2 * sz * n)
            rec("sum", lambda: sm.launch(x, out=o), sz * n)
            # back-to-back overlapped reductions (programmatic dependent launch):
            # mean of a 20-launch burst, as a stream of reductions would run
            def sum_burst():
                for _ in range(20):
                    sm.launch(x, out=o, overlap_previous=True)
            ms = dev_ms(sum_burst) / 20
            res["sum_overlapped"] = {"us": round(ms * 1e3, 2), "GB/s": round(sz * n / ms / 1e6, 1)}
            rec("max", lambda: mx.launch(x, out=o), sz * n)
            rec("dot", lambda: dot.launch(x, y, out=o), 2 * sz * n)
            row[dname] = res
            for arr in (x, y, z, o):
                arr.free()
        report["sizes"][f"2^{lg}"] = row
        print(f"2^{lg}", json.dumps(row), flush=True)
        pool.release_free()
    Path(a.out).parent.mkdir(exist_ok=True)
    Path(a.out).write_text(json.dumps(report, indent=1))


if __name__ == "__main__":
    main()
