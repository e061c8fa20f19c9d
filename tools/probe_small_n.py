"""Where does a small-n call's time go?  For x+y, sum, max and dot at
n = 2^16 / 2^20 / 2^24 (float32), four numbers per call:

  single_us   CUDA events around ONE call (bench.py's C5 protocol: host
              submission + kernel, what a synchronous caller sees on device)
  host_us     perf_counter per call over 2000 calls without synchronising
              (the Python + native launch path alone)
  stream_us   events around 2000 back-to-back calls / 2000 (max of host rate
              and device rate: the throughput a loop of calls gets)
  graph_us    one call captured in a CUDA graph, 200 replays / 200 (the
              kernel with no host path -- its floor on device)
  scalar_us   perf_counter around ONE synchronous call returning the host
              scalar (the reference API: ``kernel(x)``), reductions only

    python tools/probe_small_n.py > gpurun_out/small_n.json
"""
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402

from paper_0911_3456_b200 import _runtime as rt, ndarray as nd, elementwise as ew  # noqa: E402
from paper_0911_3456_b200 import reduction as rd, graph  # noqa: E402


def best_single(fn, reps=7):
    fn()
    rt.synchronize()
    s, e = rt.Event(), rt.Event()
    best = float("inf")
    for _ in range(reps):
        s.record()
        fn()
        e.record()
        e.synchronize()
        best = min(best, s.elapsed_ms(e) * 1e3)
    return best


def host_rate(fn, calls=2000):
    fn()
    rt.synchronize()
    t0 = time.perf_counter()
    for _ in range(calls):
        fn()
    t = time.perf_counter() - t0
    rt.synchronize()
    return t / calls * 1e6


def stream_rate(fn, calls=2000):
    fn()
    rt.synchronize()
    s, e = rt.Event(), rt.Event()
    s.record()
    for _ in range(calls):
        fn()
    e.record()
    e.synchronize()
    return s.elapsed_ms(e) * 1e3 / calls


def graph_rate(fn, replays=200):
    st = rt.Stream()
    with rt.use_stream(st.handle):
        fn()
        st.synchronize()
        g = graph.Graph(st)
        with g.capture():
            fn()
        g.launch()
        st.synchronize()
        s, e = rt.Event(), rt.Event()
        s.record(st.handle)
        for _ in range(replays):
            g.launch()
        e.record(st.handle)
        e.synchronize()
    g.close()
    return s.elapsed_ms(e) * 1e3 / replays


def scalar_call(fn, reps=50):
    fn()
    best = float("inf")
    for _ in range(reps):
        t0 = time.perf_counter()
        fn()
        best = min(best, time.perf_counter() - t0)
    return best * 1e6


def main():
    rt.set_device(0)
    pool = nd.MemoryPool(device=0)
    add = ew.ElementwiseKernel("float *x, float *y, float *z", "z[i] = x[i] + y[i]", "add_f32")
    red = {"sum": rd.sum_kernel(nd.float32), "max": rd.max_kernel(nd.float32),
           "dot": rd.dot_kernel(nd.float32)}
    rows = {}
    rng = np.random.default_rng(0)
    for lg in (16, 20, 24):
        n = 1 << lg
        x = nd.from_host(pool, nd.float32, rng.uniform(-1, 1, n).astype(np.float32))
        y = nd.from_host(pool, nd.float32, rng.uniform(-1, 1, n).astype(np.float32))
        z = pool.alloc(nd.float32, (n,))
        o = pool.alloc(nd.float32, ())
        calls = {"add": lambda: add(x, y, z)}
        for name, k in red.items():
            args = (x, y) if name == "dot" else (x,)
            calls[name] = (lambda k=k, args=args: k.launch(*args, out=o, overlap_previous=True))
            calls[name + "_serial"] = (lambda k=k, args=args: k.launch(*args, out=o))
        row = {}
        for name, fn in calls.items():
            r = {"single_us": round(best_single(fn), 2), "host_us": round(host_rate(fn), 2),
                 "stream_us": round(stream_rate(fn), 2)}
            try:
                r["graph_us"] = round(graph_rate(fn), 2)
            except Exception as exc:                      # noqa: BLE001
                r["graph_us"] = f"{type(exc).__name__}: {exc}"
            if name in red:
                k = red[name]
                args = (x, y) if name == "dot" else (x,)
                r["scalar_us"] = round(scalar_call(lambda: k(*args)), 2)
            row[name] = r
        rows[f"2^{lg}"] = row
        for a in (x, y, z, o):
            a.free()
    print(json.dumps({"what": __doc__.split("\n\n")[0], "rows": rows}, indent=1))


if __name__ == "__main__":
    main()
