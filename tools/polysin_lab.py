"""C3 (f64 poly+sin, 2^28) variant lab: time a list of variants, or launch one
variant a few times for ncu.

    python tools/polysin_lab.py sweep ['{"stages": [0, 4]}'] [--out gpurun_out/polysin_sweep.json]
    python tools/polysin_lab.py one '{"block":256,"prefetch":true,"waves":1}' [--fma]

Times are CUDA-event device times: the mean of a 10-launch burst, best of 3
bursts, after a warm-up launch.  GB/s uses 16 algorithmic bytes per element.
"""
import argparse
import itertools
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402
from paper_0911_3456_b200 import _runtime as rt, elementwise as ew, jit, ndarray as nd  # noqa: E402

SIG = "double a, double *x, double *z"
OP = "z[i] = ((a*x[i] + 2.0)*x[i] - 1.5)*x[i] + sin(x[i])"
N = 1 << 28


def kernel(v: dict, fma: bool = False, op: str = OP, preamble: str = ""):
    cfg = None
    if fma:
        cfg = jit.ToolchainConfig(flags=tuple("-fmad=true" if f == "-fmad=false" else f
                                              for f in jit.DEFAULT_FLAGS))
    return ew.ElementwiseKernel(SIG, op, "polysin", ew.VariantParams(**v), config=cfg,
                                preamble=preamble)


def time_ms(k, x, z, burst=10, reps=3):
    k(0.5, x, z)
    rt.synchronize()
    s, e = rt.Event(), rt.Event()
    best = float("inf")
    for _ in range(reps):
        s.record()
        for _ in range(burst):
            k(0.5, x, z)
        e.record()
        e.synchronize()
        best = min(best, s.elapsed_ms(e) / burst)
    return best


def main():
    p = argparse.ArgumentParser()
    p.add_argument("mode", choices=("sweep", "one", "ops", "sustained"))
    p.add_argument("variant", nargs="?", default="{}")
    p.add_argument("--fma", action="store_true")
    p.add_argument("--op", default=OP)
    p.add_argument("--out", default="gpurun_out/polysin_sweep.json")
    p.add_argument("--launches", type=int, default=3)
    p.add_argument("--preamble", default="", help="file with helper device code")
    p.add_argument("--ops", default="", help="file: one op per line (mode ops)")
    p.add_argument("--variants", default="[]", help="JSON list of variants (mode ops)")
    a = p.parse_args()
    rt.set_device(0)
    pool = nd.MemoryPool(device=0)
    x = nd.from_host(pool, nd.float64, np.random.default_rng(1).uniform(-2, 2, N))
    z = pool.alloc_uninitialized(nd.float64, (N,))
    pre = Path(a.preamble).read_text() if a.preamble else ""
    if a.mode == "sustained":   # variants under the board's power cap: heat, then long bursts
        rows = []
        variants = json.loads(a.variants)
        ks = [kernel(v, a.fma, a.op, pre) for v in variants]
        heat = ks[0]
        for _ in range(3000):          # ~2 s of the workload itself
            heat(0.5, x, z)
        rt.synchronize()
        for rnd in range(2):
            for v, k in zip(variants, ks):
                ms = time_ms(k, x, z, burst=100, reps=2)
                row = {**v, "round": rnd, "us": round(ms * 1e3, 1),
                       "GB/s": round(16 * N / ms / 1e6, 1)}
                rows.append(row)
                print(json.dumps(row), flush=True)
        Path(a.out).write_text(json.dumps(rows, indent=1))
        return
    if a.mode == "ops":       # every op line x every variant, same process
        rows = []
        for line in Path(a.ops).read_text().splitlines():
            if not line.strip():
                continue
            for v in json.loads(a.variants):
                try:
                    k = kernel(v, a.fma, line.strip(), pre)
                    ms = time_ms(k, x, z)
                    row = {"op": line.strip(), **v, "us": round(ms * 1e3, 1),
                           "GB/s": round(16 * N / ms / 1e6, 1),
                           "regs": rt.registers(k.vectorized.function(0))}
                except Exception as exc:  # noqa: BLE001
                    row = {"op": line.strip(), **v, "error": str(exc)[:300]}
                rows.append(row)
                print(json.dumps(row), flush=True)
        Path(a.out).write_text(json.dumps(rows, indent=1))
        return
    if a.mode == "one":
        v = json.loads(a.variant)
        k = kernel(v, a.fma, a.op, pre)
        for _ in range(a.launches):
            k(0.5, x, z)
        rt.synchronize()
        ms = time_ms(k, x, z)
        cfg = k.launch_config(0.5, x, z)
        print(json.dumps({"variant": v, "fma": a.fma, "us": round(ms * 1e3, 1),
                          "GB/s": round(16 * N / ms / 1e6, 1), **cfg}))
        return
    rows = []
    grid = itertools.product((128, 256, 512, 1024), (1, 2), (0, 1, 2, 4), (False, True),
                             ("default", "tma"), (0, 2, 3, 4, 6, 8))
    only = json.loads(a.variant) if a.variant != "{}" else {}
    for block, unroll, waves, prefetch, cache, stages in grid:
        if cache == "tma" and (unroll != 1 or prefetch or block < 128):
            continue
        if (prefetch or stages) and waves == 0:
            continue
        if stages and (prefetch or cache == "tma"):
            continue
        v = {"block": block, "unroll": unroll, "waves": waves, "prefetch": prefetch,
             "cache": cache, "stages": stages}
        if any(v.get(key) not in vals for key, vals in only.items()):
            continue
        try:
            k = kernel(v)
            ms = time_ms(k, x, z)
            cfg = k.launch_config(0.5, x, z)
            row = {**v, "us": round(ms * 1e3, 1), "GB/s": round(16 * N / ms / 1e6, 1),
                   "grid": cfg["grid"], "entry": cfg["entry"],
                   "regs": rt.registers(k.vectorized.function(0)) if k.vectorized else None}
        except Exception as exc:  # noqa: BLE001 - record and go on
            row = {**v, "error": str(exc)[:200]}
        rows.append(row)
        print(json.dumps(row), flush=True)
    ok = sorted((r for r in rows if "GB/s" in r), key=lambda r: -r["GB/s"])
    Path(a.out).parent.mkdir(parents=True, exist_ok=True)
    Path(a.out).write_text(json.dumps({"n": N, "op": OP, "rows": rows, "best": ok[:5]},
                                      indent=1))
    print("best", json.dumps(ok[:5]))


if __name__ == "__main__":
    main()
