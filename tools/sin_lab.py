"""C3 `sin` formulation lab: the f64 poly + sin statement at 2^28 with CUDA's
library `sin` (spelled `(sin)`, which skips the prelude's macro), the
prelude's `sin` (templates/prelude.cuh `rtcg_trig`) and the lean
formulations of tools/sin_variants.cuh, each over a list of kernel variants.

    python tools/sin_lab.py [--variants '[{...}, ...]'] [--fns '(sin),sin,sin_l2']
                            [--out gpurun_out/sin_lab.json]

For every (formulation, variant): registers, a short-burst time (10-launch
bursts, best of 3) and, after ~2 s of heating, 100-launch sustained bursts in
two interleaved rounds (the board's power cap governs those).  Each
formulation's output is compared bit for bit with the library's over the
whole 2^28 array.  CUDA-event device times; GB/s uses 16 algorithmic bytes
per element.
"""
import argparse
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402
import torch  # noqa: E402
from paper_0911_3456_b200 import _runtime as rt, elementwise as ew, ndarray as nd  # noqa: E402

SIG = "double a, double *x, double *z"
N = 1 << 28
DEFAULT_VARIANTS = [
    {"block": 128, "unroll": 1, "waves": 4, "prefetch": True},
    {"block": 256, "unroll": 1, "waves": 4, "prefetch": True},
    {"block": 512, "unroll": 2, "waves": 2, "stages": 2},
    {"block": 512, "unroll": 2, "waves": 4, "stages": 2},
]


def op(fn: str) -> str:
    return f"z[i] = ((a*x[i] + 2.0)*x[i] - 1.5)*x[i] + {fn}(x[i])"


def time_ms(k, x, z, burst, reps):
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
    p.add_argument("--variants", default=json.dumps(DEFAULT_VARIANTS))
    p.add_argument("--fns", default="(sin),sin,sin_l2")
    p.add_argument("--out", default="gpurun_out/sin_lab.json")
    p.add_argument("--sustained-rounds", type=int, default=2)
    a = p.parse_args()
    rt.set_device(0)
    pool = nd.MemoryPool(device=0)
    pre = (Path(__file__).resolve().parent / "sin_variants.cuh").read_text()
    hx = np.random.default_rng(1).uniform(-2, 2, N)
    x = nd.from_host(pool, nd.float64, hx)
    z = pool.alloc_uninitialized(nd.float64, (N,))
    variants = json.loads(a.variants)
    fns = a.fns.split(",")
    ks = {(f, i): ew.ElementwiseKernel(SIG, op(f), "polysin", ew.VariantParams(**v), preamble=pre)
          for f in fns for i, v in enumerate(variants)}
    rows = []
    # bit identity against the library formulation (variant 0 of each)
    ref = None
    bits = {}
    for f in fns:
        ks[(f, 0)](0.5, x, z)
        rt.synchronize()
        t = torch.as_tensor(z, device="cuda").clone()
        if ref is None:
            ref = t
        bits[f] = int((t.view(torch.int64) != ref.view(torch.int64)).sum().item())
        del t
    print(json.dumps({"bit_mismatches_vs_" + fns[0]: bits}), flush=True)
    for (f, i), k in ks.items():
        ms = time_ms(k, x, z, 10, 3)
        row = {"fn": f, **variants[i], "phase": "burst", "us": round(ms * 1e3, 1),
               "GB/s": round(16 * N / ms / 1e6, 1), "regs": rt.registers(k.vectorized.function(0))}
        rows.append(row)
        print(json.dumps(row), flush=True)
    heat = ks[(fns[0], 0)]
    for _ in range(3000):
        heat(0.5, x, z)
    rt.synchronize()
    for rnd in range(a.sustained_rounds):
        for (f, i), k in ks.items():
            ms = time_ms(k, x, z, 100, 2)
            row = {"fn": f, **variants[i], "phase": f"sustained{rnd}", "us": round(ms * 1e3, 1),
                   "GB/s": round(16 * N / ms / 1e6, 1)}
            rows.append(row)
            print(json.dumps(row), flush=True)
    Path(a.out).parent.mkdir(parents=True, exist_ok=True)
    Path(a.out).write_text(json.dumps({"bits": bits, "rows": rows}, indent=1))


if __name__ == "__main__":
    main()
