"""Untuned defaults for statements calling transcendentals: elementwise
f64 poly+sin and a sum-of-sin reduction at 2^28, the plain default vs the
register-pipelined loop (prefetch) over a few grids, sustained (100-launch
bursts after 2 s of heating: the board sits at its power cap)."""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402
from paper_0911_3456_b200 import _runtime as rt, autotune as at, elementwise as ew  # noqa: E402
from paper_0911_3456_b200 import ndarray as nd, reduction as rd  # noqa: E402

rt.set_device(0)
pool = nd.MemoryPool(device=0)
N = 1 << 28
x = nd.from_host(pool, nd.float64, np.random.default_rng(1).uniform(-2, 2, N))
z = pool.alloc_uninitialized(nd.float64, (N,))
o = pool.alloc_uninitialized(nd.float64, ())
ew_op = "z[i] = ((a*x[i] + 2.0)*x[i] - 1.5)*x[i] + sin(x[i])"
variants = [None, {"block": 128, "waves": 4, "prefetch": True},
            {"block": 256, "waves": 4, "prefetch": True}, {"block": 256, "waves": 1, "prefetch": True},
            {"block": 256, "waves": 2, "prefetch": True}, {"block": 128, "waves": 2, "prefetch": True}]
heat = ew.ElementwiseKernel("double a, double *x, double *z", ew_op, "heat")
for _ in range(2500):
    heat(0.5, x, z)
rt.synchronize()
rows = []
for kind in ("elementwise", "reduction"):
    for v in variants:
        vp = ew.VariantParams(**v) if v else None
        if kind == "elementwise":
            k = ew.ElementwiseKernel("double a, double *x, double *z", ew_op, "ps", vp)
            run, nbytes = (lambda k=k: k(0.5, x, z)), 16 * N
        else:
            k = rd.make_reduction("double *x", nd.float64, "0", "a + b", "sin(x[i]) * x[i]",
                                  name="sinsum", variant=vp)
            run, nbytes = (lambda k=k: k.launch(x, out=o, overlap_previous=True)), 8 * N
        timer = at.device_timer(run, 100)
        timer()
        s = min(timer() for _ in range(2))
        row = {"kind": kind, "variant": v or "default", "GB/s": round(nbytes / s / 1e9, 1)}
        rows.append(row)
        print(json.dumps(row), flush=True)
Path("gpurun_out/probe_heavy_defaults.json").write_text(json.dumps(rows, indent=1))
