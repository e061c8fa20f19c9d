"""Launch one benchmark kernel with a given variant a few times, for ncu.

    python tools/profile_kernels.py dot '{"block":256,"unroll":1,"waves":2}'
    ncu --set full --clock-control none --import-source on -k regex:dot_k -s 2 -c 1 \
        -o gpurun_out/prof_dot python tools/profile_kernels.py dot '{...}'

Kernels: dot (f32, 2^28, the headline), axpy (f32, 2^28), polysin (f64,
2^28, C3), maxabs / sumsq (f32, 2^28 -- C4's per-launch pattern), sum_i64
(2^28).  Data are the bench's distributions.  Prints the launch config."""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402
from paper_0911_3456_b200 import _runtime as rt, elementwise as ew, ndarray as nd  # noqa: E402
from paper_0911_3456_b200 import reduction as rd  # noqa: E402

N = 1 << 28


def main():
    which = sys.argv[1]
    variant = ew.VariantParams(**json.loads(sys.argv[2] if len(sys.argv) > 2 else "{}"))
    launches = int(sys.argv[3]) if len(sys.argv) > 3 else 3
    rt.set_device(0)
    pool = nd.MemoryPool(device=0)
    rng = np.random.default_rng(0)
    if which in ("dot", "axpy"):
        x = nd.from_host(pool, nd.float32, rng.uniform(-1, 1, N).astype(np.float32))
        y = nd.from_host(pool, nd.float32, rng.uniform(-1, 1, N).astype(np.float32))
        if which == "dot":
            k = rd.ReductionKernel(rd.ReductionSpec("float *x, float *y", nd.float32, "0",
                                                    "a + b", "x[i] * y[i]"), "dot_k", variant)
            o = pool.alloc_uninitialized(nd.float32, ())
            run, cfg = (lambda: k.launch(x, y, out=o)), k.launch_config(x, y)
        else:
            z = pool.alloc_uninitialized(nd.float32, (N,))
            k = ew.ElementwiseKernel("float a, float *x, float b, float *y, float *z",
                                     "z[i] = a * x[i] + b * y[i]", "axpy", variant)
            run, cfg = (lambda: k(2.0, x, -3.0, y, z)), k.launch_config(2.0, x, -3.0, y, z)
    elif which == "polysin":
        x = nd.from_host(pool, nd.float64, rng.uniform(-2, 2, N))
        z = pool.alloc_uninitialized(nd.float64, (N,))
        k = ew.ElementwiseKernel("double a, double *x, double *z",
                                 "z[i] = ((a*x[i] + 2.0)*x[i] - 1.5)*x[i] + sin(x[i])",
                                 "polysin", variant)
        run, cfg = (lambda: k(0.5, x, z)), k.launch_config(0.5, x, z)
    elif which in ("maxabs", "sumsq"):
        x = nd.from_host(pool, nd.float32, rng.standard_normal(N, dtype=np.float32))
        red, mp = ("a > b ? a : b", "fabsf(x[i])") if which == "maxabs" else ("a + b",
                                                                          "x[i] * x[i]")
        k = rd.ReductionKernel(rd.ReductionSpec("float *x", nd.float32, "0", red, mp), which,
                               variant)
        o = pool.alloc_uninitialized(nd.float32, ())
        run, cfg = (lambda: k.launch(x, out=o)), k.launch_config(x)
    elif which == "sum_i64":
        x = nd.from_host(pool, nd.int64, rng.integers(-(1 << 62), 1 << 62, N, dtype=np.int64))
        k = rd.ReductionKernel(rd.ReductionSpec("int64_t *x", nd.int64, "0", "a + b"),
                               "sum_k", variant)
        o = pool.alloc_uninitialized(nd.int64, ())
        run, cfg = (lambda: k.launch(x, out=o)), k.launch_config(x)
    else:
        raise SystemExit(f"unknown kernel {which!r}")
    for _ in range(launches):
        run()
    rt.synchronize()
    print(json.dumps({"kernel": which, "variant": json.loads(sys.argv[2]) if len(sys.argv) > 2
                      else {}, **cfg}))


if __name__ == "__main__":
    main()
