"""Generate the golden fixtures by running the REFERENCE implementation.

Run in the build container only (it imports rtcg-kit from /root/reference):

    python tests/golden/make_golden.py

Writes ``tests/golden/reference_outputs.json`` (sha256 digests of reference
outputs + reduction values) and ``tests/golden/poly_sin_f64.npz`` (reference
output of the C3 expression on a small sample).  Inputs are regenerated from
the seeds recorded in the JSON, so the fixtures stay small; the GPU box never
needs /root/reference.
"""

from __future__ import annotations

import hashlib
import json
import os
import sys
import tempfile
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parent.parent))  # repo root, for oracle.csem
REF_SRC = Path("/root/reference/pkg/src")


def digest(arr: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(arr).tobytes()).hexdigest()


def main() -> int:
    if not REF_SRC.is_dir():
        print("reference tree not present; fixtures unchanged", file=sys.stderr)
        return 1
    os.environ.setdefault("RTCG_CACHE_DIR", tempfile.mkdtemp(prefix="rtcg-ref-cache-"))
    sys.path.insert(0, str(REF_SRC))
    from rtcg import elementwise as ew, ndarray as nd, reduction as rd  # noqa: E402
    from oracle import csem  # noqa: E402

    pool = nd.MemoryPool()
    out: dict = {"generator": "tests/golden/make_golden.py",
                 "reference": "rtcg-kit @ /root/reference/pkg/src"}

    # 1. acceptance corpus (tests/test_acceptance.py:182-228), one variant --
    #    the reference guarantees all variants agree
    corpus = {}
    operands = csem.corpus_operands()
    for dname in csem.DTYPE_NAMES:
        d = nd.BY_NAME[dname]
        x_host, y_host = operands[dname]
        for op, shape, stmt in csem.CORPUS_OPS:
            k = ew.make_elementwise(csem.corpus_signature(shape, d.cname), stmt,
                                    f"{op}_{dname}", ew.VariantParams(unroll=4, workers=2))
            for n in csem.CORPUS_SIZES:
                ax, ay = nd.from_host(pool, d, x_host[:n]), nd.from_host(pool, d, y_host[:n])
                az = pool.alloc(d, (n,))
                args = {"xy": (ax, ay, az), "axy": (3, ax, ay, az), "x": (ax, az)}[shape]
                k(*args, n=n)
                corpus[f"{op}/{dname}/{n}"] = digest(az.to_host())
                for a in (ax, ay, az):
                    a.free()
    out["corpus"] = {"seed": csem.CORPUS_SEED, "digests": corpus}

    # 2. C1: axpy f32 n=2^20, x,y ~ U(-1,1) seed 0, a=2, b=-3 (src/cli.py:187,196-207)
    n = 1 << 20
    rng = np.random.default_rng(0)
    x = rng.uniform(-1, 1, n).astype(np.float32)
    y = rng.uniform(-1, 1, n).astype(np.float32)
    k = ew.make_elementwise("float a, float *x, float b, float *y, float *z",
                            "z[i] = a * x[i] + b * y[i]", "axpy")
    ax, ay, az = nd.from_host(pool, nd.float32, x), nd.from_host(pool, nd.float32, y), \
        pool.alloc(nd.float32, (n,))
    k(2.0, ax, -3.0, ay, az)
    z = az.to_host()
    assert np.array_equal(z, np.float32(2.0) * x + np.float32(-3.0) * y)
    out["axpy_c1"] = {"n": n, "seed": 0, "a": 2.0, "b": -3.0, "digest": digest(z)}

    # 3. reductions
    red = {}
    d = np.random.default_rng(7)
    ints = d.integers(-100, 101, size=5000).astype(np.int32)
    ai = nd.from_host(pool, nd.int32, ints)
    red["int32_sum_max_min_seed7"] = [int(rd.sum_kernel(nd.int32)(ai)),
                                      int(rd.max_kernel(nd.int32)(ai)),
                                      int(rd.min_kernel(nd.int32)(ai))]
    floats = d.uniform(0.0, 1.0, size=10**6).astype(np.float32)
    red["f32_sum_1e6_seed7_after_ints"] = float(rd.sum_kernel(nd.float32)(nd.from_host(
        pool, nd.float32, floats)))

    def dot_f32(n, seed):
        r = np.random.default_rng(seed)
        xx = r.uniform(-1, 1, n).astype(np.float32)
        yy = r.uniform(-1, 1, n).astype(np.float32)
        return float(rd.dot_kernel(nd.float32)(nd.from_host(pool, nd.float32, xx),
                                               nd.from_host(pool, nd.float32, yy)))
    red["dot_f32_2p20_seed0"] = dot_f32(1 << 20, 0)
    red["dot_f32_1000_seed3"] = dot_f32(1000, 3)

    r = np.random.default_rng(1)
    g = r.standard_normal(1 << 20).astype(np.float32)
    ag = nd.from_host(pool, nd.float32, g)
    red["maxabs_f32_2p20_seed1"] = float(rd.make_reduction(
        "float *x", nd.float32, "0", "a > b ? a : b", "fabsf(x[i])")(ag))
    red["sumsq_f32_2p20_seed1"] = float(rd.make_reduction(
        "float *x", nd.float32, "0", "a + b", "x[i] * x[i]")(ag))
    r = np.random.default_rng(1)
    big = r.integers(-(1 << 62), 1 << 62, size=1 << 20, dtype=np.int64)
    red["sum_i64_2p20_seed1"] = int(rd.sum_kernel(nd.int64)(nd.from_host(pool, nd.int64, big)))
    r = np.random.default_rng(11)
    h = r.integers(-120, 120, size=1003, dtype=np.int64)
    ah = nd.from_host(pool, nd.int64, h)
    red["int64_1003_seed11_sum_max_min"] = [int(rd.sum_kernel(nd.int64)(ah)),
                                            int(rd.max_kernel(nd.int64)(ah)),
                                            int(rd.min_kernel(nd.int64)(ah))]
    out["reductions"] = red

    # 4. C3: f64 ((a*x+2)*x-1.5)*x + sin(x), x ~ U(-2,2) seed 5, a = 0.5, n = 4096
    r = np.random.default_rng(5)
    xp = r.uniform(-2, 2, 4096)
    k = ew.make_elementwise("double a, double *x, double *z",
                            "z[i] = ((a*x[i] + 2.0)*x[i] - 1.5)*x[i] + sin(x[i])", "polysin")
    ax, az = nd.from_host(pool, nd.float64, xp), pool.alloc(nd.float64, (4096,))
    k(0.5, ax, az)
    np.savez_compressed(HERE / "poly_sin_f64.npz", x=xp, z=az.to_host(), a=0.5)

    (HERE / "reference_outputs.json").write_text(json.dumps(out, indent=1, sort_keys=True) + "\n")
    print(f"wrote {len(corpus)} corpus digests, {len(red)} reduction values")
    return 0


if __name__ == "__main__":
    raise SystemExit(main())
