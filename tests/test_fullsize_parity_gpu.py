"""Parity at the BASELINE sizes with SURVEY.md §8d's input distributions,
against the C oracle (the reference's acceptance pattern,
``tests/test_acceptance.py:274-308``, carried to n = 2^28 / 2^32).

* C2 dot f32 at 2^28, x, y ~ U(-1,1) seed 0: against the exact sum of the
  float32 products (what ``math.fsum`` gives), within the fp64-accumulation
  bound, and bit-equal to ``float32(fsum)`` -- the reference's own result
   -- for the default variant; also equal to the reference
  C kernel run on the same arrays.
* C3 f64 poly+sin at 2^28, x ~ U(-2,2), a = 0.5: 2^20 seeded random positions
  against the C oracle, within 4 ulp(sin x) + 1 ulp of the result.
* C4 at 2^32: int64 sum on x ~ U[-2^62, 2^62) seed 1 bit-exact (wrapping),
  max/min exact; max|x| on x ~ N(0,1) f32 seed 1 exact; L2 (sum of float32
  squares) within the bound and bit-equal to float32(fsum).  Inputs are
  generated on the host in 2^28-element chunks (one generator stream), each
  chunk uploaded into its slice and folded by the oracle's C reductions.
"""

import numpy as np
import pytest

from oracle import cport, csem
from paper_0911_3456_b200 import elementwise as ew, ndarray as nd, reduction as rd

pytestmark = pytest.mark.gpu

CHUNK = 1 << 28


def _threads():
    import os
    return max(1, len(os.sched_getaffinity(0)))


def test_c2_dot_2p28_against_exact_and_reference(kernel_env):
    kwargs, pool = kernel_env
    n = 1 << 28
    rng = np.random.default_rng(0)
    x = rng.uniform(-1, 1, n).astype(np.float32)
    y = rng.uniform(-1, 1, n).astype(np.float32)
    gx, gy = nd.from_host(pool, nd.float32, x), nd.from_host(pool, nd.float32, y)
    prods = x * y                                        # C: float * float -> float
    exact = csem.exact_f32_sum(prods)
    sum_abs = float(np.abs(prods, dtype=np.float64).sum())
    bound = 0.5 * float(np.spacing(np.float32(abs(exact)))) + n * 2.0**-53 * sum_abs
    want32 = np.float32(exact)
    ref = cport.Reduction("float *x, float *y", "float32", "0", "a + b", "x[i] * y[i]",
                          "dot_ref")(x, y, workers=_threads())
    assert ref == want32                                 # the reference is float32(fsum) here
    equal = 0
    variants = [None, ew.VariantParams(block=128, unroll=8), ew.VariantParams(block=1024, waves=2),
                ew.VariantParams(block=256, unroll=1, cache="tma")]
    for v in variants:
        got = rd.dot_kernel(nd.float32, v, **kwargs)(gx, gy)
        assert abs(float(got) - exact) <= bound, (v, got, exact)
        equal += got == want32
        if v is None:
            assert got == want32
    assert equal >= len(variants) - 1


def test_c3_polysin_2p28_sampled_against_oracle(kernel_env):
    kwargs, pool = kernel_env
    n = 1 << 28
    rng = np.random.default_rng(0)
    x = rng.uniform(-2, 2, n)
    gx = nd.from_host(pool, nd.float64, x)
    gz = pool.alloc_uninitialized(nd.float64, (n,))
    sig, op = "double a, double *x, double *z", \
        "z[i] = ((a*x[i] + 2.0)*x[i] - 1.5)*x[i] + sin(x[i])"
    ew.ElementwiseKernel(sig, op, "polysin_c3", **kwargs)(0.5, gx, gz)
    z = gz.to_host()
    idx = np.sort(np.random.default_rng(5).integers(0, n, 1 << 20))
    idx[0], idx[-1] = 0, n - 1                           # both ends of the span
    xs = np.ascontiguousarray(x[idx])
    want = np.zeros_like(xs)
    cport.Elementwise(sig, op, "polysin_c3")(0.5, xs, want, workers=_threads())
    got = z[idx]
    bound = 4 * np.spacing(np.abs(np.sin(xs))) + np.spacing(np.abs(want))
    assert np.all(np.abs(got - want) <= bound)
    assert np.mean(got == want) > 0.9


def _chunks(gen, total):
    for lo in range(0, total, CHUNK):
        yield lo, gen(min(CHUNK, total - lo))


def test_c4_int64_sum_max_min_2p32(kernel_env):
    kwargs, pool = kernel_env
    n = 1 << 32
    rng = np.random.default_rng(1)
    g = pool.alloc_uninitialized(nd.int64, (n,))
    s_ref = cport.Reduction("int64_t *x", "int64", "0", "a + b", None, "sum_ref")
    mx_ref = cport.Reduction("int64_t *x", "int64", "INT64_MIN", "a > b ? a : b", None, "max_ref")
    mn_ref = cport.Reduction("int64_t *x", "int64", "INT64_MAX", "a < b ? a : b", None, "min_ref")
    want_s, want_max, want_min = 0, -(1 << 63), (1 << 63) - 1
    for lo, h in _chunks(lambda m: rng.integers(-(1 << 62), 1 << 62, m, dtype=np.int64), n):
        g[lo:lo + h.size].copy_from_host(h)
        want_s += int(s_ref(h, workers=_threads()))
        want_max = max(want_max, int(mx_ref(h, workers=_threads())))
        want_min = min(want_min, int(mn_ref(h, workers=_threads())))
    want_s = (want_s + (1 << 63)) % (1 << 64) - (1 << 63)    # two's-complement wrap
    assert int(rd.sum_kernel(nd.int64, **kwargs)(g)) == want_s
    assert int(rd.max_kernel(nd.int64, **kwargs)(g)) == want_max
    assert int(rd.min_kernel(nd.int64, **kwargs)(g)) == want_min
    # a different CTA partition wraps to the same bits (order independent)
    v = ew.VariantParams(block=128, unroll=2, waves=2)
    assert int(rd.sum_kernel(nd.int64, v, **kwargs)(g)) == want_s
    g.free()


def test_c4_maxabs_and_l2_f32_2p32(kernel_env):
    kwargs, pool = kernel_env
    n = 1 << 32
    rng = np.random.default_rng(1)
    g = pool.alloc_uninitialized(nd.float32, (n,))
    mref = cport.Reduction("float *x", "float32", "0", "a > b ? a : b", "fabsf(x[i])",
                           "maxabs_ref")
    want_max = 0.0
    buckets = np.zeros(csem._EBINS, np.int64)
    sum_abs = 0.0
    for lo, h in _chunks(lambda m: rng.standard_normal(m, dtype=np.float32), n):
        g[lo:lo + h.size].copy_from_host(h)
        want_max = max(want_max, float(mref(h, workers=_threads())))
        sq = h * h                                       # C: float * float -> float
        buckets += csem.f32_buckets(sq)
        sum_abs += float(sq.sum(dtype=np.float64))
    maxabs = rd.make_reduction("float *x", nd.float32, "0", "a > b ? a : b", "fabsf(x[i])",
                               name="maxabs_c4", **kwargs)
    assert float(maxabs(g)) == want_max
    exact = float(csem.buckets_fraction(buckets))
    sumsq = rd.make_reduction("float *x", nd.float32, "0", "a + b", "x[i] * x[i]",
                              name="sumsq_c4", **kwargs)
    got = float(sumsq(g))
    bound = 0.5 * float(np.spacing(np.float32(exact))) + n * 2.0**-53 * sum_abs
    assert abs(got - exact) <= bound
    assert np.float32(got) == np.float32(exact)         # float32(fsum), the reference's result
    g.free()
