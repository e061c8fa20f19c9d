"""Seeded random C expressions: generated sm_100a kernels vs the C oracle.

Each case draws a signature (2-3 vectors of mixed dtypes, 0-2 scalars) and a
random expression tree over + - * / ?: and casts, then runs it through
``ElementwiseKernel`` on the GPU and through ``oracle.cport`` (the reference's
C semantics, gcc -O2 -ffp-contract=off) on identical inputs.  Bar: bit-exact.
Undefined behaviour is avoided by construction (divisors are nonzero and small,
no float->int casts of out-of-range values, no shifts), so both sides have one
defined answer.
"""

import numpy as np
import pytest

from oracle import cport
from paper_0911_3456_b200 import elementwise as ew, ndarray as nd, reduction as rd

pytestmark = pytest.mark.gpu

_INT = ("int8", "int16", "int32", "int64", "uint8", "uint16", "uint32", "uint64")
_FLT = ("float32", "float64")
_C = {"int8": "int8_t", "int16": "int16_t", "int32": "int32_t", "int64": "int64_t",
      "uint8": "uint8_t", "uint16": "uint16_t", "uint32": "uint32_t", "uint64": "uint64_t",
      "float32": "float", "float64": "double"}


def _expr(rng, leaves, depth, divisors, casts):
    if depth == 0 or rng.random() < 0.25:
        return str(rng.choice(leaves))
    kind = rng.integers(0, 6)
    a = _expr(rng, leaves, depth - 1, divisors, casts)
    b = _expr(rng, leaves, depth - 1, divisors, casts)
    if kind == 0:
        return f"({a} + {b})"
    if kind == 1:
        return f"({a} - {b})"
    if kind == 2:
        return f"({a} * {b})"
    if kind == 3:
        return f"({a} / {rng.choice(divisors)})"
    if kind == 4:
        return f"(({a}) < ({b}) ? {a} : {b})"
    return f"(({rng.choice(casts)}) ({a}))"


def _case(seed):
    """Three families, each free of undefined behaviour by construction:
    float (depth 3, |values| < 7^8, float->int casts in range), signed integer
    (depth 2: no signed overflow), unsigned (wrapping is defined; no casts
    through double)."""
    rng = np.random.default_rng(seed)
    family = ("float", "signed", "unsigned")[seed % 3]
    if family == "float":
        kinds, outs, scs = _FLT + ("int32", "int16"), _FLT, ("int32", "float64")
        depth, casts = 3, ["int", "long", "double", "float"]
    elif family == "signed":
        kinds, outs, scs = ("int8", "int16", "int32", "int64"), ("int32", "int64"), \
            ("int32", "int64")
        depth, casts = 2, ["int", "long", "double"]
    else:
        kinds, outs, scs = ("uint8", "uint16", "uint32", "uint64"), ("uint32", "uint64"), \
            ("uint32",)
        depth, casts = 3, ["unsigned int", "unsigned long"]
    nvec = int(rng.integers(2, 4))
    vec_types = [str(rng.choice(kinds)) for _ in range(nvec)]
    out_type = str(rng.choice(outs))
    nsc = int(rng.integers(0, 3))
    sc_types = [str(rng.choice(scs)) for _ in range(nsc)]
    names = [f"v{k}" for k in range(nvec)]
    leaves = [f"{n}[i]" for n in names] + [f"s{k}" for k in range(nsc)] + ["3", "7"]
    divisors = ["d[i]"] + [f"s{k}" for k in range(nsc) if not sc_types[k].startswith("float")]
    dtype_d = "uint32" if family == "unsigned" else "int32"
    expr = _expr(rng, leaves, depth, divisors, casts)
    sig = ", ".join([f"{_C[t]} *{n}" for t, n in zip(vec_types, names)] +
                    [f"{_C[t]} s{k}" for k, t in enumerate(sc_types)] +
                    [f"{_C[dtype_d]} *d", f"{_C[out_type]} *z"])
    return rng, sig, f"z[i] = {expr}", vec_types, sc_types, out_type, dtype_d


@pytest.mark.parametrize("seed", range(128))
def test_random_expression_bit_exact(kernel_env, seed):
    kwargs, pool = kernel_env
    rng, sig, op, vec_types, sc_types, out_type, dtype_d = _case(seed)
    n = int(rng.choice([1, 7, 1000, 65_537, 300_001]))
    host = []
    for t in vec_types:
        dt = np.dtype(t)
        host.append((rng.uniform(-4, 4, n) if dt.kind == "f" else
                     rng.integers(0 if dt.kind == "u" else -60, 60, n)).astype(dt))
    scalars = [float(rng.uniform(0.5, 3)) if t.startswith("float") else int(rng.integers(1, 9))
               for t in sc_types]
    d = rng.integers(1, 9, n).astype(np.int32)
    if dtype_d == "int32":
        d = d * rng.choice([-1, 1], n).astype(np.int32)
    d = d.astype(dtype_d)
    z_ref = np.zeros(n, np.dtype(out_type))
    cport.Elementwise(sig, op, "fz")(*host, *scalars, d, z_ref)
    variant = ew.VariantParams(unroll=int(rng.choice([1, 2, 4, 8])),
                               block=int(rng.choice([64, 256, 1024])),
                               chunking=str(rng.choice(ew.CHUNKINGS)),
                               waves=int(rng.choice([0, 1, 2])),
                               cache=str(rng.choice(["default", "default", "streaming",
                                                     "no-l1", "l2-256", "tma"])))
    k = ew.ElementwiseKernel(sig, op, f"fz{seed}", variant, **kwargs)
    dev = [nd.from_host(pool, nd.BY_NAME[t], h) for t, h in zip(vec_types, host)]
    gd = nd.from_host(pool, nd.BY_NAME[dtype_d], d)
    gz = pool.alloc(nd.BY_NAME[out_type], (n,))
    k(*dev, *scalars, gd, gz)
    got = gz.get()
    assert np.array_equal(got, z_ref, equal_nan=True), (sig, op, variant)


@pytest.mark.parametrize("seed", range(48))
def test_random_map_reduction_exact_for_integers(kernel_env, seed):
    kwargs, pool = kernel_env
    rng = np.random.default_rng(1000 + seed)
    t = str(rng.choice(("int64", "uint32", "uint64")))
    c = _C[t]
    expr = _expr(rng, ["x[i]", "y[i]", "5"], 2, ["3", "7"], ["long"] if t == "int64" else
                 ["unsigned long"])
    red, neutral = [("a + b", "0"), ("a > b ? a : b", rd._lowest(nd.BY_NAME[t])),
                    ("a < b ? a : b", rd._highest(nd.BY_NAME[t]))][seed % 3]
    n = int(rng.choice([1, 999, 100_003, 2_000_001]))
    x = rng.integers(0, 50, n).astype(t)
    y = rng.integers(0, 50, n).astype(t)
    want = cport.Reduction(f"{c} *x, {c} *y", t, neutral, red, expr)(x, y, workers=3)
    k = rd.make_reduction(f"{c} *x, {c} *y", nd.BY_NAME[t], neutral, red, expr,
                          name=f"rz{seed}", variant=ew.VariantParams(
                              unroll=int(rng.choice([1, 4, 8])),
                              block=int(rng.choice([128, 512])),
                              cache=str(rng.choice(["default", "l2-256", "tma"]))), **kwargs)
    got = k(nd.from_host(pool, nd.BY_NAME[t], x), nd.from_host(pool, nd.BY_NAME[t], y))
    assert got == want and got.dtype == want.dtype, (expr, red)
