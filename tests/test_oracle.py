"""Pin the CPU oracle to the reference's own outputs (tests/golden/).

The oracle (``oracle/``) is test infrastructure: these checks prove that it
reproduces what rtcg-kit itself computed, so GPU parity against the oracle is
parity against the reference.
"""

import hashlib

import numpy as np
import pytest

from oracle import cport, csem


def digest(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


@pytest.fixture(scope="module")
def operands():
    return csem.corpus_operands()


def test_numpy_c_semantics_matches_reference_corpus(golden, operands):
    """All 11 ops x 10 dtypes x 5 sizes (reference test_03 corpus)."""
    digests = golden["corpus"]["digests"]
    assert len(digests) == 550
    bad = []
    for dname in csem.DTYPE_NAMES:
        x, y = operands[dname]
        for op, _, _ in csem.CORPUS_OPS:
            for n in csem.CORPUS_SIZES:
                got = csem.c_elementwise(op, x[:n], y[:n], dname)
                if digest(got) != digests[f"{op}/{dname}/{n}"]:
                    bad.append((op, dname, n))
    assert not bad, bad[:10]


@pytest.mark.parametrize("dname", ["int8", "uint16", "int64", "float32", "float64"])
def test_c_port_matches_reference_corpus(golden, operands, dname):
    digests = golden["corpus"]["digests"]
    x, y = operands[dname]
    cname = csem.CNAMES[dname]
    for op, shape, stmt in csem.CORPUS_OPS:
        k = cport.Elementwise(csem.corpus_signature(shape, cname), stmt, f"{op}_{dname}")
        for n in (7, 1000, 10**6):
            z = np.zeros(n, dtype=dname)
            args = {"xy": (x[:n], y[:n], z), "axy": (3, x[:n], y[:n], z), "x": (x[:n], z)}[shape]
            k(*args, workers=3)
            assert digest(z) == digests[f"{op}/{dname}/{n}"], (op, n)


def test_c_port_axpy_c1(golden):
    g = golden["axpy_c1"]
    rng = np.random.default_rng(g["seed"])
    x = rng.uniform(-1, 1, g["n"]).astype(np.float32)
    y = rng.uniform(-1, 1, g["n"]).astype(np.float32)
    z = np.zeros_like(x)
    cport.Elementwise("float a, float *x, float b, float *y, float *z",
                      "z[i] = a * x[i] + b * y[i]", "axpy")(g["a"], x, g["b"], y, z, workers=4)
    assert digest(z) == g["digest"]
    assert np.array_equal(z, np.float32(g["a"]) * x + np.float32(g["b"]) * y)


def test_c_port_reductions_match_reference(golden):
    r = golden["reductions"]
    d = np.random.default_rng(7)
    ints = d.integers(-100, 101, size=5000).astype(np.int32)
    got = [int(cport.Reduction("int32_t *x", "int32", "0", "a + b")(ints, workers=4)),
           int(cport.Reduction("int32_t *x", "int32", "INT32_MIN", "a > b ? a : b")(ints)),
           int(cport.Reduction("int32_t *x", "int32", "INT32_MAX", "a < b ? a : b")(ints))]
    assert got == r["int32_sum_max_min_seed7"]
    floats = d.uniform(0.0, 1.0, size=10**6).astype(np.float32)
    # the reference used os.cpu_count() workers; fp64 accumulation makes the
    # rounded float32 result insensitive to the split on this input
    s = cport.Reduction("float *x", "float32", "0", "a + b")(floats, workers=8)
    assert float(s) == r["f32_sum_1e6_seed7_after_ints"]

    def dot(n, seed):
        rng = np.random.default_rng(seed)
        x = rng.uniform(-1, 1, n).astype(np.float32)
        y = rng.uniform(-1, 1, n).astype(np.float32)
        return float(cport.Reduction("float *x, float *y", "float32", "0", "a + b",
                                     "x[i] * y[i]")(x, y, workers=8))
    assert dot(1 << 20, 0) == r["dot_f32_2p20_seed0"]
    assert dot(1000, 3) == r["dot_f32_1000_seed3"]

    rng = np.random.default_rng(1)
    g = rng.standard_normal(1 << 20).astype(np.float32)
    assert float(cport.Reduction("float *x", "float32", "0", "a > b ? a : b",
                                 "fabsf(x[i])")(g)) == r["maxabs_f32_2p20_seed1"]
    assert float(cport.Reduction("float *x", "float32", "0", "a + b",
                                 "x[i] * x[i]")(g, workers=8)) == r["sumsq_f32_2p20_seed1"]
    rng = np.random.default_rng(1)
    big = rng.integers(-(1 << 62), 1 << 62, size=1 << 20, dtype=np.int64)
    assert int(cport.Reduction("int64_t *x", "int64", "0", "a + b")(big, workers=5)) \
        == r["sum_i64_2p20_seed1"]


def test_c_port_poly_sin_matches_reference():
    from pathlib import Path
    data = np.load(Path(__file__).parent / "golden" / "poly_sin_f64.npz")
    z = np.zeros_like(data["x"])
    cport.Elementwise("double a, double *x, double *z",
                      "z[i] = ((a*x[i] + 2.0)*x[i] - 1.5)*x[i] + sin(x[i])", "ps")(
        float(data["a"]), data["x"], z)
    assert np.array_equal(z, data["z"])


def test_float_reduction_bound_is_sound_on_reference_values(golden):
    """The stated tolerance accepts the reference's own f32 sum."""
    d = np.random.default_rng(7)
    d.integers(-100, 101, size=5000)
    floats = d.uniform(0.0, 1.0, size=10**6).astype(np.float32)
    ref = golden["reductions"]["f32_sum_1e6_seed7_after_ints"]
    assert abs(ref - csem.exact_sum(floats)) <= csem.float_reduction_bound(floats, "float32")
