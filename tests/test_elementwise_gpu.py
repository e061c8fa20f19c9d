"""GPU parity of generated elementwise kernels against the CPU oracle.

Everything here runs through ``ElementwiseKernel`` -> NVRTC cubin -> C-ABI
launch on the B200 and is compared with the reference's results: the golden
digests produced by rtcg-kit itself, and the pinned C oracle (``oracle/``) on
the same seeded inputs.  Bar: bit-exact (default ``-fmad=false``).
"""

import hashlib

import numpy as np
import pytest

from oracle import cport, csem
from paper_0911_3456_b200 import elementwise as ew, jit, ndarray as nd

pytestmark = pytest.mark.gpu


def digest(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


# --- the reference acceptance corpus (test_03): 11 ops x 10 dtypes x 5 sizes --------------

_VARIANTS = (ew.VariantParams(unroll=1, block=128, chunking="contiguous-blocks"),
             ew.VariantParams(unroll=4, block=256),
             ew.VariantParams(unroll=8, block=512, workers=3, chunking="contiguous-blocks"),
             ew.VariantParams(unroll=2, block=64, workers=5),
             ew.VariantParams(cache="tma", block=128, workers=3),
             ew.VariantParams(unroll=2, block=64, workers=3, prefetch=True))


@pytest.mark.parametrize("dname", csem.DTYPE_NAMES)
def test_corpus_bit_exact_vs_reference(golden, kernel_env, dname):
    kwargs, pool = kernel_env
    digests = golden["corpus"]["digests"]
    x_all, y_all = csem.corpus_operands()[dname]
    d = nd.BY_NAME[dname]
    bad = []
    from concurrent.futures import ThreadPoolExecutor
    jobs = [(op, shape, stmt, v) for op, shape, stmt in csem.CORPUS_OPS for v in _VARIANTS]
    with ThreadPoolExecutor(8) as ex:  # NVRTC runs outside the GIL
        kernels = list(ex.map(lambda j: ew.make_elementwise(
            csem.corpus_signature(j[1], d.cname), j[2], f"{j[0]}_{dname}", j[3], **kwargs), jobs))
    for (op, shape, stmt, variant), k in zip(jobs, kernels):
        if True:
            for n in csem.CORPUS_SIZES:
                ax = nd.from_host(pool, d, x_all[:n])
                ay = nd.from_host(pool, d, y_all[:n])
                az = pool.alloc(d, (n,))
                args = {"xy": (ax, ay, az), "axy": (3, ax, ay, az), "x": (ax, az)}[shape]
                k(*args, n=n)
                if digest(az.to_host()) != digests[f"{op}/{dname}/{n}"]:
                    bad.append((op, n, variant))
                for a in (ax, ay, az):
                    a.free()
    assert not bad, bad[:5]


def test_axpy_c1_bit_exact(golden, kernel_env):
    kwargs, pool = kernel_env
    g = golden["axpy_c1"]
    rng = np.random.default_rng(g["seed"])
    x = rng.uniform(-1, 1, g["n"]).astype(np.float32)
    y = rng.uniform(-1, 1, g["n"]).astype(np.float32)
    k = ew.ElementwiseKernel("float a, float *x, float b, float *y, float *z",
                             "z[i] = a * x[i] + b * y[i]", "axpy", **kwargs)
    ax, ay = nd.from_host(pool, nd.float32, x), nd.from_host(pool, nd.float32, y)
    az = pool.alloc(nd.float32, (g["n"],))
    k(g["a"], ax, g["b"], ay, az)
    assert k.launch_config(g["a"], ax, g["b"], ay, az)["entry"] == "axpy"  # vector path
    z = az.to_host()
    assert digest(z) == g["digest"]
    assert np.array_equal(z, np.float32(2.0) * x + np.float32(-3.0) * y)


def test_poly_sin_f64_within_ulp_bound(kernel_env):
    """C3 expression: sin differs between CUDA and glibc (parity unpinned by
    the reference's tests) -- bound: 4 ulp of sin(x) (CUDA <= 2 ulp, glibc <= 1)
    plus 1 ulp of the result for the final add."""
    from pathlib import Path
    kwargs, pool = kernel_env
    data = np.load(Path(__file__).parent / "golden" / "poly_sin_f64.npz")
    k = ew.ElementwiseKernel("double a, double *x, double *z",
                             "z[i] = ((a*x[i] + 2.0)*x[i] - 1.5)*x[i] + sin(x[i])", "polysin",
                             **kwargs)
    ax = nd.from_host(pool, nd.float64, data["x"])
    az = pool.alloc(nd.float64, data["x"].shape)
    k(float(data["a"]), ax, az)
    z = az.to_host()
    bound = 4 * np.spacing(np.abs(np.sin(data["x"]))) + np.spacing(np.abs(data["z"]))
    assert np.all(np.abs(z - data["z"]) <= bound)
    assert np.mean(z == data["z"]) > 0.9  # mostly bit-identical in practice


def test_fma_mode_within_term_magnitude_bound(shared_cache, pool):
    """-fmad=true: |err| <= 2 ulp(|a x| + |b y|) (BASELINE.md parity rule)."""
    cfg = jit.ToolchainConfig().with_fmad(True)
    rng = np.random.default_rng(0)
    n = 1 << 18
    x = rng.uniform(-1, 1, n).astype(np.float32)
    y = rng.uniform(-1, 1, n).astype(np.float32)
    k = ew.ElementwiseKernel("float a, float *x, float b, float *y, float *z",
                             "z[i] = a * x[i] + b * y[i]", "axpy_fma", config=cfg,
                             cache=shared_cache)
    ax, ay = nd.from_host(pool, nd.float32, x), nd.from_host(pool, nd.float32, y)
    az = pool.alloc(nd.float32, (n,))
    k(2.0, ax, -3.0, ay, az)
    z = az.to_host().astype(np.float64)
    ref = (np.float32(2.0) * x + np.float32(-3.0) * y).astype(np.float64)
    terms = np.abs(2.0 * x.astype(np.float64)) + np.abs(3.0 * y.astype(np.float64))
    assert np.all(np.abs(z - ref) <= 2 * np.spacing(terms.astype(np.float32)))


# --- reference execution tests (tests/test_elementwise.py:187-304) ----------------------------


def test_lincomb_matches_hand_oracle(kernel_env):
    kwargs, pool = kernel_env
    k = ew.make_elementwise("float a, float b, float *x, float *y, float *z",
                            "z[i] = a * x[i] + b * y[i]", "lin5", **kwargs)
    x = nd.from_host(pool, nd.float32, [1.0, 1.0])
    y = nd.from_host(pool, nd.float32, [1.0, 1.0])
    z = pool.alloc(nd.float32, (2,))
    k(2, 3, x, y, z)
    assert list(z.to_host()) == [5.0, 5.0]


def test_doubling_kernel(kernel_env):
    kwargs, pool = kernel_env
    k = ew.make_elementwise("float *x, float *y", "y[i] = 2 * x[i]", "dbl2", **kwargs)
    host = np.arange(7, dtype=np.float32)
    x = nd.from_host(pool, nd.float32, host)
    y = pool.alloc(nd.float32, (7,))
    k(x, y)
    assert np.array_equal(y.to_host(), host * 2)


def test_n_zero_writes_nothing(kernel_env):
    kwargs, pool = kernel_env
    k = ew.make_elementwise("float *x, float *z", "z[i] = 9", "nines", **kwargs)
    x = pool.alloc(nd.float32, (4,))
    z = nd.from_host(pool, nd.float32, [1.0, 2.0, 3.0, 4.0])
    k(x, z, n=0)
    assert list(z.to_host()) == [1.0, 2.0, 3.0, 4.0]


def test_explicit_n_limits_range(kernel_env):
    kwargs, pool = kernel_env
    k = ew.make_elementwise("float *x, float *z", "z[i] = x[i] + 1", "inc1", **kwargs)
    x = nd.from_host(pool, nd.float32, [1.0, 2.0, 3.0, 4.0])
    z = pool.alloc(nd.float32, (4,))
    k(x, z, n=2)
    assert list(z.to_host()) == [2.0, 3.0, 0.0, 0.0]


def test_arity_dtype_shape_errors(kernel_env):
    kwargs, pool = kernel_env
    k = ew.make_elementwise("float *x, float *z", "z[i] = x[i]", "cpy", **kwargs)
    x = pool.alloc(nd.float32, (2,))
    with pytest.raises(ew.ArityMismatch):
        k(x)
    with pytest.raises(ew.DtypeMismatch) as err:
        k(pool.alloc(nd.float64, (2,)), x)
    assert "x" in str(err.value)
    with pytest.raises(nd.ShapeMismatch):
        k(x, pool.alloc(nd.float32, (8,)), n=8)
    with pytest.raises(ew.DtypeMismatch):
        k(x, 3.0)
    with pytest.raises(nd.ShapeMismatch):
        k(x, x, n=-1)


def test_scalar_argument_conversion(kernel_env):
    kwargs, pool = kernel_env
    k = ew.make_elementwise("int32_t s, int32_t *x, int32_t *z", "z[i] = s * x[i]", "smul",
                            **kwargs)
    x = nd.from_host(pool, nd.int32, [1, 2, 3])
    z = pool.alloc(nd.int32, (3,))
    k(-4, x, z)
    assert list(z.to_host()) == [-4, -8, -12]


def test_scalar_widening_chain_matches_c(kernel_env):
    """Python float -> double -> declared type (uint8 wraps, float rounds)."""
    kwargs, pool = kernel_env
    k = ew.make_elementwise("uint8_t s, float f, uint8_t *x, float *z",
                            "z[i] = x[i] + s + f", "widen", **kwargs)
    x = nd.from_host(pool, nd.uint8, [1, 2, 3])
    z = pool.alloc(nd.float32, (3,))
    k(300, 0.1, x, z)
    zc = np.zeros(3, np.float32)
    cport.Elementwise("uint8_t s, float f, uint8_t *x, float *z", "z[i] = x[i] + s + f")(
        300, 0.1, np.array([1, 2, 3], np.uint8), zc)
    assert np.array_equal(z.to_host(), zc)


def test_multi_statement_operation(kernel_env):
    kwargs, pool = kernel_env
    k = ew.make_elementwise("float *x, float *z", "float t = x[i] * 2; z[i] = t + 1",
                            "two_step", **kwargs)
    x = nd.from_host(pool, nd.float32, [1.0, 2.0])
    z = pool.alloc(nd.float32, (2,))
    k(x, z)
    assert list(z.to_host()) == [3.0, 5.0]


def test_variant_invariance(kernel_env):
    kwargs, pool = kernel_env
    rng = np.random.default_rng(5)
    hx = rng.integers(-50, 50, size=1037, dtype=np.int32)
    hy = rng.integers(-50, 50, size=1037, dtype=np.int32)
    x, y = nd.from_host(pool, nd.int32, hx), nd.from_host(pool, nd.int32, hy)
    for unroll in (1, 2, 8, 16):
        for workers in (None, 1, 3):
            for chunking in ew.CHUNKINGS:
                z = pool.alloc(nd.int32, (1037,))
                v = ew.VariantParams(unroll=unroll, workers=workers, chunking=chunking,
                                     block=64)
                ew.make_elementwise("int32_t *x, int32_t *y, int32_t *z",
                                    "z[i] = x[i] * y[i] - x[i]", "vinv", v, **kwargs)(x, y, z)
                assert np.array_equal(z.to_host(), hx * hy - hx), v
                z.free()


# --- paths the vector analysis must route correctly -----------------------------------------


def test_index_value_and_neighbour_access(kernel_env):
    """Uses of i as a value and x[i+1] force the general path; results match C."""
    kwargs, pool = kernel_env
    n = 4099
    host = np.random.default_rng(1).uniform(-1, 1, n + 1).astype(np.float32)
    x = nd.from_host(pool, nd.float32, host)
    z = pool.alloc(nd.float32, (n,))
    k = ew.make_elementwise("float *x, float *z", "z[i] = x[i + 1] - x[i] + (float) i",
                            "diffi", **kwargs)
    assert k.vectorized is None
    k(x, z, n=n)
    zc = np.zeros(n, np.float32)
    cport.Elementwise("float *x, float *z", "z[i] = x[i + 1] - x[i] + (float) i")(host, zc, n=n)
    assert np.array_equal(z.to_host(), zc)


def test_i_as_value_on_vector_path(kernel_env):
    kwargs, pool = kernel_env
    n = 100_003
    z = pool.alloc(nd.int64, (n,))
    k = ew.make_elementwise("long *z", "z[i] = i * 3 - 7", "iota3", **kwargs)
    assert k.vectorized is not None
    k(z)
    assert np.array_equal(z.to_host(), np.arange(n, dtype=np.int64) * 3 - 7)


def test_conditional_write_keeps_untouched_elements(kernel_env):
    kwargs, pool = kernel_env
    host = np.arange(-500, 500, dtype=np.float32)
    x = nd.from_host(pool, nd.float32, host)
    z = nd.from_host(pool, nd.float32, np.full(1000, 7.0, np.float32))
    k = ew.make_elementwise("float *x, float *z", "if (x[i] > 0) z[i] = x[i]", "relu_keep",
                            **kwargs)
    k(x, z)
    assert np.array_equal(z.to_host(), np.where(host > 0, host, 7.0).astype(np.float32))


def test_in_place_and_compound_assignment(kernel_env):
    kwargs, pool = kernel_env
    host = np.random.default_rng(2).integers(-9, 9, 5001).astype(np.int16)
    x = nd.from_host(pool, nd.int16, host)
    ew.make_elementwise("int16_t *x", "x[i] *= 3; x[i] += 1", "inplace", **kwargs)(x)
    assert np.array_equal(x.to_host(), (host * 3 + 1).astype(np.int16))


def test_aliased_arguments_take_general_path(kernel_env):
    """z aliases x: the call must not use the restrict vector entry point."""
    kwargs, pool = kernel_env
    host = np.arange(4096, dtype=np.float32)
    a = nd.from_host(pool, nd.float32, host)
    k = ew.make_elementwise("float *x, float *z", "z[i] = x[i] * 2", "alias2", **kwargs)
    assert k.launch_config(a, a)["entry"] == "alias2_g"
    k(a, a)
    assert np.array_equal(a.to_host(), host * 2)


def test_mixed_width_vectors(kernel_env):
    """int8 and float64 vectors in one kernel: 16-element chunks."""
    kwargs, pool = kernel_env
    rng = np.random.default_rng(4)
    n = 70_001
    b = rng.integers(-100, 100, n).astype(np.int8)
    d = rng.uniform(-1, 1, n)
    k = ew.make_elementwise("int8_t *b, double *d, double *z", "z[i] = b[i] * d[i] + 0.5",
                            "mixw", **kwargs)
    assert k.width == 16
    gb, gd = nd.from_host(pool, nd.int8, b), nd.from_host(pool, nd.float64, d)
    gz = pool.alloc(nd.float64, (n,))
    k(gb, gd, gz)
    zc = np.zeros(n)
    cport.Elementwise("int8_t *b, double *d, double *z", "z[i] = b[i] * d[i] + 0.5")(b, d, zc)
    assert np.array_equal(gz.to_host(), zc)


def test_sharded_base_keeps_global_index(kernel_env):
    """A shard holding global indices [base, base+m) sees i as global."""
    kwargs, pool = kernel_env
    k = ew.make_elementwise("long *z", "z[i] = i", "gidx", **kwargs)
    for base, m in ((0, 1000), (3, 999), (1 << 20, 4097), (5, 3)):
        z = pool.alloc(nd.int64, (m,))
        k(z, base=base)
        assert np.array_equal(z.to_host(), np.arange(base, base + m)), base
        z.free()


def test_large_n_sampled_against_oracle(kernel_env):
    """2^26 elements; a random sample of positions checked against C."""
    kwargs, pool = kernel_env
    n = 1 << 26
    rng = np.random.default_rng(9)
    x = rng.uniform(-2, 2, n).astype(np.float32)
    y = rng.uniform(-2, 2, n).astype(np.float32)
    k = ew.make_elementwise("float a, float *x, float b, float *y, float *z",
                            "z[i] = a * x[i] + b * y[i]", "axpy_big", **kwargs)
    gx, gy = nd.from_host(pool, nd.float32, x), nd.from_host(pool, nd.float32, y)
    gz = pool.alloc(nd.float32, (n,))
    k(1.37, gx, -0.71, gy, gz)
    z = gz.to_host()
    assert np.array_equal(z, np.float32(1.37) * x + np.float32(-0.71) * y)


# --- adaptive factory and operators ------------------------------------------------------------


def test_adaptive_kernels(kernel_env):
    kwargs, pool = kernel_env
    x = nd.from_host(pool, nd.float64, [1.0, 2.0, 3.0, 4.0])
    y = nd.from_host(pool, nd.float32, np.full(4, 0.5, np.float32))
    k = ew.make_elementwise_adaptive([("x", x), ("y", y)], "out[i] = x[i] + y[i]",
                                     "ada_mix", **kwargs)
    assert k.result_dtype is nd.float64 and "float *y" in k.signature.render()
    out = pool.alloc(nd.float64, (4,))
    k(x, y, out)
    assert list(out.to_host()) == [1.5, 2.5, 3.5, 4.5]
    xi = nd.from_host(pool, nd.int32, [1, 2, 3])
    ks = ew.make_elementwise_adaptive([("x", xi), ("s", 2)], "out[i] = s * x[i]", "ada_s",
                                      **kwargs)
    assert "int32_t s" in ks.source
    o = pool.alloc(nd.int32, (3,))
    ks(xi, 2, o)
    assert list(o.to_host()) == [2, 4, 6]


def test_operators_promote_and_match_c(pool):
    x = nd.from_host(pool, nd.int32, [1, 2, 3])
    y = nd.from_host(pool, nd.float32, [1.5, 1.5, 1.5])
    z = x + y
    assert z.dtype is nd.float64 and list(z.to_host()) == [2.5, 3.5, 4.5]
    assert list((x * x).to_host()) == [1, 4, 9]
    assert (2 * x).dtype is nd.int32 and list((2 * x).to_host()) == [2, 4, 6]
    assert (nd.from_host(pool, nd.float32, [1.0]) * 0.5).dtype is nd.float64
    assert list((10 - x).to_host()) == [9, 8, 7]
    assert list((nd.from_host(pool, nd.int32, [7, -7]) / 2).to_host()) == [3, -3]
    assert list((12 / nd.from_host(pool, nd.float64, [2.0, 4.0])).to_host()) == [6.0, 3.0]
    with pytest.raises(nd.DivisionByZero):
        x / 0
    with pytest.raises(nd.ShapeMismatch):
        x + pool.alloc(nd.int32, (4,))
    h = np.random.default_rng(0).uniform(-1, 1, (4, 4)).astype(np.float32)
    z = nd.from_host(pool, nd.float32, h) * np.float32(2)
    assert z.shape == (4, 4) and np.array_equal(z.to_host(), h * np.float32(2))


def test_operator_matrix_against_c_port(pool):
    """Every dtype pair for + and /: promotion + C arithmetic vs the oracle."""
    rng = np.random.default_rng(8)
    for a in nd.DTYPES:
        for b in nd.DTYPES:
            ha = rng.integers(1, 50, 257).astype(a.np)
            hb = rng.integers(1, 50, 257).astype(b.np)
            ga, gb = nd.from_host(pool, a, ha), nd.from_host(pool, b, hb)
            for sym, pyop in (("+", lambda p, q: p + q), ("/", lambda p, q: p / q)):
                got = pyop(ga, gb)
                rt = nd.promote(a, b)
                assert got.dtype is rt
                zc = np.zeros(257, rt.np)
                cport.Elementwise(f"{a.cname} *x, {b.cname} *y, {rt.cname} *z",
                                  f"z[i] = ({rt.cname}) x[i] {sym} ({rt.cname}) y[i]")(ha, hb, zc)
                assert np.array_equal(got.to_host(), zc), (a, b, sym)
                got.free()


def test_cuda_array_interface_exposes_device_buffer(pool):
    torch = pytest.importorskip("torch")
    x = nd.from_host(pool, nd.float32, np.arange(10, dtype=np.float32))
    t = torch.as_tensor(x, device="cuda")
    assert t.data_ptr() == x.address
    assert torch.equal(t.cpu(), torch.arange(10, dtype=torch.float32))


def test_pinned_host_round_trip(pool):
    n = 1 << 20
    h = nd.pinned_empty((n,), nd.float32)
    h[:] = np.arange(n, dtype=np.float32)
    g = nd.from_host(pool, nd.float32, h)
    out = nd.pinned_empty((n,), nd.float32)
    g.to_host(out=out)
    assert np.array_equal(out, h)


def test_preamble_and_range(kernel_env):
    kwargs, pool = kernel_env
    pre = "__device__ float cube(float v) { return v * v * v; }"
    k = ew.ElementwiseKernel("float *x, float *z", "z[i] = cube(x[i])", "cubed",
                             preamble=pre, **kwargs)
    assert "__device__ float cube" in k.source and k.vectorized is not None
    h = np.arange(1000, dtype=np.float32) - 500
    x = nd.from_host(pool, nd.float32, h)
    z = nd.from_host(pool, nd.float32, np.full(1000, -1.0, np.float32))
    k(x, z, range=slice(10, 990))
    want = np.full(1000, -1.0, np.float32)
    want[10:990] = h[10:990] * h[10:990] * h[10:990]
    assert np.array_equal(z.get(), want)
    with pytest.raises(ValueError):
        k(x, z, range=slice(0, 10, 2))
    from paper_0911_3456_b200 import reduction as rd
    r = rd.ReductionKernel(np.float32, "0", "a + b", "cube(x[i])", "float *x", preamble=pre,
                           cache=kwargs["cache"], config=kwargs["config"])
    cubes = (h * h * h).astype(np.float64)      # float products, exact fp64 sum
    assert float(r(x).get()) == float(np.float32(np.sum(cubes)))


@pytest.mark.parametrize("n", [1, 3, 17, 1000, 65_537, 1_000_003])
def test_partition_covers_every_index_exactly_once(kernel_env, n):
    """SPEC 'worker-range partition' invariant, GPU form: a guard array
    incremented once per visited index ends up all ones inside [0, n) and
    untouched outside, for every partition / grid policy and both paths."""
    kwargs, pool = kernel_env
    guard = pool.alloc(nd.int32, (n + 5,))
    variants = [ew.VariantParams(unroll=u, block=b, chunking=c, waves=w, workers=wk)
                for u, b, c, w, wk in ((1, 256, "strided", None, None), (4, 64, "strided", 1, None),
                                       (16, 1024, "contiguous-blocks", 0, None),
                                       (2, 128, "contiguous-blocks", None, 7),
                                       (8, 32, "strided", None, 3))]
    variants += [ew.VariantParams(cache="tma", block=b, waves=w, workers=wk)
                 for b, w, wk in ((256, None, None), (64, None, 2), (1024, 2, None))]
    variants += [ew.VariantParams(unroll=u, block=b, waves=1, workers=wk, prefetch=True)
                 for u, b, wk in ((1, 256, None), (4, 64, 3), (2, 128, 1))]
    for v in variants:
        for op in ("g[i] += 1", "g[i] = g[i] + 1; if (i < 0) g[0] = 9"):
            guard.fill(0)
            ew.ElementwiseKernel("int32_t *g", op, "guard", v, **kwargs)(guard, n=n)
            got = guard.get()
            assert np.all(got[:n] == 1) and np.all(got[n:] == 0), (v, op)


def test_dot_invariants_and_f64_sum_tolerance(kernel_env):
    from paper_0911_3456_b200 import reduction as rd
    import math
    kwargs, pool = kernel_env
    rng = np.random.default_rng(13)
    h = rng.standard_normal(257)
    x = nd.from_host(pool, nd.float64, h)
    k = rd.dot_kernel(nd.float64, **kwargs)
    assert k(x, x) >= 0 and k(x, pool.alloc(nd.float64, (257,))) == 0.0
    big = rng.uniform(-1, 1, 10**6)
    got = float(rd.sum_kernel(nd.float64, **kwargs)(nd.from_host(pool, nd.float64, big)))
    exact = math.fsum(big.tolist())
    assert abs(got - exact) <= 1e-12 * abs(exact) or abs(got - exact) <= 1e-12 * np.abs(big).sum()


def test_double_sin_cos_within_two_ulp_of_glibc(kernel_env):
    """Double sin / cos in generated kernels (CUDA's libdevice) against glibc
    (math.sin / math.cos, the reference's libm) over |x| < 2, 1e5, 2^19,
    next to multiples of pi/2 and beyond 2^19: <= 2 ulp; signed zeros,
    infinities and NaNs as in C."""
    import math
    kwargs, pool = kernel_env
    rng = np.random.default_rng(31)
    half_pi = np.pi / 2
    k = np.arange(1, 3000, dtype=np.float64)
    near = np.concatenate([k * half_pi, np.nextafter(k * half_pi, 0),
                           np.nextafter(k * half_pi, np.inf)])
    x = np.concatenate([rng.uniform(-2, 2, 100_000), rng.uniform(-1e5, 1e5, 100_000),
                        rng.uniform(-2.0**19, 2.0**19, 50_000), near, -near,
                        rng.uniform(2.0**19, 1e9, 5_000), [0.0, -0.0, 5e-324, -1e-300, 1e-8]])
    gx = nd.from_host(pool, nd.float64, x)
    for fn, ref in (("sin", math.sin), ("cos", math.cos)):
        kern = ew.ElementwiseKernel("double *x, double *z", f"z[i] = {fn}(x[i])", f"t_{fn}",
                                    **kwargs)
        gz = pool.alloc(nd.float64, x.shape)
        kern(gx, gz)
        got = gz.to_host()
        want = np.array([ref(v) for v in x])
        ulps = np.abs(got - want) / np.spacing(np.abs(want))
        assert ulps.max() <= 2.0, (fn, x[np.argmax(ulps)], ulps.max())
        assert np.signbit(got[-4]) == np.signbit(want[-4])          # sin(-0) = -0
        assert np.mean(got == want) > 0.8       # measured 0.88-0.9: mostly identical
    special = nd.from_host(pool, nd.float64, np.array([np.inf, -np.inf, np.nan]))
    out = pool.alloc(nd.float64, (3,))
    ew.ElementwiseKernel("double *x, double *z", "z[i] = sin(x[i]) + cos(x[i])", "t_sc",
                         **kwargs)(special, out)
    assert np.all(np.isnan(out.to_host()))


@pytest.mark.parametrize("fn", ["sin", "cos"])
def test_double_sin_cos_bit_identical_to_cuda_library(kernel_env, fn):
    """The prelude's lean sin / cos (templates/prelude.cuh ``rtcg_trig``)
    return exactly the bits of CUDA's own double sin / cos (torch calls the
    library) -- on |x| < 2^31 by construction, beyond it, at inf / NaN and
    the signed zeros by the out-of-line library call -- over several
    magnitudes, next to multiples of pi/2, both quadrant parities, and
    through the vector, prefetch and cp.async-ring entry points."""
    torch = pytest.importorskip("torch")
    kwargs, pool = kernel_env
    rng = np.random.default_rng(41)
    half_pi = np.pi / 2
    k = np.arange(-5000, 5000, dtype=np.float64)
    near = np.concatenate([k * half_pi, np.nextafter(k * half_pi, -np.inf),
                           np.nextafter(k * half_pi, np.inf), (k + 0.5) * half_pi])
    x = np.concatenate([rng.uniform(-2, 2, 200_000), rng.uniform(-1e3, 1e3, 100_000),
                        rng.uniform(-2.0**31, 2.0**31, 100_000), near,
                        np.ldexp(rng.uniform(-1, 1, 20_000), rng.integers(-1074, 31, 20_000)),
                        rng.uniform(2.0**31 - 64, 2.0**31 + 64, 1000),
                        [2.0**31, -2.0**31, np.nextafter(2.0**31, 0), 1e300, -1e22,
                         0.0, -0.0, 5e-324, -5e-324, np.inf, -np.inf, np.nan]])
    want = getattr(torch, fn)(torch.from_numpy(x).cuda()).cpu().numpy()
    gx = nd.from_host(pool, nd.float64, x)
    for v in (ew.VariantParams(), ew.VariantParams(block=128, waves=4, prefetch=True),
              ew.VariantParams(block=256, unroll=2, waves=2, stages=2)):
        kern = ew.ElementwiseKernel("double *x, double *z", f"z[i] = {fn}(x[i])", f"b_{fn}",
                                    v, **kwargs)
        gz = pool.alloc(nd.float64, x.shape)
        kern(gx, gz)
        got = gz.to_host()
        same = (got.view(np.int64) == want.view(np.int64)) | (np.isnan(got) & np.isnan(want))
        assert same.all(), (fn, v, x[~same][:5], got[~same][:5], want[~same][:5])



@pytest.mark.parametrize("stages, unroll, block", [(2, 1, 128), (3, 2, 256), (4, 1, 256),
                                                   (8, 4, 64), (6, 1, 1024)])
def test_cp_async_ring_matches_the_register_path(kernel_env, stages, unroll, block):
    """``stages`` (per-thread cp.async ring) computes exactly what the plain
    vector path computes: read-only, read-write and mixed-width vectors,
    spans with unaligned heads/tails, shard bases, grids shorter than the
    ring (tiny n) -- and the C oracle agrees."""
    kwargs, pool = kernel_env
    rng = np.random.default_rng(stages * 10 + unroll)
    sig = "float a, float *x, double *y, double *z"
    op = "z[i] += a * x[i] * y[i] - (double) i"
    v_ring = ew.VariantParams(unroll=unroll, block=block, stages=stages, waves=1)
    v_plain = ew.VariantParams(unroll=unroll, block=block, waves=1)
    ring = ew.ElementwiseKernel(sig, op, "ring", v_ring, **kwargs)
    plain = ew.ElementwiseKernel(sig, op, "plain", v_plain, **kwargs)
    assert ring._async == (ring.smem > 0)
    assert ("rtcg::async::issue" in ring.source) == ring._async
    for n, lo in ((1 << 20, 0), (1_000_003, 3), (37, 1), (5, 0), (0, 0)):
        x = rng.uniform(-1, 1, n + lo).astype(np.float32)
        y = rng.uniform(-1, 1, n + lo)
        z0 = rng.uniform(-1, 1, n + lo)
        gx, gy = nd.from_host(pool, nd.float32, x), nd.from_host(pool, nd.float64, y)
        outs = []
        for k in (ring, plain):
            gz = nd.from_host(pool, nd.float64, z0)
            k(1.5, gx[lo:], gy[lo:], gz[lo:], base=7)
            outs.append(gz.to_host())
        assert outs[0].tobytes() == outs[1].tobytes(), (n, lo)
        want = z0.copy()
        cport.Elementwise(sig, op.replace("(double) i", "(double) (i + 7)"))(
            1.5, np.ascontiguousarray(x[lo:]), np.ascontiguousarray(y[lo:]), want[lo:])
        assert outs[0].tobytes() == want.tobytes(), (n, lo)


def test_cp_async_ring_variant_validation():
    with pytest.raises(ValueError):
        ew.VariantParams(stages=5)
    with pytest.raises(ValueError):
        ew.VariantParams(stages=4, prefetch=True)
    with pytest.raises(ValueError):
        ew.VariantParams(stages=4, cache="tma")
    # write-only statements have nothing to stage: the plain path is used
    k = ew.ElementwiseKernel("float *z", "z[i] = 1.0f", "wo", ew.VariantParams(stages=4))
    assert k.smem == 0 and not k._async and "cp.async.cg" not in k.source.split("end prelude")[1]
    # a ring beyond the shared-memory budget falls back to the plain path
    k = ew.ElementwiseKernel("float *x, double *y, double *z", "z[i] = x[i] * y[i]", "big",
                             ew.VariantParams(stages=8, unroll=4, block=1024))
    assert k.smem == 0 and not k._async


def test_general_entry_is_compiled_on_first_need(kernel_env, tmp_path):
    """Construction runs NVRTC once (the vector entry); aligned calls never
    build the general entry; a misaligned view builds it once, runs it
    correctly, and later misaligned calls go through the native plan."""
    from paper_0911_3456_b200 import jit
    kwargs, pool = kernel_env
    cache = jit.CacheStore(tmp_path / "lazy-cache")
    before = jit.compiler_spawn_count()
    k = ew.ElementwiseKernel("float a, float *x, float *z", "z[i] = a * x[i] + 1.0f",
                             "lazy_g", cache=cache, config=kwargs["config"])
    assert jit.compiler_spawn_count() - before == 1
    assert not k.generic.ready and "lazy_g_g(" not in k.source
    n = 100_003
    host = np.random.default_rng(2).uniform(-1, 1, n + 1).astype(np.float32)
    x, z = nd.from_host(pool, nd.float32, host), pool.alloc(nd.float32, (n + 1,))
    k(2.0, x, z)
    assert jit.compiler_spawn_count() - before == 1 and not k.generic.ready
    z2 = pool.alloc(nd.float32, (n,))
    k(2.0, x[1:], z2)                                   # 4-byte offset: general path
    assert k.generic.ready and jit.compiler_spawn_count() - before == 2
    assert np.array_equal(z2.get(), np.float32(2.0) * host[1:] + np.float32(1.0))
    assert np.array_equal(z.get(), np.float32(2.0) * host + np.float32(1.0))
    k(2.0, x[1:], z2)
    assert jit.compiler_spawn_count() - before == 2
    assert k.launch_config(2.0, x[1:], z2)["entry"] == "lazy_g_g"
