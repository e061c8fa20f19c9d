"""GPU parity of generated reductions against the reference and the oracle.

Bars (BASELINE.md §2 / SURVEY.md §8c):
* integer reductions and max/min: bit-exact;
* float sums with fp64 accumulation: |got - fsum(terms)| <=
  1/2 ulp_out(result) + n * 2^-53 * sum|terms| (``oracle.csem.float_reduction_bound``),
  plus bitwise reproducibility for a fixed variant.
"""

import numpy as np
import pytest

from oracle import cport, csem
from paper_0911_3456_b200 import elementwise as ew, ndarray as nd, reduction as rd

pytestmark = pytest.mark.gpu

_VARIANTS = (ew.VariantParams(), ew.VariantParams(unroll=1, block=64, workers=7),
             ew.VariantParams(unroll=8, block=512, chunking="contiguous-blocks"),
             ew.VariantParams(unroll=2, block=1024, workers=1),
             ew.VariantParams(cache="tma", block=256),
             ew.VariantParams(cache="tma", block=64, workers=3),
             ew.VariantParams(unroll=4, block=256, chunk=8192),
             ew.VariantParams(unroll=1, block=128, chunk=1024, workers=5))


def test_reference_known_answers(kernel_env, golden):
    kwargs, pool = kernel_env
    assert rd.sum_kernel(nd.int32, **kwargs)(nd.from_host(pool, nd.int32, [1, 2, 3, 4])) == 10
    x = nd.from_host(pool, nd.float64, [1.0, 2.0])
    y = nd.from_host(pool, nd.float64, [3.0, 4.0])
    v = rd.dot_kernel(nd.float64, **kwargs)(x, y)
    assert v == 11.0 and isinstance(v, np.float64)
    assert rd.max_kernel(nd.float64, **kwargs)(pool.alloc(nd.float64, (0,))) == -np.inf
    assert rd.sum_kernel(nd.uint16, **kwargs)(pool.alloc(nd.uint16, (0,))) == 0
    i8 = nd.from_host(pool, nd.int8, [-128, 5, 127, -1])
    assert rd.max_kernel(nd.int8, **kwargs)(i8) == 127
    assert rd.min_kernel(nd.int8, **kwargs)(i8) == -128
    s16 = rd.sum_kernel(nd.int16, **kwargs)(nd.from_host(pool, nd.int16, [1, 2, 3]))
    assert s16.dtype == np.int16 and s16 == 6
    assert rd.sum_kernel(nd.int32, **kwargs)(nd.from_host(pool, nd.int32, [10, 20, 30, 40]),
                                             n=2) == 30
    cnt = rd.make_reduction("float t, float *x", nd.float32, "0", "a + b",
                            map_expr="(x[i] > t) ? 1.0f : 0.0f", name="count_above", **kwargs)
    assert cnt(0.6, nd.from_host(pool, nd.float32, [0.1, 0.9, 0.5, 0.7])) == 2.0


def test_int32_and_f32_folds_vs_reference_goldens(kernel_env, golden):
    kwargs, pool = kernel_env
    r = golden["reductions"]
    d = np.random.default_rng(7)
    ints = d.integers(-100, 101, size=5000).astype(np.int32)
    ai = nd.from_host(pool, nd.int32, ints)
    for v in _VARIANTS:
        got = [int(rd.sum_kernel(nd.int32, v, **kwargs)(ai)),
               int(rd.max_kernel(nd.int32, v, **kwargs)(ai)),
               int(rd.min_kernel(nd.int32, v, **kwargs)(ai))]
        assert got == r["int32_sum_max_min_seed7"], v
    floats = d.uniform(0.0, 1.0, size=10**6).astype(np.float32)
    af = nd.from_host(pool, nd.float32, floats)
    bound = csem.float_reduction_bound(floats, "float32")
    exact = csem.exact_sum(floats)
    for v in _VARIANTS:
        got = float(rd.sum_kernel(nd.float32, v, **kwargs)(af))
        assert abs(got - exact) <= bound
        assert abs(got - r["f32_sum_1e6_seed7_after_ints"]) / exact <= 1e-6


def test_int64_variants_exact(kernel_env, golden):
    kwargs, pool = kernel_env
    want = golden["reductions"]["int64_1003_seed11_sum_max_min"]
    host = np.random.default_rng(11).integers(-120, 120, size=1003, dtype=np.int64)
    x = nd.from_host(pool, nd.int64, host)
    for v in _VARIANTS:
        assert [int(rd.sum_kernel(nd.int64, v, **kwargs)(x)),
                int(rd.max_kernel(nd.int64, v, **kwargs)(x)),
                int(rd.min_kernel(nd.int64, v, **kwargs)(x))] == want


def test_wrapping_int64_sum_bit_exact(kernel_env, golden):
    """C4's int64 sum: values in [-2^62, 2^62) wrap; order independent."""
    kwargs, pool = kernel_env
    rng = np.random.default_rng(1)
    big = rng.integers(-(1 << 62), 1 << 62, size=1 << 20, dtype=np.int64)
    x = nd.from_host(pool, nd.int64, big)
    for v in _VARIANTS:
        assert int(rd.sum_kernel(nd.int64, v, **kwargs)(x)) == \
            golden["reductions"]["sum_i64_2p20_seed1"]


def test_dot_f32_vs_reference(kernel_env, golden):
    kwargs, pool = kernel_env
    for n, seed, key in ((1 << 20, 0, "dot_f32_2p20_seed0"), (1000, 3, "dot_f32_1000_seed3")):
        rng = np.random.default_rng(seed)
        x = rng.uniform(-1, 1, n).astype(np.float32)
        y = rng.uniform(-1, 1, n).astype(np.float32)
        gx, gy = nd.from_host(pool, nd.float32, x), nd.from_host(pool, nd.float32, y)
        terms = (x * y).astype(np.float64)   # products rounded in fp32, as in C
        bound = csem.float_reduction_bound(terms, "float32")
        exact = csem.exact_sum(terms)
        ref = golden["reductions"][key]
        equal = 0
        for v in _VARIANTS:
            got = float(rd.dot_kernel(nd.float32, v, **kwargs)(gx, gy))
            assert abs(got - exact) <= bound, (v, got, exact)
            equal += got == ref
        assert equal >= len(_VARIANTS) - 1  # fp64 accumulation: ties aside, bit-equal


def test_maxabs_and_sumsq_c4_expressions(kernel_env, golden):
    kwargs, pool = kernel_env
    rng = np.random.default_rng(1)
    g = rng.standard_normal(1 << 20).astype(np.float32)
    ag = nd.from_host(pool, nd.float32, g)
    mx = rd.make_reduction("float *x", nd.float32, "0", "a > b ? a : b", "fabsf(x[i])",
                           name="maxabs", **kwargs)
    assert float(mx(ag)) == golden["reductions"]["maxabs_f32_2p20_seed1"]
    sq = rd.make_reduction("float *x", nd.float32, "0", "a + b", "x[i] * x[i]",
                           name="sumsq", **kwargs)
    terms = (g * g).astype(np.float64)
    got = float(sq(ag))
    assert abs(got - csem.exact_sum(terms)) <= csem.float_reduction_bound(terms, "float32")
    assert abs(got - golden["reductions"]["sumsq_f32_2p20_seed1"]) <= \
        csem.float_reduction_bound(terms, "float32")


@pytest.mark.parametrize("dname", csem.DTYPE_NAMES)
def test_every_dtype_sum_max_min_vs_c_port(kernel_env, dname):
    kwargs, pool = kernel_env
    d = nd.BY_NAME[dname]
    rng = np.random.default_rng(17)
    n = 123_457
    host = (rng.uniform(-50, 50, n) if d.kind == "f" else
            rng.integers(0 if d.kind == "u" else -50, 50, n)).astype(d.np)
    x = nd.from_host(pool, d, host)
    for kind, neutral, expr in (("sum", "0", "a + b"),
                                ("max", rd._lowest(d), "a > b ? a : b"),
                                ("min", rd._highest(d), "a < b ? a : b")):
        got = rd.make_reduction(f"{d.cname} *x", d, neutral, expr, name=f"{kind}_{dname}",
                                **kwargs)(x)
        want = cport.Reduction(f"{d.cname} *x", dname, neutral, expr)(host, workers=4)
        if d.kind == "f" and kind == "sum":
            terms = host.astype(np.float64)
            assert abs(float(got) - csem.exact_sum(terms)) <= \
                csem.float_reduction_bound(terms, dname)
        else:
            assert got == want and got.dtype == want.dtype, (kind, got, want)


def test_float_sum_bitwise_reproducible(kernel_env):
    kwargs, pool = kernel_env
    host = np.random.default_rng(9).uniform(-1, 1, 1_000_003).astype(np.float32)
    x = nd.from_host(pool, nd.float32, host)
    for v in _VARIANTS:
        k = rd.sum_kernel(nd.float32, v, **kwargs)
        first = k(x)
        assert all(k(x) == first for _ in range(5))


def test_general_path_reduction_with_neighbour_access(kernel_env):
    kwargs, pool = kernel_env
    n = 50_001
    host = np.random.default_rng(3).uniform(-1, 1, n + 1)
    x = nd.from_host(pool, nd.float64, host)
    k = rd.make_reduction("double *x", nd.float64, "0", "a + b", "x[i+1] - x[i]",
                          name="tv", **kwargs)
    assert k.vectorized is None
    terms = np.diff(host)
    got = float(k(x, n=n))
    assert abs(got - csem.exact_sum(terms)) <= csem.float_reduction_bound(terms, "float64")


def test_neutral_probe(kernel_env):
    kwargs, pool = kernel_env
    with pytest.raises(ValueError):
        rd.make_reduction("int32_t *x", nd.int32, "7", "a + b", name="bad_neutral",
                          debug=True, **kwargs)
    k = rd.make_reduction("int32_t *x", nd.int32, "0", "a + b", name="good_neutral",
                          debug=True, **kwargs)
    assert k(nd.from_host(pool, nd.int32, [4, 5])) == 9


def test_pycuda_constructor_returns_device_scalar(kernel_env):
    kwargs, pool = kernel_env
    k = rd.ReductionKernel(np.float32, neutral="0", reduce_expr="a+b",
                           map_expr="x[i]*y[i]", arguments="float *x, float *y",
                           cache=kwargs["cache"], config=kwargs["config"])
    x = nd.from_host(pool, nd.float32, [1.0, 2.0, 3.0])
    y = nd.from_host(pool, nd.float32, [4.0, 5.0, 6.0])
    out = k(x, y)
    assert isinstance(out, nd.NdArray) and out.shape == () and out.get() == 32.0
    assert k(x, y, return_device=False) == np.float32(32.0)


def test_large_reduction_properties(kernel_env):
    """2^27 elements: dot(x, 1) == sum(x) bitwise for integers; float dot vs bound."""
    kwargs, pool = kernel_env
    n = 1 << 27
    rng = np.random.default_rng(21)
    xi = rng.integers(-1000, 1000, n, dtype=np.int64)
    ones = np.ones(n, np.int64)
    gx, go = nd.from_host(pool, nd.int64, xi), nd.from_host(pool, nd.int64, ones)
    assert int(rd.dot_kernel(nd.int64, **kwargs)(gx, go)) == int(xi.sum())
    assert int(rd.sum_kernel(nd.int64, **kwargs)(gx)) == int(xi.sum())
    xf = rng.uniform(-1, 1, n).astype(np.float32)
    gf = nd.from_host(pool, nd.float32, xf)
    got = float(rd.dot_kernel(nd.float32, **kwargs)(gf, gf))
    terms = (xf * xf).astype(np.float64)
    assert abs(got - float(np.sum(terms))) <= csem.float_reduction_bound(terms, "float32")


def test_c4_full_size_closed_forms(kernel_env):
    """BASELINE C4 sizes (n = 2^32) through size-independent properties with
    closed-form answers: inputs are generated on the device from i, and every
    checked value is exactly representable, so the bar stays bit-exact."""
    kwargs, pool = kernel_env
    n = 1 << 32
    xi = pool.alloc_uninitialized(nd.int64, (n,))
    ew.ElementwiseKernel("long *x", "x[i] = i", "iota64", **kwargs)(xi)
    s = int(rd.sum_kernel(nd.int64, **kwargs)(xi))
    assert s == (n * (n - 1) // 2 + 2**63) % 2**64 - 2**63
    assert int(rd.max_kernel(nd.int64, **kwargs)(xi)) == n - 1
    assert int(rd.min_kernel(nd.int64, **kwargs)(xi)) == 0
    xi.free()
    xf = pool.alloc_uninitialized(nd.float32, (n,))
    ew.ElementwiseKernel("float *x", "x[i] = (float) (i % 1024) - 511.0f", "saw",
                         **kwargs)(xf)
    block = np.arange(1024, dtype=np.float64) - 511.0
    reps = n // 1024
    mx = rd.make_reduction("float *x", nd.float32, "0", "a > b ? a : b", "fabsf(x[i])",
                           name="maxabs_c4", **kwargs)
    assert float(mx(xf)) == 512.0
    sq = rd.make_reduction("float *x", nd.float32, "0", "a + b", "x[i] * x[i]",
                           name="sumsq_c4", **kwargs)
    assert float(sq(xf)) == float(np.float32(reps * float(np.sum(block * block))))
    assert float(rd.sum_kernel(nd.float32, **kwargs)(xf)) == float(np.float32(
        reps * float(block.sum())))
    # elementwise at full size, checked through a reduction of its output
    z = pool.alloc_uninitialized(nd.float32, (n,))
    ew.ElementwiseKernel("float a, float *x, float b, float *z", "z[i] = a * x[i] + b",
                         "axpb_c4", **kwargs)(2.0, xf, 3.0, z)
    assert float(rd.sum_kernel(nd.float32, **kwargs)(z)) == float(np.float32(
        reps * float(np.sum(2.0 * block + 3.0))))


def test_threads_sharing_a_kernel_get_their_own_results(kernel_env):
    """Kernel objects are shareable between threads (reference SPEC:331): 8
    threads calling one sum kernel on the same stream each read their own
    result, every time."""
    from concurrent.futures import ThreadPoolExecutor
    kwargs, pool = kernel_env
    k = rd.sum_kernel(nd.int64, **kwargs)
    arrays = [nd.from_host(pool, nd.int64, np.full(100_000 + t, t, np.int64)) for t in range(8)]
    want = [t * (100_000 + t) for t in range(8)]

    def worker(t):
        from paper_0911_3456_b200 import _runtime
        _runtime.set_device(0)
        return all(int(k(arrays[t])) == want[t] for _ in range(50))
    with ThreadPoolExecutor(8) as ex:
        assert all(ex.map(worker, range(8)))


def test_synchronous_results_land_in_the_host_slot(kernel_env):
    """``kernel(x)`` has the last CTA store the value straight into a
    page-locked host slot (one per thread, shared by every kernel): calls
    alternating kernels, dtypes, empty spans (the combine kernel writes the
    neutral), streams and device-returning calls each read their own value."""
    from paper_0911_3456_b200 import _runtime
    kwargs, pool = kernel_env
    i8 = nd.from_host(pool, nd.int8, [-7, 3, 100, -128])
    f64 = nd.from_host(pool, nd.float64, np.arange(1000, dtype=np.float64))
    u64 = nd.from_host(pool, nd.uint64, np.full(5000, 3, np.uint64))
    mx8, s64, su = (rd.max_kernel(nd.int8, **kwargs), rd.sum_kernel(nd.float64, **kwargs),
                    rd.sum_kernel(nd.uint64, **kwargs))
    st = _runtime.Stream()
    for rep in range(20):
        assert mx8(i8) == 100
        assert s64(f64) == 499500.0
        assert s64(f64, n=0) == 0.0
        assert su(u64, stream=st) == 15000
        assert mx8(i8, n=2) == 3
        dev = s64(f64, return_device=True)
        assert s64(f64, n=10) == 45.0
        assert dev.to_host()[()] == 499500.0
        dev.free()
    assert rd._host_slot() == rd._host_slot()
    st.close()


def test_synchronous_call_waits_on_the_completion_word(kernel_env):
    """A synchronous call spins on its host slot's completion word (stored
    by the last CTA after the value) and blocks on the stream only after
    ``_SPIN_S``: behind a long kernel queued on the same stream the value is
    still this call's, and the word is set exactly when the kernel wrote
    the slot (empty spans fold through the combine entry and block)."""
    kwargs, pool = kernel_env
    big = pool.alloc(nd.float64, (1 << 27,))
    fill = ew.ElementwiseKernel("double *z", "z[i] = sin((double) i)", "fill_big", **kwargs)
    x = nd.from_host(pool, nd.float32, np.arange(1, 4097, dtype=np.float32))
    s = rd.sum_kernel(nd.float32, **kwargs)
    slot = rd._slot_object()
    for rep in range(5):
        fill(big)                           # ~1 ms of queued work ahead of the sum
        assert s(x) == 4096 * 4097 / 2
        assert slot.done.value == 1
        assert s(x, n=100) == 5050.0        # no queued work: the spin path
        assert s(x, n=0) == 0.0             # combine entry: no completion word
        assert slot.done.value == 0
    # a device-returning call and launch() without a host slot never write it
    dev = s(x, return_device=True)
    assert dev.to_host()[()] == 4096 * 4097 / 2 and slot.done.value == 0
    sc = s.launch(x, host_flag=True)
    assert sc.host_flagged is False
    dev.free()
    big.free()


@pytest.mark.parametrize("unroll,block,workers", [(1, 256, 296), (2, 128, 592), (4, 64, 148)])
def test_prefetch_pipeline_is_bit_identical(kernel_env, unroll, block, workers):
    """prefetch=True only moves loads earlier: with the same grid (pinned
    here -- the two variants' occupancy, hence their default grid, can
    differ) each thread folds the same chunks in the same order, so results
    are bitwise those of the plain loop (float dot, a transcendental map,
    wrapping int64 sum)."""
    kwargs, pool = kernel_env
    rng = np.random.default_rng(44)
    n = 2_000_003
    hx = rng.uniform(-2, 2, n).astype(np.float32)
    hy = rng.uniform(-2, 2, n).astype(np.float32)
    hi = rng.integers(-(1 << 62), 1 << 62, n, dtype=np.int64)
    x, y = nd.from_host(pool, nd.float32, hx), nd.from_host(pool, nd.float32, hy)
    xi = nd.from_host(pool, nd.int64, hi)
    got = {}
    for pf in (False, True):
        v = ew.VariantParams(unroll=unroll, block=block, workers=workers, prefetch=pf)
        got[pf] = (rd.dot_kernel(nd.float32, v, **kwargs)(x, y),
                   rd.make_reduction("float *x", nd.float64, "0", "a + b", "sin(x[i])",
                                     "sumsin", v, **kwargs)(x),
                   rd.sum_kernel(nd.int64, v, **kwargs)(xi))
    assert [g.tobytes() for g in got[True]] == [g.tobytes() for g in got[False]]
    assert int(got[True][2]) == int(hi.sum())


def test_overlapped_launches_give_the_same_results(kernel_env):
    """overlap_previous=True (programmatic dependent launch): consecutive
    reductions sharing one scratch, on the same and on different inputs,
    each produce exactly the result of an ordinary launch."""
    kwargs, pool = kernel_env
    rng = np.random.default_rng(51)
    n = 3_000_017
    hx = rng.uniform(-1, 1, n).astype(np.float32)
    hy = rng.uniform(-1, 1, n).astype(np.float32)
    x, y = nd.from_host(pool, nd.float32, hx), nd.from_host(pool, nd.float32, hy)
    dot = rd.dot_kernel(nd.float32, ew.VariantParams(waves=1), **kwargs)
    sq = rd.make_reduction("float *x", nd.float32, "0", "a + b", "x[i] * x[i]", "sq_ov",
                           ew.VariantParams(waves=2), **kwargs)
    want = (float(dot(x, y)), float(sq(x)), float(sq(y)))
    outs = [pool.alloc_uninitialized(nd.float32, ()) for _ in range(90)]
    for j in range(30):
        dot.launch(x, y, out=outs[3 * j], overlap_previous=True)
        sq.launch(x, out=outs[3 * j + 1], overlap_previous=True)
        sq.launch(y, out=outs[3 * j + 2], overlap_previous=True)
    got = [float(o.get()) for o in outs]
    assert got == list(want) * 30
    ints = nd.from_host(pool, nd.int64, rng.integers(-(1 << 62), 1 << 62, n, dtype=np.int64))
    for v in (ew.VariantParams(), ew.VariantParams(cache="tma", block=256, workers=5)):
        s = rd.sum_kernel(nd.int64, v, **kwargs)
        o = pool.alloc_uninitialized(nd.int64, ())
        for _ in range(20):
            s.launch(ints, out=o, overlap_previous=True)
        assert int(o.get()) == int(s(ints))
    general = rd.make_reduction("float *x", nd.float64, "0", "a + b", "x[i] * (double) (i & 3)",
                                "gen_ov", **kwargs)                       # uses i: general path
    og = pool.alloc_uninitialized(nd.float64, ())
    for _ in range(10):
        general.launch(x, out=og, overlap_previous=True)
    assert float(og.get()) == float(general(x))


def test_reduction_general_entry_is_compiled_on_first_need(kernel_env, tmp_path):
    """A reduction builds its vector entry and combine at construction, the
    general entry only when a call needs it (misaligned view), and both give
    the same fold."""
    from paper_0911_3456_b200 import jit
    kwargs, pool = kernel_env
    cache = jit.CacheStore(tmp_path / "lazy-red")
    before = jit.compiler_spawn_count()
    k = rd.sum_kernel(nd.int64, cache=cache, config=kwargs["config"])
    assert jit.compiler_spawn_count() - before == 1 and not k.generic.ready
    host = np.arange(100_001, dtype=np.int64)
    x = nd.from_host(pool, nd.int64, host)
    assert int(k(x)) == int(host.sum()) and not k.generic.ready
    assert int(k(x, n=0)) == 0 and not k.generic.ready          # empty span: the combine
    assert int(k(x[1:])) == int(host[1:].sum())                  # 8-byte offset: general
    assert k.generic.ready and jit.compiler_spawn_count() - before == 2
    assert int(k(x[1:])) == int(host[1:].sum())
    assert jit.compiler_spawn_count() - before == 2


def test_dynamic_chunks_exact_and_deterministic(kernel_env):
    """VariantParams.chunk (persistent CTAs taking chunks from a counter, one
    partial per chunk folded in chunk order): integer sums bit-exact against
    the C oracle at ragged sizes, base offsets and when the chunks must grow
    (more than MAX_CHUNKS minimum-size chunks); float results identical for
    every grid and call (the partials depend on the span, not on which CTA
    took a chunk) and within the n*eps bound."""
    kwargs, pool = kernel_env
    rng = np.random.default_rng(77)
    n_big = (ew.MAX_CHUNKS * 1024) + 4099           # chunk=1024 must grow to 2048
    hi = rng.integers(-(1 << 62), 1 << 62, n_big, dtype=np.int64)
    xi = nd.from_host(pool, nd.int64, hi)
    oracle = cport.Reduction("int64_t *x", "int64", "0", "a + b", None, "sum_dyn")
    for chunk, workers in ((1024, None), (8192, 3), (65536, 1)):
        k = rd.sum_kernel(nd.int64, ew.VariantParams(chunk=chunk, workers=workers), **kwargs)
        assert k.launch_config(xi)["entry"] == k.name          # the vector entry
        for n in (1, 7, 1023, 1024, 1025, 3 * 8192 + 5, (1 << 20) + 3, n_big):
            assert int(k(xi, n=n)) == int(oracle(hi, n=n)), (chunk, n)
        # a span starting at an aligned global offset that is not a chunk multiple
        o = pool.alloc_uninitialized(nd.int64, ())
        base = 12348
        k.launch(xi[base:], n=(1 << 20), base=base, out=o)
        assert int(o.get()) == int(oracle(hi[base:], n=1 << 20))
    hf = rng.uniform(-1, 1, n_big).astype(np.float32)
    hg = rng.uniform(-1, 1, n_big).astype(np.float32)
    xf, yf = nd.from_host(pool, nd.float32, hf), nd.from_host(pool, nd.float32, hg)
    terms = (hf * hg).astype(np.float64)
    exact, bound = csem.exact_sum(terms), csem.float_reduction_bound(terms, "float32")
    results = set()
    for workers in (None, 1, 7, 296):
        k = rd.dot_kernel(nd.float32, ew.VariantParams(unroll=2, chunk=1024, workers=workers),
                          **kwargs)
        for _ in range(3):
            got = float(k(xf, yf))
            assert abs(got - exact) <= bound
            results.add(got)
    assert len(results) == 1


def test_dynamic_chunks_overlapped_serial_and_captured(kernel_env):
    """The chunk counters are per scratch slot and re-armed by the last CTA:
    overlapped launches (alternating slots), serial launches and CUDA-graph
    replays, interleaved on one scratch, each give the ordinary result."""
    from paper_0911_3456_b200 import _runtime, graph
    kwargs, pool = kernel_env
    rng = np.random.default_rng(52)
    n = 5_000_011
    hx = rng.uniform(-1, 1, n).astype(np.float32)
    hy = rng.uniform(-1, 1, n).astype(np.float32)
    x, y = nd.from_host(pool, nd.float32, hx), nd.from_host(pool, nd.float32, hy)
    dot = rd.dot_kernel(nd.float32, ew.VariantParams(unroll=4, chunk=4096), **kwargs)
    want = float(dot(x, y))
    outs = [pool.alloc_uninitialized(nd.float32, ()) for _ in range(60)]
    for j in range(60):
        dot.launch(x, y, out=outs[j], overlap_previous=j % 3 != 2)
    assert [float(o.get()) for o in outs] == [want] * 60
    st = _runtime.Stream()
    with _runtime.use_stream(st.handle):
        o = pool.alloc_uninitialized(nd.float32, ())
        dot.launch(x, y, out=o)
        st.synchronize()
        g = graph.Graph(st)
        with g.capture():
            dot.launch(x, y, out=o, overlap_previous=True)
        for _ in range(5):
            g.launch()
        st.synchronize()
        assert float(o.get()) == want
        g.close()
    st.synchronize()
