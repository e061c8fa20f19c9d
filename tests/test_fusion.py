"""Expression-chain fusion: traced chains equal the eager operator chain bit
for bit, in one kernel launch and without temporaries."""

import ctypes

import numpy as np
import pytest

from paper_0911_3456_b200 import fusion, ndarray as nd


def host_pool():
    return nd.MemoryPool(lambda n: ctypes.create_string_buffer(n), zero_fill=lambda a, n: None)


def test_tracing_applies_eager_promotion_and_casts():
    pool = host_pool()
    x, y = pool.alloc(nd.int8, (10,)), pool.alloc(nd.float32, (10,))
    e = (fusion.lazy(x) * 2 + y) - x
    assert e.dtype is nd.float32 and len(e.arrays) == 2 and len(e.scalars) == 1
    assert e.scalars[0][1] is nd.int8          # Python int adopts the array dtype
    assert "((int8_t) ((int8_t) rtcg_fa0 * (int8_t) rtcg_fs0))" in e.text
    assert (fusion.lazy(y) * 0.5).dtype is nd.float64       # Python float is float64
    assert (fusion.lazy(y) * np.float32(0.5)).dtype is nd.float32
    assert (10 - fusion.lazy(x)).text.startswith("((int8_t) ((int8_t) rtcg_fs0 -")
    with pytest.raises(nd.DivisionByZero):
        fusion.lazy(x) / 0
    with pytest.raises(nd.ShapeMismatch):
        fusion.lazy(x) + pool.alloc(nd.int8, (11,))


def test_shared_leaves_are_deduplicated():
    pool = host_pool()
    x, y = pool.alloc(nd.float32, (4,)), pool.alloc(nd.float32, (4,))
    e = (fusion.lazy(x) + y) * (fusion.lazy(y) - x)
    assert len(e.arrays) == 2
    assert e.text.count("rtcg_fa0") == 2 and e.text.count("rtcg_fa1") == 2


@pytest.mark.gpu
@pytest.mark.parametrize("a_name, b_name", [("float32", "float32"), ("int8", "float32"),
                                            ("int16", "uint8"), ("int32", "float64"),
                                            ("uint32", "int64"), ("float32", "float64")])
def test_fused_chain_equals_eager_chain(pool, a_name, b_name):
    rng = np.random.default_rng(11)
    n = 100_003
    a_t, b_t = nd.BY_NAME[a_name], nd.BY_NAME[b_name]
    ha = (rng.uniform(-3, 3, n) if a_t.kind == "f" else rng.integers(1, 100, n)).astype(a_t.np)
    hb = (rng.uniform(-3, 3, n) if b_t.kind == "f" else rng.integers(1, 100, n)).astype(b_t.np)
    x, y = nd.from_host(pool, a_t, ha), nd.from_host(pool, b_t, hb)
    chains = [lambda p, q: (p * 2 + q) - p,
              lambda p, q: (p + q) * (q - p) / 3,
              lambda p, q: 7 - p * q + 0.25,
              lambda p, q: p * np.float32(1.5) - q / 2]
    for chain in chains:
        eager = chain(x, y)
        fused = fusion.fused(chain)(x, y)
        assert fused.dtype is eager.dtype
        assert np.array_equal(fused.get(), eager.get(), equal_nan=True)


@pytest.mark.gpu
def test_fused_chain_is_one_launch_and_no_temporaries(pool):
    x = nd.from_host(pool, nd.float32, np.arange(1 << 20, dtype=np.float32))
    y = nd.from_host(pool, nd.float32, np.ones(1 << 20, np.float32))
    before = pool.stats()["allocations_served"]
    f = fusion.fused(lambda p, q: ((p * 2 + q) - p) * q)
    z = f(x, y)
    assert pool.stats()["allocations_served"] - before == 1   # only the result
    kernel = fusion._kernel(fusion.lazy(x) * 2 + y - x, nd.float32)
    assert kernel.vectorized is not None
    assert np.array_equal(z.get(), (np.arange(1 << 20, dtype=np.float32) + 1))
    out = pool.alloc(nd.float32, (1 << 20,))
    assert f(x, y, out=out) is out


@pytest.mark.gpu
@pytest.mark.parametrize("dname", ["int8", "int32", "int64", "uint16", "float32", "float64"])
def test_fused_reductions_match_the_eager_chain(pool, dname):
    """reduce(chain) == gpuarray.<op>(evaluate(chain)): integer sums and
    max/min bit for bit; float sums fold the same per-element values in a
    possibly different CTA partition (the fused kernel's occupancy sets its
    grid), so they agree within the fp64-accumulation bound."""
    from paper_0911_3456_b200 import gpuarray as ga
    d = nd.BY_NAME[dname]
    rng = np.random.default_rng(12)
    n = 1_000_003
    hx = rng.integers(-50, 50, n).astype(d.np) if d.kind != "f" else \
        rng.uniform(-1, 1, n).astype(d.np)
    hy = rng.integers(0, 7, n).astype(d.np) if d.kind != "f" else \
        rng.uniform(-1, 1, n).astype(d.np)
    x, y = nd.from_host(pool, d, hx), nd.from_host(pool, d, hy)
    chain = (fusion.lazy(x) * 3 + y) - x
    eager = fusion.evaluate(chain)
    terms = np.abs(eager.get().astype(np.float64))
    bound = n * 2.0**-53 * terms.sum() + 0.5 * float(np.spacing(d.np.type(terms.sum()))) \
        if d.kind == "f" else 0
    for op, ref in (("sum", ga.sum), ("max", ga.max), ("min", ga.min)):
        got = fusion.reduce(chain, op).get()
        want = ref(eager).get()
        assert got.dtype == want.dtype
        if op == "sum" and d.kind == "f":
            assert abs(float(got) - float(want)) <= 2 * bound, (got, want)
        else:
            assert got.tobytes() == want.tobytes(), (op, got, want)
    f = fusion.fused(lambda p, q: p * q, reduce="max")
    assert f(x, y).get().tobytes() == ga.max(x * y).get().tobytes()


@pytest.mark.gpu
def test_fused_reduction_is_one_pass_without_temporaries(pool):
    n = 1 << 22
    x = nd.from_host(pool, nd.float32, np.ones(n, np.float32))
    y = nd.from_host(pool, nd.float32, np.full(n, 2.0, np.float32))
    before = pool.stats()["allocations_served"]
    r = fusion.reduce(fusion.lazy(x) * 2.5 + y, "sum", return_device=False)
    assert pool.stats()["allocations_served"] == before        # no temporaries, host scalar
    assert float(r) == 4.5 * n and isinstance(r, np.float64)   # Python float scalar -> f64
    with pytest.raises(ValueError):
        fusion.reduce(fusion.lazy(x), "prod")


# --- fused chains against the C oracle (not against the eager GPU chain) --------

from oracle import chain as och, cport  # noqa: E402

PAIRS = [("float32", "float32"), ("int8", "float32"), ("int16", "uint8"), ("int32", "float64"),
         ("uint32", "int64"), ("float32", "float64"), ("int8", "int8"), ("uint64", "int32"),
         ("int64", "int64"), ("uint16", "uint16")]
CHAINS = [lambda p, q: (p * 2 + q) - p,
          lambda p, q: (p + q) * (q - p) / 3,
          lambda p, q: 7 - p * q + 0.25,
          lambda p, q: p * np.float32(1.5) - q / 2,
          lambda p, q: (q - 100) / (p + 1) * p,
          lambda p, q: 2.5 / (q * q + 1) + np.int16(3) * p]


def _operands(a_name, b_name, n, seed=11):
    rng = np.random.default_rng(seed)
    out = []
    for name in (a_name, b_name):
        d = np.dtype(name)
        v = rng.uniform(-3, 3, n) if d.kind == "f" else rng.integers(1, 100, n)
        out.append(v.astype(d))
    return out


def _fused_source(expr):
    """Signature and statement of the kernel ``fusion`` generates for expr."""
    key, arrays, scalars = expr._leaves()
    params = [f"{a.dtype.cname} *rtcg_fa{k}" for k, a in enumerate(arrays)]
    params += [f"{sd.cname} rtcg_fs{k}" for k, (_, sd) in enumerate(scalars)]
    params.append(f"{expr.dtype.cname} *rtcg_fo")
    return ", ".join(params), "rtcg_fo[i] = " + fusion._render(key, "[i]") + ";", arrays, scalars


@pytest.mark.parametrize("a_name, b_name", PAIRS)
def test_fused_text_has_eager_c_semantics(a_name, b_name):
    """Host-only: the statement the fuser renders, compiled as C by the
    oracle, stores exactly what the reference's eager operator chain stores
    (each operator a separate reference kernel, src/elementwise.py:528-576)."""
    n = 4099
    ha, hb = _operands(a_name, b_name, n)
    pool = host_pool()
    x, y = pool.alloc(nd.BY_NAME[a_name], (n,)), pool.alloc(nd.BY_NAME[b_name], (n,))
    for chain in CHAINS:
        try:
            want = chain(och.HostArray(ha), och.HostArray(hb)).values
        except ZeroDivisionError:
            continue
        expr = chain(fusion.lazy(x), fusion.lazy(y))
        assert expr.dtype.name == want.dtype.name
        sig, stmt, arrays, scalars = _fused_source(expr)
        host = {id(x): ha, id(y): hb}
        got = np.zeros(n, want.dtype)
        cport.Elementwise(sig, stmt, "fused")(*[host[id(a)] for a in arrays],
                                              *[v for v, _ in scalars], got)
        assert got.tobytes() == want.tobytes(), (a_name, b_name, stmt)


@pytest.mark.gpu
@pytest.mark.parametrize("a_name, b_name", PAIRS)
def test_fused_and_eager_gpu_chains_equal_the_oracle(pool, a_name, b_name):
    n = 100_003
    ha, hb = _operands(a_name, b_name, n)
    x, y = nd.from_host(pool, nd.BY_NAME[a_name], ha), nd.from_host(pool, nd.BY_NAME[b_name], hb)
    for chain in CHAINS:
        try:
            want = chain(och.HostArray(ha), och.HostArray(hb)).values
        except ZeroDivisionError:
            continue
        fused = fusion.fused(chain)(x, y).get()
        eager = chain(x, y).get()
        assert fused.tobytes() == want.tobytes() == eager.tobytes(), (a_name, b_name)


@pytest.mark.gpu
@pytest.mark.parametrize("dname", ["int8", "int32", "int64", "uint16", "float32", "float64"])
def test_fused_reductions_equal_the_oracle(pool, dname):
    """reduce(chain) against the reference's stock reductions folded
    sequentially over the oracle's eager chain: integers and max/min bit for
    bit; float sums within the fp64-accumulation bound."""
    from oracle import csem
    d = nd.BY_NAME[dname]
    rng = np.random.default_rng(12)
    n = 1_000_003
    hx = rng.integers(-50, 50, n).astype(d.np) if d.kind != "f" else \
        rng.uniform(-1, 1, n).astype(d.np)
    hy = rng.integers(0, 7, n).astype(d.np) if d.kind != "f" else \
        rng.uniform(-1, 1, n).astype(d.np)
    x, y = nd.from_host(pool, d, hx), nd.from_host(pool, d, hy)
    terms = ((och.HostArray(hx) * 3 + och.HostArray(hy)) - och.HostArray(hx)).values
    for op in ("sum", "max", "min"):
        got = fusion.reduce((fusion.lazy(x) * 3 + y) - x, op).get()
        want = och.reduce(terms, op)
        assert got.dtype == want.dtype
        if op == "sum" and d.kind == "f":
            assert abs(float(got) - float(want)) <= 2 * csem.float_reduction_bound(terms, dname)
        else:
            assert got.tobytes() == np.asarray(want).tobytes(), (op, got, want)


@pytest.mark.gpu
def test_fused_trace_cache_is_keyed_by_dtypes_shapes_and_aliasing(pool):
    """A pure chain is traced once per argument signature; hits run the same
    kernel on the new arrays and give the uncached bits."""
    rng = np.random.default_rng(21)
    h = [rng.uniform(-2, 2, 4099).astype(np.float32) for _ in range(3)]
    x, y, w = (nd.from_host(pool, nd.float32, a) for a in h)
    f = fusion.fused(lambda p, q: (p * 2 + q) - p)
    first = f(x, y).get()
    assert f.cache_hits == 0
    again = f(w, y).get()                       # same signature, new arrays: a hit
    assert f.cache_hits == 1
    assert first.tobytes() == (och.HostArray(h[0]) * 2 + och.HostArray(h[1]) -
                               och.HostArray(h[0])).values.tobytes()
    assert again.tobytes() == (och.HostArray(h[2]) * 2 + och.HostArray(h[1]) -
                               och.HostArray(h[2])).values.tobytes()
    aliased = f(x, x).get()                     # aliasing changes the trace: a miss
    assert f.cache_hits == 1
    assert aliased.tobytes() == (och.HostArray(h[0]) * 2 + och.HostArray(h[0]) -
                                 och.HostArray(h[0])).values.tobytes()
    xd = nd.from_host(pool, nd.float64, h[0].astype(np.float64))
    assert f(xd, y).dtype is nd.float64 and f.cache_hits == 1     # new dtypes: a miss
    out = pool.alloc(nd.float32, (4099,))
    assert f(w, y, out=out) is out and f.cache_hits == 2
    assert out.get().tobytes() == again.tobytes()
    with pytest.raises(nd.ShapeMismatch):
        f(w, y, out=pool.alloc(nd.float64, (4099,)))
    r = fusion.fused(lambda p, q: p * q + 1, reduce="max")
    want = np.max(h[0] * h[1] + np.float32(1))
    assert r(x, y).get() == want and r(x, y).get() == want and r.cache_hits == 1
    scale = [2.0]
    g = fusion.fused(lambda p: p * scale[0])    # a closure: never cached
    g(x)
    scale[0] = 3.0
    assert np.array_equal(g(x).get(), h[0].astype(np.float64) * 3.0) and g.cache_hits == 0
