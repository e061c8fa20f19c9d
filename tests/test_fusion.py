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
