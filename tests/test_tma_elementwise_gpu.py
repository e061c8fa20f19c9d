"""The elementwise TMA path (``cache="tma"``): inputs staged into a shared-
memory ring by cp.async.bulk, statements run by consumer warps.  It must give
bit-identical results to the LDG vector path and to the C oracle on every
shape the vector path accepts: head/tail elements outside whole tiles,
shard bases, ``range=`` slices, read-write and conditionally written vectors,
mixed element widths, spans shorter than one tile."""

import numpy as np
import pytest

from oracle import cport
from paper_0911_3456_b200 import elementwise as ew, ndarray as nd

pytestmark = pytest.mark.gpu

_TMA = (ew.VariantParams(cache="tma", block=256),
        ew.VariantParams(cache="tma", block=1024, waves=2),
        ew.VariantParams(cache="tma", block=64, workers=3),
        ew.VariantParams(cache="tma", block=128, waves=0))


def _tile(k):
    return k._per_thread_tma * k.variant.block


@pytest.mark.parametrize("v", _TMA, ids=lambda v: f"b{v.block}w{v.waves}k{v.workers}")
def test_axpy_bit_exact_across_tile_edges(kernel_env, v):
    kwargs, pool = kernel_env
    sig, op = "float a, float *x, float b, float *y, float *z", "z[i] = a * x[i] + b * y[i]"
    k = ew.make_elementwise(sig, op, "axpy_tma", v, **kwargs)
    assert k.smem > 0 and k.launch_config(*_dummy(pool, 1 << 16))["smem"] == k.smem
    tile = _tile(k)
    rng = np.random.default_rng(2)
    for n in (0, 1, 5, tile - 1, tile, tile + 3, 3 * tile + 17, 1_000_003):
        x = rng.uniform(-1, 1, n).astype(np.float32)
        y = rng.uniform(-1, 1, n).astype(np.float32)
        gx, gy = nd.from_host(pool, nd.float32, x), nd.from_host(pool, nd.float32, y)
        gz = pool.alloc(nd.float32, (max(n, 1),))
        k(2.0, gx, -3.0, gy, gz, n=n)
        zc = np.zeros(n, np.float32)
        cport.Elementwise(sig, op)(2.0, x, -3.0, y, zc)
        assert np.array_equal(gz.to_host()[:n], zc), n
        for a in (gx, gy, gz):
            a.free()


def _dummy(pool, n):
    x = pool.alloc(nd.float32, (n,))
    return 2.0, x, -3.0, x, pool.alloc(nd.float32, (n,))


def test_polysin_tma_equals_ldg_path(kernel_env):
    """Same compiled math on both paths: bit-identical f64 poly + sin."""
    kwargs, pool = kernel_env
    sig = "double a, double *x, double *z"
    op = "z[i] = ((a*x[i] + 2.0)*x[i] - 1.5)*x[i] + sin(x[i])"
    n = (1 << 22) + 11
    x = np.random.default_rng(3).uniform(-2, 2, n)
    gx = nd.from_host(pool, nd.float64, x)
    outs = []
    for v in (ew.VariantParams(), ew.VariantParams(cache="tma", block=1024),
              ew.VariantParams(cache="tma", block=512, waves=2)):
        gz = pool.alloc(nd.float64, (n,))
        ew.make_elementwise(sig, op, "polysin", v, **kwargs)(0.5, gx, gz)
        outs.append(gz.to_host())
    assert np.array_equal(outs[0], outs[1]) and np.array_equal(outs[0], outs[2])


@pytest.mark.parametrize("v", _TMA[:2], ids=["b256", "b1024"])
def test_read_write_and_conditional_vectors(kernel_env, v):
    kwargs, pool = kernel_env
    rng = np.random.default_rng(5)
    n = 300_007
    x = rng.integers(-50, 50, n).astype(np.int32)
    z0 = rng.integers(-50, 50, n).astype(np.int32)
    for op in ("z[i] += 3 * x[i]", "if (x[i] > 0) z[i] = x[i] * 2", "z[i] = z[i] ^ x[i]"):
        k = ew.make_elementwise("int32_t *x, int32_t *z", op, "rw_tma", v, **kwargs)
        assert k.smem > 0
        gx, gz = nd.from_host(pool, nd.int32, x), nd.from_host(pool, nd.int32, z0)
        k(gx, gz)
        zc = z0.copy()
        cport.Elementwise("int32_t *x, int32_t *z", op)(x, zc)
        assert np.array_equal(gz.to_host(), zc), op
        gx.free()
        gz.free()


def test_mixed_widths_and_write_only_outputs(kernel_env):
    kwargs, pool = kernel_env
    rng = np.random.default_rng(4)
    n = 170_001
    b = rng.integers(-100, 100, n).astype(np.int8)
    d = rng.uniform(-1, 1, n)
    sig = "int8_t *b, double *d, double *z, float *w"
    op = "z[i] = b[i] * d[i] + 0.5; w[i] = (float) d[i]"
    k = ew.make_elementwise(sig, op, "mixw_tma", ew.VariantParams(cache="tma"), **kwargs)
    assert k.width == 16 and k.smem > 0
    gb, gd = nd.from_host(pool, nd.int8, b), nd.from_host(pool, nd.float64, d)
    gz, gw = pool.alloc(nd.float64, (n,)), pool.alloc(nd.float32, (n,))
    k(gb, gd, gz, gw)
    zc, wc = np.zeros(n), np.zeros(n, np.float32)
    cport.Elementwise(sig, op)(b, d, zc, wc)
    assert np.array_equal(gz.to_host(), zc) and np.array_equal(gw.to_host(), wc)


def test_shard_base_and_range_slices(kernel_env):
    kwargs, pool = kernel_env
    k = ew.make_elementwise("long *x, long *z", "z[i] = x[i] + i", "gidx_tma",
                            ew.VariantParams(cache="tma", block=128), **kwargs)
    tile = _tile(k)
    for base, m in ((0, 5 * tile + 3), (3, 4 * tile), (1 << 20, 2 * tile + 1), (7, 9)):
        x = np.arange(m, dtype=np.int64) * 10
        gx, gz = nd.from_host(pool, nd.int64, x), pool.alloc(nd.int64, (m,))
        k(gx, gz, base=base)
        assert np.array_equal(gz.to_host(), x + np.arange(base, base + m)), base
        gx.free()
        gz.free()
    m = 6 * tile
    x = np.arange(m, dtype=np.int64)
    gx, gz = nd.from_host(pool, nd.int64, x), pool.alloc(nd.int64, (m,))
    lo, hi = tile // 2 + 1, 5 * tile - 3
    k(gx, gz, range=slice(lo, hi))
    want = np.zeros(m, np.int64)
    want[lo:hi] = 2 * x[lo:hi]
    assert np.array_equal(gz.to_host(), want)


def test_write_only_statement_has_no_tma_entry(kernel_env):
    """Nothing to stage: the variant keeps the LDG vector path."""
    kwargs, pool = kernel_env
    k = ew.make_elementwise("float *z", "z[i] = 1.5f", "fill_tma", ew.VariantParams(cache="tma"),
                            **kwargs)
    assert k.smem == 0
    z = pool.alloc(nd.float32, (1001,))
    k(z)
    assert np.all(z.to_host() == 1.5)


@pytest.mark.parametrize("cache", ["default", "tma"])
def test_user_names_that_match_template_locals(kernel_env, cache):
    """A scalar called ``k`` used to be shadowed by the chunk loop counter on
    the vector path (silently wrong values); names are now namespaced."""
    kwargs, pool = kernel_env
    rng = np.random.default_rng(8)
    n = 100_003
    c = rng.uniform(-1, 1, n).astype(np.float32)
    b = rng.uniform(-1, 1, n).astype(np.float32)
    k = ew.make_elementwise("float k, float *c, double E, float *b, float *s",
                            "s[i] = k * c[i] + (float) E * b[i]", "clash",
                            ew.VariantParams(cache=cache, unroll=2), **kwargs)
    gc, gb, gs = (nd.from_host(pool, nd.float32, c), nd.from_host(pool, nd.float32, b),
                  pool.alloc(nd.float32, (n,)))
    k(1.25, gc, -0.5, gb, gs)
    assert np.array_equal(gs.to_host(), np.float32(1.25) * c + np.float32(-0.5) * b)


@pytest.mark.parametrize("block", [64, 256, 1024])
def test_wide_tiles_shrink_or_fall_back_to_ldg(kernel_env, block):
    """int8 + double chunks are 16 elements (144 staged bytes per chunk): at
    block 1024 one chunk per consumer already exceeds the shared-memory budget
    for a 2-stage ring, so the variant keeps the LDG path; smaller blocks use
    the ring.  Results are identical either way."""
    kwargs, pool = kernel_env
    n = 250_007
    rng = np.random.default_rng(6)
    b = rng.integers(-9, 9, n).astype(np.int8)
    x = rng.uniform(-1, 1, n)
    k = ew.make_elementwise("int8_t *b, double *x, double *z", "z[i] = b[i] * x[i]", "wide",
                            ew.VariantParams(cache="tma", block=block), **kwargs)
    assert (k.smem > 0) == (block < 1024) and k.smem <= 227 * 1024
    gz = pool.alloc(nd.float64, (n,))
    k(nd.from_host(pool, nd.int8, b), nd.from_host(pool, nd.float64, x), gz)
    assert np.array_equal(gz.get(), b * x)
