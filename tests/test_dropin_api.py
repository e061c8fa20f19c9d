"""The reference's public execution helpers, present under the same names
with GPU meaning (VERDICT r1 "drop-in API names"):
``elementwise.build_arg_pack`` / ``worker_ranges`` / ``run_ranges``
(``src/elementwise.py:29-35,276-366``), ``jit.KERNEL_ARGTYPES``
(``src/jit.py:538``) and ``csyntax.UNROLLED_ADD_TEMPLATE``
(``src/csyntax.py:535``).  Host-side behaviour runs here; the launches are
GPU tests."""

import ctypes

import numpy as np
import pytest
from hypothesis import given
from hypothesis import strategies as st

from paper_0911_3456_b200 import csyntax, elementwise as ew, jit, ndarray as nd


def host_pool():
    return nd.MemoryPool(lambda n: ctypes.create_string_buffer(n), zero_fill=lambda a, n: None)


def test_names_are_exported():
    for name in ("build_arg_pack", "run_ranges", "worker_ranges"):
        assert name in ew.__all__ and callable(getattr(ew, name))
    assert "KERNEL_ARGTYPES" in jit.__all__
    assert jit.KERNEL_ARGTYPES == (ctypes.POINTER(ctypes.c_void_p), ctypes.c_long, ctypes.c_long)
    assert "UNROLLED_ADD_TEMPLATE" in csyntax.__all__
    assert "${unroll}" in csyntax.UNROLLED_ADD_TEMPLATE
    assert csyntax.render(csyntax.UNROLLED_ADD_TEMPLATE, {
        "name": "v", "ctype": "float", "unroll": 2, "unrolled": True}) == \
        csyntax.unrolled_add_template(2, name="v")


@given(st.integers(0, 10_000), st.integers(1, 4), st.sampled_from(ew.CHUNKINGS))
def test_worker_ranges_partition(n, workers, chunking):
    """The reference's own property (tests/test_elementwise.py:113-129)."""
    ranges = ew.worker_ranges(n, ew.VariantParams(workers=workers, chunking=chunking))
    assert len(ranges) == workers
    if chunking == "contiguous-blocks":
        seen = set()
        for start, end in ranges:
            assert 0 <= start <= end <= n
            span = set(range(start, end))
            assert not (span & seen)
            seen |= span
        assert seen == set(range(n))
    else:
        assert ranges == [(k, n) for k in range(workers)]


def test_build_arg_pack_slots_and_errors():
    pool = host_pool()
    sig = ew.parse_signature("float a, float *x, uint16_t s, long *y")
    x, y = pool.alloc(nd.float32, (10,)), pool.alloc(nd.int64, (12,))
    pack, keep, n = ew.build_arg_pack(sig, [1.5, x, -1, y], None, extra_slots=3)
    assert n == 10 and len(pack) == 4 + 2 + 3 and pack.span_slot == 4
    assert ctypes.c_double.from_address(pack[0]).value == 1.5          # widened double
    assert ctypes.c_uint64.from_address(pack[1]).value == x.address     # device address
    assert ctypes.c_uint64.from_address(pack[2]).value == 2**64 - 1     # uint64, masked
    assert ctypes.c_uint64.from_address(pack[3]).value == y.address
    assert all(ctypes.c_int64.from_address(pack[k]).value == 0 for k in range(4, 9))
    assert len(keep) == 9
    with pytest.raises(ew.ArityMismatch):
        ew.build_arg_pack(sig, [1.5, x], None)
    with pytest.raises(ew.DtypeMismatch) as err:
        ew.build_arg_pack(sig, [1.5, y, 1, y], None)
    assert err.value.param == "x"
    with pytest.raises(ew.DtypeMismatch):
        ew.build_arg_pack(sig, [x, x, 1, y], None)
    with pytest.raises(ew.ShapeMismatch):
        ew.build_arg_pack(sig, [1.5, x, 1, y], 11)
    pack, _, n = ew.build_arg_pack("float *x", [x], 4)
    assert n == 4


def test_handle_call_needs_a_built_pack():
    handle = jit.KernelHandle("k", None)
    with pytest.raises(TypeError):
        handle((ctypes.c_void_p * 3)(), 0, 5)
    handle((ctypes.c_void_p * 3)(), 5, 5)          # empty range: nothing touched


@pytest.mark.gpu
@pytest.mark.parametrize("workers", [1, 3, 7])
def test_run_ranges_over_worker_ranges_launches_the_generated_kernel(pool, workers):
    """The reference's driving loop, verbatim in shape: pack once, one task
    per worker range, run_ranges -- here each task is a launch of the
    generated general entry point over its range."""
    n = 100_003
    host = np.random.default_rng(3).uniform(-1, 1, n).astype(np.float32)
    k = ew.ElementwiseKernel("float a, float *x, float *z", "z[i] = a * x[i] + 1", "ax1")
    x, z = nd.from_host(pool, nd.float32, host), pool.alloc(nd.float32, (n,))
    variant = ew.VariantParams(workers=workers)
    tasks = []
    for start, end in ew.worker_ranges(n, variant):
        pack, keep, _ = ew.build_arg_pack(k.signature, [2.0, x, z], n)
        tasks.append((pack, start, end, keep))
    ew.run_ranges(k.generic, [(p, s, e) for p, s, e, _ in tasks])
    assert np.array_equal(z.get(), np.float32(2.0) * host + np.float32(1.0))
    # a partial range touches only its span
    z2 = pool.alloc(nd.float32, (n,))
    pack, keep, _ = ew.build_arg_pack(k.signature, [2.0, x, z2], n)
    k.generic(pack, 10, 20)
    got = z2.get()
    assert np.all(got[:10] == 0) and np.all(got[20:] == 0)
    assert np.array_equal(got[10:20], np.float32(2.0) * host[10:20] + np.float32(1.0))


@pytest.mark.gpu
def test_numpy_scalar_on_the_left_follows_the_reference(pool):
    """``np.int16(3) * x`` reaches the array as the Python int 3 (numpy's
    fallback for unknown operands), so the result keeps x's dtype -- what
    the reference computes; ``x * np.int16(3)`` keeps the scalar's dtype."""
    x = nd.from_host(pool, nd.int8, np.arange(4, dtype=np.int8))
    left = np.int16(3) * x
    assert left.dtype is nd.int8 and list(left.get()) == [0, 3, 6, 9]
    assert (x * np.int16(3)).dtype is nd.int16
    assert (np.float32(0.5) * x).dtype is nd.float64       # Python float -> float64
    assert (np.int8(10) - x).get().tolist() == [10, 9, 8, 7]
