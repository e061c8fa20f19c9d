"""The native launch path (``csrc/fastlaunch.cpp``) against the Python binder,
on CPU: a recording launcher stands in for ``rtcg_launch`` and captures the
entry point, grid, block, shared memory, stream and every 8-byte kernel
parameter; the same calls are marshalled by ``_codegen.Binder`` + the
vector-path rule + ``cg.grid_for``, and must agree exactly.  Calls the native
path must decline (wrong dtype, freed array, short vector, bad scalar) fall
back to the Python binder, which raises the reference's exceptions."""

import ctypes
import itertools
import subprocess

import numpy as np
import pytest

from paper_0911_3456_b200 import _build, _codegen as cg, _runtime
from paper_0911_3456_b200 import elementwise as ew, ndarray as nd

RECORDER = r"""
#include <stdint.h>
#include <string.h>
uint64_t rec_vals[128];
uint64_t rec_fn, rec_stream;
unsigned rec_grid, rec_block, rec_smem;
int rec_count, rec_calls;
unsigned rec_flags;
int record(void *fn, unsigned grid, unsigned block, unsigned smem, void *stream, void **params,
           unsigned flags) {
    rec_fn = (uint64_t)fn; rec_grid = grid; rec_block = block; rec_smem = smem; rec_flags = flags;
    rec_stream = (uint64_t)stream; rec_calls++;
    for (int k = 0; k < rec_count; ++k) memcpy(&rec_vals[k], params[k], 8);
    return 0;
}
"""

GEN_FN, VEC_FN, SMS, OCC = 0x1000, 0x2000, 148, 4


@pytest.fixture(scope="module")
def fl(tmp_path_factory):
    _build.build_fastlaunch()
    d = tmp_path_factory.mktemp("rec")
    (d / "rec.c").write_text(RECORDER)
    subprocess.run(["gcc", "-O1", "-shared", "-fPIC", str(d / "rec.c"), "-o", str(d / "rec.so")],
                   check=True)
    rec = ctypes.CDLL(str(d / "rec.so"))
    from paper_0911_3456_b200 import _fastlaunch
    _fastlaunch.set_launcher(ctypes.cast(rec.record, ctypes.c_void_p).value)
    yield _fastlaunch, rec
    # restore the real launcher: plans cached by other tests call it directly
    _fastlaunch.set_launcher(ctypes.cast(_runtime.lib().rtcg_launch_ex, ctypes.c_void_p).value)


@pytest.fixture()
def pool():
    addr = itertools.count(1 << 40, 1 << 24)   # 16 MiB apart, 256-byte aligned
    return nd.MemoryPool(system_alloc=lambda nbytes: next(addr), system_free=lambda a: None,
                         zero_fill=lambda a, n: None)


def _plan(fl_mod, sig, op, variant, nextra=0):
    sig = ew.parse_signature(sig)
    op = ew._normalize_operation(op)
    access = cg.analyze(op, [p.name for p in sig.vectors])
    width = cg.chunk_width(sig, access) if access else 0
    params = []
    for p in sig.params:
        acc = access[p.name] if access is not None and p.is_vector else None
        params.append((p.is_vector, p.dtype, p.dtype.size, p.dtype.kind,
                       bool(acc and acc.used), bool(acc and acc.written)))
    waves = 0 if variant.waves is None else variant.waves
    gen = (GEN_FN, variant.unroll, SMS * OCC, waves, 0)
    vec = (VEC_FN, variant.unroll * width, SMS * OCC, waves, 0) if access and width else None
    plan = fl_mod.Plan(params, nd.NdArray, variant.block, variant.workers or 0, gen, vec, nextra)
    return plan, sig, access, width


def _python_reference(sig, access, width, variant, args, n, base, nextra_vals=()):
    """What the Python binder + pick + grid policy would launch."""
    binder = cg.Binder(sig, extra=len(nextra_vals))
    errors = (ew.ArityMismatch, ew.DtypeMismatch, nd.ShapeMismatch, nd.NdArray)
    vals, _, vectors, n = binder.bind(args, n, base, "k", errors)
    binder.set_range(vals, base, base + n)
    for j, v in enumerate(nextra_vals):
        vals[binder.count + 2 + j] = v
    used = [(a, loc, p.dtype.size, access[p.name]) for p, a, loc in vectors
            if access and access[p.name].used] if access else []
    vec = access is not None and width and cg.vector_path_ok(used, n)
    fn = VEC_FN if vec else GEN_FN
    per = variant.unroll * width if vec else variant.unroll
    waves = 0 if variant.waves is None else variant.waves
    useful = max(1, -(-n // (variant.block * per)))
    grid = variant.workers or (useful if waves == 0 else min(SMS * OCC * waves, useful))
    return fn, grid, list(vals)


CASES = [
    ("float a, float *x, float b, float *y, float *z", "z[i] = a * x[i] + b * y[i]",
     lambda p, n: (2.5, p.alloc(nd.float32, (n,)), -3, p.alloc(nd.float32, (n,)),
                   p.alloc(nd.float32, (n,)))),
    ("int8_t *b, double *d, double *z", "z[i] = b[i] * d[i]",
     lambda p, n: (p.alloc(nd.int8, (n,)), p.alloc(nd.float64, (n,)), p.alloc(nd.float64, (n,)))),
    ("long k, uint64_t u, long *z", "z[i] = k + (long) u + i",
     lambda p, n: (-7, -1, p.alloc(nd.int64, (n,)))),
    ("float *x, float *z", "z[i] = x[i + 1]",      # general path only
     lambda p, n: (p.alloc(nd.float32, (n + 1,)), p.alloc(nd.float32, (n,)))),
]
VARIANTS = [ew.VariantParams(), ew.VariantParams(unroll=4, block=128, waves=1),
            ew.VariantParams(unroll=2, block=512, workers=7)]


@pytest.mark.parametrize("case", range(len(CASES)))
@pytest.mark.parametrize("variant", VARIANTS, ids=["default", "u4b128w1", "u2b512k7"])
@pytest.mark.parametrize("n,base", [(1, 0), (1000, 0), (1 << 20, 0), (4097, 3), (99, 1 << 33)])
def test_native_marshalling_equals_python_binder(fl, pool, case, variant, n, base):
    fl_mod, rec = fl
    sig_text, op, make = CASES[case]
    plan, sig, access, width = _plan(fl_mod, sig_text, op, variant)
    args = make(pool, n)
    total = len(sig.params) + 2
    ctypes.c_int.in_dll(rec, "rec_count").value = total
    got = plan.launch(args, None if case != 3 else n, base, 0x77, -1, ())
    fn, grid, vals = _python_reference(sig, access, width, variant, args,
                                       None if case != 3 else n, base)
    assert got == grid
    assert ctypes.c_uint64.in_dll(rec, "rec_fn").value == fn
    assert ctypes.c_uint.in_dll(rec, "rec_grid").value == grid
    assert ctypes.c_uint.in_dll(rec, "rec_block").value == variant.block
    assert ctypes.c_uint64.in_dll(rec, "rec_stream").value == 0x77
    assert list((ctypes.c_uint64 * total).in_dll(rec, "rec_vals")) == vals[:total]


def test_misalignment_and_aliasing_take_the_general_entry(fl, pool):
    fl_mod, rec = fl
    plan, *_ = _plan(fl_mod, "float *x, float *z", "z[i] = x[i] * 2", ew.VariantParams())
    ctypes.c_int.in_dll(rec, "rec_count").value = 4
    x = pool.alloc(nd.float32, (1000,))
    assert plan.launch((x, pool.alloc(nd.float32, (1000,))), None, 0, 0, -1, ()) > 0
    assert ctypes.c_uint64.in_dll(rec, "rec_fn").value == VEC_FN
    assert plan.launch((x, x), None, 0, 0, -1, ()) > 0            # in place: z aliases x
    assert ctypes.c_uint64.in_dll(rec, "rec_fn").value == GEN_FN
    assert plan.launch((x, pool.alloc(nd.float32, (1000,))), 999, 1, 0, -1, ()) > 0
    assert ctypes.c_uint64.in_dll(rec, "rec_fn").value == GEN_FN  # base 1: x[i] not 16B aligned


def test_declined_calls_and_limits(fl, pool):
    fl_mod, rec = fl
    plan, *_ = _plan(fl_mod, "float a, float *x, float *z", "z[i] = a * x[i]",
                     ew.VariantParams(), nextra=2)
    x, z = pool.alloc(nd.float32, (64,)), pool.alloc(nd.float32, (64,))
    calls = ctypes.c_int.in_dll(rec, "rec_calls")
    before = calls.value
    assert plan.launch((1.0, x), None, 0, 0, -1, (1, 2)) is None                # arity
    assert plan.launch((1.0, pool.alloc(nd.float64, (64,)), z), None, 0, 0, -1, (1, 2)) is None
    assert plan.launch((x, x, z), None, 0, 0, -1, (1, 2)) is None              # array scalar
    assert plan.launch(("a", x, z), None, 0, 0, -1, (1, 2)) is None            # bad scalar
    assert plan.launch((1.0, x, z), 65, 0, 0, -1, (1, 2)) is None               # short
    assert plan.launch((1.0, x, z), -1, 0, 0, -1, (1, 2)) is None               # negative n
    assert plan.launch((1.0, x, z), None, 0, 0, 0, (1, 2)) is None              # grid cap
    assert plan.launch((1.0, x, z), None, 0, 0, -1, (1,)) is None               # extras
    assert plan.launch((1.0, x, z), 0, 0, 0, -1, (1, 2)) == 0                   # empty
    gone = pool.alloc(nd.float32, (64,))
    gone.free()
    assert plan.launch((1.0, gone, z), None, 0, 0, -1, (1, 2)) is None         # freed
    assert calls.value == before
    ctypes.c_int.in_dll(rec, "rec_count").value = 7
    assert plan.launch((1.0, x, z), None, 0, 0, -1, (11, 22)) == 1
    assert ctypes.c_uint.in_dll(rec, "rec_flags").value == 0
    assert plan.launch((1.0, x, z), None, 0, 0, -1, (11, 22), 1) == 1
    assert ctypes.c_uint.in_dll(rec, "rec_flags").value == 1
    vals = list((ctypes.c_uint64 * 7).in_dll(rec, "rec_vals"))
    assert vals[3:] == [0, 64, 11, 22]
    assert np.float64(1.0).view(np.uint64) == vals[0]
