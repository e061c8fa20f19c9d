"""Signature parsing, variants, vector-path analysis and CUDA generation.

NVRTC compiles sm_100a cubins without a GPU, so generated kernels are
compiled here and their SASS inspected for 128-bit accesses."""

import os
import shutil
import subprocess

import pytest
from hypothesis import given
from hypothesis import strategies as st

from paper_0911_3456_b200 import _codegen as cg
from paper_0911_3456_b200 import elementwise as ew
from paper_0911_3456_b200 import jit
from paper_0911_3456_b200 import ndarray as nd
from paper_0911_3456_b200 import reduction as rd


# --- signatures (reference tests/test_elementwise.py:21-92) -------------------------------


def test_parse_scalar_vector_and_aliases():
    sig = ew.parse_signature("float a, float *x")
    assert [(p.name, p.is_vector, p.dtype.name) for p in sig.params] == \
        [("a", False, "float32"), ("x", True, "float32")]
    sig = ew.parse_signature("double *z, int n0")
    assert [(p.name, p.is_vector, p.dtype.name) for p in sig.params] == \
        [("z", True, "float64"), ("n0", False, "int32")]
    assert ew.parse_signature("long *q").params[0].dtype is nd.int64
    assert ew.parse_signature("uint8_t *b").params[0].dtype is nd.uint8
    assert ew.parse_signature("short *s").params[0].dtype is nd.int16


def test_parse_errors():
    with pytest.raises(ew.ParseError):
        ew.parse_signature("")
    with pytest.raises(ew.ParseError) as err:
        ew.parse_signature("float a, float b")
    assert "vector" in str(err.value)
    for bad in ("float *i", "long n, float *v", "float *args, float *z", "int start, float *v",
                "int end, float *v", "float *rtcg_x"):
        with pytest.raises(ew.ParseError):
            ew.parse_signature(bad)
    with pytest.raises(ew.ParseError):
        ew.parse_signature("float *x, float *x")
    with pytest.raises(ew.UnknownType):
        ew.parse_signature("quux *x")
    with pytest.raises(ew.UnknownType):
        ew.parse_signature("complex64 *x")
    with pytest.raises(ew.ParseError) as err:
        ew.parse_signature("float *x, ???")
    assert err.value.position == len("float *x,")


_ident = st.from_regex(r"[a-hj-mo-qs-z][a-z0-9_]{0,5}", fullmatch=True).filter(
    lambda s: s not in ew.RESERVED_NAMES)


@given(st.lists(st.tuples(_ident, st.sampled_from(sorted(nd.BY_CNAME)), st.booleans()),
                min_size=1, max_size=6, unique_by=lambda t: t[0]))
def test_parse_round_trips_generated_signatures(params):
    if not any(vec for _, _, vec in params):
        params = params + [("rv", "float", True)]  # "r..." is never drawn by _ident
    text = ", ".join(f"{c} {'*' if v else ''}{n}" for n, c, v in params)
    sig = ew.parse_signature(text)
    assert ew.parse_signature(sig.render()) == sig and len(sig.params) == len(params)


def test_variant_validation_and_defaults():
    v = ew.VariantParams()
    assert (v.unroll, v.workers, v.chunking, v.block, v.cache, v.waves) == \
        (1, None, "strided", 256, "default", None)
    assert v.resolved() is v
    for bad in (dict(unroll=3), dict(workers=0), dict(workers=ew.MAX_WORKERS + 1),
                dict(chunking="round-robin"), dict(block=100), dict(cache="bogus"),
                dict(waves=3)):
        with pytest.raises(ValueError):
            ew.VariantParams(**bad)


# --- vector-path analysis ----------------------------------------------------------------------


@pytest.mark.parametrize("text, expect", [
    ("z[i] = a*x[i] + b*y[i];", {"x": (1, 0), "y": (1, 0), "z": (0, 1)}),
    ("z[ i ] = x [i];", {"x": (1, 0), "y": (0, 0), "z": (0, 1)}),
    ("z[i] += x[i];", {"x": (1, 0), "y": (0, 0), "z": (1, 1)}),
    ("z[i]++;", {"x": (0, 0), "y": (0, 0), "z": (1, 1)}),
    ("++z[i];", {"x": (0, 0), "y": (0, 0), "z": (1, 1)}),
    ("if (x[i] > 0) z[i] = y[i];", {"x": (1, 0), "y": (1, 0), "z": (1, 1)}),
    ("float t = x[i]; z[i] = t; y[i] = t;", {"x": (1, 0), "y": (0, 1), "z": (0, 1)}),
    ("z[i] = x[i] == y[i];", {"x": (1, 0), "y": (1, 0), "z": (0, 1)}),
    ("z[i] = s.x[i];", {"x": (0, 0), "y": (0, 0), "z": (0, 1)}),
])
def test_analysis_classifies_accesses(text, expect):
    got = cg.analyze(text, ["x", "y", "z"])
    assert {k: (int(v.read), int(v.written)) for k, v in got.items()} == expect


@pytest.mark.parametrize("text", ["z[i] = x[i+1];", "z[i] = x[0];", "z[i] = *x;",
                                  "float *p = &x[i]; z[i] = *p;", "z[i] = x[j];",
                                  "z[2*i] = x[i];"])
def test_analysis_rejects_non_elementwise_uses(text):
    assert cg.analyze(text, ["x", "z"]) is None


def test_chunk_width_from_narrowest_used_vector():
    sig = ew.parse_signature("int8_t *b, double *d, float *z")
    acc = cg.analyze("z[i] = d[i];", ["b", "d", "z"])
    assert cg.chunk_width(sig, acc) == 4          # b unused: float z sets it
    sig2 = ew.parse_signature("int8_t *b, double *d, double *z")
    assert cg.chunk_width(sig2, cg.analyze("z[i] = d[i];", ["b", "d", "z"])) == 2
    acc = cg.analyze("z[i] = b[i] * d[i];", ["b", "d", "z"])
    assert cg.chunk_width(sig, acc) == 16


def test_vector_path_call_checks():
    rw = cg.Access(False, True)
    ro = cg.Access(True, False)
    assert cg.vector_path_ok([(0x1000, 0x1000, 4, ro), (0x2000, 0x2000, 4, rw)], 1024)
    assert not cg.vector_path_ok([(0x1004, 0x1004, 4, ro)], 16)         # misaligned
    assert not cg.vector_path_ok([(0x1000, 0x1000, 4, ro), (0x1000, 0x1000, 4, rw)], 16)
    assert cg.vector_path_ok([(0x1000, 0x1000, 4, ro), (0x1000, 0x1000, 4, ro)], 16)
    assert not cg.vector_path_ok([(0x1000, 0x1000, 4, rw), (0x1020, 0x1020, 4, ro)], 16)


def test_scalar_widening_rules():
    assert cg.scalar_value(1.5, nd.float32).value == 1.5
    assert cg.scalar_value(-1, nd.uint8).value == 2**64 - 1
    assert cg.scalar_value(-4, nd.int32).value == -4
    assert isinstance(cg.scalar_value(3, nd.float64).value, float)


# --- generation ---------------------------------------------------------------------------------


def test_generate_is_deterministic_and_variant_sensitive():
    sig = ew.parse_signature("float *x, float *z")
    v = ew.VariantParams(unroll=2)
    a = ew.generate(sig, "z[i] = 2 * x[i]", "dbl", v)
    assert a == ew.generate(sig, "z[i] = 2 * x[i]", "dbl", v)
    assert a != ew.generate(sig, "z[i] = 2 * x[i]", "dbl", ew.VariantParams(unroll=4))
    assert a != ew.generate(sig, "z[i] = 2 * x[i]", "dbl", ew.VariantParams(unroll=2,
                                                                             block=512))
    assert a == ew.generate(sig, "z[i] = 2 * x[i]", "dbl", ew.VariantParams(unroll=2,
                                                                             workers=7))
    assert "${" not in a and not any(t in a for t in ("{% for", "{% if", "{% end"))
    assert 'extern "C" __global__' in a and "dbl_g(" in a and "dbl(" in a
    with pytest.raises(ValueError):
        ew.generate(sig, "z[i] = 1", "not an identifier", v)


def test_reduction_spec_rules():
    with pytest.raises(rd.NonScalarResult):
        rd.ReductionSpec("float *x", nd.float32, "0", "a + 1")
    with pytest.raises(rd.NonScalarResult):
        rd.ReductionSpec("float *x", nd.float32, "0", "b * 2")
    for bad in ("float *acc", "float *out", "float *partials", "float *result"):
        with pytest.raises(ew.ParseError):
            rd.ReductionSpec(bad + ", float *v", nd.float32, "0", "a + b")
    assert rd.ReductionSpec("float s, float *x", nd.float32, "0", "a + b").mapped == "x[i]"
    assert rd.ReductionSpec("float *x", nd.float32, "0", "a+b").acc_dtype is nd.float64
    assert rd.ReductionSpec("int16_t *x", nd.int16, "0", "a+b").acc_dtype is nd.int16
    src = rd.generate_reduction_source(rd.ReductionSpec("float *x", nd.float32, "0", "a + b"),
                                       "rsum", ew.VariantParams(unroll=1))
    assert "double acc = 0;" in src and "rsum_combine(" in src and "rsum_g(" in src


@pytest.fixture(scope="module")
def nvrtc_cache(tmp_path_factory):
    return jit.CacheStore(tmp_path_factory.mktemp("codegen-cache"))


def _sass(image: bytes, tmp_path) -> str:
    tool = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    if not os.path.exists(tool):
        pytest.skip("cuobjdump not available")
    path = tmp_path / "k.cubin"
    path.write_bytes(image)
    return subprocess.run([tool, "-sass", str(path)], capture_output=True, text=True).stdout


def test_axpy_compiles_to_128bit_accesses_without_fma(nvrtc_cache, tmp_path):
    k_src = ew.generate(ew.parse_signature("float a, float *x, float b, float *y, float *z"),
                        "z[i] = a * x[i] + b * y[i]", "axpy", ew.VariantParams())
    module = jit.compile(k_src, cache=nvrtc_cache)
    assert module.has_symbol("axpy") and module.has_symbol("axpy_g")
    assert module.provenance.diagnostics.strip() == ""
    sass = _sass(module.image, tmp_path)
    body = sass.split("Function : axpy\n")[1].split("Function :")[0]
    assert "LDG.E.128" in body and "STG.E.128" in body
    assert "FFMA" not in body  # -fmad=false keeps a*x + b*y as FMUL, FMUL, FADD


def test_dot_reduction_compiles_with_fp64_accumulator(nvrtc_cache, tmp_path):
    src = rd.generate_reduction_source(
        rd.ReductionSpec("float *x, float *y", nd.float32, "0", "a + b", "x[i] * y[i]"),
        "dot_k", ew.VariantParams(unroll=8, block=512))
    module = jit.compile(src, cache=nvrtc_cache)
    sass = _sass(module.image, tmp_path)
    body = sass.split("Function : dot_k\n")[1].split("Function :")[0]
    assert "LDG.E.128" in body and "DADD" in body and "SHFL.DOWN" in body
    assert "LDL" not in body and "STL" not in body  # no local-memory spills


def test_dynamic_chunk_reduction_takes_chunks_from_a_counter(nvrtc_cache, tmp_path):
    """VariantParams.chunk: the vector entry streams 128-bit chunks, takes
    chunk ids with a global atomic, and still spills nothing."""
    spec = rd.ReductionSpec("float *x, float *y", nd.float32, "0", "a + b", "x[i] * y[i]")
    src = rd.generate_reduction_source(spec, "dot_k", ew.VariantParams(unroll=4, chunk=8192))
    assert "rtcg::chunk_plan(start, end, 8192L" in src
    static = rd.generate_reduction_source(spec, "dot_k", ew.VariantParams(unroll=4))
    assert "chunk_plan" not in static.split("// ---- end prelude")[1]
    sass = _sass(jit.compile(src, cache=nvrtc_cache).image, tmp_path)
    body = sass.split("Function : dot_k\n")[1].split("Function :")[0]
    assert "LDG.E.128" in body and "ATOMG.E.ADD" in body and "DADD" in body
    assert "LDL" not in body and "STL" not in body


@pytest.mark.parametrize("sig, op", [
    ("int8_t *b, double *d, double *z", "z[i] = b[i] * d[i] + 0.5"),
    ("uint64_t s, uint16_t *x, uint64_t *z", "z[i] = x[i] * s"),
    ("double *x, double *z", "z[i] = sin(x[i]) + pow(x[i], 2.0) + fabs(x[i])"),
    ("float *x, float *z", "z[i] = x[i+1] - x[i]"),
    ("float *x, long *z", "z[i] = i + (long) x[i]"),
    ("int32_t *x", "x[i] = abs(x[i]) % 7"),
])
def test_varied_kernels_compile(nvrtc_cache, sig, op):
    for v in (ew.VariantParams(), ew.VariantParams(unroll=16, block=1024,
                                                   chunking="contiguous-blocks",
                                                   cache="streaming")):
        jit.compile(ew.generate(ew.parse_signature(sig), op, "k", v), cache=nvrtc_cache)


@pytest.mark.parametrize("dname", [d.name for d in nd.DTYPES])
def test_stock_reductions_compile_for_every_dtype(nvrtc_cache, dname):
    d = nd.BY_NAME[dname]
    for spec in (rd.ReductionSpec(f"{d.cname} *x", d, "0", "a + b"),
                 rd.ReductionSpec(f"{d.cname} *x", d, rd._lowest(d), "a > b ? a : b"),
                 rd.ReductionSpec(f"{d.cname} *x, {d.cname} *y", d, "0", "a + b",
                                  "x[i] * y[i]")):
        module = jit.compile(rd.generate_reduction_source(spec, "r", ew.VariantParams()),
                             cache=nvrtc_cache)
        assert module.has_symbol("r_combine")


def test_c_math_semantics_in_prelude(nvrtc_cache, tmp_path):
    """sin(float) is computed in double like C: the generated code calls the
    double routine (no float-only sinf path)."""
    src = ew.generate(ew.parse_signature("float *x, float *z"), "z[i] = sin(x[i])", "csin",
                      ew.VariantParams())
    sass = _sass(jit.compile(src, cache=nvrtc_cache).image, tmp_path)
    assert "F2F.F64.F32" in sass and "DFMA" in sass


def test_elementwise_tma_entry_uses_bulk_copies():
    from paper_0911_3456_b200 import _codegen as cg, elementwise as ew
    src = ew.generate(ew.parse_signature("double *x, double *z"), "z[i] = x[i];", "cp",
                      ew.VariantParams(cache="tma"))
    assert "cp.async.bulk" in src and "rtcg_full" in src
    assert cg.tma_eligible(ew.parse_signature("double *x, double *z"),
                           cg.analyze("z[i] = x[i];", ["x", "z"]), 2)
    with pytest.raises(ValueError):
        ew.generate(ew.parse_signature("double *x, double *z"), "z[i] = x[i];", "cp",
                    ew.VariantParams(cache="tma", block=32))


# User parameter names that are also template locals (loop counters, tile
# bookkeeping, C-ish one-letter names) must neither collide nor be shadowed.
_CLASH_SIG = "float k, float *c, double E, float *b, float *s"
_CLASH_OP = "s[i] = k * c[i] + (float) E * b[i]"


@pytest.mark.parametrize("cache", ["default", "tma"])
def test_template_locals_never_clash_with_user_names(nvrtc_cache, cache):
    from paper_0911_3456_b200 import jit
    v = ew.VariantParams(cache=cache, unroll=2)
    src = ew.generate(ew.parse_signature(_CLASH_SIG), _CLASH_OP + ";", "clash", v)
    jit.compile(src, cache=nvrtc_cache)
    spec = rd.ReductionSpec("float *b, long G, float *t", nd.float64, "0", "a + b",
                            "b[i] * t[i] + G")
    jit.compile(rd.generate_reduction_source(spec, "clash_r", v), cache=nvrtc_cache)
    if cache != "tma":     # the dynamic-chunk locals (plan, ch, sp, tl) stay out of user scope
        dyn = rd.ReductionSpec("float *x, long plan, double ch, int sp, int tl", nd.float32,
                               "0", "a + b", "x[i] * plan + ch + sp + tl")
        jit.compile(rd.generate_reduction_source(dyn, "clash_d",
                                                 ew.VariantParams(unroll=2, chunk=4096)),
                    cache=nvrtc_cache)


def test_peer_descriptor_layout_matches_prelude(nvrtc_cache):
    """parallel.PeerMailbox packs rtcg::xr on the host; the device struct must
    agree (size -- 8 + 8 * XR_MAX leaves no room for padding before mbox --,
    slot count, mailbox size)."""
    from paper_0911_3456_b200 import parallel as par
    src = (cg.template("prelude.cuh")
           + f"\nstatic_assert(sizeof(rtcg::xr) == {par._XR.size}, \"xr size\");"
           + f"\nstatic_assert(rtcg::XR_MAX == {par.XR_MAX}, \"XR_MAX\");"
           + f"\nstatic_assert(rtcg::XR_ERROR == {par.XR_ERROR}, \"XR_ERROR\");"
           + '\nextern "C" __global__ void layout_probe() {}\n')
    jit.compile(src, cache=nvrtc_cache)
    assert par.MAILBOX_BYTES >= 8 * (par.XR_ERROR + 1)


def test_default_variant_pipelines_transcendental_statements():
    """Untuned statements that call transcendentals get the register-
    pipelined loop (r02_probe_heavy_defaults.json); others the plain one."""
    heavy = ew.default_variant("z[i] = ((a*x[i] + 2.0)*x[i] - 1.5)*x[i] + sin(x[i])")
    assert heavy.prefetch and heavy.waves == 4
    assert ew.default_variant("z[i] = expf (x[i])").prefetch
    assert ew.default_variant("z[i] = a * x[i] + sinus[i]") == ew.VariantParams()
    assert ew.default_variant("z[i] = x[i] + y[i]") == ew.VariantParams()
