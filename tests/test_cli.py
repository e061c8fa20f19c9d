"""``rtcg`` command line (reference tests/test_cli.py, re-targeted): exit codes,
JSON documents, CUDA source dumps, cache administration on CPU; demos, bench
and tuning campaigns on the GPU."""

import ctypes
import json

import numpy as np
import pytest

from paper_0911_3456_b200 import cli, jit


def run_cli(capsys, *argv):
    code = cli.main(list(argv))
    out, err = capsys.readouterr()
    return code, out, err


def _populate(tmp_path, count=1):
    """Compile ``count`` distinct kernels into the cache (NVRTC runs on CPU)."""
    cache = jit.CacheStore(tmp_path)
    for k in range(count):
        src = cli.csyntax.unrolled_add_template(k + 1)
        jit.compile(src, jit.ToolchainConfig.from_env(), cache)


# --- cache administration (CPU) ---------------------------------------------------------------


def test_cache_info_empty(tmp_path, capsys):
    code, out, _ = run_cli(capsys, "--format", "json", "--cache-dir", str(tmp_path),
                           "cache", "info")
    assert code == 0
    doc = json.loads(out)
    assert doc["schema"] == cli.CLI_SCHEMA
    assert doc["entries"] == 0 and doc["bytes"] == 0


def test_cache_info_counts_compiled_entries(tmp_path, capsys):
    _populate(tmp_path, 2)
    code, out, _ = run_cli(capsys, "--format", "json", "--cache-dir", str(tmp_path),
                           "cache", "info")
    assert code == 0
    doc = json.loads(out)
    assert doc["entries"] == 2 and doc["bytes"] > 0
    assert doc["oldest_unix"] is not None and doc["newest_unix"] >= doc["oldest_unix"]
    code, out, _ = run_cli(capsys, "--cache-dir", str(tmp_path), "cache", "info")
    assert "entries: 2" in out and "oldest:" in out


def test_cache_prune_zero_age_equals_clear(tmp_path, capsys):
    _populate(tmp_path)
    code, out, _ = run_cli(capsys, "--format", "json", "--cache-dir", str(tmp_path),
                           "cache", "prune", "--older-than", "0s")
    assert code == 0
    doc = json.loads(out)
    assert doc["removed"] == 1 and doc["older_than_seconds"] == 0
    _populate(tmp_path)
    code, out, _ = run_cli(capsys, "--format", "json", "--cache-dir", str(tmp_path),
                           "cache", "clear")
    assert code == 0 and json.loads(out)["removed"] == 1
    _, out, _ = run_cli(capsys, "--format", "json", "--cache-dir", str(tmp_path), "cache", "info")
    assert json.loads(out)["entries"] == 0


def test_cache_prune_keeps_young_entries(tmp_path, capsys):
    _populate(tmp_path)
    code, out, _ = run_cli(capsys, "--format", "json", "--cache-dir", str(tmp_path),
                           "cache", "prune", "--older-than", "1h")
    assert code == 0 and json.loads(out)["removed"] == 0


def test_cache_prune_requires_valid_duration(tmp_path, capsys):
    code, _, err = run_cli(capsys, "--cache-dir", str(tmp_path),
                           "cache", "prune", "--older-than", "soon")
    assert code == 2 and "duration" in err


def test_parse_duration_units():
    assert cli.parse_duration("30s") == 30
    assert cli.parse_duration("15m") == 900
    assert cli.parse_duration("2h") == 7200
    assert cli.parse_duration("7d") == 604800
    for bad in ("1.5h", "h", "10", "-3s"):
        with pytest.raises(cli.UsageError):
            cli.parse_duration(bad)


# --- codegen dump (CPU) ----------------------------------------------------------------------


def test_dump_unrolled_add_is_deterministic(tmp_path, capsys):
    argv = ("--cache-dir", str(tmp_path), "codegen", "dump", "--kind", "unrolled-add",
            "--unroll", "4")
    first, second = run_cli(capsys, *argv), run_cli(capsys, *argv)
    assert first[0] == 0 and first[1] == second[1]
    assert 'extern "C" __global__ void vadd_unrolled(' in first[1]


def _dump_fig4(capsys, tmp_path):
    sources = {}
    for method in ("template", "ast"):
        code, out, _ = run_cli(capsys, "--cache-dir", str(tmp_path), "codegen", "dump",
                               "--kind", "unrolled-add", "--method", method, "--unroll", "4")
        assert code == 0
        sources[method] = out
    return sources


def test_dump_methods_differ_in_spelling_and_both_compile(tmp_path, capsys):
    sources = _dump_fig4(capsys, tmp_path)
    assert sources["template"] != sources["ast"]
    cache = jit.CacheStore(tmp_path / "cache")
    for src in sources.values():
        module = jit.compile(src, jit.ToolchainConfig.from_env(), cache)
        assert module.has_symbol("vadd_unrolled")


def test_dump_elementwise_source(tmp_path, capsys):
    code, out, _ = run_cli(capsys, "--cache-dir", str(tmp_path), "codegen", "dump",
                           "--kind", "elementwise", "--signature", "float *x, float *z",
                           "--operation", "z[i] = 2 * x[i]", "--name", "twice", "--unroll", "2")
    assert code == 0
    assert 'extern "C" __global__' in out and "twice(" in out and "twice_g(" in out
    assert "z[i] = 2 * x[i];" in out
    # what the dump prints is exactly what the kernel object compiles
    from paper_0911_3456_b200 import elementwise as ew
    sig = ew.parse_signature("float *x, float *z")
    assert out == ew.generate(sig, "z[i] = 2 * x[i];", "twice", ew.VariantParams(unroll=2))


def test_dump_elementwise_requires_operation(tmp_path, capsys):
    code, _, err = run_cli(capsys, "--cache-dir", str(tmp_path), "codegen", "dump",
                           "--kind", "elementwise", "--signature", "float *x, float *z")
    assert code == 2 and "error:" in err


def test_dump_reduction_source(tmp_path, capsys):
    code, out, _ = run_cli(capsys, "--cache-dir", str(tmp_path), "codegen", "dump",
                           "--kind", "reduction", "--signature", "int *x", "--out-dtype", "int64",
                           "--neutral", "0", "--reduce", "a + b", "--name", "total")
    assert code == 0
    assert "total(" in out and "total_g(" in out and "total_combine(" in out


def test_dump_reduction_unknown_dtype(tmp_path, capsys):
    code, _, err = run_cli(capsys, "--cache-dir", str(tmp_path), "codegen", "dump",
                           "--kind", "reduction", "--signature", "int *x", "--out-dtype", "int99",
                           "--neutral", "0", "--reduce", "a + b")
    assert code == 2 and "int99" in err


def test_dump_reduction_without_both_operands_is_usage_error(tmp_path, capsys):
    code, _, err = run_cli(capsys, "--cache-dir", str(tmp_path), "codegen", "dump",
                           "--kind", "reduction", "--signature", "int *x", "--out-dtype", "int64",
                           "--neutral", "0", "--reduce", "a + 1")
    assert code == 2 and "error:" in err


def test_dump_unknown_signature_type_is_usage_error(tmp_path, capsys):
    code, _, err = run_cli(capsys, "--cache-dir", str(tmp_path), "codegen", "dump",
                           "--kind", "elementwise", "--signature", "quaternion *x, float *z",
                           "--operation", "z[i] = x[i]")
    assert code == 2 and "quaternion" in err


@pytest.mark.parametrize("flag,value,word", [("--unroll", "0", "unroll"),
                                             ("--unroll", "3", "unroll"),
                                             ("--block", "96", "block")])
def test_dump_rejects_bad_variant(tmp_path, capsys, flag, value, word):
    kind = ["--kind", "unrolled-add"] if value == "0" else [
        "--kind", "elementwise", "--signature", "float *x", "--operation", "x[i] = 1"]
    code, _, err = run_cli(capsys, "--cache-dir", str(tmp_path), "codegen", "dump", *kind,
                           flag, value)
    assert code == 2 and word in err


# --- tune argument parsing / dispatch (CPU) ---------------------------------------------------


def test_parse_axis_values():
    assert cli.parse_axis("unroll=1,2,4") == ("unroll", (1, 2, 4))
    assert cli.parse_axis("chunking=strided,contiguous-blocks") == \
        ("chunking", ("strided", "contiguous-blocks"))
    with pytest.raises(cli.UsageError):
        cli.parse_axis("noequals")
    with pytest.raises(cli.UsageError):
        cli.parse_axis("unroll=1,,2")


def test_unknown_command_exits_2(capsys):
    with pytest.raises(SystemExit) as err:
        cli.main(["frobnicate"])
    assert err.value.code == 2


def test_missing_subcommand_exits_2(capsys):
    with pytest.raises(SystemExit) as err:
        cli.main([])
    assert err.value.code == 2


def test_negative_n_is_usage_error(tmp_path, capsys):
    code, _, err = run_cli(capsys, "--cache-dir", str(tmp_path), "demo", "double", "--n", "-1")
    assert code == 2 and ">= 0" in err


def test_verbose_describes_config_on_stderr(tmp_path, capsys):
    code, out, err = run_cli(capsys, "--verbose", "--cache-dir", str(tmp_path), "cache", "info")
    assert code == 0
    assert "# nvrtc:" in err and "# cache_root:" in err and "# arch: sm_100a" in err
    assert "# nvrtc:" not in out


def test_flag_precedence(tmp_path, monkeypatch):
    monkeypatch.setenv("RTCG_ARCH", "sm_90a")
    args = cli.build_parser().parse_args(["--cache-dir", str(tmp_path), "cache", "info"])
    assert cli._resolve_config(args).toolchain.arch == "sm_90a"  # env over default
    args = cli.build_parser().parse_args(["--arch", "sm_100a", "--fmad", "on",
                                          "--nvrtc-flag=-G", "cache", "info"])
    cfg = cli._resolve_config(args)
    assert cfg.toolchain.arch == "sm_100a"  # flag over env
    assert "-fmad=true" in cfg.toolchain.flags and "-G" in cfg.toolchain.flags


def test_gpu_commands_fail_loudly_without_a_device(tmp_path, capsys):
    from paper_0911_3456_b200 import _runtime
    if _runtime.have_gpu():
        pytest.skip("a GPU is present")
    code, _, err = run_cli(capsys, "--cache-dir", str(tmp_path), "demo", "double")
    assert code == 1 and "error:" in err


# --- GPU: demo, bench, tune -------------------------------------------------------------------


@pytest.mark.gpu
def test_dump_methods_agree_on_gpu(tmp_path, capsys):
    from paper_0911_3456_b200 import _runtime, ndarray as nd
    sources = _dump_fig4(capsys, tmp_path)
    _runtime.set_device(0)
    pool = nd.MemoryPool(device=0)
    rng = np.random.default_rng(11)
    n = 1000
    hx = rng.uniform(-1, 1, n).astype(np.float32)
    hy = rng.uniform(-1, 1, n).astype(np.float32)
    x, y = nd.from_host(pool, nd.float32, hx), nd.from_host(pool, nd.float32, hy)
    outs = []
    for src in sources.values():
        k = jit.get_kernel(jit.compile(src, cache=jit.CacheStore(tmp_path / "c")), "vadd_unrolled")
        z = pool.alloc(nd.float32, (n,))
        vals = [ctypes.c_uint64(x.address), ctypes.c_uint64(y.address),
                ctypes.c_uint64(z.address), ctypes.c_long(n)]
        k.launch(3, 128, (ctypes.c_void_p * 4)(*[ctypes.addressof(v) for v in vals]))
        outs.append(z.to_host())
    assert np.array_equal(outs[0], outs[1]) and np.array_equal(outs[0], hx + hy)


@pytest.mark.gpu
def test_demo_double_default_grid(tmp_path, capsys):
    code, out, _ = run_cli(capsys, "--cache-dir", str(tmp_path), "demo", "double")
    assert code == 0 and "PASS" in out and "(4x4)" in out


@pytest.mark.gpu
def test_demo_lincomb_bit_exact(tmp_path, capsys):
    code, out, _ = run_cli(capsys, "--format", "json", "--cache-dir", str(tmp_path),
                           "demo", "lincomb", "--n", "257")
    doc = json.loads(out)
    assert code == 0 and doc["pass"] is True and doc["max_abs_error"] == 0.0


@pytest.mark.gpu
def test_demo_fmad_on_still_passes_double(tmp_path, capsys):
    # 2*x is exact with or without contraction
    code, out, _ = run_cli(capsys, "--fmad", "on", "--cache-dir", str(tmp_path),
                           "demo", "double", "--n", "1000")
    assert code == 0 and "PASS" in out


@pytest.mark.gpu
def test_demo_dot_empty_input_matches_neutral(tmp_path, capsys):
    code, out, _ = run_cli(capsys, "--cache-dir", str(tmp_path), "demo", "dot", "--n", "0")
    assert code == 0 and "PASS" in out


@pytest.mark.gpu
def test_demo_json_document(tmp_path, capsys):
    code, out, _ = run_cli(capsys, "--format", "json", "--cache-dir", str(tmp_path),
                           "demo", "dot", "--n", "100")
    assert code == 0
    doc = json.loads(out)
    assert doc["pass"] is True and doc["demo"] == "dot" and doc["n"] == 100
    assert doc["seconds"] > 0 and doc["schema"] == cli.CLI_SCHEMA


@pytest.mark.gpu
def test_bench_json_has_exactly_five_fields(tmp_path, capsys):
    code, out, _ = run_cli(capsys, "--format", "json", "--cache-dir", str(tmp_path),
                           "bench", "--op", "lincomb", "--n", "1000")
    assert code == 0
    doc = json.loads(out)
    assert set(doc) == {"op", "n", "seconds", "gitless_fingerprint", "pass"}
    assert doc["op"] == "lincomb" and doc["n"] == 1000 and doc["seconds"] > 0
    assert doc["pass"] is True
    assert doc["gitless_fingerprint"] == jit.fingerprint(jit.ToolchainConfig.from_env()).digest()


@pytest.mark.gpu
@pytest.mark.parametrize("op", ["double", "lincomb", "dot"])
def test_bench_human_reports_rate(tmp_path, capsys, op):
    code, out, _ = run_cli(capsys, "--cache-dir", str(tmp_path), "bench", "--op", op,
                           "--n", str((1 << 22) + 5))
    assert code == 0 and "M elements/s" in out and "GB/s" in out and "PASS" in out


@pytest.mark.gpu
def test_bench_rejects_more_devices_than_present(tmp_path, capsys):
    from paper_0911_3456_b200 import _runtime
    code, _, err = run_cli(capsys, "--cache-dir", str(tmp_path), "bench", "--op", "double",
                           "--n", "64", "--devices", str(_runtime.device_count() + 1))
    assert code == 2 and "--devices" in err


@pytest.mark.gpu
def test_tune_runs_and_then_hits_the_store(tmp_path, capsys):
    argv = ("--format", "json", "--cache-dir", str(tmp_path), "tune", "--kernel", "double",
            "--n", "2048", "--axis", "unroll=1,2", "--axis", "block=128")
    code, out, _ = run_cli(capsys, *argv)
    assert code == 0
    cold = json.loads(out)
    assert cold["cached"] is False and len(cold["table"]) == 2
    assert {e["status"] for e in cold["table"]} == {"ok"}
    assert cold["best"]["block"] == 128
    code, out, _ = run_cli(capsys, *argv)
    warm = json.loads(out)
    assert code == 0 and warm["cached"] is True
    assert warm["best"] == cold["best"] and warm["table"] == cold["table"]


@pytest.mark.gpu
def test_tune_sample_measures_one_variant(tmp_path, capsys):
    code, out, _ = run_cli(capsys, "--format", "json", "--cache-dir", str(tmp_path),
                           "tune", "--kernel", "double", "--n", "1024",
                           "--axis", "unroll=1,2,4", "--axis", "block=256",
                           "--sample", "1", "--no-prune")
    assert code == 0
    statuses = [e["status"] for e in json.loads(out)["table"]]
    assert statuses.count("ok") == 1 and statuses.count("unsampled") == 2


@pytest.mark.gpu
def test_tune_human_table_and_dot_recipe(tmp_path, capsys):
    code, out, _ = run_cli(capsys, "--cache-dir", str(tmp_path), "tune", "--kernel", "dot",
                           "--n", "100000", "--axis", "unroll=1", "--axis", "block=256")
    assert code == 0
    assert "best: block=256,unroll=1" in out and "cached: false" in out


@pytest.mark.gpu
def test_tune_unknown_kernel_or_axis_is_usage_error(tmp_path, capsys):
    code, _, err = run_cli(capsys, "--cache-dir", str(tmp_path), "tune", "--kernel", "nosuch",
                           "--n", "8")
    assert code == 2 and "nosuch" in err
    code, _, err = run_cli(capsys, "--cache-dir", str(tmp_path), "tune", "--kernel", "double",
                           "--n", "8", "--axis", "depth=1,2")
    assert code == 2 and "depth" in err


@pytest.mark.gpu
def test_compiler_failure_exits_1(tmp_path, capsys):
    code, _, err = run_cli(capsys, "--cache-dir", str(tmp_path), "--nvrtc-flag=--no-such-option",
                           "demo", "double", "--n", "4")
    assert code == 1 and "error:" in err
