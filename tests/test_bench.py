"""bench.py keeps the driver contract: exactly one JSON line on stdout with the
required keys (reference arm on the CPU; the GPU arm on the B200)."""

import json
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
BASE_KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
             "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config", "e2e"}


def _run(*args, timeout=600, env=None):
    import os
    proc = subprocess.run([sys.executable, str(ROOT / "bench.py"), *args], cwd=ROOT,
                          capture_output=True, text=True, timeout=timeout,
                          env=None if env is None else dict(os.environ, **env))
    assert proc.returncode == 0, proc.stderr[-2000:]
    lines = [ln for ln in proc.stdout.splitlines() if ln.strip()]
    assert len(lines) == 1, proc.stdout
    return json.loads(lines[0])


def test_reference_arm_line():
    line = _run("--impl", "reference", "--steps", "2", "--warmup", "1")
    assert BASE_KEYS <= set(line) and line["impl"] == "reference"
    assert line["unit"] == "GB/s" and line["value"] > 0 and line["higher_is_better"] is True
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["e2e"]["value"] == line["value"]
    cb = line["cpu_baseline"]
    assert cb["kind"] in ("reference", "port") and cb["cores"] >= 1 and "sample" in cb
    # the unmodified reference is preferred wherever it is installed
    if (ROOT / "baseline" / "_ref" / "rtcg" / "reduction.py").exists():
        assert "stock rtcg" in cb["sample"] and "baseline/_ref" in cb["sample"]


@pytest.mark.gpu
def test_gpu_arm_line():
    line = _run("--steps", "20", "--warmup", "3", "--quick", "--no-cpu")
    assert BASE_KEYS <= set(line) and "impl" not in line
    assert line["n_gpus"] == 1 and line["scaling"] == "weak" and line["dtype"] == "f32"
    roof = line["roofline"]
    assert roof["bound"] == "hbm" and roof["unit"] == "GB/s" and roof["peak"] > 0
    assert 0.5 < roof["frac"] < 1.5 and roof["achieved"] == pytest.approx(line["value"], rel=0.1)
    assert line["gpu_launches"] == 20
    assert line["e2e"]["h2d_bytes_per_step"] == 2 * 4 * (1 << 28)
    assert set(line["clocks"]) >= {"sm_mhz", "sm_max_mhz", "reasons"}
    assert line["parity_ok"] is True and line["parity"]["dot_ok"] is True
    assert line["roofline"]["isolated_launch_ms"] > 0
    assert line["config"]["variant_block"] in (128, 256, 512, 1024)


@pytest.mark.gpu
def test_gpu_arm_spawns_two_ranks_on_one_gpu():
    """``--gpus 2`` with no launcher: two ranks (sharing the one B200 over
    gloo), one line, n_gpus 2, parity checked across the ranks."""
    line = _run("--gpus", "2", "--steps", "5", "--warmup", "3", "--quick", "--no-cpu")
    assert line["n_gpus"] == 2 and line["n_ranks_seen"] == 2
    assert line["config"]["n_total"] == 2 << 28 and line["config"]["shared_gpu"] is True
    assert line["parity_ok"] is True and line["parity"]["dot_ranks_agree"] is True
    assert line["collective"] in ("auto", "allgather", "allreduce")


def test_spawn_env_sets_the_launcher_variables():
    sys.path.insert(0, str(ROOT))
    import bench
    env = bench.spawn_env({"PATH": "/bin"}, 3, 8, 12345)
    assert env["RANK"] == env["LOCAL_RANK"] == "3" and env["WORLD_SIZE"] == "8"
    assert env["LOCAL_WORLD_SIZE"] == "8" and env["MASTER_ADDR"] == "127.0.0.1"
    assert env["MASTER_PORT"] == "12345" and env["PATH"] == "/bin"


def test_spawn_ranks_runs_world_processes_and_relays_rank0(tmp_path, capsys):
    """``bench.py --gpus N`` without a launcher must start N ranks
    (not silently one).  A stand-in rank script reports what it was given."""
    sys.path.insert(0, str(ROOT))
    import bench
    script = tmp_path / "rank.py"
    script.write_text(
        "import json, os, sys, torch.distributed as dist\n"
        "dist.init_process_group('gloo')\n"
        "ranks = [None] * dist.get_world_size()\n"
        "dist.all_gather_object(ranks, int(os.environ['RANK']))\n"
        "if dist.get_rank() == 0:\n"
        "    print(json.dumps({'n_ranks_seen': len(ranks), 'ranks': ranks,\n"
        "                      'argv': sys.argv[1:]}))\n"
        "dist.destroy_process_group()\n")
    rc = bench.spawn_ranks(["--gpus", "3"], 3, timeout=120, script=str(script))
    assert rc == 0
    line = json.loads(capsys.readouterr().out.strip())
    assert line == {"n_ranks_seen": 3, "ranks": [0, 1, 2], "argv": ["--gpus", "3"]}


def test_spawn_ranks_reports_a_failing_rank(tmp_path, capsys):
    sys.path.insert(0, str(ROOT))
    import bench
    script = tmp_path / "fail.py"
    script.write_text("import os, sys\nsys.exit(7 if os.environ['RANK'] == '1' else 0)\n")
    assert bench.spawn_ranks([], 2, timeout=60, script=str(script)) == 7


def test_exact_checkers_match_fsum_and_python_ints():
    import math
    import numpy as np
    import torch
    sys.path.insert(0, str(ROOT))
    import bench
    rng = np.random.default_rng(4)
    x = rng.uniform(-1, 1, 200_003).astype(np.float32)
    y = rng.uniform(-1, 1, 200_003).astype(np.float32)
    p = x * y
    p[:5] = [0.0, 1e-45, -3e-39, 3.0e38, -3.0e38]         # zero, subnormals, huge
    exact = bench.buckets_value(bench.f32_exact_buckets(torch.from_numpy(p)))
    assert float(exact) == math.fsum(p.astype(np.float64).tolist())
    chk = bench.reduction_check(float(np.float32(float(exact))), exact, p.size,
                                float(np.abs(p.astype(np.float64)).sum()))
    assert chk["ok"] and chk["bit_equal_f32_fsum"] and chk["ulps"] <= 0.5
    v = rng.integers(-(1 << 62), 1 << 62, size=100_001, dtype=np.int64)
    want = sum(int(a) for a in v)
    assert bench.i64_wrapped_sum(torch.from_numpy(v)) == want
    assert bench.wrap64(want) == int(v.sum())                # numpy wraps too
    small = torch.from_numpy(rng.integers(-5, 5, size=1000, dtype=np.int32))
    assert bench.i64_wrapped_sum(small) == int(small.sum())


def test_workload_config_is_shared_by_both_arms():
    sys.path.insert(0, str(ROOT))
    import bench
    assert bench.workload_config(1)["n_total"] == 1 << 28
    assert bench.workload_config(8)["n_total"] == 8 << 28


@pytest.mark.gpu
def test_gpu_arm_two_processes_through_the_peer_exchange():
    """The product path across processes: two ranks on the one B200 exchange
    their accumulators inside the reduction kernel through CUDA IPC-mapped
    mailboxes (what NVLink peers do on an 8-GPU box), parity-checked."""
    line = _run("--gpus", "2", "--steps", "5", "--warmup", "3", "--quick", "--no-cpu",
                env={"RTCG_BENCH_COLLECTIVE": "p2p"})
    assert line["n_ranks_seen"] == 2 and line["collective"] == "p2p"
    assert line["parity_ok"] is True and line["parity"]["dot_ranks_agree"] is True
    assert line["gpu_launches"] == 5          # one kernel per step: the exchange is inside


def test_roofline_traffic_is_looked_up_for_the_timed_variant():
    sys.path.insert(0, str(ROOT))
    import bench
    table_hit = bench._ncu_traffic("dot_k", {"block": 128, "unroll": 1, "waves": 2})
    assert table_hit[2] is True and table_hit[1] == {"block": 128, "unroll": 1, "waves": 2}
    assert 0.99 < table_hit[0] / (8 << 28) < 1.01
    # variant keys ignore absent-vs-default spelling
    assert bench._variant_key({"block": 256}) == bench._variant_key(
        {"block": 256, "cache": "default", "unroll": 1, "waves": 1})
    assert bench._ncu_traffic("no_such_kernel", {}) == (None, None, False, None)


def test_reduction_check_bound_and_bit_equality():
    from fractions import Fraction
    sys.path.insert(0, str(ROOT))
    import bench
    exact = Fraction(1, 3)
    got = float(exact)                               # fp64 rounding of 1/3
    chk = bench.reduction_check(got, exact, n=4, sum_abs=1.0)
    assert chk["ok"] and chk["bit_equal_f32_fsum"] and chk["ulps"] < 1e-6
    far = bench.reduction_check(got + 1e-3, exact, n=4, sum_abs=1.0)
    assert not far["ok"] and not far["bit_equal_f32_fsum"]


def test_stock_c5_times_the_reference_ops():
    """The C5 CPU leg runs the unmodified reference's operators and stock
    reductions (skipped where baseline/_ref is not installed)."""
    import numpy as np
    sys.path.insert(0, str(ROOT))
    import bench
    if bench._stock_reference() is None:
        pytest.skip("baseline/_ref not installed")
    rng = np.random.default_rng(9)
    for dname, dt in (("float32", np.float32), ("int64", np.int64)):
        x = (rng.integers(-1000, 1000, 4096) / (1000 if dt is np.float32 else 1)).astype(dt)
        y = (rng.integers(-1000, 1000, 4096) / (1000 if dt is np.float32 else 1)).astype(dt)
        got = bench.stock_c5(dname, x, y, reps=2)
        assert set(got) == {"add_us", "chain_eager_us", "sum_us", "max_us", "dot_us"}
        assert all(v > 0 for v in got.values())
