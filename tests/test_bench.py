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


def _run(*args, timeout=600):
    proc = subprocess.run([sys.executable, str(ROOT / "bench.py"), *args], cwd=ROOT,
                          capture_output=True, text=True, timeout=timeout)
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
