"""The C-ABI runtime library: loads, exports every symbol include/rtcg_b200.h
declares, compiles with NVRTC without a GPU, and fails loudly (no CPU
fallback) when no device is present."""

import ctypes
import re
import subprocess
from pathlib import Path

import pytest

from paper_0911_3456_b200 import _runtime

HEADER = Path(__file__).resolve().parent.parent / "include" / "rtcg_b200.h"


def declared_symbols():
    text = re.sub(r"/\*.*?\*/", "", HEADER.read_text(), flags=re.S)
    return sorted(set(re.findall(r"\b(rtcg_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_the_bound_symbols():
    declared = declared_symbols()
    assert set(declared) == set(_runtime.EXPORTED_SYMBOLS)


def test_library_exports_every_declared_symbol():
    out = subprocess.run(["nm", "-D", "--defined-only", str(_runtime.LIB_PATH)],
                         capture_output=True, text=True, check=True).stdout
    exported = set(re.findall(r"\bT (rtcg_\w+)", out))
    missing = set(declared_symbols()) - exported
    assert not missing, missing
    lib = ctypes.CDLL(str(_runtime.LIB_PATH))
    for name in declared_symbols():
        assert hasattr(lib, name)
    assert _runtime.lib().rtcg_abi_version() == 1


def test_nvrtc_available_without_gpu():
    major, minor = _runtime.nvrtc_version()
    assert major >= 12
    image, log = _runtime.compile_cubin(
        'extern "C" __global__ void k(int *x) { x[threadIdx.x] = 1; }', ["-arch=sm_100a"])
    assert image[:4] == b"\x7fELF" and log == ""
    with pytest.raises(_runtime.CompilerFailed) as err:
        _runtime.compile_cubin("this is not CUDA", ["-arch=sm_100a"])
    assert "error" in err.value.log


def test_header_compiles_as_c_and_cxx(tmp_path):
    src = tmp_path / "t.c"
    src.write_text('#include "rtcg_b200.h"\nint main(void){return rtcg_abi_version()==1?0:1;}\n')
    for compiler, path in (("cc", src), ("c++", src)):
        subprocess.run([compiler, "-fsyntax-only", f"-I{HEADER.parent}", "-x",
                        "c" if compiler == "cc" else "c++", str(path)], check=True)


def test_no_device_fails_loudly():
    if _runtime.have_gpu():
        pytest.skip("a GPU is present")
    with pytest.raises(_runtime.NoDevice):
        _runtime.mem_alloc(1024)
    with pytest.raises(_runtime.NoDevice):
        _runtime.device_count()


def test_product_never_imports_the_oracle():
    pkg = Path(_runtime.__file__).resolve().parent
    for py in pkg.rglob("*.py"):
        text = py.read_text()
        assert "import oracle" not in text and "from oracle" not in text, py


def _build_c_client(tmp_path):
    exe = tmp_path / "abi_client"
    subprocess.run(["cc", "-std=c11", "-O2", "-Wall", "-Werror", f"-I{HEADER.parent}",
                    str(Path(__file__).resolve().parent / "c" / "abi_client.c"),
                    f"-L{_runtime.LIB_PATH.parent}", "-lrtcg_b200",
                    f"-Wl,-rpath,{_runtime.LIB_PATH.parent}", "-o", str(exe)], check=True)
    return exe


def test_c_client_compiles_through_the_abi(tmp_path):
    """A plain C program linked against librtcg_b200.so (no Python) gets an
    sm_100a cubin from NVRTC and a structured compile error."""
    out = subprocess.run([str(_build_c_client(tmp_path)), "compile"], capture_output=True,
                         text=True, timeout=120)
    assert out.returncode == 0, out.stderr
    assert "cubin" in out.stdout


@pytest.mark.gpu
def test_c_client_launches_through_the_abi(tmp_path):
    """The same C program loads, launches and verifies a kernel on the B200."""
    out = subprocess.run([str(_build_c_client(tmp_path)), "run"], capture_output=True,
                         text=True, timeout=120)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "0 mismatches" in out.stdout
    assert re.search(r"device 0 at [0-9a-fA-F]{4,8}:[0-9a-fA-F]{2}:", out.stdout), out.stdout
