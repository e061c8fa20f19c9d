"""Build the native runtime in tree: ``python -m paper_0911_3456_b200._build``.

* ``librtcg_b200.so`` -- the C-ABI runtime (NVRTC + CUDA driver; host code).
* ``_fastlaunch*.so`` -- CPython extension: per-call argument marshalling,
  vector-path / grid decisions and the launch of generated kernels in C++.
* ``prebuilt/*.cubin`` -- ahead-of-time nvcc builds of the kernel templates
  instantiated for the stock kernels (axpy, dot, sum, max|x|), compiled with
  ``-gencode arch=compute_100a,code=sm_100a -lineinfo``.  They prove the
  templates compile with nvcc as well as NVRTC and give ``cuobjdump -sass``
  something to inspect (128-bit LDG/STG) without a GPU.  Run-time kernels are
  still generated and compiled through NVRTC.
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
CSRC = PKG / "csrc"
INCLUDE = PKG.parent / "include"
LIB = PKG / "librtcg_b200.so"
PREBUILT = PKG / "prebuilt"
CUDA_HOME = Path(os.environ.get("CUDA_HOME", "/usr/local/cuda"))
GENCODE = "-gencode=arch=compute_100a,code=sm_100a"


def _run(cmd: list[str]) -> None:
    proc = subprocess.run(cmd, capture_output=True, text=True)
    if proc.returncode != 0:
        raise RuntimeError(f"build step failed: {' '.join(cmd)}\n{proc.stdout}{proc.stderr}")


def _stale(target: Path, *sources: Path) -> bool:
    if not target.exists():
        return True
    t = target.stat().st_mtime
    return any(s.stat().st_mtime > t for s in sources)


def build_runtime(force: bool = False) -> Path:
    src = CSRC / "rtcg_runtime.cpp"
    header = INCLUDE / "rtcg_b200.h"
    if force or _stale(LIB, src, header):
        cxx = os.environ.get("CXX") or shutil.which("g++") or "c++"
        tmp = LIB.with_suffix(".so.tmp")
        _run([cxx, "-O2", "-std=c++17", "-shared", "-fPIC", "-Wall",
              f"-I{CUDA_HOME / 'include'}", f"-I{INCLUDE}", str(src), "-ldl", "-pthread",
              "-o", str(tmp)])
        os.replace(tmp, LIB)
    return LIB


def build_fastlaunch(force: bool = False) -> Path:
    import sysconfig
    src = CSRC / "fastlaunch.cpp"
    target = PKG / f"_fastlaunch{sysconfig.get_config_var('EXT_SUFFIX')}"
    if force or _stale(target, src):
        cxx = os.environ.get("CXX") or shutil.which("g++") or "c++"
        tmp = target.with_suffix(".tmp")
        _run([cxx, "-O2", "-std=c++17", "-shared", "-fPIC", "-Wall",
              f"-I{sysconfig.get_paths()['include']}", str(src), "-o", str(tmp)])
        os.replace(tmp, target)
    return target


def build_prebuilt(force: bool = False) -> list[Path]:
    """nvcc-compile the stock kernel instantiations to sm_100a cubins."""
    from . import aot  # generates the stock kernel sources

    nvcc = str(CUDA_HOME / "bin" / "nvcc")
    PREBUILT.mkdir(exist_ok=True)
    out = []
    for name, source in aot.stock_sources().items():
        cu = PREBUILT / f"{name}.cu"
        cubin = PREBUILT / f"{name}.cubin"
        if not force and cu.exists() and cu.read_text() == source and cubin.exists():
            out.append(cubin)
            continue
        cu.write_text(source)
        _run([nvcc, GENCODE, "-lineinfo", "-O3", "-std=c++17", "-fmad=false",
              "-Xptxas", "-v", "-cubin", "-o", str(cubin), str(cu)])
        out.append(cubin)
    return out


def main(argv=None) -> int:
    argv = list(sys.argv[1:] if argv is None else argv)
    force = "--force" in argv
    print(build_runtime(force))
    print(build_fastlaunch(force))
    if "--no-prebuilt" not in argv:
        for p in build_prebuilt(force):
            print(p)
    return 0


if __name__ == "__main__":
    raise SystemExit(main())
