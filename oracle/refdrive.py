"""Drive the reference-generated CPU kernels in ``oracle/_ref`` -- TEST
INFRASTRUCTURE ONLY (the CPU baseline of ``bench.py``).

Kernels follow the reference ABI ``void name(void **args, long start, long
end)``; this module reproduces its driver: argument packs with 8-byte widened
scalars (``src/elementwise.py:316-366``), contiguous worker ranges and one host
thread per live range (``:276-313``), and for reductions one partial per
worker folded in worker order by ``<name>_combine`` (``src/reduction.py:
236-258``).  When ``oracle/_ref`` has not been built, :func:`load` falls back
to the C port (``oracle.cport``), which emits equivalent C.
"""

from __future__ import annotations

import ctypes
import json
import os
from pathlib import Path

import numpy as np

from . import cport

REF = Path(__file__).resolve().parent / "_ref"


def available() -> bool:
    return (REF / "manifest.json").exists()


class _RefElementwise:
    def __init__(self, name: str, entry: dict) -> None:
        self.params = cport.parse(entry["signature"])
        self.fn = cport._symbol(ctypes.CDLL(str(REF / f"{name}.so")), name)

    def __call__(self, *args, n=None, workers: int = 1):
        slots, keep, n0 = cport.pack(self.params, args)
        n = n0 if n is None else n
        cport.run_ranges(self.fn, [(slots, s, e) for s, e in cport.worker_ranges(n, workers)])
        del keep


class _RefReduction(cport.Reduction):
    def __init__(self, name: str, entry: dict) -> None:  # noqa: D107 - reuse cport driver
        self.params = cport.parse(entry["signature"])
        self.out = np.dtype(entry["out"])
        self.acc_ct = np.ctypeslib.as_ctypes_type(np.dtype(entry["acc"]))
        lib = ctypes.CDLL(str(REF / f"{name}.so"))
        self.stage1 = cport._symbol(lib, name)
        self.combine = cport._symbol(lib, f"{name}_combine")


def load(name: str):
    """(callable, kind) where kind is "reference" (oracle/_ref) or "port"."""
    from .build_ref import KERNELS
    if available():
        manifest = json.loads((REF / "manifest.json").read_text())
        entry = manifest["kernels"].get(name)
        if entry is not None and (REF / f"{name}.so").exists():
            cls = _RefElementwise if entry["kind"] == "elementwise" else _RefReduction
            return cls(name, entry), "reference"
    kind, sig, what = KERNELS[name]
    if kind == "elementwise":
        return cport.Elementwise(sig, what, name), "port"
    out, neutral, reduce_expr, map_expr = what
    return cport.Reduction(sig, out, neutral, reduce_expr, map_expr, name), "port"


def host_threads() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:  # pragma: no cover
        return os.cpu_count() or 1
