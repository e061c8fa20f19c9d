"""C restatement of rtcg-kit's generated CPU kernels -- TEST INFRASTRUCTURE ONLY.

The reference turns a signature + C text into C (``src/elementwise.py:204-270``
for elementwise, ``src/reduction.py:98-181`` for reductions), compiles it with
``cc -O2 -ffp-contract=off -shared -fPIC`` (``src/jit.py:43,452-453``) and
calls ``void name(void **args, long start, long end)`` from one host thread per
worker range (``src/elementwise.py:276-313``).  This module re-states those
rules compactly so the GPU results can be checked against the same C
semantics, compiler and libm on any host that has ``cc`` -- including the GPU
box, where ``/root/reference`` does not exist.

Arguments are numpy arrays (vectors) and Python/numpy scalars.
"""

from __future__ import annotations

import ctypes
import hashlib
import os
import re
import subprocess
import tempfile
import threading
from pathlib import Path

import numpy as np

CC = os.environ.get("RTCG_ORACLE_CC", "cc")
CFLAGS = ("-O2", "-ffp-contract=off")   # src/jit.py:43

# C spelling -> (numpy dtype name, kind); aliases as src/elementwise.py:67-72
_TYPES = {
    "int8_t": ("int8", "i"), "int16_t": ("int16", "i"), "int32_t": ("int32", "i"),
    "int64_t": ("int64", "i"), "uint8_t": ("uint8", "u"), "uint16_t": ("uint16", "u"),
    "uint32_t": ("uint32", "u"), "uint64_t": ("uint64", "u"), "float": ("float32", "f"),
    "double": ("float64", "f"), "short": ("int16", "i"), "int": ("int32", "i"),
    "long": ("int64", "i"),
}
_CNAME = {"int8": "int8_t", "int16": "int16_t", "int32": "int32_t", "int64": "int64_t",
          "uint8": "uint8_t", "uint16": "uint16_t", "uint32": "uint32_t",
          "uint64": "uint64_t", "float32": "float", "float64": "double"}
_SLOT = {"i": ("int64_t", ctypes.c_int64), "u": ("uint64_t", ctypes.c_uint64),
         "f": ("double", ctypes.c_double)}
_I = re.compile(r"\bi\b")
_AB = re.compile(r"\b([ab])\b")


def parse(signature: str):
    """[(name, numpy dtype name, kind, is_vector)] in declaration order."""
    out = []
    for piece in signature.split(","):
        m = re.fullmatch(r"\s*(\w+)\s*(\*?)\s*(\w+)\s*", piece)
        if not m or m.group(1) not in _TYPES:
            raise ValueError(f"oracle cannot parse {piece!r}")
        npname, kind = _TYPES[m.group(1)]
        out.append((m.group(3), npname, kind, m.group(2) == "*"))
    return out


def _decls(params) -> list[str]:
    lines = []
    for k, (name, npname, kind, vec) in enumerate(params):
        c = _CNAME[npname]
        if vec:
            lines.append(f"    {c} *{name} = ({c} *) args[{k}];")
        else:
            lines.append(f"    {c} {name} = ({c}) *(const {_SLOT[kind][0]} *) args[{k}];")
    return lines


def _stmt(text: str, offset: int) -> str:
    body = text if offset == 0 else _I.sub(f"(i + {offset})", text)
    return "{ " + body + " }"


def _loops(stmt_of, unroll: int) -> list[str]:
    lines = ["    long i = start;"]
    if unroll > 1:
        lines.append(f"    for (; i + {unroll - 1} < end; i += {unroll}) {{")
        lines += [f"        {stmt_of(k)}" for k in range(unroll)]
        lines.append("    }")
    lines.append("    for (; i < end; ++i) {")
    lines.append(f"        {stmt_of(0)}")
    lines.append("    }")
    return lines


def elementwise_source(signature: str, operation: str, name: str, unroll: int = 4) -> str:
    op = operation.strip()
    op = op if op.endswith(";") else op + ";"
    params = parse(signature)
    body = _decls(params) + _loops(lambda k: _stmt(op, k), unroll)
    return "\n".join(["#include <stdint.h>", "#include <math.h>",
                      f"void {name}(void **args, long start, long end)", "{",
                      *body, "}", ""])


def acc_cname(out_npname: str) -> str:
    """float32 accumulates in double (src/reduction.py:53-54)."""
    return "double" if out_npname == "float32" else _CNAME[out_npname]


def reduction_source(signature: str, out_npname: str, neutral: str, reduce_expr: str,
                     map_expr: str | None, name: str, unroll: int = 4) -> str:
    params = parse(signature)
    mapped = map_expr if map_expr is not None else \
        next(f"{p[0]}[i]" for p in params if p[3]) + ""
    acc = acc_cname(out_npname)

    def fold(k: int) -> str:
        m = mapped if k == 0 else _I.sub(f"(i + {k})", mapped)
        return "acc = " + _AB.sub(lambda g: "acc" if g.group(1) == "a" else f"({m})",
                                  reduce_expr) + ";"

    combine = _AB.sub(lambda g: "acc" if g.group(1) == "a" else "partials[i]", reduce_expr)
    stage1 = _decls(params) + [f"    {acc} *partial_out = ({acc} *) args[{len(params)}];",
                               f"    {acc} acc = {neutral};"]
    stage1 += _loops(fold, unroll) + ["    partial_out[0] = acc;"]
    return "\n".join([
        "#include <stdint.h>", "#include <math.h>",
        f"void {name}(void **args, long start, long end)", "{", *stage1, "}", "",
        f"void {name}_combine(void **args, long start, long end)", "{",
        f"    const {acc} *partials = (const {acc} *) args[0];",
        f"    {acc} *result = ({acc} *) args[1];",
        f"    {acc} acc = {neutral};",
        "    for (long i = start; i < end; ++i) {",
        f"        acc = {combine};",
        "    }",
        "    result[0] = acc;", "}", ""])


# --- compile (content-addressed, per process + on disk) ---------------------------------

_CACHE = Path(os.environ.get("RTCG_ORACLE_CACHE") or
              Path(tempfile.gettempdir()) / "rtcg-b200-oracle")
_loaded: dict[str, ctypes.CDLL] = {}
_load_lock = threading.Lock()


def build(source: str) -> ctypes.CDLL:
    key = hashlib.sha256((CC + " ".join(CFLAGS) + source).encode()).hexdigest()[:24]
    with _load_lock:
        lib = _loaded.get(key)
        if lib is not None:
            return lib
        _CACHE.mkdir(parents=True, exist_ok=True)
        so = _CACHE / f"{key}.so"
        if not so.exists():
            src = _CACHE / f"{key}.c"
            src.write_text(source)
            tmp = _CACHE / f"{key}.{os.getpid()}.so"
            proc = subprocess.run([CC, *CFLAGS, "-shared", "-fPIC", "-o", str(tmp), str(src), "-lm"],
                                  capture_output=True, text=True)
            if proc.returncode != 0:
                raise RuntimeError(f"oracle compile failed:\n{proc.stderr}\n{source}")
            os.replace(tmp, so)
        lib = _loaded[key] = ctypes.CDLL(str(so))
        return lib


def _symbol(lib, name):
    fn = getattr(lib, name)
    fn.argtypes = (ctypes.POINTER(ctypes.c_void_p), ctypes.c_long, ctypes.c_long)
    fn.restype = None
    return fn


# --- driver (src/elementwise.py:276-366, src/reduction.py:236-258) ------------------------


def worker_ranges(n: int, workers: int):
    return [(k * n // workers, (k + 1) * n // workers) for k in range(workers)]


def run_ranges(fn, tasks) -> None:
    live = [t for t in tasks if t[1] < t[2]]
    if len(live) == 1:
        fn(*live[0])
        return
    threads = [threading.Thread(target=fn, args=t) for t in live]
    for t in threads:
        t.start()
    for t in threads:
        t.join()


def pack(params, args, extra: int = 0):
    if len(args) != len(params):
        raise TypeError(f"expected {len(params)} arguments, got {len(args)}")
    slots = (ctypes.c_void_p * (len(params) + extra))()
    keep, n = [], None
    for k, ((name, npname, kind, vec), arg) in enumerate(zip(params, args)):
        if vec:
            arr = np.asarray(arg)
            if arr.dtype != np.dtype(npname) or not arr.flags.c_contiguous:
                raise TypeError(f"{name}: need contiguous {npname}")
            n = arr.size if n is None else n
            slots[k] = arr.ctypes.data
            keep.append(arr)
        else:
            ct = _SLOT[kind][1]
            v = ct(float(arg)) if kind == "f" else ct(int(arg) & 0xFFFFFFFFFFFFFFFF) \
                if kind == "u" else ct(int(arg))
            keep.append(v)
            slots[k] = ctypes.addressof(v)
    return slots, keep, n


class Elementwise:
    """``Elementwise(sig, op)(x, y, z, n=None, workers=1)`` mutates the numpy
    output arrays in place, exactly like the reference kernel would."""

    def __init__(self, signature: str, operation: str, name: str = "k", unroll: int = 4):
        self.params = parse(signature)
        self.source = elementwise_source(signature, operation, name, unroll)
        self.fn = _symbol(build(self.source), name)

    def __call__(self, *args, n: int | None = None, workers: int = 1) -> None:
        slots, keep, n0 = pack(self.params, args)
        n = n0 if n is None else n
        run_ranges(self.fn, [(slots, s, e) for s, e in worker_ranges(n, workers)])
        del keep


class Reduction:
    """``Reduction(sig, out, neutral, reduce, map)(args..., workers=1)`` ->
    numpy scalar of the out dtype, with the reference's two-stage fold."""

    def __init__(self, signature: str, out_npname: str, neutral: str, reduce_expr: str,
                 map_expr: str | None = None, name: str = "r", unroll: int = 4):
        self.params = parse(signature)
        self.out = np.dtype(out_npname)
        acc = acc_cname(out_npname)
        self.acc_ct = {"double": ctypes.c_double, "float": ctypes.c_float}.get(acc) or \
            np.ctypeslib.as_ctypes_type(np.dtype(_TYPES[acc][0]))
        self.source = reduction_source(signature, out_npname, neutral, reduce_expr,
                                       map_expr, name, unroll)
        lib = build(self.source)
        self.stage1 = _symbol(lib, name)
        self.combine = _symbol(lib, f"{name}_combine")

    def fold_partials(self, partials) -> object:
        arr = (self.acc_ct * max(1, len(partials)))(*partials)
        res = self.acc_ct()
        slots = (ctypes.c_void_p * 2)(ctypes.addressof(arr), ctypes.addressof(res))
        self.combine(slots, 0, len(partials))
        return res.value

    def partials(self, *args, n: int | None = None, workers: int = 1) -> list:
        slots, keep, n0 = pack(self.params, args, extra=1)
        n = n0 if n is None else n
        live = [r for r in worker_ranges(n, workers) if r[0] < r[1]]
        parts = (self.acc_ct * max(1, len(live)))()
        size = ctypes.sizeof(self.acc_ct)
        tasks = []
        for slot, (s, e) in enumerate(live):
            wp = (ctypes.c_void_p * len(slots))(*list(slots)[:-1],
                                                 ctypes.addressof(parts) + slot * size)
            tasks.append((wp, s, e))
        run_ranges(self.stage1, tasks)
        del keep
        return [parts[k] for k in range(len(live))]

    def __call__(self, *args, n: int | None = None, workers: int = 1):
        return self.out.type(self.fold_partials(self.partials(*args, n=n, workers=workers)))
