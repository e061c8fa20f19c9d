"""Eager GPUArray operator chains on the host -- TEST INFRASTRUCTURE ONLY.

Restates the reference's array operators so fused and eager GPU chains can
be checked against C semantics rather than against each other:

* ``array_binary_op`` (``src/elementwise.py:528-576``): one generated kernel
  per operator, ``z[i] = (rt) x[i] OP (rt) y[i]`` (vector-vector) or
  ``z[i] = (rt) x[i] OP (rt) s`` / ``(rt) s OP (rt) x[i]`` (vector-scalar),
  each result stored in a fresh array of the promoted dtype ``rt``;
* ``_scalar_dtype_of`` (``src/elementwise.py:431-440``): numpy scalars keep
  their dtype, Python floats are float64, Python ints are int64 -- and a
  plain Python int adopts the array's dtype (``:561-565``);
* ``promote`` (``src/ndarray.py:100-129``);
* integer division by a scalar zero raises (``:567-568``).

Every operator runs through ``cport.Elementwise`` -- the reference's C text
compiled with its own compiler command -- so each temporary is exactly what
the reference would store.  ``HostArray`` mirrors ``NdArray``'s ``+ - * /``
dunders (``src/ndarray.py:347-358``).
"""

from __future__ import annotations

import numpy as np

from . import cport

_SYMBOL = {"add": "+", "sub": "-", "mul": "*", "div": "/"}
_SIGNED = {1: "int8", 2: "int16", 4: "int32", 8: "int64"}


def promote(a: str, b: str) -> str:
    """Result dtype name of combining numpy dtype names a and b."""
    if a == b:
        return a
    da, db = np.dtype(a), np.dtype(b)
    if da.kind == db.kind:
        return a if da.itemsize >= db.itemsize else b
    if "f" in (da.kind, db.kind):
        f, i = (da, db) if da.kind == "f" else (db, da)
        value_bits = i.itemsize * 8 - (1 if i.kind == "i" else 0)
        return "float32" if f.itemsize == 4 and value_bits <= 24 else "float64"
    s, u = (da, db) if da.kind == "i" else (db, da)
    needed = s.itemsize if u.itemsize < s.itemsize else u.itemsize * 2
    return "float64" if needed > 8 else _SIGNED[needed]


def scalar_dtype(value, array_dtype: str) -> str:
    if isinstance(value, np.generic):
        return np.dtype(type(value)).name
    if isinstance(value, float):
        return "float64"
    return array_dtype            # plain Python int adopts the array dtype


_kernels: dict = {}


def _kernel(sig: str, op: str) -> cport.Elementwise:
    k = _kernels.get((sig, op))
    if k is None:
        k = _kernels[(sig, op)] = cport.Elementwise(sig, op, "ew_op")
    return k


class HostArray:
    """A host array whose operators run the reference's operator kernels."""

    __slots__ = ("values",)

    def __init__(self, values) -> None:
        self.values = np.ascontiguousarray(values)

    @property
    def dtype(self) -> str:
        return self.values.dtype.name

    def _binop(self, other, op: str, reverse: bool) -> "HostArray":
        sym = _SYMBOL[op]
        cn = cport._CNAME
        if isinstance(other, HostArray):
            a, b = (other, self) if reverse else (self, other)
            rt = promote(a.dtype, b.dtype)
            z = np.zeros(self.values.size, rt)
            _kernel(f"{cn[a.dtype]} *x, {cn[b.dtype]} *y, {cn[rt]} *z",
                    f"z[i] = ({cn[rt]}) x[i] {sym} ({cn[rt]}) y[i]")(a.values, b.values, z)
            return HostArray(z)
        sd = scalar_dtype(other, self.dtype)
        rt = promote(self.dtype, sd)
        if op == "div" and np.dtype(rt).kind != "f" and not reverse and int(other) == 0:
            raise ZeroDivisionError("integer division by scalar zero")
        expr = (f"z[i] = ({cn[rt]}) s {sym} ({cn[rt]}) x[i]" if reverse
                else f"z[i] = ({cn[rt]}) x[i] {sym} ({cn[rt]}) s")
        z = np.zeros(self.values.size, rt)
        _kernel(f"{cn[sd]} s, {cn[self.dtype]} *x, {cn[rt]} *z", expr)(other, self.values, z)
        return HostArray(z)

    def __add__(self, o): return self._binop(o, "add", False)
    def __radd__(self, o): return self._binop(o, "add", True)
    def __sub__(self, o): return self._binop(o, "sub", False)
    def __rsub__(self, o): return self._binop(o, "sub", True)
    def __mul__(self, o): return self._binop(o, "mul", False)
    def __rmul__(self, o): return self._binop(o, "mul", True)
    def __truediv__(self, o): return self._binop(o, "div", False)
    def __rtruediv__(self, o): return self._binop(o, "div", True)


def reduce(values: np.ndarray, op: str):
    """The reference's stock sum/max/min (``src/reduction.py:273-312``) over
    a host array, sequential fold (acc float64 for float32)."""
    d = values.dtype.name
    cn = cport._CNAME[d]
    kind = values.dtype.kind
    low = {"i": f"INT{values.dtype.itemsize * 8}_MIN", "u": "0", "f": "-INFINITY"}[kind]
    high = {"i": f"INT{values.dtype.itemsize * 8}_MAX",
            "u": f"UINT{values.dtype.itemsize * 8}_MAX", "f": "INFINITY"}[kind]
    neutral, expr = {"sum": ("0", "a + b"), "max": (low, "a > b ? a : b"),
                     "min": (high, "a < b ? a : b")}[op]
    return cport.Reduction(f"{cn} *x", d, neutral, expr)(values)
