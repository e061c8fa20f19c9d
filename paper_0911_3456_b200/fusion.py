"""Expression-chain fusion for GPUArray arithmetic.

``z = (x * 2 + y) - x`` with eager operators runs three kernels and
allocates two temporaries, each a full HBM pass (``src/ndarray.py:347-358``,
``src/elementwise.py:528-576``).  The paper motivates ``ElementwiseKernel``
precisely by removing such temporaries.  Here the same
chain is traced into one C expression and evaluated by one generated kernel:

    from paper_0911_3456_b200 import fusion
    z = fusion.evaluate((fusion.lazy(x) * 2 + y) - x)
    # or
    f = fusion.fused(lambda x, y: (x * 2 + y) - x)
    z = f(x, y)

Results are bit-identical to the eager chain: every node applies the eager
operator's promotion and scalar rules and casts its result back to the
promoted dtype, exactly the value the eager kernel would have stored in its
temporary (e.g. int8 + int8 wraps to int8 before the next operator).
"""

from __future__ import annotations

import threading

import numpy as np

from . import elementwise as ew
from . import ndarray as nd
from .ndarray import DivisionByZero, NdArray, ShapeMismatch

__all__ = ["Expr", "lazy", "evaluate", "fused", "kernel_count"]

_SYMBOLS = {"add": "+", "sub": "-", "mul": "*", "div": "/"}


class Expr:
    """A traced elementwise expression over GPUArrays and scalars."""

    __slots__ = ("text", "dtype", "arrays", "scalars", "shape")

    def __init__(self, text: str, dtype: nd.Dtype, arrays: tuple, scalars: tuple, shape):
        self.text, self.dtype, self.arrays, self.scalars, self.shape = \
            text, dtype, arrays, scalars, shape

    # -- building ------------------------------------------------------------------------

    def _merge(self, other: "Expr"):
        """Union of leaves; returns (arrays, scalars, remap of other's names)."""
        arrays, scalars = list(self.arrays), list(self.scalars)
        text = other.text
        ids = {id(a): k for k, a in enumerate(arrays)}
        renames = {}
        for k, a in enumerate(other.arrays):
            j = ids.get(id(a))
            if j is None:
                j = len(arrays)
                arrays.append(a)
                ids[id(a)] = j
            renames[f"rtcg_fa{k}"] = f"rtcg_fa{j}"
        for k, s in enumerate(other.scalars):
            renames[f"rtcg_fs{k}"] = f"rtcg_fs{len(scalars)}"
            scalars.append(s)
        if renames:
            import re
            text = re.sub(r"\brtcg_f[as]\d+\b", lambda m: renames.get(m.group(0), m.group(0)),
                          text)
        return tuple(arrays), tuple(scalars), text

    def _binop(self, other, op: str, reverse: bool) -> "Expr":
        symbol = _SYMBOLS[op]
        if isinstance(other, NdArray):
            other = lazy(other)
        if isinstance(other, Expr):
            if other.shape != self.shape:
                raise ShapeMismatch(f"operand shapes differ: {self.shape} vs {other.shape}")
            arrays, scalars, other_text = self._merge(other)
            rt = nd.promote(self.dtype, other.dtype)
            left, right = (other_text, self.text) if reverse else (self.text, other_text)
        else:
            sd = ew._scalar_dtype_of(other)
            if sd is nd.int64 and not isinstance(other, np.generic):
                sd = self.dtype  # Python ints adopt the array dtype (eager rule)
            rt = nd.promote(self.dtype, sd)
            if op == "div" and rt.kind != "f" and not reverse and int(other) == 0:
                raise DivisionByZero("integer division by scalar zero")
            arrays = self.arrays
            scalars = self.scalars + ((other, sd),)
            name = f"rtcg_fs{len(self.scalars)}"
            left, right = (name, self.text) if reverse else (self.text, name)
        c = rt.cname
        text = f"(({c}) (({c}) {left} {symbol} ({c}) {right}))"
        return Expr(text, rt, arrays, scalars, self.shape)

    def __add__(self, o): return self._binop(o, "add", False)
    def __radd__(self, o): return self._binop(o, "add", True)
    def __sub__(self, o): return self._binop(o, "sub", False)
    def __rsub__(self, o): return self._binop(o, "sub", True)
    def __mul__(self, o): return self._binop(o, "mul", False)
    def __rmul__(self, o): return self._binop(o, "mul", True)
    def __truediv__(self, o): return self._binop(o, "div", False)
    def __rtruediv__(self, o): return self._binop(o, "div", True)

    def __repr__(self) -> str:
        return f"<Expr {self.dtype.name} {self.text}>"


def lazy(array: NdArray) -> Expr:
    """A leaf expression reading *array*."""
    if not isinstance(array, NdArray):
        raise TypeError("lazy() takes a GPUArray")
    return Expr("rtcg_fa0", array.dtype, (array,), (), array.shape)


_memo: dict = {}
_memo_lock = threading.Lock()


def kernel_count() -> int:
    """Distinct fused kernels built in this process (test hook)."""
    with _memo_lock:
        return len(_memo)


def _kernel(expr: Expr, out_dtype: nd.Dtype) -> ew.ElementwiseKernel:
    params = [ew.KernelParam(f"rtcg_fa{k}", a.dtype, True) for k, a in enumerate(expr.arrays)]
    params += [ew.KernelParam(f"rtcg_fs{k}", sd, False) for k, (_, sd) in enumerate(expr.scalars)]
    params.append(ew.KernelParam("rtcg_fo", out_dtype, True))
    key = (expr.text, tuple((p.name, p.dtype.name, p.is_vector) for p in params))
    with _memo_lock:
        kernel = _memo.get(key)
    if kernel is None:
        import hashlib
        sig = ew.KernelSignature(tuple(params))
        op = "rtcg_fo[i] = " + _index(expr.text) + ";"
        tag = hashlib.sha256(repr(key).encode()).hexdigest()[:12]
        kernel = ew.ElementwiseKernel(sig, op, f"fused_{tag}")
        with _memo_lock:
            kernel = _memo.setdefault(key, kernel)
    return kernel


def _index(text: str) -> str:
    """Leaf names -> element references (``rtcg_fa0`` -> ``rtcg_fa0[i]``)."""
    import re
    return re.sub(r"\b(rtcg_fa\d+)\b", r"\1[i]", text)


def evaluate(expr, out: NdArray | None = None, stream=None) -> NdArray:
    """Run a traced expression as one kernel; returns (or fills) the result."""
    if isinstance(expr, NdArray):
        return expr
    if not isinstance(expr, Expr):
        raise TypeError("evaluate() takes an Expr")
    first = expr.arrays[0]
    if out is None:
        out = first.pool.alloc_uninitialized(expr.dtype, expr.shape)
    elif out.dtype != expr.dtype or out.shape != expr.shape:
        raise ShapeMismatch("out does not match the expression's dtype/shape")
    kernel = _kernel(expr, expr.dtype)
    kernel(*expr.arrays, *(v for v, _ in expr.scalars), out, n=out.size, stream=stream)
    return out


def fused(fn):
    """Decorator: ``fused(f)(*arrays)`` traces ``f`` over lazy leaves and
    evaluates it as one kernel."""
    def run(*args, out=None, stream=None):
        traced = fn(*(lazy(a) if isinstance(a, NdArray) else a for a in args))
        return evaluate(traced, out=out, stream=stream)
    run.__name__ = getattr(fn, "__name__", "fused")
    return run
