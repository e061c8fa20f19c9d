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

A chain that ends in a reduction (``fusion.reduce(expr, "sum")``, or
``fused(f, reduce="sum")``) becomes the map expression of one generated
ReductionKernel: one HBM pass over the leaves and no materialised result.
Integer sums and max/min equal ``gpuarray.sum/max/min(evaluate(expr))``
bit for bit; float sums fold the same per-element values (fp64 accumulation
for float32) and agree within the reference's fp64-accumulation bound --
exactly when the leaves have the result's width (same chunking).
"""

from __future__ import annotations

import threading

import numpy as np

from . import elementwise as ew
from . import ndarray as nd
from .ndarray import DivisionByZero, NdArray, ShapeMismatch

__all__ = ["Expr", "lazy", "evaluate", "reduce", "fused", "kernel_count"]

_SYMBOLS = {"add": "+", "sub": "-", "mul": "*", "div": "/"}


class Expr:
    """A traced elementwise expression over GPUArrays and scalars.

    The trace is a small tuple tree -- ``("A", array)`` leaves, ``("S", value,
    dtype)`` scalar leaves, ``(symbol, cname, left, right)`` operators --
    built with no string work; the C text is rendered only when a new kernel
    must be generated (the per-call cost of a fused chain is the trace, one
    tree walk and the native launch)."""

    __slots__ = ("node", "dtype", "shape")

    def __init__(self, node: tuple, dtype: nd.Dtype, shape) -> None:
        self.node, self.dtype, self.shape = node, dtype, shape

    # -- building ------------------------------------------------------------------------

    def _binop(self, other, op: str, reverse: bool) -> "Expr":
        symbol = _SYMBOLS[op]
        if other.__class__ is NdArray or isinstance(other, NdArray):
            other = lazy(other)
        if isinstance(other, Expr):
            if other.shape != self.shape:
                raise ShapeMismatch(f"operand shapes differ: {self.shape} vs {other.shape}")
            rt = nd.promote(self.dtype, other.dtype)
            right = other.node
        else:
            sd = ew._scalar_dtype_of(other)
            if sd is nd.int64 and not isinstance(other, np.generic):
                sd = self.dtype  # Python ints adopt the array dtype (eager rule)
            rt = nd.promote(self.dtype, sd)
            if op == "div" and rt.kind != "f" and not reverse and int(other) == 0:
                raise DivisionByZero("integer division by scalar zero")
            right = ("S", other, sd)
        left, right = (right, self.node) if reverse else (self.node, right)
        return Expr((symbol, rt.cname, left, right), rt, self.shape)

    def __add__(self, o): return self._binop(o, "add", False)
    def __radd__(self, o): return self._binop(o, "add", True)
    def __sub__(self, o): return self._binop(o, "sub", False)
    def __rsub__(self, o): return self._binop(o, "sub", True)
    def __mul__(self, o): return self._binop(o, "mul", False)
    def __rmul__(self, o): return self._binop(o, "mul", True)
    def __truediv__(self, o): return self._binop(o, "div", False)
    def __rtruediv__(self, o): return self._binop(o, "div", True)

    # -- views of the trace ----------------------------------------------------------------

    def _leaves(self):
        """(structure key, arrays in first-use order, scalars as (value, dtype))."""
        arrays, ids, scalars = [], {}, []

        def walk(n):
            tag = n[0]
            if tag == "A":
                a = n[1]
                k = ids.get(id(a))
                if k is None:
                    k = ids[id(a)] = len(arrays)
                    arrays.append(a)
                return ("a", k, a.dtype.name)
            if tag == "S":
                scalars.append((n[1], n[2]))
                return ("s", len(scalars) - 1, n[2].name)
            return (tag, n[1], walk(n[2]), walk(n[3]))
        return walk(self.node), tuple(arrays), tuple(scalars)

    @property
    def arrays(self) -> tuple:
        return self._leaves()[1]

    @property
    def scalars(self) -> tuple:
        return self._leaves()[2]

    @property
    def text(self) -> str:
        """The C expression, leaves named ``rtcg_fa<k>`` / ``rtcg_fs<k>``."""
        return _render(self._leaves()[0], "")

    def __repr__(self) -> str:
        return f"<Expr {self.dtype.name} {self.text}>"


def _render(key, index: str) -> str:
    tag = key[0]
    if tag == "a":
        return f"rtcg_fa{key[1]}{index}"
    if tag == "s":
        return f"rtcg_fs{key[1]}"
    c = key[1]
    return (f"(({c}) (({c}) {_render(key[2], index)} {tag} "
            f"({c}) {_render(key[3], index)}))")


def lazy(array: NdArray) -> Expr:
    """A leaf expression reading *array*."""
    if not isinstance(array, NdArray):
        raise TypeError("lazy() takes a GPUArray")
    return Expr(("A", array), array.dtype, array.shape)


_memo: dict = {}
_memo_lock = threading.Lock()


def kernel_count() -> int:
    """Distinct fused kernels built in this process (test hook)."""
    with _memo_lock:
        return len(_memo)


def _kernel_for(key, arrays, scalars, out_dtype: nd.Dtype) -> ew.ElementwiseKernel:
    memo_key = (key, out_dtype.name)
    kernel = _memo.get(memo_key)
    if kernel is None:
        import hashlib
        params = [ew.KernelParam(f"rtcg_fa{k}", a.dtype, True) for k, a in enumerate(arrays)]
        params += [ew.KernelParam(f"rtcg_fs{k}", sd, False) for k, (_, sd) in enumerate(scalars)]
        params.append(ew.KernelParam("rtcg_fo", out_dtype, True))
        sig = ew.KernelSignature(tuple(params))
        op = "rtcg_fo[i] = " + _render(key, "[i]") + ";"
        tag = hashlib.sha256(repr(memo_key).encode()).hexdigest()[:12]
        kernel = ew.ElementwiseKernel(sig, op, f"fused_{tag}")
        with _memo_lock:
            kernel = _memo.setdefault(memo_key, kernel)
    return kernel


def _kernel(expr: Expr, out_dtype: nd.Dtype) -> ew.ElementwiseKernel:
    key, arrays, scalars = expr._leaves()
    return _kernel_for(key, arrays, scalars, out_dtype)


def evaluate(expr, out: NdArray | None = None, stream=None) -> NdArray:
    """Run a traced expression as one kernel; returns (or fills) the result."""
    if isinstance(expr, NdArray):
        return expr
    if not isinstance(expr, Expr):
        raise TypeError("evaluate() takes an Expr")
    key, arrays, scalars = expr._leaves()
    if out is None:
        out = arrays[0].pool.alloc_uninitialized(expr.dtype, expr.shape)
    elif out.dtype != expr.dtype or out.shape != expr.shape:
        raise ShapeMismatch("out does not match the expression's dtype/shape")
    kernel = _kernel_for(key, arrays, scalars, expr.dtype)
    kernel(*arrays, *[v for v, _ in scalars], out, n=out.size, stream=stream)
    return out


_REDUCE_OPS = ("sum", "max", "min")
_reduction_memo: dict = {}


def _reduction_for(key, arrays, scalars, dtype: nd.Dtype, op: str):
    from . import reduction as rd
    memo_key = (key, dtype.name, op)
    kernel = _reduction_memo.get(memo_key)
    if kernel is None:
        import hashlib
        params = [ew.KernelParam(f"rtcg_fa{k}", a.dtype, True) for k, a in enumerate(arrays)]
        params += [ew.KernelParam(f"rtcg_fs{k}", sd, False) for k, (_, sd) in enumerate(scalars)]
        neutral, reduce_expr = {"sum": ("0", "a + b"),
                                "max": (rd._lowest(dtype), "a > b ? a : b"),
                                "min": (rd._highest(dtype), "a < b ? a : b")}[op]
        mapped = _render(key, "[i]")
        if key[0] != "a" or arrays[key[1]].dtype is not dtype:
            mapped = f"(({dtype.cname}) {mapped})"
        spec = rd.ReductionSpec(ew.KernelSignature(tuple(params)), dtype, neutral, reduce_expr,
                                mapped)
        tag = hashlib.sha256(repr(memo_key).encode()).hexdigest()[:12]
        kernel = rd.ReductionKernel(spec, f"fusedr_{tag}")
        with _memo_lock:
            kernel = _reduction_memo.setdefault(memo_key, kernel)
    return kernel


def reduce(expr, op: str = "sum", *, return_device: bool = True, stream=None):  # noqa: A001
    """Reduce a traced expression (``sum`` / ``max`` / ``min``) in one pass:
    the expression is the map of a generated ReductionKernel.  Returns a 0-d
    GPUArray (PyCUDA style) or, with ``return_device=False``, a numpy
    scalar."""
    if op not in _REDUCE_OPS:
        raise ValueError(f"op must be one of {_REDUCE_OPS}, got {op!r}")
    if isinstance(expr, NdArray):
        expr = lazy(expr)
    if not isinstance(expr, Expr):
        raise TypeError("reduce() takes an Expr or a GPUArray")
    key, arrays, scalars = expr._leaves()
    kernel = _reduction_for(key, arrays, scalars, expr.dtype, op)
    return kernel(*arrays, *[v for v, _ in scalars], n=arrays[0].size,
                  return_device=return_device, stream=stream)


def _pure(fn) -> bool:
    """Whether a traced function depends on nothing but its arguments: no
    closure cells and no global names (literal constants only), so its trace
    is a function of the arguments' dtypes, shapes and aliasing."""
    code = getattr(fn, "__code__", None)
    return code is not None and not getattr(fn, "__closure__", None) and not code.co_names


def fused(fn, reduce: str | None = None):  # noqa: A002 - keyword mirrors the function
    """Decorator: ``fused(f)(*arrays)`` traces ``f`` over lazy leaves and
    evaluates it as one kernel; ``fused(f, reduce="sum")`` reduces the traced
    chain in the same pass (a 0-d GPUArray).

    When ``f`` is pure (see :func:`_pure`, e.g. ``lambda x, y: (x*2 + y) -
    x``) and is called with GPUArrays only, the trace is kept per (dtypes,
    shapes, aliasing) of the arguments: later calls skip the tracer and go
    straight to the generated kernel (the same kernel, the same bits)."""
    reducer = reduce
    cache = {} if _pure(fn) else None

    def trace(args):
        return fn(*(Expr(("A", a), a.dtype, a.shape) if a.__class__ is NdArray else
                    lazy(a) if isinstance(a, NdArray) else a for a in args))

    def run(*args, out=None, stream=None):
        key = None
        if cache is not None and args and all(a.__class__ is NdArray for a in args):
            ids = [id(a) for a in args]
            key = (tuple((a.dtype.name, a.shape) for a in args),
                   tuple(ids.index(i) for i in ids))
            hit = cache.get(key)
            if hit is not None:
                run.cache_hits += 1
                kernel, positions, values, dtype, shape = hit
                arrays = [args[p] for p in positions]
                if reducer is not None:
                    return kernel(*arrays, *values, n=arrays[0].size, return_device=True,
                                  stream=stream)
                if out is None:
                    out = arrays[0].pool.alloc_uninitialized(dtype, shape)
                elif out.dtype != dtype or out.shape != shape:
                    raise ShapeMismatch("out does not match the expression's dtype/shape")
                kernel(*arrays, *values, out, n=out.size, stream=stream)
                return out
        traced = trace(args)
        if key is not None and isinstance(traced, Expr):
            skey, arrays, scalars = traced._leaves()
            if reducer is not None:
                kernel = _reduction_for(skey, arrays, scalars, traced.dtype, reducer)
            else:
                kernel = _kernel_for(skey, arrays, scalars, traced.dtype)
            positions = tuple(next(k for k, a in enumerate(args) if a is leaf) for leaf in arrays)
            cache[key] = (kernel, positions, tuple(v for v, _ in scalars), traced.dtype,
                          traced.shape)
        if reducer is not None:
            return globals()["reduce"](traced, reducer, stream=stream)
        return evaluate(traced, out=out, stream=stream)
    run.__name__ = getattr(fn, "__name__", "fused")
    run.cache_hits = 0
    return run
