"""PyCUDA-style ``gpuarray`` namespace over the generated kernels.

``GPUArray`` is :class:`paper_0911_3456_b200.ndarray.NdArray`; this module adds
the usual PyCUDA conveniences on top of the generators, each one a memoised
generated kernel (no hand-written special cases):

* ``to_gpu``, ``empty``, ``zeros``, ``empty_like``, ``zeros_like``;
* ``fill(a, value)``, ``astype(a, dtype)``, ``copy(a)``;
* reductions ``sum``, ``dot``, ``max``, ``min`` returning a 0-d GPUArray
  (PyCUDA's behaviour: no host synchronisation) -- ``.get()`` reads it.
"""

from __future__ import annotations

import threading

from . import _runtime
from . import elementwise as ew
from . import ndarray as nd
from . import reduction as rd
from .ndarray import GPUArray, NdArray, empty, empty_like, to_gpu, zeros, zeros_like

__all__ = ["GPUArray", "to_gpu", "empty", "zeros", "empty_like", "zeros_like", "fill",
           "astype", "copy", "sum", "dot", "max", "min"]

_lock = threading.Lock()
_kernels: dict = {}


def _memo(key, build):
    with _lock:
        k = _kernels.get(key)
    if k is None:
        k = build()
        with _lock:
            k = _kernels.setdefault(key, k)
    return k


def fill(array: NdArray, value) -> NdArray:
    """Set every element to ``value`` (converted like a kernel scalar)."""
    d = array.dtype
    k = _memo(("fill", d.name), lambda: ew.ElementwiseKernel(
        f"{d.cname} v, {d.cname} *z", "z[i] = v", f"fill_{d.name}"))
    k(value, array, n=array.size)
    return array


def astype(array: NdArray, dtype) -> NdArray:
    """A new array with every element converted by a C cast."""
    src, dst = array.dtype, nd.dtype_of(dtype)
    out = array.pool.alloc_uninitialized(dst, array.shape)
    k = _memo(("cast", src.name, dst.name), lambda: ew.ElementwiseKernel(
        f"{src.cname} *x, {dst.cname} *z", f"z[i] = ({dst.cname}) x[i]",
        f"cast_{src.name}_{dst.name}"))
    k(array, out, n=array.size)
    return out


def copy(array: NdArray) -> NdArray:
    """Device-to-device copy into a new array of the same pool."""
    out = array.pool.alloc_uninitialized(array.dtype, array.shape)
    if array.size:
        _runtime.memcpy_dtod(out.address, array.address, array.nbytes)
    return out


def _reduce(kind: str, d: nd.Dtype) -> rd.ReductionKernel:
    makers = {"sum": rd.sum_kernel, "max": rd.max_kernel, "min": rd.min_kernel,
              "dot": rd.dot_kernel}
    return _memo((kind, d.name), lambda: makers[kind](d))


def sum(array: NdArray) -> NdArray:  # noqa: A001 - PyCUDA name
    return _reduce("sum", array.dtype)(array, return_device=True)


def max(array: NdArray) -> NdArray:  # noqa: A001
    return _reduce("max", array.dtype)(array, return_device=True)


def min(array: NdArray) -> NdArray:  # noqa: A001
    return _reduce("min", array.dtype)(array, return_device=True)


def dot(a: NdArray, b: NdArray) -> NdArray:
    """Inner product; operands are promoted to a common dtype first."""
    rt = nd.promote(a.dtype, b.dtype)
    a2 = a if a.dtype is rt else astype(a, rt)
    b2 = b if b.dtype is rt else astype(b, rt)
    return _reduce("dot", rt)(a2, b2, return_device=True)
