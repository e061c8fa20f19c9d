"""Multi-GPU execution: contiguous shards, one process per GPU.

The reference parallelises over host threads with disjoint index ranges
``[k*n//w, (k+1)*n//w)`` (``src/elementwise.py:306-313``) and combines
reduction partials with an ordered host fold (``src/reduction.py:211-216``).
Here the workers are GPUs (one process each, ``torch.distributed`` for the
plumbing):

* rank r owns global indices ``shard_range(n, r, world)`` -- the same
  formula -- and keeps that slice resident in its HBM; kernels run on the
  local slice with ``base`` = the slice start, so ``i`` in user code stays the
  global index;
* elementwise kernels need no communication;
* reductions do one exchange over NCCL (NVLink / NVSwitch): an ncclAllReduce
  of the 8-byte accumulators when the reduce_expr is exactly an NCCL op
  (integer sum; max/min), otherwise an all-gather of the accumulators into a
  world-sized buffer folded in ascending rank order by the kernel's compiled
  ``<name>_combine`` -- valid for any ``reduce_expr`` and deterministic for a
  fixed world size (float sums always take this path).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _runtime
from . import ndarray as nd

__all__ = ["shard_range", "ShardedArray", "scatter_from_host", "sharded_elementwise",
           "sharded_reduce", "gather_partials", "ordered_fold", "nccl_op"]


def shard_range(n: int, rank: int, world: int) -> tuple[int, int]:
    """Global ``[lo, hi)`` owned by *rank*; the reference's worker formula."""
    if not 0 <= rank < world:
        raise ValueError(f"rank {rank} outside world of {world}")
    return rank * n // world, (rank + 1) * n // world


@dataclass
class ShardedArray:
    """This rank's slice of a global 1-d array of ``n`` elements."""

    local: nd.NdArray
    base: int
    n: int
    rank: int
    world: int

    @property
    def dtype(self):
        return self.local.dtype

    def free(self) -> None:
        self.local.free()


def scatter_from_host(host: np.ndarray | None, dtype, n: int, rank: int, world: int,
                      pool: nd.MemoryPool | None = None, fill=None) -> ShardedArray:
    """Upload this rank's slice of *host* (or of ``fill(lo, hi)``, which lets a
    rank synthesise only its own slice)."""
    lo, hi = shard_range(n, rank, world)
    pool = pool or nd.default_pool()
    values = fill(lo, hi) if fill is not None else host[lo:hi]
    return ShardedArray(nd.from_host(pool, dtype, values), lo, n, rank, world)


def _locals(args):
    base = None
    out = []
    for a in args:
        if isinstance(a, ShardedArray):
            if base is not None and a.base != base:
                raise ValueError("sharded arguments are not co-partitioned")
            base = a.base
            out.append(a.local)
        else:
            out.append(a)
    if base is None:
        raise ValueError("no sharded argument")
    return out, base


def sharded_elementwise(kernel, *args, stream=None) -> None:
    """Run an ElementwiseKernel on this rank's slices (no communication)."""
    local_args, base = _locals(args)
    n_local = next(a.size for a in local_args if isinstance(a, nd.NdArray))
    kernel(*local_args, n=n_local, base=base, stream=stream)


def ordered_fold(fold, neutral, values):
    """Host statement of the combine semantics (ascending rank order)."""
    acc = neutral
    for v in values:
        acc = fold(acc, v)
    return acc


def gather_partials(partial, group=None):
    """All-gather one accumulator per rank (torch tensor of shape (1,)) into a
    (world,) tensor ordered by rank.  NCCL for CUDA tensors, gloo for CPU."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    out = torch.empty(world, dtype=partial.dtype, device=partial.device)
    dist.all_gather_into_tensor(out, partial.reshape(1), group=group)
    return out


class _DeviceView:
    """__cuda_array_interface__ over raw device memory (scratch buffers)."""

    def __init__(self, address: int, count: int, dtype: nd.Dtype) -> None:
        self.__cuda_array_interface__ = {"shape": (count,), "typestr": dtype.np.str,
                                         "data": (address, False), "version": 3,
                                         "strides": None}


_NCCL_OPS = {"a+b": "sum", "b+a": "sum", "a>b?a:b": "max", "b>a?b:a": "max",
             "a<b?a:b": "min", "b<a?b:a": "min"}


def nccl_op(spec) -> str | None:
    """The NCCL reduction equal to ``spec.reduce_expr`` *exactly*, or None.

    sum is exact (order-independent) only for integer accumulators (two's
    complement wrap); max/min are exact for every dtype on NaN-free data.
    Float sums keep the ordered fold so results do not depend on NCCL's
    reduction order."""
    op = _NCCL_OPS.get("".join(spec.reduce_expr.split()))
    if spec.acc_dtype.name not in _NCCL_DTYPES:
        return None
    if op == "sum" and spec.acc_dtype.kind == "f":
        return None
    return op


# accumulator dtypes both NCCL and torch's NCCL backend reduce natively
_NCCL_DTYPES = {"int8", "uint8", "int32", "int64", "float32", "float64"}


def sharded_reduce(kernel, *args, group=None, return_device: bool = False,
                   collective: str = "auto"):
    """Global reduction of a ReductionKernel over sharded arguments.

    1. local two-stage reduction into the kernel's scratch accumulator;
    2. the cross-GPU step over NCCL (NVLink / NVSwitch):
       ``"allreduce"`` -- one ncclAllReduce of the 8-byte accumulators when
       :func:`nccl_op` maps ``reduce_expr`` to an exact NCCL op;
       ``"allgather"`` -- all-gather (world x 8 bytes) + ``<name>_combine``
       folding in rank order, valid for any ``reduce_expr``;
       ``"auto"`` -- allreduce when exact, else allgather;
    3. the out-dtype value is written on the device.
    Everything runs in stream order on torch's current stream.
    """
    import torch
    import torch.distributed as dist

    local_args, base = _locals(args)
    n_local = next(a.size for a in local_args if isinstance(a, nd.NdArray))
    spec = kernel.spec
    op = nccl_op(spec)
    if collective == "auto":
        collective = "allreduce" if op is not None else "allgather"
    if collective == "allreduce" and op is None:
        raise ValueError(f"reduce_expr {spec.reduce_expr!r} has no exact NCCL equivalent")
    if collective not in ("allreduce", "allgather"):
        raise ValueError(f"unknown collective {collective!r}")
    stream = torch.cuda.current_stream().cuda_stream
    with _runtime.use_stream(stream):
        scratch = kernel.launch(*local_args, n=n_local, base=base)
        acc_view = torch.as_tensor(_DeviceView(scratch.result, 1, spec.acc_dtype), device="cuda")
        first = next(a for a in local_args if isinstance(a, nd.NdArray))
        out = first.pool.alloc_uninitialized(spec.out_dtype, ())
        if collective == "allreduce":
            reduce_op = {"sum": dist.ReduceOp.SUM, "max": dist.ReduceOp.MAX,
                         "min": dist.ReduceOp.MIN}[op]
            dist.all_reduce(acc_view, op=reduce_op, group=group)
            # fold the single global accumulator once more to write the out
            # dtype (a fold of one value from the neutral is the identity)
            kernel._launch_combine(scratch.result, 1, scratch.result, out.address)
        else:
            gathered = gather_partials(acc_view, group)
            kernel._launch_combine(gathered.data_ptr(), gathered.numel(), scratch.result,
                                   out.address)
        if return_device:
            # `gathered` goes back to torch's caching allocator; its reuse is
            # ordered after the combine because both run on this stream
            return out
        value = out.to_host()
        out.free()
        return spec.out_dtype.np.type(value[()])
