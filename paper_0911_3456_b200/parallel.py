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
* reductions do one exchange.  The product path (``collective="p2p"``) does
  it inside the reduction kernel: its last CTA stores the device accumulator
  into every rank's mailbox over NVLink / NVSwitch peer memory (CUDA IPC
  mappings, :class:`PeerMailbox`), waits for the world's accumulators to land
  in its own mailbox and folds them in ascending rank order -- one launch per
  GPU, no collective call, any ``reduce_expr``, the same bits on every rank.
  The NCCL paths remain as the baseline: an ncclAllReduce of the 8-byte
  accumulators when the reduce_expr is exactly an NCCL op (integer sum;
  max/min), otherwise an all-gather of the accumulators folded in rank order
  by the kernel's compiled ``<name>_combine`` (same fold, same result).
"""

from __future__ import annotations

from dataclasses import dataclass

import ctypes
import struct
import threading

import numpy as np

from . import _runtime
from . import ndarray as nd
from .reduction import _host_slot

__all__ = ["shard_range", "ShardedArray", "scatter_from_host", "sharded_elementwise",
           "sharded_reduce", "gather_partials", "ordered_fold", "nccl_op", "PeerMailbox",
           "PeerTimeout", "peer_mailbox", "p2p_capable", "peer_plan"]


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


# --- peer-memory exchange (the fused cross-GPU combine) -------------------------------------

XR_MAX = 64                             # rtcg::XR_MAX in templates/prelude.cuh
XR_ERROR = 4 * XR_MAX                   # rtcg::XR_ERROR: epoch of a timed-out wait
MAILBOX_BYTES = 8 * (4 * XR_MAX + 8)    # two banks x 64 tagged 2-word slots, error word
_XR = struct.Struct(f"<ii{XR_MAX}QQ")    # struct rtcg::xr {int rank, world; u64 mbox[64], timeout_ns;}
DEFAULT_TIMEOUT_S = 20.0


class PeerTimeout(RuntimeError):
    """A peer never published its accumulator (the kernel gave up after the
    mailbox's timeout and poisoned result/out: all bits set, i.e. NaN for
    floats and -1 / MAX for integers)."""


class PeerMailbox:
    """Every rank's exchange mailbox, mapped into this process, plus the
    device descriptor (``rtcg::xr``) a reduction kernel reads.

    ``ReductionKernel.launch(..., peers=mailbox)`` turns the launch into a
    cross-GPU reduction (``rtcg::exchange``).  Each call takes the next epoch;
    all ranks must issue the same sequence of calls on a mailbox, one stream
    at a time (calls on one mailbox are serialised by the stream).  Not
    capturable in CUDA graphs (the epoch is a launch parameter)."""

    def __init__(self, rank: int, world: int, addresses, *, owned=(), opened=(),
                 timeout_s: float = DEFAULT_TIMEOUT_S) -> None:
        if not 1 <= world <= XR_MAX:
            raise ValueError(f"world size must be in [1, {XR_MAX}], got {world}")
        if len(addresses) != world or not 0 <= rank < world:
            raise ValueError("need one mailbox address per rank")
        self.rank, self.world = rank, world
        self.addresses = tuple(int(a) for a in addresses)
        self._owned, self._opened = list(owned), list(opened)
        self._epoch = 0
        self._lock = threading.Lock()
        if not timeout_s > 0:
            raise ValueError("timeout_s must be positive")
        self.timeout_s = float(timeout_s)
        blob = _XR.pack(rank, world, *self.addresses, *([0] * (XR_MAX - world)),
                        int(self.timeout_s * 1e9))
        self.descriptor = _runtime.mem_alloc(len(blob))
        self._owned.append(self.descriptor)
        host = ctypes.create_string_buffer(blob, len(blob))
        _runtime.memcpy_htod(self.descriptor, ctypes.addressof(host), len(blob), 0)
        _runtime.stream_synchronize(0)

    def next_epoch(self) -> int:
        with self._lock:
            self._epoch += 1
            return self._epoch

    def check(self, stream=None) -> None:
        """Synchronise ``stream`` and raise :class:`PeerTimeout` if an
        exchange on this mailbox timed out waiting for a peer since the last
        check.  The error word is cleared when it is reported, so a later
        healthy exchange checks clean."""
        word = ctypes.c_uint64()
        st = 0 if stream is None else getattr(stream, "handle", stream)
        err = self.addresses[self.rank] + 8 * XR_ERROR
        _runtime.memcpy_dtoh(ctypes.addressof(word), err, 8, st)
        _runtime.stream_synchronize(st)
        if word.value:
            _runtime.memset_async(err, 0, 8, st)
            _runtime.stream_synchronize(st)
            raise PeerTimeout(f"rank {self.rank}: the peer exchange of epoch {word.value} "
                              f"timed out waiting for another rank")

    @staticmethod
    def _new_box() -> int:
        box = _runtime.mem_alloc(MAILBOX_BYTES)   # cuMemAlloc: IPC-exportable
        _runtime.memset_async(box, 0, MAILBOX_BYTES, 0)
        _runtime.stream_synchronize(0)
        return box

    @classmethod
    def create(cls, group=None, timeout_s: float = DEFAULT_TIMEOUT_S) -> "PeerMailbox":
        """Collective over a torch.distributed group (one process per GPU):
        allocate and zero this rank's mailbox, exchange CUDA IPC handles
        (``all_gather_object``, which also orders every zeroing before any
        use) and map the peers' mailboxes."""
        import torch.distributed as dist
        rank, world = dist.get_rank(group), dist.get_world_size(group)
        box = cls._new_box()
        mine = (_runtime.current_device(), _runtime.ipc_get_handle(box))
        everyone = [None] * world
        dist.all_gather_object(everyone, mine, group=group)
        addresses, opened, error = [], [], None
        try:
            for r, (_dev, handle) in enumerate(everyone):
                if r == rank:
                    addresses.append(box)
                else:
                    addr = _runtime.ipc_open_handle(handle)
                    addresses.append(addr)
                    opened.append(addr)
        except Exception as exc:  # noqa: BLE001 - decided collectively below
            error = exc
        # every rank must take the exchange path or none: agree on success
        verdicts = [None] * world
        dist.all_gather_object(verdicts, error is None, group=group)
        if not all(verdicts):
            for addr in opened:
                _runtime.ipc_close_handle(addr)
            _runtime.mem_free(box)
            raise RuntimeError(f"peer mailboxes unavailable on ranks "
                               f"{[r for r, ok in enumerate(verdicts) if not ok]}: {error}")
        mb = cls(rank, world, addresses, owned=[box], opened=opened, timeout_s=timeout_s)
        mb.devices = tuple(d for d, _ in everyone)
        return mb

    @classmethod
    def local_group(cls, world: int, timeout_s: float = DEFAULT_TIMEOUT_S) -> list["PeerMailbox"]:
        """``world`` mailboxes on the current device, one per emulated rank
        (single-process tests of the exchange protocol: launch rank r on its
        own stream with ``peers=group[r]``)."""
        boxes = [cls._new_box() for _ in range(world)]
        group = [cls(r, world, boxes, timeout_s=timeout_s) for r in range(world)]
        group[0]._owned.extend(boxes)
        return group

    def close(self) -> None:
        for addr in self._opened:
            _runtime.ipc_close_handle(addr)
        for addr in self._owned:
            _runtime.mem_free(addr)
        self._opened, self._owned = [], []


# Per-process caches keyed by the identity of the process-group object (the
# entry holds the object, so a destroyed-and-recreated group -- possibly of
# another size, possibly reusing the address -- never matches a stale entry).
_mailboxes: dict = {}
_capable: dict = {}
_mailbox_lock = threading.Lock()


def _group_object(group):
    import torch.distributed as dist
    return group if group is not None else dist.group.WORLD


def peer_mailbox(group=None, stream: int = 0) -> PeerMailbox:
    """The cached mailbox of (group, device, stream); created collectively on
    first use (every rank must reach the first call together)."""
    g = _group_object(group)
    key = (_runtime.current_device(), stream)
    with _mailbox_lock:
        for owner, mb in _mailboxes.get(key, ()):
            if owner is g:
                return mb
    mb = PeerMailbox.create(group)
    with _mailbox_lock:
        _mailboxes.setdefault(key, []).append((g, mb))
    return mb


def peer_plan(bus_ids, visible) -> bool:
    """Whether ranks on the devices ``bus_ids`` (one PCI bus id per rank) can
    exchange through peer memory, seen from one process whose visible devices
    are ``visible`` ({bus id: local ordinal}).  Ranks must sit on distinct
    physical GPUs (bus ids, not ordinals: under per-rank CUDA_VISIBLE_DEVICES
    every rank calls its GPU device 0), and every peer's GPU must be visible
    here -- CUDA IPC cannot map memory of a device this process cannot see."""
    if len(set(bus_ids)) != len(bus_ids):
        return False
    return all(b in visible for b in bus_ids)


def p2p_capable(group=None) -> bool:
    """True when every rank runs on its own device, each rank sees the other
    ranks' devices, and all pairs have peer access (NVLink / NVSwitch on an
    HGX B200).  Decided on PCI bus ids gathered from every rank, and agreed
    collectively.  Ranks that share a device (test setups) take the NCCL path
    under ``collective="auto"``."""
    import torch.distributed as dist
    g = _group_object(group)
    for owner, ok in _capable.get(id(g), ()):
        if owner is g:
            return ok
    world = dist.get_world_size(group)
    mine = _runtime.pci_bus_id(_runtime.current_device())
    bus_ids = [None] * world
    dist.all_gather_object(bus_ids, mine, group=group)
    visible = {_runtime.pci_bus_id(d): d for d in range(_runtime.device_count())}
    ok = peer_plan(bus_ids, visible)
    if ok:
        me = visible[mine]
        ok = all(visible[b] == me or _runtime.can_access_peer(me, visible[b]) for b in bus_ids)
    verdicts = [None] * world          # every rank takes the same path
    dist.all_gather_object(verdicts, ok, group=group)
    ok = all(verdicts)
    _capable.setdefault(id(g), []).append((g, ok))
    return ok


def sharded_reduce(kernel, *args, group=None, return_device: bool = False,
                   collective: str = "auto", overlap_previous: bool = False):
    """Global reduction of a ReductionKernel over sharded arguments.

    ``"p2p"`` -- one launch per GPU: the local two-stage reduction and the
    exchange of accumulators over peer memory in the same kernel
    (:class:`PeerMailbox`), folded in rank order; any ``reduce_expr``.

    NCCL baseline -- the local reduction, then:
    ``"allreduce"`` -- one ncclAllReduce of the 8-byte accumulators when
    :func:`nccl_op` maps ``reduce_expr`` to an exact NCCL op;
    ``"allgather"`` -- all-gather (world x 8 bytes) + ``<name>_combine``
    folding in rank order, valid for any ``reduce_expr``.

    ``"auto"`` -- p2p when every rank has its own peer-accessible GPU, else
    allreduce when exact, else allgather.  Everything runs in stream order on
    torch's current stream; p2p and allgather give identical bits.
    ``overlap_previous`` (p2p only) lets this rank's reduction start while the
    previous kernel on the stream drains -- see ``ReductionKernel.launch``;
    with the exchange inside the kernel this also hides the previous step's
    exchange latency.

    ``return_device=True`` returns the 0-d result without synchronising.  On
    the p2p path a timed-out exchange leaves it poisoned (all bits set: NaN
    / -1 / MAX), never this rank's partial value; call
    ``peer_mailbox(group, stream).check(stream)`` to raise :class:`PeerTimeout`.
    Host results (the default) are checked before they are returned.
    """
    import torch
    import torch.distributed as dist

    local_args, base = _locals(args)
    n_local = next(a.size for a in local_args if isinstance(a, nd.NdArray))
    spec = kernel.spec
    op = nccl_op(spec)
    if collective == "auto":
        collective = "p2p" if p2p_capable(group) else \
            "allreduce" if op is not None else "allgather"
    if collective == "allreduce" and op is None:
        raise ValueError(f"reduce_expr {spec.reduce_expr!r} has no exact NCCL equivalent")
    if collective not in ("allreduce", "allgather", "p2p"):
        raise ValueError(f"unknown collective {collective!r}")
    stream = torch.cuda.current_stream().cuda_stream
    if collective == "p2p":
        mailbox = peer_mailbox(group, stream)
        with _runtime.use_stream(stream):
            if return_device:
                first = next(a for a in local_args if isinstance(a, nd.NdArray))
                out = first.pool.alloc_uninitialized(spec.out_dtype, ())
                kernel.launch(*local_args, n=n_local, base=base, out=out, peers=mailbox,
                              overlap_previous=overlap_previous)
                return out
            # the global value lands in this thread's page-locked slot
            slot = _host_slot()
            kernel.launch(*local_args, n=n_local, base=base, peers=mailbox,
                          overlap_previous=overlap_previous, out_address=slot)
            _runtime.stream_synchronize(stream)
            mailbox.check(stream)
            return spec.out_dtype.np.type(nd.ctype_for(spec.out_dtype).from_address(slot).value)
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
