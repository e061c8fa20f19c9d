"""Generated reductions on the GPU: sums, extrema, inner products and kin.

B200 version of the reference's ``src/reduction.py``.  A reduction is a
signature plus three pieces of C: ``map_expr`` (one value per index ``i``,
default: the first vector's element), ``reduce_expr`` over ``a`` and ``b``
(assumed commutative and associative) and a ``neutral`` literal (the fold's
identity, interpreted by the compiler, never by Python -- ``INT64_MIN`` and
``-INFINITY`` work as written).

Execution is two-stage like the reference (workers -> partials -> ordered
combine), mapped onto one launch of ``templates/reduction.cu``:

1. every CTA (a "worker") folds its index range with a thread-serial fold,
   a warp-shuffle tree and a shared-memory tree into one partial;
2. the last CTA to finish folds the partials in ascending CTA order.

Accumulation uses the out dtype, except float32 accumulates in float64 and
rounds once (``src/reduction.py:18-20,53-54``).  A fixed (n, variant) gives a
bitwise-identical result on every run: no float atomics, fixed tree order.

Both constructor forms are accepted: the reference's
``ReductionKernel(spec, name, variant, ...)`` and PyCUDA's
``ReductionKernel(dtype_out, neutral, reduce_expr, map_expr=None,
arguments=None, name=...)``.  Calls return a numpy scalar of the out dtype
(reference behaviour); ``return_device=True`` (the default in the PyCUDA form)
returns a 0-d GPUArray instead, without a host synchronisation.
"""

from __future__ import annotations

import ctypes
import re
import threading
from time import perf_counter as _perf_counter
from dataclasses import dataclass
from threading import get_ident as _get_ident

import numpy as np

from . import _runtime
from . import _codegen as cg
from . import jit
from . import ndarray as nd
from .driver import HostArg as _HostArg, In as _In, InOut as _InOut, Out as _Out
from .elementwise import (_CHUNK_TOKEN, _ERRORS, MAX_CHUNKS, ArityMismatch, DtypeMismatch,
                          KernelSignature, ParseError, VariantParams, _check_name, _LazyEntry,
                          _preamble_text, parse_signature)
from .ndarray import Dtype

_HOST_CLASSES = frozenset({_HostArg, _In, _Out, _InOut})

__all__ = [
    "NonScalarResult", "ReductionSpec", "ReductionKernel", "make_reduction",
    "generate_reduction_source", "sum_kernel", "max_kernel", "min_kernel",
    "dot_kernel",
]


class NonScalarResult(Exception):
    """map/reduce expressions cannot produce one value per element/pair."""


_AB = re.compile(r"\b([ab])\b")
_DRIVER_NAMES = ("acc", "out", "partials", "result")


def _accumulator_dtype(out_dtype: Dtype) -> Dtype:
    return nd.float64 if out_dtype == nd.float32 else out_dtype


@dataclass(frozen=True)
class ReductionSpec:
    """What to fold (``src/reduction.py:57-95``)."""

    signature: KernelSignature
    out_dtype: Dtype
    neutral: str
    reduce_expr: str
    map_expr: str | None = None

    def __post_init__(self) -> None:
        if isinstance(self.signature, str):
            object.__setattr__(self, "signature", parse_signature(self.signature))
        object.__setattr__(self, "out_dtype", nd.dtype_of(self.out_dtype))
        for p in self.signature.params:
            if p.name in _DRIVER_NAMES:
                raise ParseError(f"parameter name {p.name!r} collides with reduction "
                                 f"driver identifiers")
        if {m.group(1) for m in _AB.finditer(self.reduce_expr)} != {"a", "b"}:
            raise NonScalarResult("reduce_expr must combine both operands a and b")
        if not self.mapped.strip():
            raise NonScalarResult("map_expr must produce a value per element")

    @property
    def mapped(self) -> str:
        return self.map_expr if self.map_expr is not None else \
            f"{self.signature.vectors[0].name}[i]"

    @property
    def acc_dtype(self) -> Dtype:
        return _accumulator_dtype(self.out_dtype)


def generate_reduction_source(spec: ReductionSpec, name: str,
                              variant: VariantParams, preamble: str = "",
                              entries: str = "all") -> str:
    """CUDA source with ``<name>`` (vector path, when legal), ``<name>_g``
    (general) and ``<name>_combine`` (ordered fold of partials).
    ``entries``: "all", "vector" (``<name>`` + ``<name>_combine``) or
    "general" (``<name>_g`` only)."""
    if entries not in ("all", "vector", "general"):
        raise ValueError(f"entries must be 'all', 'vector' or 'general', got {entries!r}")
    _check_name(name)
    sig = spec.signature
    access = cg.analyze(spec.mapped, [p.name for p in sig.vectors])
    if access is not None and any(a.written for a in access.values()):
        access = None  # a map expression with side effects stays general
    width = cg.chunk_width(sig, access) if access is not None else 0
    b = cg.parts(sig, access, width, variant.cache)
    if variant.cache == "tma" and b["vector"]:
        b.update(cg.tma_parts(sig, access, width))
        b["vector"] = False  # the TMA entry point takes the vector path's name
    if entries == "general":
        b.update(vector=False, tma=False)
    b.update(general=entries != "vector", combine=entries != "general")
    b["map_tparams"] = b.pop("op_tparams")
    b["map_params"] = b.pop("op_params")
    dynamic = bool(variant.chunk) and b["vector"]
    b.update(name=name, unroll=variant.unroll, block=variant.block,
             dynamic=dynamic, static=not dynamic, chunk=variant.chunk, max_chunks=MAX_CHUNKS,
             prefetch=variant.prefetch, no_prefetch=not variant.prefetch,
             preamble=_preamble_text(preamble), chunking=_CHUNK_TOKEN[variant.chunking],
             acc_t=spec.acc_dtype.cname, out_t=spec.out_dtype.cname,
             neutral=spec.neutral, reduce_expr=spec.reduce_expr, map_expr=spec.mapped)
    return cg.render("reduction.cu", b)


_SERIAL = 1 << 63
_HOST_FLAG = 1 << 62       # seq bit: out is a host slot, write its completion word
_SPIN_S = 200e-6           # a synchronous call spins this long before blocking
_host_slots = threading.local()


class _HostSlot:
    """A 64-byte page-locked buffer, returned to the driver when its thread's
    local storage goes away: the value at +0, the completion word the last
    CTA stores after it at +32."""
    __slots__ = ("address", "done")

    def __init__(self) -> None:
        self.address = _runtime.host_alloc(64)
        self.done = ctypes.c_uint32.from_address(self.address + 32)

    def __del__(self):
        try:
            _runtime.host_free(self.address)
        except Exception:  # pragma: no cover - interpreter shutdown
            pass


def _slot_object() -> _HostSlot:
    slot = getattr(_host_slots, "slot", None)
    if slot is None:
        slot = _host_slots.slot = _HostSlot()
    return slot


def _host_slot() -> int:
    """This thread's page-locked result slot.  A synchronous call
    (``kernel(x)`` returning a host scalar) passes it as the kernel's ``out``:
    with unified addressing the last CTA stores the value straight into host
    memory, so the call is launch + wait, without a device-to-host copy (the
    call returns before the thread's next one, so one slot per thread serves
    every kernel and device)."""
    return _slot_object().address


def _await_slot(slot: _HostSlot, stream) -> None:
    """Wait for a launch that writes ``slot``'s completion word: spin on the
    word (the last CTA stores it after the value, system-scope release) for
    up to ``_SPIN_S``, then block on the stream -- which also reports a
    failed launch.  Spinning saves the stream synchronisation's wake-up
    (2^16 synchronous sum / max / dot: 14.4-15.0 -> 12.6-13.4 us per call,
    tools/probe_sync_spin.py, profiles/r02_probe_small_n_spin.json)."""
    done = slot.done
    if done.value:
        return
    deadline = _perf_counter() + _SPIN_S
    while True:
        for _ in range(64):
            if done.value:
                return
        if _perf_counter() > deadline:
            _runtime.stream_synchronize(stream)
            return


class _Scratch:
    """Per-device partials / result / out / ticket buffers of one kernel.

    Three partials regions of ``capacity`` accumulators: two alternate
    between overlapped launches (so a launch's CTAs may publish while the
    previous launch still folds the other region) and one serves serial
    launches; the 64-byte block holds result (+0), out (+16), the three
    regions' tickets (+32) and the two overlapped regions' release counters
    (+44) -- see ``rtcg::finish``.  ``seq`` numbers the overlapped launches."""

    def __init__(self, acc_size: int, out_size: int, stream: int = 0) -> None:
        self.capacity = 0
        self.partials = 0
        self.seq = 0
        self.host_flagged = False    # the last launch stores a host slot's completion word
        self.acc_size, self.out_size = acc_size, out_size
        self.stream = stream
        self.result = _runtime.mem_alloc(64)
        self.out = self.result + 16
        self.ticket = self.result + 32
        # zeroed on the stream the scratch is keyed by, so the first launch
        # there is ordered after the ticket reset (cuMemAlloc is not zeroed)
        _runtime.memset_async(self.result, 0, 64, stream)

    def ensure(self, count: int) -> None:
        if count > self.capacity:
            cap = max(count, 2048)
            if self.partials:
                # stream-ordered retirement: the old buffer is released after
                # the launches already queued on this scratch's stream (no
                # device-wide synchronisation, which would block on peers'
                # exchange kernels spinning on the same GPU)
                _runtime.mem_free_async(self.partials, self.stream)
            self.partials = _runtime.mem_alloc_async(3 * cap * self.acc_size, self.stream)
            self.capacity = cap

    def slot(self, overlapped: bool):
        """(partials region, seq parameter) of the next launch: an overlapped
        launch takes region ``seq & 1``, a serial one region 2.  The caller
        commits ``seq`` (``self.seq += 1``) once an overlapped launch was
        issued -- a number handed out but never launched would leave its
        region unreleased."""
        if not overlapped:
            return self.partials + 2 * self.capacity * self.acc_size, _SERIAL
        q = self.seq
        return self.partials + (q & 1) * self.capacity * self.acc_size, q


def _is_dtype_like(obj) -> bool:
    if isinstance(obj, Dtype):
        return True
    if isinstance(obj, (ReductionSpec, str)):
        return False
    try:
        np.dtype(obj)
        return True
    except TypeError:
        return False


class ReductionKernel:
    """A compiled reduction; ``kernel(args..., n=count)`` returns the result.

    Construction: ``ReductionKernel(spec, name="reduce", variant=None, *,
    config, cache, debug)`` (reference) or ``ReductionKernel(dtype_out,
    neutral, reduce_expr, map_expr=None, arguments=None, name=..., ...)``
    (PyCUDA; ``arguments`` is the signature text).
    """

    def __init__(self, *args, **kwargs) -> None:
        if args and _is_dtype_like(args[0]) or "dtype_out" in kwargs:
            self._init_pycuda(*args, **kwargs)
        else:
            self._init_reference(*args, **kwargs)

    def _init_pycuda(self, dtype_out=None, neutral=None, reduce_expr=None, map_expr=None,
                     arguments=None, name="reduce_kernel", variant=None, *,
                     config=None, cache=None, debug=False, return_device=True, preamble="",
                     **_ignored):
        if arguments is None:
            raise ParseError("ReductionKernel needs an 'arguments' signature")
        spec = ReductionSpec(arguments, nd.dtype_of(dtype_out), str(neutral), reduce_expr,
                             map_expr)
        self._init_reference(spec, name, variant, config=config, cache=cache, debug=debug,
                             preamble=preamble)
        self.return_device = return_device

    def _init_reference(self, spec: ReductionSpec, name: str = "reduce",
                        variant: VariantParams | None = None, *,
                        config: jit.ToolchainConfig | None = None,
                        cache: jit.CacheStore | None = None, debug: bool = False,
                        preamble: str = "") -> None:
        self.spec = spec
        self.preamble = preamble
        self.name = name
        self.variant = (variant or VariantParams()).resolved()
        self.return_device = False
        sig = spec.signature
        access = cg.analyze(spec.mapped, [p.name for p in sig.vectors])
        if access is not None and any(a.written for a in access.values()):
            access = None
        self.access = access
        self.width = cg.chunk_width(sig, access) if access is not None else 0
        self._plans: dict = {}
        if self.access and self.width:
            # vector (or TMA) entry + combine now; the general entry point
            # (misaligned / aliased arguments) on first need
            self.source = generate_reduction_source(spec, name, self.variant, preamble,
                                                    entries="vector")
            self.module = jit.compile(self.source, config, cache)
            self.vectorized = jit.get_kernel(self.module, name)
            self.generic = _LazyEntry(
                f"{name}_g", lambda: jit.compile(
                    generate_reduction_source(spec, name, self.variant, preamble,
                                              entries="general"), config, cache),
                self._plans.clear)
        else:
            self.source = generate_reduction_source(spec, name, self.variant, preamble)
            self.module = jit.compile(self.source, config, cache)
            self.vectorized = None
            self.generic = jit.get_kernel(self.module, f"{name}_g")
        self.smem = 0
        self._tma_tile = 0
        if self.vectorized is not None and self.variant.cache == "tma":
            if self.variant.block < 64:
                raise ValueError("the TMA path needs block >= 64 (a producer warp + consumers)")
            tp = cg.tma_parts(sig, access, self.width)
            self.smem, self._tma_tile = tp["tma_smem"], tp["tile"]
        self.combine = jit.get_kernel(self.module, f"{name}_combine")
        self._acc_ctype = nd.ctype_for(spec.acc_dtype)
        self._binder = cg.Binder(sig, extra=7)
        self._waves = 1 if self.variant.waves is None else self.variant.waves
        # dynamic chunks: the vector entry stores up to MAX_CHUNKS partials
        # (rtcg::chunk_plan grows the chunks to fit), whatever its grid
        self._min_parts = MAX_CHUNKS if self.variant.chunk and self.vectorized is not None \
            and not self.smem else 0
        self._scratch: dict[int, _Scratch] = {}
        self._lock = threading.Lock()
        self.launches = 0
        if debug:
            self._check_neutral()

    def __repr__(self) -> str:
        return (f"<ReductionKernel {self.name} [{self.spec.signature.render()}]"
                f" -> {self.spec.out_dtype.name}>")

    # -- plumbing --

    def scratch(self, device: int, stream: int | None = None) -> _Scratch:
        """Partials / result / ticket buffers for (device, stream, calling
        thread): launches on different streams never share a ticket, and two
        threads sharing a kernel object and a stream never read each other's
        result (the reference's kernels are shareable between threads,
        SPEC:331)."""
        key = (device, _runtime.current_stream() if stream is None else stream, _get_ident())
        with self._lock:
            s = self._scratch.get(key)
            if s is None:
                s = self._scratch[key] = _Scratch(self.spec.acc_dtype.size,
                                                 self.spec.out_dtype.size, key[1])
            return s

    def _pick(self, vectors, n):
        """(handle, elements per thread-step, dynamic shared memory)."""
        if self.vectorized is not None:
            used = [(addr, local, p.dtype.size, self.access[p.name])
                    for p, addr, local in vectors if self.access[p.name].used]
            if cg.vector_path_ok(used, n):
                if self.smem:
                    return self.vectorized, max(1, self._tma_tile // self.variant.block), \
                        self.smem
                return self.vectorized, self.variant.unroll * self.width, 0
        return self.generic, self.variant.unroll, 0

    def _read(self, address: int, dtype: Dtype, stream=None):
        """Read one value on ``stream`` (default: the current stream) -- the
        stream the producing kernel ran on, so the copy is ordered after it."""
        st = None if stream is None else getattr(stream, "handle", stream)
        box = nd.ctype_for(dtype)()
        _runtime.memcpy_dtoh(ctypes.addressof(box), address, dtype.size, st)
        _runtime.stream_synchronize(st)
        return dtype.np.type(box.value)

    def _launch_combine(self, partials: int, count: int, result: int, out: int,
                        stream=None) -> None:
        vals = [ctypes.c_uint64(partials), ctypes.c_uint64(result), ctypes.c_uint64(out),
                ctypes.c_long(0), ctypes.c_long(count)]
        _runtime.launch(self.combine.function(), 1, 32, cg.pack(vals), 0, stream)

    def _check_neutral(self) -> None:
        """fold([v]) must give v back for exactly representable samples
        (``src/reduction.py:218-234``); runs the compiled combine on device."""
        kind = self.spec.acc_dtype.kind
        samples = {"f": [0.0, 1.5, -2.25, 7.0], "u": [0, 1, 7, 200]}.get(kind, [0, 1, -3, 99])
        dev = _runtime.current_device()
        s = self.scratch(dev)
        s.ensure(1)
        for value in samples:
            box = self._acc_ctype(value)
            _runtime.memcpy_htod(s.partials, ctypes.addressof(box), self.spec.acc_dtype.size)
            self._launch_combine(s.partials, 1, s.result, s.out)
            folded = self._read(s.result, self.spec.acc_dtype)
            if folded != self.spec.acc_dtype.np.type(value):
                raise ValueError(
                    f"neutral {self.spec.neutral!r} is not an identity for "
                    f"{self.spec.reduce_expr!r}: fold([{value!r}]) gave {folded!r}")

    def _plan(self, dev: int):
        """Native launch plan on device *dev* (``csrc/fastlaunch.cpp``): the
        binder, :meth:`_pick` and the grid policy in one C call."""
        plan = self._plans.get(dev)
        if plan is not None:
            return plan
        sms = cg.sm_count(dev)
        block = self.variant.block
        gen = None              # not compiled yet: calls that need it take the Python path
        if not isinstance(self.generic, _LazyEntry) or self.generic.ready:
            gen_fn = self.generic.function(dev)
            gen = (gen_fn, self.variant.unroll,
                   sms * max(1, _runtime.occupancy(gen_fn, block, 0)), self._waves, 0)
        vec = None
        if self.vectorized is not None:
            fn = self.vectorized.function(dev)
            if self.smem:
                _runtime.set_max_dynamic_smem(fn, self.smem)
                per = max(1, self._tma_tile // block)
            else:
                per = self.variant.unroll * self.width
            vec = (fn, per, sms * max(1, _runtime.occupancy(fn, block, self.smem)), self._waves,
                   self.smem, self._min_parts)
        params = []
        for p in self.spec.signature.params:
            acc = self.access[p.name] if self.access is not None and p.is_vector else None
            params.append((p.is_vector, p.dtype, p.dtype.size, p.dtype.kind,
                           bool(acc and acc.used), bool(acc and acc.written)))
        plan = self._plans[dev] = _runtime.fastlaunch().Plan(
            params, nd.NdArray, block, self.variant.workers or 0, gen, vec, 7)
        return plan

    def launch(self, *args, n: int | None = None, base: int = 0, stream=None,
               out: nd.NdArray | None = None, peers=None, overlap_previous: bool = False,
               out_address: int = 0, host_flag: bool = False):
        """Asynchronous stage 1+2.  Returns the scratch (result address holds
        the accumulator, ``out`` -- or the scratch out slot -- the out-dtype
        value).  Used by ``__call__`` and by the multi-GPU driver.

        ``peers`` (a :class:`~paper_0911_3456_b200.parallel.PeerMailbox`)
        makes the launch a cross-GPU reduction: the kernel's last CTA
        exchanges the device accumulator with every rank over peer memory and
        result/out receive the global value (every rank must make the same
        call; an empty local span still takes part).

        ``overlap_previous=True`` launches with programmatic stream
        serialization: this reduction's CTAs may start streaming their inputs
        while the previous kernel on the stream (typically the previous
        reduction of a loop) is still folding, and wait for it only before
        touching the shared scratch (``griddepcontrol.wait`` in
        ``rtcg::finish``).  The caller asserts that the previous kernel on
        the stream writes nothing this call reads (its inputs).  With
        ``peers``, one GPU per rank is assumed (ranks emulated on one GPU
        share its SMs with each other's waiting grids).  Measured on B200:
        back-to-back dot f32 at 2^24 / 2^26 / 2^28 +19 / +5 / +2 %.

        ``out_address`` (internal) overrides the out slot with a raw address
        -- the page-locked host slot of a synchronous call; ``host_flag``
        (internal) makes the kernel store the slot's completion word after
        the value.  ``scratch.host_flagged`` tells whether this launch will
        (an empty span folds through the combine entry, which does not)."""
        if stream is not None:
            stream = getattr(stream, "handle", stream)
        # the completion word lives in a host slot only (out + 32)
        host_flag = bool(host_flag and out_address and out is None)
        if peers is None:
            tls = _runtime._tls
            dev = getattr(tls, "device", None)
            if dev is None:
                dev = _runtime.current_device()
            st = getattr(tls, "stream", 0) if stream is None else stream or 0
            s = self._scratch.get((dev, st, _get_ident())) or self.scratch(dev, st)
            plan = self._plans.get(dev) or self._plan(dev)
            rotate = overlap_previous and not _runtime.stream_is_capturing(st)
            partials, seq = s.slot(rotate)
            if host_flag:
                seq |= _HOST_FLAG
            oaddr = out.address if out is not None else out_address or s.out
            got = plan.launch(args, n, base, st or 0, s.capacity,
                              (partials, s.result, oaddr,
                               s.ticket, 0, 0, seq), 1 if overlap_previous else 0)
            if got:          # None: the Python binder below; 0: empty span
                if got < 0:
                    _runtime._check(-got, "launch")
                if rotate:
                    s.seq += 1
                self.launches += 1
                s.host_flagged = host_flag
                return s
        # the Python binder: empty spans, peer exchanges, and every call the
        # native plan declined (it raises the reference's exceptions)
        if n is not None and n < 0:
            raise nd.ShapeMismatch(f"n must be non-negative, got {n}")
        vals, ptrs, vectors, n = self._binder.bind(args, n, base, self.name, _ERRORS)
        dev = _runtime.current_device()
        s = self.scratch(dev, stream)
        out_addr = out.address if out is not None else out_address or s.out
        b = self._binder
        if peers is not None:
            # resolve (and load) every entry point before the first exchange
            # launch: nothing may wait on the device between ranks' launches
            for h in (self.generic, self.vectorized, self.combine):
                if h is not None:
                    h.function(dev)
            vals[b.count + 6], vals[b.count + 7] = peers.descriptor, peers.next_epoch()
        else:
            vals[b.count + 6] = vals[b.count + 7] = 0
        if n == 0 and peers is None:
            s.ensure(1)
            self._launch_combine(s.partials, 0, s.result, out_addr, stream)
            s.host_flagged = False
            return s
        if n == 0:
            handle, grid, smem = self.generic, 1, 0
            fn = handle.function(dev)
        else:
            handle, per_thread, smem = self._pick(vectors, n)
            fn = handle.function(dev)
            if smem:
                _runtime.set_max_dynamic_smem(fn, smem)
            grid = cg.grid_for(fn, dev, self.variant.block, self.variant.workers, n, per_thread,
                               self._waves, smem)
        s.ensure(max(grid, self._min_parts if handle is self.vectorized else 0))
        rotate = overlap_previous and not _runtime.stream_is_capturing(stream)
        partials, seq = s.slot(rotate)
        if host_flag:
            seq |= _HOST_FLAG
        b.set_range(vals, base, base + n)
        vals[b.count + 2] = partials
        vals[b.count + 3] = s.result
        vals[b.count + 4] = out_addr
        vals[b.count + 5] = s.ticket
        vals[b.count + 8] = seq
        if overlap_previous:
            _runtime.launch_overlapped(fn, grid, self.variant.block, ptrs, smem, stream)
        else:
            _runtime.launch(fn, grid, self.variant.block, ptrs, smem, stream)
        if rotate:
            s.seq += 1
        self.launches += 1
        s.host_flagged = host_flag
        return s

    def launch_config(self, *args, n: int | None = None) -> dict:
        _, _, vectors, n = self._binder.bind(args, n, 0, self.name, _ERRORS)
        handle, per_thread, smem = self._pick(vectors, n)
        dev = _runtime.current_device()
        fn = handle.function(dev)
        if smem:
            _runtime.set_max_dynamic_smem(fn, smem)
        grid = cg.grid_for(fn, dev, self.variant.block, self.variant.workers, max(n, 1),
                           per_thread, self._waves, smem)
        return {"entry": handle.name, "grid": grid, "block": self.variant.block, "n": n,
                "smem": smem}

    HOST_CHUNK_BYTES = 64 << 20

    def _call_host(self, args, n, base: int, want_device: bool, chunk: int | None = None):
        """Reduction over host arrays (``driver.In``): chunk j's uploads and
        stage-1+2 reduction run on one of two streams (uploads overlap the
        previous chunk's kernel); each chunk's accumulator lands in slot j of
        a device array, and the compiled combine folds the slots in chunk
        order -- the reference's ordered fold of worker partials with chunks
        as workers (src/reduction.py:211-216)."""
        from .driver import HostArg
        from .elementwise import _host_streams
        params = self.spec.signature.params
        if len(args) != len(params):
            raise ArityMismatch(f"kernel {self.name} takes {len(params)} arguments, "
                                f"got {len(args)}")
        host_bytes = 0
        for p, a in zip(params, args):
            if isinstance(a, HostArg):
                if not p.is_vector:
                    raise DtypeMismatch(p.name, "a host array passed for a scalar")
                if a.copy_out:
                    raise ValueError("reductions take host inputs only (driver.In)")
                if a.array.dtype != p.dtype.np:
                    raise DtypeMismatch(p.name, f"expected dtype {p.dtype.name}, "
                                                f"got {a.array.dtype}")
                host_bytes += p.dtype.size
        first = next((a for p, a in zip(params, args) if p.is_vector), None)
        total = n if n is not None else first.size
        for p, a in zip(params, args):
            if p.is_vector and a.size < total:
                raise nd.ShapeMismatch(f"vector {p.name!r} holds {a.size} elements, "
                                       f"kernel span is {total}")
        dev = _runtime.current_device()
        pool = nd.default_pool(dev)
        step = chunk or max(1 << 16, self.HOST_CHUNK_BYTES // max(1, host_bytes) // 256 * 256)
        step = max(1, min(step, total)) if total > 0 else 1
        count = -(-total // step) if total > 0 else 0
        accs = pool.alloc_uninitialized(self.spec.acc_dtype, (max(1, count),))
        streams = _host_streams(dev)
        staging = [[pool.alloc_uninitialized(p.dtype, (step,)) if isinstance(a, HostArg)
                    else None for p, a in zip(params, args)] for _ in streams]
        acc_size = self.spec.acc_dtype.size
        _runtime.order_after_current(streams)   # see ElementwiseKernel._call_host
        done = False
        try:
            for j in range(count):
                lo, hi = j * step, min(total, (j + 1) * step)
                k = j % len(streams)
                st = streams[k]
                call = []
                with _runtime.use_stream(st.handle):
                    for p, a, buf in zip(params, args, staging[k]):
                        if isinstance(a, HostArg):
                            _runtime.copy_htod(buf.address, a.array[lo:hi].ctypes.data,
                                               (hi - lo) * p.dtype.size)
                            call.append(buf)
                        elif p.is_vector:
                            call.append(a[lo:hi])
                        else:
                            call.append(a)
                    s = self.launch(*call, n=hi - lo, base=base + lo)
                    _runtime.memcpy_dtod(accs.address + j * acc_size, s.result, acc_size)
            for st in streams:
                st.synchronize()
            done = True
            s = self.scratch(dev)
            s.ensure(1)
            if want_device:
                out = pool.alloc_uninitialized(self.spec.out_dtype, ())
                self._launch_combine(accs.address, count, s.result, out.address)
                return out
            slot = _host_slot()
            self._launch_combine(accs.address, count, s.result, slot)
            _runtime.stream_synchronize()
            dt = self.spec.out_dtype
            return dt.np.type(nd.ctype_for(dt).from_address(slot).value)
        finally:
            if not done:       # drain in-flight copies before the staging is reused
                for st in streams:
                    st.synchronize()
            accs.free()
            for stage in staging:
                for buf in stage:
                    if buf is not None:
                        buf.free()

    def __call__(self, *args, n: int | None = None, stream=None,
                 return_device: bool | None = None, base: int = 0):
        want_device = self.return_device if return_device is None else return_device
        for a in args:                       # host arrays: the streamed path
            if a.__class__ in _HOST_CLASSES:
                return self._call_host(args, n, base, want_device)
        if want_device:
            first = next(a for a, p in zip(args, self.spec.signature.params) if p.is_vector)
            out = first.pool.alloc_uninitialized(self.spec.out_dtype, ())
            self.launch(*args, n=n, base=base, stream=stream, out=out)
            return out
        slot = _slot_object()
        st = None if stream is None else getattr(stream, "handle", stream)
        slot.done.value = 0
        s = self.launch(*args, n=n, base=base, stream=stream, out_address=slot.address,
                        host_flag=True)
        if s.host_flagged:
            _await_slot(slot, st)
        else:
            _runtime.stream_synchronize(st)
        dt = self.spec.out_dtype
        return dt.np.type(nd.ctype_for(dt).from_address(slot.address).value)


def make_reduction(signature, out_dtype, neutral: str, reduce_expr: str,
                   map_expr: str | None = None, name: str = "reduce",
                   variant: VariantParams | None = None, **kwargs) -> ReductionKernel:
    """Reduction from the raw spec pieces (``src/reduction.py:261-268``)."""
    spec = ReductionSpec(signature, nd.dtype_of(out_dtype), neutral, reduce_expr, map_expr)
    return ReductionKernel(spec, name, variant, **kwargs)


# --- stock reductions (src/reduction.py:273-312) -----------------------------------------------


def _lowest(d: Dtype) -> str:
    return {"i": f"INT{d.size * 8}_MIN", "u": "0", "f": "-INFINITY"}[d.kind]


def _highest(d: Dtype) -> str:
    return {"i": f"INT{d.size * 8}_MAX", "u": f"UINT{d.size * 8}_MAX", "f": "INFINITY"}[d.kind]


def sum_kernel(dtype, variant: VariantParams | None = None, **kwargs) -> ReductionKernel:
    d = nd.dtype_of(dtype)
    return make_reduction(f"{d.cname} *x", d, "0", "a + b", name="sum_k",
                          variant=variant, **kwargs)


def max_kernel(dtype, variant: VariantParams | None = None, **kwargs) -> ReductionKernel:
    d = nd.dtype_of(dtype)
    return make_reduction(f"{d.cname} *x", d, _lowest(d), "a > b ? a : b", name="max_k",
                          variant=variant, **kwargs)


def min_kernel(dtype, variant: VariantParams | None = None, **kwargs) -> ReductionKernel:
    d = nd.dtype_of(dtype)
    return make_reduction(f"{d.cname} *x", d, _highest(d), "a < b ? a : b", name="min_k",
                          variant=variant, **kwargs)


def dot_kernel(dtype, variant: VariantParams | None = None, **kwargs) -> ReductionKernel:
    """Inner product of two same-dtype vectors."""
    d = nd.dtype_of(dtype)
    return make_reduction(f"{d.cname} *x, {d.cname} *y", d, "0", "a + b",
                          map_expr="x[i] * y[i]", name="dot_k", variant=variant, **kwargs)
