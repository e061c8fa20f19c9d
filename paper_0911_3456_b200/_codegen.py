"""Shared CUDA code generation and launch plumbing for the kernel templates.

Both generators (elementwise, reduction) turn a parsed signature plus user C
text into the placeholder bindings of a template under ``templates/``.  The
interesting decision made here is whether the *vector path* may be emitted:

* every occurrence of every vector parameter in the user text must be the
  exact element reference ``name[i]`` (whitespace allowed), not address-taken
  and not a member of something else;
* then each vector is classified as read, written, or both -- the register
  chunk is loaded only when read, stored only when written, and a vector that
  is written conditionally (or only sometimes) is loaded first so untouched
  elements are stored back unchanged.

The same analysis generalises the reference's ``\\bi\\b`` rewriting trick
(``src/elementwise.py:185,195-201``): instead of rewriting text, the user's
statement becomes the body of a template function instantiated once with
pointers and once with register ``rtcg::lane`` wrappers.
"""

from __future__ import annotations

import ctypes
import re
import struct
import threading
from dataclasses import dataclass
from functools import lru_cache
from pathlib import Path

from . import _runtime
from . import csyntax as cs

TEMPLATES = Path(__file__).resolve().parent / "templates"

_WIDE = {"i": ("long", ctypes.c_int64), "u": ("unsigned long", ctypes.c_uint64),
         "f": ("double", ctypes.c_double)}

CACHE_POLICIES = {
    # name: (load policy for read-only vectors, load policy for read-write
    #        vectors, store policy) -- see rtcg::ld16 / rtcg::st16
    "default": (1, 0, 0),
    "streaming": (2, 2, 1),
    "no-l1": (3, 0, 2),
    # read-only loads ask L2 for the whole 256-byte block (ld...L2::256B)
    "l2-256": (4, 0, 0),
    "l2-256-no-l1": (5, 0, 2),
    # inputs staged through shared memory by TMA bulk copies (the "TMA path"
    # of templates/reduction.cu and templates/elementwise.cu); the policies
    # apply to the pointer-path head/tail and to elementwise stores
    "tma": (1, 0, 0),
}
TMA_STAGES = 4
TMA_STAGE_BYTES = 32 * 1024
TMA_HEADER = 128


TMA_SMEM_BUDGET = 200 * 1024   # of the 227 KB a CTA may opt in to


def _tma_layout(sig, access, width: int, block: int | None, staged: str):
    """(staged vectors, tile elements, stages) or None when no ring of >= 2
    stages fits the shared-memory budget."""
    pick = (lambda a: a.used) if staged == "used" else (lambda a: a.read)
    used = [p for p in sig.vectors if pick(access[p.name])]
    per_elem = sum(p.dtype.size for p in used)
    if not used:
        return None
    if block is None:
        tile = max(width * 16, (TMA_STAGE_BYTES // per_elem) // width * width)
    else:
        consumers = block - 32
        per_thread = max(1, TMA_STAGE_BYTES // (consumers * width * per_elem))
        tile = per_thread * consumers * width
    stages = min(TMA_STAGES, (TMA_SMEM_BUDGET - TMA_HEADER) // (tile * per_elem))
    if stages < 2:
        return None
    return used, tile, stages


def tma_parts(sig, access, width: int, block: int | None = None,
              staged: str = "used") -> dict:
    """Bindings of a template's TMA path: shared-memory rings (one per staged
    vector), the producer's bulk copies, the consumers' shared-memory chunk
    loads and the dynamic shared-memory size.

    Reductions stage every used vector (``staged="used"``) in 32 KB-ish tiles.
    Elementwise kernels stage the vectors they *read* (``staged="read"``;
    written vectors are stored straight from registers) and size the tile so
    every consumer thread (all warps but the producer) owns the same number of
    16-byte chunks -- an uneven split idles consumers on compute-heavy
    statements.  The ring has up to 4 stages, fewer when a tile of wide
    vectors is large (at least 2, see :func:`tma_eligible`)."""
    used, tile, stages = _tma_layout(sig, access, width, block, staged)
    per_elem = sum(p.dtype.size for p in used)
    rings, bulks, loads = [], [], []
    offset = 0
    for p in used:
        c = p.dtype.cname
        rings.append(f"    {c} *rtcg_r_{p.name} = reinterpret_cast<{c} *>(rtcg_ring + {offset});")
        bulks.append(f"                    rtcg::tma::bulk_load(rtcg_r_{p.name} + s * TE, "
                     f"rtcg_p_{p.name} + t * TE, (unsigned)(TE * sizeof({c})), rtcg_full + s);")
        loads.append(f"                    rtcg::tma::load_smem(rtcg_v_{p.name}[u], "
                     f"rtcg_r_{p.name} + s * TE, c);")
        offset += stages * tile * p.dtype.size
    return {"tma": True, "stages": stages, "tile": tile, "tile_bytes": tile * per_elem,
            "ring_decls": "\n".join(rings), "bulk_loads": "\n".join(bulks),
            "smem_loads": "\n".join(loads), "tma_smem": TMA_HEADER + offset}


def tma_eligible(sig, access, width: int, block: int | None = None,
                 staged: str = "read") -> bool:
    """A TMA path needs the vector path, something to stage and a ring of at
    least two stages within the shared-memory budget."""
    if access is None or width <= 0:
        return False
    return _tma_layout(sig, access, width, block, staged) is not None

def async_eligible(sig, access, width: int) -> bool:
    """A per-thread cp.async ring needs the vector path and a vector to read."""
    return access is not None and width > 0 and any(access[p.name].read for p in sig.vectors)


def async_parts(sig, access, width: int, stages: int, unroll: int, block: int) -> dict:
    """Bindings of the elementwise vector path's cp.async ring (``stages``
    steps of ``unroll`` chunks per read vector, ``block`` threads): ring
    pointers into dynamic shared memory, the copy issue and the register
    fetch per read vector, and the dynamic shared-memory size."""
    rings, issue, issue_ahead, fetch = [], [], [], []
    offset = 0
    for p in sig.vectors:
        if not access[p.name].read:
            continue
        c = p.dtype.cname
        q = width * p.dtype.size // 16          # 16-byte words per chunk of this vector
        rings.append(f"    int4 *rtcg_a_{p.name} = reinterpret_cast<int4 *>(rtcg_smem + {offset});")
        slot = f"rtcg_a_{p.name} + ({{s}} * U + u) * {q * block}"
        issue.append(f"                rtcg::async::issue<{c}, E, {block}>("
                     f"{slot.format(s='s')}, rtcg_p_{p.name}, cu);")
        issue_ahead.append(f"                    rtcg::async::issue<{c}, E, {block}>("
                           f"{slot.format(s='sa')}, rtcg_p_{p.name}, cu);")
        fetch.append(f"                rtcg::async::fetch<{c}, E, {block}>(rtcg_v_{p.name}[u], "
                     f"{slot.format(s='s')});")
        offset += stages * unroll * q * 16 * block
    return {"stages": stages, "async_ring_decls": "\n".join(rings),
            "async_issue": "\n".join(issue), "async_issue_ahead": "\n".join(issue_ahead),
            "async_fetch": "\n".join(fetch), "async_smem": offset}


_CONTROL = re.compile(r"\b(?:if|else|for|while|do|switch|case|goto|return|break|continue)\b|[{}]")


@lru_cache(maxsize=None)
def template(name: str) -> str:
    return (TEMPLATES / name).read_text()


@dataclass(frozen=True)
class Access:
    read: bool
    written: bool

    @property
    def used(self) -> bool:
        return self.read or self.written


def _occurrences(name: str, text: str):
    """All uses of identifier *name* that are not member accesses."""
    pat = re.compile(r"(?<![\w.])(?<!->)" + re.escape(name) + r"\b")
    return list(pat.finditer(text))


_REF_TAIL = re.compile(r"\s*\[\s*i\s*\]")
_PURE_ASSIGN = re.compile(r"\s*=(?!=)")
_COMPOUND = re.compile(r"\s*(?:<<|>>|[-+*/%&|^])=")
_POSTFIX = re.compile(r"\s*(?:\+\+|--)")


def analyze(text: str, vectors) -> dict | None:
    """Per-vector :class:`Access` if the vector path is legal for *text*,
    else None.  *vectors* are parameter names."""
    result = {}
    unconditional_stores = not _CONTROL.search(text)
    for name in vectors:
        read = written = False
        for m in _occurrences(name, text):
            tail = _REF_TAIL.match(text, m.end())
            if tail is None:
                return None  # x used as a pointer / with another index
            before = text[:m.start()].rstrip()
            if before.endswith("&") and not before.endswith("&&"):
                return None  # address of the element
            after = tail.end()
            prefix_incdec = before.endswith("++") or before.endswith("--")
            if prefix_incdec or _COMPOUND.match(text, after) or _POSTFIX.match(text, after):
                read = written = True
            elif _PURE_ASSIGN.match(text, after):
                written = True
                at_statement_start = before == "" or before.endswith(";")
                if not (at_statement_start and unconditional_stores):
                    read = True  # partial/conditional write: keep old values
            else:
                read = True
        result[name] = Access(read, written)
    return result


def chunk_width(sig, access) -> int:
    """Elements per 16-byte chunk: set by the narrowest accessed vector."""
    sizes = [p.dtype.size for p in sig.vectors if access[p.name].used]
    return 16 // min(sizes) if sizes else 0


def parts(sig, access, width: int, policy: str) -> dict:
    """Placeholder bindings shared by the elementwise and reduction templates.

    User identifiers never appear in kernel scope: kernel parameters are
    ``rtcg_p_<name>`` (vectors) / ``rtcg_w_<name>`` (widened scalars), the
    converted scalars ``rtcg_s_<name>``; the user's names exist only as the
    parameters of ``rtcg_op`` / ``rtcg_map``.  So a parameter called ``b``,
    ``k`` or ``E`` cannot collide with, or be shadowed by, template locals
    (``rtcg_`` is a reserved prefix)."""
    ld_ro, ld_rw, st = CACHE_POLICIES[policy]
    vec_ok = access is not None and width > 0
    op_tparams, op_params, kgen, kvec, unpack = [], [], [], [], []
    ptr_gen, ptr_vec, lane_types, lane_args, call_args = [], [], [], [], []
    decls, loads, stores = [], [], []
    decls_next, loads_next, copies_next = [], [], []
    for p in sig.params:
        c = p.dtype.cname
        if not p.is_vector:
            wide = _WIDE[p.dtype.kind][0]
            op_params.append(f", {c} {p.name}")
            kgen.append(f"{wide} rtcg_w_{p.name}")
            kvec.append(f"{wide} rtcg_w_{p.name}")
            unpack.append(f"    const {c} rtcg_s_{p.name} = ({c}) rtcg_w_{p.name};")
            call_args.append(f", rtcg_s_{p.name}")
            lane_args.append(f", rtcg_s_{p.name}")
            continue
        call_args.append(f", rtcg_p_{p.name}")
        op_tparams.append(f"class rtcg_T_{p.name}")
        op_params.append(f", rtcg_T_{p.name} {p.name}")
        kgen.append(f"{c} *rtcg_p_{p.name}")
        ptr_gen.append(f"{c} *")
        acc = access[p.name] if vec_ok else Access(True, True)
        read_only = acc.read and not acc.written
        qual = "const " if read_only else ""
        kvec.append(f"{qual}{c} *__restrict__ rtcg_p_{p.name}")
        ptr_vec.append(f"{qual}{c} *")
        if vec_ok and acc.used:
            lane_types.append(f"rtcg::lane<{c}>")
            lane_args.append(f", rtcg::lane<{c}>{{rtcg_v_{p.name}[u].e[k]}}")
            decls.append(f"        rtcg::chunk<{c}, E> rtcg_v_{p.name}[U];")
            if acc.read:
                hint = ld_ro if read_only else ld_rw
                loads.append(f"                rtcg::load<{hint}>(rtcg_v_{p.name}[u], rtcg_p_{p.name}, cu);")
                decls_next.append(f"    rtcg::chunk<{c}, E> rtcg_n_{p.name}[U];")
                loads_next.append(f"            rtcg::load<{hint}>(rtcg_n_{p.name}[u], "
                                  f"rtcg_p_{p.name}, cu);")
                copies_next.append(f"#pragma unroll\n        for (int u = 0; u < U; ++u) "
                                   f"rtcg_v_{p.name}[u] = rtcg_n_{p.name}[u];")
            if acc.written:
                stores.append(f"                rtcg::store<{st}>(rtcg_p_{p.name}, cu, rtcg_v_{p.name}[u]);")
        else:
            lane_types.append(f"{qual}{c} *")
            lane_args.append(f", rtcg_p_{p.name}")
    return {
        "vector": vec_ok,
        "tma": False,
        "width": width,
        "op_tparams": ", ".join(op_tparams),
        "op_params": "".join(op_params),
        "kparams_generic": ", ".join(kgen),
        "kparams_vector": ", ".join(kvec),
        "unpack": "\n".join(unpack),
        "ptr_types_generic": ", ".join(ptr_gen),
        "ptr_types_vector": ", ".join(ptr_vec),
        "call_args": "".join(call_args),
        "lane_types": ", ".join(lane_types),
        "lane_args": "".join(lane_args),
        "vec_decls": "\n".join(decls),
        "vec_loads": "\n".join(loads),
        "vec_stores": "\n".join(stores),
        "vec_decls_next": "\n".join(decls_next),
        "vec_loads_next": "\n".join(loads_next),
        "vec_copy_next": "\n".join(copies_next),
        "prefetch": False,
        "stages": 0,
    }


def render(template_name: str, bindings: dict) -> str:
    return cs.render(template(template_name),
                     {"prelude": template("prelude.cuh").rstrip("\n"), **bindings})


# --- launch plumbing ---------------------------------------------------------------------


def scalar_value(value, dtype):
    """Widen a Python/numpy scalar the way the reference does
    (``src/elementwise.py:316-321``): float kinds -> double, unsigned ->
    uint64 modulo 2**64, signed -> int64; the kernel casts to the declared
    type."""
    if dtype.kind == "f":
        return ctypes.c_double(float(value))
    if dtype.kind == "u":
        return ctypes.c_uint64(int(value) & 0xFFFFFFFFFFFFFFFF)
    return ctypes.c_int64(int(value))


_MASK64 = (1 << 64) - 1
_PACK_D = struct.Struct("<d").pack
_UNPACK_Q = struct.Struct("<Q").unpack


def _bits(value, kind: str) -> int:
    """The 8 bytes of the widened scalar slot, as an unsigned integer."""
    if kind == "f":
        return _UNPACK_Q(_PACK_D(float(value)))[0]
    return int(value) & _MASK64


class Binder:
    """Argument marshalling for one kernel signature into preallocated
    per-thread parameter slots (every kernel parameter is 8 bytes: pointers,
    widened scalars, ``long start/end``, scratch pointers).  cuLaunchKernel
    copies parameter values at launch, so the slots are reusable as soon as
    the launch call returns.  Validation follows ``src/elementwise.py:324-366``.
    """

    def __init__(self, sig, extra: int = 0) -> None:
        self.params = sig.params
        self.count = len(self.params)
        self.total = self.count + 2 + extra
        self._tls = threading.local()
        # (slot, is_vector, dtype, element size, scalar kind, name) per parameter
        self._plan = tuple((k, p.is_vector, p.dtype, p.dtype.size, p.dtype.kind, p.name, p)
                           for k, p in enumerate(self.params))

    def slots(self):
        held = getattr(self._tls, "slots", None)
        if held is None:
            vals = (ctypes.c_uint64 * self.total)()
            base = ctypes.addressof(vals)
            ptrs = (ctypes.c_void_p * self.total)(*[base + 8 * k for k in range(self.total)])
            held = self._tls.slots = (vals, ptrs)
        return held

    def bind(self, args, n, base: int, name: str, errors):
        """-> (vals, ptrs, vectors, n); ``vectors`` = [(param, addr0, local)].
        ``errors`` = (ArityMismatch, DtypeMismatch, ShapeMismatch, NdArray)."""
        if len(args) != self.count:
            raise errors[0](f"kernel {name} takes {self.count} arguments, got {len(args)}")
        array_t = errors[3]
        try:
            vals, ptrs = self._tls.slots
        except AttributeError:
            vals, ptrs = self.slots()
        vectors = []
        for k, is_vector, dtype, size, kind, pname, p in self._plan:
            arg = args[k]
            if is_vector:
                if arg.__class__ is not array_t and not isinstance(arg, array_t):
                    raise errors[1](pname, f"expected a GPUArray, got {type(arg).__name__}")
                if arg.dtype is not dtype and arg.dtype != dtype:
                    raise errors[1](pname, f"expected dtype {dtype.name}, got {arg.dtype.name}")
                asize = arg.size
                if n is None:
                    n = asize
                elif asize < n:
                    raise errors[2](f"vector {pname!r} holds {asize} elements, "
                                    f"kernel span is {n}")
                if arg._freed:
                    raise ValueError("array was freed")
                block = arg._block
                local = block.address if block is not None else 0
                addr0 = (local - base * size) & _MASK64 if base else local
                vals[k] = addr0
                vectors.append((p, addr0, local))
            else:
                if isinstance(arg, array_t):
                    raise errors[1](pname, "expected a scalar, got a GPUArray")
                vals[k] = _UNPACK_Q(_PACK_D(float(arg)))[0] if kind == "f" \
                    else int(arg) & _MASK64
        if n is None:
            raise errors[0]("cannot infer n: no vector arguments")
        return vals, ptrs, vectors, n

    def set_range(self, vals, start: int, end: int) -> None:
        vals[self.count] = start & _MASK64
        vals[self.count + 1] = end & _MASK64


def pack(values) -> ctypes.Array:
    """cuLaunchKernel parameter array: pointers to each ctypes value."""
    arr = (ctypes.c_void_p * len(values))()
    for k, v in enumerate(values):
        arr[k] = ctypes.addressof(v)
    return arr


def vector_path_ok(entries, n: int) -> bool:
    """entries: (index-0 address, local address, itemsize, Access) per used
    vector.  True when every index-0 address is 16-byte aligned and no written
    vector overlaps another used vector over the n local elements."""
    bits = 0
    for e in entries:
        bits |= e[0]
    if bits & 15:
        return False
    for a, (_, lo_a, size_a, acc_a) in enumerate(entries):
        if not acc_a.written:
            continue
        hi_a = lo_a + n * size_a
        for b, (_, lo_b, size_b, _acc) in enumerate(entries):
            if b != a and lo_a < lo_b + n * size_b and lo_b < hi_a:
                return False
    return True


_sm_count: dict[int, int] = {}


def sm_count(device: int) -> int:
    hit = _sm_count.get(device)
    if hit is None:
        hit = _sm_count[device] = _runtime.device_info(device)["sm_count"]
    return hit


_grid_cache: dict = {}


def grid_for(function: int, device: int, block: int, workers: int | None,
             n: int, per_thread: int, waves: int = 1, smem: int = 0) -> int:
    """CTAs to launch: explicit ``workers``; else ``waves`` x the resident CTAs
    (SMs x occupancy), never more than the work needs; ``waves=0`` = exactly
    the work (one step per thread)."""
    key = (function, device, block, workers, n, per_thread, waves, smem)
    hit = _grid_cache.get(key)
    if hit is not None:
        return hit
    if len(_grid_cache) > 4096:
        _grid_cache.clear()
    grid = _grid_cache[key] = _compute_grid(function, device, block, workers, n, per_thread,
                                            waves, smem)
    return grid


def _compute_grid(function, device, block, workers, n, per_thread, waves, smem=0) -> int:
    useful = max(1, -(-n // (block * per_thread)))
    if workers is not None:
        grid = workers
    elif waves == 0:
        grid = useful
    else:
        resident = sm_count(device) * max(1, _runtime.occupancy(function, block, smem))
        grid = min(resident * waves, useful)
    return max(1, min(grid, 2**31 - 1))
