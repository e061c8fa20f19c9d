"""ctypes binding of ``librtcg_b200.so`` (declared in ``include/rtcg_b200.h``).

This is the only module that talks to the native runtime.  It mirrors what
the reference does at its native seams -- ``ctypes.CDLL`` of compiled code
(``src/jit.py:439-443``) and ctypes kernel calls (``src/jit.py:553-554``) --
except that the library here is the fixed NVRTC + CUDA-driver runtime and the
kernels it launches live on the GPU.

There is no CPU fallback: if the library is missing, importing a submodule
that needs it raises :class:`RuntimeMissing`; if there is no GPU, every driver
call raises :class:`NoDevice`.  NVRTC compilation works without a GPU.
"""

from __future__ import annotations

import ctypes
import os
import threading
from pathlib import Path

__all__ = [
    "CudaError", "NoDevice", "DeviceOutOfMemory", "ModuleLoadFailed",
    "SymbolMissing", "CompilerFailed", "RuntimeMissing", "LIB_PATH", "lib",
    "nvrtc_version", "compile_cubin", "device_count", "device_info",
    "set_device", "current_device", "synchronize", "Module", "launch",
    "mem_alloc", "mem_free", "memset_async", "memcpy_htod", "memcpy_dtoh",
    "memcpy_dtod", "host_alloc", "host_free", "Stream", "Event",
    "current_stream", "use_stream", "have_gpu",
]

LIB_PATH = Path(__file__).resolve().parent / "librtcg_b200.so"

RTCG_OK = 0
RTCG_ERR_CUDA = 1
RTCG_ERR_OUT_OF_MEMORY = 2
RTCG_ERR_NOT_FOUND = 3
RTCG_ERR_COMPILE = 4
RTCG_ERR_NO_DEVICE = 5
RTCG_ERR_INVALID = 6
RTCG_ERR_LOAD = 7
RTCG_ERR_NO_COMPILER = 8


class RuntimeMissing(ImportError):
    """librtcg_b200.so has not been built (run ``python -m paper_0911_3456_b200._build``)."""


class CudaError(RuntimeError):
    def __init__(self, status: int, message: str) -> None:
        super().__init__(message)
        self.status = status


class NoDevice(CudaError):
    """No NVIDIA driver or no visible CUDA device."""


class DeviceOutOfMemory(CudaError, MemoryError):
    """CUDA_ERROR_OUT_OF_MEMORY; a MemoryError so pools can release and retry."""


class ModuleLoadFailed(CudaError):
    """The driver rejected a module image."""


class SymbolMissing(CudaError):
    """A kernel symbol is not present in a loaded module."""


class CompilerFailed(CudaError):
    """NVRTC rejected the source; ``log`` holds its diagnostics."""

    def __init__(self, status: int, message: str, log: str = "") -> None:
        super().__init__(status, message)
        self.log = log


_ERRORS = {
    RTCG_ERR_OUT_OF_MEMORY: DeviceOutOfMemory,
    RTCG_ERR_NOT_FOUND: SymbolMissing,
    RTCG_ERR_NO_DEVICE: NoDevice,
    RTCG_ERR_LOAD: ModuleLoadFailed,
    RTCG_ERR_COMPILE: CompilerFailed,
    RTCG_ERR_NO_COMPILER: CompilerFailed,
}


class _DeviceInfo(ctypes.Structure):
    _fields_ = [
        ("name", ctypes.c_char * 128),
        ("cc_major", ctypes.c_int), ("cc_minor", ctypes.c_int),
        ("sm_count", ctypes.c_int),
        ("max_threads_per_sm", ctypes.c_int),
        ("max_threads_per_block", ctypes.c_int),
        ("l2_bytes", ctypes.c_int),
        ("driver_version", ctypes.c_int),
        ("mem_clock_khz", ctypes.c_int), ("mem_bus_width", ctypes.c_int),
        ("total_mem", ctypes.c_uint64),
    ]


_vp = ctypes.c_void_p
_u64 = ctypes.c_uint64
_int = ctypes.c_int
_pint = ctypes.POINTER(ctypes.c_int)

# name -> argtypes; every function returns int status
_PROTOTYPES = {
    "rtcg_nvrtc_version": (_pint, _pint),
    "rtcg_compile": (ctypes.c_char_p, ctypes.c_char_p,
                     ctypes.POINTER(ctypes.c_char_p), _int,
                     ctypes.POINTER(_vp), ctypes.POINTER(ctypes.c_size_t),
                     ctypes.POINTER(_vp)),
    "rtcg_init": (),
    "rtcg_device_count": (_pint,),
    "rtcg_device_info_get": (_int, ctypes.POINTER(_DeviceInfo)),
    "rtcg_set_device": (_int,),
    "rtcg_get_device": (_pint,),
    "rtcg_synchronize": (),
    "rtcg_mem_get_info": (ctypes.POINTER(_u64), ctypes.POINTER(_u64)),
    "rtcg_module_load": (_vp, ctypes.c_size_t, ctypes.POINTER(_vp)),
    "rtcg_module_unload": (_vp,),
    "rtcg_module_function": (_vp, ctypes.c_char_p, ctypes.POINTER(_vp)),
    "rtcg_function_occupancy": (_vp, _int, ctypes.c_size_t, _pint),
    "rtcg_function_registers": (_vp, _pint),
    "rtcg_function_set_max_dynamic_smem": (_vp, _int),
    "rtcg_launch": (_vp, ctypes.c_uint, ctypes.c_uint, ctypes.c_uint, _vp,
                    ctypes.POINTER(_vp)),
    "rtcg_launch_ex": (_vp, ctypes.c_uint, ctypes.c_uint, ctypes.c_uint, _vp,
                       ctypes.POINTER(_vp), ctypes.c_uint),
    "rtcg_mem_alloc": (_u64, ctypes.POINTER(_u64)),
    "rtcg_mem_free": (_u64,),
    "rtcg_mem_alloc_async": (_u64, _vp, ctypes.POINTER(_u64)),
    "rtcg_mem_free_async": (_u64, _vp),
    "rtcg_mem_trim": (),
    "rtcg_memset_async": (_u64, ctypes.c_ubyte, _u64, _vp),
    "rtcg_memcpy_htod_async": (_u64, _vp, _u64, _vp),
    "rtcg_memcpy_dtoh_async": (_vp, _u64, _u64, _vp),
    "rtcg_memcpy_dtod_async": (_u64, _u64, _u64, _vp),
    "rtcg_copy_htod": (_u64, _vp, _u64, _vp),
    "rtcg_copy_dtoh": (_vp, _u64, _u64, _vp),
    "rtcg_host_alloc": (_u64, ctypes.POINTER(_vp)),
    "rtcg_host_free": (_vp,),
    "rtcg_host_register": (_vp, _u64),
    "rtcg_host_is_pinned": (_vp, ctypes.POINTER(ctypes.c_int)),
    "rtcg_host_unregister": (_vp,),
    "rtcg_stream_create": (ctypes.POINTER(_vp),),
    "rtcg_stream_destroy": (_vp,),
    "rtcg_stream_synchronize": (_vp,),
    "rtcg_event_create": (ctypes.POINTER(_vp),),
    "rtcg_event_destroy": (_vp,),
    "rtcg_event_record": (_vp, _vp),
    "rtcg_device_pci_bus_id": (_int, ctypes.c_char_p, _int),
    "rtcg_stream_wait_event": (_vp, _vp),
    "rtcg_stream_is_capturing": (_vp, _pint),
    "rtcg_event_synchronize": (_vp,),
    "rtcg_event_elapsed_ms": (_vp, _vp, ctypes.POINTER(ctypes.c_float)),
    "rtcg_stream_begin_capture": (_vp,),
    "rtcg_stream_end_capture": (_vp, ctypes.POINTER(_vp)),
    "rtcg_graph_launch": (_vp, _vp),
    "rtcg_graph_destroy": (_vp,),
    "rtcg_ipc_get_handle": (_u64, ctypes.c_char_p),
    "rtcg_ipc_open_handle": (ctypes.c_char_p, ctypes.POINTER(_u64)),
    "rtcg_ipc_close_handle": (_u64,),
    "rtcg_device_can_access_peer": (_int, _int, _pint),
}

EXPORTED_SYMBOLS = tuple(sorted(_PROTOTYPES)) + (
    "rtcg_abi_version", "rtcg_last_error", "rtcg_free_buffer")

_lib = None
_lib_lock = threading.Lock()


def lib() -> ctypes.CDLL:
    """The loaded runtime library (loaded once, prototypes attached)."""
    global _lib
    if _lib is not None:
        return _lib
    with _lib_lock:
        if _lib is not None:
            return _lib
        path = os.environ.get("RTCG_RUNTIME_LIBRARY") or str(LIB_PATH)
        if not Path(path).exists():
            raise RuntimeMissing(
                f"{path} is not built; run `python -m paper_0911_3456_b200._build`")
        handle = ctypes.CDLL(path, mode=ctypes.RTLD_LOCAL)
        for name, argtypes in _PROTOTYPES.items():
            fn = getattr(handle, name)
            fn.argtypes = list(argtypes)
            fn.restype = ctypes.c_int
        handle.rtcg_abi_version.restype = ctypes.c_int
        handle.rtcg_abi_version.argtypes = []
        handle.rtcg_last_error.restype = ctypes.c_char_p
        handle.rtcg_last_error.argtypes = []
        handle.rtcg_free_buffer.restype = None
        handle.rtcg_free_buffer.argtypes = [_vp]
        if handle.rtcg_abi_version() != 1:
            raise RuntimeMissing(f"{path}: unexpected ABI version")
        _lib = handle
        return _lib


_fast = None


def fastlaunch():
    """The native launch-path extension (``_fastlaunch``), wired to this
    library's ``rtcg_launch``.  Built with the runtime; missing = not built."""
    global _fast
    if _fast is None:
        try:
            from . import _fastlaunch as mod
        except ImportError as exc:
            raise RuntimeMissing(
                f"_fastlaunch is not built ({exc}); run `python -m paper_0911_3456_b200._build`"
            ) from exc
        mod.set_launcher(ctypes.cast(lib().rtcg_launch_ex, ctypes.c_void_p).value)
        _fast = mod
    return _fast


def _check(status: int, what: str = "") -> None:
    if status == RTCG_OK:
        return
    message = (lib().rtcg_last_error() or b"").decode(errors="replace")
    cls = _ERRORS.get(status, CudaError)
    raise cls(status, f"{what}: {message}" if what else message)


# --- NVRTC ---------------------------------------------------------------------


def nvrtc_version() -> tuple[int, int]:
    major, minor = ctypes.c_int(), ctypes.c_int()
    _check(lib().rtcg_nvrtc_version(ctypes.byref(major), ctypes.byref(minor)),
           "nvrtc")
    return major.value, minor.value


def compile_cubin(source: str, options, program_name: str = "rtcg.cu"):
    """Compile CUDA C++ to an sm_XXX cubin with NVRTC, in process.

    Returns ``(cubin_bytes, log)``; raises :class:`CompilerFailed` carrying
    the NVRTC log on a compile error.
    """
    opts = [o.encode() for o in options]
    arr = (ctypes.c_char_p * max(1, len(opts)))(*opts)
    image, size, log = _vp(), ctypes.c_size_t(), _vp()
    status = lib().rtcg_compile(source.encode(), program_name.encode(), arr,
                                len(opts), ctypes.byref(image),
                                ctypes.byref(size), ctypes.byref(log))
    text = ""
    if log.value:
        text = ctypes.string_at(log.value).decode(errors="replace")
        lib().rtcg_free_buffer(log)
    if status != RTCG_OK:
        message = (lib().rtcg_last_error() or b"").decode(errors="replace")
        cls = _ERRORS.get(status, CudaError)
        if cls is CompilerFailed:
            raise CompilerFailed(status, message, text)
        raise cls(status, message)
    data = ctypes.string_at(image.value, size.value)
    lib().rtcg_free_buffer(image)
    return data, text


# --- devices -----------------------------------------------------------------------

_tls = threading.local()
_info_cache: dict[int, dict] = {}


def have_gpu() -> bool:
    """True when the runtime is built, the driver loads, and a device exists."""
    try:
        return lib().rtcg_init() == RTCG_OK
    except RuntimeMissing:
        return False


def device_count() -> int:
    count = ctypes.c_int()
    _check(lib().rtcg_device_count(ctypes.byref(count)), "device count")
    return count.value


def device_info(device: int | None = None) -> dict:
    dev = current_device() if device is None else device
    cached = _info_cache.get(dev)
    if cached is not None:
        return cached
    info = _DeviceInfo()
    _check(lib().rtcg_device_info_get(dev, ctypes.byref(info)), "device info")
    out = {k: getattr(info, k) for k, _ in _DeviceInfo._fields_}
    out["name"] = info.name.decode(errors="replace")
    out["arch"] = f"sm_{info.cc_major}{info.cc_minor}"
    _info_cache[dev] = out
    return out


def pci_bus_id(device: int) -> str:
    """Process-independent identity of a visible device ("0000:1b:00.0")."""
    buf = ctypes.create_string_buffer(32)
    _check(lib().rtcg_device_pci_bus_id(device, buf, len(buf)), "pci bus id")
    return buf.value.decode().lower()


def set_device(device: int) -> None:
    """Make ``device``'s primary context current on this thread."""
    if getattr(_tls, "device", None) == device:
        return
    _check(lib().rtcg_set_device(device), f"set device {device}")
    _tls.device = device


def current_device() -> int:
    dev = getattr(_tls, "device", None)
    if dev is None:
        out = ctypes.c_int()
        _check(lib().rtcg_get_device(ctypes.byref(out)), "current device")
        dev = _tls.device = out.value
    return dev


def synchronize() -> None:
    current_device()
    _check(lib().rtcg_synchronize(), "synchronize")


def mem_get_info() -> tuple[int, int]:
    free, total = _u64(), _u64()
    _check(lib().rtcg_mem_get_info(ctypes.byref(free), ctypes.byref(total)),
           "mem info")
    return free.value, total.value


# --- streams ---------------------------------------------------------------------------


class Stream:
    """A non-blocking CUDA stream owned by this runtime (or a borrowed handle)."""

    def __init__(self, handle: int | None = None) -> None:
        self._owned = handle is None
        if handle is None:
            current_device()
            out = _vp()
            _check(lib().rtcg_stream_create(ctypes.byref(out)), "stream create")
            handle = out.value
        self.handle = handle or 0

    def synchronize(self) -> None:
        _check(lib().rtcg_stream_synchronize(self.handle or None), "stream sync")

    def wait(self, event: "Event") -> None:
        """Order work submitted to this stream after ``event``."""
        stream_wait_event(self.handle, event)

    def close(self) -> None:
        if self._owned and self.handle:
            _check(lib().rtcg_stream_destroy(self.handle), "stream destroy")
            self.handle = 0

    def __repr__(self) -> str:
        return f"<Stream 0x{self.handle:x}>"


def current_stream() -> int:
    """Raw handle of the stream launches go to on this thread (0 = legacy default)."""
    return getattr(_tls, "stream", 0)


class use_stream:
    """Context manager routing this thread's launches/copies to a stream.

    Accepts a :class:`Stream`, a raw handle (e.g. ``torch.cuda.current_stream()
    .cuda_stream``) or None for the legacy default stream.
    """

    def __init__(self, stream) -> None:
        if isinstance(stream, Stream):
            stream = stream.handle
        self.handle = stream or 0

    def __enter__(self):
        self._saved = current_stream()
        _tls.stream = self.handle
        return self

    def __exit__(self, *exc):
        _tls.stream = self._saved


class Event:
    def __init__(self) -> None:
        current_device()
        out = _vp()
        _check(lib().rtcg_event_create(ctypes.byref(out)), "event create")
        self.handle = out.value

    def record(self, stream: int | None = None) -> "Event":
        s = current_stream() if stream is None else stream
        _check(lib().rtcg_event_record(self.handle, s or None), "event record")
        return self

    def synchronize(self) -> None:
        _check(lib().rtcg_event_synchronize(self.handle), "event sync")

    def elapsed_ms(self, end: "Event") -> float:
        ms = ctypes.c_float()
        _check(lib().rtcg_event_elapsed_ms(self.handle, end.handle,
                                           ctypes.byref(ms)), "elapsed")
        return ms.value

    def __del__(self):
        handle = getattr(self, "handle", None)
        if handle and _lib is not None:
            try:
                _lib.rtcg_event_destroy(handle)
            except Exception:  # pragma: no cover - interpreter shutdown
                pass


def stream_wait_event(stream, event: Event) -> None:
    """Work submitted to ``stream`` (raw handle, 0 = legacy) after this call
    waits for ``event`` (cuStreamWaitEvent)."""
    _check(lib().rtcg_stream_wait_event(stream or None, event.handle), "stream wait event")


def stream_is_capturing(stream=None) -> bool:
    """Whether ``stream`` (default: this thread's current stream) is being
    captured into a CUDA graph."""
    s = current_stream() if stream is None else getattr(stream, "handle", stream)
    out = ctypes.c_int()
    _check(lib().rtcg_stream_is_capturing(s or None, ctypes.byref(out)), "is capturing")
    return bool(out.value)


def order_after_current(streams) -> None:
    """Make every stream in ``streams`` wait for the work already submitted
    to this thread's current stream (one event, recorded now)."""
    ev = _order_event()
    ev.record(current_stream())
    for st in streams:
        stream_wait_event(getattr(st, "handle", st), ev)


def _order_event() -> Event:
    dev = current_device()
    evs = getattr(_tls, "order_events", None)
    if evs is None:
        evs = _tls.order_events = {}
    ev = evs.get(dev)
    if ev is None:
        ev = evs[dev] = Event()
    return ev


# --- graphs ------------------------------------------------------------------------------


def begin_capture(stream: int) -> None:
    _check(lib().rtcg_stream_begin_capture(stream or None), "begin capture")


def end_capture(stream: int) -> int:
    out = _vp()
    _check(lib().rtcg_stream_end_capture(stream or None, ctypes.byref(out)), "end capture")
    return out.value


def graph_launch(graph: int, stream: int) -> None:
    _check(lib().rtcg_graph_launch(graph, stream or None), "graph launch")


def graph_destroy(graph: int) -> None:
    _check(lib().rtcg_graph_destroy(graph), "graph destroy")


# --- modules and launches ------------------------------------------------------------


class Module:
    """A cubin loaded into the current device's primary context."""

    def __init__(self, image: bytes) -> None:
        current_device()
        out = _vp()
        self._image = image  # keep alive for the driver's lifetime of the call
        _check(lib().rtcg_module_load(image, len(image), ctypes.byref(out)),
               "module load")
        self.handle = out.value
        self._functions: dict[str, int] = {}

    def function(self, name: str) -> int:
        fn = self._functions.get(name)
        if fn is None:
            out = _vp()
            _check(lib().rtcg_module_function(self.handle, name.encode(),
                                              ctypes.byref(out)), "function")
            fn = self._functions[name] = out.value
        return fn


_occupancy_cache: dict[tuple[int, int], int] = {}


_smem_optin: dict[int, int] = {}


def set_max_dynamic_smem(function: int, nbytes: int) -> None:
    """Allow ``function`` to launch with ``nbytes`` of dynamic shared memory."""
    if _smem_optin.get(function, 0) >= nbytes:
        return
    _check(lib().rtcg_function_set_max_dynamic_smem(function, nbytes), "smem opt-in")
    _smem_optin[function] = nbytes


def occupancy(function: int, block: int, smem: int = 0) -> int:
    key = (function, block, smem)
    hit = _occupancy_cache.get(key)
    if hit is None:
        out = ctypes.c_int()
        _check(lib().rtcg_function_occupancy(function, block, smem,
                                             ctypes.byref(out)), "occupancy")
        hit = _occupancy_cache[key] = out.value
    return hit


def registers(function: int) -> int:
    out = ctypes.c_int()
    _check(lib().rtcg_function_registers(function, ctypes.byref(out)), "regs")
    return out.value


def launch(function: int, grid: int, block: int, params, smem: int = 0,
           stream: int | None = None) -> None:
    """cuLaunchKernel with ``params`` = ctypes array of pointers to values."""
    s = current_stream() if stream is None else getattr(stream, "handle", stream)
    _check(lib().rtcg_launch(function, grid, block, smem, s or None, params),
           "launch")


def launch_overlapped(function: int, grid: int, block: int, params, smem: int = 0,
                      stream: int | None = None) -> None:
    """Programmatic dependent launch (see rtcg_launch_ex in the header)."""
    s = current_stream() if stream is None else getattr(stream, "handle", stream)
    _check(lib().rtcg_launch_ex(function, grid, block, smem, s or None, params, 1),
           "launch (overlapped)")


# --- memory ------------------------------------------------------------------------------


def _alloc_with_trim(call, what: str) -> None:
    """Run an allocation; on out-of-memory, trim the stream-ordered pool's
    cached memory and retry once before raising DeviceOutOfMemory."""
    status = call()
    if status == RTCG_ERR_OUT_OF_MEMORY:
        _check(lib().rtcg_mem_trim(), "trim")
        status = call()
    _check(status, what)


def mem_alloc(nbytes: int) -> int:
    current_device()
    out = _u64()
    _alloc_with_trim(lambda: lib().rtcg_mem_alloc(nbytes, ctypes.byref(out)),
                     f"cuMemAlloc({nbytes})")
    return out.value


def mem_free(dptr: int) -> None:
    _check(lib().rtcg_mem_free(dptr), "cuMemFree")


def mem_alloc_async(nbytes: int, stream=None) -> int:
    """Stream-ordered allocation (cuMemAllocAsync from the device mempool)."""
    current_device()
    s = current_stream() if stream is None else stream
    out = _u64()
    _alloc_with_trim(lambda: lib().rtcg_mem_alloc_async(nbytes, s or None, ctypes.byref(out)),
                     f"cuMemAllocAsync({nbytes})")
    return out.value


def mem_free_async(dptr: int, stream=None) -> None:
    s = current_stream() if stream is None else stream
    _check(lib().rtcg_mem_free_async(dptr, s or None), "cuMemFreeAsync")


def memset_async(dptr: int, value: int, nbytes: int, stream=None) -> None:
    s = current_stream() if stream is None else stream
    _check(lib().rtcg_memset_async(dptr, value, nbytes, s or None), "memset")


def memcpy_htod(dst: int, src: int, nbytes: int, stream=None) -> None:
    s = current_stream() if stream is None else stream
    _check(lib().rtcg_memcpy_htod_async(dst, src, nbytes, s or None), "HtoD")


def memcpy_dtoh(dst: int, src: int, nbytes: int, stream=None) -> None:
    s = current_stream() if stream is None else stream
    _check(lib().rtcg_memcpy_dtoh_async(dst, src, nbytes, s or None), "DtoH")


def copy_htod(dst: int, src: int, nbytes: int, stream=None) -> None:
    """Host->device copy; pageable sources go through pinned staging."""
    s = current_stream() if stream is None else stream
    _check(lib().rtcg_copy_htod(dst, src, nbytes, s or None), "HtoD")


def copy_dtoh(dst: int, src: int, nbytes: int, stream=None) -> None:
    """Device->host copy into pinned or pageable memory; returns when filled."""
    s = current_stream() if stream is None else stream
    _check(lib().rtcg_copy_dtoh(dst, src, nbytes, s or None), "DtoH")


def memcpy_dtod(dst: int, src: int, nbytes: int, stream=None) -> None:
    s = current_stream() if stream is None else stream
    _check(lib().rtcg_memcpy_dtod_async(dst, src, nbytes, s or None), "DtoD")


def stream_synchronize(stream=None) -> None:
    s = current_stream() if stream is None else stream
    _check(lib().rtcg_stream_synchronize(s or None), "stream sync")


def ipc_get_handle(dptr: int) -> bytes:
    """64-byte CUDA IPC handle of an ``mem_alloc`` buffer."""
    buf = ctypes.create_string_buffer(64)
    _check(lib().rtcg_ipc_get_handle(dptr, buf), "cuIpcGetMemHandle")
    return buf.raw


def ipc_open_handle(handle: bytes) -> int:
    """Map another process's buffer into this context (peer access lazily
    enabled); returns its device address here."""
    if len(handle) != 64:
        raise ValueError("an IPC handle is 64 bytes")
    out = _u64()
    _check(lib().rtcg_ipc_open_handle(handle, ctypes.byref(out)), "cuIpcOpenMemHandle")
    return out.value


def ipc_close_handle(dptr: int) -> None:
    _check(lib().rtcg_ipc_close_handle(dptr), "cuIpcCloseMemHandle")


def can_access_peer(device: int, peer: int) -> bool:
    out = _int()
    _check(lib().rtcg_device_can_access_peer(device, peer, ctypes.byref(out)),
           "cuDeviceCanAccessPeer")
    return bool(out.value)


def host_alloc(nbytes: int) -> int:
    current_device()
    out = _vp()
    _check(lib().rtcg_host_alloc(max(1, nbytes), ctypes.byref(out)),
           "cuMemHostAlloc")
    return out.value


def host_free(ptr: int) -> None:
    _check(lib().rtcg_host_free(ptr), "cuMemFreeHost")


def host_is_pinned(ptr: int) -> bool:
    """Whether host address ``ptr`` lies in page-locked memory (the test the
    host copies use to DMA directly instead of staging)."""
    current_device()
    out = ctypes.c_int(0)
    _check(lib().rtcg_host_is_pinned(ptr, ctypes.byref(out)), "host is pinned")
    return bool(out.value)
