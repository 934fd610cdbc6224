"""ctypes binding to ``libkaas_b200.so`` (C ABI in ``include/kaas_b200.h``).

There is no fallback: if the library or a CUDA device is missing, every
device-touching call raises.  ctypes releases the GIL for the duration of
each call, so one worker thread per GPU overlaps host work with the others.
"""

from __future__ import annotations

import ctypes as C
import os
import threading

import numpy as np

from .faults import (
    ArityMismatchError,
    BackendFaultError,
    DeviceError,
    KaasError,
    UnknownKernelError,
)

LIB_NAME = "libkaas_b200.so"
LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), LIB_NAME)

KAAS_E_INVALID = -1
KAAS_E_ARITY = -2
KAAS_E_BOUNDS = -3
KAAS_E_UNKNOWN_KERNEL = -4
KAAS_E_UNSUPPORTED = -5

# kernel ids (kaas_b200.h)
K_VECTOR_ADD = 1
K_SAXPY = 2
K_MATMUL = 3
K_REDUCE_SUM = 4
K_FILL = 5
K_CGEMM = 6
K_JACOBI = 7

LIT_TAGS = {"i32": 0, "i64": 1, "f32": 2, "f64": 3}
MAX_LITS = 4
MAX_ARGS = 8


class Literal(C.Structure):
    _fields_ = [("tag", C.c_int32), ("reserved", C.c_int32),
                ("i", C.c_int64), ("f", C.c_double)]


class LaunchDesc(C.Structure):
    _fields_ = [
        ("kernel", C.c_int32), ("n_lits", C.c_int32), ("n_args", C.c_int32),
        ("flags", C.c_int32), ("dims", C.c_uint32 * 6), ("reserved", C.c_uint32 * 2),
        ("lits", Literal * MAX_LITS), ("ptrs", C.c_uint64 * MAX_ARGS),
        ("sizes", C.c_uint64 * MAX_ARGS),
    ]


class StreamOut(C.Structure):
    _fields_ = [("desc_index", C.c_int32), ("arg_index", C.c_int32),
                ("out_stream", C.c_uint64), ("host_dst", C.c_void_p), ("bytes", C.c_uint64)]


class DeviceInfo(C.Structure):
    _fields_ = [
        ("ordinal", C.c_int32), ("sm_count", C.c_int32), ("cc_major", C.c_int32),
        ("cc_minor", C.c_int32), ("total_mem", C.c_uint64), ("l2_bytes", C.c_uint64),
        ("max_smem_per_block", C.c_int32), ("clock_khz", C.c_int32),
        ("name", C.c_char * 128),
    ]


def _desc_dtype():
    import numpy as np
    lit = np.dtype({"names": ["tag", "reserved", "i", "f"],
                    "formats": ["<i4", "<i4", "<i8", "<f8"],
                    "offsets": [0, 4, 8, 16], "itemsize": C.sizeof(Literal)})
    f = LaunchDesc
    return np.dtype({
        "names": ["kernel", "n_lits", "n_args", "flags", "dims", "reserved", "lits", "ptrs", "sizes"],
        "formats": ["<i4", "<i4", "<i4", "<i4", ("<u4", 6), ("<u4", 2), (lit, MAX_LITS),
                    ("<u8", MAX_ARGS), ("<u8", MAX_ARGS)],
        "offsets": [f.kernel.offset, f.n_lits.offset, f.n_args.offset, f.flags.offset,
                    f.dims.offset, f.reserved.offset, f.lits.offset, f.ptrs.offset,
                    f.sizes.offset],
        "itemsize": C.sizeof(LaunchDesc)})


DESC_DTYPE = _desc_dtype()

_u64 = C.c_uint64
_pu64 = C.POINTER(C.c_uint64)
_vp = C.c_void_p

# name -> (argtypes) ; every function returns int
# kaas_launch_desc.flags for cgemm (include/kaas_b200.h)
F_CG_A_USE, F_CG_B_USE, F_CG_A_FILL, F_CG_B_FILL = 1, 2, 4, 8
F_MM_BT_USE, F_MM_BT_FILL = 16, 32

EXPORTS = {
    "kaas_last_error": [C.c_char_p, C.c_size_t],
    "kaas_version": [C.POINTER(C.c_int), C.POINTER(C.c_int)],
    "kaas_device_count": [C.POINTER(C.c_int)],
    "kaas_init_device": [C.c_int],
    "kaas_device_info_get": [C.c_int, C.POINTER(DeviceInfo)],
    "kaas_launch_counter": [_pu64],
    "kaas_device_check": [C.c_int],
    "kaas_inject_fault": [_u64],
    "kaas_stream_create": [C.c_int, C.c_int, _pu64],
    "kaas_stream_destroy": [_u64],
    "kaas_stream_sync": [_u64],
    "kaas_event_create": [C.c_int, C.c_int, _pu64],
    "kaas_event_destroy": [_u64],
    "kaas_event_record": [_u64, _u64],
    "kaas_stream_wait_event": [_u64, _u64],
    "kaas_event_sync": [_u64],
    "kaas_event_query": [_u64, C.POINTER(C.c_int)],
    "kaas_event_elapsed_ms": [_u64, _u64, C.POINTER(C.c_float)],
    "kaas_event_elapsed_many": [C.c_int, _pu64, _pu64, C.POINTER(C.c_float)],
    "kaas_malloc_async": [_u64, _u64, _pu64],
    "kaas_free_async": [_u64, _u64],
    "kaas_memset_async": [_u64, C.c_int, _u64, _u64],
    "kaas_host_alloc": [_u64, C.POINTER(_vp)],
    "kaas_host_free": [_vp],
    "kaas_host_register": [_vp, _u64],
    "kaas_host_unregister": [_vp],
    "kaas_memcpy_h2d_async": [_u64, _vp, _u64, _u64],
    "kaas_memcpy_d2h_async": [_vp, _u64, _u64, _u64],
    "kaas_memcpy_d2d_async": [_u64, _u64, _u64, _u64],
    "kaas_enable_peer": [C.c_int, C.c_int],
    "kaas_can_access_peer": [C.c_int, C.c_int, C.POINTER(C.c_int)],
    "kaas_memcpy_p2p_async": [_u64, C.c_int, _u64, C.c_int, _u64, _u64],
    "kaas_launch": [C.c_int, _u64, C.POINTER(LaunchDesc)],
    # descriptor tables go in as void*: a ctypes array or a numpy buffer's address
    "kaas_launch_batch": [C.c_int, _u64, C.c_void_p, C.c_int],
    "kaas_launch_batch_memo": [C.c_int, _u64, C.c_void_p, C.c_int, _u64],
    "kaas_launch_batch_timed": [C.c_int, _u64, C.c_void_p, C.c_int, _u64, _u64, _u64, _u64, _u64,
                                C.c_void_p, C.c_int],
    "kaas_launch_batch_ex": [C.c_int, _u64, C.c_void_p, C.c_int,
                             C.POINTER(StreamOut), C.c_int],
}

_lib = None
_lib_lock = threading.Lock()


def load(path: str | None = None) -> C.CDLL:
    """Load the shared library (cached).  Raises if it is missing."""
    global _lib
    lib = _lib
    if lib is not None:  # lock-free fast path (called on every native call)
        return lib
    with _lib_lock:
        if _lib is not None:
            return _lib
        p = path or os.environ.get("KAAS_B200_LIB", LIB_PATH)
        if not os.path.exists(p):
            raise DeviceError(f"{LIB_NAME} not built at {p}: run __graft_entry__.build()")
        lib = C.CDLL(p)
        for name, argtypes in EXPORTS.items():
            fn = getattr(lib, name)
            fn.argtypes = argtypes
            fn.restype = C.c_int
        _lib = lib
        return lib


def last_error() -> str:
    buf = C.create_string_buffer(1024)
    load().kaas_last_error(buf, len(buf))
    return buf.value.decode("utf-8", "replace")


def check(rc: int, what: str) -> None:
    """Map a C ABI status onto the KaaS error taxonomy."""
    if rc == 0:
        return
    msg = f"{what}: {last_error()}"
    if rc == KAAS_E_BOUNDS:
        raise BackendFaultError(msg)
    if rc == KAAS_E_ARITY:
        raise ArityMismatchError(msg)
    if rc == KAAS_E_UNKNOWN_KERNEL:
        raise UnknownKernelError(msg)
    raise DeviceError(msg, rc)


def call(name: str, *args) -> None:
    check(getattr(load(), name)(*args), name)


_FAST: dict = {}


def _fn(name: str):
    """The bound C function (hot paths: skip call()'s per-call lookup)."""
    f = _FAST.get(name)
    if f is None:
        f = _FAST[name] = getattr(load(), name)
    return f


def device_count() -> int:
    n = C.c_int(0)
    call("kaas_device_count", C.byref(n))
    return n.value


def device_info(dev: int) -> DeviceInfo:
    info = DeviceInfo()
    call("kaas_device_info_get", dev, C.byref(info))
    return info


def launch_counter() -> int:
    v = C.c_uint64(0)
    call("kaas_launch_counter", C.byref(v))
    return v.value


def device_check(dev: int) -> str | None:
    """None when ``dev`` is usable, else the sticky error's text."""
    rc = load().kaas_device_check(dev)
    return None if rc == 0 else f"{last_error()} (code {rc})"


def inject_fault(stream: "Stream") -> None:
    """Tests only: a trapping kernel on ``stream`` (poisons the context)."""
    call("kaas_inject_fault", stream.handle)


_inited: set[int] = set()
_init_lock = threading.Lock()


def init_device(dev: int) -> None:
    with _init_lock:
        if dev in _inited:
            return
        call("kaas_init_device", dev)
        _inited.add(dev)


def bind_thread(dev: int) -> None:
    """Make ``dev`` the calling thread's current device (a pool worker does
    this once at start; the C exports also bind each call's stream device)."""
    init_device(dev)
    call("kaas_init_device", dev)


class Stream:
    """A CUDA stream owned by one executor (plus its per-stream scratch)."""

    __slots__ = ("dev", "handle")

    def __init__(self, dev: int, priority: int = 0):
        init_device(dev)
        h = C.c_uint64(0)
        call("kaas_stream_create", dev, priority, C.byref(h))
        self.dev = dev
        self.handle = h.value

    def sync(self) -> None:
        call("kaas_stream_sync", self.handle)

    def wait(self, event: "Event") -> None:
        rc = _fn("kaas_stream_wait_event")(self.handle, event.handle)
        if rc:
            check(rc, "kaas_stream_wait_event")

    def destroy(self) -> None:
        if self.handle:
            call("kaas_stream_destroy", self.handle)
            self.handle = 0


class Event:
    __slots__ = ("dev", "handle")

    def __init__(self, dev: int, timing: bool = False):
        h = C.c_uint64(0)
        call("kaas_event_create", dev, 1 if timing else 0, C.byref(h))
        self.dev = dev
        self.handle = h.value

    def record(self, stream: Stream) -> "Event":
        rc = _fn("kaas_event_record")(self.handle, stream.handle)
        if rc:
            check(rc, "kaas_event_record")
        return self

    def sync(self) -> None:
        call("kaas_event_sync", self.handle)

    def done(self) -> bool:
        d = C.c_int(0)
        call("kaas_event_query", self.handle, C.byref(d))
        return bool(d.value)

    def elapsed_ms(self, end: "Event") -> float:
        ms = C.c_float(0.0)
        call("kaas_event_elapsed_ms", self.handle, end.handle, C.byref(ms))
        return float(ms.value)

    def destroy(self) -> None:
        if self.handle:
            call("kaas_event_destroy", self.handle)
            self.handle = 0

    def __del__(self):
        # CUDA releases an event's resources once pending work on it is done
        h = getattr(self, "handle", 0)
        if h and _lib is not None:
            try:
                _lib.kaas_event_destroy(h)
            except Exception:
                pass


def elapsed_many(pairs) -> list[float]:
    """cudaEventElapsedTime over (start, end) Event pairs in one crossing."""
    n = len(pairs)
    starts = (C.c_uint64 * n)(*(a.handle for a, _ in pairs))
    ends = (C.c_uint64 * n)(*(b.handle for _, b in pairs))
    out = (C.c_float * n)()
    call("kaas_event_elapsed_many", n, starts, ends, out)
    return list(out)


def malloc_async(stream: Stream, nbytes: int) -> int:
    p = C.c_uint64(0)
    call("kaas_malloc_async", stream.handle, nbytes, C.byref(p))
    return p.value


def free_async(stream: Stream, ptr: int) -> None:
    call("kaas_free_async", stream.handle, ptr)


def memset_async(ptr: int, value: int, nbytes: int, stream: Stream) -> None:
    call("kaas_memset_async", ptr, value, nbytes, stream.handle)


def h2d_async(dst: int, src_addr: int, nbytes: int, stream: Stream) -> None:
    rc = _fn("kaas_memcpy_h2d_async")(dst, src_addr, nbytes, stream.handle)
    if rc:
        check(rc, "kaas_memcpy_h2d_async")


def d2h_async(dst_addr: int, src: int, nbytes: int, stream: Stream) -> None:
    rc = _fn("kaas_memcpy_d2h_async")(dst_addr, src, nbytes, stream.handle)
    if rc:
        check(rc, "kaas_memcpy_d2h_async")


def d2d_async(dst: int, src: int, nbytes: int, stream: Stream) -> None:
    call("kaas_memcpy_d2d_async", dst, src, nbytes, stream.handle)


def p2p_async(dst: int, dst_dev: int, src: int, src_dev: int, nbytes: int,
              stream: Stream) -> None:
    call("kaas_memcpy_p2p_async", dst, dst_dev, src, src_dev, nbytes, stream.handle)


def enable_peer(dev: int, peer: int) -> bool:
    can = C.c_int(0)
    call("kaas_can_access_peer", dev, peer, C.byref(can))
    if not can.value:
        return False
    call("kaas_enable_peer", dev, peer)
    return True


def host_alloc(nbytes: int) -> int:
    p = C.c_void_p(0)
    call("kaas_host_alloc", nbytes, C.byref(p))
    return p.value or 0


def host_free(addr: int) -> None:
    call("kaas_host_free", C.c_void_p(addr))


def launch_batch_timed(dev: int, stream: Stream, descs, memo_key: int = 0, join_stream: Stream | None = None,
                       join_event: Event | None = None, ev_start: Event | None = None,
                       ev_end: Event | None = None, outs=None) -> None:
    """launch_batch with the join / kernel-span events in the same crossing
    (kaas_launch_batch_timed).  ``outs``: (desc_index, arg_index, host_addr,
    nbytes) write-backs that are complete once ``ev_end`` is (a fused Jacobi
    chain writes its last sweep there from the kernel; anything else is
    copied on ``stream`` after the batch)."""
    n = len(descs)
    ptr = descs.__array_interface__["data"][0] if isinstance(descs, np.ndarray) else descs
    arr, n_outs = None, 0
    if isinstance(outs, C.Array):  # a prebuilt StreamOut array (the caller keeps it current)
        arr, n_outs = outs, len(outs)
    elif outs:
        n_outs = len(outs)
        arr = (StreamOut * n_outs)()
        for i, (di, ai, addr, nb) in enumerate(outs):
            arr[i].desc_index, arr[i].arg_index = di, ai
            arr[i].out_stream, arr[i].host_dst, arr[i].bytes = stream.handle, addr, nb
    rc = _fn("kaas_launch_batch_timed")(dev, stream.handle, ptr, n, memo_key,
                                        join_stream.handle if join_event is not None else 0,
                                        join_event.handle if join_event is not None else 0,
                                        ev_start.handle if ev_start is not None else 0,
                                        ev_end.handle if ev_end is not None else 0, arr, n_outs)
    if rc:
        check(rc, "kaas_launch_batch_timed")


def launch_batch(dev: int, stream: Stream, descs, outs=None, memo_key: int = 0) -> None:
    """Enqueue LaunchDescs in order (ctypes array or DESC_DTYPE numpy array).

    ``outs``: optional list of (desc_index, arg_index, out_stream, host_addr,
    nbytes) progressive write-backs (kaas_launch_batch_ex).  ``memo_key``:
    nonzero promises ``descs`` has the content of the last call on this
    stream with the same key (kaas_launch_batch_memo)."""
    n = len(descs)
    if n == 0:
        return
    if isinstance(descs, np.ndarray):
        ptr = descs.__array_interface__["data"][0]
    else:
        ptr = descs
    if not outs:
        if memo_key:
            rc = _fn("kaas_launch_batch_memo")(dev, stream.handle, ptr, n, memo_key)
            if rc:
                check(rc, "kaas_launch_batch_memo")
        else:
            check(load().kaas_launch_batch(dev, stream.handle, ptr, n), "kaas_launch_batch")
        return
    arr = (StreamOut * len(outs))()
    for i, (di, ai, st, addr, nb) in enumerate(outs):
        arr[i].desc_index, arr[i].arg_index = di, ai
        arr[i].out_stream, arr[i].host_dst, arr[i].bytes = st.handle, addr, nb
    check(load().kaas_launch_batch_ex(dev, stream.handle, ptr, n, arr, len(outs)),
          "kaas_launch_batch_ex")


def is_available() -> bool:
    """True when the library loads and at least one CUDA device is visible."""
    try:
        return device_count() > 0
    except KaasError:
        return False
    except OSError:
        return False


_util_streams: dict[int, Stream] = {}
_util_lock = threading.Lock()


def util_stream(dev: int) -> Stream:
    """A per-device stream for synchronous helper copies (tests, snapshots)."""
    with _util_lock:
        s = _util_streams.get(dev)
        if s is None:
            s = _util_streams[dev] = Stream(dev)
        return s
