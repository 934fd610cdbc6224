"""GPU executor: the reference request lifecycle on one B200.

``GpuExecutor`` keeps the public surface of the reference ``Executor``
(``pkg/src/kaas/executor.py:215-436``): ``execute(req) -> KaasResponse``
(never raises for request-level failures), ``resolve_buffer``, ``stats()``,
``cache`` / ``clock`` / ``backend`` / ``requests_served`` attributes.

Split of work:

* host, synchronously, in request order -- everything that decides:
  validation, static checks, the 5-way ``resolve_buffer`` tree against the
  byte ledger (``cache.CacheState``), per-invocation bounds checks, virtual
  clock and IoStats.  These are the reference's own rules, so responses and
  cache states are bit-exact.
* device, asynchronously, on three streams per executor -- everything that
  moves or computes bytes:
    ``s_in``   H2D cache fills straight from pinned store objects
    ``s_exec`` zero-fills + the whole invocation list in ONE
               ``kaas_launch_batch`` crossing (Jacobi sweep runs fuse into one
               persistent launch)
    ``s_out``  D2H write-back into fresh pinned blobs adopted by the store
  linked by events (fills -> kernels -> flush).

Failure atomicity (``executor.py:371-384``): every failure the reference can
produce is detected on the host before the first kernel is enqueued, so a
failed request launches nothing and puts nothing; it leaves exactly the
cache side effects the reference leaves (evictions, completed fetches,
clean zero-filled outputs).

Device memory: entries are ``cudaMallocAsync`` allocations from the device
pool (pages retained).  A buffer dropped while the current request may still
touch it is freed only after the request's streams drain.
"""

from __future__ import annotations

import itertools
import threading
import os
import time

from collections import OrderedDict, deque
from dataclasses import dataclass, field, replace

import numpy as np

from . import native
from .api import (
    BufferArg,
    InvocationStats,
    IoStats,
    KaasRequest,
    KaasResponse,
    Status,
    validate_request,
)
from .cache import CacheState, DeviceBuffer
from .faults import (
    BufferBusyError,
    DeviceError,
    InvalidRequestError,
    KaasError,
    SizeMismatchError,
)
from .hoststore import PinnedBlob, PinnedStore
from .kernels import GpuKernel, KernelRegistry, default_registry, fill_desc
from .timing import TimingModel, VirtualClock


@dataclass(frozen=True)
class ExecutorConfig:
    """``executor.py:41-50`` plus the CUDA device ordinal."""

    capacity: int
    timing: TimingModel = field(default_factory=TimingModel)
    executor_id: int = 0
    debug: bool = False
    device: int = 0
    # device bytes for cGEMM's prepared operands of const inputs (outside the
    # ledger, which stays the reference's; None = 4x capacity, 0 = off)
    prepared_capacity: int | None = None
    # device-pool bytes to map at start-up (a server reserves its cache memory
    # once, so no request pays for growing the pool); 0 = grow on demand
    reserve_bytes: int = 0

    def __post_init__(self):
        if not isinstance(self.capacity, int) or self.capacity <= 0:
            raise ValueError(f"capacity must be a positive byte count, got {self.capacity!r}")


class GpuBackend:
    """Kernel lookup + pricing (``SimulatedBackend``, ``backend.py:246-266``);
    the launch itself goes through the executor's batched C-ABI call."""

    def __init__(self, registry: KernelRegistry | None = None,
                 timing: TimingModel | None = None):
        self.registry = registry if registry is not None else default_registry()
        self.timing = timing if timing is not None else TimingModel()

    def kernel(self, kernel_id: str) -> GpuKernel:
        return self.registry.get(kernel_id)


class _ReqStats:
    __slots__ = ("store_gets", "store_puts", "bytes_fetched", "bytes_flushed",
                 "cache_hits", "cache_misses")

    def __init__(self):
        self.store_gets = self.store_puts = 0
        self.bytes_fetched = self.bytes_flushed = 0
        self.cache_hits = self.cache_misses = 0

    def freeze(self) -> IoStats:
        return IoStats(self.store_gets, self.store_puts, self.bytes_fetched,
                       self.bytes_flushed, self.cache_hits, self.cache_misses)


class DeviceStats:
    """Measured (not virtual) device activity of one executor.

    A request's event spans are read lazily: ``complete()`` queues the
    request's events and the elapsed-time query (one C-ABI crossing, ~10 us)
    runs when a timing field is read or while the next request's kernels run
    -- not between a request's last event and its response."""

    __slots__ = ("requests", "_device_ms", "_last_device_ms", "_kernel_ms", "_last_kernel_ms",
                 "h2d_bytes", "_h2d_ms", "d2h_bytes", "p2p_bytes", "kernel_launches", "_pending",
                 "_release", "_lock", "host_ms")
    FIELDS = ("requests", "device_ms", "last_device_ms", "kernel_ms", "last_kernel_ms",
              "h2d_bytes", "h2d_ms", "d2h_bytes", "p2p_bytes", "kernel_launches", "host_ms")

    def __init__(self, release=None):
        self.requests = 0
        self._device_ms = 0.0
        self._last_device_ms = 0.0
        self._kernel_ms = 0.0      # time inside the batched invocation list
        self._last_kernel_ms = 0.0
        self.h2d_bytes = 0
        self._h2d_ms = 0.0         # time the H2D fill stream was busy (first fill -> last fill done)
        self.d2h_bytes = 0
        self.p2p_bytes = 0
        self.kernel_launches = 0
        # host time in begin() and complete() (decisions, enqueues, puts,
        # response), excluding the waits for the device: the per-request
        # Python/GIL work a pool of executors shares
        self.host_ms = 0.0
        self._pending: list = []   # (events, has_kernels, has_fills), all complete on the device
        self._release = release    # events -> the executor's pool once read
        self._lock = threading.Lock()  # the worker resolves while a reader may too

    def defer(self, events, has_kernels: bool, has_fills: bool) -> None:
        with self._lock:
            self._pending.append((events, has_kernels, has_fills))
            full = len(self._pending) >= 16
        if full:
            self.resolve()

    def resolve(self) -> None:
        if not self._pending:
            return
        with self._lock:
            self._resolve_locked()

    def _resolve_locked(self) -> None:
        pend = self._pending
        if not pend:
            return
        pairs = []
        for ev, hk, hf in pend:
            pairs.append((ev[0], ev[1]))
            if hk:
                pairs.append((ev[2], ev[3]))
            if hf:
                pairs.append((ev[4], ev[5]))
        spans = native.elapsed_many(pairs)  # one crossing for all queued requests
        self._pending = []
        i = 0
        for ev, hk, hf in pend:
            self._last_device_ms = spans[i]
            self._device_ms += spans[i]
            i += 1
            if hk:
                self._last_kernel_ms = spans[i]
                self._kernel_ms += spans[i]
                i += 1
            if hf:
                self._h2d_ms += spans[i]
                i += 1
            if self._release is not None:
                self._release(ev)

    def _get(name):
        def get(self):
            self.resolve()
            return getattr(self, name)
        return property(get)

    device_ms = _get("_device_ms")
    last_device_ms = _get("_last_device_ms")
    kernel_ms = _get("_kernel_ms")
    last_kernel_ms = _get("_last_kernel_ms")
    h2d_ms = _get("_h2d_ms")
    del _get

    def as_dict(self) -> dict:
        return {k: getattr(self, k) for k in self.FIELDS}


# keys naming one immutable descriptor table (kaas_launch_batch_memo); never reused
# dev A/B only: KAAS_DEV_NO_WB=1 turns the Jacobi in-kernel write-back off
_NO_WB = os.environ.get("KAAS_DEV_NO_WB") == "1"
_DESC_KEYS = itertools.count(1)


def _written_prefix(kernel_id: str, inv, w: int) -> int:
    """Bytes [0, n) that invocation ``inv`` of ``kernel_id`` writes into its
    argument ``w`` (coverage rules of backend.py:137-211 / kernels.py); 0 when
    not known to be a full prefix."""
    total = inv.dims.total_threads
    lits = [lit.value for lit in inv.literals]
    if kernel_id in ("vector_add", "saxpy") and w == 2:
        return 4 * max(0, min(total, lits[0]))
    if kernel_id == "fill" and w == 0:
        return 4 * max(0, min(total, lits[0]))
    if kernel_id == "reduce_sum" and w == 1:
        return 4
    if kernel_id == "matmul" and w == 2:
        return 4 * max(0, min(total, lits[0] * lits[1]))
    if kernel_id == "cgemm" and w == 2:
        return 8 * max(0, min(total, lits[0] * lits[1]))
    if kernel_id == "jacobi_sweep":
        if w == 3:
            return 4 * max(0, min(total, lits[0]))
        if w == 4:
            return 4
    return 0


class _Plan:
    """Everything about a request that does not depend on cache state.

    Validation, static checks, per-invocation bounds checks (resolved
    buffers always have the declared sizes), virtual compute time and the
    launch descriptors are pure functions of the request, so they are
    computed once per distinct request and replayed: a 500-sweep Jacobi
    request costs a few numpy ops on the host instead of ~4 ms of Python."""

    __slots__ = ("error", "kernels", "fail_at", "fail_exc", "advance_ns", "per_inv",
                 "template", "slots", "names", "dirty_names", "n", "stream_outs", "wb_outs", "wb_arr",
                 "wb_next", "prepared",
                 "last_ptrs", "last_descs", "last_key", "skip_zero")


class _LRU(OrderedDict):
    def __init__(self, cap: int):
        super().__init__()
        self.cap = cap

    def put(self, k, v):
        self[k] = v
        self.move_to_end(k)
        if len(self) > self.cap:
            self.popitem(last=False)


def _plan_key(req: KaasRequest):
    """Exact structural key of what a plan depends on: the buffer table and
    the invocation list.  Numeric fields carry their types (``4``, ``4.0``
    and ``True`` compare equal in Python, but validation tells them apart),
    floats are keyed by their exact bits (``0.0 == -0.0``), and the tuples
    are plain, so hashing and comparing run at C speed."""
    bufs = tuple([(b.name, b.size, type(b.size), b.direction, b.key, b.is_const,
                   type(b.is_const), b.is_ephemeral, type(b.is_ephemeral))
                  for b in req.buffers])
    out = []
    ap = out.append
    for i in req.invocations:
        d = i.dims
        ap((i.kernel_id, d.grid_x, d.grid_y, d.grid_z, d.block_x, d.block_y, d.block_z,
            type(d.grid_x), type(d.grid_y), type(d.grid_z),
            type(d.block_x), type(d.block_y), type(d.block_z),
            tuple([(lit.type, type(lit.value),
                    lit.value.hex() if type(lit.value) is float else lit.value)
                   for lit in i.literals]), i.args))
    return bufs, tuple(out)


class _Req:
    """One request between ``begin`` (decisions made, device work enqueued)
    and ``complete`` (device done, store puts, response)."""

    __slots__ = ("seq", "req", "response", "pending", "graveyard", "keepalive", "events",
                 "has_kernels", "has_fills", "streamed", "wb")

    def __init__(self, seq, req):
        self.seq = seq
        self.req = req
        self.response = None
        self.pending = []      # (key, blob, size) store puts, table order
        self.graveyard = []    # device pointers to free once this request's work is done
        self.keepalive = []    # host blobs referenced by this request's copies
        self.events = None     # (start, end, k0, k1, in0, in1)
        self.has_kernels = False
        self.has_fills = False
        self.streamed = {}
        self.wb = False        # streamed buffers written back on the exec stream (by the kernel)


class GpuExecutor:
    """Owns one device cache on one GPU; requests are decided strictly in
    arrival order and may overlap on the device (``begin`` / ``complete``)."""

    recycle_blocks = True  # device block free list (class-level switch for A/B runs)

    def __init__(self, config: ExecutorConfig, store, backend: GpuBackend | None = None,
                 time_requests: bool = True):
        self.config = config
        self.executor_id = config.executor_id
        self.store = store
        self.backend = backend if backend is not None else GpuBackend(timing=config.timing)
        self.device = config.device
        native.init_device(self.device)
        self.s_in = native.Stream(self.device)
        self.s_exec = native.Stream(self.device)
        self.s_out = native.Stream(self.device)
        self._ev_fill = native.Event(self.device)
        self._ev_exec = native.Event(self.device)
        self._ev_pool: list = []
        self.time_requests = time_requests
        self.cache = CacheState(config.capacity, debug=config.debug, on_drop=self._drop)
        if config.reserve_bytes > 0:
            # the pool keeps freed memory mapped (release threshold = max)
            p = native.malloc_async(self.s_exec, config.reserve_bytes)
            native.free_async(self.s_exec, p)
            self.s_exec.sync()
        self.clock = VirtualClock()
        self.total_hits = 0
        self.total_misses = 0
        self.requests_served = 0
        self.dev_stats = DeviceStats(release=self._ev_pool.append)
        self._pinned_store = isinstance(store, PinnedStore)
        self._req_seq = 0
        self._cur: _Req | None = None             # request being begun
        self._skip_zero: frozenset = frozenset()  # names whose zero-fill the plan proved dead
        self._inflight: OrderedDict[int, _Req] = OrderedDict()  # seq -> begun, not completed
        self._pending_puts: dict[str, int] = {}   # key -> seq of the request that will put it
        self.on_complete = None                   # callback(req_record, response) (pool)
        self.peers = None                         # PeerDirectory shared by a pool (peers.py)
        self._versioned = hasattr(store, "get_versioned")
        self._closed = False
        self._plans_by_id: _LRU = _LRU(256)     # id(req) -> (req, plan)
        self._plans_by_value: _LRU = _LRU(256)  # (buffers, invocations) -> plan
        self._plans_by_parts: _LRU = _LRU(256)  # (id(buffers), id(invocations)) -> plan
        pc = config.prepared_capacity
        if pc is None:
            # outside the ledger: 4x the ledger, but never more than half of
            # what the device has beyond it (several executors may share a GPU)
            total = native.device_info(self.device).total_mem
            pc = max(0, min(4 * config.capacity, (total - config.capacity) // 2))
        self._prep_cap = pc
        self._prep_bytes = 0
        self._skipped: list = []  # zero-fills elided for the request being begun
        self._blocks: dict[int, deque] = {}  # recycled device blocks by size (FIFO)
        self._block_bytes = 0
        self._block_cap = max(256 << 20, min(2 << 30, config.capacity // 2))
        # set when a CUDA fault left the device unusable (a sticky error): the
        # executor then answers Internal without touching the device, and a
        # pool's router stops placing requests here (service.py:71-78 analogue)
        self.poisoned: str | None = None
        self._timing_depth = 0  # host-time accounting (begin / complete may nest)
        self._wait_s = 0.0

    # -- device memory ------------------------------------------------------

    def _mark(self, buf: DeviceBuffer) -> None:
        buf.dev = self.device
        buf._req = self._req_seq

    def _alloc(self, buf: DeviceBuffer, stream: native.Stream) -> None:
        buf.ptr = self._dmalloc(buf.size, stream)
        buf.dev = self.device

    # Device blocks are recycled by exact size: a block whose last user has
    # completed on the device goes back to a per-executor free list instead
    # of cudaFreeAsync, and the next allocation of that size takes it
    # without a C-ABI crossing (a warm Jacobi request replaces 4 blocks).
    # The free list is outside the ledger (decisions never see it) and is
    # emptied before any allocation is allowed to fail.
    def _dmalloc(self, nbytes: int, stream: native.Stream) -> int:
        lst = self._blocks.get(nbytes)
        if lst:
            # first freed, first reused: a steady request stream gets the same
            # block for the same buffer every time, so its memoised launch
            # (descriptor table keyed by the buffer addresses) keeps hitting
            self._block_bytes -= nbytes
            return lst.popleft()
        try:
            return native.malloc_async(stream, nbytes)
        except DeviceError:
            if not self._block_bytes:
                raise
            self._release_blocks()
            return native.malloc_async(stream, nbytes)

    def _dfree(self, ptr: int, nbytes: int, stream: native.Stream) -> None:
        """``ptr``'s last user is done on the device (or ordered by stream waits)."""
        if self.poisoned is not None:
            return  # a faulted context frees nothing (it is torn down whole)
        if nbytes and self.recycle_blocks and self._block_bytes + nbytes <= self._block_cap:
            lst = self._blocks.get(nbytes)
            if lst is None:
                lst = self._blocks[nbytes] = deque()
            lst.append(ptr)
            self._block_bytes += nbytes
        else:
            native.free_async(stream, ptr)

    def _release_blocks(self) -> None:
        for lst in self._blocks.values():
            for ptr in lst:
                native.free_async(self.s_exec, ptr)
        self._blocks.clear()
        self._block_bytes = 0

    def _alloc_zeroed(self, buf: DeviceBuffer, name: str | None = None) -> None:
        self._alloc(buf, self.s_exec)
        if name is None or name not in self._skip_zero:
            native.memset_async(buf.ptr, 0, buf.size, self.s_exec)
        else:
            # the plan proved the first kernel overwrites every byte; if the
            # request fails before that kernel runs, begin() zero-fills it
            self._skipped.append(buf)
        if self._cur is None:  # a direct resolve_buffer call: contents final on return
            self.s_exec.sync()

    def _drop(self, buf: DeviceBuffer) -> None:
        """on_drop hook: an entry left the table or an ephemeral was freed.
        The allocation is released once the last request that used it is done."""
        if not buf.ptr:
            return
        self._fence_lends(buf)
        self._clear_derived(buf)
        ptr, buf.ptr = buf.ptr, 0
        self._free_after_user(buf, ptr, buf.size)

    def _free_after_user(self, buf: DeviceBuffer, ptr: int, nbytes: int, stream=None) -> None:
        owner = self._inflight.get(buf._req)
        if owner is None and self._cur is not None and buf._req == self._cur.seq:
            owner = self._cur
        if owner is not None:
            owner.graveyard.append((ptr, nbytes))  # released when the owner completes
        else:
            self._dfree(ptr, nbytes, self.s_in if stream is None else stream)

    # -- prepared operands ------------------------------------------------------
    # cGEMM's scaled 3xFP16 split of A and split + 4M expansion + transpose of B are
    # pure functions of a const input's bytes: they are kept beside the cache
    # entry, so a warm request skips the preparation pass.  They die with the
    # entry's contents (fill, kernel write, eviction); decisions are unaffected.

    def _clear_derived(self, buf: DeviceBuffer) -> None:
        buf._hits = 0
        d = buf._derived
        if not d:
            return
        buf._derived = None
        for ptr, nbytes, _ in d.values():
            self._prep_bytes -= nbytes
            # allocated and used on s_exec: free there too, so the pool can
            # hand the block straight to the next prepared operand
            self._free_after_user(buf, ptr, nbytes, self.s_exec)

    def _derived_slot(self, buf: DeviceBuffer, key, nbytes: int):
        """-> [ptr, nbytes, ready] for ``key`` on ``buf``, allocating (on the
        exec stream) within the prepared-operand budget; None when over it or
        when ``buf`` has not been reused yet."""
        d = buf._derived
        if d is not None:
            hit = d.get(key)
            if hit is not None:
                return hit
        # promote on reuse: an operand seen once (a cold fetch, or churn under
        # eviction) keeps using scratch; the first cache hit prepares it
        if buf._hits == 0 or self._prep_bytes + nbytes > self._prep_cap:
            return None
        try:
            ptr = self._dmalloc(nbytes, self.s_exec)
        except DeviceError:  # device memory short: this launch uses scratch instead
            return None
        slot = [ptr, nbytes, False]
        self._prep_bytes += nbytes
        if d is None:
            buf._derived = d = {}
        d[key] = slot
        return slot

    def _fence_lends(self, buf: DeviceBuffer) -> None:
        """Withdraw ``buf`` from the peer directory and order any later free
        or rewrite of it after every peer copy still reading it."""
        if self.peers is None or buf.key is None:
            return
        self.peers.withdraw(self.executor_id, buf)
        for ev in self.peers.take_lends(buf):
            self.s_in.wait(ev)
            self.s_exec.wait(ev)

    def _events(self):
        if self._ev_pool:
            return self._ev_pool.pop()
        return tuple(native.Event(self.device, timing=True) for _ in range(6))

    def _wait_for_user(self, buf: DeviceBuffer) -> None:
        """A fill is about to overwrite ``buf`` in place: order it after every
        in-flight request that may still read or copy it."""
        owner = self._inflight.get(buf._req)
        if owner is not None and owner is not self._cur:
            self.s_in.wait(owner.events[1])

    # -- buffer resolution (executor.py:233-316) ------------------------------

    def resolve_buffer(self, arg: BufferArg, stats: _ReqStats | None = None) -> DeviceBuffer:
        if stats is None:
            stats = _ReqStats()
        cache = self.cache

        if arg.is_ephemeral:
            cache.evict_until(arg.size)
            buf = cache.alloc_ephemeral(arg.size)
            self._mark(buf)
            self._alloc_zeroed(buf, arg.name)
            return buf

        cached = cache.entries.get(arg.key)

        if arg.is_const:
            if cached is not None:
                if cached.size != arg.size:
                    raise SizeMismatchError(
                        f"buffer {arg.name!r}: cached object under {arg.key!r} is"
                        f" {cached.size} bytes, request declares {arg.size}")
                stats.cache_hits += 1
                cached._hits += 1
                cache.pin(cached)
                cache.touch(cached)
                cached.is_const = True
                self._mark(cached)
                return cached
            cache.evict_until(arg.size)
            buf = DeviceBuffer(arg.key, arg.size, is_const=True)
            self._fetch_into(buf, arg, stats)
            cache.insert(buf)
            cache.pin(buf)
            return buf

        if arg.direction == "output":
            if cached is not None:
                if cached.pinned > 0:
                    raise BufferBusyError(
                        f"buffer {arg.name!r}: key {arg.key!r} pinned elsewhere")
                cache.remove(arg.key)
            cache.evict_until(arg.size)
            buf = DeviceBuffer(arg.key, arg.size, is_const=False)
            self._mark(buf)
            self._alloc_zeroed(buf, arg.name)
            stats.cache_misses += 1
            cache.insert(buf)
            cache.pin(buf)
            return buf

        # non-const input / inout: always re-fetched
        if cached is not None and cached.pinned > 0:
            raise BufferBusyError(f"buffer {arg.name!r}: key {arg.key!r} pinned elsewhere")
        if cached is not None and cached.size == arg.size:
            self._fetch_into(cached, arg, stats)  # overwrite in place
            cached.is_const = False
            cache.pin(cached)
            cache.touch(cached)
            return cached
        if cached is not None:
            cache.remove(arg.key)
        cache.evict_until(arg.size)
        buf = DeviceBuffer(arg.key, arg.size, is_const=False)
        self._fetch_into(buf, arg, stats)
        cache.insert(buf)
        cache.pin(buf)
        return buf

    def _fetch_into(self, buf: DeviceBuffer, arg: BufferArg, stats: _ReqStats) -> None:
        owner = self._pending_puts.get(arg.key)
        if owner is not None:  # read-your-writes: that put must land first
            self.complete(through=owner)
        if self._versioned:
            payload, version = self.store.get_versioned(arg.key)  # NotFound propagates
        else:
            payload, version = self.store.get(arg.key), None
        if len(payload) != arg.size:
            raise SizeMismatchError(
                f"buffer {arg.name!r}: store object {arg.key!r} is"
                f" {len(payload)} bytes, request declares {arg.size}")
        cur = self._cur
        standalone = cur is None  # resolve_buffer called directly (executor.py:233 API)
        if standalone:
            cur = _Req(0, None)
        if buf.ptr:
            self._wait_for_user(buf)
            self._fence_lends(buf)
            self._clear_derived(buf)
        self._mark(buf)
        if not buf.ptr:
            self._alloc(buf, self.s_in)
        if self.time_requests and not cur.has_fills and cur.events is not None:
            cur.events[4].record(self.s_in)
        cur.has_fills = True
        borrowed = False
        if self.peers is not None and version is not None:
            def copy_from_peer(src, ready):
                if ready is not None:
                    self.s_in.wait(ready)
                native.p2p_async(buf.ptr, self.device, src.ptr, src.dev, arg.size, self.s_in)
                return native.Event(self.device).record(self.s_in)
            borrowed = self.peers.borrow(arg.key, version, self.executor_id, copy_from_peer)
        if borrowed:
            self.dev_stats.p2p_bytes += arg.size
        else:
            src = payload if isinstance(payload, PinnedBlob) else PinnedBlob.from_bytes(payload)
            native.h2d_async(buf.ptr, src.addr, arg.size, self.s_in)
            cur.keepalive.append(src)
            self.dev_stats.h2d_bytes += arg.size
        if self.peers is not None and version is not None:
            if buf._ready is None:
                buf._ready = native.Event(self.device)
            buf._ready.record(self.s_in)
            self.peers.publish(self.executor_id, buf, version, buf._ready)
        buf.dirty = False
        if standalone:  # no request owns the copy: finish it before returning
            self.s_in.sync()
            cur.keepalive.clear()
        self.clock.advance_ns(self.backend.timing.fetch_time_ns(arg.size))
        stats.store_gets += 1
        stats.bytes_fetched += arg.size
        stats.cache_misses += 1

    # -- request planning -----------------------------------------------------

    def _plan(self, req: KaasRequest) -> _Plan:
        """Plans depend on the buffer table and invocation list only (the
        request id matters just for its own validity check), so a client
        that rebuilds the same request each call still hits the cache."""
        hit = self._plans_by_id.get(id(req))
        if hit is not None and hit[0] is req:
            return hit[1]
        if not isinstance(req.request_id, str) or not req.request_id:
            return self._build_plan(req)  # invalid id: never cached
        # a client resending one kernel graph under new request ids reuses
        # the (immutable) buffer and invocation tuples: O(1) by identity
        parts = (id(req.buffers), id(req.invocations))
        hit = self._plans_by_parts.get(parts)
        if hit is not None and hit[0] is req.buffers and hit[1] is req.invocations:
            self._plans_by_id.put(id(req), (req, hit[2]))
            return hit[2]
        try:
            key = _plan_key(req)
            plan = self._plans_by_value.get(key)
        except TypeError:  # unhashable field values: plan without caching
            return self._build_plan(req)
        if plan is None:
            plan = self._build_plan(req)
            self._plans_by_value.put(key, plan)
        self._plans_by_id.put(id(req), (req, plan))
        # strong references keep the ids from being recycled while cached
        self._plans_by_parts.put(parts, (req.buffers, req.invocations, plan))
        return plan

    def _build_plan(self, req: KaasRequest) -> _Plan:
        p = _Plan()
        p.error = None
        p.last_ptrs = p.last_descs = None
        p.last_key = 0
        p.skip_zero = frozenset()
        violations = validate_request(req)
        if violations:
            p.error = Status.make_error("InvalidRequest", "; ".join(violations))
            return p
        try:  # static checks (executor.py:331-345)
            kernels = []
            for inv in req.invocations:
                kernel = self.backend.kernel(inv.kernel_id)
                kernel.check_arity(inv.literals, len(inv.args))
                for idx in kernel.writes:
                    arg = req.by_name[inv.args[idx]]
                    if not arg.is_ephemeral and arg.direction == "input":
                        raise InvalidRequestError(
                            f"kernel {inv.kernel_id!r} writes to read-only"
                            f" buffer {arg.name!r}")
                kernels.append(kernel)
        except KaasError as exc:
            p.error = Status.make_error(exc.kind, exc.message)
            return p
        p.kernels = kernels
        names = [b.name for b in req.referenced_buffers()]
        slot_of = {nm: i for i, nm in enumerate(names)}
        by_name = req.by_name
        timing = self.backend.timing
        n = len(req.invocations)
        descs = (native.LaunchDesc * n)() if n else None
        slots = np.full((n, native.MAX_ARGS), len(names), dtype=np.int64)
        per_inv, dirty, advance = [], [], 0
        p.fail_at, p.fail_exc = None, None
        for i, (inv, kernel) in enumerate(zip(req.invocations, kernels)):
            sizes = [by_name[nm].size for nm in inv.args]
            try:
                fma = kernel.plan(inv.dims, inv.literals, sizes)
            except KaasError as exc:  # BackendFault at invocation i
                p.fail_at, p.fail_exc = i, exc
                break
            compute_ns = timing.compute_time_ns(fma)
            overhead_ns = timing.launch_overhead_ns()
            advance += overhead_ns + compute_ns
            fill_desc(descs[i], kernel, inv.dims, inv.literals, [0] * len(sizes), sizes)
            for j, nm in enumerate(inv.args):
                slots[i, j] = slot_of[nm]
            for idx in kernel.writes:
                nm = inv.args[idx]
                if not by_name[nm].is_ephemeral and nm not in dirty:
                    dirty.append(nm)
            per_inv.append(InvocationStats(inv.kernel_id, compute_ns, overhead_ns))
        # outputs a kernel can write back progressively while it still runs:
        # a cgemm's C that is keyed (flushed at the end) and not rewritten later
        outs = []
        if p.fail_at is None:
            for i, (inv, kernel) in enumerate(zip(req.invocations, kernels)):
                if kernel.kernel_id != "cgemm":
                    continue
                nm = inv.args[2]
                if by_name[nm].is_ephemeral:
                    continue
                later = any(inv2.args[w] == nm for inv2, k2 in
                            zip(req.invocations[i + 1:], kernels[i + 1:]) for w in k2.writes)
                if not later and all(o[2] != nm for o in outs):
                    outs = [o for o in outs if o[2] != nm] + [(i, 2, nm)]
        p.stream_outs = tuple(outs)
        # a request ending in a jacobi_sweep: its keyed x_out / resid are
        # written back to their host blobs by the chain kernel itself (no D2H
        # copy after it; kaas_launch_batch_timed copies when it cannot)
        wb = []
        if (p.fail_at is None and req.invocations and kernels[-1].kernel_id == "jacobi_sweep" and not outs
                and not _NO_WB):
            last = req.invocations[-1]
            n_ = last.literals[0].value
            for ai, nbytes in ((3, 4 * n_), (4, 4)):
                nm = last.args[ai]
                arg = by_name[nm]
                # the kernel writes exactly x[0:n] / the one residual: a
                # larger buffer's tail must come from the device copy
                if (not arg.is_ephemeral and arg.key is not None and arg.size == nbytes
                        and all(w[2] != nm for w in wb)):
                    wb.append((len(req.invocations) - 1, ai, nm))
        p.wb_outs = tuple(wb)
        p.wb_arr = None   # native.StreamOut array for wb_outs, built on first launch
        p.wb_next = None  # host blobs for the next launch, allocated after this one
        # operands whose prepared forms may be cached: const inputs the request
        # does not rewrite -- cgemm's split A / expanded B, matmul's Bt
        prep = []
        if p.fail_at is None:
            for i, (inv, kernel) in enumerate(zip(req.invocations, kernels)):
                if kernel.kernel_id == "matmul":
                    n_, m_, k_ = (lit.value for lit in inv.literals)
                    if n_ * m_ * k_ == 0 or k_ % 4 or inv.dims.total_threads == 0:
                        continue
                    arg = by_name[inv.args[1]]
                    if arg.is_const and not arg.is_ephemeral and arg.name not in dirty:
                        prep.append((i, None, (arg.name, ("mm", k_, m_), 4 * m_ * k_)))
                    continue
                if kernel.kernel_id != "cgemm":
                    continue
                n_, m_, k_ = (lit.value for lit in inv.literals)
                if n_ * m_ * k_ == 0 or inv.dims.total_threads == 0:
                    continue  # nothing is computed, so nothing would be prepared
                # fp16 hi/lo planes (rows of 2k rounded up to 64) + 4 B of
                # scale max-bits per row of A / complex column of B
                # (cgemm_prepared_bytes, csrc/kaas_internal.cuh)
                ldk = (2 * k_ + 63) // 64 * 64
                sides = []
                for j, nbytes in ((0, 4 * n_ * ldk + 4 * n_), (1, 8 * m_ * ldk + 4 * m_)):
                    arg = by_name[inv.args[j]]
                    ok = arg.is_const and not arg.is_ephemeral and arg.name not in dirty
                    sides.append((arg.name, ("cg", j, n_, m_, k_), nbytes) if ok else None)
                if any(sides):
                    prep.append((i, sides[0], sides[1]))
        p.prepared = tuple(prep)
        # new outputs / ephemerals whose zero-fill no one can observe: the
        # first invocation touching them overwrites every byte without
        # reading them first (a planned BackendFault keeps every zero-fill:
        # never-written outputs stay cached as zeros)
        skip = set()
        if p.fail_at is None:
            seen = set()
            for inv, kernel in zip(req.invocations, kernels):
                written = {inv.args[w]: _written_prefix(kernel.kernel_id, inv, w) for w in kernel.writes}
                for j, nm in enumerate(inv.args):
                    if nm in seen:
                        continue
                    seen.add(nm)
                    arg = by_name[nm]
                    if arg.is_const or not (arg.is_ephemeral or arg.direction == "output"):
                        continue
                    reads = any(nm == a for jj, a in enumerate(inv.args) if jj not in kernel.writes)
                    if not reads and written.get(nm, 0) >= arg.size:
                        skip.add(nm)
        p.skip_zero = frozenset(skip)
        p.advance_ns = advance
        p.per_inv = tuple(per_inv)
        p.dirty_names = tuple(dirty)
        p.names = tuple(names)
        p.n = n if p.fail_at is None else 0
        p.slots = slots
        p.template = (np.frombuffer(bytes(descs), dtype=native.DESC_DTYPE).copy()
                      if n else None)
        return p

    # -- request lifecycle (executor.py:320-425) ------------------------------

    def execute(self, req: KaasRequest) -> KaasResponse:
        """Run one request to completion (the reference's synchronous call)."""
        rec = self.begin(req)
        if isinstance(rec, KaasResponse):
            return rec
        self.complete(through=rec.seq)
        return rec.response

    def begin(self, req: KaasRequest):
        """Make every decision for ``req`` and enqueue its device work (see
        ``_begin``); host time is accounted in ``dev_stats.host_ms``."""
        if self._timing_depth:
            return self._begin(req)
        self._timing_depth += 1
        t = time.perf_counter()
        self._wait_s = 0.0
        try:
            return self._begin(req)
        finally:
            self._timing_depth -= 1
            self.dev_stats.host_ms += (time.perf_counter() - t - self._wait_s) * 1e3

    def _begin(self, req: KaasRequest):
        """Make every decision for ``req`` and enqueue its device work.

        Returns the finished ``KaasResponse`` when the request fails on the
        host (nothing enqueued), else an in-flight record whose response is
        produced by ``complete``.  Decisions, ledger, ticks, virtual time and
        statistics are final here -- exactly as if the reference had run the
        request -- so requests begun later see the same cache state."""
        t0 = self.clock.now_ns
        stats = _ReqStats()
        if self.poisoned is not None:
            return self._finish(req, stats, t0, Status.make_error(
                "Internal", f"device {self.device} is unusable after a fault: {self.poisoned}"))
        plan = self._plan(req)
        if plan.error is not None:
            return self._finish(req, stats, t0, plan.error)

        self._req_seq += 1
        self._skip_zero = plan.skip_zero
        self._skipped = []
        rec = _Req(self._req_seq, req)
        self._cur = rec
        resolved: dict[str, DeviceBuffer] = {}
        ephemerals: list[DeviceBuffer] = []
        try:
            rec.events = ev = self._events()
            if self.time_requests:
                # the request's first device op: its fills follow on s_in, its
                # kernels wait on the fills' join (recorded on s_in later) and
                # its flush waits on the kernels, so every span is ordered
                # after this event without further cross-stream waits
                ev[0].record(self.s_in)
            by_name = req.by_name
            for nm in plan.names:
                arg = by_name[nm]
                buf = self.resolve_buffer(arg, stats)
                resolved[nm] = buf
                if arg.is_ephemeral:
                    ephemerals.append(buf)
            self._skip_zero = frozenset()
            self._launch(rec, plan, resolved)
            self._enqueue_flush(rec, plan.names, resolved, stats)
        except KaasError as exc:
            if isinstance(exc, DeviceError):
                self._check_poison()
            self._skip_zero = frozenset()
            # the kernel that would have overwritten these never runs: they
            # must read as zeros, like the reference's fresh allocations
            # (a clean output entry survives the failure)
            for buf in self._skipped:
                if buf.ptr and self.poisoned is None:
                    native.memset_async(buf.ptr, 0, buf.size, self.s_exec)
            self._skipped = []
            # a host-detected failure enqueued no kernels; drain so the
            # request's fills/zero-fills finish before its buffers are freed
            self._cur = None
            self.complete()
            self._drain_streams_quietly()
            self._release(resolved, ephemerals, drop_dirty=True)
            for ptr, nbytes in rec.graveyard:
                self._dfree(ptr, nbytes, self.s_exec)
            if rec.events is not None:
                self._ev_pool.append(rec.events)
            return self._finish(req, stats, t0, Status.make_error(exc.kind, exc.message))
        self._release(resolved, ephemerals, drop_dirty=False)
        for key, _, _, _ in rec.pending:
            self._pending_puts[key] = rec.seq
        rec.response = self._finish(req, stats, t0, Status.make_ok(), list(plan.per_inv))
        self._inflight[rec.seq] = rec
        self._cur = None
        return rec

    def complete(self, through: int | None = None, block: bool = True) -> int:
        """Finish in-flight requests in order: wait for the device, put the
        flushed objects, release deferred frees.  ``through`` = last seq to
        finish (all when None).  With ``block=False`` only requests whose
        device work is already done are finished.  Returns how many."""
        if self._timing_depth:
            return self._complete(through, block)
        self._timing_depth += 1
        t = time.perf_counter()
        self._wait_s = 0.0
        try:
            return self._complete(through, block)
        finally:
            self._timing_depth -= 1
            self.dev_stats.host_ms += (time.perf_counter() - t - self._wait_s) * 1e3

    def _complete(self, through: int | None, block: bool) -> int:
        done = 0
        while self._inflight:
            seq, rec = next(iter(self._inflight.items()))
            if through is not None and seq > through:
                break
            ev = rec.events
            if not block:
                try:
                    if not ev[1].done():
                        break
                except DeviceError:
                    pass  # faulted: the sync below reports it for this request
            try:
                tw = time.perf_counter()
                ev[1].sync()
                self._wait_s += time.perf_counter() - tw
            except DeviceError as exc:
                # the device faulted under this request: nothing it computed
                # may reach the store; it (and every later one) fails in band
                self._check_poison()
                rec.pending = []
                rec.response = replace(rec.response, per_invocation=(),
                                       status=Status.make_error("Internal", str(exc)))
            for key, blob, size, buf in rec.pending:
                if self._pinned_store:
                    version = self.store.put_owned(key, blob)
                else:
                    version = self.store.put(key, bytes(blob))
                if self._pending_puts.get(key) == seq:
                    del self._pending_puts[key]
                self.dev_stats.d2h_bytes += size
                # the cached copy now equals the object the store serves
                if (self.peers is not None and isinstance(version, int) and buf.ptr
                        and self.cache.entries.get(key) is buf and not buf.dirty):
                    self.peers.publish(self.executor_id, buf, version, None)
            for ptr, nbytes in rec.graveyard:
                self._dfree(ptr, nbytes, self.s_exec)
            self.dev_stats.requests += 1
            del self._inflight[seq]
            if self.time_requests and self.poisoned is None:  # spans read later (DeviceStats.resolve)
                self.dev_stats.defer(ev, rec.has_kernels, rec.has_fills)
            else:
                self._ev_pool.append(ev)
            rec.keepalive.clear()
            done += 1
            if self.on_complete is not None:
                self.on_complete(rec, rec.response)
        return done

    @property
    def inflight(self) -> int:
        return len(self._inflight)

    def _launch(self, rec: _Req, plan: _Plan, resolved) -> None:
        """Replay the plan: clock, dirty marks, one batched enqueue.  On a
        planned BackendFault the clock and dirty marks stop where the
        reference's would and nothing is enqueued (the failed request's
        kernel effects are unobservable: every buffer they could write is
        dropped or ephemeral)."""
        self.clock.advance_ns(plan.advance_ns)
        for nm in plan.dirty_names:
            b = resolved[nm]
            b.dirty = True
            self._fence_lends(b)  # a kernel is about to rewrite it
            self._clear_derived(b)
        if plan.fail_at is not None:
            raise plan.fail_exc
        ev = rec.events
        timed = self.time_requests
        # the usual launch (no stream-outs): the fills' join, the kernel span
        # and the launch in one C crossing (kaas_launch_batch_timed)
        one_call = bool(plan.n) and not plan.stream_outs
        if timed and rec.has_fills and not one_call:
            ev[5].record(self.s_in)
        if plan.n:
            ptrs = tuple(resolved[nm].ptr for nm in plan.names)
            memo_key = 0
            if not plan.prepared and ptrs == plan.last_ptrs:
                # the pool handed back the same blocks as last time (the usual
                # steady state): the 500-descriptor table is already built --
                # kaas_launch_batch copies what it needs before returning --
                # and its key lets the C side relaunch a fused chain as is
                descs = plan.last_descs
                memo_key = plan.last_key
            else:
                table = np.fromiter(ptrs, dtype=np.uint64, count=len(ptrs))
                table = np.append(table, np.uint64(0))
                descs = plan.template.copy()
                descs["ptrs"] = table[plan.slots]
                if not plan.prepared:
                    plan.last_ptrs, plan.last_descs = ptrs, descs
                    plan.last_key = memo_key = next(_DESC_KEYS)
            filled = self._attach_prepared(plan, descs, resolved) if plan.prepared else ()
            if one_call:
                wb = None
                if plan.wb_outs:
                    # the write-back blobs were allocated after the previous
                    # launch of this plan: nothing but two field stores here
                    blobs = plan.wb_next or [PinnedBlob(resolved[nm].size) for _, _, nm in plan.wb_outs]
                    plan.wb_next = None
                    wb = plan.wb_arr
                    if wb is None:
                        wb = plan.wb_arr = (native.StreamOut * len(plan.wb_outs))()
                        for o, (di, ai, nm) in enumerate(plan.wb_outs):
                            wb[o].desc_index, wb[o].arg_index = di, ai
                            wb[o].out_stream, wb[o].bytes = self.s_exec.handle, resolved[nm].size
                    for o, (_, _, nm) in enumerate(plan.wb_outs):
                        blob = blobs[o]
                        rec.keepalive.append(blob)
                        rec.streamed[nm] = blob
                        wb[o].host_dst = blob.addr
                    rec.wb = True
                # s_exec waits for everything enqueued on s_in so far (the fills)
                native.launch_batch_timed(self.device, self.s_exec, descs, memo_key, self.s_in,
                                          ev[5] if timed and rec.has_fills else self._ev_fill,
                                          ev[2] if timed else None, ev[3] if timed else None, wb)
                if plan.wb_outs:  # the next launch's write-back blobs, off its critical path
                    plan.wb_next = [PinnedBlob(resolved[nm].size) for _, _, nm in plan.wb_outs]
                self.dev_stats.resolve()  # earlier requests' spans, while this one runs
                for slot in filled:
                    slot[2] = True  # later launches on s_exec are ordered after the fill
                rec.has_kernels = True
                self.dev_stats.kernel_launches += plan.n
                return
            if self.time_requests and rec.has_fills:
                self.s_exec.wait(ev[5])  # recorded on s_in just above: the fills' end
            else:
                self._ev_fill.record(self.s_in)
                self.s_exec.wait(self._ev_fill)
            outs = []
            for di, ai, nm in plan.stream_outs:
                buf = resolved[nm]
                blob = PinnedBlob(buf.size)
                rec.keepalive.append(blob)
                rec.streamed[nm] = blob
                outs.append((di, ai, self.s_out, blob.addr, buf.size))
            if self.time_requests:
                ev[2].record(self.s_exec)
            native.launch_batch(self.device, self.s_exec, descs, outs, memo_key)
            self.dev_stats.resolve()  # earlier requests' spans, while this one runs
            for slot in filled:
                slot[2] = True  # later launches on s_exec are ordered after the fill
            if self.time_requests:
                ev[3].record(self.s_exec)
            rec.has_kernels = True
            self.dev_stats.kernel_launches += plan.n

    def _attach_prepared(self, plan: _Plan, descs, resolved):
        filled = []
        for i, *sides in plan.prepared:
            flags = 0
            for j, side in enumerate(sides):
                if side is None:
                    continue
                name, key, nbytes = side
                slot = self._derived_slot(resolved[name], key, nbytes)
                if slot is None:
                    continue
                if key[0] == "mm":  # matmul: Bt in ptrs[3]
                    descs["ptrs"][i, 3] = slot[0]
                    descs["sizes"][i, 3] = nbytes
                    flags |= native.F_MM_BT_USE if slot[2] else native.F_MM_BT_FILL
                    if not slot[2]:
                        filled.append(slot)
                    continue
                descs["ptrs"][i, 3 + j] = slot[0]
                descs["sizes"][i, 3 + j] = nbytes
                if slot[2]:
                    flags |= (native.F_CG_A_USE, native.F_CG_B_USE)[j]
                else:
                    flags |= (native.F_CG_A_FILL, native.F_CG_B_FILL)[j]
                    filled.append(slot)
            descs["flags"][i] = flags
        return filled

    def _enqueue_flush(self, rec: _Req, names, resolved, stats: _ReqStats) -> None:
        """Write-back of dirty keyed buffers in table order
        (executor.py:371-380): the D2H copies are enqueued now, the puts
        happen in ``complete``; virtual time, IoStats and the clean marks are
        final now, as the next request's decisions depend on them."""
        # Alone on the executor (nothing else in flight), the copies go on the
        # exec stream right behind the kernels: no cross-stream hand-over
        # between the last kernel and the write-back (a warm Jacobi request's
        # kernel-end -> flush-done tail was 13 us).  With requests pipelined,
        # they go on the copy-out stream so the next request's kernels
        # overlap them.
        alone = rec.wb or (not rec.streamed and len(self._inflight) == 0)
        fs = self.s_exec if alone else self.s_out
        if rec.has_fills and not rec.has_kernels:
            # no kernel joined the fills: the request's end event must not
            # come before them (complete() releases the fills' host sources)
            join = rec.events[5] if self.time_requests else self._ev_fill
            join.record(self.s_in)
            fs.wait(join)
        if alone:
            pass
        elif self.time_requests and rec.has_kernels:
            self.s_out.wait(rec.events[3])  # _launch recorded it on s_exec after the batch, just now
        else:
            self._ev_exec.record(self.s_exec)
            self.s_out.wait(self._ev_exec)
        for nm in names:
            buf = resolved[nm]
            # only non-const keyed buffers get dirty, and validation forbids
            # binding one non-const key twice, so no buffer appears twice here
            if buf.dirty:
                blob = rec.streamed.get(nm)
                if blob is None:
                    blob = PinnedBlob(buf.size)
                    native.d2h_async(blob.addr, buf.ptr, buf.size, fs)
                rec.pending.append((buf.key, blob, buf.size, buf))
                self.clock.advance_ns(self.backend.timing.flush_time_ns(buf.size))
                stats.store_puts += 1
                stats.bytes_flushed += buf.size
                buf.dirty = False
        rec.events[1].record(fs)

    def _check_poison(self) -> None:
        if self.poisoned is None:
            self.poisoned = native.device_check(self.device)

    def _drain_streams_quietly(self) -> None:
        """Failure-path drain: a sticky device error must not escape execute."""
        try:
            self.s_in.sync()
            self.s_exec.sync()
            self.s_out.sync()
        except KaasError:
            pass

    def _release(self, resolved, ephemerals, drop_dirty: bool) -> None:
        for buf in ephemerals:
            self.cache.free_ephemeral(buf)
        for buf in resolved.values():
            if buf.key is None:
                continue
            self.cache.unpin(buf)
        if drop_dirty:
            for buf in resolved.values():
                if buf.key is not None and buf.dirty and buf.key in self.cache.entries:
                    self.cache.remove(buf.key)
                    buf.dirty = False

    def _finish(self, req, stats, t0, status, per_inv=None) -> KaasResponse:
        self.total_hits += stats.cache_hits
        self.total_misses += stats.cache_misses
        self.requests_served += 1
        if self.config.debug:
            self.cache.check_accounting()
        return KaasResponse(
            request_id=req.request_id,
            status=status,
            per_invocation=tuple(per_inv or ()),
            io_stats=stats.freeze(),
            simulated_total_time=self.clock.now_ns - t0,
        )

    def stats(self) -> dict:
        return {
            "executor_id": self.executor_id,
            "used_bytes": self.cache.used_bytes,
            "entries": len(self.cache.entries),
            "cache_hits": self.total_hits,
            "cache_misses": self.total_misses,
            "requests": self.requests_served,
            "clock_ns": self.clock.now_ns,
        }

    def device_stats(self) -> dict:
        d = self.dev_stats.as_dict()
        d["device"] = self.device
        return d

    def close(self) -> None:
        """Finish in-flight work, release every device allocation and the streams."""
        if self._closed:
            return
        self._closed = True
        try:
            self.complete()
        except KaasError:
            pass
        if self.poisoned is not None:
            # a faulted context: every device call fails; its memory goes
            # with the process (or a device reset), only the ledger is cleared
            self.cache.entries.clear()
            return
        self._drain_streams_quietly()
        for key in list(self.cache.entries):
            buf = self.cache.entries[key]
            self._clear_derived(buf)
            buf._pinned = 0
            buf._dirty = False
            self.cache.remove(key)
        self._release_blocks()
        self._drain_streams_quietly()
        for s in (self.s_in, self.s_exec, self.s_out):
            s.sync()
            s.destroy()
        for e in (self._ev_fill, self._ev_exec):
            e.destroy()
        try:
            self.dev_stats.resolve()  # returns the queued requests' events to the pool
        except Exception:  # noqa: BLE001 -- a faulted context: the events are destroyed below anyway
            self._ev_pool.extend(ev for ev, _, _ in self.dev_stats._pending)
            self.dev_stats._pending = []
        for evs in self._ev_pool:
            for e in evs:
                e.destroy()


# reference-compatible name
Executor = GpuExecutor
