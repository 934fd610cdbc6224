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

from dataclasses import dataclass, field

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
    """Measured (not virtual) device activity of one executor."""

    __slots__ = ("requests", "device_ms", "last_device_ms", "h2d_bytes", "d2h_bytes",
                 "p2p_bytes", "kernel_launches")

    def __init__(self):
        self.requests = 0
        self.device_ms = 0.0
        self.last_device_ms = 0.0
        self.h2d_bytes = 0
        self.d2h_bytes = 0
        self.p2p_bytes = 0
        self.kernel_launches = 0

    def as_dict(self) -> dict:
        return {k: getattr(self, k) for k in self.__slots__}


class GpuExecutor:
    """Owns one device cache on one GPU and runs requests one at a time."""

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
        self._ev_start = native.Event(self.device, timing=True)
        self._ev_end = native.Event(self.device, timing=True)
        self.time_requests = time_requests
        self.cache = CacheState(config.capacity, debug=config.debug, on_drop=self._drop)
        self.clock = VirtualClock()
        self.total_hits = 0
        self.total_misses = 0
        self.requests_served = 0
        self.dev_stats = DeviceStats()
        self._pinned_store = isinstance(store, PinnedStore)
        self._req_seq = 0
        self._graveyard: list[int] = []   # device ptrs to free once streams drain
        self._keepalive: list = []        # host blobs referenced by in-flight copies
        self._closed = False

    # -- device memory ------------------------------------------------------

    def _mark(self, buf: DeviceBuffer) -> None:
        buf.dev = self.device
        buf._req = self._req_seq

    def _alloc(self, buf: DeviceBuffer, stream: native.Stream) -> None:
        buf.ptr = native.malloc_async(stream, buf.size)
        buf.dev = self.device

    def _alloc_zeroed(self, buf: DeviceBuffer) -> None:
        self._alloc(buf, self.s_exec)
        native.memset_async(buf.ptr, 0, buf.size, self.s_exec)

    def _drop(self, buf: DeviceBuffer) -> None:
        """on_drop hook: an entry left the table or an ephemeral was freed."""
        if not buf.ptr:
            return
        ptr, buf.ptr = buf.ptr, 0
        if buf._req == self._req_seq:
            self._graveyard.append(ptr)  # may still be touched by this request
        else:
            native.free_async(self.s_in, ptr)

    def _drain(self) -> None:
        """Wait for every stream, then free deferred allocations."""
        self.s_in.sync()
        self.s_exec.sync()
        self.s_out.sync()
        for ptr in self._graveyard:
            native.free_async(self.s_exec, ptr)
        self._graveyard.clear()
        self._keepalive.clear()

    # -- buffer resolution (executor.py:233-316) ------------------------------

    def resolve_buffer(self, arg: BufferArg, stats: _ReqStats | None = None) -> DeviceBuffer:
        if stats is None:
            stats = _ReqStats()
        cache = self.cache

        if arg.is_ephemeral:
            cache.evict_until(arg.size)
            buf = cache.alloc_ephemeral(arg.size)
            self._mark(buf)
            self._alloc_zeroed(buf)
            return buf

        cached = cache.entries.get(arg.key)

        if arg.is_const:
            if cached is not None:
                if cached.size != arg.size:
                    raise SizeMismatchError(
                        f"buffer {arg.name!r}: cached object under {arg.key!r} is"
                        f" {cached.size} bytes, request declares {arg.size}")
                stats.cache_hits += 1
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
            self._alloc_zeroed(buf)
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
        payload = self.store.get(arg.key)  # NotFound propagates
        if len(payload) != arg.size:
            raise SizeMismatchError(
                f"buffer {arg.name!r}: store object {arg.key!r} is"
                f" {len(payload)} bytes, request declares {arg.size}")
        self._mark(buf)
        if not buf.ptr:
            self._alloc(buf, self.s_in)
        src = payload if isinstance(payload, PinnedBlob) else PinnedBlob.from_bytes(payload)
        native.h2d_async(buf.ptr, src.addr, arg.size, self.s_in)
        self._keepalive.append(src)
        self.dev_stats.h2d_bytes += arg.size
        buf.dirty = False
        self.clock.advance_ns(self.backend.timing.fetch_time_ns(arg.size))
        stats.store_gets += 1
        stats.bytes_fetched += arg.size
        stats.cache_misses += 1

    # -- request lifecycle (executor.py:320-425) ------------------------------

    def execute(self, req: KaasRequest) -> KaasResponse:
        t0 = self.clock.now_ns
        stats = _ReqStats()

        violations = validate_request(req)
        if violations:
            return self._finish(req, stats, t0,
                                Status.make_error("InvalidRequest", "; ".join(violations)))

        try:
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
            return self._finish(req, stats, t0, Status.make_error(exc.kind, exc.message))

        self._req_seq += 1
        if self.time_requests:
            self._ev_start.record(self.s_in)
            self.s_exec.wait(self._ev_start)
            self.s_out.wait(self._ev_start)
        resolved: dict[str, DeviceBuffer] = {}
        ephemerals: list[DeviceBuffer] = []
        try:
            for arg in req.referenced_buffers():
                buf = self.resolve_buffer(arg, stats)
                resolved[arg.name] = buf
                if arg.is_ephemeral:
                    ephemerals.append(buf)

            per_inv = self._plan_and_launch(req, kernels, resolved)
            self._flush(req, resolved, stats)
            status = Status.make_ok()
        except KaasError as exc:
            self._drain_quietly()
            self._release(resolved, ephemerals, drop_dirty=True)
            self._drain_quietly()
            return self._finish(req, stats, t0, Status.make_error(exc.kind, exc.message))

        self._release(resolved, ephemerals, drop_dirty=False)
        self._drain()
        if self.time_requests:
            ms = self._ev_start.elapsed_ms(self._ev_end)
            self.dev_stats.last_device_ms = ms
            self.dev_stats.device_ms += ms
        self.dev_stats.requests += 1
        return self._finish(req, stats, t0, status, per_inv)

    def _plan_and_launch(self, req: KaasRequest, kernels, resolved) -> list[InvocationStats]:
        """Check + price every invocation in order (backend.launch semantics),
        then enqueue them all in one C-ABI crossing."""
        timing = self.backend.timing
        n = len(req.invocations)
        descs = (native.LaunchDesc * n)() if n else None
        per_inv = []
        for i, (inv, kernel) in enumerate(zip(req.invocations, kernels)):
            bufs = [resolved[name] for name in inv.args]
            sizes = [b.size for b in bufs]
            kernel.check_arity(inv.literals, len(bufs))
            fma = kernel.plan(inv.dims, inv.literals, sizes)  # BackendFault before any effect
            compute_ns = timing.compute_time_ns(fma)
            overhead_ns = timing.launch_overhead_ns()
            self.clock.advance_ns(overhead_ns + compute_ns)
            fill_desc(descs[i], kernel, inv.dims, inv.literals, [b.ptr for b in bufs], sizes)
            for idx in kernel.writes:
                b = bufs[idx]
                if b.key is not None:
                    b.dirty = True
            per_inv.append(InvocationStats(inv.kernel_id, compute_ns, overhead_ns))
        if n:
            self._ev_fill.record(self.s_in)
            self.s_exec.wait(self._ev_fill)
            native.launch_batch(self.device, self.s_exec, descs)
            self.dev_stats.kernel_launches += n
        return per_inv

    def _flush(self, req: KaasRequest, resolved, stats: _ReqStats) -> None:
        """Write back dirty keyed buffers, table order (executor.py:371-380)."""
        self._ev_exec.record(self.s_exec)
        self.s_out.wait(self._ev_exec)
        pending = []
        for arg in req.referenced_buffers():
            buf = resolved[arg.name]
            # only non-const keyed buffers get dirty, and validation forbids
            # binding one non-const key twice, so no buffer appears twice here
            if buf.dirty:
                blob = PinnedBlob(buf.size)
                native.d2h_async(blob.addr, buf.ptr, buf.size, self.s_out)
                pending.append((buf, blob))
        if self.time_requests:
            self._ev_end.record(self.s_out)
        if pending:
            self.s_out.sync()
        else:
            self.s_exec.sync()
        for buf, blob in pending:
            if self._pinned_store:
                self.store.put_owned(buf.key, blob)
            else:
                self.store.put(buf.key, bytes(blob))
            self.clock.advance_ns(self.backend.timing.flush_time_ns(buf.size))
            stats.store_puts += 1
            stats.bytes_flushed += buf.size
            buf.dirty = False
            self.dev_stats.d2h_bytes += buf.size

    def _drain_quietly(self) -> None:
        """Failure-path drain: a sticky device error must not escape execute."""
        try:
            self._drain()
        except KaasError:
            self._graveyard.clear()
            self._keepalive.clear()

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
        """Release every device allocation and the streams."""
        if self._closed:
            return
        self._closed = True
        self._drain_quietly()
        for key in list(self.cache.entries):
            buf = self.cache.entries[key]
            buf._pinned = 0
            buf._dirty = False
            self.cache.remove(key)
        self._req_seq += 1
        self._drain()
        for s in (self.s_in, self.s_exec, self.s_out):
            s.sync()
            s.destroy()
        for e in (self._ev_fill, self._ev_exec, self._ev_start, self._ev_end):
            e.destroy()


# reference-compatible name
Executor = GpuExecutor
