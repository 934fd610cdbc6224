"""Multi-GPU request pool: the ``KaasService`` surface over B200 executors.

Same public surface as the reference service (``pkg/src/kaas/service.py:22-112``):
``KaasService(store, n_executors, capacity, policy, timing, digest_cap,
strict_schema, debug)``, ``submit`` / ``submit_async`` / ``stats`` /
``close``, context manager, ``executors`` / ``router`` / ``store`` attributes.

Executor ``i`` owns GPU ``devices[i % len(devices)]`` (one executor per GPU by
default; several executors may share a GPU, each with its own ledger and
streams).  Each executor has one consumer thread and a FIFO queue, so
requests on one executor run in arrival order; the router decision is made
at submission time under its lock.  ctypes drops the GIL inside every CUDA
call, so the per-GPU workers overlap.  No NCCL: requests shard by request.
"""

from __future__ import annotations

import queue
import threading
from concurrent.futures import Future

from . import native
from .api import KaasRequest, KaasResponse, Status
from .gpu_executor import ExecutorConfig, GpuBackend, GpuExecutor
from .peers import PeerDirectory
from .placement import Router, parse_policy
from .timing import TimingModel


def visible_devices() -> list[int]:
    return list(range(native.device_count()))


class KaasService:
    def __init__(self, store, n_executors: int | None = None, capacity: int = 256 * 2**20,
                 policy="affinity:8", timing: TimingModel | None = None,
                 digest_cap: int = 1024, strict_schema: bool = False, debug: bool = False,
                 devices: list[int] | None = None, executor_factory=None,
                 log_decisions: bool = False, max_inflight: int = 3, peer_fills: bool = True,
                 reserve_bytes: int = 0):
        explicit_devices = devices is not None
        if executor_factory is None:
            devices = devices if devices is not None else visible_devices()
            if not devices:
                raise RuntimeError("no CUDA devices visible (libkaas_b200 has no CPU path)")
        if n_executors is None:
            # the reference default is one executor (service.py:24); an explicit
            # device list means one executor per listed GPU
            n_executors = len(devices) if explicit_devices else 1
        if n_executors < 1:
            raise ValueError("need at least one executor")
        self.store = store
        self.strict_schema = strict_schema
        self.max_inflight = max_inflight
        self.timing = timing if timing is not None else TimingModel()
        self.devices = devices
        if executor_factory is None:
            def executor_factory(i):
                cfg = ExecutorConfig(capacity=capacity, timing=self.timing, executor_id=i,
                                     debug=debug, device=devices[i % len(devices)],
                                     reserve_bytes=reserve_bytes)
                return GpuExecutor(cfg, store, GpuBackend(timing=self.timing))
        self.executors = [executor_factory(i) for i in range(n_executors)]
        # peer fills between this pool's executors (NVLink across GPUs, D2D on one)
        self.peers = None
        gpu_execs = [e for e in self.executors if hasattr(e, "peers")]
        if peer_fills and len(gpu_execs) > 1:
            self.peers = PeerDirectory()
            devs = sorted({e.device for e in gpu_execs})
            for d in devs:
                for q in devs:
                    if d != q:
                        native.enable_peer(d, q)
            for e in gpu_execs:
                e.peers = self.peers
        if isinstance(policy, str):
            policy = parse_policy(policy)
        self.router = Router([e.executor_id for e in self.executors], policy,
                             digest_cap=digest_cap, log_decisions=log_decisions)
        self._queues = {e.executor_id: queue.Queue() for e in self.executors}
        self._by_id = {e.executor_id: e for e in self.executors}
        # a GPU executor is driven either by its worker thread or, when it is
        # idle (nothing queued, nothing in flight), inline by a synchronous
        # submit() -- saving two thread hand-offs (~40 us) per request; this
        # lock says who owns it
        self._dispatch = threading.Lock()  # route + enqueue / inline claim, atomically
        # requests routed to an executor and not yet claimed by its worker
        # (a dequeued item counts until the worker owns the executor)
        self._pending = {e.executor_id: 0 for e in self.executors}
        self._owners = {e.executor_id: threading.Lock() for e in self.executors
                        if hasattr(e, "begin")}
        self._threads = [threading.Thread(target=self._worker, args=(e,), daemon=True,
                                          name=f"kaas-executor-{e.executor_id}")
                         for e in self.executors]
        self._closed = False
        for t in self._threads:
            t.start()

    def _after(self, executor) -> None:
        """A faulted (poisoned) executor leaves the placement set."""
        if getattr(executor, "poisoned", None) is not None and \
                executor.executor_id not in self.router.down:
            self.router.mark_down(executor.executor_id)

    def _worker(self, executor) -> None:
        dev = getattr(executor, "device", None)
        if dev is not None:
            native.bind_thread(dev)  # this thread's current device, once
        if hasattr(executor, "begin"):
            return self._pipelined_worker(executor)
        q = self._queues[executor.executor_id]
        while True:
            item = q.get()
            if item is None:
                return
            with self._dispatch:
                self._pending[executor.executor_id] -= 1
            req, fut = item
            try:
                resp = executor.execute(req)
            except BaseException as exc:  # execute() reports request errors in-band
                failed = KaasResponse(req.request_id, Status.make_error("Internal", str(exc)))
                self.router.update_digest(executor.executor_id, failed, req)
                fut.set_exception(exc)
                continue
            self.router.update_digest(executor.executor_id, resp, req)
            fut.set_result(resp)

    def _pipelined_worker(self, executor) -> None:
        """Up to ``max_inflight`` requests per executor overlap on the device:
        request i's write-back and epilogue run while request i+1's fills and
        kernels are queued.  Decisions are still taken strictly in arrival
        order inside ``begin`` (bit-exact), puts and responses in ``complete``."""
        eid = executor.executor_id
        q = self._queues[eid]
        owner = self._owners[eid]
        futs: dict[int, tuple] = {}

        def on_complete(rec, resp):
            entry = futs.pop(rec.seq, None)
            if entry is None:  # an inline submit(): the caller finishes it
                return
            req, fut = entry
            self.router.update_digest(eid, resp, req)
            self._after(executor)
            fut.set_result(resp)

        executor.on_complete = on_complete
        held = False
        while True:
            if executor.inflight:
                executor.complete(block=False)
            if executor.inflight:
                try:
                    item = q.get_nowait()
                except queue.Empty:
                    executor.complete(through=next(iter(futs)))  # block on the oldest
                    continue
            else:
                if held:  # idle: inline submits may drive the executor meanwhile
                    owner.release()
                    held = False
                item = q.get()
                owner.acquire()
                held = True
            if item is not None:
                with self._dispatch:
                    self._pending[eid] -= 1
            if item is None:
                executor.complete()
                owner.release()
                return
            req, fut = item
            try:
                rec = executor.begin(req)
            except BaseException as exc:
                try:
                    executor.complete()
                except BaseException:
                    pass
                failed = KaasResponse(req.request_id, Status.make_error("Internal", str(exc)))
                self.router.update_digest(eid, failed, req)
                fut.set_exception(exc)
                continue
            if isinstance(rec, KaasResponse):  # failed on the host: nothing in flight
                self.router.update_digest(eid, rec, req)
                self._after(executor)
                fut.set_result(rec)
                continue
            futs[rec.seq] = (req, fut)
            while executor.inflight > self.max_inflight:
                executor.complete(through=next(iter(futs)))

    def submit_async(self, req: KaasRequest) -> Future:
        if self._closed:
            raise RuntimeError("service is closed")
        fut: Future = Future()
        with self._dispatch:  # routing order = queue order per executor
            eid = self.router.route(req)
            fut.executor_id = eid  # placement, for benches and tests
            self._pending[eid] += 1
            self._queues[eid].put((req, fut))
        return fut

    def submit(self, req: KaasRequest) -> KaasResponse:
        if self._closed:
            raise RuntimeError("service is closed")
        # Route and claim under one lock, so every executor runs its requests
        # in routing order (the decision log replays against a FIFO
        # executor): a request routed later can neither be queued ahead of
        # this one nor run inline before it.
        with self._dispatch:
            eid = self.router.route(req)
            owner = self._owners.get(eid)
            q = self._queues[eid]
            inline = owner is not None and not self._pending[eid] and owner.acquire(blocking=False)
            if inline:
                ex = self._by_id[eid]
                if ex.inflight:
                    owner.release()
                    inline = False
            if not inline:
                fut: Future = Future()
                fut.executor_id = eid
                self._pending[eid] += 1
                q.put((req, fut))
        if not inline:
            return fut.result()
        # idle and nobody queued ahead: run it on this thread
        try:
            try:
                resp = ex.execute(req)
            except BaseException as exc:
                failed = KaasResponse(req.request_id, Status.make_error("Internal", str(exc)))
                self.router.update_digest(eid, failed, req)
                raise
            self.router.update_digest(eid, resp, req)
            self._after(ex)
            return resp
        finally:
            owner.release()

    def stats(self) -> dict:
        out = {"executors": [e.stats() for e in self.executors],
               "router": self.router.snapshot()}
        dev = [e.device_stats() for e in self.executors if hasattr(e, "device_stats")]
        if dev:
            out["devices"] = dev
        return out

    def close(self) -> None:
        if self._closed:
            return
        self._closed = True
        for q in self._queues.values():
            q.put(None)
        for t in self._threads:
            t.join(timeout=60)
        for e in self.executors:
            if hasattr(e, "close"):
                e.close()

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()


GpuKaasService = KaasService
