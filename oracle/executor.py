"""Oracle executor -- TEST INFRASTRUCTURE ONLY.

Restates the reference request lifecycle (``pkg/src/kaas/executor.py``) over
host memory: the byte ledger with unique ticks and an O(E) LRU victim scan
(``executor.py:91-195``), the 5-way ``resolve_buffer`` tree (``233-303``),
``_fetch_into`` (``305-316``), ``execute`` (``320-387``), ``_release``
(``394-410``) and the virtual timing model (``backend.py:37-68``).  Kernels
come from ``oracle.kernels``.  Observable outputs -- responses, cache
snapshots, eviction sequence, store bytes -- are what the GPU executor must
reproduce.
"""

from __future__ import annotations

import numpy as np

from paper_2212_08146_b200.api import (
    InvocationStats,
    IoStats,
    KaasResponse,
    Status,
    validate_request,
)

from .kernels import KERNELS, OracleFault

NS = 1_000_000_000


def ns(seconds: float) -> int:  # backend.py:37-38
    return int(round(seconds * NS))


class OracleTiming:
    """backend.py:41-68 with the default parameters."""

    def __init__(self, h2d=12 * 2**30, d2h=12 * 2**30, fetch_latency=200e-6,
                 launch_overhead=10e-6, flop_rate=1e12):
        self.h2d, self.d2h = h2d, d2h
        self.fetch_latency, self.launch_overhead, self.flop_rate = (
            fetch_latency, launch_overhead, flop_rate)

    @classmethod
    def from_model(cls, t) -> "OracleTiming":
        return cls(t.h2d_bandwidth, t.d2h_bandwidth, t.fetch_latency, t.launch_overhead,
                   t.flop_rate)

    def fetch(self, nbytes):
        return ns(self.fetch_latency) + ns(nbytes / self.h2d)

    def flush(self, nbytes):
        return ns(nbytes / self.d2h)

    def overhead(self):
        return ns(self.launch_overhead)

    def compute(self, fma):
        return ns(fma / self.flop_rate)


class Fail(Exception):
    def __init__(self, kind: str, message: str):
        super().__init__(message)
        self.kind, self.message = kind, message


class Entry:
    __slots__ = ("key", "size", "const", "pins", "dirty", "tick", "data")

    def __init__(self, key, size, const):
        self.key, self.size, self.const = key, size, const
        self.pins, self.dirty, self.tick = 0, False, 0
        self.data = bytearray(size)  # zero-filled like executor.py:70


class OracleExecutor:
    def __init__(self, capacity: int, store, timing: OracleTiming | None = None,
                 kernels=None):
        self.capacity = capacity
        self.store = store  # any object with get/put (bytes)
        self.t = timing or OracleTiming()
        self.kernels = kernels or KERNELS
        self.table: dict[str, Entry] = {}
        self.used = 0
        self.eph = 0
        self.tick = 0
        self.now = 0
        self.victims: list[str] = []  # eviction sequence, for parity checks
        self.removed: list[str] = []  # every table removal (evict/replace/drop)
        self.hits = self.misses = self.served = 0

    # -- ledger ---------------------------------------------------------

    def _tick(self) -> int:
        self.tick += 1
        return self.tick

    def _insert(self, e: Entry):
        self.table[e.key] = e
        self.used += e.size
        e.tick = self._tick()

    def _remove(self, key: str) -> Entry:
        self.removed.append(key)
        e = self.table.pop(key)
        self.used -= e.size
        return e

    def _make_room(self, needed: int):
        while self.capacity - self.used - self.eph < needed:
            best = None
            for e in self.table.values():
                if e.pins == 0 and not e.dirty and (best is None or e.tick < best.tick):
                    best = e
            if best is None:
                raise Fail("OutOfDeviceMemory",
                           f"need {needed} bytes, {self.capacity - self.used - self.eph}"
                           " free and no evictable entries")
            self._remove(best.key)
            self.victims.append(best.key)

    # -- resolution -----------------------------------------------------

    def _fetch(self, e: Entry, arg, st):
        try:
            payload = self.store.get(arg.key)
        except KeyError:
            raise Fail("NotFound", f"no object under key {arg.key!r}") from None
        if len(payload) != arg.size:
            raise Fail("SizeMismatch",
                       f"buffer {arg.name!r}: store object {arg.key!r} is"
                       f" {len(payload)} bytes, request declares {arg.size}")
        e.data[:] = bytes(payload)
        e.dirty = False
        self.now += self.t.fetch(arg.size)
        st["store_gets"] += 1
        st["bytes_fetched"] += arg.size
        st["cache_misses"] += 1

    def _resolve(self, arg, st) -> Entry:
        if arg.is_ephemeral:
            self._make_room(arg.size)
            e = Entry(None, arg.size, False)
            self.eph += arg.size
            e.pins = 1
            return e
        cur = self.table.get(arg.key)
        if arg.is_const:
            if cur is not None:
                if cur.size != arg.size:
                    raise Fail("SizeMismatch",
                               f"buffer {arg.name!r}: cached object under {arg.key!r} is"
                               f" {cur.size} bytes, request declares {arg.size}")
                st["cache_hits"] += 1
                cur.pins += 1
                cur.tick = self._tick()
                cur.const = True
                return cur
            self._make_room(arg.size)
            e = Entry(arg.key, arg.size, True)
            self._fetch(e, arg, st)
            self._insert(e)
            e.pins += 1
            return e
        if arg.direction == "output":
            if cur is not None:
                if cur.pins > 0:
                    raise Fail("BufferBusy", f"buffer {arg.name!r}: key {arg.key!r} pinned elsewhere")
                self._remove(arg.key)
            self._make_room(arg.size)
            e = Entry(arg.key, arg.size, False)
            st["cache_misses"] += 1
            self._insert(e)
            e.pins += 1
            return e
        if cur is not None and cur.pins > 0:
            raise Fail("BufferBusy", f"buffer {arg.name!r}: key {arg.key!r} pinned elsewhere")
        if cur is not None and cur.size == arg.size:
            self._fetch(cur, arg, st)
            cur.const = False
            cur.pins += 1
            cur.tick = self._tick()
            return cur
        if cur is not None:
            self._remove(arg.key)
        self._make_room(arg.size)
        e = Entry(arg.key, arg.size, False)
        self._fetch(e, arg, st)
        self._insert(e)
        e.pins += 1
        return e

    # -- lifecycle ------------------------------------------------------

    def execute(self, req) -> KaasResponse:
        t0 = self.now
        st = dict.fromkeys(("store_gets", "store_puts", "bytes_fetched", "bytes_flushed",
                            "cache_hits", "cache_misses"), 0)
        problems = validate_request(req)
        if problems:
            return self._done(req, st, t0, Status.make_error("InvalidRequest", "; ".join(problems)))
        try:
            specs = []
            for inv in req.invocations:
                if inv.kernel_id not in self.kernels:
                    raise Fail("UnknownKernel", f"no kernel registered as {inv.kernel_id!r}")
                spec = self.kernels[inv.kernel_id]
                self._arity(inv.kernel_id, spec, inv.literals, len(inv.args))
                for w in spec[2]:
                    a = req.by_name[inv.args[w]]
                    if not a.is_ephemeral and a.direction == "input":
                        raise Fail("InvalidRequest",
                                   f"kernel {inv.kernel_id!r} writes to read-only buffer {a.name!r}")
                specs.append(spec)
        except Fail as f:
            return self._done(req, st, t0, Status.make_error(f.kind, f.message))

        got: dict[str, Entry] = {}
        temps: list[Entry] = []
        try:
            for arg in req.referenced_buffers():
                e = self._resolve(arg, st)
                got[arg.name] = e
                if arg.is_ephemeral:
                    temps.append(e)
            per = []
            for inv, spec in zip(req.invocations, specs):
                views = [np.frombuffer(got[nm].data, dtype=np.uint8) for nm in inv.args]
                self._arity(inv.kernel_id, spec, inv.literals, len(views))
                try:
                    with np.errstate(all="ignore"):
                        fma = spec[3](inv.dims, inv.literals, views)
                except OracleFault as f:
                    raise Fail("BackendFault", str(f)) from None
                c_ns = self.t.compute(fma)
                o_ns = self.t.overhead()
                self.now += o_ns + c_ns
                for w in spec[2]:
                    e = got[inv.args[w]]
                    if e.key is not None:
                        e.dirty = True
                per.append(InvocationStats(inv.kernel_id, c_ns, o_ns))
            for arg in req.referenced_buffers():
                e = got[arg.name]
                if e.dirty:
                    self.store.put(e.key, bytes(e.data))
                    self.now += self.t.flush(e.size)
                    st["store_puts"] += 1
                    st["bytes_flushed"] += e.size
                    e.dirty = False
        except Fail as f:
            self._release(got, temps, True)
            return self._done(req, st, t0, Status.make_error(f.kind, f.message))
        self._release(got, temps, False)
        return self._done(req, st, t0, Status.make_ok(), per)

    @staticmethod
    def _arity(kid, spec, literals, n_args):
        if n_args != spec[1]:
            raise Fail("ArityMismatch", f"{kid}: expected {spec[1]} buffer args, got {n_args}")
        tags = tuple(l.type for l in literals)
        if tags != spec[0]:
            raise Fail("ArityMismatch", f"{kid}: expected literals {spec[0]}, got {tags}")

    def _release(self, got, temps, drop_dirty):
        for e in temps:
            self.eph -= e.size
            e.pins = 0
        for e in got.values():
            if e.key is not None:
                e.pins -= 1
        if drop_dirty:
            for e in got.values():
                if e.key is not None and e.dirty and self.table.get(e.key) is e:
                    self._remove(e.key)
                    e.dirty = False

    def _done(self, req, st, t0, status, per=None) -> KaasResponse:
        self.hits += st["cache_hits"]
        self.misses += st["cache_misses"]
        self.served += 1
        return KaasResponse(req.request_id, status, tuple(per or ()), IoStats(**st),
                            self.now - t0)

    def snapshot(self) -> dict:
        return {k: (e.size, e.tick, e.pins, e.dirty) for k, e in self.table.items()}


class DictStore:
    """Minimal oracle store: key -> bytes (NotFound as KeyError)."""

    def __init__(self, objects=None):
        self.objects: dict[str, bytes] = dict(objects or {})

    def get(self, key):
        return self.objects[key]

    def put(self, key, payload):
        self.objects[key] = bytes(payload)

    def keys(self):
        return sorted(self.objects)
