"""Per-GPU device-buffer cache: the byte ledger and its LRU eviction.

Decisions are bit-exact with the reference ``CacheState``
(``pkg/src/kaas/executor.py:91-195``): unique ticks from ``insert``/``touch``
(``pin``/``unpin`` do not tick), ``used_bytes`` = sum of keyed entry sizes,
live ephemerals count against capacity outside the table, and
``evict_until(needed)`` removes the minimum-``last_use`` entry among
``pinned == 0 and not dirty`` until ``capacity - used - ephemeral >= needed``,
raising ``OutOfDeviceMemory`` -- with the partial evictions kept -- when no
candidate is left.

The reference scans every entry per victim (O(E)); here candidates live in a
lazy min-heap keyed by ``last_use``.  Ticks are unique, so the heap minimum
that is still a valid candidate is exactly the reference's victim.  Every
transition *into* the evictable state (insert, touch, unpin to zero, dirty
cleared) pushes a fresh heap item; stale items (entry gone, tick moved, not
evictable now) are discarded on pop.

Ledger objects hold no device memory themselves: ``DeviceBuffer.ptr`` is
attached by the executor, and the cache calls ``on_drop(buf)`` whenever an
entry leaves the table so the executor can release the allocation.
"""

from __future__ import annotations

import heapq

from .faults import OutOfDeviceMemoryError


class DeviceBuffer:
    """A device-resident allocation (``executor.py:53-88``).

    ``pinned`` holds the buffer against eviction while a request uses it;
    ``dirty`` marks device contents newer than the store.  Setting either
    field notifies the owning cache so the LRU index stays exact.
    """

    __slots__ = ("key", "size", "is_const", "_pinned", "_dirty", "last_use",
                 "ptr", "dev", "_cache", "_epoch", "_req", "_lends", "_ready", "_derived", "_hits",
                 "__weakref__")

    def __init__(self, key: str | None, size: int, is_const: bool):
        self.key = key
        self.size = size
        self.is_const = is_const
        self._pinned = 0
        self._dirty = False
        self.last_use = 0
        self.ptr = 0        # device address, 0 until the executor allocates
        self.dev = -1
        self._cache = None  # owning CacheState while in its table
        self._epoch = 0     # bumps on every table (re)insertion
        self._req = -1      # last request (executor sequence no.) that used it
        self._lends = []    # events of peer copies reading this buffer (peers.py)
        self._ready = None  # event recorded after the last fill (peers.py)
        self._derived = None  # kernel-prepared forms of the contents (gpu_executor.py)
        self._hits = 0        # const cache hits since the last fill

    @property
    def pinned(self) -> int:
        return self._pinned

    @pinned.setter
    def pinned(self, value: int) -> None:
        self._pinned = value
        if value == 0 and self._cache is not None:
            self._cache._maybe_candidate(self)

    @property
    def dirty(self) -> bool:
        return self._dirty

    @dirty.setter
    def dirty(self, value: bool) -> None:
        self._dirty = value
        if not value and self._cache is not None:
            self._cache._maybe_candidate(self)

    def evictable(self) -> bool:
        return self._pinned == 0 and not self._dirty

    # -- host views of the device bytes (DeviceBuffer.snapshot/load,
    #    executor.py:78-82); synchronous, for tests and tools ------------

    def snapshot(self) -> bytes:
        if self.ptr == 0:
            return bytes(self.size)
        from . import native
        from .hoststore import PinnedBlob
        s = native.util_stream(self.dev)
        blob = PinnedBlob(self.size)
        native.d2h_async(blob.addr, self.ptr, self.size, s)
        s.sync()
        return bytes(blob)

    def load(self, payload) -> None:
        from . import native
        from .hoststore import PinnedBlob
        blob = PinnedBlob.from_bytes(payload)
        s = native.util_stream(self.dev)
        native.h2d_async(self.ptr, blob.addr, self.size, s)
        s.sync()

    def canaries_intact(self) -> bool:
        # device allocations carry no canaries: every launch is bounds-checked
        # on the host before it is enqueued (kernels.py plan functions)
        return True

    def __repr__(self) -> str:
        return (f"DeviceBuffer(key={self.key!r}, size={self.size}, pinned={self._pinned},"
                f" dirty={self._dirty}, last_use={self.last_use})")


class CacheState:
    """Keyed device-buffer table plus the accounting ledger."""

    def __init__(self, capacity: int, debug: bool = False, on_drop=None):
        self.capacity = capacity
        self.debug = debug
        self.entries: dict[str, DeviceBuffer] = {}
        self.used_bytes = 0
        self.ephemeral_bytes = 0
        self.tick = 0
        self.on_drop = on_drop
        self._heap: list[tuple[int, int, str, int]] = []  # (last_use, seq, key, epoch)
        self._seq = 0
        self.evictions = 0

    # -- ledger -------------------------------------------------------------

    def check_accounting(self) -> None:
        total = sum(b.size for b in self.entries.values())
        assert self.used_bytes == total, (
            f"ledger drift: used_bytes={self.used_bytes} actual={total}")
        assert self.used_bytes + self.ephemeral_bytes <= self.capacity, (
            f"capacity exceeded: {self.used_bytes}+{self.ephemeral_bytes} > {self.capacity}")
        assert self.ephemeral_bytes >= 0
        for key, buf in self.entries.items():
            assert buf.key == key
            assert buf.pinned >= 0
            assert not (buf.dirty and buf.key is None)

    def _after_step(self) -> None:
        if self.debug:
            self.check_accounting()

    # -- LRU index ----------------------------------------------------------

    def _push(self, buf: DeviceBuffer) -> None:
        self._seq += 1
        heapq.heappush(self._heap, (buf.last_use, self._seq, buf.key, buf._epoch))
        if len(self._heap) > 4 * len(self.entries) + 64:
            self._compact()

    def _compact(self) -> None:
        # drop stale items: one item per currently evictable entry
        self._heap = [(b.last_use, i, k, b._epoch)
                      for i, (k, b) in enumerate(self.entries.items()) if b.evictable()]
        heapq.heapify(self._heap)
        self._seq = len(self._heap)

    def _maybe_candidate(self, buf: DeviceBuffer) -> None:
        if buf.evictable() and self.entries.get(buf.key) is buf:
            self._push(buf)

    def _pop_victim(self) -> DeviceBuffer | None:
        heap = self._heap
        while heap:
            last_use, _, key, epoch = heap[0]
            buf = self.entries.get(key)
            if (buf is None or buf._epoch != epoch or buf.last_use != last_use
                    or not buf.evictable()):
                heapq.heappop(heap)
                continue
            return buf
        return None

    # -- mutations ----------------------------------------------------------

    def next_tick(self) -> int:
        self.tick += 1
        return self.tick

    def touch(self, buf: DeviceBuffer) -> None:
        buf.last_use = self.next_tick()
        if buf._cache is self:
            self._maybe_candidate(buf)
        self._after_step()

    def pin(self, buf: DeviceBuffer) -> None:
        buf.pinned += 1
        self._after_step()

    def unpin(self, buf: DeviceBuffer) -> None:
        assert buf.pinned > 0, "unbalanced unpin"
        buf.pinned -= 1
        self._after_step()

    def insert(self, buf: DeviceBuffer) -> None:
        assert buf.key is not None and buf.key not in self.entries
        self.entries[buf.key] = buf
        self.used_bytes += buf.size
        buf._cache = self
        buf._epoch += 1
        buf.last_use = self.next_tick()
        self._maybe_candidate(buf)
        self._after_step()

    def remove(self, key: str) -> DeviceBuffer:
        buf = self.entries.pop(key)
        self.used_bytes -= buf.size
        buf._cache = None
        if self.on_drop is not None:
            self.on_drop(buf)
        self._after_step()
        return buf

    def alloc_ephemeral(self, size: int) -> DeviceBuffer:
        buf = DeviceBuffer(key=None, size=size, is_const=False)
        self.ephemeral_bytes += size
        buf.pinned = 1
        self._after_step()
        return buf

    def free_ephemeral(self, buf: DeviceBuffer) -> None:
        assert buf.key is None
        self.ephemeral_bytes -= buf.size
        buf.pinned = 0
        if self.on_drop is not None:
            self.on_drop(buf)
        self._after_step()

    # -- eviction -----------------------------------------------------------

    def free_space(self) -> int:
        return self.capacity - self.used_bytes - self.ephemeral_bytes

    def evict_until(self, needed: int) -> int:
        assert needed >= 0
        freed = 0
        while self.free_space() < needed:
            victim = self._pop_victim()
            if victim is None:
                raise OutOfDeviceMemoryError(
                    f"need {needed} bytes, {self.free_space()} free and no"
                    " evictable entries")
            self.remove(victim.key)
            self.evictions += 1
            freed += victim.size
        return freed

    def snapshot(self) -> dict[str, tuple[int, int, int, bool]]:
        """``{key: (size, last_use, pinned, dirty)}`` for parity checks."""
        return {k: (b.size, b.last_use, b.pinned, b.dirty) for k, b in self.entries.items()}
