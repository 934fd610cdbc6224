"""Object stores: the reference's in-memory store and a pinned-memory store.

``MemoryStore`` keeps the reference semantics (``pkg/src/kaas/store.py:43-98``):
per-key locks, ``put`` copies the payload, ``get`` returns the stored bytes,
``NotFound`` / ``InvalidKey`` errors.

``PinnedStore`` is the B200 data plane: every object
lives in page-locked host memory, so a cache fill is one DMA straight from the
object (``cudaMemcpyAsync`` at PCIe line rate, no staging copy), and a flush
D2H-copies into a fresh pinned blob that the store adopts without copying.
Objects are ``PinnedBlob``s: read-only bytes-like values (buffer protocol via
PEP 688, ``==`` against ``bytes``, ``len``, ``bytes()``), so code written
against the reference store keeps working.  Pinned blocks are recycled
through ``PinnedPool`` because ``cudaHostAlloc`` costs milliseconds.
"""

from __future__ import annotations

import collections
import ctypes as C
import threading

from . import native
from .api import valid_store_key
from .faults import InvalidKeyError, NotFoundError


def _checked_key(key: str) -> str:
    if not valid_store_key(key):
        raise InvalidKeyError(f"invalid store key {key!r}")
    return key


class _KeyLocks:
    def __init__(self):
        self._locks: dict[str, threading.Lock] = {}
        self._guard = threading.Lock()

    def get(self, key: str) -> threading.Lock:
        with self._guard:
            lk = self._locks.get(key)
            if lk is None:
                lk = self._locks[key] = threading.Lock()
            return lk


class ObjectStore:
    """Store interface (``store.py:43-62``)."""

    def put(self, key: str, payload) -> None:
        raise NotImplementedError

    def get(self, key: str):
        raise NotImplementedError

    def delete(self, key: str) -> None:
        raise NotImplementedError

    def exists(self, key: str) -> bool:
        raise NotImplementedError

    def size_of(self, key: str) -> int:
        raise NotImplementedError

    def keys(self) -> list[str]:
        raise NotImplementedError


class MemoryStore(ObjectStore):
    """Dict-backed store with the reference semantics, plus a per-key put
    counter (``version``) so peer GPUs can tell whether a cached copy is the
    object the store serves now (the reference has no versioning,
    SPEC.md:171; the counter is invisible to reference callers)."""

    def __init__(self):
        self._objects: dict[str, bytes] = {}
        self._locks = _KeyLocks()
        self.version: dict[str, int] = {}

    def put(self, key: str, payload) -> int:
        """Store a copy; returns the key's new version."""
        _checked_key(key)
        data = bytes(payload)
        with self._locks.get(key):
            self._objects[key] = data
            v = self.version[key] = self.version.get(key, 0) + 1
            return v

    def get(self, key: str):
        _checked_key(key)
        with self._locks.get(key):
            try:
                return self._objects[key]
            except KeyError:
                raise NotFoundError(f"no object under key {key!r}") from None

    def get_versioned(self, key: str):
        """(payload, version) read atomically under the key lock."""
        _checked_key(key)
        with self._locks.get(key):
            try:
                return self._objects[key], self.version.get(key, 0)
            except KeyError:
                raise NotFoundError(f"no object under key {key!r}") from None

    def delete(self, key: str) -> None:
        _checked_key(key)
        with self._locks.get(key):
            self._objects.pop(key, None)

    def exists(self, key: str) -> bool:
        _checked_key(key)
        with self._locks.get(key):
            return key in self._objects

    def size_of(self, key: str) -> int:
        return len(self.get(key))

    def keys(self) -> list[str]:
        return sorted(self._objects)


# ---------------------------------------------------------------------------
# pinned host memory


def _size_class(n: int) -> int:
    if n <= 4096:
        return 4096
    if n <= (1 << 20):
        return 1 << (n - 1).bit_length()
    return (n + (2 << 20) - 1) // (2 << 20) * (2 << 20)


class PinnedPool:
    """Recycles page-locked host blocks by size class.

    ``pinned=False`` backs blocks with ordinary heap memory (for CPU-only
    tests of the store logic; the GPU executor still works, just without
    true DMA overlap)."""

    def __init__(self, pinned: bool = True, keep_bytes: int = 32 << 30):
        self.pinned = pinned
        self.keep_bytes = keep_bytes
        self._free: dict[int, list[int]] = {}
        self._cached = 0
        # blocks come back from PinnedBlob.__del__, which the garbage collector
        # may run at any allocation -- including one made while this thread
        # already holds the pool lock; __del__ therefore never takes the lock,
        # it only appends to this deque (atomic), drained under the lock.
        self._returns: collections.deque = collections.deque()
        self._lock = threading.RLock()
        self._heap_blocks: dict[int, C.Array] = {}
        self.allocated = 0

    def _drain_returns(self) -> None:
        while True:
            try:
                addr, cap = self._returns.popleft()
            except IndexError:
                return
            self._release_locked(addr, cap)

    def alloc(self, nbytes: int) -> tuple[int, int]:
        cap = _size_class(max(1, nbytes))
        with self._lock:
            self._drain_returns()
            lst = self._free.get(cap)
            if lst:
                self._cached -= cap
                return lst.pop(), cap
        if self.pinned:
            addr = native.host_alloc(cap)
        else:
            buf = (C.c_uint8 * cap)()
            addr = C.addressof(buf)
            self._heap_blocks[addr] = buf
        self.allocated += cap
        return addr, cap

    def release(self, addr: int, cap: int) -> None:
        """Lock-free hand-back (safe from __del__); recycled on the next alloc."""
        self._returns.append((addr, cap))

    def _release_locked(self, addr: int, cap: int) -> None:
        if self._cached + cap <= self.keep_bytes:
            self._free.setdefault(cap, []).append(addr)
            self._cached += cap
            return
        self.allocated -= cap
        if self.pinned:
            native.host_free(addr)
        else:
            self._heap_blocks.pop(addr, None)


_default_pool: PinnedPool | None = None
_pool_lock = threading.Lock()


def default_pool() -> PinnedPool:
    global _default_pool
    with _pool_lock:
        if _default_pool is None:
            _default_pool = PinnedPool(pinned=native.is_available())
        return _default_pool


class PinnedBlob:
    """Immutable-by-convention bytes living in a pinned host block."""

    __slots__ = ("addr", "nbytes", "_cap", "_pool", "_arr", "__weakref__")

    def __init__(self, nbytes: int, pool: PinnedPool | None = None):
        self._pool = pool or default_pool()
        self.addr, self._cap = self._pool.alloc(nbytes)
        self.nbytes = nbytes
        self._arr = (C.c_uint8 * nbytes).from_address(self.addr) if nbytes else None

    @classmethod
    def from_bytes(cls, payload, pool: PinnedPool | None = None) -> "PinnedBlob":
        mv = memoryview(payload).cast("B")
        blob = cls(mv.nbytes, pool)
        if mv.nbytes:
            blob._writable()[:] = mv
        return blob

    def _writable(self) -> memoryview:
        return memoryview(self._arr).cast("B") if self._arr is not None else memoryview(b"")

    def __buffer__(self, flags):
        return self._writable().toreadonly()

    def __release_buffer__(self, view):
        pass

    def __len__(self) -> int:
        return self.nbytes

    def __bytes__(self) -> bytes:
        return bytes(self._writable())

    def __eq__(self, other):
        try:
            return self._writable() == memoryview(other).cast("B")
        except TypeError:
            return NotImplemented

    def __hash__(self):
        return hash(bytes(self))

    def __repr__(self) -> str:
        return f"PinnedBlob({self.nbytes} bytes @ {self.addr:#x})"

    def __del__(self):
        pool = getattr(self, "_pool", None)
        if pool is not None and getattr(self, "_cap", 0):
            try:
                pool.release(self.addr, self._cap)
            except Exception:
                pass


class PinnedStore(MemoryStore):
    """``MemoryStore`` whose objects are ``PinnedBlob``s (zero-copy DMA)."""

    def __init__(self, pool: PinnedPool | None = None):
        super().__init__()
        self.pool = pool or default_pool()

    def put(self, key: str, payload) -> int:
        _checked_key(key)
        # copy, as the reference does (store.py:72): later caller writes
        # must not reach the stored object
        return self._adopt(key, PinnedBlob.from_bytes(payload, self.pool))

    def put_owned(self, key: str, blob: PinnedBlob) -> int:
        """Store ``blob`` without copying; the caller gives up ownership."""
        _checked_key(key)
        return self._adopt(key, blob)

    def _adopt(self, key: str, blob: PinnedBlob) -> int:
        with self._locks.get(key):
            self._objects[key] = blob
            v = self.version[key] = self.version.get(key, 0) + 1
            return v
