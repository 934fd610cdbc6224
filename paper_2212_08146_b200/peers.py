"""Peer cache directory: NVLink (or same-GPU) fills from another executor.

A cache fill in the reference always reads the object store
(``executor.py:305-316``).  When another executor of the same pool already
holds the store object *at the version the store serves now*, the bytes are
identical, so the fill can be a device-to-device copy (``cudaMemcpyPeerAsync``
over NVLink 5 / NVSwitch, ~700 GB/s, or a same-GPU D2D copy) instead of a PCIe
H2D (~55 GB/s).  Nothing observable changes: the fill still counts as a store
get / miss / bytes_fetched and still performs the NotFound / SizeMismatch
checks against the store; only ``DeviceStats.p2p_bytes`` records it.

Lifetime rules (all transitions under one lock):
* an entry is published only once its bytes equal a store version: after a
  fill (with the fill's completion event) or after a flush's put;
* it is withdrawn when a kernel is about to write it (dirty) or it leaves
  the cache;
* a borrower records an event after its copy; the owner's later free or
  in-place overwrite of that buffer is stream-ordered after every such event.
"""

from __future__ import annotations

import threading


class _Entry:
    __slots__ = ("owner", "buf", "version", "ready")

    def __init__(self, owner, buf, version, ready):
        self.owner, self.buf, self.version, self.ready = owner, buf, version, ready


class PeerDirectory:
    def __init__(self):
        self._lock = threading.Lock()
        self._by_key: dict[str, dict[int, _Entry]] = {}
        self.lends = 0

    def publish(self, owner: int, buf, version: int, ready=None) -> None:
        if buf.key is None or version is None:
            return
        with self._lock:
            self._by_key.setdefault(buf.key, {})[owner] = _Entry(owner, buf, version, ready)

    def withdraw(self, owner: int, buf) -> None:
        if buf.key is None:
            return
        with self._lock:
            d = self._by_key.get(buf.key)
            if d is not None:
                e = d.get(owner)
                if e is not None and e.buf is buf:
                    del d[owner]
                    if not d:
                        del self._by_key[buf.key]

    def borrow(self, key: str, version: int, borrower: int, copy_fn) -> bool:
        """Find a peer copy of ``key`` at ``version`` and run
        ``copy_fn(src_buf, ready_event) -> lend_event`` while the directory
        lock guarantees the source cannot be withdrawn mid-enqueue.  The
        returned event is attached to the source buffer.  True if copied."""
        with self._lock:
            d = self._by_key.get(key)
            if not d:
                return False
            for owner, e in d.items():
                if owner == borrower or e.version != version or not e.buf.ptr:
                    continue
                ev = copy_fn(e.buf, e.ready)
                e.buf._lends.append(ev)
                self.lends += 1
                return True
        return False

    def take_lends(self, buf) -> list:
        """Events the owner must order a free / overwrite of ``buf`` after."""
        with self._lock:
            evs, buf._lends = buf._lends, []
            return evs
