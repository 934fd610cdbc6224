"""Object stores (CPU): reference MemoryStore semantics (pkg/tests/test_store.py
restated for the in-memory backend) and the pinned store's bytes-like blobs,
recycling and GC-safety."""

import gc
import threading

import pytest

from paper_2212_08146_b200.faults import InvalidKeyError, NotFoundError
from paper_2212_08146_b200.hoststore import MemoryStore, PinnedBlob, PinnedPool, PinnedStore


@pytest.fixture(params=["mem", "pinned"])
def store(request):
    if request.param == "mem":
        return MemoryStore()
    return PinnedStore(PinnedPool(pinned=False))


def test_put_get_roundtrip_and_copy_semantics(store):
    buf = bytearray(b"abcd")
    store.put("k", buf)
    buf[0] = ord("z")  # later caller writes must not reach the object
    assert store.get("k") == b"abcd"
    assert bytes(store.get("k")) == b"abcd" and len(store.get("k")) == 4
    assert store.exists("k") and store.size_of("k") == 4
    assert store.keys() == ["k"]
    store.delete("k")
    assert not store.exists("k")
    with pytest.raises(NotFoundError):
        store.get("k")


def test_invalid_keys_rejected(store):
    for bad in ("", "a b", "x" * 257, "ü"):
        with pytest.raises(InvalidKeyError):
            store.put(bad, b"x")


def test_concurrent_puts_never_tear(store):
    def writer(v):
        for _ in range(200):
            store.put("hot", bytes([v]) * 4096)

    ts = [threading.Thread(target=writer, args=(i,)) for i in range(8)]
    for t in ts:
        t.start()
    for _ in range(200):
        data = bytes(store.get("hot")) if store.exists("hot") else None
        if data is not None:
            assert len(set(data)) == 1
    for t in ts:
        t.join()


def test_pinned_blob_is_read_only_and_outlives_store_entry():
    pool = PinnedPool(pinned=False)
    st = PinnedStore(pool)
    st.put("k", b"\x01\x02\x03\x04")
    mv = memoryview(st.get("k"))
    assert mv.readonly
    st.put("k", b"\x09" * 4)  # replaces the entry; the old blob lives while viewed
    gc.collect()
    assert bytes(mv) == b"\x01\x02\x03\x04"
    assert st.version["k"] == 2


def test_pool_recycles_blocks_and_is_gc_reentrant():
    pool = PinnedPool(pinned=False)
    a = PinnedBlob(5000, pool)
    addr = a.addr
    del a
    b = PinnedBlob(6000, pool)  # same 8 KiB size class: recycled block
    assert b.addr == addr
    # blobs freed by the cyclic GC while the pool is busy must not deadlock
    for _ in range(2000):
        x = PinnedBlob(64, pool)
        cyc = [x]
        cyc.append(cyc)
        del x, cyc
    gc.collect()
    PinnedBlob(64, pool)
