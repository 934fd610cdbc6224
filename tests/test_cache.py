"""Ledger / LRU of the GPU cache (host-side, no device memory needed).

Hand scenarios restate pkg/tests/test_executor.py:110-201; the randomized
test checks the O(log E) heap victim choice against the reference's O(E)
scan rule (oracle-style model) over long op sequences."""

import random

import pytest

from paper_2212_08146_b200.cache import CacheState, DeviceBuffer
from paper_2212_08146_b200.faults import OutOfDeviceMemoryError


def test_hand_simulated_lru():
    cache = CacheState(capacity=64, debug=True)
    a, b = DeviceBuffer("a", 32, False), DeviceBuffer("b", 32, False)
    cache.insert(a)
    cache.insert(b)
    cache.touch(a)
    cache.touch(b)
    assert cache.evict_until(32) == 32 and set(cache.entries) == {"b"}
    cache.insert(DeviceBuffer("c", 32, False))
    assert set(cache.entries) == {"b", "c"}


def test_needed_zero_is_noop_and_all_pinned_raises():
    cache = CacheState(capacity=64, debug=True)
    cache.insert(DeviceBuffer("a", 64, False))
    assert cache.evict_until(0) == 0
    cache = CacheState(capacity=64, debug=True)
    for k in ("a", "b"):
        buf = DeviceBuffer(k, 32, False)
        cache.insert(buf)
        cache.pin(buf)
    with pytest.raises(OutOfDeviceMemoryError):
        cache.evict_until(32)


def test_dirty_is_not_a_candidate_until_cleared():
    cache = CacheState(capacity=64, debug=True)
    d = DeviceBuffer("d", 64, False)
    cache.insert(d)
    d.dirty = True
    with pytest.raises(OutOfDeviceMemoryError):
        cache.evict_until(32)
    d.dirty = False
    assert cache.evict_until(32) == 64


def test_partial_evictions_persist_on_oom():
    cache = CacheState(capacity=96, debug=True)
    a, b, c = (DeviceBuffer(k, 32, False) for k in "abc")
    for x in (a, b, c):
        cache.insert(x)
    cache.pin(c)
    with pytest.raises(OutOfDeviceMemoryError):
        cache.evict_until(96)
    assert set(cache.entries) == {"c"}  # a, b evicted before the failure


def _scan_victim(cache):
    best = None
    for buf in cache.entries.values():
        if buf.pinned == 0 and not buf.dirty and (best is None or buf.last_use < best.last_use):
            best = buf
    return best


@pytest.mark.parametrize("seed", [2024, 515151, 7])
def test_heap_victims_equal_reference_scan(seed):
    rng = random.Random(seed)
    cache = CacheState(capacity=1 << 14, debug=False)
    live, counter = [], 0
    victims = []
    orig = cache.remove
    cache.remove = lambda k: (victims.append(k), orig(k))[1]
    for _ in range(6000):
        op = rng.random()
        if op < 0.4 or not live:
            size = rng.choice((256, 512, 1024, 2048))
            # model the reference scan on a copy of the state
            expect = []
            shadow = {k: (b.last_use, b.pinned, b.dirty, b.size) for k, b in cache.entries.items()}
            free = cache.free_space()
            while free < size:
                cands = [(v[0], k) for k, v in shadow.items() if v[1] == 0 and not v[2]]
                if not cands:
                    expect = None
                    break
                _, k = min(cands)
                expect.append(k)
                free += shadow.pop(k)[3]
            victims.clear()
            if expect is None:
                with pytest.raises(OutOfDeviceMemoryError):
                    cache.evict_until(size)
                live = [b for b in live if b.key in cache.entries]
                continue
            cache.evict_until(size)
            assert victims == expect
            live = [b for b in live if b.key in cache.entries]
            buf = DeviceBuffer(f"k{counter}", size, False)
            counter += 1
            cache.insert(buf)
            live.append(buf)
        elif op < 0.6:
            cache.touch(rng.choice(live))
        elif op < 0.75:
            cache.pin(rng.choice(live))
        elif op < 0.9:
            b = rng.choice(live)
            if b.pinned:
                cache.unpin(b)
        else:
            b = rng.choice(live)
            b.dirty = not b.dirty
        v = _scan_victim(cache)
        h = cache._pop_victim()
        assert (v.key if v else None) == (h.key if h else None)
    cache.check_accounting()
