"""DeviceStats: request spans are queued and read lazily (one elapsed-time
crossing for all queued requests), with events returned to the pool once read."""
import threading

from paper_2212_08146_b200 import gpu_executor as G


def test_lazy_spans_resolve_in_order_and_release_events(monkeypatch):
    calls = []

    def fake_elapsed_many(pairs):
        calls.append(len(pairs))
        return [float(a) * 10 + float(b) for a, b in pairs]  # "events" are ints here

    monkeypatch.setattr(G.native, "elapsed_many", fake_elapsed_many)
    pool = []
    st = G.DeviceStats(release=pool.append)
    ev1 = (1, 2, 3, 4, 5, 6)
    ev2 = (7, 8, 9, 1, 0, 0)
    st.defer(ev1, True, True)
    st.defer(ev2, True, False)
    assert calls == [] and pool == []          # nothing read yet
    assert st.last_device_ms == 78.0           # the latest request's span
    assert calls == [5]                        # one crossing: 3 + 2 pairs
    assert st.device_ms == 12.0 + 78.0
    assert st.kernel_ms == 34.0 + 91.0 and st.last_kernel_ms == 91.0
    assert st.h2d_ms == 56.0
    assert pool == [ev1, ev2]
    assert st.as_dict()["device_ms"] == 90.0 and calls == [5]


def test_queue_is_bounded(monkeypatch):
    monkeypatch.setattr(G.native, "elapsed_many", lambda pairs: [1.0] * len(pairs))
    pool = []
    st = G.DeviceStats(release=pool.append)
    for i in range(40):
        st.defer((i,) * 6, False, False)
    assert len(st._pending) < 16 and len(pool) >= 32


def test_concurrent_readers_release_each_event_once(monkeypatch):
    monkeypatch.setattr(G.native, "elapsed_many", lambda pairs: [1.0] * len(pairs))
    pool = []
    st = G.DeviceStats(release=pool.append)
    for i in range(10):
        st.defer((i,) * 6, True, False)
    ts = [threading.Thread(target=lambda: st.device_ms) for _ in range(8)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert sorted(e[0] for e in pool) == list(range(10))
    assert st.device_ms == 10.0
