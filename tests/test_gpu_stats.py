"""Measured device spans through the real executor: read lazily, consistent,
and every request's events return to the executor's pool once read."""
import pytest

pytestmark = pytest.mark.gpu


def test_lazy_device_spans_on_b200():
    from paper_2212_08146_b200 import native
    from paper_2212_08146_b200 import workloads as W
    from paper_2212_08146_b200.hoststore import PinnedStore
    from paper_2212_08146_b200.pool import KaasService

    if native.device_count() < 1:
        pytest.skip("no CUDA device")
    store = PinnedStore()
    W.seed_jacobi(store, 1024, prefix="st")
    svc = KaasService(store, n_executors=1, capacity=256 << 20, policy="rr", devices=[0])
    try:
        ex = svc.executors[0]
        for i in range(5):
            r = svc.submit(W.jacobi_request(f"st/{i}", 1024, 50, "st/A/1024", "st/b/1024",
                                            "st/x0/1024", "st/x", "st/r"))
            assert r.status.ok, r.status
        st = ex.dev_stats
        assert st.requests == 5
        assert len(st._pending) >= 1           # the last request is still queued ...
        last_dev, last_kern = st.last_device_ms, st.last_kernel_ms
        assert not st._pending                 # ... until a timing field is read
        assert 0.0 < last_kern <= last_dev
        assert st.kernel_ms <= st.device_ms
        assert st.device_ms >= last_dev        # five requests accumulated
        assert len(ex._ev_pool) >= 1            # events recycled after the read
    finally:
        svc.close()
