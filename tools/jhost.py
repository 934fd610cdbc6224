"""Dev: host timeline of a warm Jacobi request and the chain's true device cost.

1. Chain kernel behind a busy stream (a 1 GiB memset first, so the host has
   enqueued the launch before the GPU reaches it): device-only fixed cost.
2. Per-request host timeline through KaasService.submit: submit -> launch_batch
   call -> its return -> last event sync -> submit return.

    python tools/jhost.py
"""
import sys
import time

import numpy as np

sys.path.insert(0, ".")
sys.path.insert(0, "tools")
from kbench import LaunchDims, default_registry, dev_buf, fill_desc, i32, native  # noqa: E402


def chain_device_only(n=4096):
    k = default_registry().get("jacobi_sweep")
    s = native.Stream(0)
    rng = np.random.default_rng(0)
    A = rng.random((n, n), dtype=np.float32)
    A[np.arange(n), np.arange(n)] = A.sum(1) + 1
    b = (A.astype(np.float64) @ np.ones(n)).astype(np.float32)
    pA, pb = dev_buf(s, A.tobytes()), dev_buf(s, b.tobytes())
    px = [dev_buf(s, bytes(4 * n)) for _ in range(3)]
    pr = dev_buf(s, bytes(4))
    busy = native.malloc_async(s, 1 << 30)
    res = {}
    for sweeps in (2, 10, 100, 500):
        descs = (native.LaunchDesc * sweeps)()
        for t in range(sweeps):
            src = px[0] if t == 0 else px[1 + (t - 1) % 2]
            fill_desc(descs[t], k, LaunchDims(grid_x=n), (i32(n),), [pA, pb, src, px[1 + t % 2], pr],
                      [4 * n * n, 4 * n, 4 * n, 4 * n, 4])
        ts = []
        for _ in range(12):
            native.memset_async(busy, 0x5A, 1 << 30, s)  # also flushes L2
            e0, e1 = native.Event(0, True), native.Event(0, True)
            e0.record(s)
            t = time.perf_counter()
            native.launch_batch(0, s, descs)
            host = (time.perf_counter() - t) * 1e6
            e1.record(s)
            e1.sync()
            ts.append((e0.elapsed_ms(e1) * 1e3, host))
        ts = sorted(ts[2:])
        res[sweeps] = ts[len(ts) // 2][0]
        print(f"sweeps {sweeps:4d}: device {ts[len(ts) // 2][0]:8.1f} us  (launch_batch host {ts[len(ts) // 2][1]:.1f} us)",
              flush=True)
    x = np.array(list(res), float)
    y = np.array(list(res.values()), float)
    slope, icpt = np.polyfit(x, y, 1)
    print(f"device only: {slope:.3f} us/sweep + {icpt:.1f} us fixed")


def request_timeline(count=40):
    import bench
    from paper_2212_08146_b200.hoststore import PinnedStore
    from paper_2212_08146_b200.pool import KaasService
    store = PinnedStore()
    make = bench.jacobi_setup(store)
    svc = KaasService(store, n_executors=1, capacity=1 << 30, policy="rr", devices=[0])
    flush = bench.L2Flusher(0)
    bench.run_requests(svc, make, 5, 0, flush)
    marks = {}
    orig_lb, orig_sync = native.launch_batch, native.Event.sync

    def lb(*a, **kw):
        marks["lb0"] = time.perf_counter()
        r = orig_lb(*a, **kw)
        marks["lb1"] = time.perf_counter()
        return r

    def sync(self):
        r = orig_sync(self)
        marks["sync"] = time.perf_counter()
        return r
    native.launch_batch, native.Event.sync = lb, sync
    ex = svc.executors[0]
    rows = []
    for i in range(count):
        flush()
        r = make(100 + i)
        t0 = time.perf_counter()
        resp = svc.submit(r)
        t1 = time.perf_counter()
        assert resp.status.ok
        rows.append(((marks["lb0"] - t0) * 1e6, (marks["lb1"] - marks["lb0"]) * 1e6,
                     (marks["sync"] - marks["lb1"]) * 1e6, (t1 - marks["sync"]) * 1e6,
                     (t1 - t0) * 1e6, ex.dev_stats.last_kernel_ms * 1e3, ex.dev_stats.last_device_ms * 1e3))
    native.launch_batch, native.Event.sync = orig_lb, orig_sync
    med = np.median(np.array(rows), axis=0)
    print("request p50 (us): submit->launch_batch {:.1f}, launch_batch {:.1f}, ->last sync {:.1f}, "
          "sync->return {:.1f}, total {:.1f}; kernel span {:.1f}, device span {:.1f}".format(*med))
    svc.close()


if __name__ == "__main__":
    chain_device_only()
    request_timeline()
