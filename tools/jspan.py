"""Dev: where a Jacobi request's device time goes.

1. The fused chain kernel alone at 1..500 sweeps, after an L2 flush: the
   intercept is the per-launch fixed cost (launch, band fill from HBM, first
   exchange), the slope the per-sweep cost.
2. 40 bench requests: device span vs kernel span vs x0 fill span.

    python tools/jspan.py
"""
import sys

import numpy as np

sys.path.insert(0, ".")
sys.path.insert(0, "tools")
from kbench import LaunchDims, default_registry, dev_buf, fill_desc, i32, native  # noqa: E402


def chain_fixed(n=4096):
    k = default_registry().get("jacobi_sweep")
    s = native.Stream(0)
    rng = np.random.default_rng(0)
    A = rng.random((n, n), dtype=np.float32)
    A[np.arange(n), np.arange(n)] = A.sum(1) + 1
    b = (A.astype(np.float64) @ np.ones(n)).astype(np.float32)
    pA, pb = dev_buf(s, A.tobytes()), dev_buf(s, b.tobytes())
    px = [dev_buf(s, bytes(4 * n)) for _ in range(3)]
    pr = dev_buf(s, bytes(4))
    flush = native.malloc_async(s, 256 << 20)
    rows = []
    for sweeps in (1, 2, 10, 100, 500):
        descs = (native.LaunchDesc * sweeps)()
        for t in range(sweeps):
            src = px[0] if t == 0 else px[1 + (t - 1) % 2]
            fill_desc(descs[t], k, LaunchDims(grid_x=n), (i32(n),), [pA, pb, src, px[1 + t % 2], pr],
                      [4 * n * n, 4 * n, 4 * n, 4 * n, 4])
        for cold in (False, True):
            ts = []
            for _ in range(12):
                if cold:
                    native.memset_async(flush, 0x5A, 256 << 20, s)
                e0, e1 = native.Event(0, True), native.Event(0, True)
                e0.record(s)
                native.launch_batch(0, s, descs)
                e1.record(s)
                e1.sync()
                ts.append(e0.elapsed_ms(e1) * 1e3)
            ts = sorted(ts[2:])
            rows.append((sweeps, cold, ts[len(ts) // 2]))
            print(f"sweeps {sweeps:4d} {'flushed' if cold else 'warm   '} chain p50 {ts[len(ts) // 2]:8.1f} us", flush=True)
    for cold in (False, True):
        pts = [(sw, t) for sw, c, t in rows if c == cold]
        x = np.array([p[0] for p in pts], float)
        y = np.array([p[1] for p in pts], float)
        slope, icpt = np.polyfit(x, y, 1)
        print(f"{'flushed' if cold else 'warm'}: {slope:.3f} us/sweep + {icpt:.1f} us fixed")


def request_spans(count=40):
    import bench
    from paper_2212_08146_b200.hoststore import PinnedStore
    from paper_2212_08146_b200.pool import KaasService
    store = PinnedStore()
    make = bench.jacobi_setup(store)
    svc = KaasService(store, n_executors=1, capacity=1 << 30, policy="rr", devices=[0])
    flush = bench.L2Flusher(0)
    bench.run_requests(svc, make, 5, 0, flush)
    ex = svc.executors[0]
    dev, kern, fill = [], [], []
    for i in range(count):
        flush()
        h0 = ex.dev_stats.h2d_ms
        r = svc.submit(make(100 + i))
        assert r.status.ok
        dev.append(ex.dev_stats.last_device_ms * 1e3)
        kern.append(ex.dev_stats.last_kernel_ms * 1e3)
        fill.append((ex.dev_stats.h2d_ms - h0) * 1e3)
    med = lambda v: sorted(v)[len(v) // 2]  # noqa: E731
    print(f"request p50: device {med(dev):.1f} us, kernels {med(kern):.1f} us, x0 fill {med(fill):.1f} us")
    svc.close()


if __name__ == "__main__":
    chain_fixed()
    request_spans()
