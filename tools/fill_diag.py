"""Dev: cold cache-fill bandwidth -- raw pinned H2D vs the executor's fills."""
import statistics
import sys
import time

sys.path.insert(0, ".")
from paper_2212_08146_b200 import native  # noqa: E402
from paper_2212_08146_b200 import workloads as W  # noqa: E402
from paper_2212_08146_b200.hoststore import PinnedBlob, PinnedStore  # noqa: E402
from paper_2212_08146_b200.pool import KaasService  # noqa: E402

native.init_device(0)
s = native.Stream(0)
for mb in (8, 64, 512):
    blob = PinnedBlob(mb << 20)
    d = native.malloc_async(s, mb << 20)
    e0, e1 = native.Event(0, True), native.Event(0, True)
    native.h2d_async(d, blob.addr, mb << 20, s)
    s.sync()
    v = []
    for _ in range(5):
        e0.record(s)
        native.h2d_async(d, blob.addr, mb << 20, s)
        e1.record(s)
        e1.sync()
        v.append((mb << 20) / (e0.elapsed_ms(e1) * 1e6))
    print(f"raw pinned H2D {mb:4d} MiB: {statistics.median(v):6.1f} GB/s")

for n in (1024, 8192):
    store = PinnedStore()
    for c in range(4):
        W.seed_cgemm(store, n, prefix=f"c{c}", seed=c)
    cap = 16 * n * n * 8
    with KaasService(store, n_executors=1, capacity=cap, policy="rr", devices=[0],
                     reserve_bytes=cap + 64 * n * n) as svc:
        ex = svc.executors[0]
        for c in range(4):
            h0, b0 = ex.dev_stats.h2d_ms, ex.dev_stats.h2d_bytes
            t = time.perf_counter()
            r = svc.submit(W.cgemm_request(f"c{c}/r", n, f"c{c}/A/{n}", f"c{c}/B/{n}", f"c{c}/C"))
            wall = (time.perf_counter() - t) * 1e3
            ms = ex.dev_stats.h2d_ms - h0
            print(f"cgemm {n} cold request {c}: fills {(ex.dev_stats.h2d_bytes - b0) >> 20} MiB in {ms:.2f} ms "
                  f"= {(ex.dev_stats.h2d_bytes - b0) / (ms * 1e6):.1f} GB/s; request {wall:.1f} ms, "
                  f"pinned src: {type(store.get(f'c{c}/A/{n}')).__name__}")
