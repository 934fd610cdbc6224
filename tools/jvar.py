"""Dev: per-request device/kernel time of the bench's Jacobi request (variance hunt)."""
import sys
import time

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_2212_08146_b200 import native  # noqa: E402
from paper_2212_08146_b200.hoststore import PinnedStore  # noqa: E402
from paper_2212_08146_b200.pool import KaasService  # noqa: E402

native.init_device(0)
store = PinnedStore()
make_req = bench.jacobi_setup(store)
svc = KaasService(store, n_executors=1, capacity=1 << 30, policy="rr", devices=[0])
ex = svc.executors[0]
flush = bench.L2Flusher(0) if "--flush" in sys.argv else None
for i in range(60):
    if flush:
        flush()
    t = time.perf_counter()
    svc.submit(make_req(i))
    w = (time.perf_counter() - t) * 1e3
    print(f"{i:3d} wall {w:6.3f} dev {ex.dev_stats.last_device_ms:6.3f} kern {ex.dev_stats.last_kernel_ms:6.3f}")
svc.close()
