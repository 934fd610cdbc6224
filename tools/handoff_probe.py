"""Dev: per-request wall time through KaasService.submit (queue + worker
thread + Future) vs GpuExecutor.execute called directly (same requests)."""
import statistics
import sys
import time

sys.path.insert(0, ".")
from paper_2212_08146_b200 import workloads as W  # noqa: E402
from paper_2212_08146_b200.hoststore import PinnedStore  # noqa: E402
from paper_2212_08146_b200.pool import KaasService  # noqa: E402

store = PinnedStore()
W.seed_jacobi(store, 4096, prefix="j")
svc = KaasService(store, n_executors=1, capacity=4 << 30, policy="rr", devices=[0])
ex = svc.executors[0]


def mk(i):
    return W.jacobi_request(f"j/{i}", 4096, 500, "j/A/4096", "j/b/4096", "j/x0/4096", "j/x", "j/r")


for i in range(5):
    svc.submit(mk(i))
from paper_2212_08146_b200.gpu_executor import ExecutorConfig, GpuExecutor  # noqa: E402


def timeit(label, fn, exr):
    ts = []
    for i in range(40):
        t = time.perf_counter()
        r = fn(mk(100 + i))
        ts.append((time.perf_counter() - t) * 1e3)
        assert r.status.ok
    print(f"{label:8s} p50 {statistics.median(ts):.3f} ms  mean {statistics.mean(ts):.3f} ms  "
          f"device {exr.dev_stats.last_device_ms:.3f} ms", flush=True)


timeit("submit", svc.submit, ex)
svc.close()
direct = GpuExecutor(ExecutorConfig(capacity=4 << 30), store)
for i in range(5):
    direct.execute(mk(i))
timeit("execute", direct.execute, direct)
direct.close()
svc = KaasService(store, n_executors=1, capacity=4 << 30, policy="rr", devices=[0])
for i in range(5):
    svc.submit(mk(i))
timeit("submit", svc.submit, svc.executors[0])
svc.close()
