"""Dev: where the host time of a warm Jacobi request goes (cProfile over
KaasService.submit, BASELINE configs[1] shape)."""
import cProfile
import pstats
import sys
import time

sys.path.insert(0, ".")
from paper_2212_08146_b200 import workloads as W  # noqa: E402
from paper_2212_08146_b200.hoststore import PinnedStore  # noqa: E402
from paper_2212_08146_b200.pool import KaasService  # noqa: E402
from paper_2212_08146_b200.gpu_executor import GpuExecutor  # noqa: E402

if len(sys.argv) > 1 and sys.argv[1] == "norecycle":
    GpuExecutor.recycle_blocks = False

store = PinnedStore()
W.seed_jacobi(store, 4096, prefix="j")
req = lambda i: W.jacobi_request(f"j/{i}", 4096, 500, "j/A/4096", "j/b/4096", "j/x0/4096", "j/x", "j/r")  # noqa
svc = KaasService(store, capacity=1 << 30, policy="rr", devices=[0])
for i in range(20):
    svc.submit(req(i))
ex = svc.executors[0]
h0 = ex.dev_stats.host_ms
t = time.perf_counter()
for i in range(100):
    svc.submit(req(100 + i))
wall = time.perf_counter() - t
print(f"wall {wall / 100 * 1e6:.1f} us/request, executor host time {(ex.dev_stats.host_ms - h0) / 100 * 1e3:.1f} us/request")
if len(sys.argv) > 2:
    sys.exit(0)
pr = cProfile.Profile()
pr.enable()
for i in range(200):
    svc.submit(req(1000 + i))
pr.disable()
st = pstats.Stats(pr)
st.sort_stats("tottime").print_stats(30)
st.sort_stats("cumulative").print_callees("_begin")
st.print_callees("_complete")
st.print_callees("_launch")
svc.close()
