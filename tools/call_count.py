"""Dev: C-ABI calls (name -> count, host us) per warm Jacobi request."""
import collections
import sys
import time

sys.path.insert(0, ".")
from paper_2212_08146_b200 import native  # noqa: E402
from paper_2212_08146_b200 import workloads as W  # noqa: E402
from paper_2212_08146_b200.hoststore import PinnedStore  # noqa: E402
from paper_2212_08146_b200.pool import KaasService  # noqa: E402

store = PinnedStore()
W.seed_jacobi(store, 4096, prefix="j")
svc = KaasService(store, n_executors=1, capacity=4 << 30, policy="rr", devices=[0])


def mk(i):
    return W.jacobi_request(f"j/{i}", 4096, 500, "j/A/4096", "j/b/4096", "j/x0/4096", "j/x", "j/r")


for i in range(5):
    svc.submit(mk(i))
counts = collections.Counter()
times = collections.Counter()
orig = native.call


def counting(name, *args):
    t = time.perf_counter()
    orig(name, *args)
    counts[name] += 1
    times[name] += time.perf_counter() - t


native.call = counting
N = 20
for i in range(N):
    svc.submit(mk(100 + i))
native.call = orig
for name, c in counts.most_common():
    print(f"{name:28s} {c / N:5.1f} per request  {times[name] / c * 1e6:8.1f} us each")
svc.close()
