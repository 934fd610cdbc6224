"""Dev: which C-ABI calls a warm Jacobi request makes, and the host time in
each (native.call wrapped; perf_counter around every crossing), plus the
request's host phases.

    python tools/jcalls.py
"""
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
mk = lambda i: W.jacobi_request(f"j/{i}", 4096, 500, "j/A/4096", "j/b/4096", "j/x0/4096", "j/x", "j/r")  # noqa
svc = KaasService(store, n_executors=1, capacity=4 << 30, policy="rr", devices=[0])
for i in range(5):
    svc.submit(mk(i))
stats = collections.defaultdict(lambda: [0, 0.0])
orig = native.call
log = []


def wrapped(name, *args):
    t = time.perf_counter()
    try:
        return orig(name, *args)
    finally:
        dt = time.perf_counter() - t
        stats[name][0] += 1
        stats[name][1] += dt
        log.append((name, t, dt))


native.call = wrapped
N = 40
reqs = [mk(100 + i) for i in range(N)]
t0s = []
for r in reqs:
    log.clear()
    t0 = time.perf_counter()
    svc.submit(r)
    t1 = time.perf_counter()
    t0s.append((t0, t1, list(log)))
native.call = orig
print(f"per request over {N} warm requests: {sum(t1 - t0 for t0, t1, _ in t0s) / N * 1e6:.1f} us wall")
for name, (c, dt) in sorted(stats.items(), key=lambda kv: -kv[1][1]):
    print(f"  {name:34s} calls/req {c / N:5.1f}   host us/req {dt / N * 1e6:8.1f}")
t0, t1, lg = t0s[-1]
print("timeline of the last request (us from submit):")
for name, t, dt in lg:
    print(f"  {(t - t0) * 1e6:8.1f} +{dt * 1e6:7.1f}  {name}")
print(f"  {(t1 - t0) * 1e6:8.1f}  submit returns")
svc.close()
