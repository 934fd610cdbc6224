"""Dev: host time of each step of a warm Jacobi request's begin() (resolve
per buffer, plan, launch), by wrapping the executor's methods.

    python tools/jresolve.py
"""
import collections
import sys
import time

sys.path.insert(0, ".")
from paper_2212_08146_b200 import workloads as W  # noqa: E402
from paper_2212_08146_b200.gpu_executor import GpuExecutor  # noqa: E402
from paper_2212_08146_b200.hoststore import PinnedStore  # noqa: E402
from paper_2212_08146_b200.pool import KaasService  # noqa: E402

store = PinnedStore()
W.seed_jacobi(store, 4096, prefix="j")
mk = lambda i: W.jacobi_request(f"j/{i}", 4096, 500, "j/A/4096", "j/b/4096", "j/x0/4096", "j/x", "j/r")  # noqa
svc = KaasService(store, n_executors=1, capacity=4 << 30, policy="rr", devices=[0])
ex = svc.executors[0]
for i in range(5):
    svc.submit(mk(i))
acc = collections.defaultdict(float)
cnt = collections.defaultdict(int)


def wrap(obj, name, key=None):
    orig = getattr(obj, name)

    def f(*a, **k):
        t = time.perf_counter()
        try:
            return orig(*a, **k)
        finally:
            kk = key(a) if key else name
            acc[kk] += time.perf_counter() - t
            cnt[kk] += 1
    setattr(obj, name, f)


wrap(ex, "resolve_buffer", key=lambda a: f"resolve_buffer[{a[0].name}]")
for nm in ("_plan", "_launch", "_enqueue_flush", "_events", "_finish", "_release", "_alloc_zeroed", "_fetch_into",
           "_mark", "complete", "begin"):
    if hasattr(ex, nm):
        wrap(ex, nm)
wrap(svc, "submit")
from paper_2212_08146_b200 import native  # noqa: E402
import paper_2212_08146_b200.gpu_executor as GE  # noqa: E402
wrap(GE.native, "launch_batch")
wrap(type(ex.dev_stats), "resolve", key=lambda a: "dev_stats.resolve")
_orig_lib = native.load()


class _Timed:
    def __init__(self, lib):
        self._lib = lib

    def __getattr__(self, name):
        fn = getattr(self._lib, name)
        if not name.startswith("kaas_launch"):
            return fn

        def g(*a):
            t = time.perf_counter()
            try:
                return fn(*a)
            finally:
                acc["C " + name] += time.perf_counter() - t
                cnt["C " + name] += 1
        return g


native.load = lambda: _Timed(_orig_lib)
if ex.peers is not None:
    wrap(ex.peers, "borrow", key=lambda a: "peers.borrow")
    wrap(ex.peers, "publish", key=lambda a: "peers.publish")
wrap(ex.store, "get_versioned", key=lambda a: "store.get_versioned")
wrap(GE.native, "h2d_async", key=lambda a: "native.h2d_async")
wrap(native.Event, "record", key=lambda a: "Event.record")
wrap(native.Stream, "wait", key=lambda a: "Stream.wait")
for nm in ("_wait_for_user", "_fence_lends", "_clear_derived", "_alloc", "_derived_slot", "_attach_prepared"):
    if hasattr(ex, nm):
        wrap(ex, nm)
N = 50
for i in range(N):
    svc.submit(mk(100 + i))
for k in sorted(acc, key=lambda k: -acc[k]):
    print(f"{k:34s} {acc[k] / N * 1e6:8.1f} us/req  ({cnt[k] / N:.1f} calls/req)")
svc.close()
