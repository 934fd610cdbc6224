"""Dev: host timeline of one warm Jacobi request (perf_counter at each step of
begin(): plan, each resolve_buffer, _launch, flush, release) -- light wrappers,
so the absolute numbers are close to the unwrapped path.

    python tools/jtimeline.py
"""
import statistics
import sys
import time

sys.path.insert(0, ".")
from paper_2212_08146_b200 import workloads as W  # noqa: E402
from paper_2212_08146_b200.hoststore import PinnedStore  # noqa: E402
from paper_2212_08146_b200.pool import KaasService  # noqa: E402

store = PinnedStore()
W.seed_jacobi(store, 4096, prefix="j")
mk = lambda i: W.jacobi_request(f"j/{i}", 4096, 500, "j/A/4096", "j/b/4096", "j/x0/4096", "j/x", "j/r")  # noqa
svc = KaasService(store, n_executors=1, capacity=4 << 30, policy="rr", devices=[0])
ex = svc.executors[0]
for i in range(5):
    svc.submit(mk(i))
marks = []
T = time.perf_counter


def wrap(obj, name, label):
    orig = getattr(obj, name)

    def f(*a, **k):
        marks.append((label(a) + ">", T()))
        try:
            return orig(*a, **k)
        finally:
            marks.append(("<" + label(a), T()))
    setattr(obj, name, f)


wrap(ex, "resolve_buffer", lambda a: f"resolve[{a[0].name}]")
for nm in ("_plan", "_launch", "_enqueue_flush", "_release", "_finish", "complete"):
    wrap(ex, nm, lambda a, nm=nm: nm)
rows = {}
for i in range(60):
    marks.clear()
    t0 = T()
    svc.submit(mk(100 + i))
    t1 = T()
    for lab, t in marks:
        rows.setdefault(lab, []).append((t - t0) * 1e6)
    rows.setdefault("submit returns", []).append((t1 - t0) * 1e6)
order = sorted(rows, key=lambda k: statistics.median(rows[k]))
for k in order:
    print(f"{statistics.median(rows[k]):9.1f} us  {k}")
svc.close()
