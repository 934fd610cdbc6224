"""Dev: device-side phases of warm Jacobi requests from the executor's own
events: ev0 (first op) -> ev2 (kernel launch point) -> ev3 (kernel end) ->
ev1 (flush copies done).

    python tools/jtail.py
"""
import statistics
import sys

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
ds = ex.dev_stats
cls = type(ds)
orig = cls.defer
rows = []


def defer(self, events, hk, hf):
    ev = events
    ev[1].sync()
    rows.append((ev[0].elapsed_ms(ev[5]) * 1e3 if hf else 0.0, ev[0].elapsed_ms(ev[2]) * 1e3,
                 ev[2].elapsed_ms(ev[3]) * 1e3, ev[3].elapsed_ms(ev[1]) * 1e3, ev[0].elapsed_ms(ev[1]) * 1e3))
    return orig(self, events, hk, hf)


cls.defer = defer
for i in range(50):
    svc.submit(mk(100 + i))
for j, nm in enumerate(["ev0 -> fills done", "ev0 -> launch point (ev2)", "kernel span ev2 -> ev3",
                        "kernel end -> flush done (ev3 -> ev1)", "device span ev0 -> ev1"]):
    print(f"{nm:40s} median {statistics.median(r[j] for r in rows):8.1f} us")
svc.close()
