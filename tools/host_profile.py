"""cProfile the host side of warm Jacobi / cGEMM requests (dev tool)."""

import cProfile
import pstats
import sys
import time

sys.path.insert(0, ".")
from paper_2212_08146_b200 import workloads as W  # noqa: E402
from paper_2212_08146_b200.hoststore import PinnedStore  # noqa: E402
from paper_2212_08146_b200.pool import KaasService  # noqa: E402


def main(kind="jacobi", n_req=30, n=1024):
    store = PinnedStore()
    if kind == "jacobi":
        W.seed_jacobi(store, 4096, prefix="j")
        mk = lambda i: W.jacobi_request(f"j/{i}", 4096, 500, "j/A/4096", "j/b/4096", "j/x0/4096",  # noqa: E731
                                        "j/x", "j/r")
    else:
        W.seed_cgemm(store, n, prefix="c")
        mk = lambda i: W.cgemm_request(f"c/{i}", n, f"c/A/{n}", f"c/B/{n}", "c/C")  # noqa: E731
    svc = KaasService(store, n_executors=1, capacity=4 << 30, policy="rr", devices=[0])
    ex = svc.executors[0]
    for i in range(3):
        svc.submit(mk(i))
    reqs = [mk(100 + i) for i in range(n_req)]
    pr = cProfile.Profile()
    t = time.perf_counter()
    pr.enable()
    dev = 0.0
    for r in reqs:
        svc.submit(r)
        dev += ex.dev_stats.last_device_ms
    pr.disable()
    wall = time.perf_counter() - t
    print(f"{kind}: wall {wall / n_req * 1e3:.3f} ms/req, device {dev / n_req:.3f} ms/req, "
          f"kernel {ex.dev_stats.last_kernel_ms:.3f} ms")
    pstats.Stats(pr).sort_stats("tottime").print_stats(18)
    svc.close()


if __name__ == "__main__":
    a = sys.argv[1:]
    main(a[0] if a else "jacobi", int(a[1]) if len(a) > 1 else 30, int(a[2]) if len(a) > 2 else 1024)
