"""Dev: per-request breakdown of the mixed multi-tenant workload (slowest requests)."""
import statistics
import sys
import time

sys.path.insert(0, ".")
from paper_2212_08146_b200 import workloads as W  # noqa: E402
from paper_2212_08146_b200.benchlib import run_stream  # noqa: E402
from paper_2212_08146_b200.hoststore import PinnedStore  # noqa: E402
from paper_2212_08146_b200.pool import KaasService  # noqa: E402

store = PinnedStore()
uni = W.mixed_universe(store)
reqs = W.mixed_requests(uni, 160)
with KaasService(store, n_executors=1, capacity=512 << 20, policy="affinity:8", devices=[0]) as svc:
    ex = svc.executors[0]
    log = []
    inner = ex.on_complete

    def hook(rec, resp):
        d = ex.dev_stats
        log.append((time.perf_counter(), resp.request_id, d.last_device_ms, d.last_kernel_ms,
                    resp.io_stats.bytes_fetched))
        if inner is not None:
            inner(rec, resp)
    ex.on_complete = hook
    run_stream(svc, reqs[:8], 1)
    for rep in range(3):
        log.clear()
        t0 = time.perf_counter()
        resps, lat = run_stream(svc, reqs, 16)
        wall = time.perf_counter() - t0
        dev = [x[2] for x in log]
        print(f"run {rep}: {len(reqs) / wall:.1f} req/s, wall {wall * 1e3:.0f} ms, sum device {sum(dev):.0f} ms, "
              f"p50 lat {statistics.median(lat) * 1e3:.1f} ms, max lat {max(lat) * 1e3:.0f} ms")
        gaps = sorted(((log[i][0] - log[i - 1][0]) * 1e3, i) for i in range(1, len(log)))[-5:]
        for g, i in gaps:
            print(f"   completion gap {g:7.1f} ms before {log[i][1]} (dev {log[i][2]:.2f} ms, kern {log[i][3]:.2f} ms, "
                  f"fetched {log[i][4] >> 20} MiB)")
        worst = sorted(log, key=lambda x: -x[2])[:5]
        for w in worst:
            print(f"   slow device span {w[2]:8.2f} ms  kern {w[3]:7.2f} ms  {w[1]}  fetched {w[4] >> 20} MiB")
