"""Dev: speculative Jacobi chain start on/off (needs the reverted patch
profiles/r02/probes/jacobi_speculative_start.diff; --off-only on the product), interleaved blocks of warm
N=4096 x 500-sweep requests under the bench's conditions (L2 flushed before
each request, outside the timed span): submit latency and device span."""
import statistics
import sys
import time

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_2212_08146_b200 import native  # noqa: E402
from paper_2212_08146_b200.hoststore import PinnedStore  # noqa: E402
from paper_2212_08146_b200.pool import KaasService  # noqa: E402

native.init_device(0)
store = PinnedStore()
mk = bench.jacobi_setup(store)
svc = KaasService(store, n_executors=1, capacity=1 << 30, policy="rr", devices=[0])
ex = svc.executors[0]
flush = bench.L2Flusher(0)
for i in range(5):
    svc.submit(mk(i))
res = {True: ([], [], []), False: ([], [], [])}
i = 100
modes = (False,) if "--off-only" in sys.argv else (True, False)
for rnd in range(8):
    for spec in modes if rnd % 2 == 0 else modes[::-1]:
        ex.speculative = spec
        lat, dev, kern = bench.run_requests(svc, mk, 25, i, flush)
        i += 25
        res[spec][0].extend(lat[2:])
        res[spec][1].extend(dev[2:])
        res[spec][2].extend(kern[2:])
for spec, (lat, dev, kern) in res.items():
    if not lat:
        continue
    print(f"speculative={spec!s:5}: submit p50 {statistics.median(lat) * 1e3:.4f} ms "
          f"(mean {statistics.fmean(lat) * 1e3:.4f}, {1 / statistics.fmean(lat):.1f} req/s)  "
          f"device p50 {statistics.median(dev):.4f} ms  kernel p50 {statistics.median(kern):.4f} ms")
print("spec launches", getattr(ex, "spec_launches", None))
svc.close()
