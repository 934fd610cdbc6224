"""Dev: Jacobi chain time per launch under the bench's conditions -- back to
back, after a 256 MiB L2-flushing memset, and after an idle gap."""
import sys
import time

sys.path.insert(0, ".")
sys.path.insert(0, "tools")
import kbench  # noqa: E402
from paper_2212_08146_b200 import native  # noqa: E402
from paper_2212_08146_b200.api import LaunchDims, i32  # noqa: E402
from paper_2212_08146_b200.kernels import default_registry, fill_desc  # noqa: E402
import numpy as np  # noqa: E402

n, sweeps = 4096, 500
k = default_registry().get("jacobi_sweep")
s = native.Stream(0)
rng = np.random.default_rng(0)
A = rng.random((n, n), dtype=np.float32)
A[np.arange(n), np.arange(n)] = A.sum(1) + 1
b = A.astype(np.float64) @ np.ones(n)
pA = kbench.dev_buf(s, A.tobytes())
pb = kbench.dev_buf(s, b.astype(np.float32).tobytes())
px = [kbench.dev_buf(s, bytes(4 * n)) for _ in range(3)]
pr = kbench.dev_buf(s, bytes(4))
descs = (native.LaunchDesc * sweeps)()
for t in range(sweeps):
    src = px[0] if t == 0 else px[1 + (t - 1) % 2]
    fill_desc(descs[t], k, LaunchDims(grid_x=n), (i32(n),), [pA, pb, src, px[1 + t % 2], pr],
              [4 * n * n, 4 * n, 4 * n, 4 * n, 4])
flush = native.malloc_async(s, 256 << 20)
e0, e1 = native.Event(0, True), native.Event(0, True)


def one(pre):
    pre()
    e0.record(s)
    native.launch_batch(0, s, descs)
    e1.record(s)
    e1.sync()
    return e0.elapsed_ms(e1) * 1e3 / sweeps


modes = {
    "back-to-back": lambda: None,
    "after 256 MiB memset": lambda: native.memset_async(flush, 0, 256 << 20, s),
    "after 2 ms idle": lambda: time.sleep(0.002),
    "after memset + 2 ms idle": lambda: (native.memset_async(flush, 0, 256 << 20, s), s.sync(), time.sleep(0.002)),
}
for name, pre in modes.items():
    one(pre)
    v = sorted(one(pre) for _ in range(15))
    print(f"{name:28s} us/sweep  p50 {v[7]:.3f}  min {v[0]:.3f}  max {v[-1]:.3f}")

# host cost of one 500-invocation launch_batch call (descriptor walk, chain
# detection, ChainParams, cooperative launch) -- GPU idle inside the bench's
# kernel window when nothing else is queued
ts = []
for _ in range(20):
    s.sync()
    t = time.perf_counter()
    native.launch_batch(0, s, descs)
    ts.append((time.perf_counter() - t) * 1e6)
s.sync()
ts.sort()
print(f"launch_batch host time: p50 {ts[10]:.1f} us  min {ts[0]:.1f} us")
