"""Dev: launch phases of the fused Jacobi chain kernel (dev build, stamps
from k_jacobi_tmem's prologue): CTA entry spread, TMEM alloc, band fill,
first sweeps, teardown.  L2 flushed before the traced launch.

    make -C paper_2212_08146_b200/csrc dev
    python tools/jpro.py [sweeps]
"""
import ctypes as C
import os
import sys

import numpy as np

os.environ.setdefault("KAAS_B200_LIB", "paper_2212_08146_b200/libkaas_b200_dev.so")
if not os.environ.get("JPRO_NOSTAMPS"):
    os.environ.setdefault("KAAS_JACOBI_TRACE", "1")
sys.path.insert(0, ".")
sys.path.insert(0, "tools")
from kbench import LaunchDims, default_registry, dev_buf, fill_desc, i32, native  # noqa: E402

n = 4096
sweeps = int(sys.argv[1]) if len(sys.argv) > 1 else 500
k = default_registry().get("jacobi_sweep")
s = native.Stream(0)
rng = np.random.default_rng(0)
A = rng.random((n, n), dtype=np.float32)
A[np.arange(n), np.arange(n)] = A.sum(1) + 1
b = (A.astype(np.float64) @ np.ones(n)).astype(np.float32)
pA, pb = dev_buf(s, A.tobytes()), dev_buf(s, b.tobytes())
px = [dev_buf(s, bytes(4 * n)) for _ in range(3)]
pr = dev_buf(s, bytes(4))
flush = native.malloc_async(s, 256 << 20)
dims = LaunchDims(grid_x=n)
descs = (native.LaunchDesc * sweeps)()
for i in range(sweeps):
    xi = px[0] if i == 0 else px[1 + (i - 1) % 2]
    xo = px[1 + i % 2]
    fill_desc(descs[i], k, dims, (i32(n),), [pA, pb, xi, xo, pr], [4 * n * n, 4 * n, 4 * n, 4 * n, 4])
lib = native.load()
times = []
for rep in range(int(os.environ.get("JPRO_REPS", "4"))):
    native.memset_async(flush, rep, 256 << 20, s)
    if os.environ.get("JPRO_IDLE"):  # the GPU idles before the launch (as in a request)
        s.sync()
    e0, e1 = native.Event(0, True), native.Event(0, True)
    e0.record(s)
    native.launch_batch(0, s, descs)
    e1.record(s)
    e1.sync()
    times.append(e0.elapsed_ms(e1))
ms = float(np.median(times[1:])) if len(times) > 1 else times[0]
if os.environ.get("JPRO_NOSTAMPS"):
    print(f"{os.environ['KAAS_B200_LIB']}: chain of {sweeps} sweeps: median {ms * 1e3:.1f} us over "
          f"{len(times) - 1} L2-flushed launches")
    sys.exit(0)
nst = 32 * 148 * 5
buf = (C.c_uint * (nst + 148 * 8))()
assert lib.kaas_dev_jacobi_trace(buf, C.sizeof(buf)) == 0
t = np.frombuffer(buf, dtype=np.uint32)[nst:].astype(np.int64).reshape(148, 8)[:, :6]
t = (t - t[:, 0].min()) % (1 << 32)
names = ["entry", "tmem allocated", "band filled", "sweep 0 published", "sweep 1 published", "teardown"]
print(f"chain of {sweeps} sweeps: {ms * 1e3:.1f} us event-timed (median, L2 flushed first)")
for i, nm in enumerate(names):
    print(f"{nm:20s} min {t[:, i].min() / 1e3:8.2f} us  median {np.median(t[:, i]) / 1e3:8.2f} us  max {t[:, i].max() / 1e3:8.2f} us")
