"""Dev: does the fused Jacobi chain's speed depend on which stream (hence
which per-stream exchange scratch) it runs on -- or, with JMODE=xt and the
dev build, on which window of the stream's exchange pool
(KAAS_JACOBI_XT_SEL)?  One process, L2 flushed before each launch.

    python tools/jstreams.py [count]
    JMODE=xt KAAS_B200_LIB=paper_2212_08146_b200/libkaas_b200_dev.so python tools/jstreams.py 16
"""
import os
import sys

import numpy as np

sys.path.insert(0, ".")
sys.path.insert(0, "tools")
from kbench import LaunchDims, default_registry, dev_buf, fill_desc, i32, native  # noqa: E402

n, sweeps = 4096, 500
nst = int(sys.argv[1]) if len(sys.argv) > 1 else 6
k = default_registry().get("jacobi_sweep")
s0 = native.Stream(0)
rng = np.random.default_rng(0)
A = rng.random((n, n), dtype=np.float32)
A[np.arange(n), np.arange(n)] = A.sum(1) + 1
b = (A.astype(np.float64) @ np.ones(n)).astype(np.float32)
pA, pb = dev_buf(s0, A.tobytes()), dev_buf(s0, b.tobytes())
px = [dev_buf(s0, bytes(4 * n)) for _ in range(3)]
pr = dev_buf(s0, bytes(4))
flush = native.malloc_async(s0, 256 << 20)
s0.sync()
dims = LaunchDims(grid_x=n)
descs = (native.LaunchDesc * sweeps)()
for i in range(sweeps):
    xi = px[0] if i == 0 else px[1 + (i - 1) % 2]
    fill_desc(descs[i], k, dims, (i32(n),), [pA, pb, xi, px[1 + i % 2], pr], [4 * n * n, 4 * n, 4 * n, 4 * n, 4])
mode = os.environ.get("JMODE", "streams")
streams = [native.Stream(0) for _ in range(nst)] if mode == "streams" else [native.Stream(0)] * nst
for rnd in range(2):
    for si, s in enumerate(streams):
        if mode == "xt":
            os.environ["KAAS_JACOBI_XT_SEL"] = str(si)
        t = []
        for rep in range(8):
            native.memset_async(flush, rep, 256 << 20, s)
            e0, e1 = native.Event(0, True), native.Event(0, True)
            e0.record(s)
            native.launch_batch(0, s, descs)
            e1.record(s)
            e1.sync()
            t.append(e0.elapsed_ms(e1))
        print(f"round {rnd} {mode} {si}: median {np.median(t[1:]) * 1e3:.1f} us", flush=True)
