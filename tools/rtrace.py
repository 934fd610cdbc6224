"""Dev: per-task timeline of the invocation-run kernel on the ResNet-50 chain.

    make -C paper_2212_08146_b200/csrc dev   # the trace exists only in the dev build
    python tools/rtrace.py [--cfg N]

Each CTA stamps (globaltimer) the start of a task (after its dependency wait)
and the end of its items.  Per task: op, shape, tile config, items, the task
it waits for, when its first CTA started / last CTA finished relative to the
launch, and its span.  Summary: kernel time, time in matmul spans, gaps.
"""

import ctypes as C
import os
import sys

import numpy as np

sys.path.insert(0, ".")
os.environ.setdefault("KAAS_RUN_TRACE", "1")
os.environ.setdefault("KAAS_B200_LIB", "paper_2212_08146_b200/libkaas_b200_dev.so")
from paper_2212_08146_b200 import native  # noqa: E402
from paper_2212_08146_b200 import workloads as W  # noqa: E402
from paper_2212_08146_b200.gpu_executor import ExecutorConfig, GpuExecutor  # noqa: E402
from paper_2212_08146_b200.hoststore import PinnedStore  # noqa: E402

OPS = ["mm", "add", "saxpy", "fill", "reduce", "transpose", "copy", "addc"]

native.init_device(0)
store = PinnedStore()
W.seed_resnet(store)
ex = GpuExecutor(ExecutorConfig(capacity=1 << 30), store)
for i in range(3):
    r = ex.execute(W.resnet_chain_request(f"rt/{i}"))
    assert r.status.ok, r.status
print(f"kernel ms (last request): {ex.dev_stats.last_kernel_ms:.3f}")
meta = (C.c_int * (7 * 128))()
stamps = (C.c_uint * (128 * 1024 * 2))()
nt, grid = C.c_int(), C.c_int()
rc = native.load().kaas_dev_run_trace(meta, len(meta), stamps, len(stamps), C.byref(nt), C.byref(grid))
assert rc == 0, rc
n, G = nt.value, grid.value
m = np.frombuffer(meta, dtype=np.int32)[: 7 * n].reshape(n, 7)
s = np.frombuffer(stamps, dtype=np.uint32)[: n * G * 2].astype(np.int64).reshape(n, G, 2)
t0 = s[:, :, 0].min()
s = (s - t0) % (1 << 32)
mm_total = 0
rows = []
for t in range(n):
    op, cfg, wait, items, nn, mm, kk = m[t]
    busy = [(b + 0) for b in range(G)]  # all CTAs stamp every task
    start = s[t, :, 0].min()
    end = s[t, :, 1].max()
    span = end - start
    if OPS[op] == "mm":
        mm_total += span
    rows.append((t, OPS[op], cfg, wait, items, nn, mm, kk, start, end, span))
    shape = f"{nn}x{mm}x{kk}" if OPS[op] in ("mm", "transpose") else ""
    print(f"{t:3d} {OPS[op]:9s} cfg {cfg:2d} wait {wait:3d} items {items:5d} {shape:16s} "
          f"start {start / 1e3:8.2f} us end {end / 1e3:8.2f} us span {span / 1e3:7.2f} us")
end_all = s[:, :, 1].max()
print(f"launch span {end_all / 1e3:.1f} us; matmul task spans sum {mm_total / 1e3:.1f} us; tasks {n}, grid {G}")
