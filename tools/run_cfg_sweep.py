"""Dev: time every matmul tile configuration of the invocation-run kernel on the
ResNet-50 layer shapes (dev build: KAAS_RUN_CFG="cfg,per" forces one).

    make -C paper_2212_08146_b200/csrc dev
    python tools/run_cfg_sweep.py [layer-name-substring]

Each request is [fill, matmul] (a run of two); the matmul task's span comes
from the run kernel's dev trace (first CTA start to last CTA end), median of
3.  Prints, per distinct shape, the cost model's pick and the five fastest
configurations.
"""

import ctypes as C
import os
import statistics
import sys

import numpy as np

sys.path.insert(0, ".")
os.environ.setdefault("KAAS_B200_LIB", "paper_2212_08146_b200/libkaas_b200_dev.so")
os.environ.setdefault("KAAS_RUN_TRACE", "1")
from paper_2212_08146_b200 import native  # noqa: E402
from paper_2212_08146_b200 import workloads as W  # noqa: E402
from paper_2212_08146_b200.api import BufferArg, KaasRequest, KernelInvocation, LaunchDims, f32, i32  # noqa: E402
from paper_2212_08146_b200.gpu_executor import ExecutorConfig, GpuExecutor  # noqa: E402
from paper_2212_08146_b200.hoststore import PinnedStore  # noqa: E402

SUB = sys.argv[1] if len(sys.argv) > 1 else ""
# (ty, tx, tm, tn) by index -- must match kCfgs in csrc/runs.cu
BT = [(16, 16, 4, 4), (16, 16, 2, 4), (16, 16, 4, 2), (16, 16, 2, 2), (16, 16, 1, 2), (16, 16, 2, 1), (16, 16, 1, 1),
      (64, 4, 1, 1), (16, 8, 1, 2), (8, 16, 2, 2), (16, 8, 2, 2), (32, 4, 2, 1), (8, 8, 2, 2), (4, 16, 2, 2),
      (16, 4, 2, 2), (32, 2, 2, 2), (1, 64, 1, 4), (1, 256, 1, 1)]
CFGS = list(enumerate(BT))
meta = (C.c_int * (7 * 128))()
stamps = (C.c_uint * (128 * 1024 * 2))()
nt, grid = C.c_int(), C.c_int()


def mm_span_us():
    rc = native.load().kaas_dev_run_trace(meta, len(meta), stamps, len(stamps), C.byref(nt), C.byref(grid))
    assert rc == 0, rc
    n, g = nt.value, grid.value
    s = np.frombuffer(stamps, dtype=np.uint32)[: n * g * 2].astype(np.int64).reshape(n, g, 2)
    t = n - 1  # the matmul is the last task
    return ((s[t, :, 1].max() - s[t, :, 0].min()) % (1 << 32)) / 1e3


native.init_device(0)
store = PinnedStore()
ex = GpuExecutor(ExecutorConfig(capacity=4 << 30), store)
rng = np.random.default_rng(0)
seen = set()
for name, m, n, k in W.resnet50_gemms():
    if (m, n, k) in seen or SUB not in name or k % 4:
        continue
    seen.add((m, n, k))
    store.put(f"sw/a/{name}", rng.standard_normal(m * k, dtype=np.float32).tobytes())
    store.put(f"sw/w/{name}", rng.standard_normal(k * n, dtype=np.float32).tobytes())
    req = KaasRequest(f"sw/{name}", (
        BufferArg("a", 4 * m * k, "input", key=f"sw/a/{name}", is_const=True),
        BufferArg("w", 4 * k * n, "input", key=f"sw/w/{name}", is_const=True),
        BufferArg("z", 64, "inout", is_ephemeral=True),
        BufferArg("o", 4 * m * n, "inout", is_ephemeral=True)), (
        KernelInvocation("fill", LaunchDims(grid_x=16), (i32(16), f32(0.0)), ("z",)),
        KernelInvocation("matmul", LaunchDims(grid_x=m * n), (i32(m), i32(n), i32(k)), ("a", "w", "o"))))

    def timed():
        ts = []
        for _ in range(3):
            r = ex.execute(req)
            assert r.status.ok, r.status
            ts.append(mm_span_us())
        return statistics.median(ts)

    os.environ.pop("KAAS_RUN_CFG", None)
    timed()
    model = timed()
    res = []
    for idx, c in CFGS:
        for per in range(1, 5):
            if per > 256 // (c[0] * c[1]):
                break
            os.environ["KAAS_RUN_CFG"] = f"{idx},{per}"
            try:
                res.append((timed(), idx, per, c))
            except AssertionError as e:
                print("  fail", idx, per, e)
    os.environ.pop("KAAS_RUN_CFG", None)
    res.sort()
    best = " | ".join(f"{t:6.1f} us cfg {i:2d}x{p} {c}" for t, i, p, c in res[:5])
    print(f"{name:10s} {m}x{n}x{k}: model pick {model:6.1f} us; best: {best}", flush=True)
