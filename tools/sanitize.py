"""Small requests through every kernel family, for compute-sanitizer runs
(tools/sanitize.sh): Jacobi on-chip chain (tagged exchange + grid barrier),
cGEMM (TMA + tcgen05, K chunks, split-K red.add, progressive write-back),
bit-exact matmul (cp.async ring, PDL), elementwise, reduce_sum."""

import sys

import numpy as np

sys.path.insert(0, ".")
from paper_2212_08146_b200 import workloads as W  # noqa: E402
from paper_2212_08146_b200.api import (BufferArg, KaasRequest, KernelInvocation,  # noqa: E402
                                       LaunchDims, f32, i32)
from paper_2212_08146_b200.gpu_executor import ExecutorConfig, GpuExecutor  # noqa: E402
from paper_2212_08146_b200.hoststore import PinnedStore  # noqa: E402

store = PinnedStore()
ex = GpuExecutor(ExecutorConfig(capacity=1 << 30), store)
n = 2048
W.seed_jacobi(store, n, prefix="sj")
reqs = [W.jacobi_request("sj", n, 12, f"sj/A/{n}", f"sj/b/{n}", f"sj/x0/{n}", "sj/x", "sj/r")]
for cn, key in ((256, "c256"), (1100, "c1100")):  # split-K path and the multi-panel path
    W.seed_cgemm(store, cn, prefix=key)
    reqs.append(W.cgemm_request(key, cn, f"{key}/A/{cn}", f"{key}/B/{cn}", f"{key}/C"))
rng = np.random.default_rng(1)
store.put("ma", rng.standard_normal(96 * 200, dtype=np.float32).tobytes())
store.put("mb", rng.standard_normal(200 * 72, dtype=np.float32).tobytes())
reqs.append(KaasRequest("mm", (
    BufferArg("a", 4 * 96 * 200, "input", key="ma", is_const=True),
    BufferArg("b", 4 * 200 * 72, "input", key="mb", is_const=True),
    BufferArg("o", 4 * 96 * 72, "output", key="mo"),
    BufferArg("t", 4 * 96 * 72, "inout", is_ephemeral=True),
    BufferArg("r", 4, "output", key="mr")), (
    KernelInvocation("matmul", LaunchDims(grid_x=96 * 72), (i32(96), i32(72), i32(200)), ("a", "b", "t")),
    KernelInvocation("saxpy", LaunchDims(grid_x=96 * 72), (i32(96 * 72), f32(0.5)), ("t", "t", "o")),
    KernelInvocation("vector_add", LaunchDims(grid_x=96 * 72), (i32(96 * 72),), ("o", "t", "t")),
    KernelInvocation("reduce_sum", LaunchDims(), (i32(96 * 72),), ("t", "r")))))
# invocation-run fusions: fill + add -> one pass, matmul + residual add -> fused store
store.put("fx", rng.standard_normal(96 * 72, dtype=np.float32).tobytes())
reqs.append(KaasRequest("fu", (
    BufferArg("a", 4 * 96 * 200, "input", key="ma", is_const=True),
    BufferArg("b", 4 * 200 * 72, "input", key="mb", is_const=True),
    BufferArg("x", 4 * 96 * 72, "input", key="fx"),
    BufferArg("s", 4 * 96 * 72, "inout", is_ephemeral=True),
    BufferArg("d", 4 * 96 * 72, "output", key="fd")), (
    KernelInvocation("fill", LaunchDims(grid_x=96 * 72), (i32(96 * 72), f32(0.0)), ("s",)),
    KernelInvocation("vector_add", LaunchDims(grid_x=96 * 72), (i32(96 * 72),), ("x", "s", "s")),
    KernelInvocation("matmul", LaunchDims(grid_x=96 * 72), (i32(96), i32(72), i32(200)), ("a", "b", "d")),
    KernelInvocation("vector_add", LaunchDims(grid_x=96 * 72), (i32(96 * 72),), ("d", "s", "d")))))
for rep in range(2):  # second pass: const hits, prepared operands, memoised chain
    for r in reqs:
        resp = ex.execute(r)
        assert resp.status.ok, resp.status
ex.close()
print("sanitize workload ok")
