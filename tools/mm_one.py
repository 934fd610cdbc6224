"""Dev: run one bit-exact matmul request (a [fill, matmul] run) REPS times through
the executor, for an ncu capture of the run kernel on that shape.

    python tools/mm_one.py M N K [REPS]
"""

import sys

import numpy as np

sys.path.insert(0, ".")
from paper_2212_08146_b200 import native  # noqa: E402
from paper_2212_08146_b200.api import BufferArg, KaasRequest, KernelInvocation, LaunchDims, f32, i32  # noqa: E402
from paper_2212_08146_b200.gpu_executor import ExecutorConfig, GpuExecutor  # noqa: E402
from paper_2212_08146_b200.hoststore import PinnedStore  # noqa: E402

m, n, k = (int(a) for a in sys.argv[1:4])
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 6
native.init_device(0)
store = PinnedStore()
ex = GpuExecutor(ExecutorConfig(capacity=4 << 30), store)
rng = np.random.default_rng(0)
store.put("mo/a", rng.standard_normal(m * k, dtype=np.float32).tobytes())
store.put("mo/w", rng.standard_normal(k * n, dtype=np.float32).tobytes())
req = KaasRequest("mo", (
    BufferArg("a", 4 * m * k, "input", key="mo/a", is_const=True),
    BufferArg("w", 4 * k * n, "input", key="mo/w", is_const=True),
    BufferArg("z", 64, "inout", is_ephemeral=True),
    BufferArg("o", 4 * m * n, "inout", is_ephemeral=True)), (
    KernelInvocation("fill", LaunchDims(grid_x=16), (i32(16), f32(0.0)), ("z",)),
    KernelInvocation("matmul", LaunchDims(grid_x=m * n), (i32(m), i32(n), i32(k)), ("a", "w", "o"))))
for _ in range(reps):
    r = ex.execute(req)
    assert r.status.ok, r.status
print("ok")
