"""Quick end-to-end probe of the native path on a GPU box (dev tool).

Runs each kernel through GpuExecutor on small random inputs, compares with a
numpy restatement, and times the two headline kernels.  Prints one line per
check; exits non-zero on the first mismatch.
"""

import sys
import time

import numpy as np

sys.path.insert(0, ".")
from paper_2212_08146_b200 import native  # noqa: E402
from paper_2212_08146_b200.api import BufferArg, KaasRequest, KernelInvocation, LaunchDims, f32, i32  # noqa: E402
from paper_2212_08146_b200.gpu_executor import ExecutorConfig, GpuExecutor  # noqa: E402
from paper_2212_08146_b200.hoststore import PinnedStore  # noqa: E402

F32 = np.float32
rng = np.random.default_rng(0)


def grid(cells):
    b = min(256, max(1, cells))
    return LaunchDims(grid_x=max(1, -(-cells // b)), block_x=b)


def run(ex, store, req):
    t = time.perf_counter()
    r = ex.execute(req)
    dt = time.perf_counter() - t
    if not r.status.ok:
        print("FAIL", req.request_id, r.status)
        sys.exit(1)
    return r, dt


def main():
    print("devices", native.device_count(), native.device_info(0).name, flush=True)
    store = PinnedStore()
    ex = GpuExecutor(ExecutorConfig(capacity=40 << 30), store)

    # vector_add / saxpy / fill / reduce
    n = 100003
    x = rng.standard_normal(n).astype(F32)
    y = rng.standard_normal(n).astype(F32)
    store.put("x", x.tobytes())
    store.put("y", y.tobytes())
    req = KaasRequest("ew", buffers=(
        BufferArg("x", 4 * n, "input", key="x", is_const=True),
        BufferArg("y", 4 * n, "input", key="y", is_const=True),
        BufferArg("o1", 4 * n, "output", key="o1"),
        BufferArg("o2", 4 * n, "output", key="o2"),
        BufferArg("o3", 4 * n, "output", key="o3"),
        BufferArg("o4", 4, "output", key="o4"),
    ), invocations=(
        KernelInvocation("vector_add", LaunchDims(grid_x=n - 5), (i32(n),), ("x", "y", "o1")),
        KernelInvocation("saxpy", grid(n), (i32(n), f32(1.7)), ("x", "y", "o2")),
        KernelInvocation("fill", grid(n), (i32(n), f32(-2.25)), ("o3",)),
        KernelInvocation("reduce_sum", LaunchDims(), (i32(n),), ("x", "o4")),
    ))
    run(ex, store, req)
    exp1 = np.zeros(n, F32)
    exp1[: n - 5] = x[: n - 5] + y[: n - 5]
    ok = [
        np.frombuffer(bytes(store.get("o1")), F32).tobytes() == exp1.tobytes(),
        np.frombuffer(bytes(store.get("o2")), F32).tobytes() == (F32(1.7) * x + y).tobytes(),
        np.frombuffer(bytes(store.get("o3")), F32).tobytes() == np.full(n, -2.25, F32).tobytes(),
        np.frombuffer(bytes(store.get("o4")), F32)[0] == np.add.accumulate(x)[-1],
    ]
    print("elementwise+reduce bit-exact:", ok, flush=True)

    # matmul bit-exact
    for (mn, mm, mk) in [(7, 5, 3), (64, 64, 64), (130, 70, 33), (300, 200, 147)]:
        a = (rng.standard_normal(mn * mk) * 3).astype(F32)
        b = (rng.standard_normal(mk * mm) * 3).astype(F32)
        store.put("ma", a.tobytes())
        store.put("mb", b.tobytes())
        req = KaasRequest("mm", buffers=(
            BufferArg("a", a.nbytes, "input", key="ma"),
            BufferArg("b", b.nbytes, "input", key="mb"),
            BufferArg("c", 4 * mn * mm, "output", key="mc")),
            invocations=(KernelInvocation("matmul", grid(mn * mm), (i32(mn), i32(mm), i32(mk)), ("a", "b", "c")),))
        run(ex, store, req)
        A = a.reshape(mn, mk)
        B = b.reshape(mk, mm)
        acc = np.zeros((mn, mm), F32)
        for kk in range(mk):
            acc += A[:, kk:kk + 1] * B[kk:kk + 1, :]
        got = np.frombuffer(bytes(store.get("mc")), F32)
        print(f"matmul {mn}x{mm}x{mk} bit-exact:", got.tobytes() == acc.tobytes(), flush=True)

    # jacobi
    N = 4096
    A = rng.random((N, N), dtype=F32)
    np.fill_diagonal(A, 0)
    A[np.arange(N), np.arange(N)] = A.sum(1) + 1
    A = A.astype(F32)
    bvec = (A.astype(np.float64) @ np.ones(N)).astype(F32)
    store.put("jA", A.tobytes())
    store.put("jb", bvec.tobytes())
    store.put("jx0", np.zeros(N, F32).tobytes())
    for sweeps in (1, 2, 500):
        invs = []
        for s in range(sweeps):
            src = "x0" if s == 0 else ("e1" if s % 2 == 1 else "e2")
            dst = "x" if s == sweeps - 1 else ("e1" if s % 2 == 0 else "e2")
            invs.append(KernelInvocation("jacobi_sweep", grid(N), (i32(N),), ("A", "b", src, dst, "r")))
        req = KaasRequest(f"jac{sweeps}", buffers=(
            BufferArg("A", A.nbytes, "input", key="jA", is_const=True),
            BufferArg("b", 4 * N, "input", key="jb", is_const=True),
            BufferArg("x0", 4 * N, "input", key="jx0"),
            BufferArg("e1", 4 * N, "inout", is_ephemeral=True),
            BufferArg("e2", 4 * N, "inout", is_ephemeral=True),
            BufferArg("x", 4 * N, "output", key="jx"),
            BufferArg("r", 4, "output", key="jr")), invocations=tuple(invs))
        run(ex, store, req)
        _, dt = run(ex, store, req)
        xk = np.zeros(N)
        A64 = A.astype(np.float64)
        d = np.diag(A64).copy()
        b64 = bvec.astype(np.float64)
        for _ in range(sweeps):
            xn = ((b64 - (A64 @ xk - d * xk)) / d).astype(F32).astype(np.float64)
            res = np.abs(xn - xk).sum()
            xk = xn
        got = np.frombuffer(bytes(store.get("jx")), F32)
        r = np.frombuffer(bytes(store.get("jr")), F32)[0]
        print(f"jacobi sweeps={sweeps}: max|dx|={np.abs(got - xk).max():.3e} resid={r:.4e} vs {res:.4e}"
              f"  warm request {dt*1e3:.2f} ms device {ex.dev_stats.last_device_ms:.2f} ms", flush=True)

    # cgemm
    for (cn, cm, ck) in [(128, 128, 64), (256, 192, 80), (200, 100, 17), (1024, 1024, 1024), (8192, 8192, 8192)]:
        Ac = (rng.standard_normal((cn, ck)) + 1j * rng.standard_normal((cn, ck))).astype(np.complex64)
        Bc = (rng.standard_normal((ck, cm)) + 1j * rng.standard_normal((ck, cm))).astype(np.complex64)
        ka, kb = f"cA{cn}_{ck}", f"cB{ck}_{cm}"
        store.put(ka, Ac.tobytes())
        store.put(kb, Bc.tobytes())
        req = KaasRequest("cg", buffers=(
            BufferArg("A", Ac.nbytes, "input", key=ka, is_const=True),
            BufferArg("B", Bc.nbytes, "input", key=kb, is_const=True),
            BufferArg("C", 8 * cn * cm, "output", key="cC")),
            invocations=(KernelInvocation("cgemm", grid(cn * cm), (i32(cn), i32(cm), i32(ck)), ("A", "B", "C")),))
        run(ex, store, req)
        for _ in range(2):
            _, dt = run(ex, store, req)
        got = np.frombuffer(store.get("cC"), np.complex64).reshape(cn, cm)
        if cn <= 1024:
            ref = Ac.astype(np.complex128) @ Bc.astype(np.complex128)
            err = np.linalg.norm(got - ref) / np.linalg.norm(ref)
        else:  # spot-check 64 rows
            rows = rng.choice(cn, 64, replace=False)
            ref = Ac[rows].astype(np.complex128) @ Bc.astype(np.complex128)
            err = np.linalg.norm(got[rows] - ref) / np.linalg.norm(ref)
        print(f"cgemm {cn}x{cm}x{ck}: rel.fro={err:.3e}  warm request {dt*1e3:.2f} ms device {ex.dev_stats.last_device_ms:.3f} ms", flush=True)

    print("launches", native.launch_counter())


if __name__ == "__main__":
    main()
