"""Kernel-only microbenchmarks through the C ABI (dev tool; also used by ncu runs).

    python tools/kbench.py jacobi [n] [sweeps] [reps]
    python tools/kbench.py cgemm [n] [reps]
    python tools/kbench.py matmul M N K [reps]
    python tools/kbench.py resnet [reps]      per-layer bit-exact matmul vs. its floor
"""

import sys

import numpy as np

sys.path.insert(0, ".")
from paper_2212_08146_b200 import native  # noqa: E402
from paper_2212_08146_b200.api import LaunchDims, i32  # noqa: E402
from paper_2212_08146_b200.kernels import default_registry, fill_desc  # noqa: E402
from paper_2212_08146_b200.hoststore import PinnedBlob  # noqa: E402


def dev_buf(stream, data: bytes):
    p = native.malloc_async(stream, len(data))
    blob = PinnedBlob.from_bytes(data)
    native.h2d_async(p, blob.addr, len(data), stream)
    stream.sync()
    return p


def timed(stream, fn, reps):
    e0, e1 = native.Event(0, True), native.Event(0, True)
    fn()
    stream.sync()
    e0.record(stream)
    for _ in range(reps):
        fn()
    e1.record(stream)
    e1.sync()
    return e0.elapsed_ms(e1) / reps


def jacobi(n=4096, sweeps=500, reps=3):
    reg = default_registry()
    k = reg.get("jacobi_sweep")
    s = native.Stream(0)
    rng = np.random.default_rng(0)
    A = rng.random((n, n), dtype=np.float32)
    A[np.arange(n), np.arange(n)] = A.sum(1) + 1
    b = A.astype(np.float64) @ np.ones(n)
    pA = dev_buf(s, A.tobytes())
    pb = dev_buf(s, b.astype(np.float32).tobytes())
    px = [dev_buf(s, bytes(4 * n)) for _ in range(3)]
    pr = dev_buf(s, bytes(4))
    dims = LaunchDims(grid_x=n)
    descs = (native.LaunchDesc * sweeps)()
    for t in range(sweeps):
        src = px[0] if t == 0 else px[1 + (t - 1) % 2]
        dst = px[1 + t % 2]
        fill_desc(descs[t], k, dims, (i32(n),), [pA, pb, src, dst, pr],
                  [4 * n * n, 4 * n, 4 * n, 4 * n, 4])
    ms = timed(s, lambda: native.launch_batch(0, s, descs), reps)
    one = (native.LaunchDesc * 1)()
    fill_desc(one[0], k, dims, (i32(n),), [pA, pb, px[0], px[1], pr], [4 * n * n, 4 * n, 4 * n, 4 * n, 4])
    ms1 = timed(s, lambda: native.launch_batch(0, s, one), 20)
    per = ms / sweeps
    bytes_sweep = 4 * n * n + 12 * n
    print(f"jacobi n={n} sweeps={sweeps}: chain {ms:.3f} ms = {per*1e3:.2f} us/sweep "
          f"({bytes_sweep / per / 1e6:.0f} GB/s); single-sweep launch {ms1*1e3:.2f} us "
          f"({bytes_sweep / ms1 / 1e6:.0f} GB/s)")


def cgemm(n=8192, reps=3):
    reg = default_registry()
    k = reg.get("cgemm")
    s = native.Stream(0)
    rng = np.random.default_rng(0)
    A = rng.standard_normal(2 * n * n, dtype=np.float32)
    B = rng.standard_normal(2 * n * n, dtype=np.float32)
    pA, pB = dev_buf(s, A.tobytes()), dev_buf(s, B.tobytes())
    pC = native.malloc_async(s, 8 * n * n)
    d = (native.LaunchDesc * 1)()
    fill_desc(d[0], k, LaunchDims(grid_x=n * n), (i32(n), i32(n), i32(n)), [pA, pB, pC],
              [8 * n * n] * 3)
    ms = timed(s, lambda: native.launch_batch(0, s, d), reps)
    useful = 8.0 * n ** 3
    print(f"cgemm n={n}: {ms:.3f} ms/launch  useful {useful / ms / 1e9:.1f} TFLOP/s  "
          f"f16-issued (3 products) {3 * useful / ms / 1e9:.1f} TFLOP/s")


def matmul(M, N, K, reps=5):
    reg = default_registry()
    k = reg.get("matmul")
    s = native.Stream(0)
    rng = np.random.default_rng(0)
    pa = dev_buf(s, rng.standard_normal(M * K, dtype=np.float32).tobytes())
    pb = dev_buf(s, rng.standard_normal(K * N, dtype=np.float32).tobytes())
    pc = native.malloc_async(s, 4 * M * N)
    d = (native.LaunchDesc * 1)()
    fill_desc(d[0], k, LaunchDims(grid_x=M * N), (i32(M), i32(N), i32(K)), [pa, pb, pc],
              [4 * M * K, 4 * K * N, 4 * M * N])
    ms = timed(s, lambda: native.launch_batch(0, s, d), reps)
    print(f"matmul {M}x{N}x{K}: {ms*1e3:.1f} us  {M*N*K/ms/1e9:.2f} TMAC/s")
    for p in (pa, pb, pc):
        native.free_async(s, p)
    s.sync()
    return ms


def resnet(reps=20):
    """Each ResNet-50 conv-as-GEMM layer alone, against its floor: issue
    (FMUL+FADD per MAC over 148x128 lanes) or the serial FADD chain (4
    cycles per k), at 1.9 GHz; then the whole chain as one batch."""
    from paper_2212_08146_b200.workloads import resnet50_gemms
    layers = resnet50_gemms()
    seen, tot, floor_tot = {}, 0.0, 0.0
    for name, m, n, k in layers:
        key = (m, n, k)
        if key not in seen:
            seen[key] = matmul(m, n, k, reps)
        ms = seen[key]
        fl = max(m * n * k * 2 / (148 * 128), 4 * k) / 1.9e6
        tot += ms
        floor_tot += fl
        print(f"  {name:12s} {ms*1e3:8.1f} us  floor {fl*1e3:6.1f} us  x{ms/fl:5.1f}")
    print(f"sum of layers {tot*1e3:.1f} us, floor {floor_tot*1e3:.1f} us, "
          f"{sum(m*n*k for _, m, n, k in layers)/tot/1e9:.2f} TMAC/s")


if __name__ == "__main__":
    what = sys.argv[1]
    args = [int(a) for a in sys.argv[2:]]
    {"jacobi": jacobi, "cgemm": cgemm, "matmul": matmul, "resnet": resnet}[what](*args)
