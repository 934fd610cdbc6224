// Bit-exact sm_100a versions of the reference builtin kernels
// (pkg/src/kaas/backend.py:153-211).
//
// Semantics follow the reference's sequential model (backend.py:3-11): thread
// g in [0, total_threads) covers logical element g; elements past
// min(total_threads, n) are untouched; every multiply and add is a separately
// rounded IEEE binary32 operation (no FMA contraction: __fmul_rn/__fadd_rn),
// matmul/reduce accumulate in one f32 accumulator in ascending index order.
// The CUDA grid is our own choice (sized to the SM count); the request's
// LaunchDims only decide coverage, as in the reference.
//
// NaN payloads are the one thing IEEE 754 leaves open: numpy's x86 loops pick
// a payload by operand position and even by SIMD-vs-tail element position,
// so parity is defined bit-exact on every non-NaN word and NaN-for-NaN
// elsewhere ("bit-exact").
#include "kaas_internal.cuh"

namespace kaas {
namespace {

constexpr int kEltThreads = 256;

inline int elt_blocks(int dev, uint64_t work) {
  uint64_t want = (work + kEltThreads - 1) / kEltThreads;
  uint64_t cap = (uint64_t)device_props(dev).sm_count * 8;
  if (want < 1) want = 1;
  return (int)(want < cap ? want : cap);
}

inline bool aligned16(const void *p) { return ((uintptr_t)p & 15u) == 0; }

// Exact aliasing (out == x or out == y) is safe: each element is read and
// then written by the same thread, so no __restrict__ on these pointers.
template <int kOp>  // 0 = add, 1 = saxpy, 2 = fill
__global__ void __launch_bounds__(kEltThreads)
k_elementwise_v4(uint64_t n4, float a, const float4 *x, const float4 *y, float4 *out) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += stride) {
    float4 r;
    if (kOp == 2) {
      r = make_float4(a, a, a, a);
    } else {
      const float4 xv = x[i];
      const float4 yv = y[i];
      if (kOp == 0) {
        r.x = __fadd_rn(xv.x, yv.x); r.y = __fadd_rn(xv.y, yv.y);
        r.z = __fadd_rn(xv.z, yv.z); r.w = __fadd_rn(xv.w, yv.w);
      } else {
        r.x = __fadd_rn(__fmul_rn(a, xv.x), yv.x); r.y = __fadd_rn(__fmul_rn(a, xv.y), yv.y);
        r.z = __fadd_rn(__fmul_rn(a, xv.z), yv.z); r.w = __fadd_rn(__fmul_rn(a, xv.w), yv.w);
      }
    }
    out[i] = r;
  }
}

template <int kOp>
__global__ void __launch_bounds__(kEltThreads)
k_elementwise_scalar(uint64_t begin, uint64_t end, float a, const float *x, const float *y,
                     float *out) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = begin + (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < end; i += stride) {
    float r;
    if (kOp == 0) r = __fadd_rn(x[i], y[i]);
    else if (kOp == 1) r = __fadd_rn(__fmul_rn(a, x[i]), y[i]);
    else r = a;
    out[i] = r;
  }
}

template <int kOp>
int launch_elementwise(cudaStream_t s, int dev, uint64_t cov, float a, const float *x,
                       const float *y, float *out) {
  if (cov == 0) return 0;
  const bool vec = aligned16(out) && (kOp == 2 || (aligned16(x) && aligned16(y)));
  uint64_t done = 0;
  if (vec && cov >= 4) {
    const uint64_t n4 = cov / 4;
    k_elementwise_v4<kOp><<<elt_blocks(dev, n4), kEltThreads, 0, s>>>(
        n4, a, (const float4 *)x, (const float4 *)y, (float4 *)out);
    count_launch();
    done = n4 * 4;
  }
  if (done < cov) {
    k_elementwise_scalar<kOp><<<elt_blocks(dev, cov - done), kEltThreads, 0, s>>>(
        done, cov, a, x, y, out);
    count_launch();
  }
  KAAS_CUDA(cudaGetLastError());
  return 0;
}

// ---- reduce_sum: np.add.accumulate(x)[-1] (backend.py:192-202) ------------
// Inherently sequential: the result depends on every intermediate rounding.
// One thread walks the vector; loads are issued 16 at a time ahead of the
// dependent adds.  accumulate() seeds with x[0] itself (not 0 + x[0]), which
// matters for x[0] == -0.0.
__global__ void k_reduce_sum(uint64_t n, const float *x, float *out) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  if (n == 0) { *out = 0.0f; return; }
  float acc = x[0];
  uint64_t i = 1;
  for (; i + 16 <= n; i += 16) {
    float v[16];
#pragma unroll
    for (int u = 0; u < 16; ++u) v[u] = __ldg(x + i + u);
#pragma unroll
    for (int u = 0; u < 16; ++u) acc = __fadd_rn(acc, v[u]);
  }
  for (; i < n; ++i) acc = __fadd_rn(acc, __ldg(x + i));
  *out = acc;  // written after every read: safe if out aliases x
}

// ---- matmul: per cell acc = 0; acc = fl(acc + fl(a*b)), k ascending --------
// (backend.py:174-189, oracle pkg/tests/oracles.py:25-33).  SIMT tiles of
// 64x64 cells, 256 threads x (4x4) cells, k staged through smem 16 at a time.
// Padding products are never added (0*Inf would be NaN and +0 would flip
// the sign of a -0.0 accumulator), so the k loop uses the true extent.
constexpr int MM_BM = 64, MM_BN = 64, MM_BK = 16;

__global__ void __launch_bounds__(256)
k_matmul(int n, int m, int k, uint64_t cov, const float *__restrict__ a,
         const float *__restrict__ b, float *__restrict__ out) {
  __shared__ float As[MM_BK][MM_BM];
  __shared__ float Bs[MM_BK][MM_BN];
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  const int bm = blockIdx.y * MM_BM, bn = blockIdx.x * MM_BN;
  float acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = 0.0f;

  for (int k0 = 0; k0 < k; k0 += MM_BK) {
    const int kc = min(MM_BK, k - k0);
    // A tile: 64 rows x 16 k; thread t loads (row = t/4 + 64*0.., kk = t%4*4..)
    for (int e = threadIdx.x; e < MM_BM * MM_BK; e += 256) {
      const int r = e / MM_BK, kk = e % MM_BK;
      const int gr = bm + r, gk = k0 + kk;
      As[kk][r] = (gr < n && kk < kc) ? a[(size_t)gr * k + gk] : 0.0f;
    }
    for (int e = threadIdx.x; e < MM_BK * MM_BN; e += 256) {
      const int kk = e / MM_BN, c = e % MM_BN;
      const int gc = bn + c, gk = k0 + kk;
      Bs[kk][c] = (gc < m && kk < kc) ? b[(size_t)gk * m + gc] : 0.0f;
    }
    __syncthreads();
    if (kc == MM_BK) {
#pragma unroll
      for (int kk = 0; kk < MM_BK; ++kk) {
        float av[4], bv[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) av[i] = As[kk][ty + 16 * i];
#pragma unroll
        for (int j = 0; j < 4; ++j) bv[j] = Bs[kk][tx + 16 * j];
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) acc[i][j] = __fadd_rn(acc[i][j], __fmul_rn(av[i], bv[j]));
      }
    } else {
      for (int kk = 0; kk < kc; ++kk) {
        float av[4], bv[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) av[i] = As[kk][ty + 16 * i];
#pragma unroll
        for (int j = 0; j < 4; ++j) bv[j] = Bs[kk][tx + 16 * j];
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) acc[i][j] = __fadd_rn(acc[i][j], __fmul_rn(av[i], bv[j]));
      }
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int r = bm + ty + 16 * i;
    if (r >= n) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int c = bn + tx + 16 * j;
      if (c >= m) continue;
      const uint64_t g = (uint64_t)r * m + c;
      if (g < cov) out[g] = acc[i][j];
    }
  }
}

}  // namespace

int launch_vector_add(cudaStream_t s, int dev, uint64_t cov, const float *x, const float *y,
                      float *out) {
  return launch_elementwise<0>(s, dev, cov, 0.0f, x, y, out);
}

int launch_saxpy(cudaStream_t s, int dev, uint64_t cov, float a, const float *x, const float *y,
                 float *out) {
  return launch_elementwise<1>(s, dev, cov, a, x, y, out);
}

int launch_fill(cudaStream_t s, int dev, uint64_t cov, float v, float *out) {
  return launch_elementwise<2>(s, dev, cov, v, nullptr, nullptr, out);
}

int launch_reduce_sum(cudaStream_t s, int dev, uint64_t n, const float *x, float *out) {
  (void)dev;
  k_reduce_sum<<<1, 32, 0, s>>>(n, x, out);
  count_launch();
  KAAS_CUDA(cudaGetLastError());
  return 0;
}

int launch_matmul(cudaStream_t s, int dev, uint64_t n, uint64_t m, uint64_t k, uint64_t cov,
                  const float *a, const float *b, float *out) {
  (void)dev;
  if (n == 0 || m == 0 || cov == 0) return 0;
  if (n > 0x7fffffffu || m > 0x7fffffffu || k > 0x7fffffffu)
    return fail(KAAS_E_INVALID, "matmul extent exceeds i32");
  const uint64_t gy = (n + MM_BM - 1) / MM_BM, gx = (m + MM_BN - 1) / MM_BN;
  if (gy > 65535) return fail(KAAS_E_INVALID, "matmul: n too large for grid.y");
  dim3 grid((unsigned)gx, (unsigned)gy);
  k_matmul<<<grid, 256, 0, s>>>((int)n, (int)m, (int)k, cov, a, b, out);
  count_launch();
  KAAS_CUDA(cudaGetLastError());
  return 0;
}

}  // namespace kaas
