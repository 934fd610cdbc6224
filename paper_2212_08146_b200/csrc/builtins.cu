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
// (backend.py:174-189, oracle pkg/tests/oracles.py:25-33).  Bit-exactness
// forbids split-K, so all parallelism comes from output cells: 256 threads
// (16 x 16) each own TM x TN cells of a (16*TM) x (16*TN) tile, k staged
// through smem BK at a time.  The tile shape is picked per launch so small-M
// / long-K layers (ResNet stage 4: M = 49, K = 4608) still fill the SMs,
// while big layers get 4x4 register blocking (0.5 smem loads per MAC).
// Padding products are never added (0*Inf would be NaN and +0 would flip
// the sign of a -0.0 accumulator), so the k loop uses the true extent.
constexpr int MM_BK = 16;

template <int TM, int TN>
__global__ void __launch_bounds__(256)
k_matmul(int n, int m, int k, uint64_t cov, const float *__restrict__ a,
         const float *__restrict__ b, float *__restrict__ out) {
  constexpr int BM = 16 * TM, BN = 16 * TN;
  constexpr int LA = BM * MM_BK / 256, LB = MM_BK * BN / 256;  // elements per thread
  __shared__ float As[2][MM_BK][BM];
  __shared__ float Bs[2][MM_BK][BN];
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  const int bm = blockIdx.y * BM, bn = blockIdx.x * BN;
  float acc[TM][TN];
#pragma unroll
  for (int i = 0; i < TM; ++i)
#pragma unroll
    for (int j = 0; j < TN; ++j) acc[i][j] = 0.0f;

  // register staging: the next k-chunk's global loads are in flight while
  // the current chunk computes out of the other smem buffer
  float ra[LA], rb[LB];
  auto load = [&](int k0) {
    const int kc = min(MM_BK, k - k0);
#pragma unroll
    for (int u = 0; u < LA; ++u) {
      const int e = threadIdx.x + 256 * u;
      const int r = e / MM_BK, kk = e % MM_BK;
      ra[u] = (bm + r < n && kk < kc) ? __ldg(a + (size_t)(bm + r) * k + k0 + kk) : 0.0f;
    }
#pragma unroll
    for (int u = 0; u < LB; ++u) {
      const int e = threadIdx.x + 256 * u;
      const int kk = e / BN, c = e % BN;
      rb[u] = (bn + c < m && kk < kc) ? __ldg(b + (size_t)(k0 + kk) * m + bn + c) : 0.0f;
    }
  };
  auto stash = [&](int buf) {
#pragma unroll
    for (int u = 0; u < LA; ++u) {
      const int e = threadIdx.x + 256 * u;
      As[buf][e % MM_BK][e / MM_BK] = ra[u];
    }
#pragma unroll
    for (int u = 0; u < LB; ++u) {
      const int e = threadIdx.x + 256 * u;
      Bs[buf][e / BN][e % BN] = rb[u];
    }
  };
  if (k > 0) load(0);
  int buf = 0;
  for (int k0 = 0; k0 < k; k0 += MM_BK, buf ^= 1) {
    const int kc = min(MM_BK, k - k0);
    stash(buf);
    __syncthreads();
    if (k0 + MM_BK < k) load(k0 + MM_BK);
    auto step = [&](int kk) {
      float av[TM], bv[TN];
#pragma unroll
      for (int i = 0; i < TM; ++i) av[i] = As[buf][kk][ty + 16 * i];
#pragma unroll
      for (int j = 0; j < TN; ++j) bv[j] = Bs[buf][kk][tx + 16 * j];
#pragma unroll
      for (int i = 0; i < TM; ++i)
#pragma unroll
        for (int j = 0; j < TN; ++j) acc[i][j] = __fadd_rn(acc[i][j], __fmul_rn(av[i], bv[j]));
    };
    if (kc == MM_BK) {
#pragma unroll
      for (int kk = 0; kk < MM_BK; ++kk) step(kk);
    } else {
      for (int kk = 0; kk < kc; ++kk) step(kk);
    }
  }
#pragma unroll
  for (int i = 0; i < TM; ++i) {
    const int r = bm + ty + 16 * i;
    if (r >= n) continue;
#pragma unroll
    for (int j = 0; j < TN; ++j) {
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
  if (n == 0 || m == 0 || cov == 0) return 0;
  if (n > 0x7fffffffu || m > 0x7fffffffu || k > 0x7fffffffu)
    return fail(KAAS_E_INVALID, "matmul extent exceeds i32");
  // largest register tile that still gives >= 2 CTAs per SM
  const uint64_t want = 2ull * device_props(dev).sm_count;
  auto ctas = [&](int tm, int tn) {
    return ((n + 16 * tm - 1) / (16 * tm)) * ((m + 16 * tn - 1) / (16 * tn));
  };
  int tm = 1, tn = 1;
  const int cand[][2] = {{4, 4}, {2, 4}, {4, 2}, {2, 2}, {1, 2}, {2, 1}};
  for (auto &c : cand) {
    if (ctas(c[0], c[1]) >= want) {
      tm = c[0];
      tn = c[1];
      break;
    }
  }
  const uint64_t gy = (n + 16 * tm - 1) / (16 * tm), gx = (m + 16 * tn - 1) / (16 * tn);
  if (gy > 65535) return fail(KAAS_E_INVALID, "matmul: n too large for grid.y");
  dim3 grid((unsigned)gx, (unsigned)gy);
#define MM_LAUNCH(TM, TN) \
  k_matmul<TM, TN><<<grid, 256, 0, s>>>((int)n, (int)m, (int)k, cov, a, b, out)
  if (tm == 4 && tn == 4) MM_LAUNCH(4, 4);
  else if (tm == 2 && tn == 4) MM_LAUNCH(2, 4);
  else if (tm == 4 && tn == 2) MM_LAUNCH(4, 2);
  else if (tm == 2 && tn == 2) MM_LAUNCH(2, 2);
  else if (tm == 1 && tn == 2) MM_LAUNCH(1, 2);
  else if (tm == 2 && tn == 1) MM_LAUNCH(2, 1);
  else MM_LAUNCH(1, 1);
#undef MM_LAUNCH
  count_launch();
  KAAS_CUDA(cudaGetLastError());
  return 0;
}

}  // namespace kaas
