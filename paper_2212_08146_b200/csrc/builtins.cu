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

#include <atomic>

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
// (16 x 16) each own TM x TN cells of a (16*TM) x (16*TN) tile.  The tile
// shape is picked per launch so small-M / long-K layers (ResNet stage 4:
// M = 49, K = 4608) still fill the SMs, while big layers get 4x4 blocking.
//
// Operands stream through an S-deep ring of BK = 32 k-chunks filled by
// cp.async (4-byte copies, zero-filled out of bounds, so any shape and
// alignment works): S-1 chunks of loads are in flight behind the chunk being
// computed, which is what long-K layers need -- a 2-deep ring pays the full
// L2/HBM latency once per chunk.  A tiles are row-major in smem (k
// contiguous, rows padded to 36 floats) so a thread reads 4 k of a row with
// one LDS.128; a thread owns TN contiguous columns of B, read as one vector.
// Padding products are never added (0*Inf would be NaN and +0 would flip
// the sign of a -0.0 accumulator), so the tail chunk uses the true extent.
constexpr int MM_BK = 32, MM_LDA = MM_BK + 4;

__device__ __forceinline__ void cp_async4(float *dst, const float *src, bool ok) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;\n" ::"r"(d), "l"(src),
               "r"(ok ? 4 : 0)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}

template <int TN>
__device__ __forceinline__ void lds_vec(const float *p, float (&v)[TN]) {
  if constexpr (TN == 4) {
    const float4 t = *reinterpret_cast<const float4 *>(p);
    v[0] = t.x; v[1] = t.y; v[2] = t.z; v[3] = t.w;
  } else if constexpr (TN == 2) {
    const float2 t = *reinterpret_cast<const float2 *>(p);
    v[0] = t.x; v[1] = t.y;
  } else {
#pragma unroll
    for (int j = 0; j < TN; ++j) v[j] = p[j];
  }
}

template <int TM, int TN, int S>
constexpr int mm_smem_bytes() {
  return S * (16 * TM * MM_LDA + MM_BK * 16 * TN) * 4;
}

template <int TM, int TN, int S>
__global__ void __launch_bounds__(256)
k_matmul(int n, int m, int k, uint64_t cov, const float *__restrict__ a,
         const float *__restrict__ b, float *__restrict__ out) {
  constexpr int BM = 16 * TM, BN = 16 * TN;
  constexpr int A_ST = BM * MM_LDA, B_ST = MM_BK * BN;
  extern __shared__ __align__(16) float mm_smem[];
  float *As = mm_smem, *Bs = mm_smem + S * A_ST;
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  const int bm = blockIdx.y * BM, bn = blockIdx.x * BN;
  const int nk = (k + MM_BK - 1) / MM_BK;

  auto issue = [&](int t) {
    const int k0 = t * MM_BK;
    float *as = As + (t % S) * A_ST, *bs = Bs + (t % S) * B_ST;
#pragma unroll
    for (int u = 0; u < BM * MM_BK / 256; ++u) {
      const int e = threadIdx.x + 256 * u;
      const int r = e / MM_BK, kk = e % MM_BK;
      const bool ok = bm + r < n && k0 + kk < k;
      cp_async4(as + r * MM_LDA + kk, ok ? a + (size_t)(bm + r) * k + k0 + kk : a, ok);
    }
#pragma unroll
    for (int u = 0; u < MM_BK * BN / 256; ++u) {
      const int e = threadIdx.x + 256 * u;
      const int kk = e / BN, c = e % BN;
      const bool ok = bn + c < m && k0 + kk < k;
      cp_async4(bs + kk * BN + c, ok ? b + (size_t)(k0 + kk) * m + bn + c : b, ok);
    }
  };

  float acc[TM][TN];
#pragma unroll
  for (int i = 0; i < TM; ++i)
#pragma unroll
    for (int j = 0; j < TN; ++j) acc[i][j] = 0.0f;

#pragma unroll
  for (int t = 0; t < S - 1; ++t) {
    if (t < nk) issue(t);
    cp_async_commit();
  }
  for (int t = 0; t < nk; ++t) {
    cp_async_wait<S - 2>();
    __syncthreads();  // chunk t landed; everyone is done with chunk t-1's stage
    if (t + S - 1 < nk) issue(t + S - 1);
    cp_async_commit();
    const float *as = As + (t % S) * A_ST + ty * TM * MM_LDA;
    const float *bs = Bs + (t % S) * B_ST + tx * TN;
    const int kc = min(MM_BK, k - t * MM_BK);
    if (kc == MM_BK) {
#pragma unroll
      for (int k4 = 0; k4 < MM_BK; k4 += 4) {
        float4 av[TM];
#pragma unroll
        for (int i = 0; i < TM; ++i) av[i] = *reinterpret_cast<const float4 *>(as + i * MM_LDA + k4);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          float bv[TN];
          lds_vec<TN>(bs + (k4 + q) * BN, bv);
#pragma unroll
          for (int i = 0; i < TM; ++i) {
            const float x = q == 0 ? av[i].x : q == 1 ? av[i].y : q == 2 ? av[i].z : av[i].w;
#pragma unroll
            for (int j = 0; j < TN; ++j) acc[i][j] = __fadd_rn(acc[i][j], __fmul_rn(x, bv[j]));
          }
        }
      }
    } else {
      for (int kk = 0; kk < kc; ++kk) {
        float bv[TN];
        lds_vec<TN>(bs + kk * BN, bv);
#pragma unroll
        for (int i = 0; i < TM; ++i) {
          const float x = as[i * MM_LDA + kk];
#pragma unroll
          for (int j = 0; j < TN; ++j) acc[i][j] = __fadd_rn(acc[i][j], __fmul_rn(x, bv[j]));
        }
      }
    }
  }
  cp_async_wait<0>();
#pragma unroll
  for (int i = 0; i < TM; ++i) {
    const int r = bm + ty * TM + i;
    if (r >= n) continue;
#pragma unroll
    for (int j = 0; j < TN; ++j) {
      const int c = bn + tx * TN + j;
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
#define MM_LAUNCH(TM, TN)                                                               \
  do {                                                                                  \
    constexpr int S_ = (TM) * (TN) >= 8 ? 4 : 8;                                        \
    constexpr int SM_ = mm_smem_bytes<TM, TN, S_>();                                    \
    static std::atomic<uint64_t> attr_done{0}; /* per device (dev < 64) */               \
    if (!(attr_done.load(std::memory_order_relaxed) >> (dev & 63) & 1)) {               \
      KAAS_CUDA(cudaFuncSetAttribute(k_matmul<TM, TN, S_>,                              \
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, SM_)); \
      attr_done.fetch_or(1ull << (dev & 63));                                           \
    }                                                                                   \
    k_matmul<TM, TN, S_><<<grid, 256, SM_, s>>>((int)n, (int)m, (int)k, cov, a, b, out); \
  } while (0)
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
