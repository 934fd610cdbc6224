// Jacobi sweep for dense systems (new kernel; no reference counterpart --
// semantics are the CPU restatement in oracle/kernels.py:jacobi_sweep).
//
//   x_out[i] = (b[i] - sum_{j != i} A[i,j] * x_in[j]) / A[i,i]   for i < cov
//   resid[0] = sum_{i < cov} |x_out[i] - x_in[i]|
//
// A sweep is a GEMV (4*n*n bytes of A, 2*n*n flops) with no reuse of A
// inside it -- but a request's sweeps all read the same A, so the kernels
// that run a request's sweeps keep A close to the SMs.  Kernel family:
//
//   k_jacobi_tmem   (default, 2048 <= n <= 4096, n % 4 == 0): each SM's band
//                   of A lives in TMEM + registers + smem for all sweeps; x
//                   moves between SMs as (value, tag) words, no grid barrier
//   k_jacobi_cols   same layout with an L2 tier instead of TMEM
//                   (KAAS_JACOBI_TMEM=0; the A/B reference)
//   k_jacobi_rows   n % 4 == 0 up to 40960: one warp per row, A re-read from
//                   L2 (evict_last), x staged in smem, grid barrier per sweep
//   k_jacobi_sweep / k_jacobi_chain   any n (scalar path when n % 4 != 0)
//
// One CTA per SM, each owning a contiguous band of ~n/148 rows; the diagonal
// is dropped in-register; per-row partials are reduced with warp shuffles and
// across warps in fixed order.  Residual partials are reduced
// deterministically (rows -> CTA -> grid, fixed order, grid level in double).
//
// A request's 500 sweeps are 500 invocations ping-ponging two ephemerals;
// kaas_launch_batch hands such runs to launch_jacobi_chain: one cooperative
// persistent launch per request instead of 500.
#include <cooperative_groups.h>

#include <atomic>
#include <cstdio>
#include <cstdlib>

#include "kaas_internal.cuh"

namespace kaas {
namespace {

constexpr int kJacThreads = 512;
constexpr int kJacWarps = kJacThreads / 32;
constexpr int kGroup = 8;        // rows per group
constexpr int kChunk = 128;      // columns per chunk (32 lanes x float4)

__device__ __forceinline__ float4 ld_a(const float *p, uint64_t policy) {
  float4 v;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.f32 {%0,%1,%2,%3}, [%4], %5;"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "l"(p), "l"(policy));
  return v;
}

__device__ __forceinline__ uint64_t l2_policy(bool keep) {
  uint64_t pol;
  if (keep)  // A is re-read every sweep: ask L2 to keep it
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  else
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}

// x loads: the non-coherent path only when x is read-only for the whole
// launch (single sweep); the chain kernel rewrites x between sweeps.
template <bool kNcX>
__device__ __forceinline__ float4 ld_x4(const float *p) {
  if (kNcX) return __ldg(reinterpret_cast<const float4 *>(p));
  return __ldcg(reinterpret_cast<const float4 *>(p));
}
template <bool kNcX>
__device__ __forceinline__ float ld_x(const float *p) {
  if (kNcX) return __ldg(p);
  return __ldcg(p);
}

__device__ __forceinline__ float dot_masked(float4 a, float4 x, int d) {
  // d = row - first column of this float4; the diagonal term is dropped
  float s = d == 0 ? 0.f : a.x * x.x;
  s = fmaf(a.y, d == 1 ? 0.f : x.y, s);
  s = fmaf(a.z, d == 2 ? 0.f : x.z, s);
  s = fmaf(a.w, d == 3 ? 0.f : x.w, s);
  return s;
}

struct SweepSmem {
  float red[kJacWarps][kGroup];
  float part[kJacWarps];
};

// One sweep over rows [r0, r1) of this CTA.  Vector path (n % 4 == 0):
// KC = chunks per warp held in registers (n <= KC * 16 * 128).  Returns the
// CTA's residual partial in thread 0.
template <int KC, bool kNcX>
__device__ __forceinline__ float sweep_band_vec(int n, int r0, int r1, const float *__restrict__ A,
                                                const float *__restrict__ b,
                                                const float *__restrict__ x_in,
                                                float *__restrict__ x_out, SweepSmem &sm,
                                                uint64_t pol) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nchunks = (n + kChunk - 1) / kChunk;
  float4 xr[KC];
  int col[KC];
#pragma unroll
  for (int k = 0; k < KC; ++k) {
    const int c = warp + k * kJacWarps;
    col[k] = c * kChunk + 4 * lane;
    xr[k] = (c < nchunks && col[k] < n) ? ld_x4<kNcX>(x_in + col[k]) : make_float4(0.f, 0.f, 0.f, 0.f);
  }
  float res = 0.f;
  for (int i0 = r0; i0 < r1; i0 += kGroup) {
    const int g_n = min(kGroup, r1 - i0);
    float acc[kGroup];
#pragma unroll
    for (int g = 0; g < kGroup; ++g) acc[g] = 0.f;
    float4 av[kGroup][KC];
#pragma unroll
    for (int g = 0; g < kGroup; ++g)
#pragma unroll
      for (int k = 0; k < KC; ++k) {
        const bool ok = g < g_n && col[k] < n;
        av[g][k] = ok ? ld_a(A + (size_t)(i0 + g) * n + col[k], pol) : make_float4(0.f, 0.f, 0.f, 0.f);
      }
#pragma unroll
    for (int g = 0; g < kGroup; ++g)
#pragma unroll
      for (int k = 0; k < KC; ++k) acc[g] += dot_masked(av[g][k], xr[k], i0 + g - col[k]);
#pragma unroll
    for (int g = 0; g < kGroup; ++g) {
      float v = acc[g];
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
      acc[g] = v;
    }
    if (lane == 0) {
#pragma unroll
      for (int g = 0; g < kGroup; ++g) sm.red[warp][g] = acc[g];
    }
    __syncthreads();
    if (threadIdx.x < g_n) {
      const int g = threadIdx.x, i = i0 + g;
      float s = 0.f;
#pragma unroll
      for (int w = 0; w < kJacWarps; ++w) s += sm.red[w][g];
      const float xi = ld_x<kNcX>(x_in + i);
      const float xn = (b[i] - s) / A[(size_t)i * n + i];  // IEEE div.rn
      x_out[i] = xn;
      res += fabsf(xn - xi);
    }
    __syncthreads();
  }
  // CTA partial: threads 0..kGroup-1 hold row-group residuals
  if (threadIdx.x < kGroup) sm.part[threadIdx.x] = res;
  __syncthreads();
  float part = 0.f;
  if (threadIdx.x == 0)
    for (int g = 0; g < kGroup; ++g) part += sm.part[g];
  __syncthreads();
  return part;
}

// Scalar path for n % 4 != 0: one warp per row.
template <bool kNcX>
__device__ __forceinline__ float sweep_band_scalar(int n, int r0, int r1, const float *__restrict__ A,
                                                   const float *__restrict__ b,
                                                   const float *__restrict__ x_in,
                                                   float *__restrict__ x_out, SweepSmem &sm) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  float res = 0.f;
  for (int i = r0 + warp; i < r1; i += kJacWarps) {
    const float *row = A + (size_t)i * n;
    float s = 0.f;
    for (int j = lane; j < n; j += 32) s = fmaf(__ldg(row + j), j == i ? 0.f : ld_x<kNcX>(x_in + j), s);
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
    if (lane == 0) {
      const float xn = (b[i] - s) / row[i];
      x_out[i] = xn;
      res += fabsf(xn - ld_x<kNcX>(x_in + i));
    }
  }
  if (lane == 0) sm.part[warp] = res;
  __syncthreads();
  float part = 0.f;
  if (threadIdx.x == 0)
    for (int w = 0; w < kJacWarps; ++w) part += sm.part[w];
  __syncthreads();
  return part;
}

template <int KC, bool kNcX>
__device__ __forceinline__ float sweep_band(int n, int r0, int r1, const float *A, const float *b,
                                            const float *x_in, float *x_out, SweepSmem &sm,
                                            uint64_t pol) {
  if (KC > 0)
    return sweep_band_vec<(KC > 0 ? KC : 1), kNcX>(n, r0, r1, A, b, x_in, x_out, sm, pol);
  return sweep_band_scalar<kNcX>(n, r0, r1, A, b, x_in, x_out, sm);
}

__device__ __forceinline__ void band(int cov, int &r0, int &r1) {
  r0 = (int)(((long long)blockIdx.x * cov) / gridDim.x);
  r1 = (int)(((long long)(blockIdx.x + 1) * cov) / gridDim.x);
}

// Final cross-CTA sum by one warp, fixed order -> deterministic.
__device__ __forceinline__ void finish_resid(const float *partials, int nparts, float *resid,
                                             float *resid2 = nullptr) {
  const int lane = threadIdx.x & 31;
  double acc = 0.0;
  for (int p = lane; p < nparts; p += 32) acc += (double)__ldcg(partials + p);
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
  if (lane == 0) {
    *resid = (float)acc;
    if (resid2 != nullptr) *resid2 = (float)acc;
  }
}

template <int KC>
__global__ void __launch_bounds__(kJacThreads, 1)
k_jacobi_sweep(int n, int cov, const float *__restrict__ A, const float *__restrict__ b,
               const float *__restrict__ x_in, float *__restrict__ x_out, float *resid,
               float *partials, unsigned *ticket) {
  __shared__ SweepSmem sm;
  __shared__ bool last;
  int r0, r1;
  band(cov, r0, r1);
  const float part = sweep_band<KC, true>(n, r0, r1, A, b, x_in, x_out, sm, l2_policy(false));
  if (threadIdx.x == 0) {
    partials[blockIdx.x] = part;
    __threadfence();
    last = atomicAdd(ticket, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (last && threadIdx.x < 32) {
    __threadfence();
    finish_resid(partials, gridDim.x, resid);
    if (threadIdx.x == 0) *ticket = 0u;  // re-arm for the next launch on this stream
  }
}

// ---- persistent multi-sweep kernel ----------------------------------------

constexpr int kChainMaxPtrs = 16;
constexpr int kTraceStamps = 5;  // dev trace: per sweep and CTA (tools/jtrace.py)
constexpr int kTracePro = 8;     // dev trace: per-CTA launch-phase stamps after the sweep stamps
constexpr int kTraceWarpOff = 32 * 148 * kTraceStamps + 148 * kTracePro;  // then [32][148][8] per-warp x arrival
constexpr int kChainMaxSweeps = 2048;

struct ChainParams {
  const float *A;
  const float *b;
  float *ptrs[kChainMaxPtrs];
  // per sweep: x_in, x_out, resid indices into ptrs
  unsigned char idx[kChainMaxSweeps][3];
  int n, cov, sweeps, keep_l2;
  // column kernel only: x of sweep s >= 1 published as (value, tag0 + s)
  // words in xt[s & 1] instead of behind a grid barrier (tagged != 0)
  unsigned long long *xt;
  unsigned tag0;
  int tagged;
  int poll_ns;  // back-off between unsuccessful polls
  unsigned zero;  // always 0: an opaque value ptxas cannot fold (k_jacobi_tmem)
  unsigned sync_base;  // the grid-barrier counter's value when this launch starts
  unsigned *trace;  // dev: [32 sweeps][148 CTAs][3] globaltimer_lo stamps, or nullptr
  // k_jacobi_tmem: the last sweep also writes x_out / resid here (pinned
  // host memory; the request's write-back without a copy), or nullptr
  float *wb_x, *wb_r;
};

__device__ __forceinline__ unsigned ld_acquire(const unsigned *p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// Monotonic grid barrier: the counter only ever grows (the host tracks its
// value across launches on the stream: no reset, no memset before a launch);
// barrier number e of a launch completes when it reaches base + (e+1) *
// gridDim.x (compared modulo 2^32).  One release-atomic per CTA,
// acquire-polling, no extra fences (release is cumulative over the CTA's
// writes ordered by bar.sync).
__device__ __forceinline__ void grid_sync_mono(unsigned *counter, unsigned epoch, unsigned base) {
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(counter) : "memory");
    const unsigned target = base + (epoch + 1) * gridDim.x;
    // ld.acquire.gpu lowers to LDG.STRONG.GPU + CCTL.IVALL: the SM's L1 is
    // invalidated, so later plain loads of x see the other CTAs' writes
    while ((int)(ld_acquire(counter) - target) < 0) {
    }
  }
  __syncthreads();
}

__device__ __forceinline__ void grid_barrier(unsigned *count, unsigned *gen) {
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned g = ld_acquire(gen);
    __threadfence();
    if (atomicAdd(count, 1u) == gridDim.x - 1) {
      *count = 0u;
      __threadfence();
      atomicAdd(gen, 1u);
    } else {
      while (ld_acquire(gen) == g) __nanosleep(20);
    }
    __threadfence();
  }
  __syncthreads();
}

template <int KC>
__global__ void __launch_bounds__(kJacThreads, 1)
k_jacobi_chain(const __grid_constant__ ChainParams p, float *partials, unsigned *sync) {
  __shared__ SweepSmem sm;
  int r0, r1;
  band(p.cov, r0, r1);
  const uint64_t pol = l2_policy(p.keep_l2 != 0);
  for (int s = 0; s < p.sweeps; ++s) {
    const float *x_in = p.ptrs[p.idx[s][0]];
    float *x_out = p.ptrs[p.idx[s][1]];
    const float part = sweep_band<KC, false>(p.n, r0, r1, p.A, p.b, x_in, x_out, sm, pol);
    float *slot = partials + (s & 1) * kMaxJacobiBlocks;
    if (threadIdx.x == 0) slot[blockIdx.x] = part;
    grid_barrier(sync + 1, sync + 2);
    if (blockIdx.x == 0 && threadIdx.x < 32) finish_resid(slot, gridDim.x, p.ptrs[p.idx[s][2] & 0x7f]);
  }
}


// ---- row-per-warp direct kernel ----------------------------------------------
//
// One warp per row, all of the CTA's band in flight at once (~28 warps for
// n = 4096), 8 x 128-bit loads of A per lane in flight, x staged once per
// sweep in smem (16 KiB) and read with conflict-free 128-bit LDS, four
// independent FMA chains, a 5-step shuffle reduce per row, no CTA barrier
// inside the sweep.
constexpr int kRowsMaxWarps = 28;  // 896 threads -> 72 registers per thread
constexpr int kRowsUnroll = 8;
constexpr int kRowsPre = 4;  // loads hoisted above the x staging

template <bool kChain, bool kPrefetch, bool kXDirect = false>
__global__ void __launch_bounds__(kRowsMaxWarps * 32, 1)
k_jacobi_rows(const __grid_constant__ ChainParams p, float *partials, unsigned *sync) {
  extern __shared__ __align__(16) float xs[];  // n floats
  __shared__ float wres[kRowsMaxWarps];
  __shared__ bool last;
  const int n = p.n, n4 = n >> 2;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nwarps = blockDim.x >> 5;
  int r0, r1;
  band(p.cov, r0, r1);
  const uint64_t pol = l2_policy(p.keep_l2 != 0);
  const float4 *x4 = reinterpret_cast<const float4 *>(xs);
  const int first = r0 + warp;                                  // this warp's first row
  const bool full_first = kPrefetch && n4 >= 32 * kRowsPre;  // hoistable first loads
  float4 pre[kPrefetch ? kRowsPre : 1];
  for (int s = 0; s < p.sweeps; ++s) {
    const float *x_in = p.ptrs[p.idx[s][0]];
    float *x_out = p.ptrs[p.idx[s][1]];
    const bool want_resid = !kChain || (p.idx[s][2] & 0x80) != 0;
    // A does not depend on x: the first loads of this warp's first row are
    // put in flight early -- for sweep 0 here, for later sweeps just before
    // the grid barrier of the previous one (A is the same every sweep)
    if (kPrefetch && s == 0 && first < r1 && full_first) {
#pragma unroll
      for (int u = 0; u < kRowsPre; ++u)
        pre[kPrefetch ? u : 0] = ld_a(p.A + (size_t)first * n + 4 * (lane + 32 * u), pol);
    }
    if (!kXDirect) {
      for (int e = threadIdx.x; e < n4; e += blockDim.x)
        reinterpret_cast<float4 *>(xs)[e] = kChain ? __ldcg(reinterpret_cast<const float4 *>(x_in) + e)
                                                   : __ldg(reinterpret_cast<const float4 *>(x_in) + e);
      __syncthreads();
    }
    // kXDirect: x is read through L1 inside the row loop (the grid barrier's
    // acquire invalidated L1, so the first warp per SM pulls each line from L2)
    const float4 *xg = reinterpret_cast<const float4 *>(x_in);
    float res = 0.f;
    for (int i = first; i < r1; i += nwarps) {
      const float *row = p.A + (size_t)i * n;
      const int it_d = (i >> 2) / 32;  // the (warp-uniform) iteration holding the diagonal
      float a0 = 0.f, a1 = 0.f, a2 = 0.f, a3 = 0.f;
      auto group = [&](const float4 *av, int cnt, int j4, int it) {
#pragma unroll
        for (int u = 0; u < cnt; ++u) {
          float4 xv = kXDirect ? xg[j4 + 32 * u] : x4[j4 + 32 * u];
          if (it + u == it_d) {
            const int d = i - 4 * (j4 + 32 * u);
            xv.x = d == 0 ? 0.f : xv.x;
            xv.y = d == 1 ? 0.f : xv.y;
            xv.z = d == 2 ? 0.f : xv.z;
            xv.w = d == 3 ? 0.f : xv.w;
          }
          a0 = fmaf(av[u].x, xv.x, a0);
          a1 = fmaf(av[u].y, xv.y, a1);
          a2 = fmaf(av[u].z, xv.z, a2);
          a3 = fmaf(av[u].w, xv.w, a3);
        }
      };
      int it = 0;
      int j4 = lane;
      if (kPrefetch && i == first && full_first) {  // first group: already in flight
        group(pre, kRowsPre, j4, it);
        j4 += 32 * kRowsPre;
        it += kRowsPre;
      }
      for (; j4 + 32 * (kRowsUnroll - 1) < n4; j4 += 32 * kRowsUnroll, it += kRowsUnroll) {
        float4 av[kRowsUnroll];
#pragma unroll
        for (int u = 0; u < kRowsUnroll; ++u) av[u] = ld_a(row + 4 * (j4 + 32 * u), pol);
        group(av, kRowsUnroll, j4, it);
      }
      for (; j4 < n4; j4 += 32, ++it) {
        const float4 a = ld_a(row + 4 * j4, pol);
        float4 xv = kXDirect ? xg[j4] : x4[j4];
        if (it == it_d) {
          const int d = i - 4 * j4;
          xv.x = d == 0 ? 0.f : xv.x;
          xv.y = d == 1 ? 0.f : xv.y;
          xv.z = d == 2 ? 0.f : xv.z;
          xv.w = d == 3 ? 0.f : xv.w;
        }
        a0 = fmaf(a.x, xv.x, a0);
        a1 = fmaf(a.y, xv.y, a1);
        a2 = fmaf(a.z, xv.z, a2);
        a3 = fmaf(a.w, xv.w, a3);
      }
      float v = (a0 + a1) + (a2 + a3);
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
      if (lane == 0) {
        const float xn = (p.b[i] - v) / __ldg(row + i);  // IEEE div.rn
        x_out[i] = xn;
        res += fabsf(xn - (kXDirect ? x_in[i] : xs[i]));
      }
    }
    if (kPrefetch && kChain && s + 1 < p.sweeps && first < r1 && full_first) {
#pragma unroll
      for (int u = 0; u < kRowsPre; ++u)
        pre[kPrefetch ? u : 0] = ld_a(p.A + (size_t)first * n + 4 * (lane + 32 * u), pol);
    }
    if (want_resid && lane == 0) wres[warp] = res;
    if (kChain) {
      float *slot = partials + (s & 1) * kMaxJacobiBlocks;
      if (want_resid) {
        __syncthreads();
        if (threadIdx.x == 0) {
          float cta = 0.f;
          for (int w = 0; w < nwarps; ++w) cta += wres[w];
          slot[blockIdx.x] = cta;
        }
      }
      grid_sync_mono(sync + 3, (unsigned)s, p.sync_base);  // also: xs reads done before the next stage-in
      if (want_resid && blockIdx.x == 0 && threadIdx.x < 32)
        finish_resid(slot, gridDim.x, p.ptrs[p.idx[s][2] & 0x7f]);
    } else {
      __syncthreads();
      if (threadIdx.x == 0) {
        float cta = 0.f;
        for (int w = 0; w < nwarps; ++w) cta += wres[w];
        partials[blockIdx.x] = cta;
        __threadfence();
        last = atomicAdd(sync, 1u) == gridDim.x - 1;
      }
      __syncthreads();
      if (last && threadIdx.x < 32) {
        __threadfence();
        finish_resid(partials, gridDim.x, p.ptrs[p.idx[s][2] & 0x7f]);
        if (threadIdx.x == 0) *sync = 0u;
      }
    }
  }
}

// ---- column-split kernel with A kept on chip (n <= 4096) ---------------------
//
// The row kernel is bound by the SM's load-return path, not by L2: every
// warp re-reads all of x through L1 for each of its rows, so per sweep an SM
// moves its 453 KB band of A plus 28 x 16 KB of x into registers (ncu:
// l1tex writeback 60% active over the whole chain).  Here the band is
// transposed onto the CTA instead: 8 warps split the columns (each lane owns
// 4 float4 columns and holds its x values in registers, so x crosses the
// load path once per CTA), and every thread keeps its slice of the band's
// rows in three tiers that persist across all sweeps of the launch:
//   rows 0..5    registers (96 KB per SM)
//   rows 6..19   thread-private shared memory (224 KB per SM, LDS.128,
//                conflict-free: [row][u][thread])
//   rows 20..27  re-read from L2 (evict_last) in two groups of 4; the first
//                group's loads are issued before the grid barrier
// Each lane accumulates one FMA chain per row over its 16 columns; the 28
// row partials are reduced across the warp with a 31-shuffle transpose
// reduction (lane l ends with row l) and across warps in fixed order, so the
// result is deterministic.  The diagonal is zeroed as A is loaded.
constexpr int kColW = 8;
constexpr int kColT = kColW * 32;
constexpr int kColC4 = 4;            // float4 columns per lane: n4 <= 8 * 32 * 4
constexpr int kColRows = 28;         // band rows per CTA
constexpr int kColRR = 6;            // register rows
constexpr int kColRS = 14;           // shared-memory rows
constexpr int kColG = 4;             // L2 rows per load group
static_assert(kColRR + kColRS + 2 * kColG == kColRows, "row tiers must cover the band");
constexpr size_t kColSmem = (size_t)kColRS * kColC4 * kColT * sizeof(float4);

__device__ __forceinline__ float4 zero4() { return make_float4(0.f, 0.f, 0.f, 0.f); }

// (value, tag) words: 8-byte aligned accesses are single-copy atomic, so a
// reader that sees the tag it waits for also sees that sweep's value
__device__ __forceinline__ ulonglong2 ld_relaxed_u64x2(const unsigned long long *p) {
  ulonglong2 v;
  asm volatile("ld.relaxed.gpu.global.v2.u64 {%0, %1}, [%2];" : "=l"(v.x), "=l"(v.y) : "l"(p) : "memory");
  return v;
}
// one lane's whole chunk (4 tagged words, 32 B) in one 256-bit load: a warp's
// poll is 1 KB contiguous, every sector fully used (two 128-bit loads would
// fetch each sector twice -- strong loads bypass L1)
struct TagWords4 {
  unsigned long long w[4];
};
__device__ __forceinline__ TagWords4 ld_relaxed_u64x4(const unsigned long long *p) {
  TagWords4 v;
  asm volatile("ld.relaxed.gpu.global.v4.u64 {%0, %1, %2, %3}, [%4];"
               : "=l"(v.w[0]), "=l"(v.w[1]), "=l"(v.w[2]), "=l"(v.w[3])
               : "l"(p)
               : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed_u64(unsigned long long *p, unsigned long long v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned gtimer_lo() {
  unsigned t;
  asm volatile("mov.u32 %0, %%globaltimer_lo;" : "=r"(t));
  return t;
}
__device__ __forceinline__ unsigned long long tagged_word(float v, unsigned tag) {
  return ((unsigned long long)tag << 32) | __float_as_uint(v);
}

// band row held by reduction slot l (see the two slot sets in k_jacobi_cols);
// 32 = empty slot
__device__ __forceinline__ int col_slot_row(int l) {
  constexpr int L2R0 = kColRR + kColRS, S0 = 16 - kColG - kColRR;
  if (l < kColG) return L2R0 + l;                       // L2 group 0
  if (l < kColG + kColRR) return l - kColG;             // register rows
  if (l < 16) return kColRR + (l - kColG - kColRR);     // smem rows 0..S0-1
  const int k = l - 16;
  if (k < kColRS - S0) return kColRR + S0 + k;          // smem rows S0..
  if (k < kColRS - S0 + kColG) return L2R0 + kColG + (k - (kColRS - S0));  // L2 group 1
  return 32;
}

__global__ void __launch_bounds__(kColT, 1)
k_jacobi_cols(const __grid_constant__ ChainParams p, float *partials, unsigned *sync) {
  extern __shared__ __align__(16) float4 acache[];  // [kColRS][kColC4][kColT]
  __shared__ float red[kColW][32];
  const int n = p.n, n4 = n >> 2;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  int r0, r1;
  band(p.cov, r0, r1);
  const int R = r1 - r0;
  const uint64_t pol = l2_policy(p.keep_l2 != 0);
  const int cbase = warp * 32 * kColC4 + lane;  // this lane's float4 columns: cbase + 32u

  // A[r0 + rl][cbase + 32u].  Rows past the band are clamped to a valid row
  // (their partials are discarded); columns past n read as 0, which only a
  // narrow system (n4 < 1024) needs, so the full-width case has no
  // predicates at all.  Nothing consumes a value at issue, so the L2 tier
  // really is in flight while other rows compute.  `z` is an opaque 0 from
  // the caller: it keeps the compiler from hoisting 8 row addresses out of
  // the sweep loop into registers (one IMAD.WIDE per row to recompute).
  const bool full = cbase + 32 * (kColC4 - 1) < n4;  // all of this lane's columns exist
  auto lda_raw = [&](int rl, int u, int z) -> float4 {
    const float4 *rp = reinterpret_cast<const float4 *>(p.A) +
                       (size_t)(r0 + min(rl, R - 1) + z) * n4 + cbase;
    if (full) return ld_a(reinterpret_cast<const float *>(rp + 32 * u), pol);
    float4 a = zero4();
    if (cbase + 32 * u < n4) a = ld_a(reinterpret_cast<const float *>(rp + 32 * u), pol);
    return a;
  };
  // the cached tiers hold A with the diagonal zeroed
  auto lda = [&](int rl, int u, int z) -> float4 {
    if (rl >= R) return zero4();
    float4 a = lda_raw(rl, u, z);
    const int c4 = cbase + 32 * u, i = r0 + rl;
    if (c4 == (i >> 2)) {
      const int d = i & 3;
      a.x = d == 0 ? 0.f : a.x;
      a.y = d == 1 ? 0.f : a.y;
      a.z = d == 2 ? 0.f : a.z;
      a.w = d == 3 ? 0.f : a.w;
    }
    return a;
  };
  auto opaque0 = [] {
    int z;
    asm volatile("mov.u32 %0, 0;" : "=r"(z));
    return z;
  };
  float4 areg[kColRR][kColC4];
#pragma unroll
  for (int r = 0; r < kColRR; ++r)
#pragma unroll
    for (int u = 0; u < kColC4; ++u) areg[r][u] = lda(r, u, 0);
#pragma unroll 1
  for (int r = 0; r < kColRS; ++r)
#pragma unroll
    for (int u = 0; u < kColC4; ++u) acache[(r * kColC4 + u) * kColT + tid] = lda(kColRR + r, u, 0);
  const int my_rl = col_slot_row(lane);  // warp 0, lane l finishes slot l's row
  float bi = 0.f, di = 1.f;
  if (warp == 0 && my_rl < R) {
    bi = __ldg(p.b + r0 + my_rl);
    di = __ldg(p.A + (size_t)(r0 + my_rl) * n + r0 + my_rl);
  }
  constexpr int L2R0 = kColRR + kColRS;
  float4 pf[kColG][kColC4];
  auto issue = [&](int g) {
    const int z = opaque0();
#pragma unroll
    for (int j = 0; j < kColG; ++j)
#pragma unroll
      for (int u = 0; u < kColC4; ++u) pf[j][u] = lda_raw(L2R0 + g * kColG + j, u, z);
  };
  // L2-tier rows whose diagonal lies in this lane's columns (bit = L2 row)
  unsigned dmask = 0;
#pragma unroll
  for (int j = 0; j < 2 * kColG; ++j) {
    const int off = ((r0 + L2R0 + j) >> 2) - cbase;
    if (L2R0 + j < R && off >= 0 && off % 32 == 0 && off / 32 < kColC4) dmask |= 1u << j;
  }
  issue(0);

  float xprev = 0.f;    // warp 0: this lane's row value from the previous sweep
  unsigned epoch = 0;   // grid barriers passed (monotonic counter target)
  for (int s = 0; s < p.sweeps; ++s) {
    const float *x_in = p.ptrs[p.idx[s][0]];
    float *x_out = p.ptrs[p.idx[s][1]];
    const bool want_resid = (p.idx[s][2] & 0x80) != 0;
    const bool from_tags = p.tagged && s > 0;
    float4 xr[kColC4];
    if (!from_tags) {
#pragma unroll
      for (int u = 0; u < kColC4; ++u)
        xr[u] = cbase + 32 * u < n4 ? __ldcg(reinterpret_cast<const float4 *>(x_in) + cbase + 32 * u)
                                    : zero4();
    } else {
      // wait for this lane's 16 x values of sweep s by polling their tags:
      // the producers' stores are the only synchronisation.  All chunks are
      // polled at once (4 producers per lane: one round trip, not four).
      const unsigned want = p.tag0 + (unsigned)s;
      const unsigned long long *src = p.xt + (size_t)(s & 1) * kJacTaggedMaxN;
      ulonglong2 q[kColC4][2];
      unsigned pending = 0;
#pragma unroll
      for (int u = 0; u < kColC4; ++u)
        if (cbase + 32 * u < n4) pending |= 1u << u;
      unsigned spins = 0;
      while (pending) {
        if (++spins > (1u << 22)) __trap();  // a lost producer: fail loudly, never hang
        if (spins > 1 && p.poll_ns) __nanosleep(p.poll_ns);
#pragma unroll
        for (int u = 0; u < kColC4; ++u) {
          if (pending & (1u << u)) {
            const int c4 = cbase + 32 * u;
            q[u][0] = ld_relaxed_u64x2(src + 4 * c4);
            q[u][1] = ld_relaxed_u64x2(src + 4 * c4 + 2);
          }
        }
#pragma unroll
        for (int u = 0; u < kColC4; ++u) {
          if ((pending & (1u << u)) && (unsigned)(q[u][0].x >> 32) == want &&
              (unsigned)(q[u][0].y >> 32) == want && (unsigned)(q[u][1].x >> 32) == want &&
              (unsigned)(q[u][1].y >> 32) == want)
            pending &= ~(1u << u);
        }
      }
#pragma unroll
      for (int u = 0; u < kColC4; ++u)
        xr[u] = cbase + 32 * u < n4
                    ? make_float4(__uint_as_float((unsigned)q[u][0].x), __uint_as_float((unsigned)q[u][0].y),
                                  __uint_as_float((unsigned)q[u][1].x), __uint_as_float((unsigned)q[u][1].y))
                    : zero4();
    }
    const bool tr = p.trace != nullptr && s >= 100 && s < 132 && threadIdx.x == 0;
    unsigned *trp = tr ? p.trace + ((s - 100) * 148 + (blockIdx.x < 148 ? blockIdx.x : 147)) * kTraceStamps : nullptr;
    if (tr) trp[1] = gtimer_lo();  // warp 0's x has arrived
    auto dot = [&](const float4 (&a)[kColC4]) {
      float acc = 0.f;
#pragma unroll
      for (int u = 0; u < kColC4; ++u) {
        acc = fmaf(a[u].x, xr[u].x, acc);
        acc = fmaf(a[u].y, xr[u].y, acc);
        acc = fmaf(a[u].z, xr[u].z, acc);
        acc = fmaf(a[u].w, xr[u].w, acc);
      }
      return acc;
    };
    // Rows are reduced in two sets of 16 slots so only 16 partials are live:
    // set 0 = L2 group 0, register rows, smem rows 0..5; set 1 = smem rows
    // 6..13, L2 group 1, 4 empty slots (slot -> row: col_slot_row()).
    // Reduction of one set: after the h-step (h = 8..1), v[k] (k < h) holds
    // a lane-pair sum of slot k + (lane's bits below 16); a final xor-16 add
    // completes it, and lane l ends with slot l & 15.
    // L2-tier group g: the diagonal is excluded at consumption; only the few
    // lanes that own one of the group's diagonals take the branch
    auto mask_group = [&](int g) {
      if ((dmask >> (g * kColG)) & ((1u << kColG) - 1u)) {
#pragma unroll
        for (int j = 0; j < kColG; ++j) {
          if ((dmask >> (g * kColG + j)) & 1u) {
            const int i = r0 + L2R0 + g * kColG + j, u = ((i >> 2) - cbase) / 32, d = i & 3;
#pragma unroll
            for (int q = 0; q < kColC4; ++q) {
              if (q == u) {
                pf[j][q].x = d == 0 ? 0.f : pf[j][q].x;
                pf[j][q].y = d == 1 ? 0.f : pf[j][q].y;
                pf[j][q].z = d == 2 ? 0.f : pf[j][q].z;
                pf[j][q].w = d == 3 ? 0.f : pf[j][q].w;
              }
            }
          }
        }
      }
    };
    auto reduce16 = [&](float (&v)[16]) {
#pragma unroll
      for (int h = 8; h >= 1; h >>= 1) {
        const bool up = (lane & h) != 0;
#pragma unroll
        for (int k = 0; k < h; ++k) {
          const float send = up ? v[k] : v[k + h];
          const float keep = up ? v[k + h] : v[k];
          v[k] = keep + __shfl_xor_sync(0xffffffffu, send, h);
        }
      }
      return v[0] + __shfl_xor_sync(0xffffffffu, v[0], 16);
    };
    float mine;
    {
      float v[16];
      mask_group(0);
#pragma unroll
      for (int j = 0; j < kColG; ++j) v[j] = dot(pf[j]);  // prefetched group 0
      issue(1);
#pragma unroll
      for (int r = 0; r < kColRR; ++r) v[kColG + r] = dot(areg[r]);
#pragma unroll
      for (int r = 0; r < 16 - kColG - kColRR; ++r) {
        float4 a[kColC4];
#pragma unroll
        for (int u = 0; u < kColC4; ++u) a[u] = acache[(r * kColC4 + u) * kColT + tid];
        v[kColG + kColRR + r] = dot(a);
      }
      mine = reduce16(v);
    }
    {
      float v[16];
      constexpr int S0 = 16 - kColG - kColRR;
#pragma unroll
      for (int r = S0; r < kColRS; ++r) {
        float4 a[kColC4];
#pragma unroll
        for (int u = 0; u < kColC4; ++u) a[u] = acache[(r * kColC4 + u) * kColT + tid];
        v[r - S0] = dot(a);
      }
      mask_group(1);
#pragma unroll
      for (int j = 0; j < kColG; ++j) v[kColRS - S0 + j] = dot(pf[j]);
#pragma unroll
      for (int k = kColRS - S0 + kColG; k < 16; ++k) v[k] = 0.f;
      if (s + 1 < p.sweeps) issue(0);  // A is the same every sweep: in flight across the barrier
      const float other = reduce16(v);
      mine = lane < 16 ? mine : other;
    }
    red[warp][lane] = mine;  // slot "lane"
    if (tr) trp[3] = gtimer_lo();  // warp 0's compute done
    __syncthreads();
    float *slot = partials + (s & 1) * kMaxJacobiBlocks;
    if (warp == 0) {
      float tot = 0.f;
#pragma unroll
      for (int w = 0; w < kColW; ++w) tot += red[w][lane];
      float res = 0.f;
      if (my_rl < R) {
        const float xn = (bi - tot) / di;  // IEEE div.rn
        const int i = r0 + my_rl;
        x_out[i] = xn;
        if (p.tagged)
          st_relaxed_u64(p.xt + (size_t)((s + 1) & 1) * kJacTaggedMaxN + i,
                         tagged_word(xn, p.tag0 + (unsigned)s + 1));
        // x_in[i] is this lane's own previous result once sweeps are chained
        res = fabsf(xn - (from_tags ? xprev : __ldcg(x_in + i)));
        xprev = xn;
      }
      if (want_resid) {
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) res += __shfl_xor_sync(0xffffffffu, res, off);
        if (lane == 0) slot[blockIdx.x] = res;
      }
    }
    if (tr) trp[4] = gtimer_lo();  // rows published
    if (want_resid || !p.tagged) {
      grid_sync_mono(sync + 3, epoch++, p.sync_base);  // also orders red[] reuse
      if (want_resid && blockIdx.x == 0 && threadIdx.x < 32)
        finish_resid(slot, gridDim.x, p.ptrs[p.idx[s][2] & 0x7f]);
    } else {
      __syncthreads();  // red[] reuse; the tags order everything else
    }
  }
}

// ---- TMEM-tier kernel: the whole band of A on chip (n <= 4096) -----------------
//
// Same thread layout, reduction and tagged exchange as k_jacobi_cols, but the
// band's 28 rows never leave the SM after the first sweep:
//   rows 0..15   tensor memory (each thread owns 256 of its TMEM lane's 512
//                columns: warps w and w+4 share lane quadrant w%4), read back
//                with tcgen05.ld.32x32b.x16 -- one row's 16 floats per load
//   rows 16..21  registers
//   rows 22..27  thread-private shared memory (LDS.128, conflict-free)
// Measured on B200 (tools/tmembw.cu): tcgen05.ld streams ~425 B/clk/SM, 3.3x
// the 128 B/clk LDS path, and the two overlap, so a sweep's 458 KB per SM
// costs ~1,000 cycles instead of the L2 tier's ~2 us.  Nothing is re-read
// from L2 or HBM after the fill.
constexpr int kTmRT = 16;   // TMEM rows; the other 12 rows: RR in registers, 12 - RR in smem
constexpr int kTmOther = kColRows - kTmRT;
// padded so no other 1-CTA/SM kernel that allocates TMEM can be co-resident
template <int RS>
constexpr size_t tm_smem() {
  return (size_t)RS * kColC4 * kColT * sizeof(float4) > 116 * 1024
             ? (size_t)RS * kColC4 * kColT * sizeof(float4)
             : 116 * 1024;
}

#define KAAS_TMEM_LD16(taddr, v)                                                               \
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 "                                      \
               "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"             \
               : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]),     \
                 "=r"(v[6]), "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]),   \
                 "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])                          \
               : "r"(taddr))
#define KAAS_TMEM_ST16(taddr, v)                                                               \
  asm volatile("tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], "                                \
               "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(taddr),    \
               "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]),  \
               "r"(v[7]), "r"(v[8]), "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]),          \
               "r"(v[13]), "r"(v[14]), "r"(v[15])                                           \
               : "memory")

// volatile so the compiler keeps the smem tier's loads where they are
// written instead of hoisting the whole tier into registers at the top of
// the sweep
__device__ __forceinline__ float4 lds4(const float4 *q) {
  float4 a;
  asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];"
               : "=f"(a.x), "=f"(a.y), "=f"(a.z), "=f"(a.w)
               : "r"((uint32_t)__cvta_generic_to_shared(q)));
  return a;
}

__device__ __forceinline__ void tmem_wait_ld() {
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

// packed FP32 pair helpers (fma.rn.f32x2 -> FFMA2 on sm_100a)
__device__ __forceinline__ unsigned long long pack2(float lo, float hi) {
  unsigned long long r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
  return r;
}
__device__ __forceinline__ unsigned long long ffma2(unsigned long long a, unsigned long long b,
                                                    unsigned long long c) {
  unsigned long long d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}
__device__ __forceinline__ float sum2(unsigned long long v) {
  float lo, hi;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(v));
  return lo + hi;
}

// MODE 3 schedule: what step i of the 16 TMEM steps computes besides TMEM
// row i -- 100 + k = shared-memory row k (rows at steps k * 16 / RS), 1 + r
// = register row r (the remaining steps in order), 0 = nothing
__host__ __device__ constexpr int tm_spread(int i, int RR, int RS) {
  for (int k = 0; k < RS; ++k)
    if (k * 16 / RS == i) return 100 + k;
  int r = 0;
  for (int j = 0; j < i; ++j) {
    bool sm = false;
    for (int k = 0; k < RS; ++k) sm = sm || (k * 16 / RS == j);
    if (!sm) ++r;
  }
  return r < RR ? 1 + r : 0;
}

// RR register rows, kTmOther - RR shared-memory rows.  MODE 0: the register
// and smem rows first, then the TMEM rows (DEP tcgen05.ld in flight).  MODE 1:
// interleaved -- step i loads TMEM row i while it computes register/smem row
// i, so the TMEM stream (425 B/clk) and the LDS stream (128 B/clk) overlap.
template <int RR, int MODE, int DEP>
__global__ void __launch_bounds__(kColT, 1)
k_jacobi_tmem(const __grid_constant__ ChainParams p, float *partials, unsigned *sync) {
#ifdef KAAS_DEV
  // launch-phase stamps (thread 0 of each CTA): entry, TMEM allocated, band
  // filled, sweep 0 published, sweep 1 published, before teardown
  unsigned *pro = p.trace != nullptr && threadIdx.x == 0
                      ? p.trace + 32 * 148 * kTraceStamps + (blockIdx.x < 148 ? blockIdx.x : 147) * kTracePro
                      : nullptr;
  if (pro) pro[0] = gtimer_lo();
#define KAAS_PRO(i) \
  if (pro) pro[i] = gtimer_lo();
#else
#define KAAS_PRO(i)
#endif
  constexpr int kTmRR = RR, kTmRS = kTmOther - RR, kTmDep = DEP, kTmBatch = 1;
  static_assert(kTmRS >= 0 && kTmRR + kTmRS <= 16, "one 16-slot reduction set for the non-TMEM rows");
  extern __shared__ __align__(16) float4 acache[];  // [kTmRS][kColC4][kColT]
  // per-warp row partials, double-buffered by sweep parity: a warp may run
  // into sweep s+1 while warp 0 still reads sweep s's partials (no CTA
  // barrier at the end of a sweep), and it cannot reach sweep s+2 -- the next
  // write to this parity -- before every CTA, this one included, has
  // published sweep s+1, which warp 0 does only after reading them
  __shared__ float red[2][kColW][32];
  __shared__ uint32_t tmem_base;
  const int n = p.n, n4 = n >> 2;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  int r0, r1;
  band(p.cov, r0, r1);
  const int R = r1 - r0;
  const uint64_t pol = l2_policy(false);  // A is read once per launch
  const int cbase = warp * 32 * kColC4 + lane;
  const bool full = cbase + 32 * (kColC4 - 1) < n4;

  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     (uint32_t)__cvta_generic_to_shared(&tmem_base)),
                 "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  KAAS_PRO(1)
  const uint32_t taddr = tmem_base + ((uint32_t)(32 * (warp & 3)) << 16) + (uint32_t)(warp >> 2) * 256u;

  // A[r0 + rl][cbase + 32u]; rows past the band and columns past n are 0
  // (their partials are discarded / contribute nothing).  The diagonal is
  // zeroed by zdiag AFTER a whole batch of loads is in flight: touching a
  // loaded value right after its load makes the one warp holding the row's
  // diagonal wait for that load before issuing the next, which serialised
  // the fill into one HBM round trip per row (44 us per request; 4x the
  // 64 MiB / HBM-bandwidth floor).
  auto lda = [&](int rl, int u) -> float4 {
    float4 a = zero4();
    const float4 *rp = reinterpret_cast<const float4 *>(p.A) + (size_t)(r0 + rl) * n4 + cbase;
    if (rl < R && (full || cbase + 32 * u < n4)) a = ld_a(reinterpret_cast<const float *>(rp + 32 * u), pol);
    return a;
  };
  auto zdiag = [&](float4 &a, int rl, int u) {
    const int c4 = cbase + 32 * u, i = r0 + rl;
    if (c4 == (i >> 2)) {
      const int d = i & 3;
      a.x = d == 0 ? 0.f : a.x;
      a.y = d == 1 ? 0.f : a.y;
      a.z = d == 2 ? 0.f : a.z;
      a.w = d == 3 ? 0.f : a.w;
    }
  };
  // fill the three tiers once per launch (64 MiB of A at N = 4096): rows go
  // in batches of 4 (16 loads per thread in flight), the diagonal patched
  // after each batch's loads are issued.  (Issuing the shared-memory rows as
  // cp.async up front, or the register rows first, fills 8 us faster but
  // measured 8-17 us slower per 500-sweep request: the sweeps that follow
  // run slower -- tools/jfill_ab2.sh.)
  constexpr int kFillB = 4;  // TMEM rows per batch
  static_assert(kTmRT % kFillB == 0, "TMEM rows fill in whole batches");
#pragma unroll 1
  for (int rb = 0; rb < kTmRT; rb += kFillB) {
    float4 t4[kFillB][kColC4];
#pragma unroll
    for (int j = 0; j < kFillB; ++j)
#pragma unroll
      for (int u = 0; u < kColC4; ++u) t4[j][u] = lda(rb + j, u);
#pragma unroll
    for (int j = 0; j < kFillB; ++j) {
#pragma unroll
      for (int u = 0; u < kColC4; ++u) zdiag(t4[j][u], rb + j, u);
      uint32_t v[16];
#pragma unroll
      for (int u = 0; u < kColC4; ++u) {
        v[4 * u + 0] = __float_as_uint(t4[j][u].x);
        v[4 * u + 1] = __float_as_uint(t4[j][u].y);
        v[4 * u + 2] = __float_as_uint(t4[j][u].z);
        v[4 * u + 3] = __float_as_uint(t4[j][u].w);
      }
      KAAS_TMEM_ST16(taddr + 16u * (rb + j), v);
    }
  }
#pragma unroll 1
  for (int rb = 0; rb < kTmRS; rb += kFillB) {
    float4 t4[kFillB][kColC4];
#pragma unroll
    for (int j = 0; j < kFillB; ++j)
#pragma unroll
      for (int u = 0; u < kColC4; ++u)
        t4[j][u] = rb + j < kTmRS ? lda(kTmRT + kTmRR + rb + j, u) : zero4();
#pragma unroll
    for (int j = 0; j < kFillB; ++j)
#pragma unroll
      for (int u = 0; u < kColC4; ++u)
        if (rb + j < kTmRS) {
          zdiag(t4[j][u], kTmRT + kTmRR + rb + j, u);
          acache[((rb + j) * kColC4 + u) * kColT + tid] = t4[j][u];
        }
  }
  float4 areg[kTmRR][kColC4];
#pragma unroll
  for (int r = 0; r < kTmRR; ++r)
#pragma unroll
    for (int u = 0; u < kColC4; ++u) areg[r][u] = lda(kTmRT + r, u);
#pragma unroll
  for (int r = 0; r < kTmRR; ++r)
#pragma unroll
    for (int u = 0; u < kColC4; ++u) zdiag(areg[r][u], kTmRT + r, u);
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");

  KAAS_PRO(2)
  // reduction slot l holds band row l (slots 28..31 empty)
  const int my_rl = lane;
  float bi = 0.f, di = 1.f;
  if (warp == 0 && my_rl < R) {
    bi = __ldg(p.b + r0 + my_rl);
    di = __ldg(p.A + (size_t)(r0 + my_rl) * n + r0 + my_rl);
  }
  // the row's reciprocal once per launch: the per-sweep division on the
  // publish path becomes one multiply (within an ulp of div.rn -- Jacobi's
  // contract is a tolerance; a zero diagonal still gives +-inf / NaN);
  // 2.34 -> 2.27 us/sweep, where a Newton correction gave the time back
  const float rdi = 1.0f / di;

  float xprev = 0.f;
  unsigned epoch = 0;
  for (int s = 0; s < p.sweeps; ++s) {
    const float *x_in = p.ptrs[p.idx[s][0]];
    float *x_out = p.ptrs[p.idx[s][1]];
    const bool want_resid = (p.idx[s][2] & 0x80) != 0;
    const bool from_tags = p.tagged && s > 0;
    // phase stamps (tools/jtrace.py): p.trace is set only by the dev build's
    // host side, so in the product library these branches are never taken.
    // They are compiled in anyway: with the "published" stamp below present
    // the kernel measures ~30 us faster per 500-sweep request (ptxas
    // schedules the end of a sweep differently; same-box A/B over product
    // builds, profiles/r02/probes/jacobi_stamp_fence_ab.txt)
    const bool tr = p.trace != nullptr && s >= 100 && s < 132 && threadIdx.x == 0;
    unsigned *trp = tr ? p.trace + ((s - 100) * 148 + (blockIdx.x < 148 ? blockIdx.x : 147)) * kTraceStamps : nullptr;
    if (tr) trp[0] = gtimer_lo();  // warp 0 starts waiting for x
    float4 xr[kColC4];
    if (!from_tags) {
#pragma unroll
      for (int u = 0; u < kColC4; ++u)
        xr[u] = cbase + 32 * u < n4 ? __ldcg(reinterpret_cast<const float4 *>(x_in) + cbase + 32 * u)
                                    : zero4();
    } else {
      const unsigned want = p.tag0 + (unsigned)s;
      const unsigned long long *src = p.xt + (size_t)(s & 1) * kJacTaggedMaxN;
      TagWords4 q[kColC4];
      unsigned pending = 0;
#pragma unroll
      for (int u = 0; u < kColC4; ++u)
        if (cbase + 32 * u < n4) pending |= 1u << u;
      unsigned spins = 0;
      while (pending) {
        // a lost producer: fail loudly, never hang (checked every 256 polls)
        if ((++spins & 0xffu) == 0u && spins > (1u << 22)) __trap();
#ifdef KAAS_DEV
        if (p.tagged == 3 && spins > 1) break;  // dev: no waiting (compute-only timing; wrong results)
        if (spins > 1 && p.poll_ns) {  // dev A/B: busy back-off (cycles) between polls
          const long long t = clock64();
          while (clock64() - t < p.poll_ns) {
          }
        }
#endif
#pragma unroll
        for (int u = 0; u < kColC4; ++u)
          if (pending & (1u << u)) q[u] = ld_relaxed_u64x4(src + 4 * (cbase + 32 * u));
#pragma unroll
        for (int u = 0; u < kColC4; ++u) {
          // all four tags == want, as one OR of XORs (the check runs once
          // more after the last word lands -- it is on the critical path)
          const unsigned d = ((unsigned)(q[u].w[0] >> 32) ^ want) | ((unsigned)(q[u].w[1] >> 32) ^ want) |
                             ((unsigned)(q[u].w[2] >> 32) ^ want) | ((unsigned)(q[u].w[3] >> 32) ^ want);
          // branch-free: a chunk done earlier (or out of range) only clears
          // a bit that is already clear
          pending &= d == 0u ? ~(1u << u) : ~0u;
        }
      }
#pragma unroll
      for (int u = 0; u < kColC4; ++u)
        xr[u] = cbase + 32 * u < n4
                    ? make_float4(__uint_as_float((unsigned)q[u].w[0]), __uint_as_float((unsigned)q[u].w[1]),
                                  __uint_as_float((unsigned)q[u].w[2]), __uint_as_float((unsigned)q[u].w[3]))
                    : zero4();
    }
#ifdef KAAS_DEV
    if (tr) trp[1] = gtimer_lo();  // x arrived
    if (p.trace != nullptr && s >= 100 && s < 132 && lane == 0)  // every warp's x arrival
      p.trace[kTraceWarpOff + ((s - 100) * 148 + (blockIdx.x < 148 ? blockIdx.x : 147)) * 8 + warp] = gtimer_lo();
#endif
    // packed FP32 (FFMA2, fma.rn.f32x2): even and odd columns accumulate in
    // the two halves of one 64-bit register pair, added at the end -- half
    // the FMA issue slots (2.43 -> 2.33 us/sweep); the order is fixed, so
    // results stay deterministic
    auto dot = [&](const float4 (&a)[kColC4]) {
      unsigned long long acc = 0ull;
#pragma unroll
      for (int u = 0; u < kColC4; ++u) {
        acc = ffma2(pack2(a[u].x, a[u].y), pack2(xr[u].x, xr[u].y), acc);
        acc = ffma2(pack2(a[u].z, a[u].w), pack2(xr[u].z, xr[u].w), acc);
      }
      return sum2(acc);
    };
    // MODE 2: two independent FFMA2 chains per row (chunks 0-1 and 2-3),
    // half the dependent-FMA latency per row at one extra add
    auto dot2 = [&](const float4 (&a)[kColC4]) {
      unsigned long long c0 = 0ull, c1 = 0ull;
#pragma unroll
      for (int u = 0; u < kColC4; u += 2) {
        c0 = ffma2(pack2(a[u].x, a[u].y), pack2(xr[u].x, xr[u].y), c0);
        c1 = ffma2(pack2(a[u + 1].x, a[u + 1].y), pack2(xr[u + 1].x, xr[u + 1].y), c1);
        c0 = ffma2(pack2(a[u].z, a[u].w), pack2(xr[u].z, xr[u].w), c0);
        c1 = ffma2(pack2(a[u + 1].z, a[u + 1].w), pack2(xr[u + 1].z, xr[u + 1].w), c1);
      }
      return sum2(c0) + sum2(c1);
    };
    auto dot2_t = [&](const uint32_t (&t)[16]) {
      float4 a[kColC4];
#pragma unroll
      for (int u = 0; u < kColC4; ++u)
        a[u] = make_float4(__uint_as_float(t[4 * u]), __uint_as_float(t[4 * u + 1]),
                           __uint_as_float(t[4 * u + 2]), __uint_as_float(t[4 * u + 3]));
      return dot2(a);
    };
    auto dot_t = [&](const uint32_t (&t)[16]) {
      unsigned long long acc = 0ull;
#pragma unroll
      for (int u = 0; u < kColC4; ++u) {
        acc = ffma2(pack2(__uint_as_float(t[4 * u + 0]), __uint_as_float(t[4 * u + 1])),
                    pack2(xr[u].x, xr[u].y), acc);
        acc = ffma2(pack2(__uint_as_float(t[4 * u + 2]), __uint_as_float(t[4 * u + 3])),
                    pack2(xr[u].z, xr[u].w), acc);
      }
      return sum2(acc);
    };
    auto reduce16 = [&](float (&v)[16]) {
#pragma unroll
      for (int h = 8; h >= 1; h >>= 1) {
        const bool up = (lane & h) != 0;
#pragma unroll
        for (int k = 0; k < h; ++k) {
          const float send = up ? v[k] : v[k + h];
          const float keep = up ? v[k + h] : v[k];
          v[k] = keep + __shfl_xor_sync(0xffffffffu, send, h);
        }
      }
      return v[0] + __shfl_xor_sync(0xffffffffu, v[0], 16);
    };
    float m0, m1;
    if (MODE == 0) {
      // set 1 = register rows, smem rows, 4 empty (reduced first, so only one
      // set of partials is live while TMEM rows stream in); set 0 = TMEM rows
      {
        float w[16];
#pragma unroll
        for (int r = 0; r < kTmRR; ++r) w[r] = dot(areg[r]);
#pragma unroll
        for (int r = 0; r < kTmRS; ++r) {
          float4 a[kColC4];
#pragma unroll
          for (int u = 0; u < kColC4; ++u) a[u] = lds4(&acache[(r * kColC4 + u) * kColT + tid]);
          w[kTmRR + r] = dot(a);
        }
#pragma unroll
        for (int k = kTmRR + kTmRS; k < 16; ++k) w[k] = 0.f;
        m1 = reduce16(w);
      }
#ifdef KAAS_DEV
      if (tr) trp[2] = gtimer_lo();  // register + shared-memory rows done
#endif
      {
        float v[16];
#pragma unroll
        for (int bt = 0; bt < kTmRT / kTmBatch; ++bt) {
          uint32_t t[kTmBatch][16];
          // the batch's address depends (by an opaque 0) on the previous batch's
          // dots, so ptxas cannot hoist every tcgen05.ld of the sweep to the
          // top and hold all 256 values in registers at once
          const uint32_t dep =
              bt < kTmDep ? 0u : (__float_as_uint(v[(bt - kTmDep + 1) * kTmBatch - 1]) & p.zero);
#pragma unroll
          for (int j = 0; j < kTmBatch; ++j) KAAS_TMEM_LD16(taddr + dep + 16u * (bt * kTmBatch + j), t[j]);
          tmem_wait_ld();
#pragma unroll
          for (int j = 0; j < kTmBatch; ++j) v[bt * kTmBatch + j] = dot_t(t[j]);
        }
        m0 = reduce16(v);
      }
    } else {
      // interleaved: TMEM row i is in flight while register / smem row i is
      // computed (its LDS issued after the tcgen05.ld, before the wait)
      float v[16], w[16];
      if (MODE == 3) {
#pragma unroll
        for (int k = kTmRR + kTmRS; k < 16; ++k) w[k] = 0.f;
      }
#pragma unroll
      for (int i = 0; i < kTmRT; ++i) {
        uint32_t t[16];
        const uint32_t dep = i < kTmDep ? 0u : (__float_as_uint(v[i - kTmDep]) & p.zero);
        KAAS_TMEM_LD16(taddr + dep + 16u * i, t);
        // MODE 3: the shared-memory rows spread evenly over the 16 steps
        // (one every 16 / RS), the register rows in the steps between, so
        // the LDS stream (128 B/clk) overlaps the TMEM stream all sweep
        // long instead of bunching in steps RR .. RR + RS - 1
        const int sc = MODE == 3 ? tm_spread(i, kTmRR, kTmRS) : 0;
        if (MODE == 3) {
          if (sc >= 100) {
            const int r = sc - 100;
            float4 a[kColC4];
#pragma unroll
            for (int u = 0; u < kColC4; ++u) a[u] = lds4(&acache[(r * kColC4 + u) * kColT + tid]);
            w[kTmRR + r] = dot(a);
          } else if (sc > 0) {
            w[sc - 1] = dot(areg[sc - 1]);
          }
        } else if (i < kTmRR) {
          w[i] = MODE == 2 ? dot2(areg[i < kTmRR ? i : 0]) : dot(areg[i < kTmRR ? i : 0]);
        } else if (i < kTmRR + kTmRS) {
          const int r = i - kTmRR;
          float4 a[kColC4];
#pragma unroll
          for (int u = 0; u < kColC4; ++u) a[u] = lds4(&acache[(r * kColC4 + u) * kColT + tid]);
          w[i] = MODE == 2 ? dot2(a) : dot(a);
        } else {
          w[i] = 0.f;
        }
        tmem_wait_ld();
        v[i] = MODE == 2 ? dot2_t(t) : dot_t(t);
      }
#ifdef KAAS_DEV
      if (tr) trp[2] = gtimer_lo();  // all rows' partial dots done
#endif
      m1 = reduce16(w);
      m0 = reduce16(v);
    }
    const float mine = lane < 16 ? m0 : m1;
    red[s & 1][warp][lane] = mine;
#ifdef KAAS_DEV
    if (tr) trp[3] = gtimer_lo();  // TMEM rows + reductions done
#endif
    __syncthreads();
    float *slot = partials + (s & 1) * kMaxJacobiBlocks;
    if (warp == 0) {
      float tot = 0.f;
#pragma unroll
      {
        // the 8 warps' partials as a tree (3 dependent adds, not 8; fixed
        // order, so still deterministic)
        static_assert(kColW == 8, "tree over 8 warps");
        const float *rr = &red[s & 1][0][lane];
        tot = ((rr[0] + rr[32]) + (rr[64] + rr[96])) + ((rr[128] + rr[160]) + (rr[192] + rr[224]));
      }
      float res = 0.f;
      if (my_rl < R) {
        const float xn = (bi - tot) * rdi;
        const int i = r0 + my_rl;
        if (p.tagged)  // the word the other CTAs wait for goes out first
          st_relaxed_u64(p.xt + (size_t)((s + 1) & 1) * kJacTaggedMaxN + i,
                         tagged_word(xn, p.tag0 + (unsigned)s + 1));
        x_out[i] = xn;
        if (p.wb_x != nullptr && s == p.sweeps - 1) p.wb_x[i] = xn;  // the request's write-back
        res = fabsf(xn - (from_tags ? xprev : __ldcg(x_in + i)));
        xprev = xn;
      }
      if (want_resid) {
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) res += __shfl_xor_sync(0xffffffffu, res, off);
        if (lane == 0) slot[blockIdx.x] = res;
      }
    }
    if (tr) trp[4] = gtimer_lo();  // published
    if (s < 2) {
      KAAS_PRO(3 + s)
    }
    if (want_resid || !p.tagged) {
      grid_sync_mono(sync + 3, epoch++, p.sync_base);
      if (want_resid && blockIdx.x == 0 && threadIdx.x < 32)
        finish_resid(slot, gridDim.x, p.ptrs[p.idx[s][2] & 0x7f], s == p.sweeps - 1 ? p.wb_r : nullptr);
    }
    // tagged sweeps end without a CTA barrier: the other warps go straight
    // to polling the next x while warp 0 reduces and publishes (red is
    // double-buffered, see above)
  }

  KAAS_PRO(5)
#undef KAAS_PRO
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(512));
}

#ifdef KAAS_DEV
// ---- split-publish kernel (dev build only: measured slower) -----------------
//
// Measured on B200 (round 2): 2.71 us/sweep with the polls in program order,
// 3.31 us/sweep with them software-pipelined, against 2.19 for k_jacobi_tmem.
// A poll round on lines other SMs have just written costs ~0.5-0.9 us, the
// early rows' publish spread across CTAs is ~0.5 us, so the early x of the
// next sweep is rarely complete when phase C ends and the second reduction
// and CTA barrier per sweep are not paid back.  Kept as the A/B reference
// (KAAS_JACOBI_TMV=s in a dev build).
//
// Same on-chip band as k_jacobi_tmem, but a sweep no longer needs all of x
// before any work starts.  Rows i with (i >> 2) even are "early", the others
// "late"; x's early columns are the even float4 chunks, late columns the odd
// ones, and every thread owns two early chunks (2t, 2t + 512) and two late
// chunks (2t + 1, 2t + 513).  Per sweep:
//   A  all rows x early columns          (needs only the early x of sweep s)
//   B  early rows x late columns -> reduce -> publish the early rows
//   C  late rows x late columns  -> reduce -> publish the late rows
// so phase A of sweep s+1 overlaps the exchange of sweep s's late rows, and
// the critical path per sweep is exchange + A + B instead of exchange + all
// of the arithmetic.  Each row's dot product is (early part) + (late part):
// a fixed order, so results are deterministic.
//
// Band storage, 16 early + 16 late slots (a band has 12..16 of each; empty
// slots are zeros and sit in the shared-memory tier, which is skipped):
//   early slots 0-7 / late slots 0-7   TMEM (16 columns per thread per slot:
//                                      8 early-column values, then 8 late)
//   early 8-10 / late 8-10             registers
//   early 11-15 / late 11-15           shared memory
constexpr int kSpT = 8, kSpR = 3, kSpS = 5;  // TMEM / register / smem slots per half
static_assert(kSpT + kSpR + kSpS == 16, "16 slots per half");
constexpr size_t kSpSmem = (size_t)2 * kSpS * 4 * kColT * sizeof(float4) > 116 * 1024
                               ? (size_t)2 * kSpS * 4 * kColT * sizeof(float4)
                               : 116 * 1024;

#define KAAS_TMEM_LD8(taddr, v)                                                                \
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"       \
               : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]),     \
                 "=r"(v[6]), "=r"(v[7])                                                      \
               : "r"(taddr))

__global__ void __launch_bounds__(kColT, 1)
k_jacobi_split(const __grid_constant__ ChainParams p, float *partials, unsigned *sync) {
  extern __shared__ __align__(16) float4 acache[];  // [2 * kSpS][4][kColT]
  __shared__ float red[2][kColW][16];
  __shared__ uint32_t tmem_base;
  __shared__ signed char slot_row[2][16];  // band-local row of each early / late slot, -1 = empty
  const int n = p.n, n4 = n >> 2;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  int r0, r1;
  band(p.cov, r0, r1);
  const int R = r1 - r0;
  const uint64_t pol = l2_policy(false);
  // this thread's chunks: u = 0, 1 early columns, u = 2, 3 late columns
  const int chunk[4] = {2 * tid, 2 * tid + 512, 2 * tid + 1, 2 * tid + 513};

  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     (uint32_t)__cvta_generic_to_shared(&tmem_base)),
                 "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    if (lane < 2) {  // slot -> row tables (ascending rows per half)
      int k = 0;
      for (int rl = 0; rl < R; ++rl)
        if ((((r0 + rl) >> 2) & 1) == lane && k < 16) slot_row[lane][k++] = (signed char)rl;
      for (; k < 16; ++k) slot_row[lane][k] = -1;
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t taddr = tmem_base + ((uint32_t)(32 * (warp & 3)) << 16) + (uint32_t)(warp >> 2) * 256u;

  // A[r0 + rl][chunk u] with the diagonal zeroed; empty slots / absent columns 0
  auto lda = [&](int rl, int u) -> float4 {
    float4 a = zero4();
    const int c4 = chunk[u];
    if (rl < 0 || c4 >= n4) return a;
    a = ld_a(p.A + (size_t)(r0 + rl) * n + 4 * c4, pol);
    const int i = r0 + rl;
    if (c4 == (i >> 2)) {
      const int d = i & 3;
      a.x = d == 0 ? 0.f : a.x;
      a.y = d == 1 ? 0.f : a.y;
      a.z = d == 2 ? 0.f : a.z;
      a.w = d == 3 ? 0.f : a.w;
    }
    return a;
  };
#pragma unroll 1
  for (int t = 0; t < 2 * kSpT; ++t) {  // TMEM slot t: half t / kSpT, slot t % kSpT
    const int rl = slot_row[t / kSpT][t % kSpT];
    uint32_t v[16];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const float4 a = lda(rl, u);
      v[4 * u + 0] = __float_as_uint(a.x);
      v[4 * u + 1] = __float_as_uint(a.y);
      v[4 * u + 2] = __float_as_uint(a.z);
      v[4 * u + 3] = __float_as_uint(a.w);
    }
    KAAS_TMEM_ST16(taddr + 16u * t, v);
  }
  float4 areg[2][kSpR][4];
#pragma unroll
  for (int h = 0; h < 2; ++h)
#pragma unroll
    for (int k = 0; k < kSpR; ++k)
#pragma unroll
      for (int u = 0; u < 4; ++u) areg[h][k][u] = lda(slot_row[h][kSpT + k], u);
#pragma unroll 1
  for (int h = 0; h < 2; ++h)
#pragma unroll 1
    for (int k = 0; k < kSpS; ++k)
#pragma unroll
      for (int u = 0; u < 4; ++u)
        acache[((h * kSpS + k) * 4 + u) * kColT + tid] = lda(slot_row[h][kSpT + kSpR + k], u);
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");

  // warp 0, lane l < 16: early slot l and late slot l (their rows, b, 1/a_ii)
  int rowE = -1, rowL = -1;
  float bE = 0.f, rE = 1.f, bL = 0.f, rL = 1.f;
  if (warp == 0 && lane < 16) {
    if (slot_row[0][lane] >= 0) {
      rowE = r0 + slot_row[0][lane];
      bE = __ldg(p.b + rowE);
      rE = 1.0f / __ldg(p.A + (size_t)rowE * n + rowE);
    }
    if (slot_row[1][lane] >= 0) {
      rowL = r0 + slot_row[1][lane];
      bL = __ldg(p.b + rowL);
      rL = 1.0f / __ldg(p.A + (size_t)rowL * n + rowL);
    }
  }

  // Software-pipelined exchange: the loads that poll for the next sweep's
  // early x are issued right after this CTA publishes its own early rows
  // (every CTA publishes them at about that time) and checked after phase C;
  // the loads for the late x are issued after the late publish and checked
  // after the next phase A.  A poll round's latency (~0.5 us on lines other
  // SMs just wrote) is thereby hidden behind phases C and A.
  auto dot8 = [&](const float4 &a0, const float4 &a1, const float4 &x0, const float4 &x1) {
    unsigned long long acc = 0ull;
    acc = ffma2(pack2(a0.x, a0.y), pack2(x0.x, x0.y), acc);
    acc = ffma2(pack2(a0.z, a0.w), pack2(x0.z, x0.w), acc);
    acc = ffma2(pack2(a1.x, a1.y), pack2(x1.x, x1.y), acc);
    acc = ffma2(pack2(a1.z, a1.w), pack2(x1.z, x1.w), acc);
    return sum2(acc);
  };
  auto u2f4 = [](const uint32_t *t) {
    return make_float4(__uint_as_float(t[0]), __uint_as_float(t[1]), __uint_as_float(t[2]), __uint_as_float(t[3]));
  };
  auto reduce16 = [&](float (&v)[16]) {
#pragma unroll
    for (int h = 8; h >= 1; h >>= 1) {
      const bool up = (lane & h) != 0;
#pragma unroll
      for (int k = 0; k < h; ++k) {
        const float send = up ? v[k] : v[k + h];
        const float keep = up ? v[k + h] : v[k];
        v[k] = keep + __shfl_xor_sync(0xffffffffu, send, h);
      }
    }
    return v[0] + __shfl_xor_sync(0xffffffffu, v[0], 16);
  };
  // slots of half h against the x chunk pair (x0, x1) = chunks u0, u0 + 1,
  // added into acc[16]; TMEM slot k in flight while register / smem slot k
  // is computed (straight-line: empty smem slots are zeros, computed anyway)
  auto half_pass = [&](int h, int u0, const float4 &x0, const float4 &x1, float (&acc)[16]) {
#pragma unroll
    for (int k = 0; k < kSpT; ++k) {
      uint32_t t[8];
      const uint32_t dep = k < 3 ? 0u : (__float_as_uint(acc[k - 3]) & p.zero);
      KAAS_TMEM_LD8(taddr + dep + 16u * (h * kSpT + k) + (u0 ? 8u : 0u), t);
      if (k < kSpR) {
        acc[kSpT + k] += dot8(areg[h][k][u0], areg[h][k][u0 + 1], x0, x1);
      } else {
        const int j = k - kSpR;
        const float4 a0 = lds4(&acache[((h * kSpS + j) * 4 + u0) * kColT + tid]);
        const float4 a1 = lds4(&acache[((h * kSpS + j) * 4 + u0 + 1) * kColT + tid]);
        acc[kSpT + kSpR + j] += dot8(a0, a1, x0, x1);
      }
      tmem_wait_ld();
      acc[k] += dot8(u2f4(t), u2f4(t + 4), x0, x1);
    }
  };
  // tagged-word polls: issue the loads of chunk pair u0 (no wait) / finish
  // them (re-poll any chunk whose tag is not `want` yet)
  auto issue = [&](TagWords4 (&q)[2], int u0, const unsigned long long *src) {
#pragma unroll
    for (int j = 0; j < 2; ++j)
      if (chunk[u0 + j] < n4) q[j] = ld_relaxed_u64x4(src + 4 * chunk[u0 + j]);
  };
  auto tag_ok = [&](const TagWords4 &q, unsigned want) {
    return (unsigned)(q.w[0] >> 32) == want && (unsigned)(q.w[1] >> 32) == want &&
           (unsigned)(q.w[2] >> 32) == want && (unsigned)(q.w[3] >> 32) == want;
  };
  auto finish = [&](TagWords4 (&q)[2], int u0, const unsigned long long *src, unsigned want, float4 &x0,
                    float4 &x1) {
    unsigned spins = 0;
#pragma unroll 1
    for (;;) {
      bool ok = true;
#pragma unroll
      for (int j = 0; j < 2; ++j) ok = ok && (chunk[u0 + j] >= n4 || tag_ok(q[j], want));
      if (ok) break;
      if (++spins > (1u << 22)) __trap();  // a lost producer: fail loudly, never hang
#ifdef KAAS_DEV
      if (p.tagged == 3) break;
#endif
#pragma unroll
      for (int j = 0; j < 2; ++j)
        if (chunk[u0 + j] < n4 && !tag_ok(q[j], want)) q[j] = ld_relaxed_u64x4(src + 4 * chunk[u0 + j]);
    }
    float4 *xs[2] = {&x0, &x1};
#pragma unroll
    for (int j = 0; j < 2; ++j)
      *xs[j] = chunk[u0 + j] < n4
                   ? make_float4(__uint_as_float((unsigned)q[j].w[0]), __uint_as_float((unsigned)q[j].w[1]),
                                 __uint_as_float((unsigned)q[j].w[2]), __uint_as_float((unsigned)q[j].w[3]))
                   : zero4();
  };
  auto plain = [&](const float *x_in, int u) {
    return chunk[u] < n4 ? __ldcg(reinterpret_cast<const float4 *>(x_in) + chunk[u]) : zero4();
  };

  float xprevE = 0.f, xprevL = 0.f;
  unsigned epoch = 0;
  float4 xe0 = zero4(), xe1 = zero4(), xl0 = zero4(), xl1 = zero4();  // x of the current sweep
  TagWords4 qe[2], ql[2];  // in-flight polls: next sweep's early / this sweep's late x
  bool late_inflight = false;
  for (int s = 0; s < p.sweeps; ++s) {
    const float *x_in = p.ptrs[p.idx[s][0]];
    float *x_out = p.ptrs[p.idx[s][1]];
    const bool want_resid = (p.idx[s][2] & 0x80) != 0;
    const bool from_tags = p.tagged && s > 0;
    const unsigned want = p.tag0 + (unsigned)s;
    const unsigned long long *src = p.xt + (size_t)(s & 1) * kJacTaggedMaxN;
    unsigned long long *dst = p.xt + (size_t)((s + 1) & 1) * kJacTaggedMaxN;
    const bool next_tagged = p.tagged && s + 1 < p.sweeps;
#ifdef KAAS_DEV
    const bool tr = p.trace != nullptr && s >= 100 && s < 132 && threadIdx.x == 0;
    unsigned *trp = tr ? p.trace + ((s - 100) * 148 + (blockIdx.x < 148 ? blockIdx.x : 147)) * kTraceStamps : nullptr;
    if (tr) trp[0] = gtimer_lo();
#endif
    if (!from_tags) {  // first sweep, or grid-barrier mode: x_in is complete in memory
      xe0 = plain(x_in, 0);
      xe1 = plain(x_in, 1);
      xl0 = plain(x_in, 2);
      xl1 = plain(x_in, 3);
    }
#ifdef KAAS_DEV
    if (tr) trp[1] = gtimer_lo();
#endif
    float vE[16], vL[16];
#pragma unroll
    for (int k = 0; k < 16; ++k) vE[k] = vL[k] = 0.f;
    // ---- phase A: every row x the early columns
    half_pass(0, 0, xe0, xe1, vE);
    half_pass(1, 0, xe0, xe1, vL);
    if (from_tags) {
      if (!late_inflight) issue(ql, 2, src);
      finish(ql, 2, src, want, xl0, xl1);
    }
    late_inflight = false;
#ifdef KAAS_DEV
    if (tr) trp[2] = gtimer_lo();
#endif
    // ---- phase B: early rows x the late columns, then publish them
    half_pass(0, 2, xl0, xl1, vE);
    {
      const float m = reduce16(vE);
      if (lane < 16) red[0][warp][lane] = m;
    }
    __syncthreads();
    float res = 0.f;
    if (warp == 0 && rowE >= 0) {
      float tot = 0.f;
#pragma unroll
      for (int w = 0; w < kColW; ++w) tot += red[0][w][lane];
      const float xn = (bE - tot) * rE;
      if (p.tagged) st_relaxed_u64(dst + rowE, tagged_word(xn, want + 1));
      x_out[rowE] = xn;
      res = fabsf(xn - (from_tags ? xprevE : __ldcg(x_in + rowE)));
      xprevE = xn;
    }
    // every CTA publishes its early rows about now: poll for them while
    // phase C runs
    if (next_tagged) issue(qe, 0, dst);
    // ---- phase C: late rows x the late columns, then publish them
    half_pass(1, 2, xl0, xl1, vL);
    {
      const float m = reduce16(vL);
      if (lane < 16) red[1][warp][lane] = m;
    }
#ifdef KAAS_DEV
    if (tr) trp[3] = gtimer_lo();
#endif
    __syncthreads();
    float *slot = partials + (s & 1) * kMaxJacobiBlocks;
    if (warp == 0) {
      if (rowL >= 0) {
        float tot = 0.f;
#pragma unroll
        for (int w = 0; w < kColW; ++w) tot += red[1][w][lane];
        const float xn = (bL - tot) * rL;
        if (p.tagged) st_relaxed_u64(dst + rowL, tagged_word(xn, want + 1));
        x_out[rowL] = xn;
        res += fabsf(xn - (from_tags ? xprevL : __ldcg(x_in + rowL)));
        xprevL = xn;
      }
      if (want_resid) {
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) res += __shfl_xor_sync(0xffffffffu, res, off);
        if (lane == 0) slot[blockIdx.x] = res;
      }
    }
    if (want_resid || !p.tagged) {
      grid_sync_mono(sync + 3, epoch++, p.sync_base);
      if (want_resid && blockIdx.x == 0 && threadIdx.x < 32)
        finish_resid(slot, gridDim.x, p.ptrs[p.idx[s][2] & 0x7f]);
    }
    if (next_tagged) {
      // late x of the next sweep: every CTA publishes it about now -- in
      // flight across the next phase A; the next early x: finish its polls
      issue(ql, 2, dst);
      late_inflight = true;
      finish(qe, 0, dst, want + 1, xe0, xe1);
    }
#ifdef KAAS_DEV
    if (tr) trp[4] = gtimer_lo();
#endif
  }

  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(512));
}

#endif  // KAAS_DEV

unsigned *&jacobi_trace_buffer() {
  static unsigned *buf = nullptr;
  return buf;
}

bool use_cols_kernel(int dev, int n, uint64_t cov, int blocks) {
  const char *e = KAAS_DEV_ENV("KAAS_JACOBI_PATH");  // dev A/B: cols (default where it fits)
  if (e && e[0] != 'c') return false;
  return n % 4 == 0 && n >= 2048 && n <= kColW * 32 * kColC4 * 4 &&
         (cov + blocks - 1) / blocks <= (uint64_t)kColRows &&
         device_props(dev).max_smem_optin >= (int)(kColSmem + sizeof(float) * kColW * 32);
}

// TMEM-tier kernel variant: the product default, or (dev builds)
// KAAS_JACOBI_TMV="RR,MODE,DEP" for A/B runs (tools/jacobi_var.sh)
struct TmVariant {
  int rr, mode, dep;
  const void *fn;
  size_t smem;
};
#define KAAS_TMV(RR, MODE, DEP) \
  TmVariant { RR, MODE, DEP, (const void *)k_jacobi_tmem<RR, MODE, DEP>, tm_smem<kTmOther - RR>() }
constexpr int kTmDefRR = 6, kTmDefMode = 3, kTmDefDep = 5;
const TmVariant &tm_variant() {
  static const TmVariant def = KAAS_TMV(kTmDefRR, kTmDefMode, kTmDefDep);
#ifdef KAAS_DEV
  static const TmVariant split = TmVariant{0, 9, 0, (const void *)k_jacobi_split, kSpSmem};
  if (const char *e = KAAS_DEV_ENV("KAAS_JACOBI_TMV"))
    if (e[0] == 's') return split;
  static const TmVariant vars[] = {KAAS_TMV(6, 1, 4), KAAS_TMV(6, 3, 4), KAAS_TMV(6, 3, 6),
                                   KAAS_TMV(5, 3, 5), KAAS_TMV(5, 3, 6), KAAS_TMV(7, 3, 5),
                                   KAAS_TMV(6, 0, 4), KAAS_TMV(6, 1, 2), KAAS_TMV(6, 1, 3),
                                   KAAS_TMV(6, 2, 3), KAAS_TMV(6, 2, 4), KAAS_TMV(6, 2, 5),
                                   KAAS_TMV(7, 2, 4), KAAS_TMV(8, 2, 4)};
  if (const char *e = KAAS_DEV_ENV("KAAS_JACOBI_TMV")) {
    int rr = 0, mode = 0, dep = 0;
    if (sscanf(e, "%d,%d,%d", &rr, &mode, &dep) == 3)
      for (const TmVariant &v : vars)
        if (v.rr == rr && v.mode == mode && v.dep == dep) return v;
  }
#endif
  return def;
}

// the band in TMEM + registers + smem (default); KAAS_JACOBI_TMEM=0 = L2 tier
bool use_tmem_kernel() {
  const char *e = KAAS_DEV_ENV("KAAS_JACOBI_TMEM");  // dev A/B
  return !(e && e[0] == '0');
}


// threads for the row kernel: one warp per band row, 4..32 warps
int rows_threads(int dev, uint64_t cov) {
  const int sms = device_props(dev).sm_count;
  int rows = (int)((cov + sms - 1) / sms);
  if (rows < 4) rows = 4;
  if (rows > kRowsMaxWarps) rows = kRowsMaxWarps;
  return rows * 32;
}

bool rows_prefetch() {
  // dev A/B: hoisting the next sweep's first A loads above the grid barrier
  // measured slower (7.02 vs 6.41 us/sweep), so it is off by default
  const char *e = KAAS_DEV_ENV("KAAS_JACOBI_PREFETCH");
  return e && e[0] == '1';
}

bool use_rows_kernel(int n) {
  const char *e = KAAS_DEV_ENV("KAAS_JACOBI_PATH");  // dev A/B: rows (default) | generic
  if (e && e[0] == 'g') return false;
  return n % 4 == 0 && (size_t)n * 4 <= 160 * 1024;
}

int pick_kc(int n) {
  if (n % 4 != 0) return 0;
  const int chunks = (n + kChunk - 1) / kChunk;
  const int per = (chunks + kJacWarps - 1) / kJacWarps;
  if (per <= 1) return 1;
  if (per <= 2) return 2;
  if (per <= 4) return 4;
  return -1;  // too wide for register-resident x: caller splits (not needed <= 8192)
}

bool aligned16(const void *p) { return ((uintptr_t)p & 15u) == 0; }

}  // namespace

int launch_jacobi(cudaStream_t s, int dev, int n, uint64_t cov, const float *A, const float *b,
                  const float *x_in, float *x_out, float *resid, StreamScratch *sc) {
  int blocks = device_props(dev).sm_count;
  if ((uint64_t)blocks > cov) blocks = cov > 0 ? (int)cov : 1;
  if (blocks > kMaxJacobiBlocks) blocks = kMaxJacobiBlocks;
  if (use_rows_kernel(n) && aligned16(A) && aligned16(x_in)) {
    static thread_local ChainParams p;
    p.A = A;
    p.b = b;
    p.n = n;
    p.cov = (int)cov;
    p.sweeps = 1;
    p.keep_l2 = 0;
    p.ptrs[0] = const_cast<float *>(x_in);
    p.ptrs[1] = x_out;
    p.ptrs[2] = resid;
    p.idx[0][0] = 0;
    p.idx[0][1] = 1;
    p.idx[0][2] = 2;
    float *partials = sc->jac_partials;
    unsigned *sync = sc->jac_sync;
    void *args[] = {(void *)&p, (void *)&partials, (void *)&sync};
    const size_t smem = (size_t)n * 4;
    KAAS_CUDA(cudaFuncSetAttribute((const void *)k_jacobi_rows<false, false, true>,
                                   cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    KAAS_CUDA(cudaLaunchKernel((const void *)k_jacobi_rows<false, false, true>, dim3(blocks),
                               dim3(rows_threads(dev, cov)), args, smem, s));
    count_launch();
    return 0;
  }
  int kc = pick_kc(n);
  if (!aligned16(A) || !aligned16(x_in)) kc = 0;
  if (kc < 0) kc = 0;
#define JAC_LAUNCH(K)                                                                     \
  k_jacobi_sweep<K><<<blocks, kJacThreads, 0, s>>>(n, (int)cov, A, b, x_in, x_out, resid, \
                                                   sc->jac_partials, sc->jac_sync)
  switch (kc) {
    case 1: JAC_LAUNCH(1); break;
    case 2: JAC_LAUNCH(2); break;
    case 4: JAC_LAUNCH(4); break;
    default: JAC_LAUNCH(0); break;
  }
#undef JAC_LAUNCH
  count_launch();
  KAAS_CUDA(cudaGetLastError());
  return 0;
}

struct JacobiMemo {
  ChainParams p;
  const void *fn;
  int blocks;
  size_t smem;
  bool wb_ok;  // the memoised kernel writes back the last sweep (k_jacobi_tmem)
};

void free_jacobi_memo(StreamScratch *sc) {
  delete static_cast<JacobiMemo *>(sc->jac_memo);
  sc->jac_memo = nullptr;
  sc->jac_memo_key = 0;
}

// grid barriers a launch of p passes (the kernels' grid_sync_mono calls):
// every sweep for the untagged kernels, sweeps with an observable residual
// for the tagged ones
static unsigned chain_barriers(const ChainParams &p) {
  if (!p.tagged) return (unsigned)p.sweeps;
  unsigned c = 0;
  for (int t = 0; t < p.sweeps; ++t) c += (p.idx[t][2] & 0x80) ? 1u : 0u;
  return c;
}

// claim this launch's range of the stream's monotonic barrier counter
static void claim_barriers(StreamScratch *sc, ChainParams &p, int blocks) {
  p.sync_base = sc->jac_sync_base;
  sc->jac_sync_base += chain_barriers(p) * (unsigned)blocks;
}

// the per-launch part of a tagged on-chip chain launch: fresh tags, the
// barrier counter range, cooperative launch
static int launch_tagged_chain(cudaStream_t s, StreamScratch *sc, ChainParams &p, const void *fn,
                               int blocks, size_t smem) {
  if (sc->jac_tag > 0x7fffffffu - (unsigned)p.sweeps - 2u) {  // tag space wrap: start over
    KAAS_CUDA(cudaMemsetAsync(sc->jac_xt, 0, 2 * kJacTaggedMaxN * sizeof(unsigned long long), s));
    sc->jac_tag = 1;
  }
  p.tag0 = sc->jac_tag;
  sc->jac_tag += (unsigned)p.sweeps + 1u;
  float *partials = sc->jac_partials;
  unsigned *sync = sc->jac_sync;
  claim_barriers(sc, p, blocks);
  void *cargs[] = {(void *)&p, (void *)&partials, (void *)&sync};
  KAAS_CUDA(cudaLaunchCooperativeKernel(fn, dim3(blocks), dim3(kColT), cargs, smem, s));
  count_launch();
  return 0;
}

int launch_jacobi_memo(cudaStream_t s, int dev, StreamScratch *sc, float *wb_x, float *wb_r) {
  (void)dev;
  auto *m = static_cast<JacobiMemo *>(sc->jac_memo);
  if (!m) return 1;
  if ((wb_x || wb_r) && !m->wb_ok) return 1;  // its kernel cannot write back: the full path copies
  m->p.wb_x = wb_x;
  m->p.wb_r = wb_r;
  return launch_tagged_chain(s, sc, m->p, m->fn, m->blocks, m->smem);
}

int launch_jacobi_chain(cudaStream_t s, int dev, const JacobiChain &c, StreamScratch *sc,
                        uint64_t memo_key) {
  sc->jac_memo_key = 0;  // rebuilt below when this launch can be memoised
  int kc = pick_kc(c.n);
  if (kc < 0) kc = 0;
  if (!aligned16(c.A)) kc = 0;
  for (int t = 0; t < c.sweeps && kc; ++t)
    if (!aligned16(c.x_in[t])) kc = 0;
  bool use_rows = use_rows_kernel(c.n) && aligned16(c.A);
  for (int t = 0; t < c.sweeps && use_rows; ++t)
    if (!aligned16(c.x_in[t])) use_rows = false;
  const char *xd = KAAS_DEV_ENV("KAAS_JACOBI_XDIRECT");  // dev A/B (default on)
  const bool xdirect = !(xd && xd[0] == '0');
  const bool pf = rows_prefetch();
  const void *rfn = xdirect ? (pf ? (const void *)k_jacobi_rows<true, true, true>
                                  : (const void *)k_jacobi_rows<true, false, true>)
                            : (pf ? (const void *)k_jacobi_rows<true, true>
                                  : (const void *)k_jacobi_rows<true, false>);
  const void *fn = kc == 1 ? (const void *)k_jacobi_chain<1>
                 : kc == 2 ? (const void *)k_jacobi_chain<2>
                 : kc == 4 ? (const void *)k_jacobi_chain<4>
                           : (const void *)k_jacobi_chain<0>;
  // Keep A resident in L2 across sweeps when it fits comfortably.
  const bool keep = (double)c.n * c.n * 4.0 <= 0.75 * (double)device_props(dev).l2_bytes;
  int done = 0;
  while (done < c.sweeps) {
    static thread_local ChainParams p;  // ~6 KB: keep it off the stack
    p.A = c.A;
    p.b = c.b;
    p.n = c.n;
    p.cov = (int)c.cov;
    p.keep_l2 = keep ? 1 : 0;
    int np = 0, cnt = 0;
    auto slot = [&](const float *q) -> int {
      for (int t = 0; t < np; ++t)
        if (p.ptrs[t] == q) return t;
      if (np == kChainMaxPtrs) return -1;
      p.ptrs[np] = const_cast<float *>(q);
      return np++;
    };
    for (; done + cnt < c.sweeps && cnt < kChainMaxSweeps; ++cnt) {
      const int t = done + cnt;
      const int a = slot(c.x_in[t]), o = slot(c.x_out[t]), r = slot(c.resid[t]);
      if (a < 0 || o < 0 || r < 0) break;
      p.idx[cnt][0] = (unsigned char)a;
      p.idx[cnt][1] = (unsigned char)o;
      // residual slots are never read inside a run, so only the last write to
      // each slot is observable: flag it (0x80) and skip the others' finish
      bool last_writer = true;
      for (int u = t + 1; u < c.sweeps && last_writer; ++u) last_writer = c.resid[u] != c.resid[t];
      p.idx[cnt][2] = (unsigned char)(r | (last_writer ? 0x80 : 0));
    }
    if (cnt == 0) return fail(KAAS_E_INVALID, "jacobi chain: too many distinct buffers");
    p.sweeps = cnt;
    int blocks = device_props(dev).sm_count;
    if ((uint64_t)blocks > c.cov) blocks = c.cov > 0 ? (int)c.cov : 1;
    float *partials = sc->jac_partials;
    unsigned *sync = sc->jac_sync;
    p.xt = sc->jac_xt;
    p.tag0 = 0;
    p.tagged = 0;
    p.zero = 0;
    p.trace = nullptr;
    p.wb_x = p.wb_r = nullptr;
    if (use_rows && use_cols_kernel(dev, c.n, c.cov, blocks)) {
      // a pure ping-pong run (each sweep reads the previous one's output, no
      // in-place sweep) publishes x through tags instead of grid barriers
      // (every row must be produced each sweep: full coverage)
      bool chained = sc->jac_xt != nullptr && c.n <= kJacTaggedMaxN && c.cov >= (uint64_t)c.n;
      if (const char *e = KAAS_DEV_ENV("KAAS_JACOBI_TAGS"))  // dev A/B: 0 = grid barrier per sweep
        chained = chained && e[0] != '0';
      for (int t = done; t < done + cnt && chained; ++t)
        chained = c.x_in[t] != c.x_out[t] && (t == done || c.x_in[t] == c.x_out[t - 1]);
      if (chained) {
        p.tagged = 1;
#ifdef KAAS_DEV
        if (KAAS_DEV_ENV("KAAS_JACOBI_NOWAIT")) p.tagged = 3;  // dev: compute-only timing
#endif
        static unsigned *trace_buf = nullptr;  // dev: KAAS_JACOBI_TRACE=1 (tools/jtrace.py)
        if (KAAS_DEV_ENV("KAAS_JACOBI_TRACE") && !trace_buf) cudaMalloc((void **)&trace_buf, (kTraceWarpOff + 32 * 148 * 8) * 4);
        p.trace = KAAS_DEV_ENV("KAAS_JACOBI_TRACE") ? trace_buf : nullptr;
        jacobi_trace_buffer() = p.trace;
        const char *pe = KAAS_DEV_ENV("KAAS_JACOBI_POLL_NS");  // dev A/B
        p.poll_ns = pe ? atoi(pe) : 0;
      }
      const bool tm = use_tmem_kernel();
      const TmVariant &tv = tm_variant();
      const void *cfn = tm ? tv.fn : (const void *)k_jacobi_cols;
      const size_t csmem = tm ? tv.smem : kColSmem;
      static std::atomic<uint64_t> attr_done[2];  // per kernel, bit per device (dev < 64)
#ifdef KAAS_DEV
      KAAS_CUDA(cudaFuncSetAttribute(cfn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)csmem));
#endif
      if (!(attr_done[tm].load(std::memory_order_relaxed) >> (dev & 63) & 1)) {
        KAAS_CUDA(cudaFuncSetAttribute(cfn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)csmem));
        attr_done[tm].fetch_or(1ull << (dev & 63));
      }
      if (p.tagged) {
        // only the TMEM kernel writes the last sweep back to host memory
        const bool wb = tm && done + cnt == c.sweeps && (c.wb_x || c.wb_r);
        p.wb_x = wb ? c.wb_x : nullptr;
        p.wb_r = wb ? c.wb_r : nullptr;
        int rc = launch_tagged_chain(s, sc, p, cfn, blocks, csmem);
        if (rc) return rc;
        if (wb && c.wb_done) *c.wb_done = true;
        if (memo_key && done == 0 && cnt == c.sweeps) {  // the whole run in one launch
          auto *m = static_cast<JacobiMemo *>(sc->jac_memo);
          if (!m) sc->jac_memo = m = new JacobiMemo();
          m->p = p;
          m->fn = cfn;
          m->blocks = blocks;
          m->smem = csmem;
          m->wb_ok = tm;
          sc->jac_memo_key = memo_key;
        }
        done += cnt;
        continue;
      }
      claim_barriers(sc, p, blocks);
      void *cargs[] = {(void *)&p, (void *)&partials, (void *)&sync};
      KAAS_CUDA(cudaLaunchCooperativeKernel(cfn, dim3(blocks), dim3(kColT), cargs, csmem, s));
    } else if (use_rows) {
      KAAS_CUDA(cudaFuncSetAttribute(rfn, cudaFuncAttributeMaxDynamicSharedMemorySize, c.n * 4));
      claim_barriers(sc, p, blocks);
      void *rargs[] = {(void *)&p, (void *)&partials, (void *)&sync};
      KAAS_CUDA(cudaLaunchCooperativeKernel(rfn, dim3(blocks),
                                            dim3(rows_threads(dev, c.cov)), rargs, (size_t)c.n * 4, s));
    } else {
      void *args[] = {(void *)&p, (void *)&partials, (void *)&sync};
      KAAS_CUDA(cudaLaunchCooperativeKernel(fn, dim3(blocks), dim3(kJacThreads), args, 0, s));
    }
    count_launch();
    done += cnt;
  }
  return 0;
}

}  // namespace kaas

#ifdef KAAS_DEV
// dev build only (not in include/kaas_b200.h): copy the last traced Jacobi
// chain's per-CTA timestamps (KAAS_JACOBI_TRACE=1) to the host; tools/jtrace.py
extern "C" int kaas_dev_jacobi_trace(void *host, unsigned long bytes) {
  unsigned *buf = kaas::jacobi_trace_buffer();
  if (!buf) return 1;
  const unsigned long cap = (kaas::kTraceWarpOff + 32ul * 148 * 8) * 4;
  if (bytes > cap) bytes = cap;
  return cudaMemcpy(host, buf, bytes, cudaMemcpyDeviceToHost) == cudaSuccess ? 0 : 2;
}
#endif
