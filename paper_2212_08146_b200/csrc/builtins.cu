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
#include <cuda.h>

#include "kaas_internal.cuh"
#include "mm_tile.cuh"

#include <atomic>

namespace kaas {
// 2-D f32 TMA descriptor (cgemm.cu): rows x ld, box box_rows x box_k,
// swizzle_bytes 0 / 64 / 128
int encode_map_f32(CUtensorMap *map, const float *base, uint64_t rows, uint64_t ld, uint32_t box_rows,
                   uint32_t box_k, int swizzle_bytes);
namespace {

constexpr int kEltThreads = 256;

inline int elt_blocks(int dev, uint64_t work) {
  uint64_t want = (work + kEltThreads - 1) / kEltThreads;
  uint64_t cap = (uint64_t)device_props(dev).sm_count * 8;
  if (want < 1) want = 1;
  return (int)(want < cap ? want : cap);
}

inline bool aligned16(const void *p) { return ((uintptr_t)p & 15u) == 0; }

// Programmatic dependent launch: a request's builtin kernels run back to back
// on one stream (ResNet chain: ~100 of them), so each is launched with
// programmatic stream serialization and may be scheduled while its
// predecessor drains.  Every such kernel waits (griddepcontrol.wait: the
// previous grid has completed and its writes are visible) before touching
// memory, and lets its own dependents launch once its main work is issued.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_release() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

template <typename... KArgs, typename... Args>
cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                       Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kernel, (KArgs)args...);
}

// Exact aliasing (out == x or out == y) is safe: each element is read and
// then written by the same thread, so no __restrict__ on these pointers.
template <int kOp>  // 0 = add, 1 = saxpy, 2 = fill
__global__ void __launch_bounds__(kEltThreads)
k_elementwise_v4(uint64_t n4, float a, const float4 *x, const float4 *y, float4 *out) {
  pdl_wait();
  pdl_release();
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
  pdl_wait();
  pdl_release();
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
    KAAS_CUDA(launch_pdl(k_elementwise_v4<kOp>, dim3(elt_blocks(dev, n4)), dim3(kEltThreads), 0, s,
                         n4, a, (const float4 *)x, (const float4 *)y, (float4 *)out));
    count_launch();
    done = n4 * 4;
  }
  if (done < cov) {
    KAAS_CUDA(launch_pdl(k_elementwise_scalar<kOp>, dim3(elt_blocks(dev, cov - done)), dim3(kEltThreads), 0,
                         s, done, cov, a, x, y, out));
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

// 1-D grid, column tiles fastest (the 2-D raster order without grid.y's
// 65535 limit on n); the tile body is mm_tile (mm_tile.cuh)
template <int TY, int TX, int TM, int TN, int S, int BK, bool AV, bool BT>
__global__ void __launch_bounds__(TY *TX)
k_matmul(int n, int m, int k, uint64_t cov, const float *__restrict__ a,
         const float *__restrict__ b, float *__restrict__ out) {
  extern __shared__ __align__(16) float mm_smem[];
  constexpr int BM = TY * TM, BN = TX * TN;
  const unsigned gx = (unsigned)((m + BN - 1) / BN);
  const int bm = (int)(blockIdx.x / gx) * BM, bn = (int)(blockIdx.x % gx) * BN;
  mm_tile<TY, TX, TM, TN, S, BK, AV, BT, true>(n, m, k, cov, a, b, out, bm, bn, mm_smem);
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

#ifdef KAAS_DEV
// ---- long-K, few-cell layers: TMA-fed chain kernel (dev build only) --------
//
// Measured on B200 (round 2, profiles/r02/probes/matmul_lk.txt): correct
// (bit-exact) but SLOWER than the cp.async-ring kernel on every ResNet shape
// it targets (49x512x4608: 60-99 us vs 48-53; fc 1x1000x2048: 29-37 vs 21),
// and still ~26 cycles per k in a compute-only run (no copies, no waits)
// against the 4.1 cycles per step a lone FMUL+FADD chain measures
// (tools/chainlat.cu).  Not understood yet; kept as the A/B starting point
// (KAAS_MATMUL_LK=1 in a dev build).
//
// Per cell the serial FADD chain is the floor (k dependent adds, 4 cycles
// each); these layers have only 1k-100k cells, so the kernel keeps every
// chain fed with as few instructions per k as possible:
//   * operands are staged by 2-D TMA (one cp.async.bulk.tensor per operand
//     tile per 32-k stage: A rows and the transposed B are k-contiguous) into
//     an S-deep ring guarded by mbarriers -- no per-thread copy work, no
//     __syncthreads; one lane issues the copies, every warp releases a stage
//     with one elected arrive;
//   * 128-byte swizzled tiles, so a warp's LDS.128 of different rows at the
//     same k hit different banks;
//   * each thread owns TN cells (one row, TN columns) and holds a whole stage
//     of its operands in registers: the next stage's first half is loaded
//     while the current stage's second half is in the chain, and vice versa.
// Products and their order are exactly the reference's (k ascending, one f32
// accumulator per cell, multiply and add rounded separately); a partial last
// stage adds only its valid k.
__device__ __forceinline__ uint32_t smem_addr(const void *p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mb_init(uint64_t *bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count));
}
__device__ __forceinline__ void mb_expect(uint64_t *bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mb_arrive(uint64_t *bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_addr(bar)) : "memory");
}
__device__ __forceinline__ void mb_wait(uint64_t *bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n"
      "LAB_WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@!P1 bra LAB_WAIT_%=;\n\t}" ::"r"(smem_addr(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma2d(const CUtensorMap *map, uint64_t *bar, void *dst, int k0, int row0) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], "
      "[%2];" ::"r"(smem_addr(dst)),
      "l"(map), "r"(smem_addr(bar)), "r"(k0), "r"(row0)
      : "memory");
}
// LDS.128 of 16-byte chunk c (0..7) of 128-byte row r in a SWIZZLE_128B tile
__device__ __forceinline__ float4 lds_sw(const uint8_t *tile, int r, int c) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "r"(smem_addr(tile + r * 128 + ((c ^ (r & 7)) << 4))));
  return v;
}

constexpr int kLkBK = 32;  // k per stage: one 128-byte swizzle row per tile row
template <int TY, int TX, int TN>
struct LkShape {
  static constexpr int BN = TX * TN;
  static constexpr int A_BYTES = ((TY * 128 + 1023) / 1024) * 1024;  // boxes 1024-aligned (swizzle atom)
  static constexpr int B_BYTES = ((BN * 128 + 1023) / 1024) * 1024;
  static constexpr int STAGE = A_BYTES + B_BYTES;
};
template <int TY, int TX, int TN, int S>
constexpr int lk_smem_bytes() {
  return S * LkShape<TY, TX, TN>::STAGE + 2 * S * 8 + 1024;
}

template <int TY, int TX, int TN, int S>
__global__ void __launch_bounds__(TY *TX)
k_matmul_lk(const __grid_constant__ CUtensorMap map_a, const __grid_constant__ CUtensorMap map_b, int n,
            int m, int k, uint64_t cov, float *__restrict__ out, int dev_flags) {
  using L = LkShape<TY, TX, TN>;
  constexpr int T = TY * TX, NW = T / 32, G = kLkBK / 4;
  static_assert(T % 32 == 0 && (S & (S - 1)) == 0, "whole warps, power-of-two ring");
  extern __shared__ uint8_t lk_raw[];
  uint8_t *ring = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(lk_raw) + 1023) & ~uintptr_t(1023));
  uint64_t *full = reinterpret_cast<uint64_t *>(ring + S * L::STAGE);
  uint64_t *empty = full + S;
  const int tid = threadIdx.x, lane = tid & 31;
  const int tx = tid % TX, ty = tid / TX;
  const unsigned gx = (unsigned)((m + L::BN - 1) / L::BN);
  const int bm = (int)(blockIdx.x / gx) * TY, bn = (int)(blockIdx.x % gx) * L::BN;
  const int nk = (k + kLkBK - 1) / kLkBK;
  const int nfull = k / kLkBK;  // stages with all 32 k valid
  const bool producer = tid == 0;

  if (producer) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(&map_a) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&map_b) : "memory");
    for (int i = 0; i < S; ++i) {
      mb_init(&full[i], 1);
      mb_init(&empty[i], NW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  pdl_wait();  // the operands may be the previous kernel's output
  auto produce = [&](int t) {  // one thread; boxes past the matrix edges are zero-filled
    const int st = t & (S - 1);
    if (t >= S) mb_wait(&empty[st], ((t / S) - 1) & 1);
    mb_expect(&full[st], (uint32_t)(TY * 128 + L::BN * 128));
    uint8_t *base = ring + st * L::STAGE;
    tma2d(&map_a, &full[st], base, t * kLkBK, bm);
    tma2d(&map_b, &full[st], base + L::A_BYTES, t * kLkBK, bn);
  };
  if (producer && !(dev_flags & 2))
    for (int t = 0; t < S - 1 && t < nk; ++t) produce(t);

  // shared-memory byte offsets of this thread's 16-byte chunks (128B swizzle)
  uint32_t oa[G], ob[TN][G];
#pragma unroll
  for (int c = 0; c < G; ++c) {
    oa[c] = smem_addr(ring) + ty * 128 + ((c ^ (ty & 7)) << 4);
#pragma unroll
    for (int j = 0; j < TN; ++j) {
      const int r = tx + TX * j;
      ob[j][c] = smem_addr(ring) + L::A_BYTES + r * 128 + ((c ^ (r & 7)) << 4);
    }
  }
  auto lds = [](uint32_t addr) {
    float4 v;
    asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(addr));
    return v;
  };
  float acc[TN];
#pragma unroll
  for (int j = 0; j < TN; ++j) acc[j] = 0.0f;
  float4 ra[G], rb[TN][G];
  auto load = [&](int t, int g0) {
    const uint32_t sb = (uint32_t)((t & (S - 1)) * L::STAGE);
#pragma unroll
    for (int g = g0; g < g0 + G / 2; ++g) {
      ra[g] = lds(oa[g] + sb);
#pragma unroll
      for (int j = 0; j < TN; ++j) rb[j][g] = lds(ob[j][g] + sb);
    }
  };
  auto step = [&](int g) {
#pragma unroll
    for (int j = 0; j < TN; ++j) {
      acc[j] = __fadd_rn(acc[j], __fmul_rn(ra[g].x, rb[j][g].x));
      acc[j] = __fadd_rn(acc[j], __fmul_rn(ra[g].y, rb[j][g].y));
      acc[j] = __fadd_rn(acc[j], __fmul_rn(ra[g].z, rb[j][g].z));
      acc[j] = __fadd_rn(acc[j], __fmul_rn(ra[g].w, rb[j][g].w));
    }
  };
  if (!(dev_flags & 1)) mb_wait(&full[0], 0);
  load(0, 0);
  load(0, G / 2);
  // full stages: stage t's second half is in the chain while stage t+1's
  // first half loads, and the other way round
#pragma unroll 1
  for (int t = 0; t < nfull; ++t) {
    if (producer && t + S - 1 < nk && !(dev_flags & 2)) produce(t + S - 1);
#pragma unroll
    for (int g = 0; g < G / 2; ++g) step(g);
    const bool more = t + 1 < nk;
    if (more) {
      if (!(dev_flags & 1)) mb_wait(&full[(t + 1) & (S - 1)], ((t + 1) / S) & 1);
      load(t + 1, 0);
    }
#pragma unroll
    for (int g = G / 2; g < G; ++g) step(g);
    __syncwarp();
    if (lane == 0) mb_arrive(&empty[t & (S - 1)]);  // this warp is done reading stage t
    if (more) load(t + 1, G / 2);
  }
  if (nfull < nk) {  // the partial last stage: only its valid 4-k groups
    const int gn = (k - nfull * kLkBK) >> 2;  // k % 4 == 0
#pragma unroll
    for (int g = 0; g < G; ++g)
      if (g < gn) step(g);
  }
  pdl_release();
  const int r = bm + ty;
  if (r < n) {
#pragma unroll
    for (int j = 0; j < TN; ++j) {
      const int c = bn + tx + TX * j;
      if (c >= m) continue;
      const uint64_t gi = (uint64_t)r * m + c;
      if (gi < cov) out[gi] = acc[j];
    }
  }
}

template <int TY, int TX, int TN>
int lk_launch(int dev, cudaStream_t s, uint64_t n, uint64_t m, uint64_t k, uint64_t cov, const float *a,
              const float *bt, float *out) {
  constexpr int S = LkShape<TY, TX, TN>::STAGE <= 3072 ? 32 : 16;  // >= 512 k in flight
  constexpr int SM = lk_smem_bytes<TY, TX, TN, S>();
  static std::atomic<uint64_t> attr_done{0};
  if (!(attr_done.load(std::memory_order_relaxed) >> (dev & 63) & 1)) {
    KAAS_CUDA(cudaFuncSetAttribute(k_matmul_lk<TY, TX, TN, S>, cudaFuncAttributeMaxDynamicSharedMemorySize, SM));
    attr_done.fetch_or(1ull << (dev & 63));
  }
  CUtensorMap ma, mb;
  int rc = encode_map_f32(&ma, a, n, k, TY, kLkBK, 128);
  if (!rc) rc = encode_map_f32(&mb, bt, m, k, TX * TN, kLkBK, 128);
  if (rc) return rc;
  const uint64_t grid = ((n + TY - 1) / TY) * ((m + TX * TN - 1) / (TX * TN));
  int dev_flags = 0;  // dev A/B: 1 = no data waits, 3 = no copies either (wrong results)
  if (const char *e = KAAS_DEV_ENV("KAAS_LK_FLAGS")) dev_flags = atoi(e);
  KAAS_CUDA(launch_pdl(k_matmul_lk<TY, TX, TN, S>, dim3((unsigned)grid), dim3(TY * TX), SM, s, ma, mb, (int)n,
                       (int)m, (int)k, cov, out, dev_flags));
  return 0;
}

#endif  // KAAS_DEV

// B [k][m] -> Bt [m][k] (32 x 32 smem tiles).  A 1-D grid walks the tiles,
// so no extent hits the 65535 grid.y limit (k up to 2^31 - 1).
__global__ void k_transpose_b(int k, int m, const float *__restrict__ b, float *__restrict__ bt) {
  __shared__ float t[32][33];
  const uint64_t tiles_m = ((uint64_t)m + 31) / 32, tiles = tiles_m * (((uint64_t)k + 31) / 32);
  for (uint64_t tile = blockIdx.x; tile < tiles; tile += gridDim.x) {
    const int c0 = (int)(tile % tiles_m) * 32, r0 = (int)(tile / tiles_m) * 32;
    for (int i = threadIdx.y; i < 32; i += blockDim.y) {
      const int r = r0 + i, c = c0 + threadIdx.x;
      if (r < k && c < m) t[i][threadIdx.x] = b[(size_t)r * m + c];
    }
    __syncthreads();
    for (int i = threadIdx.y; i < 32; i += blockDim.y) {
      const int c = c0 + i, r = r0 + threadIdx.x;
      if (r < k && c < m) bt[(size_t)c * k + r] = t[threadIdx.x][i];
    }
    __syncthreads();
  }
}

template <int TY, int TX, int TM, int TN, int S, int BK>
int mm_launch_sb(int dev, cudaStream_t s, dim3 grid, const float *bt, bool a_vec, uint64_t n, uint64_t m,
                 uint64_t k, uint64_t cov, const float *a, const float *b, float *out) {
  constexpr int SM = mm_smem_bytes<TY, TX, TM, TN, S, BK>();
  static_assert(SM <= 227 * 1024, "matmul ring exceeds shared memory");
  static std::atomic<uint64_t> attr_done{0};  // per device (dev < 64)
  if (!(attr_done.load(std::memory_order_relaxed) >> (dev & 63) & 1)) {
    KAAS_CUDA(cudaFuncSetAttribute(k_matmul<TY, TX, TM, TN, S, BK, true, true>,
                                   cudaFuncAttributeMaxDynamicSharedMemorySize, SM));
    KAAS_CUDA(cudaFuncSetAttribute(k_matmul<TY, TX, TM, TN, S, BK, true, false>,
                                   cudaFuncAttributeMaxDynamicSharedMemorySize, SM));
    KAAS_CUDA(cudaFuncSetAttribute(k_matmul<TY, TX, TM, TN, S, BK, false, false>,
                                   cudaFuncAttributeMaxDynamicSharedMemorySize, SM));
    attr_done.fetch_or(1ull << (dev & 63));
  }
  KAAS_CUDA(launch_pdl(bt ? k_matmul<TY, TX, TM, TN, S, BK, true, true>
                          : a_vec ? k_matmul<TY, TX, TM, TN, S, BK, true, false>
                                  : k_matmul<TY, TX, TM, TN, S, BK, false, false>,
                       grid, dim3(TY * TX), SM, s, (int)n, (int)m, (int)k, cov, a, bt ? bt : b, out));
  return 0;
}

// Ring depth: 4 x 32-k chunks for the big tiles; 3 x 64-k for the small ones,
// whose CTAs are small and many -- a shallower ring keeps more of them
// resident (measured over the ResNet-50 layers: 1364 -> 1207 us vs 6-8 stages
// for every layer).  For the long-K layers alone, a deeper ring (4, 6 or 8
// stages) and 128-k chunks both measured flat or slower: ~1.5 warps per
// scheduler stall on shared-memory latency and the FADD chain (ncu: short
// scoreboard 1.14 + wait 1.24 cycles per issue), not on L2 or chunk overhead.
template <int TY, int TX, int TM, int TN>
int mm_launch(int dev, cudaStream_t s, dim3 grid, const float *bt, bool a_vec, uint64_t n, uint64_t m,
              uint64_t k, uint64_t cov, const float *a, const float *b, float *out) {
  if constexpr (TM * TN >= 8) {
    return mm_launch_sb<TY, TX, TM, TN, 4, 32>(dev, s, grid, bt, a_vec, n, m, k, cov, a, b, out);
  } else {
    return mm_launch_sb<TY, TX, TM, TN, 3, 64>(dev, s, grid, bt, a_vec, n, m, k, cov, a, b, out);
  }
}

#ifdef KAAS_DEV
// dev: KAAS_MATMUL_LK=1 routes eligible layers to the chain kernel
bool lk_eligible(int dev, uint64_t n, uint64_t m, uint64_t k) {
  (void)dev;
  (void)n;
  (void)m;
  const char *e = KAAS_DEV_ENV("KAAS_MATMUL_LK");
  return e && e[0] == '1' && k >= 256;
}

// 1 x 32 tiles for single-row outputs (fc), otherwise the largest tile that
// still gives every SM at least ~4 warps
int lk_pick(int dev, uint64_t n, uint64_t m) {
  if (n <= 2) return 0;
  const uint64_t sms = (uint64_t)device_props(dev).sm_count;
  const uint64_t warps = n * m / 32;
  if (warps >= 16 * sms) return 3;  // two cells per thread
  if (n >= 8) return 2;
  return 1;
}

#endif

int launch_matmul(cudaStream_t s, int dev, uint64_t n, uint64_t m, uint64_t k, uint64_t cov,
                  const float *a, const float *b, float *out, StreamScratch *sc, const float *bt_prep,
                  bool bt_ready) {
  if (n > 0x7fffffffu || m > 0x7fffffffu || k > 0x7fffffffu)
    return fail(KAAS_E_INVALID, "matmul extent exceeds i32");
  // B transposed (16-byte B copies): from the executor's prepared-operand
  // cache when it has one for this weight, else built into per-stream
  // scratch for this launch (one extra pass over B)
  const char *be = KAAS_DEV_ENV("KAAS_MATMUL_BT");  // dev A/B: 0 = B as given
  const bool use_bt = !(be && be[0] == '0') && k > 0 && k % 4 == 0 && aligned16(a);
  auto transpose_into = [&](float *dst) -> int {
    const uint64_t tiles = ((m + 31) / 32) * ((k + 31) / 32);
    const uint64_t cap = (uint64_t)device_props(dev).sm_count * 16;
    KAAS_CUDA(launch_pdl(k_transpose_b, dim3((unsigned)(tiles < cap ? tiles : cap)),
                         dim3(32, 8), 0, s, (int)k, (int)m, b, dst));
    count_launch();
    return 0;
  };
  // a prepared buffer the executor asked to fill is always filled (it will
  // be trusted as Bt by later launches), whether or not this one uses it
  if (bt_prep && !bt_ready && k > 0 && m > 0) {
    int rc = transpose_into(const_cast<float *>(bt_prep));
    if (rc) return rc;
    bt_ready = true;
  }
  if (n == 0 || m == 0 || cov == 0) return 0;
  const float *bt = nullptr;
  if (use_bt) {
    if (bt_prep) {
      bt = bt_prep;
    } else {
      int rc = ensure_matmul_scratch(sc, s, (size_t)m * k * 4);
      if (!rc) rc = transpose_into((float *)sc->mm_buf);
      if (rc) return rc;
      bt = (const float *)sc->mm_buf;
    }
  }
#ifdef KAAS_DEV
  // Long-K, few-cell layers: the TMA-fed chain kernel (operands k-contiguous
  // and 16-byte aligned: A rows and the transposed B)
  if (bt && (k % 4) == 0 && aligned16(a) && aligned16(bt) && k >= 256 && lk_eligible(dev, n, m, k)) {
    int which = lk_pick(dev, n, m);
    if (const char *ce = KAAS_DEV_ENV("KAAS_LK_CFG")) which = atoi(ce);
    int rc = 0;
    switch (which) {
      case 0: rc = lk_launch<1, 32, 1>(dev, s, n, m, k, cov, a, bt, out); break;
      case 1: rc = lk_launch<4, 16, 1>(dev, s, n, m, k, cov, a, bt, out); break;
      case 2: rc = lk_launch<8, 8, 1>(dev, s, n, m, k, cov, a, bt, out); break;
      case 4: rc = lk_launch<8, 16, 1>(dev, s, n, m, k, cov, a, bt, out); break;
      case 5: rc = lk_launch<16, 8, 1>(dev, s, n, m, k, cov, a, bt, out); break;
      case 6: rc = lk_launch<8, 16, 2>(dev, s, n, m, k, cov, a, bt, out); break;
      case 7: rc = lk_launch<1, 128, 1>(dev, s, n, m, k, cov, a, bt, out); break;
      default: rc = lk_launch<8, 8, 2>(dev, s, n, m, k, cov, a, bt, out); break;
    }
    if (rc) return rc;
    count_launch();
    KAAS_CUDA(cudaGetLastError());
    return 0;
  }
#endif
  // Cost model: a config's rate ~ (warps it can field, up to 2 per
  // scheduler) x (useful fraction of its tiles) / (instructions per MAC:
  // 2 FP + (TM + TN) / 4 LDS.128 per k + ~0.5 copy/loop overhead, per cell).
  struct Cfg { int ty, tx, tm, tn; };
  static const Cfg cfgs[] = {{16, 16, 4, 4}, {16, 16, 2, 4}, {16, 16, 4, 2}, {16, 16, 2, 2},
                             {8, 16, 2, 2},  {16, 8, 2, 2},  {8, 8, 2, 2},   {8, 8, 1, 2},
                             {8, 8, 2, 1},   {8, 8, 1, 1}};
  const int sms = device_props(dev).sm_count;
  const double want_warps = 8.0 * sms;
  int best = 0;
  double best_score = -1.0;
  for (int i = 0; i < (int)(sizeof(cfgs) / sizeof(cfgs[0])); ++i) {
    const Cfg &c = cfgs[i];
    const uint64_t tbm = (uint64_t)c.ty * c.tm, tbn = (uint64_t)c.tx * c.tn;
    const uint64_t gy = (n + tbm - 1) / tbm, gx = (m + tbn - 1) / tbn;
    if (gy * gx > 0x7fffffffull) continue;
    const double warps = (double)(gy * gx) * (c.ty * c.tx / 32.0);
    const double useful = (double)(n * m) / (double)(gy * tbm * gx * tbn);
    const double cells = c.tm * c.tn;
    const double ipm = (2.0 * cells + (c.tm + c.tn) / 4.0 + 0.5) / cells;
    const double score = (warps < want_warps ? warps : want_warps) * useful / ipm;
    if (score > best_score * 1.02) {  // ties -> the larger tile (earlier)
      best_score = score;
      best = i;
    }
  }
  if (best_score < 0) return fail(KAAS_E_INVALID, "matmul: too many output tiles for one grid");
  if (const char *fe = KAAS_DEV_ENV("KAAS_MATMUL_CFG")) {  // dev: force a config (tools/mm_cfg_sweep.py)
    const int f = atoi(fe);
    const Cfg &c = cfgs[f < 0 ? 0 : f % (int)(sizeof(cfgs) / sizeof(cfgs[0]))];
    (void)c;
    best = f % (int)(sizeof(cfgs) / sizeof(cfgs[0]));
  }
  const Cfg &c = cfgs[best];
  const unsigned gy = (unsigned)((n + c.ty * c.tm - 1) / (c.ty * c.tm));
  const unsigned gx = (unsigned)((m + c.tx * c.tn - 1) / (c.tx * c.tn));
  dim3 grid(gx * gy);
  const int a_vec = (k % 4 == 0) && aligned16(a);
  int rc = 0;
  switch (best) {
    case 0: rc = mm_launch<16, 16, 4, 4>(dev, s, grid, bt, a_vec, n, m, k, cov, a, b, out); break;
    case 1: rc = mm_launch<16, 16, 2, 4>(dev, s, grid, bt, a_vec, n, m, k, cov, a, b, out); break;
    case 2: rc = mm_launch<16, 16, 4, 2>(dev, s, grid, bt, a_vec, n, m, k, cov, a, b, out); break;
    case 3: rc = mm_launch<16, 16, 2, 2>(dev, s, grid, bt, a_vec, n, m, k, cov, a, b, out); break;
    case 4: rc = mm_launch<8, 16, 2, 2>(dev, s, grid, bt, a_vec, n, m, k, cov, a, b, out); break;
    case 5: rc = mm_launch<16, 8, 2, 2>(dev, s, grid, bt, a_vec, n, m, k, cov, a, b, out); break;
    case 6: rc = mm_launch<8, 8, 2, 2>(dev, s, grid, bt, a_vec, n, m, k, cov, a, b, out); break;
    case 7: rc = mm_launch<8, 8, 1, 2>(dev, s, grid, bt, a_vec, n, m, k, cov, a, b, out); break;
    case 8: rc = mm_launch<8, 8, 2, 1>(dev, s, grid, bt, a_vec, n, m, k, cov, a, b, out); break;
    default: rc = mm_launch<8, 8, 1, 1>(dev, s, grid, bt, a_vec, n, m, k, cov, a, b, out); break;
  }
  if (rc) return rc;
  count_launch();
  KAAS_CUDA(cudaGetLastError());
  return 0;
}

}  // namespace kaas
