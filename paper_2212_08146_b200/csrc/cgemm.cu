// Complex64 GEMM on the 5th-gen tensor cores (tcgen05, TMEM, TMA) -- the
// `cgemm` KaaS library kernel (new; CPU restatement: oracle/kernels.py cgemm).
//
//   C[n x m] = A[n x k] . B[k x m], complex64 interleaved (re, im), row-major.
//
// 4M decomposition as ONE real GEMM on the interleaved data:
//   C_il[n x 2m] = A_il[n x 2k] . B_exp[2k x 2m]
//   B_exp[2p,2j] = Br, B_exp[2p+1,2j] = -Bi, B_exp[2p,2j+1] = Bi, B_exp[2p+1,2j+1] = Br
// so A needs no de-interleave and C is written interleaved directly.
//
// 3xFP16 split with power-of-two scaling for FP32 accuracy.  Each row of A
// (and each complex column of B) gets a scale 2^e that puts its largest
// magnitude in [2^14, 2^15); then x*2^e = hi + lo with hi = rn_f16(x*2^e),
// lo = rn_f16(x*2^e - hi): 22 significant bits, like a TF32 hi/lo pair, at
// twice the tensor rate (kind::f16 runs K=16 per MMA where kind::tf32 runs
// K=8, from the same 32 bytes of shared memory per row).  C =
// A_hi.B_lo + A_lo.B_hi + A_hi.B_hi, small terms first, and the epilogue
// multiplies by 2^-(e_row + e_col) (exact: powers of two).  (The round-1
// kernel ran the same three products as 3xTF32: same accuracy, half the
// rate; 1xTF32 measures 2.9e-4 rel. Frobenius at 1024^3 -- over the 1e-4
// budget.)  The tensor core's accumulation is not round-to-nearest, so K is
// accumulated in chunks of 512: each chunk in a fresh TMEM accumulator, the
// chunks summed in FP32 round-to-nearest by the epilogue in fixed order
// (error flat in K).
//
// Pipeline per launch:
//   1. prep kernels (HBM-bound): A -> [A_hi; A_lo] + row maxima (K-major
//      fp16, K padded to 64) and B -> column maxima, then [Bt_hi; Bt_lo] =
//      B_exp^T (K-major fp16), built with an smem transpose; skipped when the
//      executor has them cached for a const input.  The GEMM kernel sees each
//      fp16 row as 4-byte words (two k per word): TMA boxes and smem
//      descriptors are the same bytes either way.
//   2. persistent warp-specialised GEMM, one CTA per SM:
//        warp 0  TMA producer (cp.async.bulk.tensor, SWIZZLE_64B, all four
//                operand tiles per stage)
//        warp 1  TMEM allocator + single-thread tcgen05.mma issuer (kind::f16,
//                M=128, N=BN, K=16), three products per k-step; commits release
//                smem stages and publish finished K chunks
//        warps 2-9 epilogue: tcgen05.ld 32x32b -> FP32 running sums in
//                registers -> unscale -> st.global (C interleaved complex,
//                row-major), coverage-masked
//      TMEM holds two BN-column accumulators that alternate per K chunk, so
//      draining chunk c overlaps the MMAs of chunk c+1 (and a tile's write-out
//      overlaps the next tile's first chunk).
#include <cuda.h>
#include <cuda_fp16.h>

#include <atomic>
#include <cstdlib>

#include "kaas_internal.cuh"

namespace kaas {
namespace {

constexpr int BM = 128;
constexpr int BK = 32;  // fp32 elements per k-block = 128 B rows -> SWIZZLE_128B
constexpr int STAGES = 4;
constexpr int GEMM_THREADS = 192;

// ---------------------------------------------------------------------------
// prep kernels

// Operand scaling.  mx = the bits of max |x| over a row of A (or a complex
// column of B); integer max on |x| bits, so a NaN beats Inf beats every
// finite value.  e puts mx * 2^e in [2^14, 2^15) (fp16 max 65504); rows that
// are all zero, or hold Inf / NaN, keep e = 0 (their results are Inf / NaN
// as in FP32); e is clamped to +-125 so 2^e and 2^-e are normal floats.
__host__ __device__ __forceinline__ int cg_exp(uint32_t mx) {
  const int E = (int)((mx >> 23) & 0xffu);
  if (E == 0xff) return 0;
  if (E == 0) return mx == 0 ? 0 : 125;
  const int e = 141 - E;  // 14 - (E - 127)
  return e > 125 ? 125 : e;
}
__device__ __forceinline__ float cg_pow2(int e) { return __int_as_float((127 + e) << 23); }

__device__ __forceinline__ uint32_t abs_bits(float x) { return __float_as_uint(x) & 0x7fffffffu; }

// x (already scaled) -> (hi, lo) fp16 pair
__device__ __forceinline__ void split16(float x, __half &hi, __half &lo) {
  hi = __float2half_rn(x);
  lo = __float2half_rn(x - __half2float(hi));
}

// A_il [n x k2] (k2 = 2k) -> Ahi/Alo [n x ldk] fp16 (zero padded past k2)
// and amax[r] = max-bits of row r.  One CTA per row (grid-stride): the row is
// read twice (max, then split), the second time from L1/L2.
__global__ void k_prep_a(int n, int k2, int ldk, const float *__restrict__ A, __half *__restrict__ Ahi,
                         __half *__restrict__ Alo, uint32_t *__restrict__ amax) {
  __shared__ uint32_t wmax[32];
  const bool vec = (k2 & 3) == 0;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int r = blockIdx.x; r < n; r += gridDim.x) {
    const float *src = A + (size_t)r * k2;
    __half *hi = Ahi + (size_t)r * ldk, *lo = Alo + (size_t)r * ldk;
    uint32_t mx = 0;
    if (vec) {
      for (int q4 = threadIdx.x; q4 < (k2 >> 2); q4 += blockDim.x) {
        const float4 x = __ldg(reinterpret_cast<const float4 *>(src) + q4);
        mx = max(max(mx, max(abs_bits(x.x), abs_bits(x.y))), max(abs_bits(x.z), abs_bits(x.w)));
      }
    } else {
      for (int q = threadIdx.x; q < k2; q += blockDim.x) mx = max(mx, abs_bits(src[q]));
    }
    mx = __reduce_max_sync(0xffffffffu, mx);
    if (lane == 0) wmax[warp] = mx;
    __syncthreads();
    mx = lane < nw ? wmax[lane] : 0u;
    mx = __reduce_max_sync(0xffffffffu, mx);
    const float sc = cg_pow2(cg_exp(mx));
    if (threadIdx.x == 0) amax[r] = mx;
    if (vec) {
      for (int q4 = threadIdx.x; q4 < (ldk >> 2); q4 += blockDim.x) {
        const int q = q4 << 2;
        const float4 x = q < k2 ? __ldg(reinterpret_cast<const float4 *>(src) + q4)
                                : make_float4(0.f, 0.f, 0.f, 0.f);
        __align__(8) __half h[4], l[4];
        split16(x.x * sc, h[0], l[0]);
        split16(x.y * sc, h[1], l[1]);
        split16(x.z * sc, h[2], l[2]);
        split16(x.w * sc, h[3], l[3]);
        reinterpret_cast<uint2 *>(hi)[q4] = *reinterpret_cast<const uint2 *>(h);
        reinterpret_cast<uint2 *>(lo)[q4] = *reinterpret_cast<const uint2 *>(l);
      }
    } else {
      for (int q = threadIdx.x; q < ldk; q += blockDim.x) {
        const float x = q < k2 ? src[q] : 0.f;
        split16(x * sc, hi[q], lo[q]);
      }
    }
    __syncthreads();  // wmax is reused by the next row
  }
}

// bmax[j] = max-bits over p of |Br[p][j]|, |Bi[p][j]| (bmax zeroed first).
// 1-D grid over (64-row p strip, 256-column j strip) tiles: no grid.y limit.
constexpr int kColMaxRows = 64;
__global__ void k_colmax_b(int k, int m, const float2 *__restrict__ B, uint32_t *__restrict__ bmax) {
  const uint64_t jt = ((uint64_t)m + 255) / 256, tiles = jt * (((uint64_t)k + kColMaxRows - 1) / kColMaxRows);
  for (uint64_t t = blockIdx.x; t < tiles; t += gridDim.x) {
    const int j = (int)(t % jt) * 256 + threadIdx.x;
    const int p0 = (int)(t / jt) * kColMaxRows, p1 = min(k, p0 + kColMaxRows);
    if (j >= m) continue;
    uint32_t mx = 0;
    for (int p = p0; p < p1; ++p) {
      const float2 v = __ldg(B + (size_t)p * m + j);
      mx = max(mx, max(abs_bits(v.x), abs_bits(v.y)));
    }
    atomicMax(bmax + j, mx);
  }
}

// B [k x m] complex -> Bt_hi/Bt_lo [2m x ldk] fp16, column j scaled by 2^e_j:
//   Bt[2j][2p] = Br[p][j]  Bt[2j][2p+1] = -Bi[p][j]
//   Bt[2j+1][2p] = Bi[p][j]  Bt[2j+1][2p+1] = Br[p][j]
// 32 (p) x 32 (j) complex tile through smem; block 32x8 threads.  The tiles
// cover p < ceil(k/32)*32 = ldk/2, so they also zero the K padding.
__global__ void k_prep_b(int k, int m, int ldk, const float2 *__restrict__ B, const uint32_t *__restrict__ bmax,
                         __half *__restrict__ Bhi, __half *__restrict__ Blo) {
  __shared__ float2 tile[32][33];
  const int tx = threadIdx.x, ty = threadIdx.y;
  // 1-D grid over the tiles (no 65535 grid.y limit on k)
  const uint64_t tiles_m = ((uint64_t)m + 31) / 32, tiles = tiles_m * (((uint64_t)k + 31) / 32);
  for (uint64_t t = blockIdx.x; t < tiles; t += gridDim.x) {
    const int p0 = (int)(t / tiles_m) * 32, j0 = (int)(t % tiles_m) * 32;
    for (int r = ty; r < 32; r += 8) {
      const int p = p0 + r, j = j0 + tx;
      tile[r][tx] = (p < k && j < m) ? B[(size_t)p * m + j] : make_float2(0.f, 0.f);
    }
    __syncthreads();
    // write: for each j (row pair 2j, 2j+1), lanes cover p = p0 + tx
    for (int c = ty; c < 32; c += 8) {
      const int j = j0 + c;
      if (j >= m) continue;
      const int p = p0 + tx;
      const int q = 2 * p;
      if (q >= ldk) continue;
      const float sc = cg_pow2(cg_exp(bmax[j]));
      const float2 v = tile[tx][c];  // (Br, Bi) at [p][j]
      __half2 eh, el, oh, ol;
      split16(v.x * sc, eh.x, el.x);
      split16(-v.y * sc, eh.y, el.y);
      split16(v.y * sc, oh.x, ol.x);
      oh.y = eh.x;
      ol.y = el.x;
      *reinterpret_cast<__half2 *>(Bhi + (size_t)(2 * j) * ldk + q) = eh;
      *reinterpret_cast<__half2 *>(Bhi + (size_t)(2 * j + 1) * ldk + q) = oh;
      *reinterpret_cast<__half2 *>(Blo + (size_t)(2 * j) * ldk + q) = el;
      *reinterpret_cast<__half2 *>(Blo + (size_t)(2 * j + 1) * ldk + q) = ol;
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------
// PTX helpers

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
  const uint32_t addr = smem_u32(bar);
  asm volatile(
      "{\n\t.reg .pred P1;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@!P1 bra WAIT_%=;\n\t}" ::"r"(addr),
      "r"(parity)
      : "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t *bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void tma_load_2d(const CUtensorMap *map, uint64_t *bar, void *dst, int c0,
                                            int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, "
      "%4}], [%2];" ::"r"(smem_u32(dst)),
      "l"(map), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
      : "memory");
}

__device__ __forceinline__ void tma_prefetch_desc(const CUtensorMap *map) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(map) : "memory");
}

__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}

__device__ __forceinline__ void tc_commit(uint64_t *bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   smem_u32(bar))
               : "memory");
}

__device__ __forceinline__ void tc_mma_f16(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc,
                                            uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}

// K-major operand tile, SWIZZLE_128B: rows of 128 B, 8-row groups 1024 B apart.
__device__ __forceinline__ uint64_t make_sw128_desc(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr & 0x3FFFFu) >> 4);  // start address
  d |= (uint64_t)1 << 16;                     // LBO (unused for swizzled K-major)
  d |= (uint64_t)(1024 >> 4) << 32;           // SBO: 8 rows x 128 B
  d |= (uint64_t)1 << 46;                     // descriptor version (sm_100)
  d |= (uint64_t)2 << 61;                     // SWIZZLE_128B
  return d;
}

// kind::f16 instruction descriptor: D=F32 (bits 4-5 = 1), A=B=F16 (bits
// 7-9, 10-12 = 0), both K-major, N>>3 at bit 17, M>>4 at bit 24.
__host__ __device__ constexpr uint32_t make_idesc(int mdim, int ndim) {
  return (1u << 4) | (0u << 7) | (0u << 10) | ((uint32_t)(ndim >> 3) << 17) |
         ((uint32_t)(mdim >> 4) << 24);
}

__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&v)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
        "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]),
        "=r"(v[14]), "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]),
        "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]),
        "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

// ---------------------------------------------------------------------------
// GEMM kernel

struct GemmShape {
  int M, N;          // output rows (n), output real columns (2m)
  int kb_per_seg;    // k-blocks per segment (ldk / BK)
  int a_lo_row;      // row offset of A_lo inside the A tensor map (= n)
  int b_lo_row;      // row offset of Bt_lo inside the B tensor map (= 2m)
  int num_m, num_n;  // tile grid
  int m_complex;     // m (complex columns) for coverage indexing
  unsigned long long cov;  // covered complex cells
  int ksplit;        // 1, or 2 = each tile's K in two halves on two CTAs,
                     // both red.add-ed onto a zeroed C ((0+a)+b == (0+b)+a
                     // exactly, so the result is deterministic)
  int kb_chunk;      // k-blocks per fresh-accumulator chunk (see k_cgemm_fused4)
  int group_m;       // m-blocks per raster group
  int panel_m;       // m-blocks (of 128 rows) per progressive write-back panel
  const uint32_t *amax;  // [M] max-bits of A's rows -> row scale 2^e (cg_exp)
  const uint32_t *bmax;  // [N/2] max-bits of B's complex columns -> column scale
};

constexpr int kGroupM = 8;  // default raster group, in m-blocks
// m-blocks per progressive write-back panel: a warm 8192^3 request is bound by
// its 512 MiB PCIe write-back, which starts when the first panel is done --
// 2-block panels start it sooner than 8 (11.85 vs 12.0 ms per request,
// tools/cgwarm_ab.sh; raster groups of 16 were 13.8-14.1 ms)
constexpr int kPanelM = 2;

__device__ __forceinline__ void tile_coords(const GemmShape &s, int t, int &mb, int &nb) {
  // group m-blocks together so concurrently running CTAs share B tiles in L2
  const int GM = s.group_m;
  const int per_group = GM * s.num_n;
  const int g = t / per_group;
  const int first_m = g * GM;
  const int gsize = min(GM, s.num_m - first_m);
  const int r = t % per_group;
  mb = first_m + r % gsize;
  nb = r / gsize;
}

// ---------------------------------------------------------------------------
// v2: all four operand tiles in every stage, three products per k-step.
//
// Stage = {A_hi, A_lo} [BM x 32] + {B_hi, B_lo} [BN x 32] fp16, 64-byte rows,
// SWIZZLE_64B (48 KiB at BN = 256, 4 stages).  Per k-step of 16 the single
// MMA thread issues A_hi.B_lo, A_lo.B_hi, A_hi.B_hi into the tile's TMEM
// accumulator, so K is walked once instead of three times.  The smem arrays
// and TMA coordinates count 4-byte words (two fp16 k each): BK2 words = 32 k.
constexpr int BK2 = 16;
// k-blocks (of 2 * BK2 interleaved k) per fresh-accumulator chunk: 512 of K
constexpr int kCgemmChunkKb = 16;
// ring depth: stages of (2 BM + 2 BN) x 16 words -- 32 KiB at BN = 128, 48 KiB
// at BN = 256 -- as many as fit next to the barriers (192 KiB either way); the
// narrow-tile case needs the depth to cover L2 latency (each stage is only
// 384 MMA cycles there)
template <int BN>
constexpr int stages2() { return BN == 128 ? 6 : 4; }

template <int BN, int STAGES2 = stages2<BN>()>
struct Smem2 {
  alignas(1024) float a_hi[STAGES2][BM * BK2];
  alignas(1024) float a_lo[STAGES2][BM * BK2];
  alignas(1024) float b_hi[STAGES2][BN * BK2];
  alignas(1024) float b_lo[STAGES2][BN * BK2];
  uint64_t full[STAGES2];
  uint64_t empty[STAGES2];
  uint64_t tfull[2];
  uint64_t tempty[2];
  uint32_t tmem_base;
};

// K-major operand tile, SWIZZLE_64B: rows of 64 B, 8-row groups 512 B apart.
__device__ __forceinline__ uint64_t make_sw64_desc(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr & 0x3FFFFu) >> 4);
  d |= (uint64_t)1 << 16;
  d |= (uint64_t)(512 >> 4) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)4 << 61;  // SWIZZLE_64B
  return d;
}

// K-chunked accumulation.  The tensor core adds each MMA's K=8 partial into
// the FP32 accumulator with less than round-to-nearest accuracy, so one
// accumulator over all of K loses accuracy about linearly in K (measured:
// 4.8e-6 rel. Frobenius at 1024^3, 3.8e-5 at 8192^3).  Instead every K chunk
// of kb_chunk k-blocks goes into a FRESH accumulator (the first MMA of the
// chunk does not accumulate); the two TMEM accumulators alternate per chunk,
// and the epilogue warps drain each finished chunk into per-thread FP32
// running sums (round-to-nearest adds, fixed chunk order -> deterministic)
// while the MMA warp fills the other accumulator.  The tile's sums are
// written out after its last chunk.  Eight epilogue warps: warps w and w+4
// share TMEM lane quarter w % 4 and split the tile's columns in halves, so a
// thread holds BN / 2 running sums.
constexpr int kEpiWarps = 8;

// sums (in the scaled domain) of row `row`, real columns col0.. -> C's
// values: times 2^-e_row, then 2^-e_col (each exact for normal results;
// columns 2j and 2j+1 share complex column j's scale).  The warp's lanes
// share the columns, so the scale loads are broadcasts.
// Applied per 32-column block q right before its stores.
template <int HALF>
__device__ __forceinline__ void unscale(const GemmShape &s, float ra, int col, float (&sum)[HALF], int q) {
#pragma unroll
  for (int j = 0; j < 16; ++j) {
    const int cj = (col >> 1) + j;
    const float cb = 2 * cj < s.N ? cg_pow2(-cg_exp(__ldg(s.bmax + cj))) : 1.f;
    sum[32 * q + 2 * j] = (sum[32 * q + 2 * j] * ra) * cb;
    sum[32 * q + 2 * j + 1] = (sum[32 * q + 2 * j + 1] * ra) * cb;
  }
}
constexpr int GEMM2_THREADS = 64 + 32 * kEpiWarps;

template <int BN>
__global__ void __launch_bounds__(GEMM2_THREADS, 1)
k_cgemm_fused4(const __grid_constant__ CUtensorMap map_a, const __grid_constant__ CUtensorMap map_b,
               const GemmShape s, float *__restrict__ C, unsigned *panel_done) {
  extern __shared__ uint8_t smem_raw[];
  Smem2<BN> &sm = *reinterpret_cast<Smem2<BN> *>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  constexpr int STAGES2 = stages2<BN>();
  constexpr int HALF = BN / 2;  // columns per epilogue thread
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  constexpr uint32_t kTmemCols = 2 * BN;
  constexpr uint32_t kStageBytes = (2 * BM + 2 * BN) * BK2 * 4;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&map_a);
    tma_prefetch_desc(&map_b);
    for (int i = 0; i < STAGES2; ++i) {
      mbar_init(&sm.full[i], 1);
      mbar_init(&sm.empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&sm.tfull[i], 1);
      mbar_init(&sm.tempty[i], kEpiWarps);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(&sm.tmem_base)),
                 "r"(kTmemCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = sm.tmem_base;
  const int total_units = s.num_m * s.num_n * s.ksplit;  // unit = (tile, K slice)
  const int kbs = s.kb_per_seg;  // k-blocks of BK2 per tile (one pass)

  if (warp == 0) {
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int u = blockIdx.x; u < total_units; u += gridDim.x) {
        int mb, nb;
        tile_coords(s, u / s.ksplit, mb, nb);
        const int arow = mb * BM, brow = nb * BN;
        const int ks = u % s.ksplit;
        for (int kb = ks * kbs / s.ksplit; kb < (ks + 1) * kbs / s.ksplit; ++kb) {
          mbar_wait(&sm.empty[stage], phase ^ 1);
          mbar_arrive_expect_tx(&sm.full[stage], kStageBytes);
          tma_load_2d(&map_a, &sm.full[stage], sm.a_hi[stage], kb * BK2, arow);
          tma_load_2d(&map_a, &sm.full[stage], sm.a_lo[stage], kb * BK2, s.a_lo_row + arow);
          tma_load_2d(&map_b, &sm.full[stage], sm.b_hi[stage], kb * BK2, brow);
          tma_load_2d(&map_b, &sm.full[stage], sm.b_lo[stage], kb * BK2, s.b_lo_row + brow);
          if (++stage == STAGES2) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t idesc = make_idesc(BM, BN);
      int stage = 0;
      uint32_t phase = 0;
      uint32_t chunk = 0;  // chunks issued by this CTA: accumulator = chunk & 1
      for (int u = blockIdx.x; u < total_units; u += gridDim.x) {
        const int ks = u % s.ksplit, kb0 = ks * kbs / s.ksplit, kb1 = (ks + 1) * kbs / s.ksplit;
        for (int c0 = kb0; c0 < kb1; c0 += s.kb_chunk, ++chunk) {
          const int c1 = min(kb1, c0 + s.kb_chunk);
          const uint32_t acc = chunk & 1;
          mbar_wait(&sm.tempty[acc], ((chunk >> 1) & 1) ^ 1);
          tc_fence_after();
          const uint32_t tmem_d = tmem_base + acc * BN;
          for (int kb = c0; kb < c1; ++kb) {
            mbar_wait(&sm.full[stage], phase);
            tc_fence_after();
            const uint32_t ah = smem_u32(sm.a_hi[stage]), al = smem_u32(sm.a_lo[stage]);
            const uint32_t bh = smem_u32(sm.b_hi[stage]), bl = smem_u32(sm.b_lo[stage]);
#pragma unroll
            for (int k = 0; k < BK2 / 8; ++k) {
              const uint32_t off = k * 32;
              // small terms first, then the main product; the chunk's first
              // MMA starts a fresh accumulator
              tc_mma_f16(tmem_d, make_sw64_desc(ah + off), make_sw64_desc(bl + off), idesc,
                          kb != c0 || k != 0);
              tc_mma_f16(tmem_d, make_sw64_desc(al + off), make_sw64_desc(bh + off), idesc, 1);
              tc_mma_f16(tmem_d, make_sw64_desc(ah + off), make_sw64_desc(bh + off), idesc, 1);
            }
            tc_commit(&sm.empty[stage]);
            if (++stage == STAGES2) {
              stage = 0;
              phase ^= 1;
            }
          }
          tc_commit(&sm.tfull[acc]);
        }
      }
    }
  } else {
    // ===== epilogue: warps 2 .. 2 + kEpiWarps - 1 =====
    const int quarter = warp & 3;               // TMEM lane quarter this warp may access
    const int half = (warp - 2) / 4;            // which half of the tile's columns
    uint32_t chunk = 0;
    for (int u = blockIdx.x; u < total_units; u += gridDim.x) {
      int mb, nb;
      tile_coords(s, u / s.ksplit, mb, nb);
      const int ks = u % s.ksplit, kb0 = ks * kbs / s.ksplit, kb1 = (ks + 1) * kbs / s.ksplit;
      const uint32_t lane_base = tmem_base + ((uint32_t)(quarter * 32) << 16) + half * HALF;
      float sum[HALF];
#pragma unroll
      for (int j = 0; j < HALF; ++j) sum[j] = 0.f;
      for (int c0 = kb0; c0 < kb1; c0 += s.kb_chunk, ++chunk) {
        const uint32_t acc = chunk & 1;
        mbar_wait(&sm.tfull[acc], (chunk >> 1) & 1);
        tc_fence_after();
#pragma unroll
        for (int q = 0; q < HALF / 32; ++q) {
          uint32_t v[32];
          tmem_ld32(lane_base + acc * BN + 32 * q, v);
#pragma unroll
          for (int j = 0; j < 32; ++j) sum[32 * q + j] = __fadd_rn(sum[32 * q + j], __uint_as_float(v[j]));
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&sm.tempty[acc]);
      }
      const int row = mb * BM + quarter * 32 + lane;
      const int col0 = nb * BN + half * HALF;
      if (row < s.M) {
        float *dst = C + (size_t)row * s.N + col0;
        const float ra = cg_pow2(-cg_exp(__ldg(s.amax + row)));
#pragma unroll
        for (int q = 0; q < HALF / 32; ++q) {
          const int col = col0 + 32 * q;
          unscale<HALF>(s, ra, col, sum, q);
          float *d = dst + 32 * q;
          const unsigned long long g0 = (unsigned long long)row * s.m_complex + (col >> 1);
          const bool full = (col + 32 <= s.N) && (g0 + 16 <= s.cov) &&
                            ((reinterpret_cast<uintptr_t>(d) & 15u) == 0);
          if (s.ksplit > 1) {  // K half: add onto the zeroed C
            if (full) {
#pragma unroll
              for (int j = 0; j < 8; ++j)
                asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(d + 4 * j),
                             "f"(sum[32 * q + 4 * j]), "f"(sum[32 * q + 4 * j + 1]),
                             "f"(sum[32 * q + 4 * j + 2]), "f"(sum[32 * q + 4 * j + 3])
                             : "memory");
            } else {
#pragma unroll
              for (int j = 0; j < 32; ++j) {
                const int c = col + j;
                if (c < s.N && (unsigned long long)row * s.m_complex + (c >> 1) < s.cov)
                  atomicAdd(d + j, sum[32 * q + j]);
              }
            }
          } else if (full) {
#pragma unroll
            for (int j = 0; j < 8; ++j)
              reinterpret_cast<float4 *>(d)[j] = make_float4(sum[32 * q + 4 * j], sum[32 * q + 4 * j + 1],
                                                             sum[32 * q + 4 * j + 2], sum[32 * q + 4 * j + 3]);
          } else {
#pragma unroll
            for (int j = 0; j < 32; ++j) {
              const int c = col + j;
              if (c < s.N && (unsigned long long)row * s.m_complex + (c >> 1) < s.cov) d[j] = sum[32 * q + j];
            }
          }
        }
      }
      if (panel_done != nullptr) {
        // publish "tile done" for its row panel (group of GM m-blocks) so the
        // copy stream can stream that panel to the host while tiles compute
        __threadfence();
        asm volatile("bar.sync 1, %0;" ::"n"(32 * kEpiWarps) : "memory");
        if (warp == 2 && lane == 0) {
          __threadfence_system();
          atomicAdd(&panel_done[mb / s.panel_m], 1u);
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 1) {
    __syncwarp();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                 "r"(kTmemCols));
  }
}

// ---------------------------------------------------------------------------
// CTA-pair kernel (cta_group::2): two SMs of a TPC compute one M256 x N256
// tile.  Each CTA loads its own 128 rows of A and 128 of the tile's 256
// Bt rows (N half) per stage -- 32 KiB instead of 48 KiB -- and the leader
// issues tcgen05.mma.cta_group::2 (M=256, N=256, K=8), which reads A and B
// from both CTAs' shared memory; each CTA's TMEM accumulates its 128 rows x
// all 256 columns.  Operand traffic per output element is 2/3 of the 1-CTA
// M128 x N256 tile's.  Everything else is k_cgemm_fused4's: three products
// per k-step, K-chunked accumulation drained by 8 epilogue warps per CTA,
// progressive write-back.
//
// Barriers (per CTA unless noted): full[s] -- the LEADER's counts both CTAs'
// TMA bytes (the peer's copies signal it through the cluster address with
// the peer bit cleared) and only the leader arms it; empty[s] -- in both
// CTAs, released by the leader's MMA commit multicast to both; tfull[a] --
// both CTAs, MMA commit multicast; tempty[a] -- the LEADER's counts the
// epilogue warps of both CTAs (the peer's arrive remotely).
constexpr int kPairStages = 6;
struct SmemPair {
  alignas(1024) float a_hi[kPairStages][BM * BK2];
  alignas(1024) float a_lo[kPairStages][BM * BK2];
  alignas(1024) float b_hi[kPairStages][128 * BK2];
  alignas(1024) float b_lo[kPairStages][128 * BK2];
  uint64_t full[kPairStages];
  uint64_t empty[kPairStages];
  uint64_t tfull[2];
  uint64_t tempty[2];
  uint32_t tmem_base;
};
constexpr uint32_t kPeerBitMask = 0xFEFFFFFFu;  // shared::cluster address of the pair's rank 0

__device__ __forceinline__ uint32_t pair_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ void tma_load_2d_pair(const CUtensorMap *map, uint64_t *bar, void *dst, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, "
      "%4}], [%2];" ::"r"(smem_u32(dst)),
      "l"(map), "r"(smem_u32(bar) & kPeerBitMask), "r"(c0), "r"(c1)
      : "memory");
}
__device__ __forceinline__ void tc_mma_f16_pair(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                                 uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, {%5, %5, %5, %5, %5, %5, %5, %5}, p;\n\t}" ::"r"(
          tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate), "r"(0u)
      : "memory");
}
__device__ __forceinline__ void tc_commit_pair(uint64_t *bar) {  // arrive on bar in both CTAs
  asm volatile(
      "{\n\t.reg .b16 m;\n\tmov.b16 m, 3;\n\t"
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], m;\n\t}" ::"r"(
          smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void mbar_arrive_leader(uint64_t *bar) {  // the pair's rank-0 copy of bar
  uint32_t remote;
  asm volatile("mapa.shared::cluster.u32 %0, %1, 0;" : "=r"(remote) : "r"(smem_u32(bar)));
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(remote) : "memory");
}

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(GEMM2_THREADS, 1)
k_cgemm_pair(const __grid_constant__ CUtensorMap map_a, const __grid_constant__ CUtensorMap map_b,
             const GemmShape s, float *__restrict__ C, unsigned *panel_done) {
  constexpr int BN = 256, HALF = BN / 2;
  extern __shared__ uint8_t smem_raw[];
  SmemPair &sm = *reinterpret_cast<SmemPair *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = pair_rank();
  const bool leader = rank == 0;
  constexpr uint32_t kTmemCols = 2 * BN;
  constexpr uint32_t kPairStageBytes = (2 * BM + 2 * 128) * BK2 * 4;  // one CTA's share

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&map_a);
    tma_prefetch_desc(&map_b);
    for (int i = 0; i < kPairStages; ++i) {
      mbar_init(&sm.full[i], 1);
      mbar_init(&sm.empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&sm.tfull[i], 1);
      mbar_init(&sm.tempty[i], 2 * kEpiWarps);  // only the leader's copy is used
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(&sm.tmem_base)),
                 "r"(kTmemCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  tc_fence_before();
  cluster_sync_all();  // both CTAs' barriers initialised and TMEM allocated
  tc_fence_after();
  const uint32_t tmem_base = sm.tmem_base;
  const int pair = blockIdx.x >> 1, npairs = gridDim.x >> 1;
  const int tiles = s.num_m * s.num_n;  // num_m counts 256-row tiles here
  const int kbs = s.kb_per_seg;

  if (warp == 0) {
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int t = pair; t < tiles; t += npairs) {
        int mb, nb;
        tile_coords(s, t, mb, nb);
        const int arow = mb * 256 + (int)rank * 128, brow = nb * BN + (int)rank * 128;
        for (int kb = 0; kb < kbs; ++kb) {
          mbar_wait(&sm.empty[stage], phase ^ 1);
          if (leader) mbar_arrive_expect_tx(&sm.full[stage], 2 * kPairStageBytes);
          tma_load_2d_pair(&map_a, &sm.full[stage], sm.a_hi[stage], kb * BK2, arow);
          tma_load_2d_pair(&map_a, &sm.full[stage], sm.a_lo[stage], kb * BK2, s.a_lo_row + arow);
          tma_load_2d_pair(&map_b, &sm.full[stage], sm.b_hi[stage], kb * BK2, brow);
          tma_load_2d_pair(&map_b, &sm.full[stage], sm.b_lo[stage], kb * BK2, s.b_lo_row + brow);
          if (++stage == kPairStages) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    if (leader && lane == 0) {
      constexpr uint32_t idesc = make_idesc(256, BN);
      int stage = 0;
      uint32_t phase = 0;
      uint32_t chunk = 0;
      for (int t = pair; t < tiles; t += npairs) {
        for (int c0 = 0; c0 < kbs; c0 += s.kb_chunk, ++chunk) {
          const int c1 = min(kbs, c0 + s.kb_chunk);
          const uint32_t acc = chunk & 1;
          mbar_wait(&sm.tempty[acc], ((chunk >> 1) & 1) ^ 1);
          tc_fence_after();
          const uint32_t tmem_d = tmem_base + acc * BN;
          for (int kb = c0; kb < c1; ++kb) {
            mbar_wait(&sm.full[stage], phase);
            tc_fence_after();
            const uint32_t ah = smem_u32(sm.a_hi[stage]), al = smem_u32(sm.a_lo[stage]);
            const uint32_t bh = smem_u32(sm.b_hi[stage]), bl = smem_u32(sm.b_lo[stage]);
#pragma unroll
            for (int k = 0; k < BK2 / 8; ++k) {
              const uint32_t off = k * 32;
              tc_mma_f16_pair(tmem_d, make_sw64_desc(ah + off), make_sw64_desc(bl + off), idesc,
                               kb != c0 || k != 0);
              tc_mma_f16_pair(tmem_d, make_sw64_desc(al + off), make_sw64_desc(bh + off), idesc, 1);
              tc_mma_f16_pair(tmem_d, make_sw64_desc(ah + off), make_sw64_desc(bh + off), idesc, 1);
            }
            tc_commit_pair(&sm.empty[stage]);
            if (++stage == kPairStages) {
              stage = 0;
              phase ^= 1;
            }
          }
          tc_commit_pair(&sm.tfull[acc]);
        }
      }
    }
  } else {
    const int quarter = warp & 3;
    const int half = (warp - 2) / 4;
    uint32_t chunk = 0;
    for (int t = pair; t < tiles; t += npairs) {
      int mb, nb;
      tile_coords(s, t, mb, nb);
      const uint32_t lane_base = tmem_base + ((uint32_t)(quarter * 32) << 16) + half * HALF;
      float sum[HALF];
#pragma unroll
      for (int j = 0; j < HALF; ++j) sum[j] = 0.f;
      for (int c0 = 0; c0 < kbs; c0 += s.kb_chunk, ++chunk) {
        const uint32_t acc = chunk & 1;
        mbar_wait(&sm.tfull[acc], (chunk >> 1) & 1);
        tc_fence_after();
#pragma unroll
        for (int q = 0; q < HALF / 32; ++q) {
          uint32_t v[32];
          tmem_ld32(lane_base + acc * BN + 32 * q, v);
#pragma unroll
          for (int j = 0; j < 32; ++j) sum[32 * q + j] = __fadd_rn(sum[32 * q + j], __uint_as_float(v[j]));
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive_leader(&sm.tempty[acc]);
      }
      const int row = mb * 256 + (int)rank * 128 + quarter * 32 + lane;
      const int col0 = nb * BN + half * HALF;
      if (row < s.M) {
        float *dst = C + (size_t)row * s.N + col0;
        const float ra = cg_pow2(-cg_exp(__ldg(s.amax + row)));
#pragma unroll
        for (int q = 0; q < HALF / 32; ++q) {
          const int col = col0 + 32 * q;
          unscale<HALF>(s, ra, col, sum, q);
          float *d = dst + 32 * q;
          const unsigned long long g0 = (unsigned long long)row * s.m_complex + (col >> 1);
          const bool full = (col + 32 <= s.N) && (g0 + 16 <= s.cov) &&
                            ((reinterpret_cast<uintptr_t>(d) & 15u) == 0);
          if (full) {
#pragma unroll
            for (int j = 0; j < 8; ++j)
              reinterpret_cast<float4 *>(d)[j] = make_float4(sum[32 * q + 4 * j], sum[32 * q + 4 * j + 1],
                                                             sum[32 * q + 4 * j + 2], sum[32 * q + 4 * j + 3]);
          } else {
#pragma unroll
            for (int j = 0; j < 32; ++j) {
              const int c = col + j;
              if (c < s.N && (unsigned long long)row * s.m_complex + (c >> 1) < s.cov) d[j] = sum[32 * q + j];
            }
          }
        }
      }
      if (panel_done != nullptr) {
        __threadfence();
        asm volatile("bar.sync 1, %0;" ::"n"(32 * kEpiWarps) : "memory");
        // each CTA reports its own 128-row m-block (the host counts panels in those)
        const int mb128 = mb * 2 + (int)rank;
        if (warp == 2 && lane == 0 && mb128 * BM < s.M) {
          __threadfence_system();
          atomicAdd(&panel_done[mb128 / s.panel_m], 1u);
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync_all();  // neither CTA leaves while the pair's MMAs may touch its smem / TMEM
  tc_fence_after();
  if (warp == 1) {
    __syncwarp();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(kTmemCols));
  }
}

// ---------------------------------------------------------------------------
// host side

typedef CUresult (*EncodeTiledFn)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *,
                                  const cuuint64_t *, const cuuint64_t *, const cuuint32_t *,
                                  const cuuint32_t *, CUtensorMapInterleave, CUtensorMapSwizzle,
                                  CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn get_encode() {
  static EncodeTiledFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void *p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  });
  return fn;
}

int make_map(CUtensorMap *map, const float *base, uint64_t rows, uint64_t ld, uint32_t box_rows,
             uint32_t box_k = BK, CUtensorMapSwizzle swz = CU_TENSOR_MAP_SWIZZLE_128B) {
  EncodeTiledFn enc = get_encode();
  if (!enc) return fail(KAAS_E_UNSUPPORTED, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t dims[2] = {ld, rows};
  cuuint64_t strides[1] = {ld * sizeof(float)};
  cuuint32_t box[2] = {box_k, box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, (void *)base, dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, swz,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(KAAS_E_INVALID, "cuTensorMapEncodeTiled failed: " + std::to_string((int)r));
  return 0;
}

typedef CUresult (*WaitValue32Fn)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);

WaitValue32Fn get_wait_value() {
  static WaitValue32Fn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void *p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuStreamWaitValue32", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<WaitValue32Fn>(p);
  });
  return fn;
}

template <int BN>
int launch_gemm2(cudaStream_t s, int dev, const CUtensorMap &ma, const CUtensorMap &mb,
                 const GemmShape &shape, float *C, StreamScratch *sc, const ProgressiveOut *po) {
  const size_t smem = sizeof(Smem2<BN>) + 1024;
  static std::atomic<uint64_t> attr_done{0};  // bit per device (dev < 64)
  if (!(attr_done.load(std::memory_order_relaxed) >> (dev & 63) & 1)) {
    KAAS_CUDA(cudaFuncSetAttribute(k_cgemm_fused4<BN>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)smem));
    attr_done.fetch_or(1ull << (dev & 63));
  }
  const int units = shape.num_m * shape.num_n * shape.ksplit;
  int grid = device_props(dev).sm_count;
  if (grid > units) grid = units;
  const int PM = shape.panel_m;
  const int npanels = (shape.num_m + PM - 1) / PM;
  WaitValue32Fn waitv = get_wait_value();
  // panels stream out while later tiles compute -- only when there are later
  // tiles: in a single wave every tile finishes at once, and the per-panel
  // waits and copies would only add latency (1024^3: 0.28 -> 0.32 ms)
  const bool progressive = po != nullptr && waitv != nullptr && npanels > 1 && units > grid &&
                           npanels <= kMaxPanels && sc->panel_done != nullptr;
  if (po && !sc->cg_ev_ready) {
    KAAS_CUDA(cudaEventCreateWithFlags(&sc->cg_ev_ready, cudaEventDisableTiming));
    KAAS_CUDA(cudaEventCreateWithFlags(&sc->cg_ev_done, cudaEventDisableTiming));
  }
  cudaEvent_t ev_ready = sc->cg_ev_ready, ev_done = sc->cg_ev_done;
  if (progressive) {
    KAAS_CUDA(cudaMemsetAsync(sc->panel_done, 0, npanels * sizeof(unsigned), s));
    KAAS_CUDA(cudaEventRecord(ev_ready, s));
    KAAS_CUDA(cudaStreamWaitEvent(po->out_stream, ev_ready, 0));
  }
  k_cgemm_fused4<BN><<<grid, GEMM2_THREADS, smem, s>>>(ma, mb, shape, C,
                                                      progressive ? sc->panel_done : nullptr);
  count_launch();
  KAAS_CUDA(cudaGetLastError());
  if (!po) return 0;
  const uint64_t row_bytes = (uint64_t)shape.m_complex * 8;
  uint64_t copied = 0;
  if (progressive) {
    for (int p = 0; p < npanels; ++p) {
      const int mb0 = p * PM, mbs = min(PM, shape.num_m - mb0);
      const int row0 = mb0 * BM, row1 = min(shape.M, (mb0 + mbs) * BM);
      const unsigned want = (unsigned)(mbs * shape.num_n * shape.ksplit);
      CUresult r = waitv((CUstream)po->out_stream, (CUdeviceptr)(sc->panel_done + p), want,
                         0 /* CU_STREAM_WAIT_VALUE_GEQ */);
      if (r != CUDA_SUCCESS) return fail(KAAS_E_UNSUPPORTED, "cuStreamWaitValue32 failed");
      const uint64_t off = (uint64_t)row0 * row_bytes, len = (uint64_t)(row1 - row0) * row_bytes;
      KAAS_CUDA(cudaMemcpyAsync((char *)po->host + off, (const char *)C + off, len,
                                cudaMemcpyDeviceToHost, po->out_stream));
      copied = off + len;
    }
  }
  // the rest (or everything, without progressive support) once the kernel is done
  KAAS_CUDA(cudaEventRecord(ev_done, s));
  KAAS_CUDA(cudaStreamWaitEvent(po->out_stream, ev_done, 0));
  if (copied < po->bytes)
    KAAS_CUDA(cudaMemcpyAsync((char *)po->host + copied, (const char *)C + copied,
                              po->bytes - copied, cudaMemcpyDeviceToHost, po->out_stream));
  return 0;
}

// CTA-pair launch: shape.num_m counts 256-row tiles, map_b's box is 128 rows
// (each CTA's half of the N256 tile).  Progressive write-back panels are in
// 128-row m-blocks as for the 1-CTA kernel.
int launch_pair(cudaStream_t s, int dev, const CUtensorMap &ma, const CUtensorMap &mb, const GemmShape &shape,
                float *C, StreamScratch *sc, const ProgressiveOut *po) {
  const size_t smem = sizeof(SmemPair) + 1024;
  static std::atomic<uint64_t> attr_done{0};
  if (!(attr_done.load(std::memory_order_relaxed) >> (dev & 63) & 1)) {
    KAAS_CUDA(cudaFuncSetAttribute(k_cgemm_pair, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    attr_done.fetch_or(1ull << (dev & 63));
  }
  const int tiles = shape.num_m * shape.num_n;
  int pairs = device_props(dev).sm_count / 2;
  if (pairs > tiles) pairs = tiles;
  const int num_m128 = (shape.M + BM - 1) / BM;
  const int PM = shape.panel_m;
  const int npanels = (num_m128 + PM - 1) / PM;
  WaitValue32Fn waitv = get_wait_value();
  const bool progressive = po != nullptr && waitv != nullptr && npanels > 1 && tiles > pairs &&
                           npanels <= kMaxPanels && sc->panel_done != nullptr;
  if (po && !sc->cg_ev_ready) {
    KAAS_CUDA(cudaEventCreateWithFlags(&sc->cg_ev_ready, cudaEventDisableTiming));
    KAAS_CUDA(cudaEventCreateWithFlags(&sc->cg_ev_done, cudaEventDisableTiming));
  }
  cudaEvent_t ev_ready = sc->cg_ev_ready, ev_done = sc->cg_ev_done;
  if (progressive) {
    KAAS_CUDA(cudaMemsetAsync(sc->panel_done, 0, npanels * sizeof(unsigned), s));
    KAAS_CUDA(cudaEventRecord(ev_ready, s));
    KAAS_CUDA(cudaStreamWaitEvent(po->out_stream, ev_ready, 0));
  }
  k_cgemm_pair<<<2 * pairs, GEMM2_THREADS, smem, s>>>(ma, mb, shape, C, progressive ? sc->panel_done : nullptr);
  count_launch();
  KAAS_CUDA(cudaGetLastError());
  if (!po) return 0;
  const uint64_t row_bytes = (uint64_t)shape.m_complex * 8;
  uint64_t copied = 0;
  if (progressive) {
    for (int p = 0; p < npanels; ++p) {
      const int mb0 = p * PM, mbs = min(PM, num_m128 - mb0);
      const int row0 = mb0 * BM, row1 = min(shape.M, (mb0 + mbs) * BM);
      const unsigned want = (unsigned)(mbs * shape.num_n);
      CUresult r = waitv((CUstream)po->out_stream, (CUdeviceptr)(sc->panel_done + p), want,
                         0 /* CU_STREAM_WAIT_VALUE_GEQ */);
      if (r != CUDA_SUCCESS) return fail(KAAS_E_UNSUPPORTED, "cuStreamWaitValue32 failed");
      const uint64_t off = (uint64_t)row0 * row_bytes, len = (uint64_t)(row1 - row0) * row_bytes;
      KAAS_CUDA(cudaMemcpyAsync((char *)po->host + off, (const char *)C + off, len, cudaMemcpyDeviceToHost,
                                po->out_stream));
      copied = off + len;
    }
  }
  KAAS_CUDA(cudaEventRecord(ev_done, s));
  KAAS_CUDA(cudaStreamWaitEvent(po->out_stream, ev_done, 0));
  if (copied < po->bytes)
    KAAS_CUDA(cudaMemcpyAsync((char *)po->host + copied, (const char *)C + copied, po->bytes - copied,
                              cudaMemcpyDeviceToHost, po->out_stream));
  return 0;
}

}  // namespace

static int plain_copy_after(cudaStream_t s, const ProgressiveOut *po, const float *C) {
  cudaEvent_t ev;
  KAAS_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
  KAAS_CUDA(cudaEventRecord(ev, s));
  KAAS_CUDA(cudaStreamWaitEvent(po->out_stream, ev, 0));
  KAAS_CUDA(cudaMemcpyAsync(po->host, C, po->bytes, cudaMemcpyDeviceToHost, po->out_stream));
  cudaEventDestroy(ev);
  return 0;
}

int launch_cgemm(cudaStream_t s, int dev, int n, int m, int k, uint64_t cov, const float *A,
                 const float *B, float *C, StreamScratch *sc, const ProgressiveOut *po,
                 const CgemmPrepared *prep) {
  if (n == 0 || m == 0 || cov == 0) return po ? plain_copy_after(s, po, C) : 0;
  if (k == 0) {
    // empty contraction: covered cells are 0 + 0i
    const uint64_t nm = (uint64_t)n * m;
    const uint64_t cells = cov < nm ? cov : nm;
    KAAS_CUDA(cudaMemsetAsync(C, 0, cells * 8, s));
    return po ? plain_copy_after(s, po, C) : 0;
  }
  // operand layout (cgemm_prepared_bytes): [hi plane | lo plane] fp16, rows
  // of ldk halves (2k rounded up to 64: whole 128-byte rows), then the
  // per-row (A) / per-complex-column (B) max-bits that fix the scales
  const int k2 = 2 * k;
  const int ldk = (int)cgemm_ldk16(k);
  const int ldkw = ldk / 2;  // the same rows in 4-byte words (TMA / MMA view)
  const size_t a_half = (size_t)n * ldk, b_half = (size_t)2 * m * ldk;
  const size_t a_bytes = cgemm_prepared_bytes(0, n, m, k), b_bytes = cgemm_prepared_bytes(1, n, m, k);
  // operands come from the executor's prepared-operand cache when it has
  // them; otherwise from per-stream scratch (only the missing side)
  const bool a_ext = prep && prep->a, b_ext = prep && prep->b;
  const size_t a_scr = a_ext ? 0 : (a_bytes + 255) / 256 * 256;
  const size_t need = a_scr + (b_ext ? 0 : b_bytes);
  int rc = need ? ensure_cgemm_scratch(sc, s, need) : 0;
  if (rc) return rc;
  char *scratch = (char *)sc->cg_buf;
  __half *Ahi = a_ext ? (__half *)prep->a : (__half *)scratch;
  __half *Alo = Ahi + a_half;
  uint32_t *amax = reinterpret_cast<uint32_t *>(Ahi + 2 * a_half);
  __half *Bhi = b_ext ? (__half *)prep->b : (__half *)(scratch + a_scr);
  __half *Blo = Bhi + b_half;
  uint32_t *bmax = reinterpret_cast<uint32_t *>(Bhi + 2 * b_half);

  const int sms = device_props(dev).sm_count;
  if (!(a_ext && prep->a_ready)) {
    k_prep_a<<<n < sms * 16 ? n : sms * 16, 256, 0, s>>>(n, k2, ldk, A, Ahi, Alo, amax);
    count_launch();
  }
  if (!(b_ext && prep->b_ready)) {
    KAAS_CUDA(cudaMemsetAsync(bmax, 0, (size_t)m * 4, s));
    const uint64_t ctiles = (((uint64_t)m + 255) / 256) * (((uint64_t)k + kColMaxRows - 1) / kColMaxRows);
    k_colmax_b<<<(unsigned)(ctiles < (uint64_t)sms * 16 ? ctiles : (uint64_t)sms * 16), 256, 0, s>>>(
        k, m, reinterpret_cast<const float2 *>(B), bmax);
    count_launch();
    const uint64_t tiles = (uint64_t)((m + 31) / 32) * (uint64_t)((k + 31) / 32);
    dim3 gb((unsigned)(tiles < (uint64_t)sms * 16 ? tiles : (uint64_t)sms * 16));
    // also zero-fills the K padding columns [2k, ldk)
    k_prep_b<<<gb, dim3(32, 8), 0, s>>>(k, m, ldk, reinterpret_cast<const float2 *>(B), bmax, Bhi, Blo);
    count_launch();
  }
  KAAS_CUDA(cudaGetLastError());

  // Small problems: narrower N tiles, or (full coverage only: C is zeroed
  // first) each tile's K split over two CTAs, so the grid covers the SMs.
  const int N = 2 * m;
  const int tiles256 = ((n + BM - 1) / BM) * ((N + 255) / 256);
  const bool full_cov = cov >= (uint64_t)n * m;
  const char *ke = KAAS_DEV_ENV("KAAS_CGEMM_KSPLIT");  // dev A/B: 0 = never split K
  const bool ksplit2 = !(ke && ke[0] == '0') && full_cov && tiles256 < sms && 2 * tiles256 <= sms &&
                       ldkw / BK2 >= 16;
  const bool narrow = tiles256 < sms && !ksplit2;
  const int BNv = narrow ? 128 : 256;

  // 1..8 waves of M256 x N256 tiles: CTA pairs (2-5% faster at 2048^3 and
  // 4096^3).  Beyond that the 1-CTA kernel: both are tensor-pipe bound under
  // the board power cap there, and the pair draws more power per flop (its
  // operand exchange between the two SMs), so it settles ~5% lower in SM
  // clock and is 2.6% slower at 8192^3 (profiles/r02/probes/cgemm_pair.txt).
  // Dev A/B: KAAS_CGEMM_PAIR=0 never, =1 always.
  const char *pe = KAAS_DEV_ENV("KAAS_CGEMM_PAIR");
  const int tiles_pair = ((n + 255) / 256) * ((N + 255) / 256);
  const bool pair = !narrow && !ksplit2 && tiles_pair >= sms / 2 &&
                    (pe ? pe[0] == '1' : tiles_pair <= 8 * (sms / 2));
  CUtensorMap ma, mbm;
  if ((rc = make_map(&ma, (const float *)Ahi, (uint64_t)2 * n, ldkw, BM, BK2, CU_TENSOR_MAP_SWIZZLE_64B))) return rc;
  if (pair) {
    if ((rc = make_map(&mbm, (const float *)Bhi, (uint64_t)2 * N, ldkw, 128, BK2, CU_TENSOR_MAP_SWIZZLE_64B))) return rc;
    GemmShape ps;
    ps.M = n;
    ps.N = N;
    ps.kb_per_seg = ldkw / BK2;
    ps.amax = amax;
    ps.bmax = bmax;
    ps.a_lo_row = n;
    ps.b_lo_row = N;
    ps.num_m = (n + 255) / 256;
    ps.num_n = (N + 255) / 256;
    ps.m_complex = m;
    ps.cov = cov;
    ps.ksplit = 1;
    ps.kb_chunk = kCgemmChunkKb;
    ps.group_m = kGroupM / 2;
    ps.panel_m = kPanelM;
    if (const char *pe2 = KAAS_DEV_ENV("KAAS_CGEMM_PANELM")) ps.panel_m = atoi(pe2) > 0 ? atoi(pe2) : kPanelM;
    if (const char *ge = KAAS_DEV_ENV("KAAS_CGEMM_GROUPM")) ps.group_m = atoi(ge) > 0 ? atoi(ge) : kGroupM / 2;
    if (const char *ce = KAAS_DEV_ENV("KAAS_CGEMM_CHUNK")) ps.kb_chunk = atoi(ce) > 0 ? atoi(ce) : 1 << 30;
    return launch_pair(s, dev, ma, mbm, ps, C, sc, po);
  }
  if ((rc = make_map(&mbm, (const float *)Bhi, (uint64_t)2 * N, ldkw, BNv, BK2, CU_TENSOR_MAP_SWIZZLE_64B))) return rc;
  GemmShape shape;
  shape.M = n;
  shape.N = N;
  shape.kb_per_seg = ldkw / BK2;
  shape.amax = amax;
  shape.bmax = bmax;
  shape.a_lo_row = n;
  shape.b_lo_row = N;
  shape.num_m = (n + BM - 1) / BM;
  shape.num_n = (N + BNv - 1) / BNv;
  shape.m_complex = m;
  shape.cov = cov;
  shape.ksplit = ksplit2 ? 2 : 1;
  shape.kb_chunk = kCgemmChunkKb;
  shape.group_m = kGroupM;
  if (const char *ge = KAAS_DEV_ENV("KAAS_CGEMM_GROUPM")) shape.group_m = atoi(ge) > 0 ? atoi(ge) : kGroupM;
  shape.panel_m = kPanelM;
  if (const char *pe2 = KAAS_DEV_ENV("KAAS_CGEMM_PANELM")) shape.panel_m = atoi(pe2) > 0 ? atoi(pe2) : kPanelM;
  if (const char *ce = KAAS_DEV_ENV("KAAS_CGEMM_CHUNK")) shape.kb_chunk = atoi(ce) > 0 ? atoi(ce) : 1 << 30;
  if (ksplit2) KAAS_CUDA(cudaMemsetAsync(C, 0, (size_t)n * m * 8, s));
  return narrow ? launch_gemm2<128>(s, dev, ma, mbm, shape, C, sc, po)
                : launch_gemm2<256>(s, dev, ma, mbm, shape, C, sc, po);
}

int encode_map_f32(CUtensorMap *map, const float *base, uint64_t rows, uint64_t ld, uint32_t box_rows,
                   uint32_t box_k, int swizzle_bytes) {
  const CUtensorMapSwizzle swz = swizzle_bytes == 128  ? CU_TENSOR_MAP_SWIZZLE_128B
                                 : swizzle_bytes == 64 ? CU_TENSOR_MAP_SWIZZLE_64B
                                                       : CU_TENSOR_MAP_SWIZZLE_NONE;
  return make_map(map, base, rows, ld, box_rows, box_k, swz);
}

}  // namespace kaas
