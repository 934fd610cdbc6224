// Bit-exact matmul tile (backend.py:174-189), shared by the per-invocation
// kernel (builtins.cu) and the persistent invocation-run kernel (runs.cu).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace kaas {

__device__ __forceinline__ void mm_pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void mm_pdl_release() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

// ---- matmul: per cell acc = 0; acc = fl(acc + fl(a*b)), k ascending --------
// (backend.py:174-189, oracle pkg/tests/oracles.py:25-33).  Bit-exactness
// forbids split-K and FMA, so each MAC is an FMUL + FADD (the SIMT roofline
// is 64 MAC/clk/SM) and all parallelism comes from output cells.  A CTA of
// TY x TX threads owns a (TY*TM) x (TX*TN) tile, each thread a TM x TN block
// of cells.  The shape is picked per launch by a small cost model
// (launch_matmul): big layers get 4x4 blocking, small-M / long-K layers
// (ResNet stage 4: M = 49, K = 4608) get small CTAs of 1x1 or 2x2 blocks so
// every scheduler has warps.
//
// Operands stream through an S-deep ring of BK = 32 k-chunks filled by
// cp.async (zero-filled out of bounds).  Both tiles are stored k-contiguous
// in smem (A row-major, B transposed, rows padded to 36 floats), so a thread
// reads 4 k of each of its rows and columns with one LDS.128: per 4 k that
// is TM + TN loads for 8 TM TN FP instructions.  A is copied 16 bytes at a
// time when K and the pointer allow it.  Padding products are never added
// (0*Inf would be NaN and +0 would flip the sign of a -0.0 accumulator), so
// the tail chunk uses the true extent.

__device__ __forceinline__ void cp_async4(float *dst, const float *src, bool ok) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;\n" ::"r"(d), "l"(src),
               "r"(ok ? 4 : 0)
               : "memory");
}
__device__ __forceinline__ void cp_async16(float *dst, const float *src, int bytes) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(d), "l"(src), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}


template <int TY, int TX, int TM, int TN, int S, int BK>
constexpr int mm_smem_bytes() {
  return S * (TY * TM + TX * TN) * (BK + 4) * 4;
}

// BT: b is given transposed ([m][k], k-contiguous, 16-byte aligned rows --
// the executor keeps that form of a const weight beside its cache entry), so
// B is copied 16 bytes at a time like A instead of one 4-byte cp.async per
// element (a third of the small-tile kernels' instructions went to those).
//
// One output tile (rows bm.., columns bn..) computed by the calling CTA's
// TY x TX threads; `smem` holds mm_smem_bytes<...>() bytes.  kPdl: the tile
// is a whole kernel launched with programmatic dependent launch (wait for the
// predecessor before the first copy, release dependents after the k loop).
// The caller must __syncthreads() between two tiles that share `smem`.
// `tid` is the thread's index in the tile's group of TY x TX threads; `bar`
// the named barrier the group synchronises on (0: the whole CTA is the group,
// __syncthreads), so a CTA can run several small tiles side by side.
template <int TY, int TX, int TM, int TN, int S, int BK, bool AV, bool BT, bool kPdl>
__device__ __forceinline__ void mm_tile(int n, int m, int k, uint64_t cov, const float *__restrict__ a,
                                        const float *__restrict__ b, float *__restrict__ out, int bm, int bn,
                                        float *mm_smem, int tid = threadIdx.x, int bar = 0,
                                        const float *__restrict__ res = nullptr, uint64_t res_cov = 0) {
  constexpr int T = TY * TX, BM = TY * TM, BN = TX * TN, LD = BK + 4;
  constexpr int A_ST = BM * LD, B_ST = BN * LD;
  constexpr int NA4 = (BM * (BK / 4) + T - 1) / T;  // 16-byte A copies per thread
  constexpr int NA1 = (BM * BK + T - 1) / T;        // 4-byte A copies per thread
  constexpr int NB = BT ? (BN * (BK / 4) + T - 1) / T  // 16-byte Bt copies per thread
                        : (BK * BN + T - 1) / T;       // 4-byte B copies per thread
  float *As = mm_smem, *Bs = mm_smem + S * A_ST;
  const int tx = tid % TX, ty = tid / TX;
  const int nk = (k + BK - 1) / BK;

  // Per-thread copy slots, fixed across chunks: a running source pointer
  // (advanced by one chunk per issue), the smem offset, and the row/column
  // validity.  Only the tail chunk checks k per element.
  constexpr int NA = AV ? NA4 : NA1;
  const float *pa[NA];
  int sa[NA], ka[NA], ba[NA];  // smem offset, k offset in chunk (-1 unused), copy bytes
  size_t step_a[NA];
#pragma unroll
  for (int u = 0; u < NA; ++u) {
    const int e = tid + T * u;
    const int r = AV ? e / (BK / 4) : e / BK;
    const int kk = AV ? 4 * (e % (BK / 4)) : e % BK;
    const bool used = r < BM;
    const bool ok = used && bm + r < n;
    ka[u] = used ? kk : -1;
    sa[u] = used ? r * LD + kk : 0;
    ba[u] = ok ? (AV ? 16 : 4) : 0;
    pa[u] = ok ? a + (size_t)(bm + r) * k + kk : a;
    step_a[u] = ok ? BK : 0;
  }
  const float *pb[NB];
  int sb[NB], kb[NB], bb[NB];
  size_t step_b[NB];
#pragma unroll
  for (int u = 0; u < NB; ++u) {
    const int e = tid + T * u;
    if (BT) {  // Bt[bn + c][k0 + kk .. +3] -> Bs[c][kk .. +3]
      const int c = e / (BK / 4), kk = 4 * (e % (BK / 4));
      const bool used = c < BN;
      const bool ok = used && bn + c < m;
      kb[u] = used ? kk : -1;
      sb[u] = used ? c * LD + kk : 0;
      bb[u] = ok ? 16 : 0;
      pb[u] = ok ? b + (size_t)(bn + c) * k + kk : b;
      step_b[u] = ok ? BK : 0;
    } else {
      const int kk = e / BN, c = e % BN;
      const bool used = kk < BK;
      const bool ok = used && bn + c < m;
      kb[u] = used ? kk : -1;
      sb[u] = used ? c * LD + kk : 0;  // B[k0 + kk][bn + c] -> Bs[c][kk]
      bb[u] = ok ? 4 : 0;
      pb[u] = ok ? b + (size_t)kk * m + bn + c : b;
      step_b[u] = ok ? (size_t)BK * m : 0;
    }
  }
  int stage_in = 0;  // stage the next issue() fills
  auto issue = [&](int t) {
    const int k0 = t * BK;
    float *as = As + stage_in * A_ST, *bs = Bs + stage_in * B_ST;
    stage_in = stage_in + 1 == S ? 0 : stage_in + 1;
    if (k0 + BK <= k) {  // full chunk: fixed per-slot sizes
#pragma unroll
      for (int u = 0; u < NA; ++u) {
        if (BM * (AV ? BK / 4 : BK) % T != 0 && ka[u] < 0) continue;
        if (AV) cp_async16(as + sa[u], pa[u], ba[u]);
        else cp_async4(as + sa[u], pa[u], ba[u] != 0);
      }
#pragma unroll
      for (int u = 0; u < NB; ++u) {
        if ((BT ? BN * (BK / 4) : BK * BN) % T != 0 && kb[u] < 0) continue;
        if (BT) cp_async16(bs + sb[u], pb[u], bb[u]);
        else cp_async4(bs + sb[u], pb[u], bb[u] != 0);
      }
    } else {  // tail chunk: k bound per element
#pragma unroll
      for (int u = 0; u < NA; ++u) {
        if (ka[u] < 0) continue;
        const int left = k - (k0 + ka[u]);
        if (AV) {
          const int bytes = (ba[u] && left > 0) ? (left >= 4 ? 16 : 4 * left) : 0;
          cp_async16(as + sa[u], bytes ? pa[u] : a, bytes);
        } else {
          const bool ok = ba[u] && left > 0;
          cp_async4(as + sa[u], ok ? pa[u] : a, ok);
        }
      }
#pragma unroll
      for (int u = 0; u < NB; ++u) {
        if (kb[u] < 0) continue;
        if (BT) {
          const int left = k - (k0 + kb[u]);
          const int bytes = (bb[u] && left > 0) ? (left >= 4 ? 16 : 4 * left) : 0;
          cp_async16(bs + sb[u], bytes ? pb[u] : b, bytes);
        } else {
          const bool ok = bb[u] && k0 + kb[u] < k;
          cp_async4(bs + sb[u], ok ? pb[u] : b, ok);
        }
      }
    }
#pragma unroll
    for (int u = 0; u < NA; ++u) pa[u] += step_a[u];
#pragma unroll
    for (int u = 0; u < NB; ++u) pb[u] += step_b[u];
  };

  float acc[TM][TN];
#pragma unroll
  for (int i = 0; i < TM; ++i)
#pragma unroll
    for (int j = 0; j < TN; ++j) acc[i][j] = 0.0f;

  if (kPdl) mm_pdl_wait();  // the operands may be the previous kernel's output
#pragma unroll
  for (int t = 0; t < S - 1; ++t) {
    if (t < nk) issue(t);
    cp_async_commit();
  }
  for (int t = 0; t < nk; ++t) {
    cp_async_wait<S - 2>();
    // chunk t landed; everyone is done with chunk t-1's stage
    if (bar == 0) __syncthreads();
    else asm volatile("bar.sync %0, %1;" ::"r"(bar), "n"(T) : "memory");
    if (t + S - 1 < nk) issue(t + S - 1);
    cp_async_commit();
    // thread (ty, tx) owns rows ty + TY*i and columns tx + TX*j: each LDS.128
    // of a warp then hits consecutive rows (4-bank steps), conflict-free
    const float *as = As + (t % S) * A_ST + ty * LD;
    const float *bs = Bs + (t % S) * B_ST + tx * LD;
    const int kc = min(BK, k - t * BK);
    if (kc == BK && TM * TN <= 2) {
      // one or two serial FADD chains per thread: load 16 k of each operand
      // before the arithmetic, so one shared-memory latency covers 16 chain
      // steps instead of 4 (ResNet chain kernels -2%)
#pragma unroll
      for (int k16 = 0; k16 < BK; k16 += 16) {
        float4 av[4][TM], bv[4][TN];
#pragma unroll
        for (int g = 0; g < 4; ++g) {
#pragma unroll
          for (int i = 0; i < TM; ++i) av[g][i] = *reinterpret_cast<const float4 *>(as + i * TY * LD + k16 + 4 * g);
#pragma unroll
          for (int j = 0; j < TN; ++j) bv[g][j] = *reinterpret_cast<const float4 *>(bs + j * TX * LD + k16 + 4 * g);
        }
#pragma unroll
        for (int g = 0; g < 4; ++g)
#pragma unroll
          for (int q = 0; q < 4; ++q)
#pragma unroll
            for (int i = 0; i < TM; ++i) {
              const float x = q == 0 ? av[g][i].x : q == 1 ? av[g][i].y : q == 2 ? av[g][i].z : av[g][i].w;
#pragma unroll
              for (int j = 0; j < TN; ++j) {
                const float y = q == 0 ? bv[g][j].x : q == 1 ? bv[g][j].y : q == 2 ? bv[g][j].z : bv[g][j].w;
                acc[i][j] = __fadd_rn(acc[i][j], __fmul_rn(x, y));
              }
            }
      }
    } else if (kc == BK) {
#pragma unroll
      for (int k4 = 0; k4 < BK; k4 += 4) {
        float4 av[TM], bv[TN];
#pragma unroll
        for (int i = 0; i < TM; ++i) av[i] = *reinterpret_cast<const float4 *>(as + i * TY * LD + k4);
#pragma unroll
        for (int j = 0; j < TN; ++j) bv[j] = *reinterpret_cast<const float4 *>(bs + j * TX * LD + k4);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
#pragma unroll
          for (int i = 0; i < TM; ++i) {
            const float x = q == 0 ? av[i].x : q == 1 ? av[i].y : q == 2 ? av[i].z : av[i].w;
#pragma unroll
            for (int j = 0; j < TN; ++j) {
              const float y = q == 0 ? bv[j].x : q == 1 ? bv[j].y : q == 2 ? bv[j].z : bv[j].w;
              acc[i][j] = __fadd_rn(acc[i][j], __fmul_rn(x, y));
            }
          }
        }
      }
    } else {
      for (int kk = 0; kk < kc; ++kk) {
#pragma unroll
        for (int i = 0; i < TM; ++i) {
          const float x = as[i * TY * LD + kk];
#pragma unroll
          for (int j = 0; j < TN; ++j)
            acc[i][j] = __fadd_rn(acc[i][j], __fmul_rn(x, bs[j * TX * LD + kk]));
        }
      }
    }
  }
  cp_async_wait<0>();
  if (kPdl) mm_pdl_release();
  if (res != nullptr) {
    // a following vector_add(out, res -> out) fused into the store:
    // fl(acc + res[g]), the add's own arithmetic on the value the matmul
    // would have stored (runs.cu).  All of the tile's residual loads go out
    // before any is used (one memory round trip, not one per cell).
    float rv[TM][TN];
#pragma unroll
    for (int i = 0; i < TM; ++i)
#pragma unroll
      for (int j = 0; j < TN; ++j) {
        const int r = bm + ty + TY * i, c = bn + tx + TX * j;
        const uint64_t g = (uint64_t)r * m + c;
        rv[i][j] = (r < n && c < m && g < res_cov) ? __ldg(res + g) : 0.0f;
      }
#pragma unroll
    for (int i = 0; i < TM; ++i) {
      const int r = bm + ty + TY * i;
      if (r >= n) continue;
#pragma unroll
      for (int j = 0; j < TN; ++j) {
        const int c = bn + tx + TX * j;
        if (c >= m) continue;
        const uint64_t g = (uint64_t)r * m + c;
        if (g < cov) out[g] = g < res_cov ? __fadd_rn(acc[i][j], rv[i][j]) : acc[i][j];
      }
    }
    return;
  }
#pragma unroll
  for (int i = 0; i < TM; ++i) {
    const int r = bm + ty + TY * i;
    if (r >= n) continue;
#pragma unroll
    for (int j = 0; j < TN; ++j) {
      const int c = bn + tx + TX * j;
      if (c >= m) continue;
      const uint64_t g = (uint64_t)r * m + c;
      if (g < cov) out[g] = acc[i][j];
    }
  }
}


}  // namespace kaas
