// Persistent invocation-run kernel: a run of consecutive builtin invocations
// of one request (matmul, vector_add, saxpy, fill, reduce_sum -- e.g. the
// 102 invocations of a ResNet-50-shaped chain, BASELINE configs[4]) executes
// as ONE cooperative launch instead of one launch per invocation.
//
// Reference semantics (backend.py:258-266, executor.py:356-369): invocations
// run one after another, each seeing every earlier invocation's writes.  Here
// every invocation becomes one or more tasks (a matmul may add a transpose of
// B and, when its output aliases an input, two copies through a temporary);
// one CTA per SM walks the task list in order and runs the task's work items
// that map to it (item i -> CTA (i + rot) % G), so independent consecutive
// tasks overlap.  Ordering is by dependency counters, not grid barriers: the
// host finds, for each task, the latest earlier task it conflicts with (RAW,
// WAR or WAW on a buffer) and the CTAs wait for that task's counter.  Every
// CTA arrives on a waited-for task after finishing its items of it, and CTAs
// walk tasks in order, so "all CTAs arrived on task w" means every task <= w
// is complete -- one counter covers all of a task's dependencies.
//
// The arithmetic is exactly the per-invocation kernels' (mm_tile.cuh for the
// bit-exact matmul tiles; separately rounded adds/multiplies elsewhere), so
// results are bit-identical to the per-launch path and to the reference.
#include "kaas_internal.cuh"
#include "mm_tile.cuh"

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <atomic>
#include <unordered_map>
#include <vector>

namespace kaas {
namespace {

constexpr int kRunThreads = 256;
constexpr int kRunMaxTasks = 128;       // per launch (kernel parameter space)
constexpr uint64_t kEltItem = 2048;    // elements per elementwise work item (2 float4 per thread)
constexpr uint64_t kCopyItem = 32768;  // bytes per copy work item (8 x 16 bytes per thread)

// R_ADDC: a fill(v) of a buffer followed by vector_add(x, that buffer -> that
// buffer) over the same elements, as one pass: out = fl(x + v)
enum : uint8_t { R_MM = 0, R_ADD, R_SAXPY, R_FILL, R_REDUCE, R_TRANSPOSE, R_COPY, R_ADDC };

struct RunTask {
  uint8_t op, cfg, arrive, vec;  // vec: 16-byte aligned operands (elementwise, copy)
  uint32_t per;     // matmul: tiles per work item (one per thread group of the CTA)
  int32_t wait;     // task whose counter must reach its target first (-1: none)
  uint32_t target;  // this task's counter once every CTA has arrived on it
  uint32_t items, rot;
  uint32_t n, m, k;  // matmul extents; transpose: k rows x m columns of B
  float a;           // saxpy a / fill value (rounded to f32 once, on the host)
  uint64_t cov;      // elements (elementwise, reduce), cells (matmul), bytes (copy)
  const float *x, *y;
  float *out;
  const float *res;  // matmul: fused residual add (out = fl(acc + res)) for cells < res_cov, or null
  uint64_t res_cov;
};

struct RunParams {
  unsigned *done;
  unsigned *trace;  // dev build: [task][cta][2] globaltimer stamps (start, end), else null
  int n_tasks;
  int pad;
  RunTask t[kRunMaxTasks];
};

__device__ __forceinline__ unsigned run_gtimer() {
  unsigned t;
  asm volatile("mov.u32 %0, %%globaltimer_lo;" : "=r"(t));
  return t;
}

// ---- matmul tile configurations --------------------------------------------
// A tile is computed by a group of TY x TX threads; groups smaller than the
// CTA run side by side (named barriers, their own slice of shared memory).
// Stage-3/4 ResNet layers have only 170-680 output cells per SM, and a
// thread's operand traffic (TM + TN words per k) is what binds them: shared
// memory returns ~3 cycles per LDS.128 warp instruction per SM
// (tools/mmchain.cu), so the small layers want 2 x 2 cells per thread in
// small groups rather than 1 x 1 cells over the whole CTA.
struct MmCfg {
  int ty, tx, tm, tn, s, bk;
};
constexpr MmCfg kCfgs[] = {
    {16, 16, 4, 4, 4, 32},  // 0: 64 x 64, 256 threads
    {16, 16, 2, 4, 4, 32},  // 1: 32 x 64
    {16, 16, 4, 2, 4, 32},  // 2: 64 x 32
    {16, 16, 2, 2, 3, 64},  // 3: 32 x 32
    {16, 16, 1, 2, 3, 64},  // 4: 16 x 32
    {16, 16, 2, 1, 3, 64},  // 5: 32 x 16
    {16, 16, 1, 1, 3, 64},  // 6: 16 x 16
    {64, 4, 1, 1, 3, 64},  // 7: 64 x 4
    {16, 8, 1, 2, 3, 64},  // 8: 16 x 16, 128 threads
    {8, 16, 2, 2, 3, 64},  // 9: 16 x 32
    {16, 8, 2, 2, 3, 64},  // 10: 32 x 16
    {32, 4, 2, 1, 3, 64},  // 11: 64 x 4
    {8, 8, 2, 2, 3, 64},  // 12: 16 x 16, 64 threads
    {4, 16, 2, 2, 3, 64},  // 13: 8 x 32
    {16, 4, 2, 2, 3, 64},  // 14: 32 x 8
    {32, 2, 2, 2, 2, 64},  // 15: 64 x 4
    {1, 64, 1, 4, 2, 32},  // 16: 1 x 256 (single-row outputs: fc)
    {1, 256, 1, 1, 2, 32},  // 17: 1 x 256, 256 threads
};
constexpr int kNumCfgs = (int)(sizeof(kCfgs) / sizeof(kCfgs[0]));
constexpr int kRunSmem = 200 * 1024;

constexpr int cfg_threads(const MmCfg &c) { return c.ty * c.tx; }
constexpr int cfg_smem(const MmCfg &c) { return c.s * (c.ty * c.tm + c.tx * c.tn) * (c.bk + 4) * 4; }
// thread groups of this configuration one CTA runs side by side
constexpr int cfg_groups(const MmCfg &c) {
  const int by_threads = kRunThreads / cfg_threads(c), by_smem = kRunSmem / cfg_smem(c);
  return by_threads < by_smem ? by_threads : by_smem;
}
constexpr bool cfgs_ok() {
  for (const MmCfg &c : kCfgs)
    if (kRunThreads % cfg_threads(c) != 0 || cfg_threads(c) % 32 != 0 || cfg_groups(c) < 1) return false;
  return 32 * 33 * 4 <= kRunSmem;  // transpose tile
}
static_assert(cfgs_ok(), "matmul tile configurations must fit the run kernel's CTA");

template <int C>
__device__ __forceinline__ void run_mm(const RunTask &T, unsigned i, float *smem, unsigned tid) {
  constexpr MmCfg c = kCfgs[C];
  constexpr int NT = cfg_threads(c), BM = c.ty * c.tm, BN = c.tx * c.tn;
  const unsigned g = tid / NT;
  const unsigned gx = (T.m + BN - 1) / BN, tiles = gx * ((T.n + BM - 1) / BM);
  const unsigned tile = i * T.per + g;
  if (g >= T.per || tile >= tiles) return;
  const int bm = (int)(tile / gx) * BM, bn = (int)(tile % gx) * BN;
  float *sm = smem + g * (cfg_smem(c) / 4);
  const int bar = NT == kRunThreads ? 0 : (int)(1 + g);
  mm_tile<c.ty, c.tx, c.tm, c.tn, c.s, c.bk, true, true, false>((int)T.n, (int)T.m, (int)T.k, T.cov, T.x, T.y, T.out,
                                                                bm, bn, sm, (int)(tid % NT), bar, T.res, T.res_cov);
}

__device__ __forceinline__ unsigned ld_acquire_u32(const unsigned *p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ float elt(uint8_t op, float a, float x, float y) {
  return op == R_ADD ? __fadd_rn(x, y) : op == R_SAXPY ? __fadd_rn(__fmul_rn(a, x), y) : op == R_ADDC ? __fadd_rn(x, a) : a;
}

__global__ void __launch_bounds__(kRunThreads, 1) k_run(const __grid_constant__ RunParams p) {
  extern __shared__ __align__(16) float run_smem[];
  const unsigned G = gridDim.x, b = blockIdx.x, tid = threadIdx.x;
  for (int t = 0; t < p.n_tasks; ++t) {
    const RunTask &T = p.t[t];
    if (T.wait >= 0) {
      if (tid == 0) {
        const unsigned want = p.t[T.wait].target;
        unsigned spins = 0;
        while ((int)(ld_acquire_u32(p.done + T.wait) - want) < 0)
          if (++spins > (1u << 26)) __trap();  // a lost CTA: fail loudly, never hang
      }
      __syncthreads();
    }
#ifdef KAAS_DEV
    if (p.trace && tid == 0) p.trace[((size_t)t * G + b) * 2] = run_gtimer();
#endif
    for (unsigned i = (b + G - T.rot) % G; i < T.items; i += G) {
      __syncthreads();  // the previous item's shared-memory readers are done
      switch (T.op) {
        case R_MM:
          switch (T.cfg) {
            case 0: run_mm<0>(T, i, run_smem, tid); break;
            case 1: run_mm<1>(T, i, run_smem, tid); break;
            case 2: run_mm<2>(T, i, run_smem, tid); break;
            case 3: run_mm<3>(T, i, run_smem, tid); break;
            case 4: run_mm<4>(T, i, run_smem, tid); break;
            case 5: run_mm<5>(T, i, run_smem, tid); break;
            case 6: run_mm<6>(T, i, run_smem, tid); break;
            case 7: run_mm<7>(T, i, run_smem, tid); break;
            case 8: run_mm<8>(T, i, run_smem, tid); break;
            case 9: run_mm<9>(T, i, run_smem, tid); break;
            case 10: run_mm<10>(T, i, run_smem, tid); break;
            case 11: run_mm<11>(T, i, run_smem, tid); break;
            case 12: run_mm<12>(T, i, run_smem, tid); break;
            case 13: run_mm<13>(T, i, run_smem, tid); break;
            case 14: run_mm<14>(T, i, run_smem, tid); break;
            case 15: run_mm<15>(T, i, run_smem, tid); break;
            case 16: run_mm<16>(T, i, run_smem, tid); break;
            default: run_mm<17>(T, i, run_smem, tid); break;
          }
          break;
        case R_ADD:
        case R_SAXPY:
        case R_ADDC:
        case R_FILL: {
          // exact aliasing (out == x or y) is safe: each element is read and
          // then written by the same thread.  All of a thread's loads are
          // issued before its stores (one memory round trip per item).
          const uint64_t e0 = (uint64_t)i * kEltItem, e1 = min(e0 + kEltItem, T.cov);
          uint64_t e = e0;
          if (T.vec) {
            constexpr int U = (int)(kEltItem / 4 / kRunThreads);
            const uint64_t q1 = e1 / 4;
            float4 xv[U], yv[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
              const uint64_t q = e0 / 4 + tid + (uint64_t)u * kRunThreads;
              if (q < q1 && T.op != R_FILL) {
                xv[u] = reinterpret_cast<const float4 *>(T.x)[q];
                yv[u] = T.op == R_ADDC ? xv[u] : reinterpret_cast<const float4 *>(T.y)[q];
              }
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
              const uint64_t q = e0 / 4 + tid + (uint64_t)u * kRunThreads;
              if (q >= q1) continue;
              float4 r;
              if (T.op == R_FILL)
                r = make_float4(T.a, T.a, T.a, T.a);
              else
                r = make_float4(elt(T.op, T.a, xv[u].x, yv[u].x), elt(T.op, T.a, xv[u].y, yv[u].y),
                                elt(T.op, T.a, xv[u].z, yv[u].z), elt(T.op, T.a, xv[u].w, yv[u].w));
              reinterpret_cast<float4 *>(T.out)[q] = r;
            }
            e = q1 * 4;
          }
          for (e += tid; e < e1; e += kRunThreads)
            T.out[e] = T.op == R_FILL ? T.a : elt(T.op, T.a, T.x[e], T.op == R_ADDC ? 0.f : T.y[e]);
          break;
        }
        case R_REDUCE:
          // np.add.accumulate(x)[-1]: one serial f32 chain seeded with x[0]
          // (backend.py:192-202); out is written after every read
          if (tid == 0) {
            const uint64_t n = T.cov;
            float acc = 0.0f;
            if (n > 0) {
              acc = T.x[0];
              uint64_t j = 1;
              for (; j + 16 <= n; j += 16) {
                float v[16];
#pragma unroll
                for (int u = 0; u < 16; ++u) v[u] = T.x[j + u];
#pragma unroll
                for (int u = 0; u < 16; ++u) acc = __fadd_rn(acc, v[u]);
              }
              for (; j < n; ++j) acc = __fadd_rn(acc, T.x[j]);
            }
            *T.out = acc;
          }
          break;
        case R_TRANSPOSE: {
          // B [k][m] -> Bt [m][k], one 32 x 32 tile per item
          float(*tile)[33] = reinterpret_cast<float(*)[33]>(run_smem);
          const unsigned tiles_m = (T.m + 31) / 32;
          const unsigned c0 = (i % tiles_m) * 32, r0 = (i / tiles_m) * 32;
          const unsigned tx = tid & 31, ty = tid >> 5;
          for (unsigned q = ty; q < 32; q += kRunThreads / 32) {
            const unsigned r = r0 + q, c = c0 + tx;
            if (r < T.k && c < T.m) tile[q][tx] = T.x[(size_t)r * T.m + c];
          }
          __syncthreads();
          for (unsigned q = ty; q < 32; q += kRunThreads / 32) {
            const unsigned c = c0 + q, r = r0 + tx;
            if (r < T.k && c < T.m) T.out[(size_t)c * T.k + r] = tile[tx][q];
          }
          break;
        }
        case R_COPY: {
          const uint64_t e0 = (uint64_t)i * kCopyItem, e1 = min(e0 + kCopyItem, T.cov);
          const unsigned char *src = reinterpret_cast<const unsigned char *>(T.x);
          unsigned char *dst = reinterpret_cast<unsigned char *>(T.out);
          uint64_t e = e0;
          if (T.vec) {
            constexpr int U = (int)(kCopyItem / 16 / kRunThreads);
            const uint64_t q1 = e1 / 16;
            uint4 v[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
              const uint64_t q = e0 / 16 + tid + (uint64_t)u * kRunThreads;
              if (q < q1) v[u] = reinterpret_cast<const uint4 *>(src)[q];
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
              const uint64_t q = e0 / 16 + tid + (uint64_t)u * kRunThreads;
              if (q < q1) reinterpret_cast<uint4 *>(dst)[q] = v[u];
            }
            e = q1 * 16;
          }
          for (e += tid; e < e1; e += kRunThreads) dst[e] = src[e];
          break;
        }
      }
    }
#ifdef KAAS_DEV
    if (p.trace) {
      __syncthreads();
      if (tid == 0) p.trace[((size_t)t * G + b) * 2 + 1] = run_gtimer();
    }
#endif
    if (T.arrive) {
      __syncthreads();  // every thread's writes of this task precede the arrival
      if (tid == 0)  // release: cumulative over the CTA's writes ordered by the bar.sync
        asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(p.done + t) : "memory");
    }
  }
}

// Pick the tile configuration and tiles per work item with the lowest
// modelled time: waves of work items over the grid x (k x cycles per k + a
// per-tile fixed cost).  Cycles per k depend on how many threads of the SM
// run tiles and on the cells per thread; the table is measured on B200
// (tools/mmchain2.cu, tools/run_cfg_sweep.py over the ResNet-50 shapes): the
// serial FADD chain (~4.1 cycles), shared-memory operand returns (~3 cycles
// per LDS.128 warp instruction per SM) and FMUL/FADD issue (~0.5 warp
// instructions per cycle for a lone warp) interact too much for a formula.
struct Pick {
  int cfg, per;
};
double cycles_per_k(int threads, int cells) {
  static const double tab[3][5] = {
      // cells per thread: 1, 2, 4, 8, 16
      {6.0, 12.0, 19.0, 30.0, 50.0},   // 64 threads per SM
      {7.4, 16.0, 21.6, 44.7, 66.0},   // 128
      {18.0, 27.5, 35.0, 62.0, 105.0}  // 256
  };
  const int ti = threads <= 64 ? 0 : threads <= 128 ? 1 : 2;
  int ci = 0;
  while ((1 << ci) < cells && ci < 4) ++ci;
  return tab[ti][ci];
}
Pick pick_cfg(uint64_t n, uint64_t m, uint64_t k, int grid) {
  Pick best{0, 1};
  double best_t = 1e300;
  for (int c = 0; c < kNumCfgs; ++c) {
    const MmCfg &g = kCfgs[c];
    const uint64_t bm = (uint64_t)g.ty * g.tm, bn = (uint64_t)g.tx * g.tn;
    const uint64_t tiles = ((n + bm - 1) / bm) * ((m + bn - 1) / bn);
    if (tiles > 0xffffffffull) continue;
    for (int per = 1; per <= cfg_groups(g); ++per) {
      const uint64_t items = (tiles + per - 1) / per;
      if (per > 1 && items * (uint64_t)per - tiles >= (uint64_t)per) continue;
      const double waves = (double)((items + grid - 1) / grid);
      const double t = waves * ((double)k * cycles_per_k(per * cfg_threads(g), g.tm * g.tn) + 2000.0);
      if (t < best_t * 0.98) {
        best_t = t;
        best = Pick{c, per};
      }
    }
  }
  return best;
}

#ifdef KAAS_DEV
unsigned *g_run_trace = nullptr;  // last traced launch (dev build, KAAS_RUN_TRACE=1)
std::vector<RunTask> g_run_tasks;
int g_run_grid = 0;
#endif

}  // namespace

bool run_eligible(const RunInv &v) {
  switch (v.kernel) {
    case KAAS_K_VECTOR_ADD:
    case KAAS_K_SAXPY:
    case KAAS_K_FILL:
    case KAAS_K_REDUCE_SUM:
      return true;
    case KAAS_K_MATMUL:
      // the run kernel's tiles read A 16 bytes at a time and B transposed
      return v.ext[2] > 0 && v.ext[2] % 4 == 0 && (v.ptr[0] & 15) == 0 && v.ext[0] <= 0x7fffffffu &&
             v.ext[1] <= 0x7fffffffu && v.ext[2] <= 0x7fffffffu;
    default:
      return false;
  }
}

int launch_builtin_run(cudaStream_t s, int dev, StreamScratch *sc, const RunInv *v, int n_inv) {
  const int G = device_props(dev).sm_count;
  // ---- pass 1: scratch for transposed B (no prepared copy) and alias temporaries
  auto align256 = [](uint64_t x) { return (x + 255) & ~uint64_t(255); };
  uint64_t scratch = 0;
  for (int i = 0; i < n_inv; ++i) {
    const RunInv &q = v[i];
    if (q.kernel != KAAS_K_MATMUL) continue;
    const uint64_t nn = q.ext[0], m = q.ext[1], k = q.ext[2];
    if (q.flags & (KAAS_F_MM_BT_USE | KAAS_F_MM_BT_FILL)) {
      if (q.size[3] < m * k * 4) return fail(KAAS_E_BOUNDS, "matmul: prepared B buffer too small");
    } else if (nn && m && q.cov) {
      scratch += align256(m * k * 4);
    }
    if (nn && m && q.cov && (q.ptr[2] == q.ptr[0] || q.ptr[2] == q.ptr[1])) scratch += align256(q.cov * 4);
  }
  if (scratch) {
    int rc = ensure_matmul_scratch(sc, s, scratch);
    if (rc) return rc;
  }
  uint64_t scr = (uint64_t)sc->mm_buf;

  // ---- pass 2: tasks with their buffer footprints
  struct Foot {
    uint64_t r[3], w;  // base pointers read / written (0: none)
  };
  std::vector<RunTask> tasks;
  std::vector<Foot> feet;
  tasks.reserve((size_t)n_inv * 2);
  feet.reserve((size_t)n_inv * 2);
  auto add = [&](RunTask t, uint64_t r0, uint64_t r1, uint64_t w, uint64_t r2 = 0) {
    tasks.push_back(t);
    feet.push_back(Foot{{r0, r1, r2}, w});
  };
  auto aligned = [](uint64_t p) { return (p & 15) == 0; };
  // Peephole fusions (results bit-identical: the fused task performs the
  // second invocation's own rounding on exactly the values it would read):
  //  * fill(F, v) then vector_add(X, F -> F) over the same elements, X != F:
  //    one pass F = fl(X + v) (R_ADDC)
  //  * matmul(A, B -> D) then vector_add(D, S -> D) (either operand order)
  //    over elements the matmul covers, S != D: fl(acc + S) in the matmul's
  //    store (a ResNet block's residual add)
  auto fused_add = [&](int i, uint64_t dst) -> const RunInv * {
    if (i + 1 >= n_inv) return nullptr;
    const RunInv &a = v[i + 1];
    if (a.kernel != KAAS_K_VECTOR_ADD || a.cov == 0 || a.ptr[2] != dst) return nullptr;
    if ((a.ptr[0] == dst) == (a.ptr[1] == dst)) return nullptr;  // exactly one operand is dst
    return &a;
  };
  for (int i = 0; i < n_inv; ++i) {
    const RunInv &q = v[i];
    RunTask t{};
    t.wait = -1;
    switch (q.kernel) {
      case KAAS_K_VECTOR_ADD:
      case KAAS_K_SAXPY:
      case KAAS_K_FILL: {
        if (q.cov == 0) break;
        if (q.kernel == KAAS_K_FILL) {
          const RunInv *a = fused_add(i, q.ptr[0]);
          if (a != nullptr && a->cov == q.cov) {
            const uint64_t x = a->ptr[0] == q.ptr[0] ? a->ptr[1] : a->ptr[0];
            t.op = R_ADDC;
            t.cov = q.cov;
            t.a = q.fval;
            t.out = (float *)q.ptr[0];
            t.x = (const float *)x;
            t.y = nullptr;
            t.vec = aligned((uint64_t)t.out) && aligned(x);
            t.items = (uint32_t)((q.cov + kEltItem - 1) / kEltItem);
            add(t, x, 0, (uint64_t)t.out);
            ++i;  // the add is done
            break;
          }
        }
        const bool fill = q.kernel == KAAS_K_FILL;
        t.op = q.kernel == KAAS_K_VECTOR_ADD ? R_ADD : q.kernel == KAAS_K_SAXPY ? R_SAXPY : R_FILL;
        t.cov = q.cov;
        t.a = q.fval;
        t.out = (float *)(fill ? q.ptr[0] : q.ptr[2]);
        t.x = fill ? nullptr : (const float *)q.ptr[0];
        t.y = fill ? nullptr : (const float *)q.ptr[1];
        t.vec = aligned((uint64_t)t.out) && (fill || (aligned(q.ptr[0]) && aligned(q.ptr[1])));
        t.items = (uint32_t)((q.cov + kEltItem - 1) / kEltItem);
        add(t, fill ? 0 : q.ptr[0], fill ? 0 : q.ptr[1], (uint64_t)t.out);
        break;
      }
      case KAAS_K_REDUCE_SUM:
        t.op = R_REDUCE;
        t.cov = q.ext[0];
        t.x = (const float *)q.ptr[0];
        t.out = (float *)q.ptr[1];
        t.items = 1;
        add(t, q.ptr[0], 0, q.ptr[1]);
        break;
      case KAAS_K_MATMUL: {
        const uint64_t nn = q.ext[0], m = q.ext[1], k = q.ext[2];
        const bool work = nn && m && q.cov;
        uint64_t bt = 0;
        bool need_t = false;
        if (q.flags & (KAAS_F_MM_BT_USE | KAAS_F_MM_BT_FILL)) {
          bt = q.ptr[3];
          // a prepared buffer the executor asked to fill is always filled
          // (later launches trust it), whether or not this launch reads it
          need_t = (q.flags & KAAS_F_MM_BT_USE) == 0;
        } else if (work) {
          bt = scr;
          scr += align256(m * k * 4);
          need_t = true;
        }
        if (need_t && m) {
          RunTask tt{};
          tt.wait = -1;
          tt.op = R_TRANSPOSE;
          tt.k = (uint32_t)k;
          tt.m = (uint32_t)m;
          tt.x = (const float *)q.ptr[1];
          tt.out = (float *)bt;
          tt.items = (uint32_t)(((m + 31) / 32) * ((k + 31) / 32));
          add(tt, q.ptr[1], 0, bt);
        }
        if (!work) break;
        uint64_t out = q.ptr[2];
        uint64_t tmp = 0;
        if (out == q.ptr[0] || out == q.ptr[1]) {
          // the reference reads every input before writing (backend.py:8-9):
          // write the covered cells to a temporary, then copy them over the
          // output (its bytes past the covered cells are never touched)
          tmp = scr;
          scr += align256(q.cov * 4);
        }
        t.op = R_MM;
        t.n = (uint32_t)nn;
        t.m = (uint32_t)m;
        t.k = (uint32_t)k;
        t.cov = q.cov;
        t.x = (const float *)q.ptr[0];
        t.y = (const float *)bt;
        t.out = (float *)(tmp ? tmp : out);
        {
          Pick pk = pick_cfg(nn, m, k, G);
          if (const char *fc = KAAS_DEV_ENV("KAAS_RUN_CFG")) {  // dev: force "cfg,per" (tools/run_cfg_sweep.py)
            int c = -1, per = 1;
            if (sscanf(fc, "%d,%d", &c, &per) == 2 && c >= 0 && c < kNumCfgs && per >= 1 &&
                per <= cfg_groups(kCfgs[c]))
              pk = Pick{c, per};
          }
          const MmCfg &g = kCfgs[pk.cfg];
          const uint64_t bm = (uint64_t)g.ty * g.tm, bn = (uint64_t)g.tx * g.tn;
          const uint64_t tiles = ((nn + bm - 1) / bm) * ((m + bn - 1) / bn);
          t.cfg = (uint8_t)pk.cfg;
          t.per = (uint32_t)pk.per;
          t.items = (uint32_t)((tiles + pk.per - 1) / pk.per);
        }
        if (!tmp) {
          const RunInv *a = fused_add(i, out);
          if (a != nullptr && a->cov <= q.cov) {
            t.res = (const float *)(a->ptr[0] == out ? a->ptr[1] : a->ptr[0]);
            t.res_cov = a->cov;
          }
        }
        add(t, q.ptr[0], (uint64_t)t.y, (uint64_t)t.out, (uint64_t)t.res);
        if (t.res) ++i;  // the residual add is done
        if (tmp) {
          RunTask c{};
          c.wait = -1;
          c.op = R_COPY;
          c.cov = q.cov * 4;
          c.x = (const float *)tmp;
          c.out = (float *)out;
          c.vec = aligned(out);
          c.items = (uint32_t)((c.cov + kCopyItem - 1) / kCopyItem);
          add(c, tmp, 0, out);
        }
        break;
      }
      default:
        return fail(KAAS_E_INVALID, "invocation run: kernel is not a builtin");
    }
  }
  if (tasks.empty()) return 0;

  // ---- per-stream arrival counters (monotonic: +G per launch per arriving task)
  if (!sc->run_done) {
    KAAS_CUDA(cudaMallocAsync((void **)&sc->run_done, kRunMaxTasks * sizeof(unsigned), s));
    KAAS_CUDA(cudaMemsetAsync(sc->run_done, 0, kRunMaxTasks * sizeof(unsigned), s));
    sc->run_expect.assign(kRunMaxTasks, 0u);
  }

  // ---- launches of <= kRunMaxTasks tasks; dependencies within a launch
  // (everything of an earlier launch is complete when the next one starts)
  static thread_local RunParams p;
  const int smem = kRunSmem;
  {
    static std::atomic<uint64_t> attr_done{0};
    if (!(attr_done.load(std::memory_order_relaxed) >> (dev & 63) & 1)) {
      KAAS_CUDA(cudaFuncSetAttribute(k_run, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
      attr_done.fetch_or(1ull << (dev & 63));
    }
  }
  std::unordered_map<uint64_t, std::pair<int, int>> state;  // base -> (last writer, last reader since)
  for (size_t base = 0; base < tasks.size(); base += kRunMaxTasks) {
    const int cnt = (int)std::min<size_t>(kRunMaxTasks, tasks.size() - base);
    state.clear();
    uint32_t rot = 0;
    for (int j = 0; j < cnt; ++j) {
      RunTask &t = tasks[base + j];
      const Foot &f = feet[base + j];
      int wait = -1;
      for (uint64_t r : f.r) {
        if (!r) continue;
        auto it = state.find(r);
        if (it != state.end()) wait = std::max(wait, it->second.first);
      }
      if (f.w) {
        auto it = state.find(f.w);
        if (it != state.end()) wait = std::max(wait, std::max(it->second.first, it->second.second));
      }
      for (uint64_t r : f.r) {
        if (!r) continue;
        auto &st = state.emplace(r, std::make_pair(-1, -1)).first->second;
        st.second = std::max(st.second, j);
      }
      if (f.w) state[f.w] = std::make_pair(j, -1);
      t.wait = wait;
      t.arrive = 0;
      if (wait >= 0) tasks[base + wait].arrive = 1;
      t.rot = rot % (uint32_t)G;
      rot = (uint32_t)((rot + t.items) % (uint32_t)G);
    }
    // counter wrap: start over from zero (stream-ordered)
    bool wrap = false;
    for (int j = 0; j < cnt; ++j)
      if (tasks[base + j].arrive && sc->run_expect[j] > 0xf0000000u) wrap = true;
    if (wrap) {
      KAAS_CUDA(cudaMemsetAsync(sc->run_done, 0, kRunMaxTasks * sizeof(unsigned), s));
      std::fill(sc->run_expect.begin(), sc->run_expect.end(), 0u);
    }
    for (int j = 0; j < cnt; ++j) {
      RunTask &t = tasks[base + j];
      if (t.arrive) {
        sc->run_expect[j] += (uint32_t)G;
        t.target = sc->run_expect[j];
      }
      p.t[j] = t;
    }
    p.done = sc->run_done;
    p.trace = nullptr;
#ifdef KAAS_DEV
    if (KAAS_DEV_ENV("KAAS_RUN_TRACE")) {
      if (!g_run_trace) KAAS_CUDA(cudaMalloc(&g_run_trace, (size_t)kRunMaxTasks * 1024 * 2 * 4));
      p.trace = g_run_trace;
      g_run_tasks.assign(p.t, p.t + cnt);
      g_run_grid = G;
    }
#endif
    p.n_tasks = cnt;
    void *args[] = {(void *)&p};
    KAAS_CUDA(cudaLaunchCooperativeKernel((const void *)k_run, dim3(G), dim3(kRunThreads), args, smem, s));
    count_launch();
  }
  return 0;
}

}  // namespace kaas

#ifdef KAAS_DEV
// dev build only (not in include/kaas_b200.h): the last traced run launch --
// its task table (op, cfg, wait, items, n, m, k per task) and per-CTA
// (start, end) globaltimer stamps; tools/rtrace.py
extern "C" int kaas_dev_run_trace(int *meta, unsigned long meta_len, unsigned *stamps, unsigned long stamps_len,
                                  int *n_tasks, int *grid) {
  using namespace kaas;
  const int n = (int)g_run_tasks.size();
  *n_tasks = n;
  *grid = g_run_grid;
  if (!g_run_trace || n == 0) return 1;
  for (int t = 0; t < n && (unsigned long)(t * 7 + 6) < meta_len; ++t) {
    const RunTask &r = g_run_tasks[t];
    int *m = meta + 7 * t;
    m[0] = r.op, m[1] = r.cfg, m[2] = r.wait, m[3] = (int)r.items, m[4] = (int)r.n, m[5] = (int)r.m, m[6] = (int)r.k;
  }
  unsigned long want = (unsigned long)n * g_run_grid * 2;
  if (want > stamps_len) want = stamps_len;
  return cudaMemcpy(stamps, g_run_trace, want * 4, cudaMemcpyDeviceToHost) == cudaSuccess ? 0 : 2;
}
#endif
