// All-to-all x exchange alone (dev tool): the Jacobi sweep's communication
// pattern without the arithmetic.  148 CTAs x 256 threads; each sweep every
// CTA publishes its 28 rows as (value, tag) words and every lane polls its
// 16 words (4 chunks x 4) until the tags of this sweep are seen.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/xchg tools/xchg.cu
//   ./tools/xchg [sweeps=2000]
//
// mode 0: per-lane polling of all 16 words (the kernel's scheme)
// (each mode also runs with a busy delay of D cycles per sweep standing in for compute)
// mode 1: polls with ld.global.cg (weak, L2) instead of ld.relaxed.gpu
// mode 2: mode 0 without the second bar.sync per sweep
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

constexpr int N = 4096, T = 256;

__device__ __forceinline__ ulonglong2 ld_rlx2(const unsigned long long *p) {
  ulonglong2 v;
  asm volatile("ld.relaxed.gpu.global.v2.u64 {%0, %1}, [%2];" : "=l"(v.x), "=l"(v.y) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ ulonglong2 ld_cg2(const unsigned long long *p) {
  ulonglong2 v;
  asm volatile("ld.global.cg.v2.u64 {%0, %1}, [%2];" : "=l"(v.x), "=l"(v.y) : "l"(p) : "memory");
  return v;
}
struct W4 {
  unsigned long long w[4];
};
__device__ __forceinline__ W4 ld_rlx4(const unsigned long long *p) {
  W4 v;
  asm volatile("ld.relaxed.gpu.global.v4.u64 {%0, %1, %2, %3}, [%4];"
               : "=l"(v.w[0]), "=l"(v.w[1]), "=l"(v.w[2]), "=l"(v.w[3])
               : "l"(p)
               : "memory");
  return v;
}
__device__ __forceinline__ unsigned ld_rlx_u32(const unsigned *p) {
  unsigned v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_rlx_u32(unsigned *p, unsigned v) {
  asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void st_rlx(unsigned long long *p, unsigned long long v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

template <int MODE, int REP = 1, int NCH = 4>
__global__ void __launch_bounds__(T, 1) xchg(unsigned long long *xt, int sweeps, int delay, unsigned tag0,
                                              float *sink) {
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int G = gridDim.x;
  const int r0 = (int)((long long)blockIdx.x * N / G), r1 = (int)((long long)(blockIdx.x + 1) * N / G);
  const int cbase = warp * 128 + lane;
  float acc = 0.f;
  for (int s = 0; s < sweeps; ++s) {
    const unsigned want = tag0 + s;
    // REP replicas of the tagged buffer: CTA b polls replica b % REP, so each
    // L2 line is polled by ~148 / REP CTAs instead of all of them
    const unsigned long long *src = xt + ((size_t)(s & 1) * REP + blockIdx.x % REP) * N;
    if (s > 0) {
      unsigned pending = (1u << NCH) - 1u;
      ulonglong2 q[4][2];
      unsigned spins = 0;
      while (pending) {
        if (++spins > (1u << 24)) __trap();  // never hang the box
#pragma unroll
        for (int u = 0; u < 4; ++u)
          if (pending & (1u << u)) {
            if (MODE == 1) {
              q[u][0] = ld_cg2(src + 4 * (cbase + 32 * u));
              q[u][1] = ld_cg2(src + 4 * (cbase + 32 * u) + 2);
            } else {
              q[u][0] = ld_rlx2(src + 4 * (cbase + 32 * u));
              q[u][1] = ld_rlx2(src + 4 * (cbase + 32 * u) + 2);
            }
          }
#pragma unroll
        for (int u = 0; u < 4; ++u)
          if ((pending & (1u << u)) && (unsigned)(q[u][0].x >> 32) == want && (unsigned)(q[u][0].y >> 32) == want &&
              (unsigned)(q[u][1].x >> 32) == want && (unsigned)(q[u][1].y >> 32) == want)
            pending &= ~(1u << u);
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) acc += __uint_as_float((unsigned)q[u][0].x) + __uint_as_float((unsigned)q[u][1].y);
    }
    if (delay) {
      const long long t = clock64();
      while (clock64() - t < delay) {
      }
    }
    __syncthreads();
    if (warp == 0) {
      const unsigned long long w = ((unsigned long long)(want + 1) << 32) | __float_as_uint(acc);
      for (int row = r0 + lane; row < r1; row += 32)
#pragma unroll
        for (int r = 0; r < REP; ++r) st_rlx(xt + ((size_t)((s + 1) & 1) * REP + r) * N + row, w);
    }
    if (MODE != 2) __syncthreads();
  }
  if (acc == 1234.5f) *sink = acc;
}


// MODE 10: each lane polls its 4 chunks with one 256-bit load each (the
//          kernel's scheme today)
// MODE 11: warp 0 polls one relaxed flag per producer CTA (~600 B per round
//          instead of 32 KB), bar.sync, then every lane loads its chunks once
//          and re-polls only words whose tag is still stale
template <int MODE>
__global__ void __launch_bounds__(T, 1) xchg2(unsigned long long *xt, unsigned *flags, int sweeps, unsigned tag0,
                                               float *sink) {
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int G = gridDim.x;
  const int r0 = (int)((long long)blockIdx.x * N / G), r1 = (int)((long long)(blockIdx.x + 1) * N / G);
  const int cbase = warp * 128 + lane;
  float acc = 0.f;
  for (int s = 0; s < sweeps; ++s) {
    const unsigned want = tag0 + s;
    const unsigned long long *src = xt + (size_t)(s & 1) * N;
    if (s > 0) {
      if (MODE == 11) {
        if (warp == 0) {  // each lane's <= 5 producer flags, all polled per round
          unsigned spins = 0;
          unsigned pend = 0;
#pragma unroll
          for (int j = 0; j < 5; ++j)
            if (lane + 32 * j < G) pend |= 1u << j;
          while (pend) {
            if (++spins > (1u << 24)) __trap();
            unsigned f[5];
#pragma unroll
            for (int j = 0; j < 5; ++j)
              if (pend & (1u << j)) f[j] = ld_rlx_u32(flags + lane + 32 * j);
#pragma unroll
            for (int j = 0; j < 5; ++j)
              if ((pend & (1u << j)) && (int)(f[j] - want) >= 0) pend &= ~(1u << j);
          }
        }
        __syncthreads();
      }
      unsigned pending = 0xf;
      W4 q[4];
      unsigned spins = 0;
      while (pending) {
        if (++spins > (1u << 24)) __trap();
#pragma unroll
        for (int u = 0; u < 4; ++u)
          if (pending & (1u << u)) q[u] = ld_rlx4(src + 4 * (cbase + 32 * u));
#pragma unroll
        for (int u = 0; u < 4; ++u)
          if ((pending & (1u << u)) && (unsigned)(q[u].w[0] >> 32) == want && (unsigned)(q[u].w[1] >> 32) == want &&
              (unsigned)(q[u].w[2] >> 32) == want && (unsigned)(q[u].w[3] >> 32) == want)
            pending &= ~(1u << u);
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) acc += __uint_as_float((unsigned)q[u].w[0]) + __uint_as_float((unsigned)q[u].w[3]);
    }
    __syncthreads();
    if (warp == 0) {
      const unsigned long long w = ((unsigned long long)(want + 1) << 32) | __float_as_uint(acc);
      for (int row = r0 + lane; row < r1; row += 32) st_rlx(xt + (size_t)((s + 1) & 1) * N + row, w);
      if (MODE == 11) {
        __syncwarp();
        if (lane == 0) st_rlx_u32(flags + blockIdx.x, want + 1);
      }
    }
    __syncthreads();
  }
  if (acc == 1234.5f) *sink = acc;
}

int main(int argc, char **argv) {
  const int sweeps = argc > 1 ? atoi(argv[1]) : 2000;
  int sms, clk;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  unsigned long long *xt;
  float *sink;
  cudaMalloc(&xt, 2 * 16 * N * 8);
  cudaMalloc(&sink, 4);
  cudaMemset(xt, 0, 2 * 16 * N * 8);
  unsigned tag = 1;
  unsigned *flags;
  cudaMalloc(&flags, 4096 * 4);
  cudaMemset(flags, 0, 4096 * 4);
  for (int mode = 10; mode <= 11; ++mode)
    for (int rep = 0; rep < 2; ++rep) {
      void *args[] = {&xt, &flags, (void *)&sweeps, &tag, &sink};
      cudaEvent_t a, b;
      cudaEventCreate(&a);
      cudaEventCreate(&b);
      cudaEventRecord(a);
      cudaLaunchCooperativeKernel(mode == 10 ? (void *)xchg2<10> : (void *)xchg2<11>, sms, T, args, 0, 0);
      cudaEventRecord(b);
      if (cudaEventSynchronize(b) != cudaSuccess) {
        printf("error\n");
        return 1;
      }
      tag += sweeps + 1;
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      printf("%s: %.3f us/sweep\n", mode == 10 ? "256-bit per-lane polls" : "flag poll + one data round", ms * 1e3 / sweeps);
    }
  void *kern[] = {(void *)xchg<0>, (void *)xchg<1>, (void *)xchg<2>, (void *)xchg<0, 2>, (void *)xchg<0, 4>,
                  (void *)xchg<0, 8>, (void *)xchg<0, 16>};
  const char *names[] = {"relaxed", "ld.cg", "1 bar", "2 replicas", "4 replicas", "8 replicas", "16 replicas"};
  {
    void *half = (void *)xchg<0, 1, 2>;
    int delay = 0;
    void *args[] = {&xt, (void *)&sweeps, &delay, &tag, &sink};
    cudaLaunchCooperativeKernel(half, sms, T, args, 0, 0);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    tag += sweeps + 1;
    cudaEventRecord(a);
    cudaLaunchCooperativeKernel(half, sms, T, args, 0, 0);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    tag += sweeps + 1;
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    printf("relaxed, %3d CTAs, each polling HALF of x (2048 words): %.3f us/sweep\n", sms, ms * 1e3 / sweeps);
  }
  const int grids[] = {sms, sms / 2, sms / 4, 16, 2};
  for (int gi = 0; gi < 5; ++gi) {
    const int g = grids[gi];
    int delay = 0;
    void *args[] = {&xt, (void *)&sweeps, &delay, &tag, &sink};
    cudaLaunchCooperativeKernel(kern[0], g, T, args, 0, 0);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    tag += sweeps + 1;
    cudaEventRecord(a);
    cudaLaunchCooperativeKernel(kern[0], g, T, args, 0, 0);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    tag += sweeps + 1;
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    printf("relaxed, %3d CTAs (all 4096 words each): %.3f us/sweep\n", g, ms * 1e3 / sweeps);
  }
  for (int mode = 0; mode < 7; ++mode)
  for (int delay : {0, 0, 1000}) {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a);
    void *args[] = {&xt, (void *)&sweeps, &delay, &tag, &sink};
    cudaLaunchCooperativeKernel(kern[mode], sms, T, args, 0, 0);
    cudaEventRecord(b);
    if (cudaEventSynchronize(b) != cudaSuccess) {
      printf("error\n");
      return 1;
    }
    tag += sweeps + 1;
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    printf("%-12s: exchange only, busy delay %4d cycles (%.0f ns): %.3f us/sweep\n", names[mode], delay, delay / (clk * 1e-6),
           ms * 1e3 / sweeps);
  }
  return 0;
}
