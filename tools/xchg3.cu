// Exchange-format probe (dev tool): the Jacobi sweep's all-to-all x exchange
// with a busy delay standing in for the arithmetic, comparing wire formats.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/xchg3 tools/xchg3.cu
//   ./tools/xchg3 [sweeps=2000]
//
// fmt 0: (value, tag) 8-byte words; each lane polls its 16 words (4 x 256-bit
//        loads) straight into registers -- the product kernel's scheme
// fmt 1: one 32-byte sector per 7 rows: 7 values + the tag, written by one
//        thread with a single 256-bit store; a CTA's 28 rows are one 128-byte
//        line.  Lanes poll the 592 sectors (<= 3 each), stage x in shared
//        memory, bar.sync, and read their 16 values back (4 x LDS.128)
// fmt 2: fmt 0's wire format staged through shared memory like fmt 1 (the
//        staging cost alone)
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

constexpr int N = 4096, T = 256;

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
__device__ __forceinline__ void st_rlx4(unsigned long long *p, const W4 &v) {
  asm volatile("st.relaxed.gpu.global.v4.u64 [%0], {%1, %2, %3, %4};" ::"l"(p), "l"(v.w[0]), "l"(v.w[1]),
               "l"(v.w[2]), "l"(v.w[3])
               : "memory");
}
__device__ __forceinline__ void st_rlx(unsigned long long *p, unsigned long long v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

__device__ __forceinline__ int band0(int b, int G) { return (int)((long long)b * N / G); }

template <int FMT>
__global__ void __launch_bounds__(T, 1) xchg3(unsigned long long *xt, int sweeps, int delay, unsigned tag0,
                                               float *sink) {
  __shared__ __align__(16) float xs[N];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int G = gridDim.x;
  const int r0 = band0(blockIdx.x, G), r1 = band0(blockIdx.x + 1, G);
  const int cbase = warp * 128 + lane;
  float acc = 0.f, mine = 0.f;
  for (int s = 0; s < sweeps; ++s) {
    const unsigned want = tag0 + s;
    float xr[16];
    if (s > 0) {
      if (FMT == 0 || FMT == 2) {
        const unsigned long long *src = xt + (size_t)(s & 1) * N;
        unsigned pending = 0xf, spins = 0;
        W4 q[4];
        while (pending) {
          if (++spins > (1u << 24)) __trap();
#pragma unroll
          for (int u = 0; u < 4; ++u)
            if (pending & (1u << u)) q[u] = ld_rlx4(src + 4 * (cbase + 32 * u));
#pragma unroll
          for (int u = 0; u < 4; ++u)
            if ((pending & (1u << u)) && (unsigned)(q[u].w[0] >> 32) == want &&
                (unsigned)(q[u].w[1] >> 32) == want && (unsigned)(q[u].w[2] >> 32) == want &&
                (unsigned)(q[u].w[3] >> 32) == want)
              pending &= ~(1u << u);
        }
        if (FMT == 0) {
#pragma unroll
          for (int u = 0; u < 4; ++u)
#pragma unroll
            for (int j = 0; j < 4; ++j) xr[4 * u + j] = __uint_as_float((unsigned)q[u].w[j]);
        } else {
#pragma unroll
          for (int u = 0; u < 4; ++u)
            *reinterpret_cast<float4 *>(&xs[4 * (cbase + 32 * u)]) =
                make_float4(__uint_as_float((unsigned)q[u].w[0]), __uint_as_float((unsigned)q[u].w[1]),
                            __uint_as_float((unsigned)q[u].w[2]), __uint_as_float((unsigned)q[u].w[3]));
          __syncthreads();
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const float4 v = *reinterpret_cast<const float4 *>(&xs[4 * (cbase + 32 * u)]);
            xr[4 * u] = v.x, xr[4 * u + 1] = v.y, xr[4 * u + 2] = v.z, xr[4 * u + 3] = v.w;
          }
        }
      } else {
        // sectors: line b (CTA b's rows) = 4 sectors; sector k holds rows
        // r0(b) + 7k .. + 6 in words 0..6 (low/high halves), tag in word 7
        const unsigned long long *src = xt + (size_t)(s & 1) * (G * 16);
        const int nsec = G * 4;
        unsigned pending = 0, spins = 0;
#pragma unroll
        for (int j = 0; j < 3; ++j)
          if (tid + T * j < nsec) pending |= 1u << j;
        W4 q[3];
        while (pending) {
          if (++spins > (1u << 24)) __trap();
#pragma unroll
          for (int j = 0; j < 3; ++j)
            if (pending & (1u << j)) q[j] = ld_rlx4(src + 4 * (tid + T * j));
#pragma unroll
          for (int j = 0; j < 3; ++j)
            if ((pending & (1u << j)) && (unsigned)(q[j].w[3] >> 32) == want) pending &= ~(1u << j);
        }
#pragma unroll
        for (int j = 0; j < 3; ++j) {
          const int sec = tid + T * j;
          if (sec < nsec) {
            const int b = sec >> 2, k = sec & 3;
            const int rb = band0(b, G), re = band0(b + 1, G);
            const int row = rb + 7 * k;
#pragma unroll
            for (int e = 0; e < 7; ++e) {
              const unsigned bits = (e & 1) ? (unsigned)(q[j].w[e >> 1] >> 32) : (unsigned)q[j].w[e >> 1];
              if (row + e < re) xs[row + e] = __uint_as_float(bits);
            }
          }
        }
        __syncthreads();
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const float4 v = *reinterpret_cast<const float4 *>(&xs[4 * (cbase + 32 * u)]);
          xr[4 * u] = v.x, xr[4 * u + 1] = v.y, xr[4 * u + 2] = v.z, xr[4 * u + 3] = v.w;
        }
      }
#pragma unroll
      for (int j = 0; j < 16; ++j) acc += xr[j];
    }
    if (delay) {
      const long long t = clock64();
      while (clock64() - t < delay) {
      }
    }
    __syncthreads();
    if (warp == 0) {
      mine = acc + lane;
      if (FMT == 0 || FMT == 2) {
        if (r0 + lane < r1)
          st_rlx(xt + (size_t)((s + 1) & 1) * N + r0 + lane,
                 ((unsigned long long)(want + 1) << 32) | __float_as_uint(mine));
      } else {
        // lane k < 4 gathers rows 7k..7k+6 and stores sector k with one 256-bit store
        float v[7];
#pragma unroll
        for (int e = 0; e < 7; ++e) v[e] = __shfl_sync(0xffffffffu, mine, (7 * lane + e) & 31);
        if (lane < 4) {
          W4 w;
          w.w[0] = ((unsigned long long)__float_as_uint(v[1]) << 32) | __float_as_uint(v[0]);
          w.w[1] = ((unsigned long long)__float_as_uint(v[3]) << 32) | __float_as_uint(v[2]);
          w.w[2] = ((unsigned long long)__float_as_uint(v[5]) << 32) | __float_as_uint(v[4]);
          w.w[3] = ((unsigned long long)(want + 1) << 32) | __float_as_uint(v[6]);
          st_rlx4(xt + (size_t)((s + 1) & 1) * (G * 16) + 16 * blockIdx.x + 4 * lane, w);
        }
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
  unsigned tag = 1;
  void *kern[] = {(void *)xchg3<0>, (void *)xchg3<1>, (void *)xchg3<2>};
  const char *names[] = {"8B tagged words -> regs", "32B sectors (7+tag) -> smem", "8B tagged words -> smem"};
  for (int rep = 0; rep < 2; ++rep)
    for (int delay : {0, 1000, 2000})
      for (int f = 0; f < 3; ++f) {
        cudaMemset(xt, 0, 2 * 16 * N * 8);
        tag = 1;
        cudaEvent_t a, b;
        cudaEventCreate(&a);
        cudaEventCreate(&b);
        void *args[] = {&xt, (void *)&sweeps, &delay, &tag, &sink};
        cudaEventRecord(a);
        cudaLaunchCooperativeKernel(kern[f], sms, T, args, 0, 0);
        cudaEventRecord(b);
        if (cudaEventSynchronize(b) != cudaSuccess) {
          printf("error %s\n", cudaGetErrorString(cudaGetLastError()));
          return 1;
        }
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        printf("%-30s busy delay %4d cyc (%4.0f ns): %.3f us/sweep\n", names[f], delay, delay / (clk * 1e-6),
               ms * 1e3 / sweeps);
      }
  return 0;
}
