// TMEM / shared-memory read-bandwidth probe (dev tool).  Question it answers:
// can the Jacobi sweep keep part of its band of A in tensor memory and read it
// back with tcgen05.ld on a path that adds to the LDS bandwidth?
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/tmembw tools/tmembw.cu
//   ./tools/tmembw [reps=2000]
//
// One CTA per SM, 256 threads (8 warps; warps w and w+4 share TMEM lane
// quadrant w%4 and split the 512 columns).  Per rep every thread reads
//   tcols  TMEM columns of its lane (tcgen05.ld.32x32b.x16, one wait per 4 lds)
//   sf4    float4 from thread-private shared memory ([k][thread], conflict-free)
// and FMAs everything into 16 accumulators against a register "x".
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

#define LD16(taddr, v)                                                                        \
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 "                                     \
               "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"            \
               : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]),    \
                 "=r"(v[6]), "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]),  \
                 "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])                         \
               : "r"(taddr))

#define ST16(taddr, v)                                                                        \
  asm volatile("tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], "                               \
               "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(taddr),   \
               "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), \
               "r"(v[7]), "r"(v[8]), "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]),         \
               "r"(v[13]), "r"(v[14]), "r"(v[15]))

template <int TCOLS, int SF4>
__global__ void __launch_bounds__(256, 1) probe(int reps, float *out, unsigned long long *cyc) {
  extern __shared__ __align__(16) float4 sm[];
  __shared__ uint32_t tbase;
  const int tid = threadIdx.x, warp = tid >> 5;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(&tbase)), "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t taddr = tbase + ((uint32_t)(32 * (warp & 3)) << 16) + (warp >= 4 ? 256u : 0u);
  {
    uint32_t v[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) v[i] = __float_as_uint(1e-3f * (i + tid));
    for (int c = 0; c < 256; c += 16) ST16(taddr + c, v);
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  }
  for (int k = 0; k < SF4; ++k) sm[k * 256 + tid] = make_float4(1e-3f * k, 2e-3f, 3e-3f, tid * 1e-6f);
  __syncthreads();
  float x[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) x[i] = 0.5f + 0.01f * i;
  float acc[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) acc[i] = 0.f;
  const unsigned long long t0 = clock64();
  for (int r = 0; r < reps; ++r) {
#pragma unroll
    for (int c = 0; c < TCOLS; c += 64) {
      uint32_t v[4][16];
      LD16(taddr + c, v[0]);
      LD16(taddr + c + 16, v[1]);
      LD16(taddr + c + 32, v[2]);
      LD16(taddr + c + 48, v[3]);
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
      for (int g = 0; g < 4; ++g)
#pragma unroll
        for (int i = 0; i < 16; ++i) acc[(g * 4 + i) & 15] = fmaf(__uint_as_float(v[g][i]), x[i], acc[(g * 4 + i) & 15]);
    }
#pragma unroll
    for (int k = 0; k < SF4; ++k) {
      float4 a;
      asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(a.x), "=f"(a.y), "=f"(a.z), "=f"(a.w)
                   : "r"(smem_u32(&sm[k * 256 + tid])));
      acc[k & 15] = fmaf(a.x, x[0], acc[k & 15]);
      acc[(k + 1) & 15] = fmaf(a.y, x[1], acc[(k + 1) & 15]);
      acc[(k + 2) & 15] = fmaf(a.z, x[2], acc[(k + 2) & 15]);
      acc[(k + 3) & 15] = fmaf(a.w, x[3], acc[(k + 3) & 15]);
    }
    x[0] += 1e-7f;
  }
  const unsigned long long t1 = clock64();
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < 16; ++i) s += acc[i];
  if (s == 1234.5f) out[0] = s;
  if (tid == 0) cyc[blockIdx.x] = t1 - t0;
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tbase), "r"(512));
}

template <int TCOLS, int SF4>
void run(int reps, int sms, float *out, unsigned long long *cyc) {
  auto k = probe<TCOLS, SF4>;
  const size_t smem = (size_t)SF4 * 256 * 16 + 16;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  k<<<sms, 256, smem>>>(4, out, cyc);
  cudaEventRecord(a);
  k<<<sms, 256, smem>>>(reps, out, cyc);
  cudaEventRecord(b);
  cudaError_t e = cudaEventSynchronize(b);
  if (e != cudaSuccess) {
    printf("error %s\n", cudaGetErrorString(e));
    exit(1);
  }
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  unsigned long long h[256];
  cudaMemcpy(h, cyc, sizeof(unsigned long long) * sms, cudaMemcpyDeviceToHost);
  unsigned long long mx = 0;
  for (int i = 0; i < sms; ++i) mx = h[i] > mx ? h[i] : mx;
  const double tb = (double)TCOLS * 4 * 256 * reps, sb = (double)SF4 * 16 * 256 * reps;
  printf("tmem %3d cols/thr  smem %2d f4/thr : %8.1f cyc/rep  tmem %6.1f B/clk/SM  smem %6.1f B/clk/SM  "
         "total %6.1f B/clk/SM  (%.3f ms, %.1f TB/s chip)\n",
         TCOLS, SF4, (double)mx / reps, tb / mx, sb / mx, (tb + sb) / mx, ms,
         (tb + sb) * sms / (ms * 1e-3) / 1e12);
}

int main(int argc, char **argv) {
  const int reps = argc > 1 ? atoi(argv[1]) : 2000;
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  float *out;
  unsigned long long *cyc;
  cudaMalloc(&out, 4);
  cudaMalloc(&cyc, 8 * 256);
  run<64, 0>(reps, sms, out, cyc);
  run<128, 0>(reps, sms, out, cyc);
  run<256, 0>(reps, sms, out, cyc);
  run<0, 16>(reps, sms, out, cyc);
  run<0, 32>(reps, sms, out, cyc);
  run<0, 48>(reps, sms, out, cyc);
  run<256, 16>(reps, sms, out, cyc);
  run<256, 24>(reps, sms, out, cyc);
  run<256, 32>(reps, sms, out, cyc);
  run<192, 32>(reps, sms, out, cyc);
  run<256, 8>(reps, sms, out, cyc);
  run<128, 16>(reps, sms, out, cyc);
  return 0;
}
