// L2 -> SM bandwidth probe (dev tool): how fast can all SMs re-read an
// L2-resident buffer?  This is the honest ceiling for the Jacobi sweep,
// whose 64 MiB matrix stays in L2 across sweeps.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/l2bw tools/l2bw.cu
//   ./tools/l2bw [MiB=64] [reps=50]
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

__global__ void ldg_read(const float4 *__restrict__ p, size_t n4, int reps, float *out) {
  float acc = 0.f;
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  for (int r = 0; r < reps; ++r) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n4; i += stride * 4) {
      float4 v[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) v[u] = (i + u * stride < n4) ? __ldcg(p + i + u * stride) : make_float4(0, 0, 0, 0);
#pragma unroll
      for (int u = 0; u < 4; ++u) acc += v[u].x + v[u].y + v[u].z + v[u].w;
    }
  }
  if (acc == 123.456f) *out = acc;
}

__device__ __forceinline__ unsigned smem_addr(const void *p) {
  return (unsigned)__cvta_generic_to_shared(p);
}

// each CTA streams its contiguous slice with cp.async.bulk into an S-deep ring
__global__ void tma_read(const char *p, size_t bytes, int chunk, int stages, int reps, float *out) {
  extern __shared__ __align__(128) char ring[];
  __shared__ unsigned long long bar[16];
  const size_t per = bytes / gridDim.x / chunk * chunk;
  const char *base = p + per * blockIdx.x;
  const int nchunks = (int)(per / chunk);
  if (threadIdx.x == 0) {
    for (int i = 0; i < stages; ++i)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_addr(&bar[i])));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  float acc = 0.f;
  int q = 0;
  for (int r = 0; r < reps; ++r) {
    for (int c = 0; c < nchunks; ++c, ++q) {
      const int st = q % stages;
      if (q >= stages) {  // wait for the copy that used this stage
        const unsigned par = ((q / stages) - 1) & 1;
        asm volatile("{\n.reg .pred P;\nW%=:\nmbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n@!P bra W%=;\n}" ::"r"(smem_addr(&bar[st])), "r"(par));
        acc += ring[(size_t)st * chunk];
      }
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(&bar[st])), "r"(chunk));
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                   ::"r"(smem_addr(ring + (size_t)st * chunk)), "l"(base + (size_t)c * chunk), "r"(chunk), "r"(smem_addr(&bar[st])) : "memory");
    }
  }
  for (int k = 0; k < stages && k < q; ++k) {
    const int qq = q - 1 - k, st = qq % stages;
    const unsigned par = (qq / stages) & 1;
    asm volatile("{\n.reg .pred P;\nW%=:\nmbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n@!P bra W%=;\n}" ::"r"(smem_addr(&bar[st])), "r"(par));
  }
  if (acc == 123.456f) *out = acc;
}

int main(int argc, char **argv) {
  const size_t mib = argc > 1 ? atoi(argv[1]) : 64;
  const int reps = argc > 2 ? atoi(argv[2]) : 50;
  const size_t bytes = mib << 20;
  char *buf;
  float *out;
  cudaMalloc(&buf, bytes);
  cudaMalloc(&out, 4);
  cudaMemset(buf, 1, bytes);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float ms;
  for (int bpsm : {1, 2, 4, 8}) {
    ldg_read<<<sms * bpsm, 512>>>((const float4 *)buf, bytes / 16, 2, out);
    cudaEventRecord(e0);
    ldg_read<<<sms * bpsm, 512>>>((const float4 *)buf, bytes / 16, reps, out);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    printf("LDG.128 %3zu MiB x%d, %d CTA/SM x 512 thr: %.1f GB/s\n", mib, reps, bpsm,
           (double)bytes * reps / ms / 1e6);
  }
  for (int chunk : {4096, 16384, 32768})
    for (int stages : {4, 8, 12}) {
      const size_t smem = (size_t)chunk * stages;
      if (smem > 200 * 1024) continue;
      cudaFuncSetAttribute(tma_read, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      for (int cps : {1, 2}) {
        if (smem * cps > 220 * 1024) continue;
        tma_read<<<sms * cps, 32, smem>>>(buf, bytes, chunk, stages, 2, out);
        cudaEventRecord(e0);
        tma_read<<<sms * cps, 32, smem>>>(buf, bytes, chunk, stages, reps, out);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        printf("TMA bulk %3zu MiB x%d, chunk %5d x %2d stages, %d CTA/SM: %.1f GB/s  %s\n", mib, reps,
               chunk, stages, cps, (double)bytes * reps / ms / 1e6,
               cudaGetErrorString(cudaGetLastError()));
      }
    }
  return 0;
}
