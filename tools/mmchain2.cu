// Bit-exact matmul inner loop probe, TM x TN cells per thread (dev tool):
// cycles per k with operands streamed from shared memory (a 64-k ring read
// modulo 64) for a tile group of TY x TX threads, one group per SM.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/mmchain2 tools/mmchain2.cu
//   ./tools/mmchain2 [K=4608]
//
// P0: per 4 k, TM + TN LDS.128 then the 4 k of arithmetic (mm_tile's general path)
// P1: the same with the next 4-k group's loads issued before the current group's arithmetic
// P2: two groups ahead
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

constexpr int LD = 68;

__device__ __forceinline__ float4 lds4(const float *p) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "r"((unsigned)__cvta_generic_to_shared(p)));
  return v;
}
__device__ __forceinline__ float comp(const float4 &v, int q) { return q == 0 ? v.x : q == 1 ? v.y : q == 2 ? v.z : v.w; }

template <int P, int TY, int TX, int TM, int TN>
__global__ void chain(int K, float *out, long long *cyc) {
  __shared__ __align__(16) float As[TY * TM][LD];
  __shared__ __align__(16) float Bs[TX * TN][LD];
  const int tid = threadIdx.x, tx = tid % TX, ty = tid / TX;
  for (int i = tid; i < TY * TM * LD; i += blockDim.x) (&As[0][0])[i] = 1.0f + 1e-3f * (i % 97);
  for (int i = tid; i < TX * TN * LD; i += blockDim.x) (&Bs[0][0])[i] = 0.5f - 1e-3f * (i % 89);
  __syncthreads();
  float acc[TM][TN];
#pragma unroll
  for (int i = 0; i < TM; ++i)
#pragma unroll
    for (int j = 0; j < TN; ++j) acc[i][j] = 0.f;
  const long long t0 = clock64();
  constexpr int D = P;  // groups ahead
  float4 av[D + 1][TM], bv[D + 1][TN];
  auto load = [&](int slot, int kk) {
#pragma unroll
    for (int i = 0; i < TM; ++i) av[slot][i] = lds4(&As[ty + TY * i][kk]);
#pragma unroll
    for (int j = 0; j < TN; ++j) bv[slot][j] = lds4(&Bs[tx + TX * j][kk]);
  };
  auto compute = [&](int slot) {
#pragma unroll
    for (int q = 0; q < 4; ++q)
#pragma unroll
      for (int i = 0; i < TM; ++i)
#pragma unroll
        for (int j = 0; j < TN; ++j)
          acc[i][j] = __fadd_rn(acc[i][j], __fmul_rn(comp(av[slot][i], q), comp(bv[slot][j], q)));
  };
#pragma unroll
  for (int d = 0; d < D; ++d) load(d, 4 * d);
  for (int k0 = 0; k0 < K; k0 += 4 * (D + 1)) {
#pragma unroll
    for (int u = 0; u <= D; ++u) {
      const int nxt = (u + D) % (D + 1);
      load(nxt, (k0 + 4 * (u + D)) & 63);
      compute(u);
    }
  }
  const long long t1 = clock64();
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < TM; ++i)
#pragma unroll
    for (int j = 0; j < TN; ++j) s += acc[i][j];
  out[blockIdx.x * blockDim.x + tid] = s;
  if (tid == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int P, int TY, int TX, int TM, int TN>
void run(int K, int sms, float *out, long long *cyc) {
  chain<P, TY, TX, TM, TN><<<sms, TY * TX>>>(K, out, cyc);
  chain<P, TY, TX, TM, TN><<<sms, TY * TX>>>(K, out, cyc);
  cudaDeviceSynchronize();
  long long h[1024];
  cudaMemcpy(h, cyc, sms * sizeof(long long), cudaMemcpyDeviceToHost);
  double mean = 0;
  for (int i = 0; i < sms; ++i) mean += h[i];
  mean /= sms;
  printf("P%d threads %3d (%2dx%2d) cells %dx%d: %6.2f cycles per k, %6.1f cells x k per cycle per SM\n", P, TY * TX,
         TY, TX, TM, TN, mean / K, TY * TX * TM * TN * K / mean);
}

int main(int argc, char **argv) {
  const int K = argc > 1 ? atoi(argv[1]) : 4608;
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  float *out;
  long long *cyc;
  cudaMalloc(&out, sms * 1024 * 4);
  cudaMalloc(&cyc, 1024 * 8);
#define ALLP(TY, TX, TM, TN) \
  run<0, TY, TX, TM, TN>(K, sms, out, cyc); \
  run<1, TY, TX, TM, TN>(K, sms, out, cyc); \
  run<2, TY, TX, TM, TN>(K, sms, out, cyc);
  ALLP(8, 8, 2, 2)
  ALLP(8, 16, 2, 2)
  ALLP(16, 16, 2, 2)
  ALLP(8, 8, 1, 2)
  ALLP(8, 16, 1, 2)
  ALLP(16, 16, 1, 2)
  ALLP(8, 16, 1, 1)
  ALLP(16, 16, 1, 1)
  ALLP(8, 8, 2, 4)
  ALLP(8, 16, 2, 4)
  ALLP(16, 16, 2, 4)
  ALLP(8, 8, 4, 4)
  ALLP(16, 16, 4, 4)
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) printf("error %s\n", cudaGetErrorString(e));
  return 0;
}
