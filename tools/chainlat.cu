// Dev probe: cycles per step of a dependent FMUL+FADD accumulation chain
// (the bit-exact matmul's inner recurrence), one warp, operands in registers.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void chain(const float *in, float *out, long long *cyc, int iters) {
  float a0 = in[threadIdx.x], a1 = in[threadIdx.x + 32], b0 = in[threadIdx.x + 64], b1 = in[threadIdx.x + 96];
  float acc = 0.f, acc2 = 0.f;
  __syncwarp();
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      acc = __fadd_rn(acc, __fmul_rn(u & 1 ? a0 : a1, u & 2 ? b0 : b1));
    }
    a0 += 1e-7f;  // keep the products from being loop-invariant
  }
  long long t1 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 16; ++u) acc2 = __fadd_rn(acc2, a1);
    a1 += 1e-7f;
  }
  long long t2 = clock64();
  out[threadIdx.x] = acc + acc2;
  if (threadIdx.x == 0) { cyc[0] = t1 - t0; cyc[1] = t2 - t1; }
}
int main() {
  float *in, *out; long long *cyc, h[2];
  cudaMalloc(&in, 512); cudaMalloc(&out, 512); cudaMalloc(&cyc, 16);
  cudaMemset(in, 0, 512);
  const int iters = 4096;
  chain<<<1, 32>>>(in, out, cyc, iters); cudaDeviceSynchronize();
  chain<<<1, 32>>>(in, out, cyc, iters); cudaDeviceSynchronize();
  cudaMemcpy(h, cyc, 16, cudaMemcpyDeviceToHost);
  printf("FMUL+FADD chain: %.2f cycles per step; FADD-only chain: %.2f cycles per step\n",
         (double)h[0] / (iters * 16), (double)h[1] / (iters * 16));
  return 0;
}
