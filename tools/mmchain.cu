// Bit-exact matmul inner loop probe (dev tool): cycles per k of the serial
// FMUL+FADD chain when operands stream from shared memory, for several
// software-pipelining schemes.  One CTA per SM, operands pre-staged in smem
// (a 64-k ring read modulo 64, like the kernel's cp.async ring).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/mmchain tools/mmchain.cu
//   ./tools/mmchain [K=4608]
//
// V0: the tile kernel's scheme: load 16 k of operands (4 + 4 LDS.128), then 16 chain steps
// V1: register double buffer, one 4-k group ahead
// V2: two 4-k groups ahead
// V3: V1 with two cells per thread (one A row, two B columns)
// V4: V2 with two cells per thread
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

constexpr int LD = 68;

__device__ __forceinline__ float4 lds4(const float *p) { return *reinterpret_cast<const float4 *>(p); }
__device__ __forceinline__ float comp(const float4 &v, int q) { return q == 0 ? v.x : q == 1 ? v.y : q == 2 ? v.z : v.w; }

template <int V, int TY, int TX, int C>
__global__ void chain(int K, float *out, long long *cyc) {
  __shared__ __align__(16) float As[TY][LD];
  __shared__ __align__(16) float Bs[TX * C][LD];
  const int tid = threadIdx.x, tx = tid % TX, ty = tid / TX;
  for (int i = tid; i < TY * LD; i += blockDim.x) (&As[0][0])[i] = 1.0f + 1e-3f * (i % 97);
  for (int i = tid; i < TX * C * LD; i += blockDim.x) (&Bs[0][0])[i] = 0.5f - 1e-3f * (i % 89);
  __syncthreads();
  const float *ar = As[ty];
  const float *br[C];
#pragma unroll
  for (int c = 0; c < C; ++c) br[c] = Bs[tx + TX * c];
  float acc[C];
#pragma unroll
  for (int c = 0; c < C; ++c) acc[c] = 0.f;
  const long long t0 = clock64();
  if (V == 5 || V == 6) {  // no shared memory: operands from registers
    float ra[8], rb[8][C];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      ra[j] = ar[j];
#pragma unroll
      for (int c = 0; c < C; ++c) rb[j][c] = br[c][j];
    }
    for (int k0 = 0; k0 < K; k0 += 8) {
#pragma unroll
      for (int j = 0; j < 8; ++j)
#pragma unroll
        for (int c = 0; c < C; ++c)
          acc[c] = V == 5 ? __fadd_rn(acc[c], __fmul_rn(ra[j], rb[j][c])) : __fadd_rn(acc[c], rb[j][c]);
    }
  } else if (V == 0) {
    for (int k0 = 0; k0 < K; k0 += 16) {
      const int kk = k0 & 63;
      float4 av[4], bv[4][C];
#pragma unroll
      for (int g = 0; g < 4; ++g) {
        av[g] = lds4(ar + kk + 4 * g);
#pragma unroll
        for (int c = 0; c < C; ++c) bv[g][c] = lds4(br[c] + kk + 4 * g);
      }
#pragma unroll
      for (int g = 0; g < 4; ++g)
#pragma unroll
        for (int q = 0; q < 4; ++q)
#pragma unroll
          for (int c = 0; c < C; ++c) acc[c] = __fadd_rn(acc[c], __fmul_rn(comp(av[g], q), comp(bv[g][c], q)));
    }
  } else {
    constexpr int D = (V == 2 || V == 4) ? 2 : 1;  // groups in flight ahead
    float4 av[D + 1], bv[D + 1][C];
#pragma unroll
    for (int d = 0; d < D; ++d) {
      av[d] = lds4(ar + 4 * d);
#pragma unroll
      for (int c = 0; c < C; ++c) bv[d][c] = lds4(br[c] + 4 * d);
    }
    // unrolled by D+1 so the register ring indices are static
    for (int k0 = 0; k0 < K; k0 += 4 * (D + 1)) {
#pragma unroll
      for (int u = 0; u <= D; ++u) {
        const int cur = u, nxt = (u + D) % (D + 1);
        const int kn = (k0 + 4 * (u + D)) & 63;
        av[nxt] = lds4(ar + kn);
#pragma unroll
        for (int c = 0; c < C; ++c) bv[nxt][c] = lds4(br[c] + kn);
#pragma unroll
        for (int q = 0; q < 4; ++q)
#pragma unroll
          for (int c = 0; c < C; ++c) acc[c] = __fadd_rn(acc[c], __fmul_rn(comp(av[cur], q), comp(bv[cur][c], q)));
      }
    }
  }
  const long long t1 = clock64();
  float s = 0.f;
#pragma unroll
  for (int c = 0; c < C; ++c) s += acc[c];
  out[blockIdx.x * blockDim.x + tid] = s;
  if (tid == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int V, int TY, int TX, int C>
void run(const char *name, int K, int sms, float *out, long long *cyc) {
  chain<V, TY, TX, C><<<sms, TY * TX>>>(K, out, cyc);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  chain<V, TY, TX, C><<<sms, TY * TX>>>(K, out, cyc);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  long long h[1024];
  cudaMemcpy(h, cyc, sms * sizeof(long long), cudaMemcpyDeviceToHost);
  double mean = 0;
  for (int i = 0; i < sms; ++i) mean += h[i];
  mean /= sms;
  printf("%-34s threads %3d cells/thread %d: %6.2f cycles per k (%.1f us for K=%d)\n", name, TY * TX, C, mean / K,
         ms * 1e3, K);
}

int main(int argc, char **argv) {
  const int K = argc > 1 ? atoi(argv[1]) : 4608;
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  float *out;
  long long *cyc;
  cudaMalloc(&out, sms * 1024 * 4);
  cudaMalloc(&cyc, 1024 * 8);
  run<5, 4, 32, 1>("V5 regs only FMUL+FADD, 128 thr", K, sms, out, cyc);
  run<5, 8, 32, 1>("V5 regs only FMUL+FADD, 256 thr", K, sms, out, cyc);
  run<5, 16, 32, 1>("V5 regs only FMUL+FADD, 512 thr", K, sms, out, cyc);
  run<5, 8, 32, 2>("V5 regs only, 2 cells, 256 thr", K, sms, out, cyc);
  run<5, 8, 32, 4>("V5 regs only, 4 cells, 256 thr", K, sms, out, cyc);
  run<6, 8, 32, 1>("V6 regs only FADD chain, 256 thr", K, sms, out, cyc);
  run<6, 16, 32, 1>("V6 regs only FADD chain, 512 thr", K, sms, out, cyc);
  run<0, 16, 16, 1>("V0 16k batch (tile kernel)", K, sms, out, cyc);
  run<1, 16, 16, 1>("V1 double buffer, 1 group ahead", K, sms, out, cyc);
  run<2, 16, 16, 1>("V2 double buffer, 2 groups ahead", K, sms, out, cyc);
  run<3, 16, 16, 2>("V3 = V1, 2 cells", K, sms, out, cyc);
  run<4, 16, 16, 2>("V4 = V2, 2 cells", K, sms, out, cyc);
  run<0, 16, 16, 2>("V0, 2 cells", K, sms, out, cyc);
  run<1, 8, 16, 1>("V1, 128 threads", K, sms, out, cyc);
  run<2, 8, 16, 1>("V2, 128 threads", K, sms, out, cyc);
  run<1, 32, 16, 1>("V1, 512 threads", K, sms, out, cyc);
  run<2, 32, 16, 1>("V2, 512 threads", K, sms, out, cyc);
  run<4, 32, 16, 2>("V4, 512 threads", K, sms, out, cyc);
  run<2, 64, 4, 1>("V2, 64x4 tile", K, sms, out, cyc);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) printf("error %s\n", cudaGetErrorString(e));
  return 0;
}
