// Dev probe: latency of one Jacobi-style poll round (each lane loads K x 32 B
// of a shared 32 KB buffer that every CTA reads) as a function of how many
// SMs poll at once, the load flavour and the buffer layout.  No stores: the
// data is static, so this isolates the L2 read path.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/l2lat tools/l2lat.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr int T = 256, REPS = 200;

template <int MODE>
__device__ __forceinline__ ulonglong4 ld32(const unsigned long long *p) {
  ulonglong4 v;
  if (MODE == 0)
    asm volatile("ld.relaxed.gpu.global.v4.u64 {%0,%1,%2,%3}, [%4];"
                 : "=l"(v.x), "=l"(v.y), "=l"(v.z), "=l"(v.w) : "l"(p) : "memory");
  else if (MODE == 1)
    asm volatile("ld.global.cg.v4.u64 {%0,%1,%2,%3}, [%4];"
                 : "=l"(v.x), "=l"(v.y), "=l"(v.z), "=l"(v.w) : "l"(p) : "memory");
  else
    asm volatile("ld.volatile.global.v4.u64 {%0,%1,%2,%3}, [%4];"
                 : "=l"(v.x), "=l"(v.y), "=l"(v.z), "=l"(v.w) : "l"(p) : "memory");
  return v;
}

// K loads of 32 B per lane; stride: lane's u-th load at word 4 * (cbase + 32 u)
// (the kernel's layout) -- one poll round per rep, all threads synchronised
template <int MODE, int K>
__global__ void __launch_bounds__(T, 1) poll(const unsigned long long *buf, int words, long long *out, unsigned *sink) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int cbase = warp * 128 + lane;
  unsigned acc = 0;
  long long tot = 0;
  for (int r = 0; r < REPS; ++r) {
    __syncthreads();
    const long long t0 = clock64();
    ulonglong4 q[K];
#pragma unroll
    for (int u = 0; u < K; ++u) q[u] = ld32<MODE>(buf + (4 * (cbase + 32 * u)) % words);
#pragma unroll
    for (int u = 0; u < K; ++u) acc += (unsigned)(q[u].x ^ q[u].w);
    const long long t1 = clock64();  // after the loads' values are used
    tot += t1 - t0;
  }
  if (threadIdx.x == 0) out[blockIdx.x] = tot / REPS;
  if (acc == 0x12345u) *sink = acc;
}

template <int MODE, int K>
void run(const char *name, const unsigned long long *buf, int words, long long *out, unsigned *sink, int grid,
         int clk_khz) {
  cudaFuncSetAttribute(poll<MODE, K>, cudaFuncAttributeMaxDynamicSharedMemorySize, 120 * 1024);
  poll<MODE, K><<<grid, T, 120 * 1024>>>(buf, words, out, sink);
  poll<MODE, K><<<grid, T, 120 * 1024>>>(buf, words, out, sink);
  cudaDeviceSynchronize();
  long long h[148];
  cudaMemcpy(h, out, sizeof(long long) * grid, cudaMemcpyDeviceToHost);
  double s = 0;
  for (int i = 0; i < grid; ++i) s += h[i];
  s /= grid;
  printf("%-10s K=%d grid=%3d buffer %6d B: %6.0f cycles = %5.0f ns per round\n", name, K, grid, words * 8, s,
         s / (clk_khz * 1e-6));
}

int main() {
  unsigned long long *buf;
  long long *out;
  unsigned *sink;
  const int big = 16 * 4096;
  cudaMalloc(&buf, big * 8);
  cudaMemset(buf, 1, big * 8);
  cudaMalloc(&out, 148 * 8);
  cudaMalloc(&sink, 4);
  int clk;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  for (int g : {1, 2, 16, 37, 74, 148}) run<0, 4>("relaxed", buf, 4096, out, sink, g, clk);
  for (int g : {1, 148}) run<0, 1>("relaxed", buf, 4096, out, sink, g, clk);
  for (int g : {1, 148}) run<0, 2>("relaxed", buf, 4096, out, sink, g, clk);
  for (int g : {1, 148}) run<1, 4>("cg", buf, 4096, out, sink, g, clk);
  for (int g : {1, 148}) run<2, 4>("volatile", buf, 4096, out, sink, g, clk);
  return 0;
}
