// Dev probe: (1) per-128B-line load latency of a 64 KB buffer from SMs on
// either die (which lines are "near"), (2) poll-round latency when the lines
// are being written by other CTAs (the Jacobi exchange) vs static lines.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/l2home tools/l2home.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr int LINES = 512;  // 64 KB

__device__ __forceinline__ unsigned long long ld_rlx(const unsigned long long *p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_rlx(unsigned long long *p, unsigned long long v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

__global__ void homemap(unsigned long long *buf, int target_sm, int *lat, unsigned *found) {
  unsigned sm;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(sm));
  if ((int)sm != target_sm || threadIdx.x != 0) return;
  *found = 1;
  unsigned long long acc = 0;
  for (int pass = 0; pass < 2; ++pass)
    for (int i = 0; i < LINES; ++i) {
      const long long t0 = clock64();
      const unsigned long long v = ld_rlx(buf + (size_t)i * 16 + (acc & 1));
      acc += v;
      const long long t1 = clock64();
      if (pass == 1) lat[i] = (int)(t1 - t0);
    }
  if (acc == 77) buf[0] = acc;
}

// MODE 0: static lines; MODE 1: each CTA first stores 28 words of its band
// into the buffer (as the Jacobi publish does), then polls the whole 32 KB
template <int MODE>
__global__ void __launch_bounds__(256, 1) poll(unsigned long long *buf, long long *out, unsigned *sink) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int cbase = warp * 128 + lane;
  const int r0 = blockIdx.x * 4096 / gridDim.x, r1 = (blockIdx.x + 1) * 4096 / gridDim.x;
  unsigned acc = 0;
  long long tot = 0;
  for (int r = 0; r < 200; ++r) {
    if (MODE == 1 && warp == 0)
      for (int row = r0 + lane; row < r1; row += 32) st_rlx(buf + row, (unsigned long long)r << 32 | row);
    __syncthreads();
    const long long t0 = clock64();
    ulonglong4 q[4];
#pragma unroll
    for (int u = 0; u < 4; ++u)
      asm volatile("ld.relaxed.gpu.global.v4.u64 {%0,%1,%2,%3}, [%4];"
                   : "=l"(q[u].x), "=l"(q[u].y), "=l"(q[u].z), "=l"(q[u].w)
                   : "l"(buf + 4 * (cbase + 32 * u))
                   : "memory");
#pragma unroll
    for (int u = 0; u < 4; ++u) acc += (unsigned)(q[u].x ^ q[u].w);
    const long long t1 = clock64();
    tot += t1 - t0;
    __syncthreads();
  }
  if (threadIdx.x == 0) out[blockIdx.x] = tot / 200;
  if (acc == 0x12345u) *sink = acc;
}

int main() {
  unsigned long long *buf;
  int *lat;
  unsigned *found;
  long long *out;
  unsigned *sink;
  cudaMalloc(&buf, LINES * 128);
  cudaMemset(buf, 0, LINES * 128);
  cudaMalloc(&lat, LINES * 4);
  cudaMalloc(&found, 4);
  cudaMalloc(&out, 148 * 8);
  cudaMalloc(&sink, 4);
  int clk;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  for (int sm : {0, 1, 36, 73, 74, 75, 110, 147}) {
    cudaMemset(found, 0, 4);
    homemap<<<148, 32>>>(buf, sm, lat, found);
    cudaDeviceSynchronize();
    unsigned f;
    int h[LINES];
    cudaMemcpy(&f, found, 4, cudaMemcpyDeviceToHost);
    cudaMemcpy(h, lat, sizeof h, cudaMemcpyDeviceToHost);
    if (!f) {
      printf("sm %3d: not scheduled\n", sm);
      continue;
    }
    int lo = 1 << 30, hi = 0, nfast = 0;
    for (int i = 0; i < LINES; ++i) {
      lo = h[i] < lo ? h[i] : lo;
      hi = h[i] > hi ? h[i] : hi;
    }
    const int mid = (lo + hi) / 2;
    char pat[65];
    for (int i = 0; i < 64; ++i) pat[i] = h[i] < mid ? '.' : 'X';
    pat[64] = 0;
    for (int i = 0; i < LINES; ++i) nfast += h[i] < mid;
    printf("sm %3d: line latency %d..%d cycles, %d of %d lines fast; first 64 lines: %s\n", sm, lo, hi, nfast,
           LINES, pat);
  }
  for (int mode = 0; mode < 2; ++mode) {
    for (int rep = 0; rep < 2; ++rep) {
      if (mode == 0) poll<0><<<148, 256>>>(buf, out, sink);
      else poll<1><<<148, 256>>>(buf, out, sink);
      cudaDeviceSynchronize();
    }
    long long h[148];
    cudaMemcpy(h, out, sizeof h, cudaMemcpyDeviceToHost);
    double s = 0, mx = 0;
    for (int i = 0; i < 148; ++i) {
      s += h[i];
      mx = h[i] > mx ? h[i] : mx;
    }
    printf("poll round, %s lines: mean %.0f cycles (%.0f ns), max CTA %.0f cycles\n",
           mode ? "just-written" : "static", s / 148, s / 148 / (clk * 1e-6), mx);
  }
  return 0;
}
