// One-way SM->SM signalling latency through L2 (dev tool): how fast can a
// value published by one CTA be observed by another?  This bounds the Jacobi
// tagged-x exchange (one publish -> poll hop per sweep).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/pingpong tools/pingpong.cu
//   ./tools/pingpong [iters=2000]
//
// CTA 0 and CTA b ping-pong a counter: each waits for the other's value and
// answers with value+1.  Half the round trip is one publish->observe hop.
// mode 0: st.relaxed.gpu / ld.relaxed.gpu      mode 1: st.release / ld.acquire
// mode 2: red.relaxed.gpu.add / ld.relaxed      mode 3: st.relaxed + ld.volatile (ld.cv)
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned ld_rlx(const unsigned *p) {
  unsigned v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned ld_acq(const unsigned *p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned ld_cv(const unsigned *p) {
  unsigned v;
  asm volatile("ld.volatile.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_rlx(unsigned *p, unsigned v) {
  asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void st_rel(unsigned *p, unsigned v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void red_add(unsigned *p, unsigned v) {
  asm volatile("red.relaxed.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

template <int MODE>
__global__ void pingpong(unsigned *a, unsigned *b, int partner, int iters, long long *out, unsigned *smid) {
  if (threadIdx.x != 0) return;
  unsigned id;
  asm("mov.u32 %0, %%smid;" : "=r"(id));
  smid[blockIdx.x] = id;
  if (blockIdx.x != 0 && (int)blockIdx.x != partner) return;
  const bool ping = blockIdx.x == 0;
  unsigned *mine = ping ? a : b, *theirs = ping ? b : a;
  auto load = [&](const unsigned *p) {
    if (MODE == 1) return ld_acq(p);
    if (MODE == 3) return ld_cv(p);
    return ld_rlx(p);
  };
  auto store = [&](unsigned *p, unsigned v) {
    if (MODE == 1) st_rel(p, v);
    else if (MODE == 2) red_add(p, 1);
    else st_rlx(p, v);
  };
  long long t0 = clock64();
  for (int i = 1; i <= iters; ++i) {
    if (ping) {
      store(mine, i);
      while (load(theirs) < (unsigned)i) {
      }
    } else {
      while (load(theirs) < (unsigned)i) {
      }
      store(mine, i);
    }
  }
  if (ping) out[0] = clock64() - t0;
}

template <int MODE>
void run(int iters, int partner, unsigned *a, unsigned *b, long long *out, unsigned *smid, int sms) {
  cudaMemset(a, 0, 256);
  cudaMemset(b, 0, 256);
  pingpong<MODE><<<sms, 32>>>(a, b, partner, iters, out, smid);
  if (cudaDeviceSynchronize() != cudaSuccess) {
    printf("error\n");
    exit(1);
  }
  long long cyc;
  unsigned ids[256];
  cudaMemcpy(&cyc, out, 8, cudaMemcpyDeviceToHost);
  cudaMemcpy(ids, smid, 4 * sms, cudaMemcpyDeviceToHost);
  int clk;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf("mode %d  sm %3u <-> sm %3u : one-way hop %6.1f cycles = %6.1f ns\n", MODE, ids[0], ids[partner],
         cyc / (2.0 * iters), cyc / (2.0 * iters) / (clk * 1e-6));
}

int main(int argc, char **argv) {
  const int iters = argc > 1 ? atoi(argv[1]) : 2000;
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  unsigned *a, *b, *smid;
  long long *out;
  cudaMalloc(&a, 1 << 20);
  b = a + (64 << 10);  // different 256 KB region: likely another L2 slice / die
  cudaMalloc(&out, 8);
  cudaMalloc(&smid, 4 * 256);
  for (int partner : {1, 2, 37, 74, 111, 147}) {
    run<0>(iters, partner, a, b, out, smid, sms);
    run<1>(iters, partner, a, b, out, smid, sms);
    run<2>(iters, partner, a, b, out, smid, sms);
    run<3>(iters, partner, a, b, out, smid, sms);
  }
  return 0;
}
