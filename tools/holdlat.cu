// Dev probe: does a tiny "hold" kernel, spinning on a host flag while the
// host prepares the next launch, hide the launch latency of a persistent
// cooperative grid that lands on an otherwise idle GPU?
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tools/holdlat tools/holdlat.cu
#include <chrono>
#include <cstdio>
#include <thread>
#include <cuda_runtime.h>

__global__ void grid_k(int *o, int iters) {
  __shared__ int sm[1];
  if (threadIdx.x == 0) sm[0] = blockIdx.x;
  __syncthreads();
  long long t = clock64();
  while (clock64() - t < iters) {
  }
  if (threadIdx.x == 0 && sm[0] == 100000) o[0] = 1;
}
__global__ void hold_k(volatile unsigned *flag, unsigned want) {
  long long t0 = clock64();
  while (*flag != want && clock64() - t0 < 200000000LL) {
  }
}

int main() {
  cudaStream_t s;
  cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  int *o;
  cudaMalloc(&o, 4);
  unsigned *flag;
  cudaHostAlloc((void **)&flag, 4, cudaHostAllocMapped);
  *flag = 0;
  const int smem = 118784;
  cudaFuncSetAttribute(grid_k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int iters : {0, 200000}) {
    for (int mode = 0; mode < 2; ++mode) {
      float tot = 0;
      const int reps = 40;
      for (int r = 0; r < reps + 5; ++r) {
        const unsigned want = (unsigned)(r + 1 + mode * 1000 + iters);
        if (mode == 1) hold_k<<<1, 32, 0, s>>>(flag, want);
        else std::this_thread::sleep_for(std::chrono::microseconds(30));  // GPU idle
        void *args[] = {&o, &iters};
        cudaEventRecord(e0, s);
        cudaLaunchCooperativeKernel((void *)grid_k, 148, 256, args, smem, s);
        cudaEventRecord(e1, s);
        if (mode == 1) {
          std::this_thread::sleep_for(std::chrono::microseconds(30));  // the host's remaining work
          *(volatile unsigned *)flag = want;
        }
        cudaEventSynchronize(e1);
        float ms = 0;
        if (cudaEventElapsedTime(&ms, e0, e1) != cudaSuccess || cudaGetLastError() != cudaSuccess) {
          printf("error\n");
          return 1;
        }
        if (r >= 5) tot += ms;
      }
      printf("grid work %7d cycles, %s: %7.2f us event-to-event\n", iters, mode ? "behind a hold kernel" : "idle GPU          ",
             tot / reps * 1e3);
    }
  }
  return 0;
}
