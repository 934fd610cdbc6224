// Dev probe: GPU-side launch-to-completion time of an empty persistent grid
// (148 x 256, 118 KB dynamic smem like the Jacobi chain), plain vs
// cooperative launch, GPU idle before each launch (event-timed).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tools/launchlat tools/launchlat.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k(int *o) {
  __shared__ int sm[1];  // the dynamic allocation only sizes the CTA
  if (threadIdx.x == 0) sm[0] = blockIdx.x;
  __syncthreads();
  if (threadIdx.x == 0 && sm[0] == 100000) o[0] = 1;
}

int main() {
  cudaStream_t s;
  cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  int *o;
  cudaMalloc(&o, 4);
  const int smem = 118784;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  void *args[] = {&o};
  for (int coop = 0; coop < 2; ++coop)
    for (int sm_on = 0; sm_on < 2; ++sm_on) {
      float tot = 0;
      const int reps = 50;
      for (int r = 0; r < reps + 5; ++r) {
        cudaEventRecord(e0, s);
        if (coop)
          cudaLaunchCooperativeKernel((void *)k, 148, 256, args, sm_on ? smem : 0, s);
        else
          cudaLaunchKernel((void *)k, 148, 256, args, sm_on ? smem : 0, s);
        cudaEventRecord(e1, s);
        cudaEventSynchronize(e1);
        float ms = 0;
        cudaError_t er = cudaEventElapsedTime(&ms, e0, e1);
        if (er != cudaSuccess || cudaGetLastError() != cudaSuccess) { printf("error %s\n", cudaGetErrorString(er)); return 1; }
        if (r >= 5) tot += ms;
      }
      printf("%-11s smem %6d: %6.2f us event-to-event (idle GPU)\n", coop ? "cooperative" : "plain",
             sm_on ? smem : 0, tot / reps * 1e3);
    }
  return 0;
}
