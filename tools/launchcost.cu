// Dev probe: host-side cost of a (cooperative) launch vs kernel parameter size.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tools/launchcost tools/launchcost.cu
#include <chrono>
#include <cstdio>
#include <cuda_runtime.h>

template <int B> struct P { unsigned char d[B]; };
template <int B> __global__ void k(const __grid_constant__ P<B> p, int *o) {
  if (threadIdx.x == 0 && blockIdx.x == 0 && p.d[0] == 7) o[0] = 1;
}

template <int B> void run(bool coop, cudaStream_t s, int *o) {
  static P<B> p{};
  void *args[] = {&p, &o};
  const int reps = 200;
  for (int w = 0; w < 20; ++w) {
    if (coop) cudaLaunchCooperativeKernel((void *)k<B>, 148, 256, args, 0, s);
    else cudaLaunchKernel((void *)k<B>, 148, 256, args, 0, s);
  }
  cudaStreamSynchronize(s);
  double tot = 0;
  for (int r = 0; r < reps; ++r) {
    auto t0 = std::chrono::high_resolution_clock::now();
    if (coop) cudaLaunchCooperativeKernel((void *)k<B>, 148, 256, args, 0, s);
    else cudaLaunchKernel((void *)k<B>, 148, 256, args, 0, s);
    auto t1 = std::chrono::high_resolution_clock::now();
    tot += std::chrono::duration<double, std::micro>(t1 - t0).count();
    cudaStreamSynchronize(s);
  }
  printf("%-11s params %5d B: %6.2f us host per launch\n", coop ? "cooperative" : "plain", B, tot / reps);
}

int main() {
  cudaStream_t s;
  cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  int *o;
  cudaMalloc(&o, 4);
  for (int c = 0; c < 2; ++c) {
    run<64>(c, s, o);
    run<1024>(c, s, o);
    run<4096>(c, s, o);
    run<6144>(c, s, o);
  }
  return 0;
}
