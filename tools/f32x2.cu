// Packed FP32 (f32x2) for the bit-exact matmul chain? (dev probe)
// acc = fl(acc + fl(a * b)) must not become one FFMA2.  Three ways of writing
// the packed multiply + add; each is checked bit-exactly against scalar
// __fmul_rn/__fadd_rn and timed.  cuobjdump -sass shows whether ptxas fused.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/f32x2 tools/f32x2.cu
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned long long mul2(unsigned long long a, unsigned long long b) {
  unsigned long long d;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
__device__ __forceinline__ unsigned long long add2(unsigned long long a, unsigned long long b) {
  unsigned long long d;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
__device__ __forceinline__ unsigned long long fma2(unsigned long long a, unsigned long long b,
                                                   unsigned long long c) {
  unsigned long long d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}
__device__ __forceinline__ unsigned long long pk(float lo, float hi) {
  unsigned long long r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
  return r;
}
__device__ __forceinline__ float lo_(unsigned long long v) { return __uint_as_float((unsigned)v); }
__device__ __forceinline__ float hi_(unsigned long long v) { return __uint_as_float((unsigned)(v >> 32)); }

// S = 0: scalar reference; 1: packed, product then add; 2: products one step
// ahead (loop-carried); 3: product laundered through a predicated select on
// a runtime flag ptxas cannot evaluate; 4: the add as fma(acc, one, p) with
// `one` a runtime 1.0 (acc * 1 is exact, so this is fl(acc + p); no
// instruction fuses a multiply into an FMA's addend)
template <int S>
__global__ void k(const float *a, const float *b, int K, float *out, long long *cyc, int flag) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  float c0 = 0.f, c1 = 0.f, c2 = 0.f, c3 = 0.f;
  unsigned long long p01 = 0, p23 = 0;
  const long long t0 = clock64();
  if (S == 2) {
    p01 = mul2(pk(a[0], a[0]), pk(b[t % 64], b[(t + 1) % 64]));
    p23 = mul2(pk(a[1], a[1]), pk(b[(t + 2) % 64], b[(t + 3) % 64]));
  }
  unsigned long long acc01 = 0, acc23 = 0;
  for (int kk = 0; kk < K; ++kk) {
    const float x = a[kk & 63], y = a[(kk + 7) & 63];
    const float b0 = b[(t + kk) & 63], b1 = b[(t + kk + 1) & 63], b2 = b[(t + kk + 2) & 63], b3 = b[(t + kk + 3) & 63];
    if (S == 0) {
      c0 = __fadd_rn(c0, __fmul_rn(x, b0));
      c1 = __fadd_rn(c1, __fmul_rn(x, b1));
      c2 = __fadd_rn(c2, __fmul_rn(y, b2));
      c3 = __fadd_rn(c3, __fmul_rn(y, b3));
    } else if (S == 1) {
      acc01 = add2(acc01, mul2(pk(x, x), pk(b0, b1)));
      acc23 = add2(acc23, mul2(pk(y, y), pk(b2, b3)));
    } else if (S == 2) {
      const unsigned long long n01 = mul2(pk(x, x), pk(b0, b1));  // next step's products
      const unsigned long long n23 = mul2(pk(y, y), pk(b2, b3));
      if (kk > 0) {
        acc01 = add2(acc01, p01);
        acc23 = add2(acc23, p23);
      }
      p01 = n01, p23 = n23;
    } else if (S == 4) {
      const unsigned long long one = pk(__int_as_float(0x3f800000 + flag), __int_as_float(0x3f800000 + flag));
      acc01 = fma2(acc01, one, mul2(pk(x, x), pk(b0, b1)));
      acc23 = fma2(acc23, one, mul2(pk(y, y), pk(b2, b3)));
    } else {
      unsigned long long q01 = mul2(pk(x, x), pk(b0, b1));
      unsigned long long q23 = mul2(pk(y, y), pk(b2, b3));
      asm("{ .reg .pred p; setp.ne.s32 p, %2, 0; @p mov.b64 %0, 0; @p mov.b64 %1, 0; }" : "+l"(q01), "+l"(q23) : "r"(flag));
      acc01 = add2(acc01, q01);
      acc23 = add2(acc23, q23);
    }
  }
  if (S == 2) {
    acc01 = add2(acc01, p01);
    acc23 = add2(acc23, p23);
  }
  const long long t1 = clock64();
  if (S != 0) c0 = lo_(acc01), c1 = hi_(acc01), c2 = lo_(acc23), c3 = hi_(acc23);
  out[4 * t] = c0, out[4 * t + 1] = c1, out[4 * t + 2] = c2, out[4 * t + 3] = c3;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

int main() {
  const int K = 4096, T = 256, B = 148;
  float ha[64], hb[64];
  srand(1);
  for (int i = 0; i < 64; ++i) ha[i] = (rand() / (float)RAND_MAX - 0.5f) * 3, hb[i] = (rand() / (float)RAND_MAX - 0.5f) * 5;
  float *a, *b, *o[5];
  long long *cyc;
  cudaMalloc(&a, 256);
  cudaMalloc(&b, 256);
  cudaMemcpy(a, ha, 256, cudaMemcpyHostToDevice);
  cudaMemcpy(b, hb, 256, cudaMemcpyHostToDevice);
  cudaMalloc(&cyc, B * 8);
  void (*fn[5])(const float *, const float *, int, float *, long long *, int) = {k<0>, k<1>, k<2>, k<3>, k<4>};
  static float h[5][4 * T * B];
  for (int s = 0; s < 5; ++s) {
    cudaMalloc(&o[s], 4 * T * B * 4);
    fn[s]<<<B, T>>>(a, b, K, o[s], cyc, 0);
    fn[s]<<<B, T>>>(a, b, K, o[s], cyc, 0);
    long long c;
    cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
    cudaMemcpy(h[s], o[s], sizeof h[s], cudaMemcpyDeviceToHost);
    int diff = 0;
    for (int i = 0; i < 4 * T * B; ++i) diff += memcmp(&h[s][i], &h[0][i], 4) != 0;
    printf("style %d: %.2f cycles per k (4 cells/thread, 256 threads/SM), %d of %d results differ from scalar\n", s,
           (double)c / K, diff, 4 * T * B);
  }
  return 0;
}
