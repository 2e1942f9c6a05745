// MUFU.EX2 throughput by operand format (cycles per warp-instruction per SMSP, 4 warps/SMSP):
// f32 (ex2.approx.ftz.f32), f16 (ex2.approx.f16, one element), f16x2 and bf16x2 (two elements,
// compiled to two MUFU ops each on sm_100a).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o mufu_rates mufu_rates.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

template <int MODE>
__global__ void k(float* out, int iters) {
  float a[8];
  uint32_t h[8];
  uint16_t s[8];
  for (int i = 0; i < 8; ++i) { a[i] = -0.001f * (threadIdx.x + i); h[i] = 0x3c003c00u ^ i; s[i] = 0x3c00 ^ i; }
  unsigned long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (MODE == 0) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a[i]));
      if (MODE == 1) asm volatile("ex2.approx.f16 %0, %0;" : "+h"(s[i]));
      if (MODE == 2) asm volatile("ex2.approx.f16x2 %0, %0;" : "+r"(h[i]));
      if (MODE == 3) asm volatile("ex2.approx.ftz.bf16x2 %0, %0;" : "+r"(h[i]));
    }
  }
  unsigned long long t1 = clock64();
  float z = 0;
  for (int i = 0; i < 8; ++i) z += a[i] + h[i] + s[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = z;
  if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = (float)(t1 - t0);
}

template <int M> void run(float* o, const char* name, int elems) {
  const int iters = 2048, w = 4;
  k<M><<<148, 128 * w>>>(o, iters); k<M><<<148, 128 * w>>>(o, iters);
  cudaDeviceSynchronize();
  float c; cudaMemcpy(&c, o, 4, cudaMemcpyDeviceToHost);
  const double per = c / (iters * 8.0 * w);
  printf("%-28s %.2f cycles per warp-instr per SMSP, %.1f exp2/clk/SM\n", name, per, 4 * 32 * elems / per);
}

int main() {
  float* o; cudaMalloc(&o, 148 * 512 * 4);
  run<0>(o, "ex2.approx.ftz.f32", 1);
  run<1>(o, "ex2.approx.f16", 1);
  run<2>(o, "ex2.approx.f16x2", 2);
  run<3>(o, "ex2.approx.ftz.bf16x2", 2);
  return 0;
}
