// Microbenchmark: per-SMSP throughput of MUFU.EX2, F2FP.BF16 pack, FFMA2, and mixes (cycles per warp-instr).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

template <int MODE>
__global__ void k(float* out, uint32_t* out2, int iters) {
  float a[8]; uint32_t u[8];
  for (int i = 0; i < 8; ++i) { a[i] = -0.001f * (threadIdx.x + i); u[i] = i; }
  unsigned long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (MODE == 0 || MODE == 2) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a[i]));
      if (MODE == 1 || MODE == 2) { uint32_t r; asm volatile("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(a[i]), "f"(a[(i+1)&7])); u[i] ^= r; }
      if (MODE == 3) { asm volatile("fma.rn.f32 %0, %0, 0f3F800001, 0f3A000000;" : "+f"(a[i])); }
    }
  }
  unsigned long long t1 = clock64();
  float s = 0; uint32_t x = 0;
  for (int i = 0; i < 8; ++i) { s += a[i]; x ^= u[i]; }
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  out2[blockIdx.x * blockDim.x + threadIdx.x] = x;
  if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = (float)(t1 - t0);
}

int main() {
  float* o; uint32_t* o2;
  cudaMalloc(&o, 148 * 1024 * 4); cudaMalloc(&o2, 148 * 1024 * 4);
  const int iters = 4096;
  const char* names[] = {"MUFU.EX2", "F2FP.BF16 pack", "EX2+F2FP (1:1)", "FFMA"};
  for (int warps_per_smsp : {1, 2, 4}) {
    for (int mode = 0; mode < 4; ++mode) {
      int threads = 128 * warps_per_smsp;
      for (int rep = 0; rep < 2; ++rep) {
        if (mode == 0) k<0><<<148, threads>>>(o, o2, iters);
        if (mode == 1) k<1><<<148, threads>>>(o, o2, iters);
        if (mode == 2) k<2><<<148, threads>>>(o, o2, iters);
        if (mode == 3) k<3><<<148, threads>>>(o, o2, iters);
      }
      cudaDeviceSynchronize();
      float cyc; cudaMemcpy(&cyc, o, 4, cudaMemcpyDeviceToHost);
      double instr_per_smsp = (double)iters * 8 * warps_per_smsp * (mode == 2 ? 2 : 1);
      printf("%-18s warps/SMSP=%d: %.2f cycles per warp-instruction per SMSP (%.1f lanes/clk/SM)\n", names[mode],
             warps_per_smsp, cyc / instr_per_smsp, 4 * 32 / (cyc / instr_per_smsp));
    }
  }
  return 0;
}
