// Per-SMSP throughput (cycles per warp-instruction) of the softmax instruction mix on sm_100a.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define NCH 8
template <int MODE>
__global__ void k(float* out, int iters, float sc, float mm) {
  float a[NCH]; uint64_t b[NCH]; uint32_t u[NCH];
  for (int i = 0; i < NCH; ++i) { a[i] = 1e-3f * (threadIdx.x + i); u[i] = threadIdx.x * 7 + i;
    asm("mov.b64 %0, {%1, %2};" : "=l"(b[i]) : "f"(a[i]), "f"(a[i] + 1.f)); }
  uint64_t s2, m2; asm("mov.b64 %0, {%1, %1};" : "=l"(s2) : "f"(sc)); asm("mov.b64 %0, {%1, %1};" : "=l"(m2) : "f"(mm));
  unsigned long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < NCH; ++i) {
      if (MODE == 0) asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+f"(a[i]) : "f"(sc), "f"(mm));          // FFMA 3-reg
      if (MODE == 1) asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(b[i]) : "l"(s2), "l"(m2));       // FFMA2
      if (MODE == 2) asm volatile("add.rn.f32x2 %0, %0, %1;" : "+l"(b[i]) : "l"(m2));                     // FADD2
      if (MODE == 3) asm volatile("add.rn.f32 %0, %0, %1;" : "+f"(a[i]) : "f"(mm));                       // FADD
      if (MODE == 4) { uint32_t r; asm volatile("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(a[i]), "f"(a[(i + 1) % NCH]));
                       a[i] = __uint_as_float(r); }                                                       // F2FP (dependent)
      if (MODE == 5) asm volatile("mad.lo.u32 %0, %0, 8388608, %1;" : "+r"(u[i]) : "r"(u[(i + 3) % NCH]));  // IMAD
      if (MODE == 6) asm volatile("max.f32 %0, %0, %1;" : "+f"(a[i]) : "f"(a[(i + 1) % NCH]));            // FMNMX
      if (MODE == 7) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a[i]));                             // MUFU
      if (MODE == 8) asm volatile("fma.rn.f32 %0, %0, 0f3F800001, %1;" : "+f"(a[i]) : "f"(mm));           // FFMA imm b
    }
  }
  unsigned long long t1 = clock64();
  float s = 0; for (int i = 0; i < NCH; ++i) { float x, y; asm("mov.b64 {%0,%1}, %2;" : "=f"(x), "=f"(y) : "l"(b[i])); s += a[i] + x + y + (float)u[i]; }
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = (float)(t1 - t0);
}

template <int M> float run(float* o, int w) {
  k<M><<<148, 128 * w>>>(o, 2048, 1.0001f, 1e-7f); k<M><<<148, 128 * w>>>(o, 2048, 1.0001f, 1e-7f);
  cudaDeviceSynchronize(); float c; cudaMemcpy(&c, o, 4, cudaMemcpyDeviceToHost);
  return c / (2048.0 * NCH * w);
}

int main() {
  float* o; cudaMalloc(&o, 148 * 1024 * 4);
  const char* n[] = {"FFMA 3-reg", "FFMA2 (f32x2)", "FADD2 (f32x2)", "FADD", "F2FP.BF16 pack", "IMAD", "FMNMX", "MUFU.EX2", "FFMA imm"};
  for (int w : {1, 2, 4}) {
    float r[9] = {run<0>(o, w), run<1>(o, w), run<2>(o, w), run<3>(o, w), run<4>(o, w), run<5>(o, w), run<6>(o, w), run<7>(o, w), run<8>(o, w)};
    for (int i = 0; i < 9; ++i) printf("warps/SMSP=%d %-16s %.2f cyc/warp-instr/SMSP\n", w, n[i], r[i]);
  }
  return 0;
}
