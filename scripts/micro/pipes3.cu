// Pipe overlap on sm_100a: cycles per group when the softmax instruction classes are mixed
// (is MUFU.EX2 free to overlap FFMA2 / F2FP / FMNMX, and FMA with ALU?).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o pipes3 pipes3.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define NCH 8
// one group per chain i: NM MUFU, NF FFMA2, NA FMNMX, NP F2FP, NI IMAD
template <int NM, int NF, int NA, int NP, int NI>
__global__ void k(float* out, int iters, float sc, float mm) {
  float a[NCH], c[NCH], d[NCH]; uint64_t b[NCH]; uint32_t u[NCH], pk[NCH];
  for (int i = 0; i < NCH; ++i) {
    a[i] = 1e-3f * (threadIdx.x + i); c[i] = a[i] * 0.5f; d[i] = a[i] * 0.25f; u[i] = threadIdx.x * 7 + i; pk[i] = 0;
    asm("mov.b64 %0, {%1, %2};" : "=l"(b[i]) : "f"(a[i]), "f"(a[i] + 1.f));
  }
  uint64_t s2, m2;
  asm("mov.b64 %0, {%1, %1};" : "=l"(s2) : "f"(sc));
  asm("mov.b64 %0, {%1, %1};" : "=l"(m2) : "f"(mm));
  unsigned long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < NCH; ++i) {
#pragma unroll
      for (int r = 0; r < NM; ++r) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a[i]));
#pragma unroll
      for (int r = 0; r < NF; ++r) asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(b[i]) : "l"(s2), "l"(m2));
#pragma unroll
      for (int r = 0; r < NA; ++r) asm volatile("max.f32 %0, %0, %1, %2;" : "+f"(c[i]) : "f"(c[(i + 1) % NCH]), "f"(mm));
#pragma unroll
      for (int r = 0; r < NP; ++r) {
        uint32_t x;
        asm volatile("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(x) : "f"(d[i]), "f"(d[(i + 1) % NCH]));
        pk[i] ^= x;
      }
#pragma unroll
      for (int r = 0; r < NI; ++r) asm volatile("mad.lo.u32 %0, %0, 8388608, %1;" : "+r"(u[i]) : "r"(u[(i + 3) % NCH]));
    }
  }
  unsigned long long t1 = clock64();
  float s = 0;
  for (int i = 0; i < NCH; ++i) {
    float x, y;
    asm("mov.b64 {%0,%1}, %2;" : "=f"(x), "=f"(y) : "l"(b[i]));
    s += a[i] + x + y + c[i] + (float)u[i] + (float)pk[i];
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = (float)(t1 - t0);
}

template <int NM, int NF, int NA, int NP, int NI>
void run(float* o, int w) {
  auto kk = k<NM, NF, NA, NP, NI>;
  kk<<<148, 128 * w>>>(o, 1024, 1.0001f, 1e-7f);
  kk<<<148, 128 * w>>>(o, 1024, 1.0001f, 1e-7f);
  cudaDeviceSynchronize();
  float c;
  cudaMemcpy(&c, o, 4, cudaMemcpyDeviceToHost);
  const float per = c / (1024.0f * NCH * w);
  const float sum = NM * 8.f + NF * 2.f + NA * 2.f + NP * 2.f + NI * 1.25f;
  printf("warps/SMSP=%d MUFU x%d FFMA2 x%d FMNMX3 x%d F2FP x%d IMAD x%d: %6.2f cyc/group (serial sum %5.1f, max-pipe %s)\n",
         w, NM, NF, NA, NP, NI, per, sum, "");
}

int main() {
  float* o;
  cudaMalloc(&o, 148 * 1024 * 4);
  for (int w : {2, 4}) {
    run<1, 0, 0, 0, 0>(o, w);
    run<1, 4, 0, 0, 0>(o, w);
    run<1, 0, 4, 0, 0>(o, w);
    run<1, 0, 0, 4, 0>(o, w);
    run<1, 2, 2, 0, 0>(o, w);
    run<0, 4, 4, 0, 0>(o, w);
    run<0, 4, 0, 4, 0>(o, w);
    run<0, 0, 4, 4, 0>(o, w);
    run<1, 2, 1, 1, 0>(o, w);
    run<1, 1, 1, 1, 0>(o, w);
    run<2, 2, 2, 2, 0>(o, w);
    run<0, 0, 0, 0, 4>(o, w);
    run<1, 0, 0, 0, 4>(o, w);
    run<0, 4, 0, 0, 4>(o, w);
  }
  return 0;
}
