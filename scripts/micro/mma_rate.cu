// tcgen05.mma issue-to-completion rate for the attention operand shapes (bf16, fp32 accumulate):
// SS (A and B from shared memory) at M=128, N in {64, 128, 256}, K=16 per instruction; TS (A from
// TMEM) at N in {64, 128}; optionally with 4 warps streaming st.shared traffic (the P stores of a
// softmax that writes P to shared memory). Cycles per MMA = the operand-feed bound.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o mma_rate mma_rate.cu
#include <cstdio>
#include "../../paper_2510_14719_b200/csrc/ws_aref.cuh"
using namespace ws;

template <int N, bool TS, bool STS, int NSTS_WARPS = 4>
__global__ void __launch_bounds__(256, 1) k(float* out, int iters) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint32_t tslot;
  __shared__ uint64_t bar;
  __shared__ volatile int done;
  __shared__ unsigned long long nsts;
  const uint32_t warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  for (int i = threadIdx.x; i < 96 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0x3c003c00u;
  if (warp == 0) { tmem_alloc<1>(&tslot, 512); tmem_relinquish<1>(); }
  if (threadIdx.x == 32) { mbar_init(&bar, 1); fence_barrier_init(); done = 0; nsts = 0; }
  fence_proxy_async_smem();
  tc_fence_before(); __syncthreads(); tc_fence_after();
  const uint32_t tmem = tslot;
  constexpr uint32_t IDESC = make_idesc(1, 128, N, 0, 0);
  if (warp == 1) {
    const uint64_t ad = make_sw128_desc(smem_u32(smem), 16, 1024);
    const uint64_t bd = make_sw128_desc(smem_u32(smem + 32768), 16, 1024);
    unsigned long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int kk = 0; kk < 8; ++kk) {
        const uint32_t off = ((kk / 4) * 16384 + (kk % 4) * 32) >> 4;
        if (TS)
          mma_f16_ts_warp(tmem + 256, tmem + kk * 8, bd + off, IDESC, 1);
        else
          mma_f16_ss_warp(tmem, ad + off, bd + off, IDESC, 1);
      }
    }
    mma_commit_warp(&bar);
    mbar_wait(&bar, 0, 1);
    unsigned long long t1 = clock64();
    if (lane == 0 && blockIdx.x == 0) { out[0] = (float)(t1 - t0) / (iters * 8.0); out[1] = (float)(t1 - t0); }
    if (lane == 0) done = 1;
  } else if (STS && warp >= 4) {
    // P-store traffic for the whole MMA run: 16 B per thread per instruction into the upper 32 KB
    // (NSTS_WARPS warps); counts the bytes stored while the MMAs ran
    const uint32_t base = smem_u32(smem + 65536) + (threadIdx.x - 128) * 16;
    unsigned long long n = 0;
    if (warp < 4 + NSTS_WARPS) {
      while (!done) {
#pragma unroll
        for (int r = 0; r < 8; ++r) st_shared_v4(base + ((r * 2048 + (int)n * 16) & 16383), (uint32_t)n, r, 0, 1);
        n += 8;
      }
      if (lane == 0) atomicAdd(&nsts, n * 32 * 16);
    }
  }
  __syncthreads();
  if (threadIdx.x == 0 && blockIdx.x == 0) out[2] = (float)nsts;
  tc_fence_before(); __syncthreads();
  if (warp == 0) { tc_fence_after(); tmem_dealloc<1>(tslot, 512); }
}

template <int N, bool TS, bool STS, int NW = 4>
void run(float* o, const char* name) {
  auto kern = k<N, TS, STS, NW>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  kern<<<148, 256, 100 * 1024>>>(o, 4000);
  kern<<<148, 256, 100 * 1024>>>(o, 4000);
  cudaError_t e = cudaDeviceSynchronize();
  float r[3] = {0, 0, 0}; cudaMemcpy(r, o, 12, cudaMemcpyDeviceToHost);
  const float c = r[0];
  const double ideal = 128.0 * N / 256.0;
  printf("%-22s N=%3d sts_warps=%d: %6.1f cycles/MMA (tensor floor %5.1f, %.0f%%), st.shared %.1f B/clk %s\n", name, N,
         STS ? NW : 0, c, ideal, 100 * ideal / c, STS ? r[2] / r[1] : 0.f, e == cudaSuccess ? "" : cudaGetErrorString(e));
}

int main() {
  float* o; cudaMalloc(&o, 64);
  run<128, false, false>(o, "SS");
  run<128, false, true, 1>(o, "SS + st.shared");
  run<128, false, true, 2>(o, "SS + st.shared");
  run<128, false, true, 4>(o, "SS + st.shared");
  run<256, false, true, 4>(o, "SS + st.shared");
  run<128, true, false>(o, "TS");
  run<128, true, true, 1>(o, "TS + st.shared");
  run<128, true, true, 4>(o, "TS + st.shared");
  return 0;
}
