// Does ncu's l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st count address conflicts only, or
// also LSU stores that lose shared-memory arbitration to the tensor pipe's operand reads? Four warps
// issue a provably conflict-free st.shared.v4 stream (8 consecutive threads cover 128 contiguous
// bytes) for a fixed time while warp 1 either issues tcgen05.mma SS (M=128, N=256, operands in
// shared memory) or just spins. Run each variant under
//   ncu --metrics l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum,\
//       l1tex__data_pipe_lsu_wavefronts_mem_shared_op_st.sum,smsp__sass_inst_executed_op_shared_st.sum,\
//       l1tex__data_pipe_tc_wavefronts_mem_shared.sum ./sts_vs_tc {0|1}
// (0 = stores alone, 1 = stores + MMA). Same store pattern in both, so any difference in the
// "conflict" counter is arbitration against the tensor pipe, not addressing.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o sts_vs_tc sts_vs_tc.cu
#include <cstdio>
#include <cstdlib>
#include "../../paper_2510_14719_b200/csrc/ws_aref.cuh"
using namespace ws;

template <bool MMA>
__global__ void __launch_bounds__(256, 1) k(float* out, int iters) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint32_t tslot;
  __shared__ uint64_t bar;
  __shared__ volatile int done;
  const uint32_t warp = threadIdx.x / 32;
  for (int i = threadIdx.x; i < 96 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0x3c003c00u;
  if (warp == 0) { tmem_alloc<1>(&tslot, 512); tmem_relinquish<1>(); }
  if (threadIdx.x == 32) { mbar_init(&bar, 1); fence_barrier_init(); done = 0; }
  fence_proxy_async_smem();
  tc_fence_before(); __syncthreads(); tc_fence_after();
  const uint32_t tmem = tslot;
  constexpr uint32_t IDESC = make_idesc(1, 128, 256, 0, 0);
  if (warp == 1) {
    const unsigned long long t0 = clock64();
    if (MMA) {
      const uint64_t ad = make_sw128_desc(smem_u32(smem), 16, 1024);
      const uint64_t bd = make_sw128_desc(smem_u32(smem + 32768), 16, 1024);
      for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          const uint32_t off = ((kk / 4) * 16384 + (kk % 4) * 32) >> 4;
          mma_f16_ss_warp(tmem, ad + off, bd + off, IDESC, 1);
        }
      }
      mma_commit_warp(&bar);
      mbar_wait(&bar, 0, 1);
    } else {
      // the MMA run's length (128 cycles per N=256 MMA at the tensor floor), spent spinning
      while (clock64() - t0 < (unsigned long long)iters * 8 * 128) { }
    }
    if (threadIdx.x == 32 && blockIdx.x == 0) out[0] = (float)(clock64() - t0);
    if (threadIdx.x == 32) done = 1;
  } else if (warp >= 4) {
    const uint32_t base = smem_u32(smem + 65536) + (threadIdx.x - 128) * 16;
    uint32_t n = 0;
    while (!done) {
#pragma unroll
      for (int r = 0; r < 8; ++r) st_shared_v4(base + ((r * 2048 + n * 16) & 16383), n, r, 0, 1);
      n += 8;
    }
    if (threadIdx.x == 128 && blockIdx.x == 0) out[1] = (float)n;
  }
  tc_fence_before(); __syncthreads();
  if (warp == 0) { tc_fence_after(); tmem_dealloc<1>(tslot, 512); }
}

int main(int argc, char** argv) {
  const int mode = argc > 1 ? atoi(argv[1]) : 1;
  float* o; cudaMalloc(&o, 64);
  auto kern = mode ? k<true> : k<false>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  kern<<<148, 256, 100 * 1024>>>(o, 2000);
  cudaError_t e = cudaDeviceSynchronize();
  float r[2] = {0, 0}; cudaMemcpy(r, o, 8, cudaMemcpyDeviceToHost);
  printf("mode=%d (%s): %.0f cycles, %.0f store iterations per thread %s\n", mode, mode ? "stores + MMA" : "stores alone",
         r[0], r[1], e == cudaSuccess ? "" : cudaGetErrorString(e));
  return 0;
}
