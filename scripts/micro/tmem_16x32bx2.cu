// Layout check of tcgen05.ld.16x32bx2 (two 16-lane halves, the upper half offset by immHalfSplitoff
// columns): thread t should read lane (base + t % 16), columns col + (t / 16) * SPLIT + i.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tmem_16x32bx2 tmem_16x32bx2.cu
#include <cstdio>
#include "../../paper_2510_14719_b200/csrc/ws_aref.cuh"
using namespace ws;

__global__ void k(int* bad, int* sample) {
  __shared__ uint32_t tslot;
  const uint32_t warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (warp == 0) { tmem_alloc<1>(&tslot, 512); tmem_relinquish<1>(); }
  tc_fence_before(); __syncthreads(); tc_fence_after();
  const uint32_t tmem = tslot;
  // every warp writes its lane quarter: value = lane * 1000 + column
  const uint32_t q = warp & 3;
  for (int c0 = 0; c0 < 256; c0 += 32) {
    uint32_t v[32];
    for (int i = 0; i < 32; ++i) v[i] = (q * 32 + lane) * 1000 + c0 + i;
    tmem_st32(tmem + ((q * 32) << 16) + c0, v);
  }
  tmem_wait_st();
  tc_fence_before(); __syncthreads(); tc_fence_after();
  // warps 0-3: lanes 32q + 0..15; warps 4-7: lanes 32q + 16..31
  const uint32_t r = warp >> 2;
  const uint32_t taddr = tmem + ((q * 32 + r * 16) << 16) + 32;
  uint32_t v[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.16x32bx2.x32.b32 "
      "{%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, "
      "%16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32], 64;"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
        "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]),
        "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]),
        "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
      : "r"(taddr));
  tmem_wait_ld();
  int nbad = 0;
  for (int i = 0; i < 32; ++i) {
    const uint32_t want = (q * 32 + r * 16 + lane % 16) * 1000 + 32 + (lane / 16) * 64 + i;
    if (v[i] != want) ++nbad;
  }
  atomicAdd(bad, nbad);
  if (warp == 5 && lane == 17) for (int i = 0; i < 4; ++i) sample[i] = v[i];
  tc_fence_before(); __syncthreads();
  if (warp == 0) { tc_fence_after(); tmem_dealloc<1>(tmem, 512); }
}

int main() {
  int *bad, *sample; cudaMalloc(&bad, 4); cudaMalloc(&sample, 16); cudaMemset(bad, 0, 4);
  k<<<1, 256>>>(bad, sample);
  cudaError_t e = cudaDeviceSynchronize();
  int hb, hs[4]; cudaMemcpy(&hb, bad, 4, cudaMemcpyDeviceToHost); cudaMemcpy(hs, sample, 16, cudaMemcpyDeviceToHost);
  printf("16x32bx2 layout: %d mismatches (%s); warp 5 lane 17 got %d %d %d %d (want lane %d cols %d..)\n", hb,
         cudaGetErrorString(e), hs[0], hs[1], hs[2], hs[3], 1 * 32 + 16 + 1, 32 + 64);
  return 0;
}
