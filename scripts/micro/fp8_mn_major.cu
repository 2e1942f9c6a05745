// Does tcgen05.mma kind::f8f6f4 accept an MN-major B operand (the layout V has in P.V when V is
// stored [keys][dh])? One CTA: D[128x128] = A[128xK] . B[KxN], A K-major, B MN-major, 128B swizzle,
// e4m3 values in {-2,..,2} (exact), compared with a host reference. Prints max |diff|.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o fp8_mn_major fp8_mn_major.cu
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include "../../paper_2510_14719_b200/csrc/ws_aref.cuh"
using namespace ws;

constexpr int M = 128, N = 128, K = 128;

__device__ __forceinline__ uint32_t sw128(int row, int byte) {  // 128B-swizzled offset in a tile of 128-byte rows
  return (row / 8) * 1024 + (row % 8) * 128 + ((((byte / 16) ^ (row % 8)) & 7) * 16) + byte % 16;
}

__global__ void k(const uint8_t* a, const uint8_t* b, float* d, int b_mn_major) {
  __shared__ __align__(1024) uint8_t sa[M * K];
  __shared__ __align__(1024) uint8_t sb[K * N];
  __shared__ uint32_t tslot;
  __shared__ uint64_t bar;
  const int tid = threadIdx.x;
  for (int i = tid; i < M * K; i += blockDim.x) sa[sw128(i / K, i % K)] = a[i];  // A[m][k], K-major
  for (int i = tid; i < K * N; i += blockDim.x) {
    const int kk = i / N, n = i % N;  // B[k][n]
    if (b_mn_major)
      sb[sw128(kk, n)] = b[i];  // rows = k, 128 bytes of n each
    else
      sb[sw128(n, kk)] = b[i];  // rows = n, 128 bytes of k each
  }
  if (tid < 32) { tmem_alloc<1>(&tslot, 128); tmem_relinquish<1>(); }
  if (tid == 32) { mbar_init(&bar, 1); fence_barrier_init(); }
  fence_proxy_async_smem();
  tc_fence_before(); __syncthreads(); tc_fence_after();
  const uint32_t tmem = tslot;
  if (tid < 32) {
    const uint32_t idesc = make_idesc(0, M, N, 0, b_mn_major ? 1 : 0);
    for (int kk = 0; kk < K / 32; ++kk) {
      const uint64_t ad = make_sw128_desc(smem_u32(sa) + kk * 32, 16, 1024);
      const uint64_t bd = b_mn_major ? make_sw128_desc(smem_u32(sb) + kk * 32 * 128, 16384, 1024)
                                     : make_sw128_desc(smem_u32(sb) + kk * 32, 16, 1024);
      if (tid == 0) mma_f8_ss<1>(tmem, ad, bd, idesc, kk != 0);
    }
    __syncwarp();
    if (tid == 0) mma_commit(&bar);
  }
  mbar_wait(&bar, 0, 1);
  tc_fence_after();
  const int w = tid / 32, lane = tid % 32;
  uint32_t v[32];
  for (int c0 = 0; c0 < N; c0 += 32) {
    tmem_ld32(tmem + ((w * 32u) << 16) + c0, v);
    tmem_wait_ld();
    for (int j = 0; j < 32; ++j) d[(w * 32 + lane) * N + c0 + j] = __uint_as_float(v[j]);
  }
  tc_fence_before(); __syncthreads();
  if (tid < 32) { tc_fence_after(); tmem_dealloc<1>(tmem, 128); }
}

static uint8_t e4m3(int x) {  // exact e4m3 encodings of -2..2
  switch (x) { case 0: return 0x00; case 1: return 0x38; case 2: return 0x40; case -1: return 0xB8; default: return 0xC0; }
}

int main() {
  uint8_t *ha = (uint8_t*)malloc(M * K), *hb = (uint8_t*)malloc(K * N);
  int *ia = (int*)malloc(M * K * 4), *ib = (int*)malloc(K * N * 4);
  srand(7);
  for (int i = 0; i < M * K; ++i) { ia[i] = rand() % 5 - 2; ha[i] = e4m3(ia[i]); }
  for (int i = 0; i < K * N; ++i) { ib[i] = rand() % 5 - 2; hb[i] = e4m3(ib[i]); }
  uint8_t *da, *db; float* dd;
  cudaMalloc(&da, M * K); cudaMalloc(&db, K * N); cudaMalloc(&dd, M * N * 4);
  cudaMemcpy(da, ha, M * K, cudaMemcpyHostToDevice); cudaMemcpy(db, hb, K * N, cudaMemcpyHostToDevice);
  float* hd = (float*)malloc(M * N * 4);
  for (int mn = 0; mn < 2; ++mn) {
    cudaMemset(dd, 0, M * N * 4);
    k<<<1, 128>>>(da, db, dd, mn);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(hd, dd, M * N * 4, cudaMemcpyDeviceToHost);
    double md = 0;
    for (int m = 0; m < M; ++m)
      for (int n = 0; n < N; ++n) {
        int s = 0;
        for (int kk = 0; kk < K; ++kk) s += ia[m * K + kk] * ib[kk * N + n];
        md = fmax(md, fabs(hd[m * N + n] - s));
      }
    printf("B %s-major: %s max|diff| = %g\n", mn ? "MN" : "K", cudaGetErrorString(e), md);
  }
  return 0;
}
