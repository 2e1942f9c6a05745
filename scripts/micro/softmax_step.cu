// One FA softmax step in isolation (TMEM load of S, row max, exp mix, row sum, pack, TMEM store of P),
// NW warps per SMSP, COLS columns per thread. Reports cycles per step per warp, i.e. the latency a
// Q tile's softmax adds to the T->C->U chain when NW warps share the SMSP.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o softmax_step softmax_step.cu
#include <cstdio>
#include "../../paper_2510_14719_b200/csrc/attn_sm100.cuh"
using namespace ws;

__device__ __forceinline__ float fmax3_(float a, float b, float c) {
  float d;
  asm("max.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c));
  return d;
}

template <int COLS, int POLY, bool XCHG, int NW, int ILP = 0, bool NOSUM = false>
__global__ void __launch_bounds__(128 * NW, 1) k(float* out, int steps) {
  __shared__ uint32_t tslot;
  __shared__ float xm[2][16][32];
  const uint32_t warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (warp == 0) { tmem_alloc<1>(&tslot, 512); tmem_relinquish<1>(); }
  tc_fence_before(); __syncthreads(); tc_fence_after();
  const uint32_t tmem = tslot + (((warp & 3) * 32u) << 16) + (warp >> 2) * COLS;
  {
    uint32_t z[32];
    for (int c = 0; c < 32; ++c) z[c] = __float_as_uint(-0.01f * (c + lane) + 0.001f * warp);
    for (int c0 = 0; c0 < COLS; c0 += 32) tmem_st32(tmem + c0, z);
    tmem_wait_st();
  }
  float sl2 = 0.12f, m_used = -INFINITY, l = 0.f;
  unsigned long long t0 = clock64();
  for (int j = 0; j < steps; ++j) {
    float s[COLS];
    uint32_t* su = reinterpret_cast<uint32_t*>(s);
#pragma unroll
    for (int c0 = 0; c0 < COLS; c0 += 32) tmem_ld32(tmem + c0, *reinterpret_cast<uint32_t(*)[32]>(su + c0));
    tmem_wait_ld();
    float mx;
    if (ILP == 0) {
      float m4[4] = {fmax3_(s[0], s[1], s[2]), fmax3_(s[3], s[4], s[5]), fmax3_(s[6], s[7], s[8]), fmax3_(s[9], s[10], s[11])};
#pragma unroll
      for (int c = 12; c + 8 <= COLS; c += 8) {
        m4[0] = fmax3_(m4[0], s[c], s[c + 1]);
        m4[1] = fmax3_(m4[1], s[c + 2], s[c + 3]);
        m4[2] = fmax3_(m4[2], s[c + 4], s[c + 5]);
        m4[3] = fmax3_(m4[3], s[c + 6], s[c + 7]);
      }
      m4[0] = fmax3_(m4[0], s[COLS - 4], s[COLS - 3]);
      m4[1] = fmax3_(m4[1], s[COLS - 2], s[COLS - 1]);
      mx = fmaxf(fmaxf(m4[0], m4[1]), fmaxf(m4[2], m4[3]));
    } else {
      // 8 independent chains over 16-column groups, then a 3-level tree
      float m8[8];
#pragma unroll
      for (int g = 0; g < 8; ++g) m8[g] = fmax3_(s[2 * g], s[2 * g + 1], s[16 + 2 * g]);
#pragma unroll
      for (int c = 32; c < COLS; c += 32)
#pragma unroll
        for (int g = 0; g < 8; ++g) m8[g] = fmax3_(m8[g], s[c + 2 * g], s[c + 2 * g + 1]);
#pragma unroll
      for (int g = 0; g < 8; ++g) m8[g] = fmax3_(m8[g], s[16 + 2 * g + 1], m8[g]);
#pragma unroll
      for (int c = 48; c < COLS; c += 32)
#pragma unroll
        for (int g = 0; g < 8; ++g) m8[g] = fmax3_(m8[g], s[c + 2 * g], s[c + 2 * g + 1]);
      mx = fmax3_(fmax3_(m8[0], m8[1], m8[2]), fmax3_(m8[3], m8[4], m8[5]), fmaxf(m8[6], m8[7]));
    }
    if (XCHG) {
      // partner warp (warp ^ 4) holds the other column half of the same rows
      // double-buffered by step parity: one barrier per step keeps the buffers race-free
      xm[j & 1][warp][lane] = mx;
      asm volatile("bar.sync %0, 64;" ::"r"(1 + (warp & 3) + 4 * (warp >> 3)));
      mx = fmaxf(mx, xm[j & 1][warp ^ 4][lane]);
    }
    const float m_blk = mx * sl2;
    float alpha = 1.f;
    if (m_blk > m_used + 8.f) { alpha = ex2_approx(m_used - m_blk); m_used = m_blk; }
    l *= alpha;
    const uint64_t sl2x2 = f2_pack(sl2, sl2), negm2 = f2_pack(-m_used, -m_used);
    uint64_t sa = f2_pack(0.f, 0.f), sb = f2_pack(0.f, 0.f), sc4[4] = {sa, sa, sa, sa};
#pragma unroll
    for (int c0 = 0; c0 < COLS; c0 += 32) {
      uint32_t pk[16];
#pragma unroll
      for (int c = c0; c < c0 + 32; c += 2) {
        const uint64_t x2 = f2_fma(f2_pack(s[c], s[c + 1]), sl2x2, negm2);
        uint64_t p2;
        if (attn_poly_pair(POLY, (c / 2) & 7)) p2 = exp2_poly2(x2);
        else { float x0, x1; f2_unpack(x2, x0, x1); p2 = f2_pack(ex2_approx(x0), ex2_approx(x1)); }
        if (NOSUM) {}
        else if (ILP) sc4[(c / 2) & 3] = f2_add(sc4[(c / 2) & 3], p2);
        else if ((c / 2) & 1) sb = f2_add(sb, p2); else sa = f2_add(sa, p2);
        float p0, p1; f2_unpack(p2, p0, p1);
        pk[(c - c0) / 2] = pack_bf16(p0, p1);
      }
      tmem_st16(tmem + c0 / 2, pk);
    }
    if (ILP) { sa = f2_add(sc4[0], sc4[1]); sb = f2_add(sc4[2], sc4[3]); }
    float a, b, c2, d2; f2_unpack(sa, a, b); f2_unpack(sb, c2, d2);
    l += (a + b) + (c2 + d2);
    tmem_wait_st();
    sl2 += 1e-9f * l;  // loop-carried
  }
  unsigned long long t1 = clock64();
  if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = (float)(t1 - t0) / steps;
  if (l == 12345.f) out[2] = l;
  tc_fence_before(); __syncthreads();
  if (warp == 0) { tc_fence_after(); tmem_dealloc<1>(tslot, 512); }
}


// Speculative split-row step: COLS columns per warp (a row's other half lives in warp ^ 8), the
// exponentials run against the running max m_used while the block max is computed alongside (no
// serial max phase); the per-row rescale decision is exchanged with the partner warp through a
// tagged shared-memory slot read after the exponentials (no barrier).
template <int COLS, int POLY, int NW>
__global__ void __launch_bounds__(128 * NW, 1) kspec(float* out, int steps) {
  __shared__ uint32_t tslot;
  __shared__ unsigned long long xs[2][16][32];
  const uint32_t warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (warp == 0) { tmem_alloc<1>(&tslot, 512); tmem_relinquish<1>(); }
  if (threadIdx.x < 16 * 32) { xs[0][threadIdx.x / 32][threadIdx.x % 32] = ~0ull; xs[1][threadIdx.x / 32][threadIdx.x % 32] = ~0ull; }
  tc_fence_before(); __syncthreads(); tc_fence_after();
  const uint32_t tmem = tslot + (((warp & 3) * 32u) << 16) + (warp >> 2) * COLS;
  {
    uint32_t z[32];
    for (int c = 0; c < 32; ++c) z[c] = __float_as_uint(-0.01f * (c + lane) + 0.001f * warp);
    for (int c0 = 0; c0 < COLS; c0 += 32) tmem_st32(tmem + c0, z);
    tmem_wait_st();
  }
  float sl2 = 0.12f, m_used = 0.f, l = 0.f;
  unsigned long long t0 = clock64();
  for (int j = 0; j < steps; ++j) {
    float s[COLS];
    uint32_t* su = reinterpret_cast<uint32_t*>(s);
#pragma unroll
    for (int c0 = 0; c0 < COLS; c0 += 32) tmem_ld32(tmem + c0, *reinterpret_cast<uint32_t(*)[32]>(su + c0));
    tmem_wait_ld();
    const uint64_t sl2x2 = f2_pack(sl2, sl2), negm2 = f2_pack(-m_used, -m_used);
    uint64_t sc4[4] = {f2_pack(0.f, 0.f), f2_pack(0.f, 0.f), f2_pack(0.f, 0.f), f2_pack(0.f, 0.f)};
    float m4[4] = {s[0], s[1], s[2], s[3]};
#pragma unroll
    for (int c0 = 0; c0 < COLS; c0 += 32) {
      uint32_t pk[16];
#pragma unroll
      for (int c = c0; c < c0 + 32; c += 2) {
        if ((c & 7) == 0 && c >= 4) {
          m4[0] = fmax3_(m4[0], s[c], s[c + 1]);
          m4[1] = fmax3_(m4[1], s[c + 2], s[c + 3]);
          m4[2] = fmax3_(m4[2], s[c + 4], s[c + 5]);
          m4[3] = fmax3_(m4[3], s[c + 6], s[c + 7]);
        }
        const uint64_t x2 = f2_fma(f2_pack(s[c], s[c + 1]), sl2x2, negm2);
        uint64_t p2;
        if (attn_poly_pair(POLY, (c / 2) & 7)) p2 = exp2_poly2(x2);
        else { float x0, x1; f2_unpack(x2, x0, x1); p2 = f2_pack(ex2_approx(x0), ex2_approx(x1)); }
        sc4[(c / 2) & 3] = f2_add(sc4[(c / 2) & 3], p2);
        float p0, p1; f2_unpack(p2, p0, p1);
        pk[(c - c0) / 2] = pack_bf16(p0, p1);
      }
      tmem_st16(tmem + c0 / 2, pk);
    }
    const float mx = fmaxf(fmaxf(m4[0], m4[1]), fmaxf(m4[2], m4[3])) * sl2;
    // publish (step, max); read the partner's, spin until its step tag matches
    const unsigned long long mine = (static_cast<unsigned long long>(j) << 32) | __float_as_uint(mx);
    // double-buffered by step parity: a warp can be at most one step ahead of its partner
    *reinterpret_cast<volatile unsigned long long*>(&xs[j & 1][warp][lane]) = mine;
    unsigned long long th;
    int spins = 0;
    do { th = *reinterpret_cast<volatile unsigned long long*>(&xs[j & 1][warp ^ 8][lane]); } while ((th >> 32) != (unsigned)j && ++spins < (1 << 22));
    const float mo = __uint_as_float(static_cast<uint32_t>(th));
    if (fmaxf(mx, mo) > m_used + 64.f) m_used = fmaxf(mx, mo);  // rare path (never taken here)
    float a, b, c2, d2; f2_unpack(f2_add(sc4[0], sc4[1]), a, b); f2_unpack(f2_add(sc4[2], sc4[3]), c2, d2);
    l += (a + b) + (c2 + d2);
    tmem_wait_st();
    sl2 += 1e-9f * l;
  }
  unsigned long long t1 = clock64();
  if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = (float)(t1 - t0) / steps;
  if (l == 12345.f) out[2] = l;
  tc_fence_before(); __syncthreads();
  if (warp == 0) { tc_fence_after(); tmem_dealloc<1>(tslot, 512); }
}

template <int COLS, int POLY, int NW>
void runspec(float* o, const char* name) {
  const int steps = 2000;
  kspec<COLS, POLY, NW><<<148, 128 * NW>>>(o, steps);
  kspec<COLS, POLY, NW><<<148, 128 * NW>>>(o, steps);
  cudaError_t e = cudaDeviceSynchronize();
  float c = 0; cudaMemcpy(&c, o, 4, cudaMemcpyDeviceToHost);
  printf("%-28s warps/SMSP=%d cols=%3d: %7.1f cycles/step/warp, %6.1f cycles per SMSP per 128 cols %s\n", name, NW,
         COLS, c, c / (NW * COLS / 128.0), e == cudaSuccess ? "" : cudaGetErrorString(e));
}

template <int COLS, int POLY, bool XCHG, int NW, int ILP = 0, bool NOSUM = false>
void run1(float* o, const char* name) {
  const int steps = 2000, nw = NW;
  k<COLS, POLY, XCHG, NW, ILP, NOSUM><<<148, 128 * nw>>>(o, steps);
  k<COLS, POLY, XCHG, NW, ILP, NOSUM><<<148, 128 * nw>>>(o, steps);
  cudaError_t e = cudaDeviceSynchronize();
  float c = 0; cudaMemcpy(&c, o, 4, cudaMemcpyDeviceToHost);
  printf("%-28s warps/SMSP=%d cols=%3d: %7.1f cycles/step/warp, %6.1f cycles per SMSP per 128 cols %s\n", name, nw,
         COLS, c, c / (nw * COLS / 128.0), e == cudaSuccess ? "" : cudaGetErrorString(e));
}

template <int COLS, int POLY, bool XCHG>
void run(float* o, int nw, const char* name) {
  if (nw == 1) run1<COLS, POLY, XCHG, 1>(o, name);
  if (nw == 2) run1<COLS, POLY, XCHG, 2>(o, name);
  if (nw == 3) run1<COLS, POLY, XCHG, 3>(o, name);
  if (nw == 4) run1<COLS, POLY, XCHG, 4>(o, name);
}

int main(int argc, char** argv) {
  float* o; cudaMalloc(&o, 64);
  if (argc > 1) {  // warps-per-SMSP sweep at 128 columns (3 or 4 Q tiles per CTA instead of 2)
    run1<128, 1, false, 1, 1>(o, "1w x128 POLY=1");
    run1<128, 2, false, 1, 1>(o, "1w x128 POLY=2");
    run1<128, 1, false, 2, 1>(o, "2w x128 POLY=1");
    run1<128, 2, false, 2, 1>(o, "2w x128 POLY=2");
    run1<128, 3, false, 2, 1>(o, "2w x128 POLY=3");
    run1<128, 1, false, 3, 1>(o, "3w x128 POLY=1");
    run1<128, 2, false, 3, 1>(o, "3w x128 POLY=2");
    run1<128, 3, false, 3, 1>(o, "3w x128 POLY=3");
    run1<128, 1, false, 4, 1>(o, "4w x128 POLY=1");
    run1<128, 2, false, 4, 1>(o, "4w x128 POLY=2");
    run1<128, 3, false, 4, 1>(o, "4w x128 POLY=3");
    return 0;
  }
  run1<128, 1, false, 2, 1>(o, "2w x128 POLY=1");
  run1<128, 2, false, 2, 1>(o, "2w x128 POLY=2");
  run1<128, 3, false, 2, 1>(o, "2w x128 POLY=3");
  runspec<64, 1, 4>(o, "spec 4w x64 POLY=1");
  runspec<64, 2, 4>(o, "spec 4w x64 POLY=2");
  runspec<64, 3, 4>(o, "spec 4w x64 POLY=3");
  run1<64, 2, true, 4, 1>(o, "4w x64 xchg POLY=2");
  return 0;
}
