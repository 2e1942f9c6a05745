// attn_sm100.cuh — warp-specialized FlashAttention forward for sm_100a.
//
// Reference semantics: the flash .k of SURVEY.md Appendix A, i.e. the coarse T/C/U pipeline of
// the reference compiler (identify_stages / apply_coarse_grained,
// ref proj/include/warpspec/pipeline.hpp:160-328; schedule ref schedule.hpp:18-74):
//   T  (tensor)  S_j = Q . K_j^T                      -> tcgen05.mma into TMEM
//   C  (compute) m, l, P_j = exp(S_j*sc - m), rescale  -> softmax warps (TMEM -> regs -> TMEM)
//   U  (update)  O += P_j . V_j                         -> tcgen05.mma, A = P from TMEM
// with o = acc / l and lse = m + log(l) produced in the epilogue.
//
// CTA work item: one (b,h) slice x 256 query rows = two 128-row Q tiles (the cooperative
// consumer row bands of ref proj/include/warpspec/grid.hpp:24-72: two softmax warpgroups share
// one K/V ring, and a K/V slot is released only after both bands' MMAs have read it).
// Warp roles:
//   warp 0       TMA producer: Q0,Q1 once, then K_j, V_j into a depth-D smem aref
//   warp 1       MMA issuer (one thread): QK_j[t] -> S_t, PV_j[t] -> O_t
//   warp 2       TMEM allocator
//   warps 4..7   softmax/correction/epilogue for Q tile 0 (thread = query row = TMEM lane)
//   warps 8..11  same for Q tile 1
// TMEM (512 columns): S_0 | S_1 | O_0 | O_1. P_t (bf16, 2 per column) is written over the first
// half of S_t once the row has been read into registers; tcgen05 ops issued by one thread
// execute in order, so QK_{j+1}[t] (which overwrites S_t) is issued after PV_j[t] (which reads
// P_t) and the hazard is ordered by the tensor pipe.
//
// The U stage of step j is issued only after C_j has written P_j (the hardware hazard noted in
// the reference can issue U_{j-1} before C_{j-1} because it materialises MMA values
// lazily; a real tensor core cannot). Overlap comes from the other Q tile: while the softmax
// warps of tile t run C_j, the tensor core runs U_j/T_{j+1} of tile 1-t.
#pragma once

#include <atomic>
#include <string>

#include "../../include/ws.h"
#include "ws_aref.cuh"

namespace ws {

constexpr int ATTN_BM = 128;  // query rows per Q tile (one TMEM lane each)
constexpr int ATTN_BN = 128;  // keys per K/V tile
constexpr int ATTN_THREADS = 384;
constexpr int ATTN_MAX_KV_STAGES = 8;
constexpr float ATTN_RESCALE_THRESHOLD = 8.0f;  // log2 units: P values stay <= 2^8 between rescales

struct AttnParams {
  int S, Dh, BH_begin, num_pairs;  // num_pairs = S / 256 work items per (b,h)
  int kv_stages;
  int causal;
  float scale_log2;  // softmax_scale * log2(e)
  float* lse;
  void* o;
  int o_elem;  // 0 = bf16, 1 = f16
};

__host__ __device__ inline uint32_t attn_tile_bytes(int Dh) { return ATTN_BM * Dh * 2; }

__host__ __device__ inline uint32_t attn_smem_bytes(int Dh, int kv_stages) {
  // Q0 | Q1 | kv slots | barriers (+1 KB alignment slack)
  return 2 * attn_tile_bytes(Dh) + kv_stages * attn_tile_bytes(Dh) + (2 * ATTN_MAX_KV_STAGES + 8) * 8 + 16 +
         1024;
}

template <int DH, bool BF16>
__global__ void __launch_bounds__(ATTN_THREADS, 1)
    ws_attn_fwd_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                       const __grid_constant__ CUtensorMap tm_v, const AttnParams p) {
  constexpr uint32_t TILE = ATTN_BM * DH * 2;      // bytes of a 128 x DH tile
  constexpr uint32_t HALF = ATTN_BM * 128;         // one 64-column (128 B) swizzle panel of a tile
  constexpr int NPANEL = DH / 64;
  constexpr uint32_t FMT = BF16 ? 1u : 0u;
  constexpr uint32_t IDESC_QK = make_idesc(FMT, ATTN_BM, ATTN_BN, 0, 0);
  constexpr uint32_t IDESC_PV = make_idesc(FMT, ATTN_BM, DH, 0, 1);  // B = V is MN-major
  constexpr uint32_t COL_S = 0, COL_O = 2 * ATTN_BN;

  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sq = smem;                  // Q0, Q1
  uint8_t* skv = smem + 2 * TILE;      // K/V ring
  uint8_t* bar_base = skv + p.kv_stages * TILE;
  auto* ring = reinterpret_cast<ArefBarriers<ATTN_MAX_KV_STAGES>*>(bar_base);
  uint64_t* q_full = reinterpret_cast<uint64_t*>(bar_base + 2 * ATTN_MAX_KV_STAGES * 8);
  uint64_t* s_full = q_full + 1;  // [2]: S_t (and everything before it) complete
  uint64_t* p_full = q_full + 3;  // [2]: P_t written (and O_t rescaled)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(q_full + 8);

  const uint32_t warp = warp_id();
  const uint32_t lane = lane_id();
  const uint32_t D = static_cast<uint32_t>(p.kv_stages);

  // work item: blockIdx.x = (b,h) slice (fastest), blockIdx.y = query pair, heaviest (latest,
  // for causal) pairs dispatched first
  const int pair = p.num_pairs - 1 - static_cast<int>(blockIdx.y);
  const int bh = p.BH_begin + static_cast<int>(blockIdx.x);
  const int q_row0 = bh * p.S + pair * 2 * ATTN_BM;  // row in the [B*H*S, Dh] view
  const int n_kv = p.causal ? (pair * 2 * ATTN_BM + 2 * ATTN_BM) / ATTN_BN : p.S / ATTN_BN;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tm_q);
    tma_prefetch_desc(&tm_k);
    tma_prefetch_desc(&tm_v);
    ring->init(D, 1, 1);
    mbar_init(q_full, 1);
    mbar_init(&s_full[0], 1);
    mbar_init(&s_full[1], 1);
    mbar_init(&p_full[0], 4);
    mbar_init(&p_full[1], 4);
    fence_barrier_init();
  } else if (warp == 2) {
    tmem_alloc<1>(tmem_slot, 512);
    tmem_relinquish<1>();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    // ===================== producer =====================
    if (lane == 0) {
      mbar_arrive_expect_tx(q_full, 2 * TILE);
#pragma unroll
      for (int t = 0; t < 2; ++t)
#pragma unroll
        for (int h = 0; h < NPANEL; ++h) tma_load_2d(sq + t * TILE + h * HALF, &tm_q, q_full, h * 64, q_row0 + t * ATTN_BM);
      ArefCursor c;
      const int kv_row0 = bh * p.S;
      for (int j = 0; j < n_kv; ++j) {
#pragma unroll
        for (int which = 0; which < 2; ++which) {  // K_j then V_j
          ring->put_acquire(c, 10);
          ring->put_expect(c, TILE);
          uint8_t* dst = skv + c.slot * TILE;
#pragma unroll
          for (int h = 0; h < NPANEL; ++h)
            tma_load_2d(dst + h * HALF, which == 0 ? &tm_k : &tm_v, &ring->full[c.slot], h * 64, kv_row0 + j * ATTN_BN);
          c.advance(D);
        }
      }
    }
  } else if (warp == 1) {
    // ===================== MMA issuer =====================
    if (lane == 0) {
      const uint32_t q_addr = smem_u32(sq);
      const uint32_t kv_addr = smem_u32(skv);
      auto issue_qk = [&](int t, uint32_t k_slot) {
        const uint32_t a0 = q_addr + t * TILE, b0 = kv_addr + k_slot * TILE;
#pragma unroll
        for (int k = 0; k < DH / 16; ++k) {
          const uint32_t off = (k / 4) * HALF + (k % 4) * 32;
          mma_f16_ss<1>(tmem + COL_S + t * ATTN_BN, make_sw128_desc(a0 + off, 16, 1024),
                        make_sw128_desc(b0 + off, 16, 1024), IDESC_QK, k != 0);
        }
      };
      auto issue_pv = [&](int t, uint32_t v_slot, bool acc) {
        const uint32_t b0 = kv_addr + v_slot * TILE;
#pragma unroll
        for (int k = 0; k < ATTN_BN / 16; ++k) {
          // A = P_t: 16 keys = 8 packed columns; B = V rows [16k, 16k+16): two 8-row groups
          mma_f16_ts(tmem + COL_O + t * DH, tmem + COL_S + t * ATTN_BN + k * 8,
                     make_sw128_desc(b0 + k * 16 * 128, HALF, 1024), IDESC_PV, (acc || k != 0) ? 1u : 0u);
        }
      };
      mbar_wait(q_full, 0, 11);
      ArefCursor c;
      // prologue: T_0 for both tiles
      ring->get(c, 12);
      tc_fence_after();
      uint32_t k_slot = c.slot;
      issue_qk(0, k_slot);
      mma_commit(&s_full[0]);
      issue_qk(1, k_slot);
      mma_commit(&s_full[1]);
      ring->consumed_by_mma(c);
      c.advance(D);
      for (int j = 0; j < n_kv; ++j) {
        ring->get(c, 13);  // V_j
        tc_fence_after();
        const ArefCursor cv = c;
        c.advance(D);
        ArefCursor ck = c;  // K_{j+1}
        const bool more = j + 1 < n_kv;
#pragma unroll
        for (int t = 0; t < 2; ++t) {
          mbar_wait(&p_full[t], j & 1, 14 + t);  // C_j[t] done: P_t in TMEM, O_t rescaled
          tc_fence_after();
          issue_pv(t, cv.slot, j > 0);
          if (more) {
            if (t == 0) {
              ring->get(ck, 16);
              tc_fence_after();
            }
            issue_qk(t, ck.slot);
          }
          mma_commit(&s_full[t]);
        }
        ring->consumed_by_mma(cv);
        if (more) {
          ring->consumed_by_mma(ck);
          c.advance(D);
        }
      }
    }
  } else if (warp >= 4) {
    // ===================== softmax / correction / epilogue =====================
    const int t = (warp - 4) / 4;     // Q tile
    const uint32_t q = warp & 3u;     // TMEM lane quarter
    const int row = q * 32 + lane;    // row within the Q tile
    const uint32_t t_lane = (q * 32u) << 16;
    const uint32_t t_s = tmem + t_lane + COL_S + t * ATTN_BN;
    const uint32_t t_o = tmem + t_lane + COL_O + t * DH;
    const int qpos = pair * 2 * ATTN_BM + t * ATTN_BM + row;  // query position in the sequence
    const float sl2 = p.scale_log2;
    float m_used = -INFINITY;  // running max (log2 units) the current P/O are relative to
    float l = 0.f;
    for (int j = 0; j < n_kv; ++j) {
      mbar_wait(&s_full[t], j & 1, 20 + t);
      tc_fence_after();
      float s[ATTN_BN];
      {
        uint32_t* su = reinterpret_cast<uint32_t*>(s);
        tmem_ld32(t_s + 0, *reinterpret_cast<uint32_t(*)[32]>(su + 0));
        tmem_ld32(t_s + 32, *reinterpret_cast<uint32_t(*)[32]>(su + 32));
        tmem_ld32(t_s + 64, *reinterpret_cast<uint32_t(*)[32]>(su + 64));
        tmem_ld32(t_s + 96, *reinterpret_cast<uint32_t(*)[32]>(su + 96));
        tmem_wait_ld();
      }
      if (p.causal && j * ATTN_BN + ATTN_BN - 1 > qpos - row) {
        // block intersects the upper triangle of this tile: mask key > query
#pragma unroll
        for (int c = 0; c < ATTN_BN; ++c)
          if (j * ATTN_BN + c > qpos) s[c] = -INFINITY;
      }
      float mx = s[0];
#pragma unroll
      for (int c = 1; c < ATTN_BN; ++c) mx = fmaxf(mx, s[c]);
      const float m_blk = mx * sl2;
      float alpha = 1.f;
      const bool need = m_blk > m_used + ATTN_RESCALE_THRESHOLD;
      if (need) {
        alpha = ex2_approx(m_used - m_blk);  // 0 on the first block (m_used = -inf)
        m_used = m_blk;
      }
      if (j > 0 && __any_sync(0xffffffffu, need)) {
        // correction: O_t row *= alpha (PV_{j-1}[t] is complete: it precedes QK_j[t] in issue order)
#pragma unroll 1
        for (int c0 = 0; c0 < DH; c0 += 32) {
          uint32_t ov[32];
          tmem_ld32(t_o + c0, ov);
          tmem_wait_ld();
#pragma unroll
          for (int e = 0; e < 32; ++e) ov[e] = __float_as_uint(__uint_as_float(ov[e]) * alpha);
          tmem_st32(t_o + c0, ov);
        }
      }
      l *= alpha;
      const float neg_m = -m_used;
      float ls = 0.f;
      uint32_t pk[ATTN_BN / 2];
#pragma unroll
      for (int c = 0; c < ATTN_BN; c += 2) {
        const float p0 = ex2_approx(fmaf(s[c], sl2, neg_m));
        const float p1 = ex2_approx(fmaf(s[c + 1], sl2, neg_m));
        ls += p0 + p1;
        pk[c / 2] = BF16 ? pack_bf16(p0, p1) : pack_f16(p0, p1);
      }
      l += ls;
      tmem_st32(t_s + 0, *reinterpret_cast<uint32_t(*)[32]>(pk + 0));
      tmem_st32(t_s + 32, *reinterpret_cast<uint32_t(*)[32]>(pk + 32));
      tmem_wait_st();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&p_full[t]);
    }
    // epilogue: O_t / l -> global, lse
    mbar_wait(&s_full[t], n_kv & 1, 22 + t);
    tc_fence_after();
    const float inv_l = 1.f / l;
    const size_t grow = static_cast<size_t>(q_row0 + t * ATTN_BM + row);
    uint8_t* orow = reinterpret_cast<uint8_t*>(p.o) + grow * DH * 2;
#pragma unroll 1
    for (int c0 = 0; c0 < DH; c0 += 32) {
      uint32_t ov[32];
      tmem_ld32(t_o + c0, ov);
      tmem_wait_ld();
      uint32_t w[16];
#pragma unroll
      for (int e = 0; e < 16; ++e) {
        const float a = __uint_as_float(ov[2 * e]) * inv_l, b = __uint_as_float(ov[2 * e + 1]) * inv_l;
        w[e] = BF16 ? pack_bf16(a, b) : pack_f16(a, b);
      }
      uint4* dst = reinterpret_cast<uint4*>(orow + c0 * 2);
#pragma unroll
      for (int e = 0; e < 4; ++e) dst[e] = make_uint4(w[4 * e], w[4 * e + 1], w[4 * e + 2], w[4 * e + 3]);
    }
    if (p.lse) p.lse[grow] = m_used * 0.69314718055994531f + __logf(l);
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc<1>(tmem, 512);
  }
}

}  // namespace ws

