// attn128_sm100.cuh — FlashAttention forward for sm_100a with 128-key K/V blocks.
//
// Same reference semantics as attn_sm100.cuh (the flash .k of SURVEY.md Appendix A: the coarse
// T/C/U pipeline of ref proj/include/warpspec/pipeline.hpp:160-328, schedule.hpp:18-74), with a
// different mapping onto the SM:
//
//   * K/V blocks of 128 keys. A 128x128xDh QK^T MMA reads 4 KB of Q and 4 KB of K from shared
//     memory per K=16 step and runs 64 cycles — inside the 128 B/clk shared-memory operand rate.
//     The 64-key kernel's QK (4 KB + 2 KB per 32-cycle step) is bound by that rate at 1.5x its
//     tensor time, which is the loss this variant removes.
//   * TMEM (512 columns for Dh = 128): S_0 | S_1 (128 columns each) | O_0 | O_1 (Dh each). The S
//     accumulator of a Q tile is single-buffered; the overlap the coarse schedule asks for (T_{j+1}
//     while C_j runs) comes from the two Q tiles (the cooperative row bands of
//     ref proj/include/warpspec/grid.hpp:24-72) ping-ponging on the tensor core: while the softmax
//     warps of tile 0 work on S_0(j), the tensor core runs PV_1(j-1) and QK_1(j) for tile 1.
//   * Issue order of the single MMA thread, per step j:
//         PV_0(j)  QK_0(j+1)  PV_1(j)  QK_1(j+1)
//     QK_t(j+1) overwrites S_t, whose first 64 columns hold P_t(j) read by PV_t(j); tcgen05 MMAs
//     of one thread execute in issue order, so the overwrite follows the read. A commit after
//     QK_t(j+1) therefore also proves PV_t(j) complete: when the softmax warps see S_t(j+1) they
//     may rescale O_t in place (the correction stage needs no separate barrier).
//   * Causal: the 256 query rows of a CTA are two 128-row tiles aligned to 128-key blocks, so the
//     diagonal block of each tile is square and is the only block that needs a mask; tile 0 stops
//     one block before tile 1.
//   * Persistent (ref proj/include/warpspec/grid.hpp:93-123): grid = min(#SMs, items), CTA b runs
//     the items of its static schedule (stride, or a snake for causal), barrier phases carry over
//     (running block counters), and q_free / o_free hand the Q tiles and the O accumulators over to
//     the next item. S_t needs no hand-over: the next item's QK_t(0) is issued after this item's
//     last PV_t(j) by the same thread, and tcgen05 MMAs execute in issue order.
#pragma once

#include "attn_sm100.cuh"  // ATTN_RESCALE_THRESHOLD, attn_poly_pair, trace layout

namespace ws {

constexpr int A128_BM = 128;          // query rows per Q tile (one TMEM lane each)
constexpr int A128_BN = 128;          // keys per K/V block
constexpr int A128_THREADS = 384;     // 8 softmax warps + producer + MMA + TMEM allocator + spare
constexpr int A128_MAX_STAGES = 8;
constexpr int A128_POLY = 2;          // default exp mix: 2 of every 8 column pairs on the FMA pipe

struct Attn128Params {
  int S, BH_begin, num_pairs;  // num_pairs = S / 256 work items per (b,h)
  int num_bh;                  // (b,h) slices in this launch (the persistent kernel's item space)
  int stagger;                 // attn_psmem: issue QK_1(j+1) after PV_0(j) (offsets the two tiles)
  int kv_stages;
  int causal;
  int bh_fast;        // grid order: 1 = blockIdx.x walks (b,h) (causal, heaviest pairs first);
                      // 0 = blockIdx.x walks the query pairs of one (b,h) (K/V stay L2-resident)
  float scale_log2;   // softmax_scale * log2(e) (* q, k descales for FP8)
  float o_scale;      // V descale folded into the epilogue (1 unless FP8)
  float* lse;
  float* mx;          // optional: exact row max of the scaled scores (natural units; the .k's %m)
  void* o;
  unsigned long long* trace;  // optional %clock64 stamps of CTA (0,0), layout of attn_sm100.cuh
};

__host__ __device__ inline uint32_t a128_q_bytes(int Dh) { return A128_BM * Dh * 2; }
__host__ __device__ inline uint32_t a128_kv_bytes(int Dh) { return A128_BN * Dh * 2; }
__host__ __device__ inline uint32_t a128_smem_bytes(int Dh, int kv_stages) {
  // Q0 | Q1 | kv slots | barriers (+1 KB alignment slack)
  return 2 * a128_q_bytes(Dh) + kv_stages * a128_kv_bytes(Dh) + (2 * A128_MAX_STAGES + 16) * 8 + 16 + 1024;
}

__device__ __forceinline__ float fmax3(float a, float b, float c) {
  float d;
  asm("max.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c));
  return d;
}

// POLY: how many of every 8 column pairs are exponentiated on the FMA pipe (exp2_poly2) instead of
// MUFU.EX2 — see attn_poly_pair in attn_sm100.cuh.
template <int DH, bool BF16, int POLY = 2, bool TRACE = false>
__global__ void __launch_bounds__(A128_THREADS, 1)
    ws_attn128_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                      const __grid_constant__ CUtensorMap tm_v, const __grid_constant__ CUtensorMap tm_o,
                      const Attn128Params p) {
  constexpr uint32_t QTILE = A128_BM * DH * 2;   // bytes of a 128 x DH Q tile
  constexpr uint32_t KVTILE = A128_BN * DH * 2;  // bytes of a 128 x DH K or V block
  constexpr uint32_t QPANEL = A128_BM * 128;     // one 64-column (128 B) swizzle panel of Q
  constexpr uint32_t KVPANEL = A128_BN * 128;    // one 64-column panel of K / V
  constexpr int NPANEL = DH / 64;
  constexpr uint32_t FMT = BF16 ? 1u : 0u;
  constexpr uint32_t IDESC_QK = make_idesc(FMT, A128_BM, A128_BN, 0, 0);
  constexpr uint32_t IDESC_PV = make_idesc(FMT, A128_BM, DH, 0, 1);  // B = V is MN-major
  constexpr uint32_t COL_O = 2 * A128_BN;
  constexpr uint32_t TMEM_COLS = 2 * A128_BN + 2 * DH <= 256 ? 256 : 512;

  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sq = smem;               // Q0, Q1
  uint8_t* skv = smem + 2 * QTILE;  // K/V ring
  uint8_t* bar_base = skv + p.kv_stages * KVTILE;
  auto* ring = reinterpret_cast<ArefBarriers<A128_MAX_STAGES>*>(bar_base);
  uint64_t* q_full = reinterpret_cast<uint64_t*>(bar_base + 2 * A128_MAX_STAGES * 8);
  uint64_t* s_full = q_full + 1;  // [2]: QK_t(j) complete (and with it PV_t(j-1))
  uint64_t* p_full = q_full + 3;  // [2]: P_t(j) in S_t, O_t rescaled
  uint64_t* o_full = q_full + 5;  // [2]: last PV_t of the item complete
  uint64_t* o_free = q_full + 7;  // [2]: O_t of the item copied out by the epilogue
  uint64_t* q_free = q_full + 9;  // the item's last QK complete: Q smem reusable
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(q_full + 10);

  const uint32_t warp = warp_id();
  const uint32_t lane = lane_id();
  const uint32_t D = static_cast<uint32_t>(p.kv_stages);

  const int nbh = p.num_bh;
  auto item_coords = [&](int i, int& pair, int& bh) {
    if (p.bh_fast) {  // causal: (b,h) fastest from the heaviest query pairs down
      pair = p.num_pairs - 1 - i / nbh;
      bh = p.BH_begin + i % nbh;
    } else {  // the query pairs of one (b,h) together: its K/V stay in L2
      pair = i % p.num_pairs;
      bh = p.BH_begin + i / p.num_pairs;
    }
  };
  // K/V blocks per tile: causal tile t of pair i sees blocks 0 .. 2i+t (its diagonal block last)
  auto nblk = [&](int pair, int t) { return p.causal ? 2 * pair + 1 + t : p.S / A128_BN; };
  const int num_items = p.num_pairs * nbh;
  const int G = static_cast<int>(gridDim.x), b_id = static_cast<int>(blockIdx.x);
  auto item_of = [&](int r) { return r * G + ((p.causal && (r & 1)) ? G - 1 - b_id : b_id); };
  // the traced instantiation (ws_attn_fwd_traced) is the only one carrying the stamps
  unsigned long long* const trace =
      (TRACE && p.trace != nullptr && blockIdx.x == 0) ? p.trace : nullptr;
  // stamps of the first item of CTA 0 only
#define WS_TRACE(role, j, ev)                                                        \
  do {                                                                              \
    if (TRACE && trace != nullptr && it == 0 && (j) < ATTN_TRACE_STEPS)             \
      trace[((role) * ATTN_TRACE_STEPS + (j)) * 8 + (ev)] = clk64();                \
  } while (0)

  if (warp == 8 && lane == 0) {
    tma_prefetch_desc(&tm_q);
    tma_prefetch_desc(&tm_k);
    tma_prefetch_desc(&tm_v);
    ring->init(D, 1, 1);
    mbar_init(q_full, 1);
    mbar_init(q_free, 1);
    for (int i = 0; i < 2; ++i) {
      mbar_init(&s_full[i], 1);
      mbar_init(&p_full[i], 4);
      mbar_init(&o_full[i], 1);
      mbar_init(&o_free[i], 4);
    }
    fence_barrier_init();
  } else if (warp == 10) {
    tmem_alloc<1>(tmem_slot, TMEM_COLS);
    tmem_relinquish<1>();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  pdl_wait();  // programmatic dependent launch: the setup above overlapped the previous grid's tail
  pdl_launch_dependents();

  if (warp == 8) {
    // ===================== producer: aref put =====================
    // ring order = MMA consumption order: K_0, then (K_{j+1}, V_j) for j = 0 .. n1-1
    regs_dec<72>();
    if (lane == 0) {
      ArefCursor c;
      for (int it = 0, item = item_of(0); item < num_items; item = item_of(++it)) {
        int pair, bh;
        item_coords(item, pair, bh);
        const int n1 = nblk(pair, 1);
        const int q_row0 = bh * p.S + pair * 2 * A128_BM;  // row in the [B*H*S, Dh] view
        const int kv_row0 = bh * p.S;
        if (it > 0) mbar_wait(q_free, (it - 1) & 1, 9);  // the previous item's QKs have read Q
        mbar_arrive_expect_tx(q_full, 2 * QTILE);
#pragma unroll
        for (int t = 0; t < 2; ++t)
#pragma unroll
          for (int h = 0; h < NPANEL; ++h)
            tma_load_2d(sq + t * QTILE + h * QPANEL, &tm_q, q_full, h * 64, q_row0 + t * A128_BM);
        auto put = [&](const CUtensorMap* m, int blk) {
          ring->put_acquire(c, 10);
          ring->put_expect(c, KVTILE);
          uint8_t* dst = skv + c.slot * KVTILE;
#pragma unroll
          for (int h = 0; h < NPANEL; ++h)
            tma_load_2d(dst + h * KVPANEL, m, &ring->full[c.slot], h * 64, kv_row0 + blk * A128_BN);
          c.advance(D);
        };
        put(&tm_k, 0);
        for (int j = 0; j < n1; ++j) {
          if (j + 1 < n1) put(&tm_k, j + 1);
          put(&tm_v, j);
        }
      }
    }
  } else if (warp == 9) {
    // ===================== MMA issuer (whole warp, one elected lane issues) =====================
    regs_dec<72>();
    const uint64_t qdesc = make_sw128_desc(smem_u32(sq), 16, 1024);
    const uint64_t kdesc = make_sw128_desc(smem_u32(skv), 16, 1024);
    const uint64_t vdesc = make_sw128_desc(smem_u32(skv), KVPANEL, 1024);
    auto issue_qk = [&](int t, uint32_t k_slot) {
      const uint64_t a0 = qdesc + ((t * QTILE) >> 4), b0 = kdesc + ((k_slot * KVTILE) >> 4);
#pragma unroll
      for (int k = 0; k < DH / 16; ++k) {
        const uint32_t off = ((k / 4) * KVPANEL + (k % 4) * 32) >> 4;
        const uint32_t qoff = ((k / 4) * QPANEL + (k % 4) * 32) >> 4;
        mma_f16_ss_warp(tmem + t * A128_BN, a0 + qoff, b0 + off, IDESC_QK, k != 0);
      }
    };
    auto issue_pv = [&](int t, uint32_t v_slot, bool acc) {
      const uint64_t b0 = vdesc + ((v_slot * KVTILE) >> 4);
#pragma unroll
      for (int k = 0; k < A128_BN / 16; ++k) {
        // A = P_t: 16 keys = 8 packed columns; B = V rows [16k, 16k+16) (two 8-row core groups)
        mma_f16_ts_warp(tmem + COL_O + t * DH, tmem + t * A128_BN + k * 8, b0 + ((k * 16 * 128) >> 4), IDESC_PV,
                        (acc || k != 0) ? 1u : 0u);
      }
    };
    ArefCursor c;
    uint32_t g0 = 0, g1 = 0;  // blocks of tile 0 / tile 1 processed by earlier items
    for (int it = 0, item = item_of(0); item < num_items; item = item_of(++it)) {
      int pair, bh;
      item_coords(item, pair, bh);
      const int n0 = nblk(pair, 0), n1 = nblk(pair, 1);
      mbar_wait(q_full, it & 1, 11);
      ring->get(c, 12);  // K_0
      tc_fence_after();
      // S_t is free: the previous item's last PV_t (reading P_t from S_t) was issued before
      issue_qk(0, c.slot);
      mma_commit_warp(&s_full[0]);
      issue_qk(1, c.slot);
      mma_commit_warp(&s_full[1]);
      mma_commit_warp(&ring->empty[c.slot]);
      c.advance(D);
      for (int j = 0; j < n1; ++j) {
        if (lane == 0) WS_TRACE(0, j, 0);
        const bool more1 = j + 1 < n1;
        uint32_t kslot = 0;
        if (more1) {
          ring->get(c, 13);  // K_{j+1}
          kslot = c.slot;
          c.advance(D);
        }
        ring->get(c, 14);  // V_j
        const uint32_t vslot = c.slot;
        c.advance(D);
        tc_fence_after();
        if (lane == 0) WS_TRACE(0, j, 1);
        if (j < n0) {
          mbar_wait(&p_full[0], (g0 + j) & 1, 15);  // C_0(j): P_0(j) in TMEM, O_0 rescaled
          if (j == 0 && it > 0) mbar_wait(&o_free[0], (it - 1) & 1, 19);  // previous O_0 copied out
          tc_fence_after();
          if (lane == 0) WS_TRACE(0, j, 2);
          issue_pv(0, vslot, j > 0);
          if (j + 1 < n0) {
            issue_qk(0, kslot);
            mma_commit_warp(&s_full[0]);
          } else {
            mma_commit_warp(&o_full[0]);
          }
          if (lane == 0) WS_TRACE(0, j, 3);
        }
        mbar_wait(&p_full[1], (g1 + j) & 1, 16);
        if (j == 0 && it > 0) mbar_wait(&o_free[1], (it - 1) & 1, 19);
        tc_fence_after();
        if (lane == 0) WS_TRACE(0, j, 4);
        issue_pv(1, vslot, j > 0);
        mma_commit_warp(&ring->empty[vslot]);
        if (more1) {
          issue_qk(1, kslot);
          mma_commit_warp(&s_full[1]);
          mma_commit_warp(&ring->empty[kslot]);
          if (j + 2 == n1) mma_commit_warp(q_free);  // that was the item's last QK: Q reusable
        } else {
          mma_commit_warp(&o_full[1]);
        }
        if (lane == 0) WS_TRACE(0, j, 5);
      }
      g0 += n0;
      g1 += n1;
    }
  } else if (warp >= 8) {
    regs_dec<72>();
  } else {
    // ===================== softmax / correction / epilogue =====================
    regs_inc<216>();
    const int t = warp / 4;        // Q tile
    const uint32_t q = warp & 3u;  // TMEM lane quarter
    const int row = q * 32 + lane;  // row within the Q tile
    const uint32_t t_lane = (q * 32u) << 16;
    const uint32_t t_s = tmem + t_lane + t * A128_BN;
    const uint32_t t_o = tmem + t_lane + COL_O + t * DH;
    const float sl2 = p.scale_log2;
    const bool tr = lane == 0 && q == 0;
    uint32_t g = 0;  // blocks of this tile processed by earlier items
    for (int it = 0, item = item_of(0); item < num_items; item = item_of(++it)) {
    int pair, bh;
    item_coords(item, pair, bh);
    const int n_t = nblk(pair, t);
    const int q_row0 = bh * p.S + pair * 2 * A128_BM;
    const int j_diag = p.causal ? n_t - 1 : -1;
    float m_used = -INFINITY;  // running max (log2 units) the current P/O are relative to
    float m_true = -INFINITY;  // exact running row max (log2 units; the .k's %m, for p.mx)
    float l = 0.f;
    for (int j = 0; j < n_t; ++j) {
      if (tr) WS_TRACE(1 + t, j, 0);
      mbar_wait(&s_full[t], (g + j) & 1, 20 + t);
      if (tr) WS_TRACE(1 + t, j, 1);
      tc_fence_after();
      float s[A128_BN];
      {
        uint32_t* su = reinterpret_cast<uint32_t*>(s);
#pragma unroll
        for (int c0 = 0; c0 < A128_BN; c0 += 32) tmem_ld32(t_s + c0, *reinterpret_cast<uint32_t(*)[32]>(su + c0));
        tmem_wait_ld();
      }
      if (tr) WS_TRACE(1 + t, j, 2);
      if (j == j_diag) {
#pragma unroll
        for (int c = 0; c < A128_BN; ++c) s[c] = c > row ? -INFINITY : s[c];
      }
      float mx;
      {
        float m4[4] = {fmax3(s[0], s[1], s[2]), fmax3(s[3], s[4], s[5]), fmax3(s[6], s[7], s[8]),
                       fmax3(s[9], s[10], s[11])};
#pragma unroll
        for (int c = 12; c + 8 <= A128_BN; c += 8) {
          m4[0] = fmax3(m4[0], s[c], s[c + 1]);
          m4[1] = fmax3(m4[1], s[c + 2], s[c + 3]);
          m4[2] = fmax3(m4[2], s[c + 4], s[c + 5]);
          m4[3] = fmax3(m4[3], s[c + 6], s[c + 7]);
        }
        m4[0] = fmax3(m4[0], s[A128_BN - 4], s[A128_BN - 3]);
        m4[1] = fmax3(m4[1], s[A128_BN - 2], s[A128_BN - 1]);
        mx = fmaxf(fmaxf(m4[0], m4[1]), fmaxf(m4[2], m4[3]));
      }
      const float m_blk = mx * sl2;
      m_true = fmaxf(m_true, m_blk);
      float alpha = 1.f;
      const bool need = m_blk > m_used + ATTN_RESCALE_THRESHOLD;
      if (need) {
        alpha = ex2_approx(m_used - m_blk);  // 0 on the first block (m_used = -inf)
        m_used = m_blk;
      }
      if (j > 0 && __any_sync(0xffffffffu, need)) {
        // correction: S_t(j) complete implies PV_t(j-1) complete (issued before QK_t(j)), and
        // PV_t(j) waits for this warp's p_full arrival — O_t is quiescent here.
        const uint64_t al2 = f2_pack(alpha, alpha);
#pragma unroll 1
        for (int c0 = 0; c0 < DH; c0 += 32) {
          uint32_t ov[32];
          tmem_ld32(t_o + c0, ov);
          tmem_wait_ld();
#pragma unroll
          for (int e = 0; e < 32; e += 2) {
            float a0, a1;
            f2_unpack(f2_mul(f2_pack(__uint_as_float(ov[e]), __uint_as_float(ov[e + 1])), al2), a0, a1);
            ov[e] = __float_as_uint(a0);
            ov[e + 1] = __float_as_uint(a1);
          }
          tmem_st32(t_o + c0, ov);
        }
      }
      l *= alpha;
      if (tr) WS_TRACE(1 + t, j, 3);
      // P = 2^(s*sl2 - m) written back over the first 64 columns of S_t as packed 16-bit pairs
      const uint64_t sl2x2 = f2_pack(sl2, sl2), negm2 = f2_pack(-m_used, -m_used);
      uint64_t sum2a = f2_pack(0.f, 0.f), sum2b = f2_pack(0.f, 0.f);
#pragma unroll
      for (int c0 = 0; c0 < A128_BN; c0 += 32) {
        uint32_t pk[16];
#pragma unroll
        for (int c = c0; c < c0 + 32; c += 2) {
          const uint64_t x2 = f2_fma(f2_pack(s[c], s[c + 1]), sl2x2, negm2);
          uint64_t p2;
          if (attn_poly_pair(POLY, (c / 2) & 7)) {
            p2 = exp2_poly2(x2);
          } else {
            float x0, x1;
            f2_unpack(x2, x0, x1);
            p2 = f2_pack(ex2_approx(x0), ex2_approx(x1));
          }
          if ((c / 2) & 1)
            sum2b = f2_add(sum2b, p2);
          else
            sum2a = f2_add(sum2a, p2);
          float p0, p1;
          f2_unpack(p2, p0, p1);
          pk[(c - c0) / 2] = BF16 ? pack_bf16(p0, p1) : pack_f16(p0, p1);
        }
        tmem_st16(t_s + c0 / 2, pk);
      }
      {
        float a, b, c2, d2;
        f2_unpack(sum2a, a, b);
        f2_unpack(sum2b, c2, d2);
        l += (a + b) + (c2 + d2);
      }
      tmem_wait_st();
      if (tr) WS_TRACE(1 + t, j, 4);
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&p_full[t]);
      if (tr) WS_TRACE(1 + t, j, 5);
    }
    // epilogue: O_t / l -> global, lse. O_t is copied to registers and released (o_free) first, so
    // the next item's PV_t(0) may overwrite it while this one is converted and stored.
    g += n_t;
    mbar_wait(&o_full[t], it & 1, 26 + t);
    tc_fence_after();
    uint32_t ov[DH];
#pragma unroll
    for (int c0 = 0; c0 < DH; c0 += 32) tmem_ld32(t_o + c0, *reinterpret_cast<uint32_t(*)[32]>(ov + c0));
    tmem_wait_ld();
    tc_fence_before();
    __syncwarp();
    if (lane == 0) mbar_arrive(&o_free[t]);
    const float inv_l = 1.f / l;
    const size_t grow = static_cast<size_t>(q_row0 + t * A128_BM + row);
    uint8_t* orow = reinterpret_cast<uint8_t*>(p.o) + grow * DH * 2;
#pragma unroll
    for (int c0 = 0; c0 < DH; c0 += 8) {
      uint32_t w[4];
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const float a = __uint_as_float(ov[c0 + 2 * e]) * inv_l, b = __uint_as_float(ov[c0 + 2 * e + 1]) * inv_l;
        w[e] = BF16 ? pack_bf16(a, b) : pack_f16(a, b);
      }
      *reinterpret_cast<uint4*>(orow + c0 * 2) = make_uint4(w[0], w[1], w[2], w[3]);
    }
    if (p.lse) p.lse[grow] = m_used * 0.69314718055994531f + __logf(l);
    if (p.mx) p.mx[grow] = m_true * 0.69314718055994531f;
    }  // items
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 10) {
    tc_fence_after();
    tmem_dealloc<1>(tmem, TMEM_COLS);
  }
#undef WS_TRACE
}

}  // namespace ws
