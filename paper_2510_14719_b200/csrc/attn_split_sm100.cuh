// attn_split_sm100.cuh — FlashAttention forward for sm_100a with split-row softmax warps.
//
// Same reference semantics, tiling, MMA schedule and barrier protocol as attn_psmem_sm100.cuh (the
// flash .k of SURVEY.md Appendix A; coarse T/C/U pipeline of ref proj/include/warpspec/pipeline.hpp:
// 160-328; persistent items of ref grid.hpp:93-123). What changes is the softmax stage C:
//
//   * 16 softmax warps instead of 8, four per SM sub-partition. Warp w serves Q tile
//     t = (w / 4) % 2 and 16 rows of TMEM lane quarter q = w % 4 (rows 32 q + 16 r .. + 15,
//     r = w / 8). S is read with tcgen05.ld.16x32bx2: thread i holds row (i % 16) and the
//     contiguous key half (i / 16) — 64 of the block's 128 keys — so each thread carries half the
//     registers of S and every SMSP has twice the warps to interleave exponentials on MUFU.
//   * The two halves of a row sit in lanes i and i ^ 16 of the same warp: the row max costs one
//     shfl.xor per block, the row sum one per item. Each thread writes its keys to its own
//     128-byte panel of the P row (the K-major P tile's panel = key half), as before.
//   * O (correction, epilogue) is split the same way: thread i owns O columns
//     [(i / 16) * DH / 2, (i / 16 + 1) * DH / 2) of its row.
#pragma once

#include "attn_psmem_sm100.cuh"

namespace ws {

// 16 softmax warps (warpgroups 0-3) + producer, MMA, TMEM allocator and a spare (warpgroup 4;
// setmaxnreg is warpgroup-wide, so the group is complete and all four use one value). Register
// budget: the launch allocates 96 per thread (ptxas, 640 threads) and setmaxnreg.inc only draws on
// what the service warpgroup releases: 128 x (96 - 56) = 5120 >= 512 x (104 - 96) = 4096.
constexpr int ASP_THREADS = 640;

__host__ __device__ inline uint32_t asp_smem_bytes(int Dh, int kv_stages) { return aps_smem_bytes(Dh, kv_stages); }

template <int DH, bool BF16, int POLY = 1, bool TRACE = false>
__global__ void __launch_bounds__(ASP_THREADS, 1)
    ws_attn_split_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                         const __grid_constant__ CUtensorMap tm_v, const __grid_constant__ CUtensorMap tm_o,
                         const Attn128Params p) {
  constexpr uint32_t QTILE = A128_BM * DH * 2;        // bytes of a 128 x DH Q tile
  constexpr uint32_t PTILE = A128_BM * A128_BN * 2;   // bytes of a 128 x 128 P tile
  constexpr uint32_t KVTILE = A128_BN * DH * 2;       // bytes of a 128 x DH K or V block
  constexpr uint32_t PANEL = 128 * 128;               // one 64-column (128 B) swizzle panel of 128 rows
  constexpr int NPANEL = DH * 2 / 128;                // 128-byte panels per Q / K / V row
  constexpr int PANEL_ELEMS = 64;
  constexpr uint32_t FMT = BF16 ? 1u : 0u;
  constexpr uint32_t IDESC_QK = make_idesc(FMT, A128_BM, A128_BN, 0, 0);
  constexpr uint32_t IDESC_PV = make_idesc(FMT, A128_BM, DH, 0, 1);  // A = P K-major, B = V MN-major
  constexpr uint32_t COL_O = 2 * A128_BN;
  constexpr uint32_t TMEM_COLS = 512;
  constexpr int HC = A128_BN / 2;  // key columns per softmax warp
  constexpr int OC = DH / 2;       // O columns per softmax warp (correction, epilogue)

  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sq = smem;
  uint8_t* sp = smem + 2 * QTILE;
  uint8_t* skv = sp + 2 * PTILE;
  uint8_t* bar_base = skv + p.kv_stages * KVTILE;
  auto* ring = reinterpret_cast<ArefBarriers<A128_MAX_STAGES>*>(bar_base);
  uint64_t* q_full = reinterpret_cast<uint64_t*>(bar_base + 2 * A128_MAX_STAGES * 8);
  uint64_t* s_full = q_full + 1;   // [2]
  uint64_t* s_free = q_full + 3;   // [2]
  uint64_t* p_full = q_full + 5;   // [2]
  uint64_t* pv_done = q_full + 7;  // [2]
  uint64_t* o_free = q_full + 9;   // [2]
  uint64_t* q_free = q_full + 11;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(q_full + 12);

  const uint32_t warp = warp_id();
  const uint32_t lane = lane_id();
  const uint32_t D = static_cast<uint32_t>(p.kv_stages);

  const int nbh = p.num_bh;
  auto item_coords = [&](int i, int& pair, int& bh) {
    if (p.bh_fast) {
      pair = p.num_pairs - 1 - i / nbh;
      bh = p.BH_begin + i % nbh;
    } else {
      pair = i % p.num_pairs;
      bh = p.BH_begin + i / p.num_pairs;
    }
  };
  auto nblk = [&](int pair, int t) { return p.causal ? 2 * pair + 1 + t : p.S / A128_BN; };
  const int num_items = p.num_pairs * nbh;
  const int G = static_cast<int>(gridDim.x), b_id = static_cast<int>(blockIdx.x);
  auto item_of = [&](int r) { return r * G + ((p.causal && (r & 1)) ? G - 1 - b_id : b_id); };
  unsigned long long* const trace =
      (TRACE && p.trace != nullptr && blockIdx.x == 0) ? p.trace : nullptr;
#define WS_TRACE(role, j, ev)                                                        \
  do {                                                                              \
    if (TRACE && trace != nullptr && (j) < ATTN_TRACE_STEPS)                        \
      trace[((role) * ATTN_TRACE_STEPS + (j)) * 8 + (ev)] = clk64();                \
  } while (0)

  if (warp == 16 && lane == 0) {
    tma_prefetch_desc(&tm_q);
    tma_prefetch_desc(&tm_k);
    tma_prefetch_desc(&tm_v);
    tma_prefetch_desc(&tm_o);
    ring->init(D, 1, 1);
    mbar_init(q_full, 1);
    mbar_init(q_free, 1);
    for (int i = 0; i < 2; ++i) {
      mbar_init(&s_full[i], 1);
      mbar_init(&s_free[i], 8);
      mbar_init(&p_full[i], 8);
      mbar_init(&pv_done[i], 1);
      mbar_init(&o_free[i], 8);
    }
    fence_barrier_init();
  } else if (warp == 18) {
    tmem_alloc<1>(tmem_slot, TMEM_COLS);
    tmem_relinquish<1>();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  pdl_wait();
  pdl_launch_dependents();

  if (warp == 16) {
    // ===================== producer: aref put (as attn_psmem) =====================
    regs_dec<56>();
    if (lane == 0) {
      ArefCursor c;
      for (int it = 0, item = item_of(0); item < num_items; item = item_of(++it)) {
        int pair, bh;
        item_coords(item, pair, bh);
        const int n1 = nblk(pair, 1);
        const int q_row0 = bh * p.S + pair * 2 * A128_BM;
        const int kv_row0 = bh * p.S;
        if (it > 0) mbar_wait(q_free, (it - 1) & 1, 9);
        mbar_arrive_expect_tx(q_full, 2 * QTILE);
#pragma unroll
        for (int t = 0; t < 2; ++t)
#pragma unroll
          for (int h = 0; h < NPANEL; ++h)
            tma_load_2d(sq + t * QTILE + h * PANEL, &tm_q, q_full, h * PANEL_ELEMS, q_row0 + t * A128_BM);
        auto put = [&](const CUtensorMap* m, int blk) {
          ring->put_acquire(c, 10);
          ring->put_expect(c, KVTILE);
          uint8_t* dst = skv + c.slot * KVTILE;
#pragma unroll
          for (int h = 0; h < NPANEL; ++h)
            tma_load_2d(dst + h * PANEL, m, &ring->full[c.slot], h * PANEL_ELEMS, kv_row0 + blk * A128_BN);
          c.advance(D);
        };
        put(&tm_k, 0);
        for (int j = 0; j < n1; ++j) {
          if (j + 1 < n1) put(&tm_k, j + 1);
          put(&tm_v, j);
        }
      }
    }
  } else if (warp == 17) {
    // ===================== MMA issuer (as attn_psmem, 16-bit operands) =====================
    regs_dec<56>();
    const uint64_t qdesc = make_sw128_desc(smem_u32(sq), 16, 1024);
    const uint64_t pdesc = make_sw128_desc(smem_u32(sp), 16, 1024);
    const uint64_t kdesc = make_sw128_desc(smem_u32(skv), 16, 1024);
    const uint64_t vdesc = make_sw128_desc(smem_u32(skv), PANEL, 1024);
    auto issue_qk = [&](int t, uint32_t k_slot) {
      const uint64_t a0 = qdesc + ((t * QTILE) >> 4), b0 = kdesc + ((k_slot * KVTILE) >> 4);
#pragma unroll
      for (int k = 0; k < DH * 2 / 32; ++k) {
        const uint32_t off = ((k / 4) * PANEL + (k % 4) * 32) >> 4;
        mma_f16_ss_warp(tmem + t * A128_BN, a0 + off, b0 + off, IDESC_QK, k != 0);
      }
    };
    auto issue_pv = [&](int t, uint32_t v_slot, bool acc) {
      const uint64_t a0 = pdesc + ((t * PTILE) >> 4), b0 = vdesc + ((v_slot * KVTILE) >> 4);
#pragma unroll
      for (int k = 0; k < A128_BN / 16; ++k) {
        const uint32_t aoff = ((k / 4) * PANEL + (k % 4) * 32) >> 4;
        mma_f16_ss_warp(tmem + COL_O + t * DH, a0 + aoff, b0 + ((k * 16 * 128) >> 4), IDESC_PV,
                        (acc || k != 0) ? 1u : 0u);
      }
    };
    ArefCursor c;
    uint32_t g0 = 0, g1 = 0;
    uint32_t k0slot = 0;
    auto first_qk0 = [&](int it_, uint32_t g0_) {
      mbar_wait(q_full, it_ & 1, 11);
      ring->get(c, 12);
      k0slot = c.slot;
      c.advance(D);
      tc_fence_after();
      if (g0_ > 0) {
        mbar_wait(&s_free[0], (g0_ - 1) & 1, 17);
        tc_fence_after();
      }
      issue_qk(0, k0slot);
      mma_commit_warp(&s_full[0]);
    };
    bool qk0_issued = false;
    for (int it = 0, item = item_of(0); item < num_items; item = item_of(++it)) {
      int pair, bh;
      item_coords(item, pair, bh);
      const int n0 = nblk(pair, 0), n1 = nblk(pair, 1);
      if (!qk0_issued) first_qk0(it, g0);
      qk0_issued = false;
      if (g1 > 0) {
        mbar_wait(&s_free[1], (g1 - 1) & 1, 18);
        tc_fence_after();
      }
      issue_qk(1, k0slot);
      mma_commit_warp(&s_full[1]);
      mma_commit_warp(&ring->empty[k0slot]);
      const int next_item = item_of(it + 1);
      for (int j = 0; j < n1; ++j) {
        if (lane == 0) WS_TRACE(0, g1 + j, 0);
        const bool more = j + 1 < n1;
        uint32_t kslot = 0;
        auto qk1 = [&]() {
          mbar_wait(&s_free[1], (g1 + j) & 1, 18);
          tc_fence_after();
          issue_qk(1, kslot);
          mma_commit_warp(&s_full[1]);
          mma_commit_warp(&ring->empty[kslot]);
          if (j + 2 == n1) mma_commit_warp(q_free);
        };
        if (more) {
          ring->get(c, 13);
          kslot = c.slot;
          c.advance(D);
          if (lane == 0) WS_TRACE(0, g1 + j, 6);
          if (j + 1 < n0) {
            mbar_wait(&s_free[0], (g0 + j) & 1, 17);
            tc_fence_after();
            issue_qk(0, kslot);
            mma_commit_warp(&s_full[0]);
          }
          if (lane == 0) WS_TRACE(0, g1 + j, 1);
          if (!p.stagger) qk1();
        }
        if (lane == 0) WS_TRACE(0, g1 + j, 2);
        ring->get(c, 14);
        const uint32_t vslot = c.slot;
        c.advance(D);
        if (lane == 0) WS_TRACE(0, g1 + j, 7);
        if (j < n0) {
          mbar_wait(&p_full[0], (g0 + j) & 1, 15);
          if (j == 0 && it > 0) mbar_wait(&o_free[0], (it - 1) & 1, 19);
          tc_fence_after();
          if (lane == 0) WS_TRACE(0, g1 + j, 3);
          issue_pv(0, vslot, j > 0);
          mma_commit_warp(&pv_done[0]);
        }
        if (more && p.stagger) qk1();
        if (!more && next_item < num_items) {
          first_qk0(it + 1, g0 + n0);
          qk0_issued = true;
        }
        mbar_wait(&p_full[1], (g1 + j) & 1, 16);
        if (j == 0 && it > 0) mbar_wait(&o_free[1], (it - 1) & 1, 19);
        tc_fence_after();
        if (lane == 0) WS_TRACE(0, g1 + j, 4);
        issue_pv(1, vslot, j > 0);
        mma_commit_warp(&pv_done[1]);
        mma_commit_warp(&ring->empty[vslot]);
        if (lane == 0) WS_TRACE(0, g1 + j, 5);
      }
      g0 += n0;
      g1 += n1;
    }
  } else if (warp >= 16) {
    regs_dec<56>();  // TMEM allocator, spare
  } else {
    // ===================== softmax (split rows) / correction / epilogue =====================
    regs_inc<104>();
    const int t = (warp >> 2) & 1;            // Q tile
    const uint32_t q = warp & 3u;             // TMEM lane quarter (= SMSP)
    const uint32_t r = warp >> 3;             // 16-row half of the quarter
    const uint32_t hh = lane >> 4;            // key half (and O column half) of this thread
    const int row = q * 32 + r * 16 + (lane & 15);  // row within the Q tile
    const uint32_t t_lane = (q * 32u + r * 16u) << 16;
    const uint32_t t_s = tmem + t_lane + t * A128_BN;
    const uint32_t t_o = tmem + t_lane + COL_O + t * DH;
    // this thread's half row of P_t: panel hh (keys 64 hh .. 64 hh + 63), 128B-swizzled
    const uint32_t p_row = smem_u32(sp + t * PTILE) + hh * PANEL + row * 128u;
    const uint32_t swz = static_cast<uint32_t>(row & 7);
    const float sl2 = p.scale_log2;
    const bool issuer = q == 0 && r == 0 && lane == 0;  // the tile's TMA-store thread
    const bool tr = issuer;
    uint32_t g = 0;  // blocks of this tile processed by earlier items
    for (int it = 0, item = item_of(0); item < num_items; item = item_of(++it)) {
      int pair, bh;
      item_coords(item, pair, bh);
      const int n_t = nblk(pair, t);
      const int q_row0 = bh * p.S + pair * 2 * A128_BM;
      const bool tile_valid = (2 * pair + t) * A128_BM < p.S;
      const int j_diag = p.causal ? n_t - 1 : -1;
      float m_used = -INFINITY;  // running max (log2 units) the current P/O are relative to
      float m_true = -INFINITY;  // exact running row max (log2 units; the .k's %m, for p.mx)
      float l = 0.f;             // this thread's half of the row sum
      for (int j = 0; j < n_t; ++j) {
        if (tr) WS_TRACE(1 + t, g + j, 0);
        mbar_wait(&s_full[t], (g + j) & 1, 20 + t);
        if (tr) WS_TRACE(1 + t, g + j, 1);
        tc_fence_after();
        float s[HC];
        uint32_t* su = reinterpret_cast<uint32_t*>(s);
        tmem_ld_h32<64>(t_s + 0, *reinterpret_cast<uint32_t(*)[32]>(su + 0));
        tmem_ld_h32<64>(t_s + 32, *reinterpret_cast<uint32_t(*)[32]>(su + 32));
        tmem_wait_ld();
        // S_t(j) is in registers: release the TMEM columns so QK_t(j+1) can run during this softmax
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&s_free[t]);
        if (tr) WS_TRACE(1 + t, g + j, 2);
        if (j == j_diag) {
#pragma unroll
          for (int c = 0; c < HC; ++c) s[c] = static_cast<int>(hh) * HC + c > row ? -INFINITY : s[c];
        }
        float mx;
        {
          float m4[4] = {fmax3(s[0], s[1], s[2]), fmax3(s[3], s[4], s[5]), fmax3(s[6], s[7], s[8]),
                         fmax3(s[9], s[10], s[11])};
#pragma unroll
          for (int c = 12; c + 8 <= HC; c += 8) {
            m4[0] = fmax3(m4[0], s[c], s[c + 1]);
            m4[1] = fmax3(m4[1], s[c + 2], s[c + 3]);
            m4[2] = fmax3(m4[2], s[c + 4], s[c + 5]);
            m4[3] = fmax3(m4[3], s[c + 6], s[c + 7]);
          }
          m4[0] = fmax3(m4[0], s[HC - 4], s[HC - 3]);
          m4[1] = fmax3(m4[1], s[HC - 2], s[HC - 1]);
          mx = fmaxf(fmaxf(m4[0], m4[1]), fmaxf(m4[2], m4[3]));
          mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 16));  // the row's other key half
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
          // correction: this thread's O columns *= alpha once PV_t(j-1) has landed
          mbar_wait(&pv_done[t], (g + j - 1) & 1, 24 + t);
          tc_fence_after();
          const uint64_t al2 = f2_pack(alpha, alpha);
#pragma unroll 1
          for (int c0 = 0; c0 < OC; c0 += 16) {
            uint32_t ov[16];
            tmem_ld_h16<OC>(t_o + c0, ov);
            tmem_wait_ld();
#pragma unroll
            for (int e = 0; e < 16; e += 2) {
              float a0, a1;
              f2_unpack(f2_mul(f2_pack(__uint_as_float(ov[e]), __uint_as_float(ov[e + 1])), al2), a0, a1);
              ov[e] = __float_as_uint(a0);
              ov[e + 1] = __float_as_uint(a1);
            }
            tmem_st_h16<OC>(t_o + c0, ov);
          }
          tmem_wait_st();
        }
        l *= alpha;
        if (tr) WS_TRACE(1 + t, g + j, 3);
        // P_t's shared-memory tile is free once PV_t(j-1) has read it
        if (g + j > 0) mbar_wait(&pv_done[t], (g + j - 1) & 1, 24 + t);
        if (j == 0 && it > 0) {
          // the previous item's O_t was staged through this P tile: its TMA store must have read it
          if (issuer) tma_store_wait_read<0>();
          named_bar_sync(1 + t, 256);
        }
        const uint64_t sl2x2 = f2_pack(sl2, sl2), negm2 = f2_pack(-m_used, -m_used);
        uint64_t sum4[4];
#pragma unroll
        for (int ch = 0; ch < HC / 8; ++ch) {
          float pf[8];
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const int c = ch * 8 + 2 * e;
            const uint64_t x2 = f2_fma(f2_pack(s[c], s[c + 1]), sl2x2, negm2);
            uint64_t p2;
            if (attn_poly_pair(POLY, (c / 2) & 7)) {
              p2 = exp2_poly2(x2);
            } else {
              float x0, x1;
              f2_unpack(x2, x0, x1);
              p2 = f2_pack(ex2_approx(x0), ex2_approx(x1));
            }
            sum4[e] = ch == 0 ? p2 : f2_add(sum4[e], p2);
            f2_unpack(p2, pf[2 * e], pf[2 * e + 1]);
          }
          uint32_t pk[4];
#pragma unroll
          for (int w = 0; w < 4; ++w)
            pk[w] = BF16 ? pack_bf16(pf[2 * w], pf[2 * w + 1]) : pack_f16(pf[2 * w], pf[2 * w + 1]);
          st_shared_v4(p_row + ((static_cast<uint32_t>(ch) ^ swz) << 4), pk[0], pk[1], pk[2], pk[3]);
        }
        {
          float a, b, c2, d2;
          f2_unpack(f2_add(sum4[0], sum4[1]), a, b);
          f2_unpack(f2_add(sum4[2], sum4[3]), c2, d2);
          l += (a + b) + (c2 + d2);
        }
        if (tr) WS_TRACE(1 + t, g + j, 4);
        fence_proxy_async_smem();  // generic-proxy stores -> visible to the tensor core's reads
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&p_full[t]);
        if (tr) WS_TRACE(1 + t, g + j, 5);
      }
      // epilogue: this thread's O columns / l -> global once the last PV_t has completed; O is
      // copied to registers and released first (o_free) so the next item's PV_t(0) can overwrite it
      g += n_t;
      const float l_row = l + __shfl_xor_sync(0xffffffffu, l, 16);
      mbar_wait(&pv_done[t], (g - 1) & 1, 26 + t);
      tc_fence_after();
      uint32_t ov[OC];
#pragma unroll
      for (int c0 = 0; c0 < OC; c0 += 16) tmem_ld_h16<OC>(t_o + c0, *reinterpret_cast<uint32_t(*)[16]>(ov + c0));
      tmem_wait_ld();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&o_free[t]);
      if (tr) WS_TRACE(1 + t, g - 1, 6);
      const float inv_l = p.o_scale / l_row;
      // stage O through this tile's P buffer (free: its last PV has completed), 128B-swizzled, 64
      // columns per 16 KB panel: hdim 128 — thread half hh writes panel hh; hdim 64 — one panel,
      // thread half hh writes its chunks 4 hh .. 4 hh + 3
      const uint32_t stage = smem_u32(sp + t * PTILE) + (DH == 128 ? hh * PANEL : 0u) + row * 128u;
#pragma unroll
      for (int k8 = 0; k8 < OC / 8; ++k8) {
        uint32_t w[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const int col = k8 * 8 + 2 * e;
          const float a = __uint_as_float(ov[col]) * inv_l, b = __uint_as_float(ov[col + 1]) * inv_l;
          w[e] = BF16 ? pack_bf16(a, b) : pack_f16(a, b);
        }
        const uint32_t chunk = static_cast<uint32_t>(k8) + (DH == 128 ? 0u : 4u * hh);
        st_shared_v4(stage + ((chunk ^ swz) << 4), w[0], w[1], w[2], w[3]);
      }
      fence_proxy_async_smem();
      named_bar_sync(1 + t, 256);
      if (issuer && tile_valid) {
#pragma unroll
        for (int c = 0; c < DH / 64; ++c)
          tma_store_2d(&tm_o, reinterpret_cast<const void*>(sp + t * PTILE + c * PANEL), c * 64, q_row0 + t * A128_BM);
        tma_store_commit();
      }
      if (p.lse && tile_valid && hh == 0) p.lse[q_row0 + t * A128_BM + row] = m_used * 0.69314718055994531f + __logf(l_row);
      if (p.mx && tile_valid && hh == 0) p.mx[q_row0 + t * A128_BM + row] = m_true * 0.69314718055994531f;
      if (tr) WS_TRACE(1 + t, g - 1, 7);
    }  // items
    if (issuer) tma_store_wait<0>();  // O stores complete before the CTA retires
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 18) {
    tc_fence_after();
    tmem_dealloc<1>(tmem, TMEM_COLS);
  }
#undef WS_TRACE
}

}  // namespace ws
