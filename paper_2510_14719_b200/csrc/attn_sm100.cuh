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
// Warp roles (the issuing roles take the highest warp ids: the sm_100 scheduler arbitrates
// highest-warp-id first, so the single MMA-issuing thread is never starved by softmax warps):
//   warps 0..3   softmax/correction/epilogue for Q tile 0 (thread = query row = TMEM lane)
//   warps 4..7   same for Q tile 1
//   warp 8       TMA producer: Q0,Q1 once, then K/V tiles (64 keys) into a depth-D smem aref
//   warp 9       MMA issuer (one thread): QK_j[t] -> S_t[j%2], PV_j[t] -> O_t
//   warp 10      TMEM allocator
// TMEM (512 columns): S_0[0] | S_0[1] | S_1[0] | S_1[1] (64 columns each) | O_0 | O_1 (Dh each).
// The S accumulator is double-buffered (a depth-2 aref between the tensor core and the softmax
// warps): T_{j+1} (QK_{j+1} into the other buffer) runs while C_j works on S_j, which is the
// coarse pipeline's "T_{j+1} overlaps C_j" (ref schedule.hpp:18-74). P_j (bf16, 2 per column) is
// written back over the first half of its S buffer and read by U_j; the next write of that
// buffer (QK_{j+2}) is issued after U_j by the same thread, and tcgen05 ops from one thread
// execute in order.
//
// The U stage of step j is issued only after C_j has written P_j (the hardware hazard noted in
// the reference can issue U_{j-1} before C_{j-1} because it materialises MMA values
// lazily; a real tensor core cannot).
#pragma once

#include <atomic>
#include <string>

#include "../../include/ws.h"
#include "ws_aref.cuh"

namespace ws {

constexpr int ATTN_BM = 128;  // query rows per Q tile (one TMEM lane each)
constexpr int ATTN_BN = 64;   // keys per K/V tile (S double-buffered in TMEM)
constexpr int ATTN_THREADS = 384;
constexpr int ATTN_MAX_KV_STAGES = 8;
constexpr float ATTN_RESCALE_THRESHOLD = 8.0f;  // log2 units: P values stay <= 2^8 between rescales

struct AttnParams {
  int S, Dh, BH_begin, num_pairs;  // num_pairs = S / 256 work items per (b,h)
  int kv_stages;
  int causal;
  float scale_log2;  // softmax_scale * log2(e)
  float* lse;
  float* mx;  // optional: exact row max of the scaled scores (natural units; the .k's %m)
  void* o;
  int o_elem;  // 0 = bf16, 1 = f16
  // optional device trace (ws_attn_fwd_traced): %clock64 stamps of CTA (0,0), see ATTN_TRACE_*
  unsigned long long* trace;
};

// trace layout: trace[(role * ATTN_TRACE_STEPS + j) * 8 + event], role 0 = MMA issuer,
// 1 / 2 = softmax warp 0 / 4 (tile 0 / 1), lane 0. Events:
//   MMA:     0 step start, 1 QK_{j+1} issued (both tiles), 2 p_full[0] passed, 3 PV0 issued,
//            4 p_full[1] passed, 5 PV1 issued
//   softmax: 0 wait s_full start, 1 s_full passed, 2 S loaded, 3 max done (+rescale),
//            4 P stored, 5 p_full arrived
constexpr int ATTN_TRACE_STEPS = 256;
__device__ __forceinline__ unsigned long long clk64() {
  unsigned long long c;
  asm volatile("mov.u64 %0, %%clock64;" : "=l"(c));
  return c;
}

__host__ __device__ inline uint32_t attn_q_bytes(int Dh) { return ATTN_BM * Dh * 2; }
__host__ __device__ inline uint32_t attn_kv_bytes(int Dh) { return ATTN_BN * Dh * 2; }

__host__ __device__ inline uint32_t attn_smem_bytes(int Dh, int kv_stages) {
  // Q0 | Q1 | kv slots | barriers (+1 KB alignment slack)
  return 2 * attn_q_bytes(Dh) + kv_stages * attn_kv_bytes(Dh) + (2 * ATTN_MAX_KV_STAGES + 16) * 8 + 16 + 1024;
}

// POLY = how many of every 8 column pairs are exponentiated on the FMA pipe (exp2_poly2) instead of
// MUFU (16 ex2/clk/SM). Measured (scripts/micro/softmax_loop.cu): 3 of 8 is the fastest mix.
__host__ __device__ constexpr bool attn_poly_pair(int POLY, int i) {
  return POLY == 0 ? false
       : POLY == 1 ? (i == 3)
       : POLY == 2 ? (i == 1 || i == 5)
       : POLY == 3 ? (i == 1 || i == 4 || i == 6)
       : POLY == 4 ? (i & 1) == 1
                   : (i != 0 && i != 3 && i != 6);
}

template <int DH, bool BF16, int POLY = 3>
__global__ void __launch_bounds__(ATTN_THREADS, 1)
    ws_attn_fwd_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                       const __grid_constant__ CUtensorMap tm_v, const AttnParams p) {
  constexpr uint32_t QTILE = ATTN_BM * DH * 2;      // bytes of a 128 x DH Q tile
  constexpr uint32_t KVTILE = ATTN_BN * DH * 2;     // bytes of a 64 x DH K or V tile
  constexpr uint32_t QPANEL = ATTN_BM * 128;        // one 64-column (128 B) swizzle panel of Q
  constexpr uint32_t KVPANEL = ATTN_BN * 128;       // one 64-column panel of K / V
  constexpr int NPANEL = DH / 64;
  constexpr uint32_t FMT = BF16 ? 1u : 0u;
  constexpr uint32_t IDESC_QK = make_idesc(FMT, ATTN_BM, ATTN_BN, 0, 0);
  constexpr uint32_t IDESC_PV = make_idesc(FMT, ATTN_BM, DH, 0, 1);  // B = V is MN-major
  constexpr uint32_t COL_O = 4 * ATTN_BN;

  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sq = smem;                  // Q0, Q1
  uint8_t* skv = smem + 2 * QTILE;     // K/V ring
  uint8_t* bar_base = skv + p.kv_stages * KVTILE;
  auto* ring = reinterpret_cast<ArefBarriers<ATTN_MAX_KV_STAGES>*>(bar_base);
  uint64_t* q_full = reinterpret_cast<uint64_t*>(bar_base + 2 * ATTN_MAX_KV_STAGES * 8);
  // Per (tile t, S buffer b) barriers, index 2*t + b: the MMA issuer runs one step ahead of the
  // softmax (T_{j+1} before waiting for C_j), so a per-tile barrier could complete two phases
  // before its waiter looks and the parity test would alias; per-buffer barriers complete once
  // every two steps and cannot.
  uint64_t* s_full = q_full + 1;   // [4]: QK_j[t] into S_t[j%2] complete
  uint64_t* p_full = q_full + 5;   // [4]: P_j[t] in S_t[j%2], O_t rescaled
  uint64_t* pv_done = q_full + 9;  // [4]: PV_j[t] (P from S_t[j%2]) complete
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(q_full + 13);

  const uint32_t warp = warp_id();
  const uint32_t lane = lane_id();
  const uint32_t D = static_cast<uint32_t>(p.kv_stages);

  // work item: blockIdx.x = (b,h) slice (fastest), blockIdx.y = query pair, heaviest (latest,
  // for causal) pairs dispatched first
  const int pair = p.num_pairs - 1 - static_cast<int>(blockIdx.y);
  const int bh = p.BH_begin + static_cast<int>(blockIdx.x);
  const int q_row0 = bh * p.S + pair * 2 * ATTN_BM;  // row in the [B*H*S, Dh] view
  const int n_kv = p.causal ? (pair * 2 * ATTN_BM + 2 * ATTN_BM) / ATTN_BN : p.S / ATTN_BN;
  unsigned long long* const trace =
      (p.trace != nullptr && blockIdx.x == 0 && blockIdx.y == 0) ? p.trace : nullptr;
#define WS_TRACE(role, j, ev)                                                        \
  do {                                                                              \
    if (trace != nullptr && (j) < ATTN_TRACE_STEPS)                                 \
      trace[((role) * ATTN_TRACE_STEPS + (j)) * 8 + (ev)] = clk64();                \
  } while (0)

  if (warp == 8 && lane == 0) {
    tma_prefetch_desc(&tm_q);
    tma_prefetch_desc(&tm_k);
    tma_prefetch_desc(&tm_v);
    ring->init(D, 1, 1);
    mbar_init(q_full, 1);
    for (int i = 0; i < 4; ++i) {
      mbar_init(&s_full[i], 1);
      mbar_init(&p_full[i], 4);
      mbar_init(&pv_done[i], 1);
    }
    fence_barrier_init();
  } else if (warp == 10) {
    tmem_alloc<1>(tmem_slot, 512);
    tmem_relinquish<1>();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  pdl_wait();  // programmatic dependent launch: the setup above overlapped the previous grid's tail
  pdl_launch_dependents();

  // Register budget: the producer/MMA warpgroup needs few registers, the two softmax warpgroups
  // hold an S row each. 72*128 + 216*256 = 64512 <= 64K (= 168 * 384 at launch). Each role
  // branch reallocates on entry so ptxas sees one budget per region.
  if (warp == 8) {
    // ===================== producer =====================
    // aref order = MMA consumption order: K_0, then (K_{j+1}, V_j) for j = 0..n-1
    regs_dec<72>();
    if (lane == 0) {
      mbar_arrive_expect_tx(q_full, 2 * QTILE);
#pragma unroll
      for (int t = 0; t < 2; ++t)
#pragma unroll
        for (int h = 0; h < NPANEL; ++h)
          tma_load_2d(sq + t * QTILE + h * QPANEL, &tm_q, q_full, h * 64, q_row0 + t * ATTN_BM);
      ArefCursor c;
      const int kv_row0 = bh * p.S;
      auto put = [&](const CUtensorMap* m, int blk) {
        ring->put_acquire(c, 10);
        ring->put_expect(c, KVTILE);
        uint8_t* dst = skv + c.slot * KVTILE;
#pragma unroll
        for (int h = 0; h < NPANEL; ++h)
          tma_load_2d(dst + h * KVPANEL, m, &ring->full[c.slot], h * 64, kv_row0 + blk * ATTN_BN);
        c.advance(D);
      };
      put(&tm_k, 0);
      for (int j = 0; j < n_kv; ++j) {
        if (j + 1 < n_kv) put(&tm_k, j + 1);
        put(&tm_v, j);
      }
    }
  } else if (warp == 9) {
    // ===================== MMA issuer =====================
    // The whole warp runs this loop (warp-uniform operands, one elected lane issues).
    regs_dec<72>();
    {
      // descriptors are computed once; a K step or a slot only moves the 14-bit address field
      // (smem addresses < 256 KB, so the add never carries out of it)
      const uint64_t qdesc = make_sw128_desc(smem_u32(sq), 16, 1024);
      const uint64_t kdesc = make_sw128_desc(smem_u32(skv), 16, 1024);
      const uint64_t vdesc = make_sw128_desc(smem_u32(skv), KVPANEL, 1024);
      auto issue_qk = [&](int t, int buf, uint32_t k_slot) {
        const uint64_t a0 = qdesc + ((t * QTILE) >> 4), b0 = kdesc + ((k_slot * KVTILE) >> 4);
#pragma unroll
        for (int k = 0; k < DH / 16; ++k) {
          const uint32_t off = ((k / 4) * KVPANEL + (k % 4) * 32) >> 4;
          const uint32_t qoff = ((k / 4) * QPANEL + (k % 4) * 32) >> 4;
          mma_f16_ss_warp(tmem + (2 * t + buf) * ATTN_BN, a0 + qoff, b0 + off, IDESC_QK, k != 0);
        }
      };
      auto issue_pv = [&](int t, int buf, uint32_t v_slot, bool acc) {
        const uint64_t b0 = vdesc + ((v_slot * KVTILE) >> 4);
#pragma unroll
        for (int k = 0; k < ATTN_BN / 16; ++k) {
          // A = P_t[buf]: 16 keys = 8 packed columns; B = V rows [16k, 16k+16): two 8-row groups
          mma_f16_ts_warp(tmem + COL_O + t * DH, tmem + (2 * t + buf) * ATTN_BN + k * 8, b0 + ((k * 16 * 128) >> 4),
                          IDESC_PV, (acc || k != 0) ? 1u : 0u);
        }
      };
      mbar_wait(q_full, 0, 11);
      ArefCursor c;
      // prologue: T_0 for both tiles
      ring->get(c, 12);
      tc_fence_after();
      issue_qk(0, 0, c.slot);
      mma_commit_warp(&s_full[0]);
      issue_qk(1, 0, c.slot);
      mma_commit_warp(&s_full[2]);
      mma_commit_warp(&ring->empty[c.slot]);
      c.advance(D);
      for (int j = 0; j < n_kv; ++j) {
        if (lane == 0) WS_TRACE(0, j, 0);
        if (j + 1 < n_kv) {
          // T_{j+1}: into the other S buffer while the softmax warps run C_j
          ring->get(c, 13);
          tc_fence_after();
          const int nb = (j + 1) & 1;
          issue_qk(0, nb, c.slot);
          mma_commit_warp(&s_full[nb]);
          issue_qk(1, nb, c.slot);
          mma_commit_warp(&s_full[2 + nb]);
          mma_commit_warp(&ring->empty[c.slot]);
          c.advance(D);
        }
        if (lane == 0) WS_TRACE(0, j, 1);
        ring->get(c, 14);  // V_j
        tc_fence_after();
#pragma unroll
        for (int t = 0; t < 2; ++t) {
          mbar_wait(&p_full[2 * t + (j & 1)], (j >> 1) & 1, 15 + t);  // C_j[t] done: P_j[t] in TMEM
          if (lane == 0) WS_TRACE(0, j, 2 + 2 * t);
          tc_fence_after();
          issue_pv(t, j & 1, c.slot, j > 0);
          mma_commit_warp(&pv_done[2 * t + (j & 1)]);
          if (lane == 0) WS_TRACE(0, j, 3 + 2 * t);
        }
        mma_commit_warp(&ring->empty[c.slot]);
        c.advance(D);
      }
    }
  } else if (warp >= 8) {
    regs_dec<72>();
  } else {
    // ===================== softmax / correction / epilogue =====================
    regs_inc<216>();
    const int t = warp / 4;           // Q tile
    const uint32_t q = warp & 3u;     // TMEM lane quarter
    const int row = q * 32 + lane;    // row within the Q tile
    const uint32_t t_lane = (q * 32u) << 16;
    const uint32_t t_o = tmem + t_lane + COL_O + t * DH;
    const int tile_q0 = pair * 2 * ATTN_BM + t * ATTN_BM;
    const int qpos = tile_q0 + row;  // query position in the sequence
    const float sl2 = p.scale_log2;
    float m_used = -INFINITY;  // running max (log2 units) the current P/O are relative to
    float m_true = -INFINITY;  // exact running row max (log2 units; the .k's %m, for p.mx)
    float l = 0.f;
    const bool tr = lane == 0 && (warp & 3u) == 0;
    for (int j = 0; j < n_kv; ++j) {
      const uint32_t t_s = tmem + t_lane + (2 * t + (j & 1)) * ATTN_BN;
      if (tr) WS_TRACE(1 + t, j, 0);
      mbar_wait(&s_full[2 * t + (j & 1)], (j >> 1) & 1, 20 + t);
      if (tr) WS_TRACE(1 + t, j, 1);
      tc_fence_after();
      float s[ATTN_BN];
      {
        uint32_t* su = reinterpret_cast<uint32_t*>(s);
        tmem_ld32(t_s + 0, *reinterpret_cast<uint32_t(*)[32]>(su + 0));
        tmem_ld32(t_s + 32, *reinterpret_cast<uint32_t(*)[32]>(su + 32));
        tmem_wait_ld();
      }
      if (tr) WS_TRACE(1 + t, j, 2);
      if (p.causal && j * ATTN_BN + ATTN_BN - 1 > tile_q0) {
        // block intersects the upper triangle of this tile: mask key > query
        const int lim = qpos - j * ATTN_BN;  // last visible column of this row
#pragma unroll
        for (int c = 0; c < ATTN_BN; ++c) s[c] = c > lim ? -INFINITY : s[c];
      }
      float mx;
      {
        float m4[4] = {s[0], s[1], s[2], s[3]};
#pragma unroll
        for (int c = 4; c < ATTN_BN; c += 4) {
          m4[0] = fmaxf(m4[0], s[c]);
          m4[1] = fmaxf(m4[1], s[c + 1]);
          m4[2] = fmaxf(m4[2], s[c + 2]);
          m4[3] = fmaxf(m4[3], s[c + 3]);
        }
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
      // U_{j-1}[t] has landed (observed every step, so no pv_done phase completes unobserved —
      // compute-sanitizer synccheck; it is long done by now). T_j completing implies U_{j-2}
      // (issued before it) completed, and U_{j+1} cannot exist yet, so the buffer barrier of
      // U_{j-1} is at most one phase behind and its parity test is unambiguous.
      if (j > 0) mbar_wait(&pv_done[2 * t + ((j - 1) & 1)], ((j - 1) >> 1) & 1, 24 + t);
      if (j > 0 && __any_sync(0xffffffffu, need)) {
        // correction: O_t row *= alpha
        tc_fence_after();
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
      // P = 2^(s*sl2 - m): packed FFMA2 for the scale/shift and FADD2 for the row sum; 3 of every
      // 8 column pairs are exponentiated on the FMA pipe (exp2_poly2), the rest on MUFU, so the
      // 16/clk/SM MUFU rate stops being the bound at hdim 128 (SURVEY.md §7 "MUFU exp throughput").
      // P goes back into TMEM over its S buffer, 32 columns (16 packed words) at a time.
      const uint64_t sl2x2 = f2_pack(sl2, sl2), negm2 = f2_pack(-m_used, -m_used);
      uint64_t sum2 = f2_pack(0.f, 0.f);
#pragma unroll
      for (int c0 = 0; c0 < ATTN_BN; c0 += 32) {
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
          sum2 = f2_add(sum2, p2);
          float p0, p1;
          f2_unpack(p2, p0, p1);
          pk[(c - c0) / 2] = BF16 ? pack_bf16(p0, p1) : pack_f16(p0, p1);
        }
        tmem_st16(t_s + c0 / 2, pk);
      }
      {
        float a, b;
        f2_unpack(sum2, a, b);
        l += a + b;
      }
      tmem_wait_st();
      if (tr) WS_TRACE(1 + t, j, 4);
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&p_full[2 * t + (j & 1)]);
      if (tr) WS_TRACE(1 + t, j, 5);
    }
    // epilogue: O_t / l -> global, lse once U_{n-1}[t] (and, in issue order, everything before it)
    // has completed
    mbar_wait(&pv_done[2 * t + ((n_kv - 1) & 1)], ((n_kv - 1) >> 1) & 1, 26 + t);
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
    if (p.mx) p.mx[grow] = m_true * 0.69314718055994531f;
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 10) {
    tc_fence_after();
    tmem_dealloc<1>(tmem, 512);
  }
#undef WS_TRACE
}

}  // namespace ws
