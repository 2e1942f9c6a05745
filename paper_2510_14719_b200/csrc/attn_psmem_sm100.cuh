// attn_psmem_sm100.cuh — FlashAttention forward for sm_100a, 128-key K/V blocks, P staged in
// shared memory.
//
// Same reference semantics as attn_sm100.cuh / attn128_sm100.cuh (the flash .k of SURVEY.md
// Appendix A: coarse T/C/U pipeline, ref proj/include/warpspec/pipeline.hpp:160-328,
// schedule.hpp:18-74). What changes is where P lives:
//
//   attn128: P_t(j) is written back over S_t in TMEM, so QK_t(j+1) can only be issued after
//            PV_t(j) — the T stage of block j+1 waits for the whole C stage of block j, and the
//            tile's chain per block is softmax + PV + QK (measured ~3000 cycles per 128 keys).
//   here:    the softmax warps copy S_t(j) into registers and release it at once (s_free), and
//            P_t(j) goes to a shared-memory tile read by an SS-form PV MMA (128x128x16 SS MMAs run
//            at the tensor floor, scripts/micro/mma_rate.cu). QK_t(j+1) therefore runs while the
//            softmax of block j is still exponentiating — the coarse schedule's "T_{j+1} overlaps
//            C_j" (ref schedule.hpp:18-74) for both Q tiles at once, with S single-buffered in TMEM.
//
// TMEM (512 columns): S_0 | S_1 (128 each) | O_0 | O_1 (Dh each).
// Shared memory: Q_0 | Q_1 | P_0 | P_1 (128 x 128 bf16, K-major SW128, the A operand of PV) | K/V ring.
// Barriers per Q tile t (each completes once per block, and no party can run a phase ahead of a
// waiter that has not yet seen the previous phase, so parity tests never alias):
//   s_full[t]  QK_t(j) complete                          (tcgen05.commit)
//   s_free[t]  S_t(j) copied to registers                 (4 softmax warps)
//   p_full[t]  P_t(j) in shared memory, O_t rescaled      (4 softmax warps)
//   pv_done[t] PV_t(j) complete: P_t and O_t reusable     (tcgen05.commit)
// The kernel is persistent (ref proj/include/warpspec/grid.hpp:93-123): grid = min(#SMs, work
// items), CTA b runs items b, b + grid, ... in a static stride, and no barrier is reset between
// items — the phases carry over, counted by running per-tile block counters (g) and an item
// counter (it). Three more barriers hand the per-item buffers over to the next item:
//   q_full     Q_0, Q_1 of item it landed                 (TMA transaction bytes)
//   q_free     the last QK of item it completed: Q smem reusable (tcgen05.commit)
//   o_free[t]  O_t of item it copied out by the epilogue: PV_t(0) of item it+1 may overwrite it
// so the next item's Q load and first QKs run under the previous item's last softmax steps and
// epilogue (what makes short sequences — 8 K/V blocks per item at S = 1K — efficient).
#pragma once

#include "attn128_sm100.cuh"

namespace ws {

// default exp mix of this kernel: 1 of every 8 column pairs on the FMA pipe. With the staggered
// issue order (p.stagger) the two softmax warpgroups overlap, so the FMA pipe is the scarcer one
// (measured, scripts/attn_ab.py: stagger + 1/8 beats 2/8 by 3-4% at hdim 128).
constexpr int APS_POLY = 1;

constexpr uint32_t APS_BAR_BYTES = (2 * A128_MAX_STAGES + 24) * 8;  // ring + per-tile / V barriers, TMEM slot

__host__ __device__ inline uint32_t aps_smem_bytes(int Dh, int kv_stages) {
  // Q0 | Q1 | P0 | P1 | kv slots | barriers (+1 KB alignment slack)
  return 2 * a128_q_bytes(Dh) + 2 * A128_BM * A128_BN * 2 + kv_stages * a128_kv_bytes(Dh) + APS_BAR_BYTES + 1024;
}

// FP8: Q, K, V in e4m3. QK^T runs in kind::f8f6f4; P stays 16-bit (f16 in shared memory) and PV
// runs in kind::f16 against V converted e4m3 -> f16 in shared memory by two converter warps
// (exact: every e4m3 value is an f16). V then has its own depth-2 aref with a transform stage:
// TMA lands V_j (e4m3) in the upper half of f16 buffer j % 2 (vfull), the converter widens it in
// place (each thread reads its whole 128-byte row before writing; f16 panel 1 of row r covers
// exactly the bytes of e4m3 row r) and signals v16_full, PV_0(j) and PV_1(j) read it and commit
// vempty. Every party walks every V position in order, so no parity test can alias; the K blocks
// keep the ring (the MMA warp is their only consumer). Quantizing P itself to e4m3 (3 mantissa bits) left O up to
// ~6% of max|V| off the fp32-accumulated oracle; f16 P keeps it at the 16-bit kernels' error.
// Per-tensor descales fold into the softmax scale (q, k) and the epilogue (v); O in bf16.

template <int DH, bool BF16, int POLY = 2, bool TRACE = false, bool FP8 = false>
__global__ void __launch_bounds__(A128_THREADS, 1)
    ws_attn_psmem_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                         const __grid_constant__ CUtensorMap tm_v, const __grid_constant__ CUtensorMap tm_o,
                         const Attn128Params p) {
  constexpr int EB = FP8 ? 1 : 2;                     // Q / K / V element bytes
  constexpr int PEB = 2;                              // P element bytes (16-bit, also for FP8)
  constexpr uint32_t QTILE = A128_BM * DH * EB;       // bytes of a 128 x DH Q tile
  constexpr uint32_t PTILE = A128_BM * A128_BN * PEB; // bytes of a 128 x 128 P tile
  constexpr uint32_t KVTILE = A128_BN * DH * EB;      // bytes of a 128 x DH K or V block
  constexpr uint32_t V16TILE = FP8 ? A128_BN * DH * 2 : 0;  // FP8: a V block converted to f16
  constexpr uint32_t PANEL = 128 * 128;              // one 64-column (128 B) swizzle panel of 128 rows
  constexpr int NPANEL = DH * EB / 128;               // 128-byte panels per Q / K / V row
  constexpr int PANEL_ELEMS = 128 / EB;
  constexpr uint32_t FMT_QK = FP8 ? 0u : BF16 ? 1u : 0u;     // kind::f8f6f4 e4m3 / kind::f16 bf16, f16
  constexpr uint32_t FMT_PV = (BF16 && !FP8) ? 1u : 0u;      // kind::f16: bf16, or f16 (FP8: f16 P, V)
  constexpr uint32_t IDESC_QK = make_idesc(FMT_QK, A128_BM, A128_BN, 0, 0);
  constexpr uint32_t IDESC_PV = make_idesc(FMT_PV, A128_BM, DH, 0, 1);  // A = P K-major, B = V MN-major
  constexpr uint32_t COL_O = 2 * A128_BN;
  constexpr uint32_t TMEM_COLS = 2 * A128_BN + 2 * DH <= 256 ? 256 : 512;

  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sq = smem;                  // Q0, Q1
  uint8_t* sp = smem + 2 * QTILE;      // P0, P1
  uint8_t* skv = sp + 2 * PTILE;       // K/V ring
  uint8_t* sv16 = skv + p.kv_stages * KVTILE;  // FP8: two f16 V buffers (the ring then holds K only)
  uint8_t* bar_base = sv16 + 2 * V16TILE;
  auto* ring = reinterpret_cast<ArefBarriers<A128_MAX_STAGES>*>(bar_base);
  uint64_t* q_full = reinterpret_cast<uint64_t*>(bar_base + 2 * A128_MAX_STAGES * 8);
  uint64_t* s_full = q_full + 1;   // [2]
  uint64_t* s_free = q_full + 3;   // [2]
  uint64_t* p_full = q_full + 5;   // [2]
  uint64_t* pv_done = q_full + 7;  // [2]
  uint64_t* o_free = q_full + 9;   // [2]
  uint64_t* q_free = q_full + 11;
  uint64_t* v16_full = q_full + 12;   // [2] FP8: V_j converted to f16 (converter warps)
  uint64_t* v16_empty = q_full + 14;  // [2] FP8: PV_0(j), PV_1(j) have read it (tcgen05.commit)
  uint64_t* vfull = q_full + 16;      // [2] FP8: V_j (e4m3) landed (TMA transaction bytes)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(q_full + 18);

  const uint32_t warp = warp_id();
  const uint32_t lane = lane_id();
  const uint32_t D = static_cast<uint32_t>(p.kv_stages);

  // work item i -> (query pair, (b,h)): causal walks (b,h) fastest from the heaviest pairs down
  // (longest first); non-causal walks the query pairs of one (b,h) together (its K/V stay in L2)
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
  // K/V blocks per tile: causal tile t of pair i sees blocks 0 .. 2i+t (its diagonal block last)
  auto nblk = [&](int pair, int t) { return p.causal ? 2 * pair + 1 + t : p.S / A128_BN; };
  const int num_items = p.num_pairs * nbh;
  // CTA b takes the r-th item of its static schedule: plain stride for uniform (non-causal) items;
  // for causal items (listed heaviest first) a snake — rounds alternate direction, so each CTA's
  // heavy and light items pair up (b with 2G-1-b) and the per-CTA totals stay balanced
  const int G = static_cast<int>(gridDim.x), b_id = static_cast<int>(blockIdx.x);
  auto item_of = [&](int r) { return r * G + ((p.causal && (r & 1)) ? G - 1 - b_id : b_id); };
  unsigned long long* const trace =
      (TRACE && p.trace != nullptr && blockIdx.x == 0) ? p.trace : nullptr;
  // stamps of CTA 0, indexed by the running block counter across its items
#define WS_TRACE(role, j, ev)                                                        \
  do {                                                                              \
    if (TRACE && trace != nullptr && (j) < ATTN_TRACE_STEPS)                        \
      trace[((role) * ATTN_TRACE_STEPS + (j)) * 8 + (ev)] = clk64();                \
  } while (0)

  if (warp == 8 && lane == 0) {
    tma_prefetch_desc(&tm_q);
    tma_prefetch_desc(&tm_k);
    tma_prefetch_desc(&tm_v);
    tma_prefetch_desc(&tm_o);
    ring->init(D, 1, 1);
    mbar_init(q_full, 1);
    mbar_init(q_free, 1);
    for (int i = 0; i < 2; ++i) {
      mbar_init(&s_full[i], 1);
      mbar_init(&s_free[i], 4);
      mbar_init(&p_full[i], 4);
      mbar_init(&pv_done[i], 1);
      mbar_init(&o_free[i], 4);
      mbar_init(&v16_full[i], 1);
      mbar_init(&v16_empty[i], 1);
      mbar_init(&vfull[i], 1);
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
      uint32_t vcnt = 0;  // FP8: V blocks put
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
        // FP8: V_j -> the upper half of f16 buffer vcnt % 2, once PV_0, PV_1 of V_{j-2} are done
        auto put_v = [&](int blk) {
          const uint32_t b = vcnt & 1u;
          mbar_wait(&v16_empty[b], ((vcnt >> 1) & 1u) ^ 1u, 10);
          mbar_arrive_expect_tx(&vfull[b], KVTILE);
          tma_load_2d(sv16 + b * V16TILE + V16TILE / 2, &tm_v, &vfull[b], 0, kv_row0 + blk * A128_BN);
          ++vcnt;
        };
        // ring order = MMA consumption order: K_0, then (K_{j+1}, V_j) for j = 0 .. n1-1
        put(&tm_k, 0);
        for (int j = 0; j < n1; ++j) {
          if (j + 1 < n1) put(&tm_k, j + 1);
          if constexpr (FP8)
            put_v(j);
          else
            put(&tm_v, j);
        }
      }
    }
  } else if (warp == 9) {
    // ===================== MMA issuer (whole warp, one elected lane issues) =====================
    regs_dec<72>();
    // shared-space barrier addresses, computed once: the loop then issues no generic -> shared
    // conversions (each re-derived the 1 KB-aligned base from the shared window)
    const uint32_t a_sfull[2] = {smem_u32_pinned(&s_full[0]), smem_u32_pinned(&s_full[1])};
    const uint32_t a_sfree[2] = {smem_u32_pinned(&s_free[0]), smem_u32_pinned(&s_free[1])};
    const uint32_t a_pfull[2] = {smem_u32_pinned(&p_full[0]), smem_u32_pinned(&p_full[1])};
    const uint32_t a_pvdone[2] = {smem_u32_pinned(&pv_done[0]), smem_u32_pinned(&pv_done[1])};
    const uint32_t a_ofree[2] = {smem_u32_pinned(&o_free[0]), smem_u32_pinned(&o_free[1])};
    const uint32_t a_qfull = smem_u32_pinned(q_full), a_qfree = smem_u32_pinned(q_free);
    const uint32_t a_v16full = smem_u32_pinned(&v16_full[0]), a_v16empty = smem_u32_pinned(&v16_empty[0]);
    const uint32_t a_rfull = smem_u32_pinned(&ring->full[0]), a_rempty = smem_u32_pinned(&ring->empty[0]);
    auto ring_get = [&](const ArefCursor& cc, uint32_t tag) { mbar_wait(a_rfull + 8u * cc.slot, cc.phase, tag); };
    const uint64_t qdesc = make_sw128_desc(smem_u32(sq), 16, 1024);
    const uint64_t pdesc = make_sw128_desc(smem_u32(sp), 16, 1024);
    const uint64_t kdesc = make_sw128_desc(smem_u32(skv), 16, 1024);
    const uint64_t vdesc = make_sw128_desc(smem_u32(FP8 ? sv16 : skv), PANEL, 1024);
    auto issue_qk = [&](int t, uint32_t k_slot) {
      const uint64_t a0 = qdesc + ((t * QTILE) >> 4), b0 = kdesc + ((k_slot * KVTILE) >> 4);
#pragma unroll
      for (int k = 0; k < DH * EB / 32; ++k) {  // one MMA per 32 bytes of the head dim
        const uint32_t off = ((k / 4) * PANEL + (k % 4) * 32) >> 4;
        if constexpr (FP8)
          mma_f8_ss_warp(tmem + t * A128_BN, a0 + off, b0 + off, IDESC_QK, k != 0);
        else
          mma_f16_ss_warp(tmem + t * A128_BN, a0 + off, b0 + off, IDESC_QK, k != 0);
      }
    };
    auto issue_pv = [&](int t, uint32_t v_slot, bool acc) {
      // V from the K/V ring slot, or (FP8) from f16 buffer v_slot
      const uint64_t a0 = pdesc + ((t * PTILE) >> 4), b0 = vdesc + ((v_slot * (FP8 ? V16TILE : KVTILE)) >> 4);
      constexpr int KEYS = 32 / PEB;  // keys per MMA (32 bytes of P)
#pragma unroll
      for (int k = 0; k < A128_BN / KEYS; ++k) {
        // A = P_t keys [KEYS k, KEYS (k+1)) (K-major, panel k/4); B = V rows of those keys
        // (MN-major, KEYS/8 eight-row core groups of 128 bytes)
        const uint32_t aoff = ((k / 4) * PANEL + (k % 4) * 32) >> 4;
        mma_f16_ss_warp(tmem + COL_O + t * DH, a0 + aoff, b0 + ((k * KEYS * 128) >> 4), IDESC_PV,
                        (acc || k != 0) ? 1u : 0u);
      }
    };
    uint32_t vcnt = 0;  // FP8: V blocks consumed (f16 buffer vcnt % 2, phase vcnt / 2 % 2)
    ArefCursor c;
    uint32_t g0 = 0, g1 = 0;  // blocks of tile 0 / tile 1 processed by earlier items
    // First QK of tile 0 of item `it` (K_0 taken from the ring, its slot kept for tile 1's QK). It
    // is issued inside the previous item's last step, right after that item's last PV_0, so the
    // next item's first S_0 is computed while tile 1 finishes the current item (cross-item
    // software pipelining of the T stage; Q of item it was loaded after the previous item's last
    // QK released it).
    uint32_t k0slot = 0;
    auto first_qk0 = [&](int it_, uint32_t g0_) {
      mbar_wait(a_qfull, it_ & 1, 11);
      ring_get(c, 12);  // K_0
      k0slot = c.slot;
      c.advance(D);
      tc_fence_after();
      if (g0_ > 0) {
        mbar_wait(a_sfree[0], (g0_ - 1) & 1, 17);  // the previous item's last S_0 copied out
        tc_fence_after();
      }
      issue_qk(0, k0slot);
      mma_commit_warp(a_sfull[0]);
    };
    bool qk0_issued = false;
    for (int it = 0, item = item_of(0); item < num_items; item = item_of(++it)) {
      int pair, bh;
      item_coords(item, pair, bh);
      const int n0 = nblk(pair, 0), n1 = nblk(pair, 1);
      if (!qk0_issued) first_qk0(it, g0);
      qk0_issued = false;
      if (g1 > 0) {
        mbar_wait(a_sfree[1], (g1 - 1) & 1, 18);
        tc_fence_after();
      }
      issue_qk(1, k0slot);
      mma_commit_warp(a_sfull[1]);
      mma_commit_warp(a_rempty + 8u * k0slot);
      const int next_item = item_of(it + 1);
      for (int j = 0; j < n1; ++j) {
        if (lane == 0) WS_TRACE(0, g1 + j, 0);
        const bool more = j + 1 < n1;
        uint32_t kslot = 0;
        auto qk1 = [&]() {
          mbar_wait(a_sfree[1], (g1 + j) & 1, 18);
          tc_fence_after();
          issue_qk(1, kslot);
          mma_commit_warp(a_sfull[1]);
          mma_commit_warp(a_rempty + 8u * kslot);
          if (j + 2 == n1) mma_commit_warp(a_qfree);  // that was the item's last QK: Q reusable
        };
        if (more) {
          ring_get(c, 13);  // K_{j+1}
          kslot = c.slot;
          c.advance(D);
          if (lane == 0) WS_TRACE(0, g1 + j, 6);
          if (j + 1 < n0) {
            mbar_wait(a_sfree[0], (g0 + j) & 1, 17);  // S_0(j) copied out
            tc_fence_after();
            issue_qk(0, kslot);
            mma_commit_warp(a_sfull[0]);
          }
          if (lane == 0) WS_TRACE(0, g1 + j, 1);
          if (!p.stagger) qk1();
        }
        if (lane == 0) WS_TRACE(0, g1 + j, 2);
        uint32_t vslot;
        if constexpr (FP8) {
          vslot = vcnt & 1u;  // V_j's f16 copy (the ring carries K only)
          mbar_wait(a_v16full + 8u * vslot, (vcnt >> 1) & 1u, 14);
        } else {
          ring_get(c, 14);  // V_j
          vslot = c.slot;
          c.advance(D);
        }
        if (lane == 0) WS_TRACE(0, g1 + j, 7);
        if (j < n0) {
          mbar_wait(a_pfull[0], (g0 + j) & 1, 15);  // C_0(j): P_0(j) in smem, O_0 rescaled
          if (j == 0 && it > 0) mbar_wait(a_ofree[0], (it - 1) & 1, 19);  // previous O_0 copied out
          tc_fence_after();
          if (lane == 0) WS_TRACE(0, g1 + j, 3);
          issue_pv(0, vslot, j > 0);
          mma_commit_warp(a_pvdone[0]);
        }
        // stagger: QK_1(j+1) after PV_0(j), so tile 1's S lands half a step after tile 0's and the
        // two softmax warpgroups' latency-bound phases (row max) interleave with the other's
        // exponentials instead of coinciding
        if (more && p.stagger) qk1();
        if (!more && next_item < num_items) {
          first_qk0(it + 1, g0 + n0);  // the next item's T_0(0), ahead of this item's last PV_1
          qk0_issued = true;
        }
        mbar_wait(a_pfull[1], (g1 + j) & 1, 16);
        if (j == 0 && it > 0) mbar_wait(a_ofree[1], (it - 1) & 1, 19);
        tc_fence_after();
        if (lane == 0) WS_TRACE(0, g1 + j, 4);
        issue_pv(1, vslot, j > 0);
        mma_commit_warp(a_pvdone[1]);
        if constexpr (FP8) {
          mma_commit_warp(a_v16empty + 8u * vslot);
          ++vcnt;
        } else {
          mma_commit_warp(a_rempty + 8u * vslot);
        }
        if (lane == 0) WS_TRACE(0, g1 + j, 5);
      }
      g0 += n0;
      g1 += n1;
    }
  } else if (FP8 && warp >= 10) {
    // ===================== FP8: V converter (warps 10, 11) =====================
    // V_j (e4m3, 128 keys x 128 B, SW128, in the upper half of f16 buffer vcnt % 2) -> f16 in the
    // bf16 kernel's MN-major V layout (two 64-column SW128 panels), in place.
    regs_dec<72>();
    constexpr int NCONV = 2;                         // converter warps
    constexpr int ROWS = A128_BN / (32 * NCONV);     // keys per thread
    const uint32_t ct = (warp - 10u) * 32u + lane;  // keys ct, ct + 32 * NCONV, ...
    // pinned shared-space addresses (vfull / v16_full are adjacent pairs, the f16 V buffers too)
    const uint32_t a_vfull = smem_u32_pinned(&vfull[0]), a_v16full = smem_u32_pinned(&v16_full[0]);
    const uint32_t a_sv16 = smem_u32_pinned(sv16);
    uint32_t vcnt = 0;
    for (int it = 0, item = item_of(0); item < num_items; item = item_of(++it)) {
      int pair, bh;
      item_coords(item, pair, bh);
      const int n1 = nblk(pair, 1);
      for (int j = 0; j < n1; ++j) {
        const uint32_t b = vcnt & 1u;
        mbar_wait(a_vfull + 8u * b, (vcnt >> 1) & 1u, 30);  // V_j landed
        const uint32_t dst = a_sv16 + b * V16TILE, src = dst + V16TILE / 2;
#pragma unroll
        for (int rr = 0; rr < ROWS; ++rr) {
          const uint32_t r = ct + 32u * NCONV * rr, sw = r & 7u;
          uint4 x[8];  // the whole e4m3 row first: its f16 panel-1 half overwrites the same 128 bytes
#pragma unroll
          for (uint32_t cc = 0; cc < 8; ++cc) x[cc] = ld_shared_v4(src + r * 128u + ((cc ^ sw) << 4));
#pragma unroll
          for (uint32_t cc = 0; cc < 8; ++cc) {  // 16 e4m3 (head dims 16cc ..) -> two f16 chunks
            const uint32_t xs[4] = {x[cc].x, x[cc].y, x[cc].z, x[cc].w};
            uint32_t h[8];
#pragma unroll
            for (int w = 0; w < 4; ++w) {
              h[2 * w] = e4m3x2_to_f16x2(xs[w] & 0xffffu);
              h[2 * w + 1] = e4m3x2_to_f16x2(xs[w] >> 16);
            }
            const uint32_t row = dst + (cc / 4u) * PANEL + r * 128u, c8 = 2u * (cc % 4u);
            st_shared_v4(row + ((c8 ^ sw) << 4), h[0], h[1], h[2], h[3]);
            st_shared_v4(row + (((c8 + 1u) ^ sw) << 4), h[4], h[5], h[6], h[7]);
          }
        }
        fence_proxy_async_smem();  // generic-proxy stores -> visible to the tensor core's reads
        if constexpr (NCONV == 2)
          named_bar_sync(3, 64);
        else
          __syncwarp();
        if (ct == 0) mbar_arrive(a_v16full + 8u * b);
        ++vcnt;
      }
    }
  } else if (warp >= 8) {
    regs_dec<72>();
  } else {
    // ===================== softmax / correction / epilogue =====================
    regs_inc<216>();
    const int t = warp / 4;         // Q tile
    const uint32_t q = warp & 3u;   // TMEM lane quarter
    const int row = q * 32 + lane;  // row within the Q tile
    const uint32_t t_lane = (q * 32u) << 16;
    const uint32_t t_s = tmem + t_lane + t * A128_BN;
    const uint32_t t_o = tmem + t_lane + COL_O + t * DH;
    // this thread's row of P_t: two 128-byte-swizzled panels (keys 0-63, 64-127)
    uint32_t p_row = smem_u32(sp + t * PTILE) + row * 128u;
    asm volatile("mov.b32 %0, %0;" : "+r"(p_row));  // pinned (see smem_u32_pinned)
    const uint32_t swz = static_cast<uint32_t>(row & 7);
    const float sl2 = p.scale_log2;
    // shared-space barrier addresses of this tile, computed once (see the MMA warp)
    const uint32_t a_sfull = smem_u32_pinned(&s_full[t]), a_sfree = smem_u32_pinned(&s_free[t]);
    const uint32_t a_pfull = smem_u32_pinned(&p_full[t]), a_pvdone = smem_u32_pinned(&pv_done[t]);
    const uint32_t a_ofree = smem_u32_pinned(&o_free[t]);
    const bool tr = lane == 0 && q == 0;
    uint32_t g = 0;  // blocks of this tile processed by earlier items
    for (int it = 0, item = item_of(0); item < num_items; item = item_of(++it)) {
    int pair, bh;
    item_coords(item, pair, bh);
    const int n_t = nblk(pair, t);
    const int q_row0 = bh * p.S + pair * 2 * A128_BM;
    // S % 256 == 128: the last pair's second tile lies past the sequence — computed on whatever the
    // loads return (the next (b,h)'s rows, or TMA zero fill) and never stored
    const bool tile_valid = (2 * pair + t) * A128_BM < p.S;
    const int j_diag = p.causal ? n_t - 1 : -1;
    float m_used = -INFINITY;  // running max (log2 units) the current P/O are relative to
    float m_true = -INFINITY;  // exact running row max (log2 units; the .k's %m, for p.mx)
    float l = 0.f;
    for (int j = 0; j < n_t; ++j) {
      if (tr) WS_TRACE(1 + t, g + j, 0);
      mbar_wait(a_sfull, (g + j) & 1, 20 + t);
      if (tr) WS_TRACE(1 + t, g + j, 1);
      tc_fence_after();
      // S in two halves: the row max of the first 64 columns runs while the second half is loading
      // (a tcgen05.wait::ld covers every outstanding load, so the halves are waited separately)
      float s[A128_BN];
      uint32_t* su = reinterpret_cast<uint32_t*>(s);
      tmem_ld32(t_s + 0, *reinterpret_cast<uint32_t(*)[32]>(su + 0));
      tmem_ld32(t_s + 32, *reinterpret_cast<uint32_t(*)[32]>(su + 32));
      tmem_wait_ld();
      tmem_ld32(t_s + 64, *reinterpret_cast<uint32_t(*)[32]>(su + 64));
      tmem_ld32(t_s + 96, *reinterpret_cast<uint32_t(*)[32]>(su + 96));
      const bool diag = j == j_diag;
      if (diag) {
#pragma unroll
        for (int c = 0; c < A128_BN / 2; ++c) s[c] = c > row ? -INFINITY : s[c];
      }
      float m4[4] = {fmax3(s[0], s[1], s[2]), fmax3(s[3], s[4], s[5]), fmax3(s[6], s[7], s[8]),
                     fmax3(s[9], s[10], s[11])};
#pragma unroll
      for (int c = 12; c + 8 <= A128_BN / 2; c += 8) {
        m4[0] = fmax3(m4[0], s[c], s[c + 1]);
        m4[1] = fmax3(m4[1], s[c + 2], s[c + 3]);
        m4[2] = fmax3(m4[2], s[c + 4], s[c + 5]);
        m4[3] = fmax3(m4[3], s[c + 6], s[c + 7]);
      }
      m4[0] = fmax3(m4[0], s[60], s[61]);
      m4[1] = fmax3(m4[1], s[62], s[63]);
      tmem_wait_ld();
      // S_t(j) is in registers: release the TMEM columns so QK_t(j+1) can run during this softmax
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(a_sfree);
      if (tr) WS_TRACE(1 + t, g + j, 2);
      if (diag) {
#pragma unroll
        for (int c = A128_BN / 2; c < A128_BN; ++c) s[c] = c > row ? -INFINITY : s[c];
      }
      float mx;
      {
#pragma unroll
        for (int c = A128_BN / 2; c + 8 <= A128_BN; c += 8) {
          m4[0] = fmax3(m4[0], s[c], s[c + 1]);
          m4[1] = fmax3(m4[1], s[c + 2], s[c + 3]);
          m4[2] = fmax3(m4[2], s[c + 4], s[c + 5]);
          m4[3] = fmax3(m4[3], s[c + 6], s[c + 7]);
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
      if (j > 0 && __any_sync(0xffffffffu, need)) {
        // correction: O_t *= alpha once PV_t(j-1) has landed. PV_t(j) needs this warp's p_full,
        // so pv_done is at most one phase behind and the parity test is unambiguous.
        mbar_wait(a_pvdone, (g + j - 1) & 1, 24 + t);
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
        tmem_wait_st();
      }
      l *= alpha;
      if (tr) WS_TRACE(1 + t, g + j, 3);
      // P_t's shared-memory tile is free once PV_t(j-1) has read it (long done by now: PV_t(j-1) was
      // issued when this warp finished block j-1)
      if (g + j > 0) mbar_wait(a_pvdone, (g + j - 1) & 1, 24 + t);
      if (tr) WS_TRACE(1 + t, g + j, 6);
      if (j == 0 && it > 0) {
        // the previous item's O_t was staged through this P tile: its TMA store must have read it
        if (warp == 4u * t && lane == 0) tma_store_wait_read<0>();
        named_bar_sync(1 + t, 128);
      }
      // P = 2^(s*sl2 - m), packed to 16-bit pairs and stored 8 keys (16 bytes) at a time into the
      // 128B-swizzled K-major P tile as it is produced, so the shared-memory writes overlap the math
      const uint64_t sl2x2 = f2_pack(sl2, sl2), negm2 = f2_pack(-m_used, -m_used);
      uint64_t sum4[4];  // row-sum partials, seeded by the first chunk (no adds of zero)
      constexpr int KPC = 16 / PEB;  // keys per 16-byte chunk of the P row
#pragma unroll
      for (int ch = 0; ch < A128_BN / KPC; ++ch) {
        float pf[KPC];
#pragma unroll
        for (int e = 0; e < KPC / 2; ++e) {
          const int c = ch * KPC + 2 * e;
          const uint64_t x2 = f2_fma(f2_pack(s[c], s[c + 1]), sl2x2, negm2);
          uint64_t p2;
          if (attn_poly_pair(POLY, (c / 2) & 7)) {
            p2 = exp2_poly2(x2);
          } else {
            float x0, x1;
            f2_unpack(x2, x0, x1);
            p2 = f2_pack(ex2_approx(x0), ex2_approx(x1));
          }
          sum4[e & 3] = ch == 0 ? p2 : f2_add(sum4[e & 3], p2);
          f2_unpack(p2, pf[2 * e], pf[2 * e + 1]);
        }
        uint32_t pk[4];
#pragma unroll
        for (int w = 0; w < 4; ++w)
          pk[w] = (BF16 && !FP8) ? pack_bf16(pf[2 * w], pf[2 * w + 1]) : pack_f16(pf[2 * w], pf[2 * w + 1]);
        // 16-byte chunk ch = keys [KPC ch, KPC (ch+1)): panel ch/8, swizzled position (ch%8) ^ (row%8)
        const uint32_t addr = p_row + (ch / 8) * PANEL + ((static_cast<uint32_t>(ch & 7) ^ swz) << 4);
        st_shared_v4(addr, pk[0], pk[1], pk[2], pk[3]);
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
      if (lane == 0) mbar_arrive(a_pfull);
      if (tr) WS_TRACE(1 + t, g + j, 5);
    }
    // epilogue: O_t / l -> global, lse once the last PV_t has completed. O_t is copied to registers
    // first and released (o_free) so the next item's PV_t(0) can overwrite it while this finishes.
    g += n_t;
    mbar_wait(a_pvdone, (g - 1) & 1, 26 + t);
    tc_fence_after();
    uint32_t ov[DH];
#pragma unroll
    for (int c0 = 0; c0 < DH; c0 += 32) tmem_ld32(t_o + c0, *reinterpret_cast<uint32_t(*)[32]>(ov + c0));
    tmem_wait_ld();
    tc_fence_before();
    __syncwarp();
    if (lane == 0) mbar_arrive(a_ofree);
    if (tr) WS_TRACE(1 + t, g - 1, 6);
    const float inv_l = p.o_scale / l;  // V's per-tensor descale (FP8) folded into 1 / l
    const uint64_t inv_l2 = f2_pack(inv_l, inv_l);
    const size_t grow = static_cast<size_t>(q_row0 + t * A128_BM + row);
    // O_t leaves through TMA: each thread writes its row (16-bit, 128B-swizzled, 64 columns per
    // 16 KB panel) into this tile's P buffer — free, since its last PV has completed — and one
    // thread stores the 128 x 64 boxes. A thread writing its own 256-byte row straight to global
    // memory would issue 32 scattered 16-byte writes per warp instruction; that epilogue cost
    // ~7000 cycles per work item (scripts/attn_trace_items.py).
    constexpr int OPANELS = DH / 64;                          // 64 output columns per panel
    constexpr int PPANELS = static_cast<int>(PTILE / PANEL);  // staging panels in the P tile
    const uint32_t ptile = smem_u32_pinned(sp + t * PTILE);
#pragma unroll
    for (int c = 0; c < OPANELS; ++c) {
      const uint32_t buf = ptile + (c % PPANELS) * PANEL;
      if (c >= PPANELS) {  // reuse of a staging panel: its previous store must have read it
        if (warp == 4u * t && lane == 0) tma_store_wait_read<0>();
        named_bar_sync(1 + t, 128);
      }
#pragma unroll
      for (int k8 = 0; k8 < 8; ++k8) {
        uint32_t w[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const int col = c * 64 + k8 * 8 + 2 * e;
          float a, b;  // packed FMUL2: one multiply per column pair
          f2_unpack(f2_mul(f2_pack(__uint_as_float(ov[col]), __uint_as_float(ov[col + 1])), inv_l2), a, b);
          w[e] = (BF16 || FP8) ? pack_bf16(a, b) : pack_f16(a, b);
        }
        st_shared_v4(buf + row * 128u + ((static_cast<uint32_t>(k8) ^ swz) << 4), w[0], w[1], w[2], w[3]);
      }
      fence_proxy_async_smem();
      named_bar_sync(1 + t, 128);
      if (warp == 4u * t && lane == 0 && tile_valid) {
        tma_store_2d(&tm_o, reinterpret_cast<const void*>(sp + t * PTILE + (c % PPANELS) * PANEL), c * 64,
                     q_row0 + t * A128_BM);
        tma_store_commit();
      }
    }
    if (p.lse && tile_valid) p.lse[grow] = m_used * 0.69314718055994531f + __logf(l);
    if (p.mx && tile_valid) p.mx[grow] = m_true * 0.69314718055994531f;
    if (tr) WS_TRACE(1 + t, g - 1, 7);
    }  // items
    if (warp == 4u * t && lane == 0) tma_store_wait<0>();  // O stores complete before the CTA retires
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
