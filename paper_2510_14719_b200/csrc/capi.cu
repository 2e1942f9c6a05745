// capi.cu — the C-ABI (include/ws.h): argument validation with the reference's error codes,
// TMA descriptor construction, kernel selection and launch.
//
// Validation mirrors the reference's rejections:
//   D < 1 / P < 1 / P > D      -> PIPELINE_INFEASIBLE   (ref proj/include/warpspec/driver.hpp:117-118,
//                                                         ref proj/include/warpspec/pipeline.hpp:84-92)
//   dimension not tile-aligned -> INDIVISIBLE_TILE      (ref proj/include/warpspec/grid.hpp:43-46)
//   stage bytes x D too large  -> SMEM_OVERFLOW         (ref proj/include/warpspec/sim.hpp:81-84;
//                                                         here against the real 227 KB sm_100a limit)
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <atomic>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <new>
#include <unordered_map>
#include <string>

#include "../../include/ws.h"
#include "attn128_sm100.cuh"
#include "attn_psmem_sm100.cuh"
#include "attn_sm100.cuh"
#include "gemm_sm100.cuh"

namespace {

thread_local std::string g_last_error;
std::atomic<int64_t> g_launches{0};

ws_status fail(ws_status s, const std::string& msg) {
  g_last_error = msg;
  return s;
}

}  // namespace

namespace ws_detail {
ws_status set_error(ws_status s, const std::string& m) { return fail(s, m); }
void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }
}  // namespace ws_detail

namespace {

#define WS_CUDA_CHECK(expr)                                                                       \
  do {                                                                                            \
    cudaError_t e_ = (expr);                                                                      \
    if (e_ != cudaSuccess)                                                                        \
      return fail(WS_CUDA_ERROR, std::string(#expr " failed: ") + cudaGetErrorString(e_));        \
  } while (0)

PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  return fn;
}

int elem_bytes(int dt) {
  switch (dt) {
    case WS_F32: return 4;
    case WS_F16: return 2;
    case WS_BF16: return 2;
    case WS_E4M3: return 1;
  }
  return 0;
}

CUtensorMapDataType tma_dtype(int dt) {
  switch (dt) {
    case WS_F32: return CU_TENSOR_MAP_DATA_TYPE_FLOAT32;
    case WS_F16: return CU_TENSOR_MAP_DATA_TYPE_FLOAT16;
    case WS_BF16: return CU_TENSOR_MAP_DATA_TYPE_BFLOAT16;
    default: return CU_TENSOR_MAP_DATA_TYPE_UINT8;
  }
}

// 2-D row-major tensor [rows x cols] with row stride `ld` elements; box [box_rows x box_cols];
// 128-byte swizzle (box_cols * elem == 128).
ws_status make_tmap_uncached(CUtensorMap* m, const void* ptr, int dt, int64_t rows, int64_t cols, int64_t ld,
                             uint32_t box_rows, uint32_t box_cols, CUtensorMapL2promotion promo);

// Tensor maps only encode address, shape, strides and box, so a map built for the same operand
// is reused (per host thread, 32 entries, round robin): repeated calls on the same buffers skip
// the driver encode (small GEMMs are host-bound; scripts/host_overhead.py)
ws_status make_tmap(CUtensorMap* m, const void* ptr, int dt, int64_t rows, int64_t cols, int64_t ld,
                    uint32_t box_rows, uint32_t box_cols, CUtensorMapL2promotion promo) {
  struct Entry {
    const void* ptr;
    int dt;
    int64_t rows, cols, ld;
    uint32_t br, bc;
    int promo;
    CUtensorMap map;
  };
  thread_local Entry cache[32];
  thread_local int n = 0, next = 0;
  for (int i = 0; i < n; ++i) {
    const Entry& e = cache[i];
    if (e.ptr == ptr && e.dt == dt && e.rows == rows && e.cols == cols && e.ld == ld && e.br == box_rows &&
        e.bc == box_cols && e.promo == static_cast<int>(promo)) {
      *m = e.map;
      return WS_OK;
    }
  }
  const ws_status s = make_tmap_uncached(m, ptr, dt, rows, cols, ld, box_rows, box_cols, promo);
  if (s != WS_OK) return s;
  Entry& e = cache[next];
  e = Entry{ptr, dt, rows, cols, ld, box_rows, box_cols, static_cast<int>(promo), *m};
  next = (next + 1) % 32;
  if (n < 32) ++n;
  return WS_OK;
}

ws_status make_tmap_uncached(CUtensorMap* m, const void* ptr, int dt, int64_t rows, int64_t cols, int64_t ld,
                             uint32_t box_rows, uint32_t box_cols, CUtensorMapL2promotion promo) {
  auto enc = get_encode();
  if (!enc) return fail(WS_CUDA_ERROR, "cuTensorMapEncodeTiled unavailable (driver too old?)");
  const int eb = elem_bytes(dt);
  cuuint64_t dims[2] = {static_cast<cuuint64_t>(cols), static_cast<cuuint64_t>(rows)};
  cuuint64_t strides[1] = {static_cast<cuuint64_t>(ld * eb)};
  cuuint32_t box[2] = {box_cols, box_rows};
  cuuint32_t estr[2] = {1, 1};
  if ((reinterpret_cast<uintptr_t>(ptr) & 15) != 0 || (ld * eb) % 16 != 0)
    return fail(WS_TYPE, "operand base / row stride must be 16-byte aligned for TMA");
  CUresult r = enc(m, tma_dtype(dt), 2, const_cast<void*>(ptr), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, promo, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(WS_CUDA_ERROR, "cuTensorMapEncodeTiled failed: " + std::to_string((int)r));
  return WS_OK;
}

// Per-device state. Everything a launch needs from the device context — SM count, the dynamic
// shared-memory opt-in of each kernel, the wait-hint / watchdog symbols — is set per device
// ordinal (one process may drive several GPUs; the launch's current device is the stream's).
constexpr int MAX_DEVICES = 64;

int current_device() {
  int dev = 0;
  cudaGetDevice(&dev);
  return dev < 0 || dev >= MAX_DEVICES ? 0 : dev;
}

int num_sms() {
  static std::atomic<int> n[MAX_DEVICES];
  const int dev = current_device();
  int v = n[dev].load(std::memory_order_relaxed);
  if (v == 0) {
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    n[dev].store(v, std::memory_order_relaxed);
  }
  return v;
}

constexpr int SMEM_LIMIT = 232448;  // 227 KB opt-in per CTA on sm_100a

// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) once per (device, kernel) and size (it costs a
// driver call per launch otherwise; small GEMMs are launch-bound). Lock-free: a per-thread table
// (a thread that has not seen the pair yet repeats the idempotent attribute call once).
cudaError_t allow_smem(const void* kern, int bytes) {
  struct Entry {
    const void* kern;
    int dev, bytes;
  };
  thread_local Entry done[64];
  thread_local int n = 0;
  const int dev = current_device();
  for (int i = 0; i < n; ++i)
    if (done[i].kern == kern && done[i].dev == dev && done[i].bytes >= bytes) return cudaSuccess;
  const cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e == cudaSuccess) {
    for (int i = 0; i < n; ++i)
      if (done[i].kern == kern && done[i].dev == dev) {
        done[i].bytes = bytes;
        return e;
      }
    done[n < 64 ? n++ : 63] = Entry{kern, dev, bytes};
  }
  return e;
}

// Suspend-time hint of blocked mbarrier waits in this module's kernels: a waiting warp sleeps in
// the barrier (woken when the phase completes) instead of re-issuing try_wait, which leaves the
// issue slots to the softmax warps sharing its SM sub-partition (hdim-64 causal attention +5-10%,
// GEMM unchanged; scripts/attn_ab.py). WS_WAIT_HINT_NS overrides (0 = hardware default). Set once
// per device context before its first launch.
ws::WatchdogRecord* g_watchdog_host = nullptr;  // pinned, mapped, portable: survives a trapped context

void apply_wait_hint() {
  static std::once_flag once[MAX_DEVICES];
  static std::once_flag host_once;
  const int dev = current_device();
  std::call_once(once[dev], [] {
    const char* e = getenv("WS_WAIT_HINT_NS");
    const uint32_t ns = e ? static_cast<uint32_t>(atoi(e)) : 200000u;
    cudaMemcpyToSymbol(ws::ws_wait_hint_ns, &ns, sizeof(ns));
    // the watchdog's host-mapped record (ws_watchdog): one portable allocation, its device
    // address written into each device's copy of the module symbol
    std::call_once(host_once, [] {
      void* h = nullptr;
      if (cudaHostAlloc(&h, sizeof(ws::WatchdogRecord), cudaHostAllocMapped | cudaHostAllocPortable) == cudaSuccess) {
        std::memset(h, 0, sizeof(ws::WatchdogRecord));
        g_watchdog_host = static_cast<ws::WatchdogRecord*>(h);
      }
    });
    void* d = nullptr;
    if (g_watchdog_host && cudaHostGetDevicePointer(&d, g_watchdog_host, 0) == cudaSuccess)
      cudaMemcpyToSymbol(ws::ws_watchdog_host, &d, sizeof(d));
  });
}

// developer knobs, read once per process
int env_int(const char* name, int dflt) {
  const char* e = getenv(name);
  return e ? atoi(e) : dflt;
}
const int g_debug_deadlock = env_int("WS_DEBUG_DEADLOCK", 0);
const bool g_trace_global = getenv("WS_GEMM_TRACE_GLOBAL") != nullptr;
// programmatic dependent launch of every kernel (WS_PDL=0 turns it off): a kernel's setup (barrier
// init, TMEM alloc, descriptor prefetch) overlaps the previous grid's tail; measured +2-4% at short K
// (scripts/pdl_ab.py), where it also puts the GEMM ahead of cuBLAS (which launches the same way)
const int g_pdl = env_int("WS_PDL", 1);


unsigned long long* g_gemm_trace = nullptr;  // ws_debug_gemm_trace
unsigned long long* g_gemm_clk = nullptr;    // ws_debug_gemm_clock

}  // namespace

// A prepared GEMM launch (ws_gemm_plan_create): kernel, tensor maps, parameters and grid, so a
// repeated call is one cudaLaunchKernelEx (small GEMMs are host-bound).
struct ws_gemm_plan {
  CUtensorMap ta, tb, tc;
  ws::GemmParams p;
  const void* kern = nullptr;
  int grid = 0, smem = 0, cg = 1, dev = 0;
};

namespace {

template <int IN, int OUT, int BN, int CG>
ws_status prepare_gemm(const ws_gemm_desc& d, ws_gemm_plan& pl) {
  using namespace ws;
  const int in_dt = d.in_dtype, out_dt = d.out_dtype;
  const int kbox = 128 / elem_bytes(in_dt);

  GemmParams& p = pl.p;
  p.M = (int)d.M;
  p.N = (int)d.N;
  p.K = (int)d.K;
  p.num_m_blocks = (int)(d.M / GEMM_BM);
  const int64_t nbat = d.batch > 1 ? d.batch : 1;
  p.batch = (int)nbat;
  p.num_n_blocks = (int)(d.N / BN);
  p.num_k_blocks = (int)(d.K / kbox);
  const GemmSmemLayout L1 = gemm_smem_layout(BN / CG, 1);
  int max_stages = (SMEM_LIMIT - (int)(L1.total - L1.stage_bytes)) / (int)L1.stage_bytes;
  if (max_stages > GEMM_MAX_STAGES) max_stages = GEMM_MAX_STAGES;
  p.stages = d.D > 0 ? d.D : max_stages;
  p.mma_depth = d.P > 0 ? d.P : p.stages;
  if (p.mma_depth > p.stages)
    return fail(WS_PIPELINE_INFEASIBLE, "MMA pipelining depth P=" + std::to_string(p.mma_depth) +
                                            " exceeds aref depth D=" + std::to_string(p.stages));
  const GemmSmemLayout L = gemm_smem_layout(BN / CG, p.stages);
  if (p.stages > GEMM_MAX_STAGES || (int)L.total > SMEM_LIMIT)
    return fail(WS_SMEM_OVERFLOW, "D=" + std::to_string(p.stages) + " stages need " + std::to_string(L.total) +
                                      " B of shared memory; limit " + std::to_string(SMEM_LIMIT));
  // raster groups are counted in scheduling M-blocks (256 rows for a CTA pair)
  // auto raster (measured on B200, scripts/gemm_ab.py): 256 x 512 pair tiles in groups of 16
  // M-blocks, 256 x 256 pair tiles in groups of 2, single-CTA tiles in groups of 4
  p.group_m = d.group_m > 0 ? d.group_m : (BN == 512 ? 16 : CG == 2 ? 2 : 4);
  if (p.group_m > p.num_m_blocks / CG) p.group_m = p.num_m_blocks / CG;
  p.scale = d.scale_a * d.scale_b;
  p.act = d.act;
  p.trace = g_gemm_trace;
  p.clk = g_gemm_clk;
  // developer diagnostics: WS_DEBUG_DEADLOCK=1 makes CTA 0's producer skip its first aref put, so
  // the MMA warp waits forever and the watchdog fires (the simulator's Deadlock verdict on hardware)
  p.debug_deadlock = g_debug_deadlock;
  p.trace_global = g_trace_global;

  CUtensorMap &ta = pl.ta, &tb = pl.tb, &tc = pl.tc;
  ws_status s;
  if ((s = make_tmap(&ta, d.A, in_dt, nbat * d.M, d.K, d.lda, GEMM_BM, kbox, CU_TENSOR_MAP_L2_PROMOTION_L2_256B)) !=
      WS_OK)
    return s;
  if ((s = make_tmap(&tb, d.B, in_dt, nbat * d.N, d.K, d.ldb, (BN > 256 ? 256 : BN) / CG, kbox,
                     CU_TENSOR_MAP_L2_PROMOTION_L2_256B)) != WS_OK)
    return s;
  const int cw = 128 / elem_bytes(out_dt);
  if ((s = make_tmap(&tc, d.C, out_dt, nbat * d.M, d.N, d.ldc, 32, cw, CU_TENSOR_MAP_L2_PROMOTION_NONE)) != WS_OK)
    return s;

  auto kern = ws_gemm_tn_kernel<IN, OUT, BN, CG>;
  WS_CUDA_CHECK(allow_smem(reinterpret_cast<const void*>(kern), (int)L.total));
  const int tiles = (p.num_m_blocks / CG) * p.num_n_blocks * p.batch;
  const int units = num_sms() / CG;  // persistent: one CTA (pair) per SM (pair)
  pl.grid = CG * (d.persistent ? (tiles < units ? tiles : units) : tiles);
  pl.kern = reinterpret_cast<const void*>(kern);
  pl.smem = (int)L.total;
  pl.cg = CG;
  pl.dev = current_device();
  return WS_OK;
}

ws_status launch_plan(ws_gemm_plan& pl, cudaStream_t stream) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(pl.grid);
  cfg.blockDim = dim3(ws::GEMM_THREADS);
  cfg.dynamicSmemBytes = pl.smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[2];
  cfg.attrs = attr;
  if (pl.cg == 2) {
    attr[cfg.numAttrs].id = cudaLaunchAttributeClusterDimension;
    attr[cfg.numAttrs].val.clusterDim.x = 2;
    attr[cfg.numAttrs].val.clusterDim.y = 1;
    attr[cfg.numAttrs].val.clusterDim.z = 1;
    ++cfg.numAttrs;
  }
  if (g_pdl) {  // programmatic dependent launch: this grid's setup overlaps the previous one's tail
    attr[cfg.numAttrs].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[cfg.numAttrs].val.programmaticStreamSerializationAllowed = 1;
    ++cfg.numAttrs;
  }
  pl.p.trace = g_gemm_trace;
  pl.p.clk = g_gemm_clk;
  apply_wait_hint();
  void* args[] = {&pl.ta, &pl.tb, &pl.tc, &pl.p};
  WS_CUDA_CHECK(cudaLaunchKernelExC(&cfg, pl.kern, args));
  g_launches.fetch_add(1, std::memory_order_relaxed);
  return WS_OK;
}

template <int IN, int BN>
ws_status dispatch_out(const ws_gemm_desc& d, ws_gemm_plan& st) {
  if constexpr (BN == 512) {
    // 256 x 512 pair tiles exist only as cta_group::2 (checked by the caller)
    switch (d.out_dtype) {
      case WS_F32: return prepare_gemm<IN, ws::OUT_F32, BN, 2>(d, st);
      case WS_BF16: return prepare_gemm<IN, ws::OUT_BF16, BN, 2>(d, st);
      case WS_F16: return prepare_gemm<IN, ws::OUT_F16, BN, 2>(d, st);
    }
    return fail(WS_TYPE, "out_dtype must be F32, BF16 or F16");
  }
  if (d.cta_pair) {
    switch (d.out_dtype) {
      case WS_F32: return prepare_gemm<IN, ws::OUT_F32, BN, 2>(d, st);
      case WS_BF16: return prepare_gemm<IN, ws::OUT_BF16, BN, 2>(d, st);
      case WS_F16: return prepare_gemm<IN, ws::OUT_F16, BN, 2>(d, st);
    }
  } else {
    switch (d.out_dtype) {
      case WS_F32: return prepare_gemm<IN, ws::OUT_F32, BN, 1>(d, st);
      case WS_BF16: return prepare_gemm<IN, ws::OUT_BF16, BN, 1>(d, st);
      case WS_F16: return prepare_gemm<IN, ws::OUT_F16, BN, 1>(d, st);
    }
  }
  return fail(WS_TYPE, "out_dtype must be F32, BF16 or F16");
}

template <int BN>
ws_status dispatch_in(const ws_gemm_desc& d, ws_gemm_plan& st) {
  switch (d.in_dtype) {
    case WS_F16: return dispatch_out<ws::IN_F16, BN>(d, st);
    case WS_BF16: return dispatch_out<ws::IN_BF16, BN>(d, st);
    case WS_E4M3: return dispatch_out<ws::IN_E4M3, BN>(d, st);
  }
  return fail(WS_TYPE, "in_dtype must be F16, BF16 or E4M3");
}


template <int DH, bool BF16>
ws_status launch_attn(const ws_attn_desc& d, int bh0, int bh1, cudaStream_t stream, unsigned long long* trace) {
  using namespace ws;
  const int dt = d.dtype;
  const int64_t rows = (int64_t)d.B * d.H * d.S;
  AttnParams p;
  p.S = d.S;
  p.Dh = DH;
  p.BH_begin = bh0;
  if (d.S % (2 * ATTN_BM))
    return fail(WS_INDIVISIBLE_TILE, "the 64-key kernel needs S % 256 == 0 (S=" + std::to_string(d.S) + ")");
  p.num_pairs = d.S / (2 * ATTN_BM);
  p.causal = d.causal;
  const float sm = d.softmax_scale > 0.f ? d.softmax_scale : 1.0f / std::sqrt((float)DH);
  p.scale_log2 = sm * 1.4426950408889634f;
  p.lse = d.LSE;
  p.mx = d.MX;
  p.o = d.O;
  p.o_elem = BF16 ? 0 : 1;
  p.trace = trace;
  int max_stages = (SMEM_LIMIT - (int)attn_smem_bytes(DH, 0)) / (int)attn_kv_bytes(DH);
  if (max_stages > ATTN_MAX_KV_STAGES) max_stages = ATTN_MAX_KV_STAGES;
  p.kv_stages = d.D > 0 ? d.D : max_stages;
  if (p.kv_stages < 2)
    return fail(WS_PIPELINE_INFEASIBLE, "the K/V aref needs D >= 2 (ref pipeline.hpp:309-315)");
  const uint32_t smem = attn_smem_bytes(DH, p.kv_stages);
  if (p.kv_stages > ATTN_MAX_KV_STAGES || (int)smem > SMEM_LIMIT)
    return fail(WS_SMEM_OVERFLOW, "D=" + std::to_string(p.kv_stages) + " K/V stages need " + std::to_string(smem) +
                                      " B of shared memory; limit " + std::to_string(SMEM_LIMIT));
  CUtensorMap tq, tk, tv;
  ws_status s;
  if ((s = make_tmap(&tq, d.Q, dt, rows, DH, DH, ATTN_BM, 64, CU_TENSOR_MAP_L2_PROMOTION_L2_256B)) != WS_OK) return s;
  if ((s = make_tmap(&tk, d.K, dt, rows, DH, DH, ATTN_BN, 64, CU_TENSOR_MAP_L2_PROMOTION_L2_256B)) != WS_OK) return s;
  if ((s = make_tmap(&tv, d.V, dt, rows, DH, DH, ATTN_BN, 64, CU_TENSOR_MAP_L2_PROMOTION_L2_256B)) != WS_OK) return s;
  auto kern = ws_attn_fwd_kernel<DH, BF16>;
  WS_CUDA_CHECK(allow_smem(reinterpret_cast<const void*>(kern), (int)smem));
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(bh1 - bh0, p.num_pairs);
  cfg.blockDim = dim3(ATTN_THREADS);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  apply_wait_hint();
  cudaLaunchAttribute pdl_attr[1];
  if (g_pdl) {
    pdl_attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    pdl_attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = pdl_attr;
    cfg.numAttrs = 1;
  }
  WS_CUDA_CHECK(cudaLaunchKernelEx(&cfg, kern, tq, tk, tv, p));
  g_launches.fetch_add(1, std::memory_order_relaxed);
  return WS_OK;
}

template <int DH, bool BF16, bool PSMEM>
ws_status launch_attn128(const ws_attn_desc& d, int bh0, int bh1, cudaStream_t stream, unsigned long long* trace) {
  using namespace ws;
  if (!PSMEM && d.S % (2 * A128_BM))
    return fail(WS_INDIVISIBLE_TILE, "the P-in-TMEM kernel needs S % 256 == 0 (S=" + std::to_string(d.S) + ")");
  const int dt = d.dtype;
  const int64_t rows = (int64_t)d.B * d.H * d.S;
  Attn128Params p;
  p.S = d.S;
  p.BH_begin = bh0;
  p.num_pairs = (d.S + 2 * A128_BM - 1) / (2 * A128_BM);  // S % 256 == 128: last pair half valid
  p.num_bh = bh1 - bh0;
  static const int stagger_env = [] {  // WS_ATTN_STAGGER (developer knob)
    const char* e = getenv("WS_ATTN_STAGGER");
    return e ? atoi(e) : -1;
  }();
  // staggered tile issue: +3-4 % at hdim 128 and, since the barrier addresses are pinned (leaner
  // softmax), +2 % at hdim 64 as well (8-round medians; profiles/r02b_attn_experiments.md)
  p.stagger = stagger_env >= 0 ? stagger_env : 1;
  p.causal = d.causal;
  // causal: (b,h) fastest so every head's heaviest query pairs run first (longest-first);
  // non-causal: the query pairs of one (b,h) run together and share its K/V in L2
  p.bh_fast = d.causal ? 1 : 0;
  const float sm = d.softmax_scale > 0.f ? d.softmax_scale : 1.0f / std::sqrt((float)DH);
  p.scale_log2 = sm * 1.4426950408889634f;
  p.o_scale = 1.f;
  p.lse = d.LSE;
  p.mx = d.MX;
  p.o = d.O;
  p.trace = trace;
  auto smem_bytes = [](int stages) { return PSMEM ? aps_smem_bytes(DH, stages) : a128_smem_bytes(DH, stages); };
  int max_stages = (SMEM_LIMIT - (int)smem_bytes(0)) / (int)a128_kv_bytes(DH);
  if (max_stages > A128_MAX_STAGES) max_stages = A128_MAX_STAGES;
  p.kv_stages = d.D > 0 ? d.D : max_stages;
  if (p.kv_stages < 2)
    return fail(WS_PIPELINE_INFEASIBLE, "the K/V aref needs D >= 2 (ref pipeline.hpp:309-315)");
  const uint32_t smem = smem_bytes(p.kv_stages);
  if (p.kv_stages > A128_MAX_STAGES || (int)smem > SMEM_LIMIT)
    return fail(WS_SMEM_OVERFLOW, "D=" + std::to_string(p.kv_stages) + " K/V stages need " + std::to_string(smem) +
                                      " B of shared memory; limit " + std::to_string(SMEM_LIMIT));
  CUtensorMap tq, tk, tv;
  ws_status s;
  if ((s = make_tmap(&tq, d.Q, dt, rows, DH, DH, A128_BM, 64, CU_TENSOR_MAP_L2_PROMOTION_L2_256B)) != WS_OK) return s;
  if ((s = make_tmap(&tk, d.K, dt, rows, DH, DH, A128_BN, 64, CU_TENSOR_MAP_L2_PROMOTION_L2_256B)) != WS_OK) return s;
  if ((s = make_tmap(&tv, d.V, dt, rows, DH, DH, A128_BN, 64, CU_TENSOR_MAP_L2_PROMOTION_L2_256B)) != WS_OK) return s;
  // WS_ATTN_POLY (developer knob for the exp-mix sweep, bf16 only): column pairs of every 8 whose
  // exponential runs on the FMA pipe instead of MUFU
  static const int poly_env = [] {
    const char* e = getenv("WS_ATTN_POLY");
    return e ? atoi(e) : -1;
  }();
  // O [B*H*S, DH] in the input's 16-bit type, stored through TMA in 128 x 64 boxes
  CUtensorMap to;
  if ((s = make_tmap(&to, d.O, dt, rows, DH, DH, A128_BM, 64, CU_TENSOR_MAP_L2_PROMOTION_NONE)) != WS_OK) return s;
  auto kern = trace ? ws_attn128_kernel<DH, BF16, A128_POLY, true> : ws_attn128_kernel<DH, BF16, A128_POLY>;
  // exp mix of the P-in-smem kernel: 1/8 of the pairs on the FMA pipe at hdim 128, 2/8 at hdim 64
  // (where the softmax alone bounds the kernel; scripts/attn_ab.py)
  constexpr int PS_POLY = DH == 64 ? 2 : APS_POLY;
  if (PSMEM)
    kern = trace ? ws_attn_psmem_kernel<DH, BF16, PS_POLY, true> : ws_attn_psmem_kernel<DH, BF16, PS_POLY>;
  if (BF16 && !trace) {
    switch (poly_env) {
      case 1: kern = PSMEM ? ws_attn_psmem_kernel<DH, BF16, 1> : ws_attn128_kernel<DH, BF16, 1>; break;
      case 2: kern = PSMEM ? ws_attn_psmem_kernel<DH, BF16, 2> : ws_attn128_kernel<DH, BF16, 2>; break;
      case 3: kern = PSMEM ? ws_attn_psmem_kernel<DH, BF16, 3> : ws_attn128_kernel<DH, BF16, 3>; break;
      default: break;
    }
  }
  WS_CUDA_CHECK(allow_smem(reinterpret_cast<const void*>(kern), (int)smem));
  cudaLaunchConfig_t cfg = {};
  {
    // persistent: one CTA per SM over the (pair, (b,h)) items (both 128-key kernels);
    // WS_ATTN_PERSIST=0 (developer knob) launches one CTA per item instead
    static const int persist_env = [] {
      const char* e = getenv("WS_ATTN_PERSIST");
      return e ? atoi(e) : 1;
    }();
    const int items = p.num_pairs * p.num_bh;
    const bool per_item = d.grid_per_item == 1 || (d.grid_per_item == 0 && persist_env == 0);
    cfg.gridDim = dim3(per_item || items < num_sms() ? items : num_sms());
  }
  cfg.blockDim = dim3(A128_THREADS);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  apply_wait_hint();
  cudaLaunchAttribute pdl_attr[1];
  if (g_pdl) {
    pdl_attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    pdl_attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = pdl_attr;
    cfg.numAttrs = 1;
  }
  WS_CUDA_CHECK(cudaLaunchKernelEx(&cfg, kern, tq, tk, tv, to, p));
  g_launches.fetch_add(1, std::memory_order_relaxed);
  return WS_OK;
}

// FP8 e4m3 attention (hdim 128): the P-in-shared-memory kernel with kind::f8f6f4 MMAs, P
// quantized to e4m3, per-tensor descales (q, k into the softmax scale, v into the epilogue), bf16 O.
ws_status launch_attn_fp8(const ws_attn_desc& d, int bh0, int bh1, cudaStream_t stream, unsigned long long* trace) {
  using namespace ws;
  constexpr int DH = 128;
  const int64_t rows = (int64_t)d.B * d.H * d.S;
  Attn128Params p;
  p.S = d.S;
  p.BH_begin = bh0;
  p.num_pairs = (d.S + 2 * A128_BM - 1) / (2 * A128_BM);  // S % 256 == 128: last pair half valid
  p.num_bh = bh1 - bh0;
  p.stagger = 1;
  p.causal = d.causal;
  p.bh_fast = d.causal ? 1 : 0;
  const float sq = d.scale_q > 0.f ? d.scale_q : 1.f, sk = d.scale_k > 0.f ? d.scale_k : 1.f;
  const float sv = d.scale_v > 0.f ? d.scale_v : 1.f;
  const float sm = d.softmax_scale > 0.f ? d.softmax_scale : 1.0f / std::sqrt((float)DH);
  p.scale_log2 = sm * sq * sk * 1.4426950408889634f;
  p.o_scale = sv;
  p.lse = d.LSE;
  p.mx = d.MX;
  p.o = d.O;
  p.trace = trace;
  const uint32_t kvb = A128_BN * DH;  // one e4m3 K block
  // Q0 | Q1 (e4m3) | P0 | P1 (f16) | K ring | two f16 V buffers (e4m3 V lands in their upper
  // halves) | barriers (+1 KB alignment slack)
  const uint32_t base = 2 * A128_BM * DH + 2 * A128_BM * A128_BN * 2 + 2 * A128_BN * DH * 2 + APS_BAR_BYTES + 1024;
  int max_stages = (SMEM_LIMIT - (int)base) / (int)kvb;
  if (max_stages > A128_MAX_STAGES) max_stages = A128_MAX_STAGES;
  p.kv_stages = d.D > 0 ? d.D : max_stages;
  if (p.kv_stages < 2)
    return fail(WS_PIPELINE_INFEASIBLE, "the K/V aref needs D >= 2 (ref pipeline.hpp:309-315)");
  const uint32_t smem = base + p.kv_stages * kvb;
  if (p.kv_stages > A128_MAX_STAGES || (int)smem > SMEM_LIMIT)
    return fail(WS_SMEM_OVERFLOW, "D=" + std::to_string(p.kv_stages) + " K/V stages need " + std::to_string(smem) +
                                      " B of shared memory; limit " + std::to_string(SMEM_LIMIT));
  CUtensorMap tq, tk, tv;
  ws_status s;
  if ((s = make_tmap(&tq, d.Q, WS_E4M3, rows, DH, DH, A128_BM, 128, CU_TENSOR_MAP_L2_PROMOTION_L2_256B)) != WS_OK)
    return s;
  if ((s = make_tmap(&tk, d.K, WS_E4M3, rows, DH, DH, A128_BN, 128, CU_TENSOR_MAP_L2_PROMOTION_L2_256B)) != WS_OK)
    return s;
  if ((s = make_tmap(&tv, d.V, WS_E4M3, rows, DH, DH, A128_BN, 128, CU_TENSOR_MAP_L2_PROMOTION_L2_256B)) != WS_OK)
    return s;
  CUtensorMap to;  // O in bf16
  if ((s = make_tmap(&to, d.O, WS_BF16, rows, DH, DH, A128_BM, 64, CU_TENSOR_MAP_L2_PROMOTION_NONE)) != WS_OK)
    return s;
  // exp mix 2 of every 8 pairs on the FMA pipe: with the tensor work halved the softmax alone bounds
  // FP8 (POLY 0/1/2/3/4 = 1586/1614/1645/1539/1483 TFLOP/s at S=16K, scripts/attn_ab.py AB_FP8=1)
  constexpr int F8_POLY = 2;
  auto kern = trace ? ws_attn_psmem_kernel<DH, true, F8_POLY, true, true> : ws_attn_psmem_kernel<DH, true, F8_POLY, false, true>;
  static const int poly_env = [] {
    const char* e = getenv("WS_ATTN_POLY");
    return e ? atoi(e) : -1;
  }();
  if (!trace) {
    switch (poly_env) {
      case 0: kern = ws_attn_psmem_kernel<DH, true, 0, false, true>; break;
      case 1: kern = ws_attn_psmem_kernel<DH, true, 1, false, true>; break;
      case 3: kern = ws_attn_psmem_kernel<DH, true, 3, false, true>; break;
      case 4: kern = ws_attn_psmem_kernel<DH, true, 4, false, true>; break;
      default: break;
    }
  }
  WS_CUDA_CHECK(allow_smem(reinterpret_cast<const void*>(kern), (int)smem));
  cudaLaunchConfig_t cfg = {};
  const int items = p.num_pairs * p.num_bh;
  // grid: persistent (one CTA per SM over the items) by default, or one CTA per item. At S = 16K
  // the two are equal in interleaved A/B runs (1566 vs 1562 TFLOP/s; the 5% of the ordered D x P
  // sweep did not reproduce), at S = 1K persistent wins (1210 vs 1060, cross-item overlap)
  const bool per_item = d.grid_per_item == 1;
  cfg.gridDim = dim3(per_item || items < num_sms() ? items : num_sms());
  cfg.blockDim = dim3(A128_THREADS);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  apply_wait_hint();
  cudaLaunchAttribute pdl_attr[1];
  if (g_pdl) {
    pdl_attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    pdl_attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = pdl_attr;
    cfg.numAttrs = 1;
  }
  WS_CUDA_CHECK(cudaLaunchKernelEx(&cfg, kern, tq, tk, tv, to, p));
  g_launches.fetch_add(1, std::memory_order_relaxed);
  return WS_OK;
}

ws_status attn_entry(const ws_attn_desc& d, cudaStream_t st, unsigned long long* trace) {
  if (d.dtype != WS_BF16 && d.dtype != WS_F16 && d.dtype != WS_E4M3)
    return fail(WS_TYPE, "attention dtype must be BF16, F16 or E4M3");
  if (d.B <= 0 || d.H <= 0 || d.S <= 0) return fail(WS_TYPE, "B, H, S must be positive");
  if (d.Dh != 64 && d.Dh != 128) return fail(WS_UNSUPPORTED_KERNEL, "head dim must be 64 or 128");
  if (d.S % 128) return fail(WS_INDIVISIBLE_TILE, "S=" + std::to_string(d.S) + " is not a multiple of 128");
  if (!d.Q || !d.K || !d.V || !d.O) return fail(WS_TYPE, "null operand pointer");
  if (d.D == 1) return fail(WS_PIPELINE_INFEASIBLE, "the K/V aref needs D >= 2 (ref pipeline.hpp:309-315)");
  if (d.D < 0) return fail(WS_PIPELINE_INFEASIBLE, "D must be >= 2 (0 = auto)");
  const int BH = d.B * d.H;
  const int bh0 = d.bh_begin, bh1 = d.bh_end > 0 ? d.bh_end : BH;
  if (bh0 < 0 || bh1 > BH || bh0 >= bh1) return fail(WS_TYPE, "bad (b,h) shard range");
  if ((int64_t)BH * d.S >= (int64_t)1 << 31) return fail(WS_TYPE, "B*H*S must fit in int32");
  if (d.kv_block != 0 && d.kv_block != 64 && d.kv_block != 128)
    return fail(WS_TYPE, "kv_block must be 0 (auto), 64 or 128");
  if (d.dtype == WS_E4M3) {
    if (d.Dh != 128) return fail(WS_UNSUPPORTED_KERNEL, "FP8 attention supports head dim 128");
    if (d.kv_block == 64) return fail(WS_UNSUPPORTED_KERNEL, "FP8 attention uses 128-key K/V blocks");
    return launch_attn_fp8(d, bh0, bh1, st, trace);
  }
  if (d.kv_block != 64) {
    // P staging: P in shared memory (S released right after the softmax copies it, QK_{j+1}
    // overlaps the softmax, persistent with TMA epilogue) for both head dims; P in TMEM
    // (attn128_sm100.cuh) measured 3-7% slower at hdim 64 and 2-5% at hdim 128 once the former
    // had its item-boundary fixes. WS_ATTN_PTMEM=1 selects it (developer knob).
    static const int ptmem_env = [] {
      const char* e = getenv("WS_ATTN_PTMEM");
      return e ? atoi(e) : -1;
    }();
    const bool ptmem = ptmem_env == 1;
    if (ptmem) {
      if (d.Dh == 128)
        return d.dtype == WS_BF16 ? launch_attn128<128, true, false>(d, bh0, bh1, st, trace)
                                  : launch_attn128<128, false, false>(d, bh0, bh1, st, trace);
      return d.dtype == WS_BF16 ? launch_attn128<64, true, false>(d, bh0, bh1, st, trace)
                                : launch_attn128<64, false, false>(d, bh0, bh1, st, trace);
    }
    if (d.Dh == 128)
      return d.dtype == WS_BF16 ? launch_attn128<128, true, true>(d, bh0, bh1, st, trace)
                                : launch_attn128<128, false, true>(d, bh0, bh1, st, trace);
    return d.dtype == WS_BF16 ? launch_attn128<64, true, true>(d, bh0, bh1, st, trace)
                              : launch_attn128<64, false, true>(d, bh0, bh1, st, trace);
  }
  if (d.Dh == 128)
    return d.dtype == WS_BF16 ? launch_attn<128, true>(d, bh0, bh1, st, trace)
                              : launch_attn<128, false>(d, bh0, bh1, st, trace);
  return d.dtype == WS_BF16 ? launch_attn<64, true>(d, bh0, bh1, st, trace)
                            : launch_attn<64, false>(d, bh0, bh1, st, trace);
}

}  // namespace

extern "C" {

const char* ws_last_error(void) { return g_last_error.c_str(); }
int64_t ws_launch_count(void) { return g_launches.load(); }
const char* ws_version(void) { return "ws-b200 0.1 sm_100a"; }

void ws_debug_gemm_trace(unsigned long long* trace) { g_gemm_trace = trace; }
void ws_debug_gemm_clock(unsigned long long* clk) { g_gemm_clk = clk; }

int32_t ws_watchdog(ws_watchdog_info* out) {
  const volatile ws::WatchdogRecord* r = g_watchdog_host;
  if (out) std::memset(out, 0, sizeof(*out));
  if (r == nullptr || r->fired != 1u) return 0;
  if (out) {
    out->fired = 1;
    out->block_x = static_cast<uint32_t>(r->block & 0xffffffffu);
    out->block_y = static_cast<uint32_t>(r->block >> 32);
    out->thread = r->thread;
    out->barrier = r->bar_smem;
    out->parity = r->parity;
    out->tag = r->tag;
  }
  return 1;
}

}  // extern "C"

namespace {
ws_status build_plan(const ws_gemm_desc* desc, ws_gemm_plan& pl) {
  if (!desc) return fail(WS_TYPE, "null descriptor");
  const ws_gemm_desc& d = *desc;
  if (d.M <= 0 || d.N <= 0 || d.K <= 0) return fail(WS_TYPE, "M, N, K must be positive");
  if (!d.A || !d.B || !d.C) return fail(WS_TYPE, "null operand pointer");
  if (d.D < 0 || d.P < 0) return fail(WS_PIPELINE_INFEASIBLE, "D and P must be >= 1 (0 = auto)");
  if (d.act != 0 && d.act != 1) return fail(WS_TYPE, "act must be 0 (none) or 1 (relu)");
  if (d.D > 0 && d.P > d.D)
    return fail(WS_PIPELINE_INFEASIBLE,
                "MMA pipelining depth P=" + std::to_string(d.P) + " exceeds aref depth D=" + std::to_string(d.D));
  const int eb = elem_bytes(d.in_dtype);
  if (eb == 0 || d.in_dtype == WS_F32) return fail(WS_TYPE, "in_dtype must be F16, BF16 or E4M3");
  // auto N tile: a 256 x 512 pair tile moves 25% fewer operand bytes per output than 256 x 256
  // (256 x 256 pairs are L2 -> SM bandwidth bound, ~600 instead of 512 cycles per K block); its
  // single TMEM accumulator is handed over half by half with an early-release epilogue
  const int64_t kblocks = d.K / (128 / (eb > 0 ? eb : 1));
  // auto: 256 x 512 pair tiles from 4 K blocks on (4-7% over 256 x 256 pairs from 16 K blocks,
  // scripts/gemm_policy_sweep.sh; and, since the epilogue releases each accumulator half after one
  // batched TMEM load, 2-5% at 4-12 K blocks too: bf16 K = 256 / 512 / 768 and FP8
  // K = 512 / 1024 / 1536, profiles/r02n_ab_gemm_short_k_tiles.txt; FP8 K = 256, 2 K blocks, was
  // 5% slower), else 256-wide
  // ... and only when the grid still fills the GPU: small problems take the smaller tile with
  // more work units (1024^3: 128 x 128 single-CTA tiles, 64 CTAs)
  const int64_t units = num_sms();
  const int64_t nbat = d.batch > 1 ? d.batch : 1;
  // 256 x 512 vs 256 x 256 pairs by rounds of the persistent schedule: a K block takes ~1040 cycles
  // in a 256x512 tile and ~712 (TMA-bound) in a 256x256 one. One full round of 512-wide tiles
  // beats two of 256-wide ones.
  // (no device, e.g. validation-only calls on a CPU host: assume a B200's 74 SM pairs)
  const int64_t pairs = units >= 2 ? units / 2 : 74, t512 = nbat * (d.M / 256) * (d.N / 512), t256 = 2 * t512;
  const int64_t full512 = t512 / pairs, tail512 = t512 % pairs;
  const double cost512 = (double)(full512 + (tail512 ? 1 : 0)) * 1040.0;
  const double cost256 = (double)((t256 + pairs - 1) / pairs) * 712.0;
  const bool fill512 = cost512 <= cost256;
  const bool fill256 = nbat * (d.M / 128) * (d.N / 256) >= units;
  // (N a multiple of 128 but not of 256: 128-wide tiles, single CTA or pair)
  int bn = d.bn > 0 ? d.bn
           : (d.cta_pair && kblocks >= 4 && d.N % 512 == 0 && fill512)   ? 512
           : (!d.cta_pair && !fill256 && d.N % 128 == 0)                 ? 128
           : (d.N % 256 != 0 && d.N % 128 == 0)                          ? 128
                                                                         : 256;
  if (bn != 128 && bn != 256 && bn != 512) return fail(WS_TYPE, "bn must be 128, 256 or 512");
  if (bn == 512 && !d.cta_pair) return fail(WS_TYPE, "bn=512 (256 x 512 tiles) needs cta_pair=1");
  const int bm = d.cta_pair ? 2 * ws::GEMM_BM : ws::GEMM_BM;
  if (d.M % bm) return fail(WS_INDIVISIBLE_TILE, "M=" + std::to_string(d.M) + " is not a multiple of " + std::to_string(bm));
  if (d.N % bn) return fail(WS_INDIVISIBLE_TILE, "N=" + std::to_string(d.N) + " is not a multiple of bn=" + std::to_string(bn));
  if (d.K % (128 / eb))
    return fail(WS_INDIVISIBLE_TILE, "K=" + std::to_string(d.K) + " is not a multiple of " + std::to_string(128 / eb));
  if (d.lda < d.K || d.ldb < d.K || d.ldc < d.N) return fail(WS_TYPE, "leading dimension smaller than the row");
  if (d.batch < 0) return fail(WS_TYPE, "batch must be >= 0 (0 or 1 = one product)");
  if (nbat * d.M >= (int64_t)1 << 31 || nbat * d.N >= (int64_t)1 << 31)
    return fail(WS_TYPE, "batch*M and batch*N must fit in int32");
  return bn == 512 ? dispatch_in<512>(d, pl) : bn == 256 ? dispatch_in<256>(d, pl) : dispatch_in<128>(d, pl);
}
}  // namespace

extern "C" {

ws_status ws_gemm_tn(const ws_gemm_desc* desc, void* cuda_stream) {
  g_last_error.clear();
  ws_gemm_plan pl;
  const ws_status s = build_plan(desc, pl);
  if (s != WS_OK) return s;
  return launch_plan(pl, reinterpret_cast<cudaStream_t>(cuda_stream));
}

ws_status ws_gemm_plan_create(const ws_gemm_desc* desc, ws_gemm_plan** out) {
  g_last_error.clear();
  if (!out) return fail(WS_TYPE, "null plan pointer");
  *out = nullptr;
  auto* pl = new (std::nothrow) ws_gemm_plan();
  if (!pl) return fail(WS_CUDA_ERROR, "out of host memory");
  const ws_status s = build_plan(desc, *pl);
  if (s != WS_OK) {
    delete pl;
    return s;
  }
  *out = pl;
  return WS_OK;
}

ws_status ws_gemm_plan_launch(ws_gemm_plan* plan, void* cuda_stream) {
  if (!plan) return fail(WS_TYPE, "null plan");
  if (current_device() != plan->dev) return fail(WS_TYPE, "plan was created for another device");
  return launch_plan(*plan, reinterpret_cast<cudaStream_t>(cuda_stream));
}

void ws_gemm_plan_destroy(ws_gemm_plan* plan) { delete plan; }



ws_status ws_attn_fwd(const ws_attn_desc* desc, void* cuda_stream) {
  g_last_error.clear();
  if (!desc) return fail(WS_TYPE, "null descriptor");
  return attn_entry(*desc, reinterpret_cast<cudaStream_t>(cuda_stream), nullptr);
}

ws_status ws_attn_fwd_traced(const ws_attn_desc* desc, void* cuda_stream, unsigned long long* trace) {
  g_last_error.clear();
  if (!desc) return fail(WS_TYPE, "null descriptor");
  return attn_entry(*desc, reinterpret_cast<cudaStream_t>(cuda_stream), trace);
}

}  // extern "C"
