/*
 * ws.h — C-ABI of the B200 (sm_100a) warp-specialized GEMM and FlashAttention-forward path.
 *
 * This is the drop-in boundary for the reference's hot path. The reference (warpspec, a
 * header-only C++20 library) has no FFI: its operator API is the `.k` kernel text plus
 *   - parse_kernel(text) -> KernelGraph           (ref proj/include/warpspec/validate.hpp:349)
 *   - interpret_sequential(g, Buffers, pid)       (ref proj/include/warpspec/interp.hpp:157)
 *   - compile_kernel(g, MachineConfig, RunSpec)   (ref proj/include/warpspec/driver.hpp:116)
 *   - simulate / run_grid                         (ref proj/include/warpspec/sim.hpp:686,
 *                                                   ref proj/include/warpspec/grid.hpp:140)
 * The entry points below replace simulate/run_grid for the two kernel shapes the path covers
 * (SURVEY.md §8a rows a1..a16):
 *   ws_gemm_tn   <- gemm.k family, c = a . b^T  (ref proj/kernels/gemm.k:2-17,
 *                   gemm_large.k:3-18, gemm_batched.k:2-22, gemm_act.k:2-18)
 *   ws_attn_fwd  <- flash-attention .k of SURVEY.md Appendix A (T/C/U coarse pipeline,
 *                   ref proj/include/warpspec/pipeline.hpp:160-328)
 * Knobs mirror RunSpec (ref proj/include/warpspec/driver.hpp:42-57): D (aref depth),
 * P (MMA pipelining depth), persistent, cooperative (2-CTA pair).
 *
 * Conventions: plain pointers and sizes only. The caller owns every device buffer; the
 * library allocates nothing on the device except TMEM and shared memory inside the kernels.
 * Calls are asynchronous on the given stream and reentrant per stream. No exceptions cross
 * this boundary: every entry point returns a ws_status; ws_last_error() returns a
 * thread-local message for the last failing call on this thread.
 */
#ifndef WS_H_
#define WS_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Status codes. 1..12 mirror warpspec::ErrorCode in declaration order
 * (ref proj/include/warpspec/errors.hpp:10-23) so a host shim can rethrow
 * CompileError{code} unchanged. */
typedef enum ws_status {
  WS_OK = 0,
  WS_PARSE = 1,
  WS_TYPE = 2,                 /* bad dtype / argument shape */
  WS_UNSUPPORTED_KERNEL = 3,   /* kernel shape not covered by this path */
  WS_PIPELINE_INFEASIBLE = 4,  /* P > D, D < 1, P < 1 (ref pipeline.hpp:84-92) */
  WS_STAGE_PLAN_AMBIGUOUS = 5,
  WS_UNLOWERED_AREF = 6,
  WS_SMEM_OVERFLOW = 7,        /* stage bytes x D over the 227 KB sm_100a limit */
  WS_INDIVISIBLE_TILE = 8,     /* a dimension is not a multiple of the tile (ref grid.hpp:43-46) */
  WS_REGISTER_BUDGET = 9,
  WS_PROTOCOL_VIOLATION = 10,
  WS_IO = 11,
  WS_EVAL = 12,
  WS_CUDA_ERROR = 100          /* a CUDA runtime/driver call failed */
} ws_status;

/* Element types of the device operands. The reference payloads are `real` (double) or `int`;
 * on the GPU the storage type is a launch attribute. */
typedef enum ws_dtype {
  WS_F32 = 0,
  WS_F16 = 1,
  WS_BF16 = 2,
  WS_E4M3 = 3
} ws_dtype;

/* c[M x N] (row stride ldc elements) = scale_a*scale_b * a[M x K] . b[N x K]^T
 * a, b row-major with row strides lda, ldb (elements). fp32 accumulate in TMEM.
 * in_dtype in {F16, BF16, E4M3}; out_dtype in {F32, BF16, F16}.
 * Tiling: M % 128 == 0 (M % 256 with cta_pair), N % bn == 0, K % (128 / elem_bytes) == 0. */
typedef struct ws_gemm_desc {
  int32_t in_dtype;
  int32_t out_dtype;
  int64_t M, N, K;
  const void* A; int64_t lda;
  const void* B; int64_t ldb;
  void* C;       int64_t ldc;
  float scale_a, scale_b;      /* per-tensor dequant scales (FP8); 1.0 otherwise */
  int32_t D;                   /* aref depth: smem ring slots; 0 = auto (max that fits) */
  int32_t P;                   /* MMA k-blocks in flight; 0 = D (commit straight to empty) */
  int32_t persistent;          /* 1 = one CTA per SM looping over tiles; 0 = one CTA per tile */
  int32_t cta_pair;            /* 1 = cta_group::2 256-row tiles (cooperative WGs analogue) */
  int32_t bn;                  /* N tile: 0 = auto, else 128, 256 or 512 (512: cta_pair only, a
                                  256 x 512 pair tile with one TMEM accumulator) */
  int32_t group_m;             /* raster: tiles grouped by this many M-blocks; 0 = auto */
  int32_t act;                 /* epilogue activation: 0 none, 1 relu (gemm_act.k, ref
                                  proj/kernels/gemm_act.k:10-16) */
  int32_t batch;               /* independent products stacked along rows, one launch (gemm_batched.k,
                                  ref proj/kernels/gemm_batched.k:1-22): A [batch*M, K], B
                                  [batch*N, K], C [batch*M, N]; product i uses rows i*M / i*N.
                                  0 or 1 = a single product */
} ws_gemm_desc;

/* FlashAttention forward. q,k,v,o: [B, H, S, Dh] contiguous; lse: [B, H, S] fp32 (natural log,
 * lse = m + log(l)); may be NULL. Only bh in [bh_begin, bh_end) is computed (the multi-GPU
 * batch*heads shard); bh_end <= 0 means B*H. dtype in {BF16, F16, E4M3 (Dh 128; o is BF16;
 * P is quantized to e4m3 for the P.V product)}; Dh in {64, 128};
 * S % 128 == 0 (kv_block 64 and the P-in-TMEM developer kernel: S % 256 == 0).
 * softmax_scale <= 0 means 1/sqrt(Dh). */
typedef struct ws_attn_desc {
  int32_t dtype;
  int32_t B, H, S, Dh;
  int32_t causal;
  float softmax_scale;
  const void* Q; const void* K; const void* V;
  void* O;
  float* LSE;
  int32_t D;                   /* K/V aref depth; 0 = auto */
  int32_t bh_begin, bh_end;
  int32_t kv_block;            /* keys per K/V block: 0 = auto (128), 64 or 128. 128-key blocks
                                  keep the QK^T MMA inside the shared-memory operand rate; 64
                                  double-buffers S per Q tile instead (csrc/attn*_sm100.cuh) */
  float scale_q, scale_k, scale_v; /* E4M3 only: per-tensor descales (0 = 1): scores use
                                  scale_q*scale_k*q.k, O = scale_v * P.v / l */
  float* MX;                   /* optional [B, H, S] fp32: the exact row max m of the scaled scores
                                  (natural units), i.e. the flash .k's stored %m; with LSE it gives
                                  the .k's row sum l = exp(lse - m) and acc = O * l. NULL = skip */
  int32_t grid_per_item;       /* grid shape (RunSpec persistent): 1 = one CTA per work item,
                                  2 = persistent (one CTA per SM looping over the work items),
                                  0 = the measured default (persistent) */
} ws_attn_desc;

ws_status ws_gemm_tn(const ws_gemm_desc* desc, void* cuda_stream);
ws_status ws_attn_fwd(const ws_attn_desc* desc, void* cuda_stream);

/* Prepared GEMM launches for repeated calls on the same buffers (small GEMMs are host-bound):
 * create validates and encodes everything ws_gemm_tn would (same status codes), launch is a single
 * kernel launch on the given stream (capturable into a CUDA graph), destroy frees the host-side
 * plan. A plan belongs to the device that was current at create. */
typedef struct ws_gemm_plan ws_gemm_plan;
ws_status ws_gemm_plan_create(const ws_gemm_desc* desc, ws_gemm_plan** plan);
ws_status ws_gemm_plan_launch(ws_gemm_plan* plan, void* cuda_stream);
void ws_gemm_plan_destroy(ws_gemm_plan* plan);

/* ws_attn_fwd plus a device trace of CTA (0,0): `trace` is a device buffer of 3*256*8 uint64
 * %clock64 stamps — per KV step j, the MMA issuer (role 0) and the first softmax warp of each Q
 * tile (roles 1, 2) record when they start waiting, pass each mbarrier and finish each stage.
 * This is the hardware counterpart of the simulator's per-unit busy intervals
 * (ref proj/include/warpspec/sim.hpp:16-36, trace.hpp:59-83); layout in csrc/attn_sm100.cuh. */
ws_status ws_attn_fwd_traced(const ws_attn_desc* desc, void* cuda_stream, unsigned long long* trace);

/* `.k` front end: run pids [pid_lo, pid_hi) of a kernel written in the
 * reference grammar (ref SPEC.md:120-134) on the GPU, like the reference's tile-by-tile oracle
 * run `interpret_tiles` (ref proj/tests/support/fixtures.hpp:148-157). Buffers are the kernel's
 * parameters by name, as host arrays: double for `real`, int64 for `int`; in/out; parameters
 * without a buffer start zeroed. Supported shapes: the gemm.k family (gemm / gemm_large /
 * gemm_batched / gemm_act forms, optional 1x1 scale epilogue) — exact for the reference's payloads
 * with device dtype BF16 — the flash .k of SURVEY.md Appendix A (its three outputs as the .k
 * defines them: o = the un-normalised accumulator acc, lsum = the row sum l and mx = the running
 * max m, within the attention tolerances) and the integer max-shift attention.k
 * (ref proj/kernels/attention.k:1-21, exact in fp16). Anything else returns WS_UNSUPPORTED_KERNEL;
 * grammar errors WS_PARSE. Synchronous w.r.t. the host buffers. */
typedef struct ws_kbuffer {
  const char* name;
  int64_t rows, cols;
  int32_t is_real;
  void* data;
} ws_kbuffer;

ws_status ws_run_kernel(const char* ktext, ws_kbuffer* buffers, int32_t nbuffers, int64_t pid_lo, int64_t pid_hi,
                        int32_t dtype, void* cuda_stream);

/* RunSpec of the reference (ref proj/include/warpspec/driver.hpp:42-57) for a `.k` run on the GPU.
 * mode: pipeline mode as parse_pipeline_mode (driver.hpp:34-40). Rejections are the reference's,
 * evaluated on the .k graph before any device work:
 *   d < 1, p < 1                                   -> PIPELINE_INFEASIBLE (driver.hpp:117-118)
 *   fine on a loop body that is not a pure dot chain (gemm_act, flash) -> PIPELINE_INFEASIBLE
 *                                                     (ref pipeline.hpp:57-75)
 *   fine (or auto on a dot-only body) with p > d   -> PIPELINE_INFEASIBLE (ref pipeline.hpp:84-92)
 *   coarse on a body without a transform stage     -> PIPELINE_INFEASIBLE (ref pipeline.hpp:264-267)
 *   coarse with d < 2                              -> PIPELINE_INFEASIBLE (ref pipeline.hpp:309-315);
 *                                                     auto degrades to plain warp specialization
 *                                                     (driver.hpp:137-150) and runs
 *   coop_wgs < 1, or .k output-tile rows % coop_wgs -> INDIVISIBLE_TILE (ref grid.hpp:26-46)
 * Mapping onto the B200 kernels: d = aref depth (GEMM smem ring; attention K/V ring, min 2 — the
 * plain warp-specialized and `none` programs run with the smallest ring), p = MMA k-blocks in
 * flight (GEMM), mode none = d = p = 1 for GEMM, coop_wgs >= 2 = 256-row CTA-pair tiles
 * (cta_group::2; attention always runs two 128-row Q bands per CTA), persistent = persistent grid.
 * d = 0 / p = 0 select the library's measured defaults instead of the reference's (2, 1). */
typedef enum ws_pipeline_mode { WS_MODE_AUTO = 0, WS_MODE_FINE = 1, WS_MODE_COARSE = 2, WS_MODE_NONE = 3 } ws_pipeline_mode;
typedef struct ws_runspec {
  int32_t d;
  int32_t p;
  int32_t mode;
  int32_t coop_wgs;
  int32_t persistent;
} ws_runspec;

/* ws_run_kernel with a RunSpec (NULL = library defaults: the fastest measured configuration). */
ws_status ws_run_kernel_spec(const char* ktext, ws_kbuffer* buffers, int32_t nbuffers, int64_t pid_lo,
                             int64_t pid_hi, int32_t dtype, const ws_runspec* spec, void* cuda_stream);

/* Message for the last non-OK status returned on this thread ("" if none). */
const char* ws_last_error(void);

/* Number of kernel launches this library has issued since load (evidence counter). */
int64_t ws_launch_count(void);

/* Library version string, e.g. "ws-b200 0.1 sm_100a". */
const char* ws_version(void);

/* Device watchdog (the simulator's Deadlock verdict, ref proj/include/warpspec/sim.hpp:49-54,
 * 112-115, on hardware): every mbarrier wait in the kernels traps after 4 s without progress;
 * the first waiter to time out records where it waited in pinned host memory, so the record is
 * readable after the trap has torn down the CUDA context. */
typedef struct ws_watchdog_info {
  int32_t fired;     /* 1: a wait timed out and the kernel trapped */
  uint32_t block_x;  /* CTA of the waiter */
  uint32_t block_y;
  uint32_t thread;   /* threadIdx.x of the waiter (warp = thread / 32: its role) */
  uint32_t barrier;  /* shared-memory address of the mbarrier */
  uint32_t parity;   /* phase parity it waited for */
  uint32_t tag;      /* wait site (aref put/get, accumulator, softmax, ...; trace.py TAGS) */
} ws_watchdog_info;

/* Returns 1 and fills `out` if a watchdog fired in this process, else 0. */
int32_t ws_watchdog(ws_watchdog_info* out);

/* Developer diagnostics: subsequent ws_gemm_tn launches stamp %clock64 events of CTAs 0 and 1
 * (first 32 tiles, 16 events each) into `trace`, a device buffer of 2*32*16 uint64; NULL turns
 * it off. Event map in csrc/gemm_sm100.cuh (GT); reader: scripts/gemm_trace.py. */
void ws_debug_gemm_trace(unsigned long long* trace);

/* Developer diagnostics: subsequent ws_gemm_tn launches have CTA 0 store {%clock64, %globaltimer}
 * at its start and when it retires into `clk` (a zeroed device buffer of 8 uint64; the last
 * launch's stamps win), so the SM clock a launch ran at is (clk[2]-clk[0]) / (clk[3]-clk[1]) GHz,
 * and add the two spans and 1 to running totals clk[4], clk[5], clk[6] (the mean clock over every
 * probed launch is clk[4] / clk[5] GHz) — the per-clock efficiency of a measured kernel without an
 * external sampler. NULL turns it off. */
void ws_debug_gemm_clock(unsigned long long* clk);

#ifdef __cplusplus
}
#endif

#endif /* WS_H_ */
