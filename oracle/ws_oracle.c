/*
 * ws_oracle.c — CPU restatement of the reference's arithmetic for the hot path.
 *
 * TEST INFRASTRUCTURE ONLY. This file is the checker: only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load it. The product path (libws.so) never
 * links or calls it, and there is no CPU fallback anywhere in the package.
 *
 * What it restates (all citations into /root/reference/proj):
 *   - generate_inputs: mt19937_64(seed ^ fnv1a64(name)); int: rng%19 - 9; real: (rng%33 - 16)/4
 *       include/warpspec/driver.hpp:70-89
 *   - eval_dot: out = acc; s = out(r,c); for i: s += a(r,i) * b(c,i)  (trans_b), double or
 *       int64 wrapping                                  include/warpspec/tile.hpp:218-247
 *   - the gemm.k loop: acc carried across K tiles, so every output element is one sequential sum
 *       over k = 0..K-1 starting from 0                 kernels/gemm.k:8-16, interp.hpp:164-176
 *   - the flash .k of SURVEY.md Appendix A (ew/reduce semantics of tile.hpp:138-215):
 *       s = q.k^T (+ mask); ss = s*sc; rm = rowmax(ss); mn = max(m, rm); pp = exp(ss - mn);
 *       al = exp(m - mn); l = l*al + rowsum(pp); acc = acc*al + pp.v; m = mn
 *     and the harness step o = acc / l, lse = m + log(l).
 *
 * Parity is pinned against the reference itself: oracle/_ref/libwsref.so (built from the
 * reference headers by oracle/Makefile) and the golden vectors under tests/golden/ produced by
 * tests/golden/make_golden.py from it; see tests/test_oracle.py.
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------------------------------ */
/* mt19937_64 (the std::mt19937_64 engine: w=64, n=312, m=156, r=31)                          */
/* ------------------------------------------------------------------------------------------ */
typedef struct {
  uint64_t mt[312];
  int idx;
} mt64;

static void mt64_seed(mt64* s, uint64_t seed) {
  s->mt[0] = seed;
  for (int i = 1; i < 312; ++i) s->mt[i] = 6364136223846793005ULL * (s->mt[i - 1] ^ (s->mt[i - 1] >> 62)) + (uint64_t)i;
  s->idx = 312;
}

static uint64_t mt64_next(mt64* s) {
  static const uint64_t UM = 0xFFFFFFFF80000000ULL, LM = 0x7FFFFFFFULL, A = 0xB5026F5AA96619E9ULL;
  if (s->idx >= 312) {
    for (int i = 0; i < 312; ++i) {
      uint64_t x = (s->mt[i] & UM) | (s->mt[(i + 1) % 312] & LM);
      uint64_t xa = x >> 1;
      if (x & 1ULL) xa ^= A;
      s->mt[i] = s->mt[(i + 156) % 312] ^ xa;
    }
    s->idx = 0;
  }
  uint64_t x = s->mt[s->idx++];
  x ^= (x >> 29) & 0x5555555555555555ULL;
  x ^= (x << 17) & 0x71D67FFFEDA60000ULL;
  x ^= (x << 37) & 0xFFF7EEE000000000ULL;
  x ^= x >> 43;
  return x;
}

uint64_t ws_oracle_fnv1a64(const char* s) {
  uint64_t h = 1469598103934665603ULL;
  for (; *s; ++s) {
    h ^= (unsigned char)*s;
    h *= 1099511628211ULL;
  }
  return h;
}

/* generate_inputs for one buffer (ref driver.hpp:79-89): real payloads in {-4, -3.75, ..., 4}. */
void ws_oracle_generate_real(uint64_t seed, const char* name, int64_t n, double* out) {
  mt64 st;
  mt64_seed(&st, seed ^ ws_oracle_fnv1a64(name));
  for (int64_t i = 0; i < n; ++i) out[i] = ((double)(mt64_next(&st) % 33) - 16.0) / 4.0;
}

/* Same stream, as small integers in [-16, 16] (value = 4 x the real payload): lets the harness
 * build exact fp16/bf16/e4m3 device inputs without a double round trip. */
void ws_oracle_generate_real_x4(uint64_t seed, const char* name, int64_t n, int8_t* out) {
  mt64 st;
  mt64_seed(&st, seed ^ ws_oracle_fnv1a64(name));
  for (int64_t i = 0; i < n; ++i) out[i] = (int8_t)((int)(mt64_next(&st) % 33) - 16);
}

void ws_oracle_generate_int(uint64_t seed, const char* name, int64_t n, int64_t* out) {
  mt64 st;
  mt64_seed(&st, seed ^ ws_oracle_fnv1a64(name));
  for (int64_t i = 0; i < n; ++i) out[i] = (int64_t)(mt64_next(&st) % 19) - 9;
}

/* ------------------------------------------------------------------------------------------ */
/* thread pool helper: split [0, n) over nthreads                                              */
/* ------------------------------------------------------------------------------------------ */
typedef void (*range_fn)(void* ctx, int64_t lo, int64_t hi);
typedef struct {
  range_fn fn;
  void* ctx;
  int64_t lo, hi;
} range_job;

static void* range_thread(void* p) {
  range_job* j = (range_job*)p;
  j->fn(j->ctx, j->lo, j->hi);
  return NULL;
}

static void parallel_for(int64_t n, int nthreads, range_fn fn, void* ctx) {
  if (nthreads <= 1 || n <= 1) {
    fn(ctx, 0, n);
    return;
  }
  if (nthreads > n) nthreads = (int)n;
  pthread_t th[256];
  range_job jobs[256];
  if (nthreads > 256) nthreads = 256;
  for (int t = 0; t < nthreads; ++t) {
    jobs[t].fn = fn;
    jobs[t].ctx = ctx;
    jobs[t].lo = n * t / nthreads;
    jobs[t].hi = n * (t + 1) / nthreads;
    pthread_create(&th[t], NULL, range_thread, &jobs[t]);
  }
  for (int t = 0; t < nthreads; ++t) pthread_join(th[t], NULL);
}

/* ------------------------------------------------------------------------------------------ */
/* GEMM: c[M x N] = scale * a[M x K] . b[N x K]^T (gemm.k with real payloads)                  */
/* ------------------------------------------------------------------------------------------ */
typedef struct {
  const double *a, *b;
  double* c;
  int64_t M, N, K, ldc;
  double scale;
  int64_t n_lo;  /* first output column (N-shard offset) */
} gemm_ctx;

static void gemm_rows(void* p, int64_t lo, int64_t hi) {
  gemm_ctx* g = (gemm_ctx*)p;
  for (int64_t r = lo; r < hi; ++r) {
    const double* ar = g->a + r * g->K;
    for (int64_t n = 0; n < g->N; ++n) {
      const double* br = g->b + n * g->K;
      double s = 0.0; /* %z = const zeros (gemm.k:8) */
      for (int64_t i = 0; i < g->K; ++i) s += ar[i] * br[i]; /* eval_dot, tile.hpp:237-241 */
      /* FP8 .k variant: %o = ew mul %acc, %s before the store */
      g->c[r * g->ldc + n] = g->scale == 1.0 ? s : s * g->scale;
    }
  }
}

void ws_oracle_gemm_real(const double* a, const double* b, double* c, int64_t M, int64_t N, int64_t K, int64_t ldc,
                         double scale, int nthreads) {
  gemm_ctx g = {a, b, c, M, N, K, ldc, scale, 0};
  parallel_for(M, nthreads, gemm_rows, &g);
}

/* int64 wrapping GEMM (the shipped integer kernels; tile.hpp:63-71, 228-235) */
void ws_oracle_gemm_int(const int64_t* a, const int64_t* b, int64_t* c, int64_t M, int64_t N, int64_t K) {
  for (int64_t r = 0; r < M; ++r)
    for (int64_t n = 0; n < N; ++n) {
      uint64_t s = 0;
      for (int64_t i = 0; i < K; ++i) s += (uint64_t)a[r * K + i] * (uint64_t)b[n * K + i];
      c[r * N + n] = (int64_t)s;
    }
}

/* ------------------------------------------------------------------------------------------ */
/* FlashAttention forward: the Appendix A flash .k, one pid = one BR-row query block of one    */
/* (b,h) slice; [BH, S, Dh] row-major operands.                                                */
/* ------------------------------------------------------------------------------------------ */
typedef struct {
  const double *q, *k, *v;
  double *o, *lse;
  int64_t S, Dh, BR, BC;
  int causal;
  double sc;
  int64_t nqb;
  int64_t pid_base;
} flash_ctx;

static void flash_blocks(void* p, int64_t lo, int64_t hi) {
  flash_ctx* f = (flash_ctx*)p;
  const int64_t BR = f->BR, BC = f->BC, Dh = f->Dh, S = f->S;
  double* acc = (double*)malloc(sizeof(double) * BR * Dh);
  double* m = (double*)malloc(sizeof(double) * BR);
  double* l = (double*)malloc(sizeof(double) * BR);
  double* ss = (double*)malloc(sizeof(double) * BR * BC);
  for (int64_t pid = f->pid_base + lo; pid < f->pid_base + hi; ++pid) {
    const int64_t bh = pid / f->nqb, qb = pid % f->nqb;
    const double* Q = f->q + (bh * S + qb * BR) * Dh;
    const double* K = f->k + bh * S * Dh;
    const double* V = f->v + bh * S * Dh;
    for (int64_t i = 0; i < BR * Dh; ++i) acc[i] = 0.0;          /* %zacc */
    for (int64_t r = 0; r < BR; ++r) m[r] = 0.0 + -1000000.0;      /* %m0 = ew add %zc, %ninf */
    for (int64_t r = 0; r < BR; ++r) l[r] = 0.0;                   /* %zc */
    const int64_t nkb = S / BC;
    for (int64_t j = 0; j < nkb; ++j) {
      /* causal selector: 0 below, 1 on, 2 above the diagonal block. Blocks above the diagonal
       * carry mask -1e7 on every element: exp(ss - mn) underflows to exactly 0, al = exp(0) = 1,
       * so the .k's update is the identity there; skipping them is bit-identical. */
      if (f->causal && j > qb) break;
      const double* Kj = K + j * BC * Dh;
      const double* Vj = V + j * BC * Dh;
      for (int64_t r = 0; r < BR; ++r) {
        for (int64_t c = 0; c < BC; ++c) {
          double s = (f->causal && j == qb && c > r) ? -10000000.0 : 0.0; /* %tm or %zs */
          for (int64_t i = 0; i < Dh; ++i) s += Q[r * Dh + i] * Kj[c * Dh + i]; /* dot %tq, %tk.T */
          ss[r * BC + c] = s * f->sc;                                             /* ew mul %s, %sc */
        }
      }
      for (int64_t r = 0; r < BR; ++r) {
        double rm = ss[r * BC];
        for (int64_t c = 1; c < BC; ++c) rm = ss[r * BC + c] > rm ? ss[r * BC + c] : rm; /* reduce max */
        const double mn = m[r] > rm ? m[r] : rm;                                       /* ew max */
        double rs = 0.0;
        for (int64_t c = 0; c < BC; ++c) {
          const double pp = exp(ss[r * BC + c] - mn); /* ew sub, ew exp */
          ss[r * BC + c] = pp;
          rs = rs + pp; /* reduce add (tile.hpp:204-209) */
        }
        const double al = exp(m[r] - mn);
        l[r] = l[r] * al + rs;
        for (int64_t d = 0; d < Dh; ++d) {
          double s = acc[r * Dh + d] * al;                                       /* %as */
          for (int64_t c = 0; c < BC; ++c) s += ss[r * BC + c] * Vj[c * Dh + d]; /* dot %pp, %tv */
          acc[r * Dh + d] = s;
        }
        m[r] = mn;
      }
    }
    double* O = f->o + (bh * S + qb * BR) * Dh;
    for (int64_t r = 0; r < BR; ++r) {
      for (int64_t d = 0; d < Dh; ++d) O[r * Dh + d] = acc[r * Dh + d] / l[r]; /* harness: o / lsum */
      if (f->lse) f->lse[bh * S + qb * BR + r] = m[r] + log(l[r]);
    }
  }
  free(acc);
  free(m);
  free(l);
  free(ss);
}

/* q, k, v, o: [BH, S, Dh]; lse: [BH, S] (may be NULL). Computes pids [pid_lo, pid_hi) where
 * pid = bh * (S/BR) + query block (the batched .k pid order). */
void ws_oracle_flash(const double* q, const double* k, const double* v, double* o, double* lse, int64_t BH,
                     int64_t S, int64_t Dh, int64_t BR, int64_t BC, int causal, double softmax_scale,
                     int64_t pid_lo, int64_t pid_hi, int nthreads) {
  flash_ctx f = {q, k, v, o, lse, S, Dh, BR, BC, causal, softmax_scale, S / BR, pid_lo};
  (void)BH;
  parallel_for(pid_hi - pid_lo, nthreads, flash_blocks, &f);
}
