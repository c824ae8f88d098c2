/*
 * darm_oracle.c — CPU restatement of the reference runtime path (see
 * darm_oracle.h).  TEST INFRASTRUCTURE ONLY; never part of the product.
 *
 * Lane semantics follow /root/reference/proj/src/interp.cpp:
 *   add/sub/mul/xor wrap as uint32        interp.cpp:118-130
 *   shl/shr mask the amount with 31       interp.cpp:126-127
 *   icmp.* signed, 0/1                    interp.cpp:145-164
 *   out-of-bounds load faults the lane    interp.cpp:172-186
 *   tid = lane index within the warp      interp.cpp:206-208
 * and the control flow of /root/reference/proj/corpus/<kernel>.ir (the line
 * numbers are cited per kernel).  The restatement is closed-form per lane: a
 * corpus lane only touches element t of each global, so the lockstep order of
 * the interpreter is unobservable except in bitonic's shared buffer, where
 * every partner read (bitonic.ir:10) precedes every store (:24, :35) and each
 * lane writes only its own slot.
 */
#include "darm_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------ mt19937_64 */
void oracle_mt64_seed(oracle_mt64 *g, uint64_t seed) {
  g->mt[0] = seed;
  for (int i = 1; i < 312; ++i)
    g->mt[i] = 6364136223846793005ULL * (g->mt[i - 1] ^ (g->mt[i - 1] >> 62)) + (uint64_t)i;
  g->idx = 312;
}

uint64_t oracle_mt64_next(oracle_mt64 *g) {
  if (g->idx >= 312) {
    for (int i = 0; i < 312; ++i) {
      uint64_t x = (g->mt[i] & 0xFFFFFFFF80000000ULL) | (g->mt[(i + 1) % 312] & 0x7FFFFFFFULL);
      uint64_t xa = x >> 1;
      if (x & 1ULL) xa ^= 0xB5026F5AA96619E9ULL;
      g->mt[i] = g->mt[(i + 156) % 312] ^ xa;
    }
    g->idx = 0;
  }
  uint64_t y = g->mt[g->idx++];
  y ^= (y >> 29) & 0x5555555555555555ULL;
  y ^= (y << 17) & 0x71D67FFFEDA60000ULL;
  y ^= (y << 37) & 0xFFF7EEE000000000ULL;
  y ^= y >> 43;
  return y;
}

/* ------------------------------------------------------ makeRandomInput */
void oracle_make_random_input(int n_params, const uint8_t *param_kinds, int n_mem,
                              const int64_t *mem_sizes, int warp, uint64_t seed,
                              int32_t *args, int32_t *mem_words) {
  oracle_mt64 g;
  oracle_mt64_seed(&g, seed);                                   /* fixtures.cpp:87 */
  for (int p = 0; p < n_params; ++p) {
    if (param_kinds[p]) {                                       /* 'j'/'k': :91-95 */
      int maxShift = 0;
      while ((1 << (maxShift + 1)) <= warp) ++maxShift;
      args[p] = 1 << (int)(oracle_mt64_next(&g) % (uint64_t)(maxShift + 1));
    } else {                                                    /* :96 */
      args[p] = (int32_t)(oracle_mt64_next(&g) % (uint64_t)(2 * warp));
    }
  }
  int64_t off = 0;
  for (int m = 0; m < n_mem; ++m)                               /* :99-106 */
    for (int64_t i = 0; i < mem_sizes[m]; ++i)
      mem_words[off++] = (int32_t)(oracle_mt64_next(&g) % 257) - 128;
}

/* ------------------------------------------------------------ lanes */
static inline int32_t wadd(int32_t a, int32_t b) { return (int32_t)((uint32_t)a + (uint32_t)b); }
static inline int32_t wsub(int32_t a, int32_t b) { return (int32_t)((uint32_t)a - (uint32_t)b); }
static inline int32_t wmul(int32_t a, int32_t b) { return (int32_t)((uint32_t)a * (uint32_t)b); }
static inline int32_t wshl(int32_t a, int32_t b) { return (int32_t)((uint32_t)a << ((uint32_t)b & 31u)); }

enum { K_SB1, K_SB1R, K_SB2, K_SB2R, K_SB3, K_SB3R, K_SB4, K_SB4R, K_NESTED, K_BITONIC, K_COUNT };
static const char *const kNames[K_COUNT] = {"sb1", "sb1r", "sb2", "sb2r", "sb3", "sb3r",
                                            "sb4", "sb4r", "nested", "bitonic"};
static const int kGlobals[K_COUNT] = {4, 2, 2, 2, 4, 4, 2, 2, 2, 1};
static const int kParams[K_COUNT] = {1, 1, 1, 1, 1, 1, 2, 2, 1, 2};

static inline int32_t arg_of(const int32_t *args, int64_t acount, int64_t n_warps, int p,
                             int64_t w, int64_t lane) {
  const int32_t *a = args + p * acount;
  if (acount == 1) return a[0];
  if (acount == n_warps) return a[w];
  return a[lane];
}

/* One lane of an sb-family / nested kernel.  G[i] points at element t of the
 * i-th global of this warp. */
static void sb_lane(int k, int32_t t, const int32_t *a, int32_t **G) {
  const int32_t n = a[0];
  switch (k) {
    case K_SB1: { /* sb1.ir:7-28 */
      int32_t e = t < n ? *G[1] : *G[2];
      *G[3] = wadd(wmul(*G[0], 3), e);
      break;
    }
    case K_SB1R: { /* sb1r.ir:5-26 */
      int32_t v = *G[0];
      *G[1] = t < n ? wshl(wadd(wmul(v, 3), n), 1) : wadd(wsub(v ^ n, 7), 2);
      break;
    }
    case K_SB2:
    case K_SB2R: { /* sb2.ir:5-36, sb2r.ir:5-36 */
      int32_t v = *G[0];
      int32_t r = v;
      if (v > n) r = (k == K_SB2R && !(t < n)) ? wsub(v ^ n, 3) : wadd(wmul(v, 2), 1);
      *G[1] = r;
      break;
    }
    case K_SB3:
    case K_SB3R: { /* sb3.ir:7-58, sb3r.ir:7-58 */
      const int alt = k == K_SB3R && !(t < n);
      int32_t v1 = *G[0];
      *G[2] = v1 > n ? (alt ? (v1 ^ 9) : wmul(v1, 2)) : v1;
      int32_t v2 = *G[1];
      *G[3] = v2 > n ? (alt ? wsub(v2, 5) : wadd(v2, 7)) : v2;
      break;
    }
    case K_SB4: /* sb4.ir:5-30: every leaf stores in+1 */
      *G[1] = wadd(*G[0], 1);
      break;
    case K_SB4R: { /* sb4r.ir:5-30 */
      const int32_t h = a[0], q = a[1];
      int32_t v = *G[0];
      *G[1] = t < h ? wadd(v, 1) : (t < q ? wmul(v, 3) : (v ^ 7));
      break;
    }
    case K_NESTED: { /* nested.ir:6-41: both sides compute the same diamond */
      int32_t v = *G[0];
      *G[1] = v > n ? wmul(v, 2) : wadd(v, 9);
      break;
    }
  }
}

int oracle_execute_warps(const char *kernel, int warp, int64_t n_warps, const int32_t *args,
                         int64_t acount, int32_t *globals, int64_t gstride,
                         const int32_t *shared, int32_t *faults) {
  int k = -1;
  for (int i = 0; i < K_COUNT; ++i)
    if (kernel && strcmp(kernel, kNames[i]) == 0) k = i;
  if (k < 0 || warp < 1 || warp > 64 || n_warps < 0 || gstride < warp) return 2;
  if (acount != 1 && acount != n_warps && acount != n_warps * warp) return 2;
  const int ng = kGlobals[k];
  if (k == K_BITONIC) {
    /* bitonic.ir:6-43; shared buf[64] per warp */
    const int64_t S = 64;
    for (int64_t w = 0; w < n_warps; ++w) {
      int32_t buf[64], nbuf[64];
      for (int i = 0; i < S; ++i) buf[i] = shared ? shared[w * S + i] : 0;
      memcpy(nbuf, buf, sizeof buf);
      int32_t nf = 0;
      int32_t *res = globals + w * gstride;
      for (int t = 0; t < warp; ++t) {
        const int64_t lane = w * warp + t;
        const int32_t kk = arg_of(args, acount, n_warps, 0, w, lane);
        const int32_t dir = arg_of(args, acount, n_warps, 1, w, lane);
        const int32_t j = t ^ kk;                               /* :9 */
        if (j < 0 || j >= S) { ++nf; continue; }                /* :10 faults */
        const int32_t b0 = buf[j];                              /* :10 */
        const int keep = t < j;                                 /* :11 */
        const int up = (t & dir) == 0;                          /* :12-13 */
        const int32_t cv = buf[t];                              /* :18 / :29 */
        const int need = up ? (keep ? cv > b0 : cv < b0)        /* :19-21 */
                            : (keep ? cv < b0 : cv > b0);       /* :30-32 */
        if (need) nbuf[t] = b0;                                 /* :24 / :35 */
        res[t] = nbuf[t];                                       /* :40-41 */
      }
      if (faults) faults[w] = nf;
    }
    return 0;
  }
  for (int64_t w = 0; w < n_warps; ++w) {
    for (int t = 0; t < warp; ++t) {
      const int64_t lane = w * warp + t;
      int32_t a[2] = {0, 0};
      for (int p = 0; p < kParams[k]; ++p) a[p] = arg_of(args, acount, n_warps, p, w, lane);
      int32_t *G[4];
      for (int g = 0; g < ng; ++g) G[g] = globals + (int64_t)g * n_warps * gstride + w * gstride + t;
      sb_lane(k, t, a, G);
    }
    if (faults) faults[w] = 0;
  }
  return 0;
}

int oracle_bitonic_sort(int32_t *keys, int64_t n, int bucket) {
  if (bucket < 2 || (bucket & (bucket - 1)) || n % bucket) return 2;
  const int B = bucket;
  for (int64_t b = 0; b < n / B; ++b) {
    int32_t *v = keys + b * B;
    for (int dir = 2; dir <= B; dir <<= 1)
      for (int k = dir >> 1; k >= 1; k >>= 1)
        for (int t = 0; t < B; ++t) {
          const int j = t ^ k;
          if (j < t) continue; /* each pair once, from its lower lane */
          const int up = (t & dir) == 0;
          /* lane t (keep) takes b0 if cv > b0 when up; lane j the converse */
          const int swap = up ? v[t] > v[j] : v[t] < v[j];
          if (swap) {
            int32_t x = v[t];
            v[t] = v[j];
            v[j] = x;
          }
        }
  }
  return 0;
}

/* Batcher odd-even merge sort of each B-key bucket (PCM; no
 * reference code): the chain of ir/oddeven_step.ir steps, p = 1..B/2,
 * k = p..1; comparator (x, x + k) for x >= k % p, (x - k % p) mod 2k < k,
 * x + k < B, x and x + k in the same 2p block. */
int oracle_oddeven_sort(int32_t *keys, int64_t n, int bucket) {
  if (bucket < 2 || (bucket & (bucket - 1)) || n % bucket) return 2;
  const int B = bucket;
  for (int64_t b = 0; b < n / B; ++b) {
    int32_t *v = keys + b * B;
    for (int p = 1; p < B; p <<= 1)
      for (int k = p; k >= 1; k >>= 1) {
        const int kp = k % p;
        for (int x = kp; x + k < B; ++x) {
          if ((x - kp) % (2 * k) >= k || x / (2 * p) != (x + k) / (2 * p)) continue;
          if (v[x] > v[x + k]) {
            int32_t t = v[x];
            v[x] = v[x + k];
            v[x + k] = t;
          }
        }
      }
  }
  return 0;
}

/* Bottom-up merge sort of keys[0..n) (MS; no reference
 * code): passes w = 1, 2, 4, .. < n merge runs [a, a+w) and [a+w, a+2w),
 * clipped to n, taking the left head on ties (the loop of
 * paper_2107_05681_b200/ir/merge_step.ir). */
int oracle_merge_sort(int32_t *keys, int64_t n) {
  if (n < 0) return 2;
  if (n < 2) return 0;
  int32_t *tmp = (int32_t *)malloc(sizeof(int32_t) * (size_t)n);
  if (!tmp) return 3;
  int32_t *src = keys, *dst = tmp;
  for (int64_t w = 1; w < n; w <<= 1) {
    for (int64_t a = 0; a < n; a += 2 * w) {
      int64_t i = a, iend = a + w < n ? a + w : n, j = iend, jend = a + 2 * w < n ? a + 2 * w : n, k = a;
      while (k < jend) {
        const int take = j >= jend || (i < iend && src[i] <= src[j]);
        dst[k++] = take ? src[i++] : src[j++];
      }
    }
    int32_t *t = src;
    src = dst;
    dst = t;
  }
  if (src != keys) memcpy(keys, src, sizeof(int32_t) * (size_t)n);
  free(tmp);
  return 0;
}

/* ------------------------------------------------------------ N-Queens
 * The reference has no NQU code; this is an independent
 * recursive restatement of the search that paper_2107_05681_b200/ir/
 * nqueens_sym.ir runs iteratively.  Prefix order: every valid placement of
 * rows 0..base-1, lowest free column first; prefix i belongs to rank i % world. */
typedef struct {
  int n, base, rank, world;
  uint32_t mask, row0;   /* row0: the columns row 0 may take */
  uint32_t *out;
  int64_t cap, idx, kept;
} nq_enum;

static void nq_prefix_rec(nq_enum *e, int row, uint32_t cols, uint32_t d1, uint32_t d2) {
  if (row == e->base) {
    if (e->idx % e->world == e->rank) {
      if (e->out && e->kept < e->cap) {
        e->out[3 * e->kept] = cols;
        e->out[3 * e->kept + 1] = d1;
        e->out[3 * e->kept + 2] = d2;
      }
      e->kept++;
    }
    e->idx++;
    return;
  }
  uint32_t av = ~(cols | d1 | d2) & (row == 0 ? e->row0 : e->mask);
  while (av) {
    uint32_t bit = av & (0u - av);
    av ^= bit;
    nq_prefix_rec(e, row + 1, cols | bit, (d1 | bit) << 1, (d2 | bit) >> 1);
  }
}

int64_t oracle_nqueens_prefixes(int n, int base, int rank, int world, uint32_t *out, int64_t cap) {
  return oracle_nqueens_prefixes_ex(n, base, rank, world, 0, out, cap);
}

/* mirror: row 0 only in the columns < ceil(n/2) (the GPU's DARM_NQ_MIRROR
 * prefix set; for even n every kept placement counts twice) */
int64_t oracle_nqueens_prefixes_ex(int n, int base, int rank, int world, int mirror, uint32_t *out, int64_t cap) {
  const uint32_t mask = n >= 32 ? 0xffffffffu : ((1u << n) - 1u);
  nq_enum e = {n, base, rank, world, mask, mirror ? ((1u << ((n + 1) / 2)) - 1u) : mask, out, cap, 0, 0};
  nq_prefix_rec(&e, 0, 0, 0, 0);
  return e.kept;
}

static uint32_t nq_count_rec(int n, uint32_t mask, int row, uint32_t cols, uint32_t d1, uint32_t d2,
                             uint64_t *nodes) {
  if (row == n) return 1;
  uint32_t av = ~(cols | d1 | d2) & mask, sols = 0;
  while (av) {
    uint32_t bit = av & (0u - av);
    av ^= bit;
    ++*nodes;
    sols += nq_count_rec(n, mask, row + 1, cols | bit, (d1 | bit) << 1, (d2 | bit) >> 1, nodes);
  }
  return sols;
}

uint64_t oracle_nqueens_count(int n, int base, const uint32_t *states, int64_t count, uint32_t *per_prefix,
                              uint64_t *nodes) {
  const uint32_t mask = n >= 32 ? 0xffffffffu : ((1u << n) - 1u);
  uint64_t total = 0, nd = 0;
  for (int64_t i = 0; i < count; ++i) {
    uint32_t s = nq_count_rec(n, mask, base, states[3 * i], states[3 * i + 1], states[3 * i + 2], &nd);
    if (per_prefix) per_prefix[i] = s;
    total += s;
  }
  if (nodes) *nodes = nd;
  return total;
}

/* ------------------------------------------------------------ LUD
 * Blocked LU without pivoting, BLOCK = 16 (no reference code; Rodinia's
 * diagonal / perimeter / internal order).  Every update is
 * written as the single-rounding fmaf / division / subtraction the CUDA
 * kernels (paper_2107_05681_b200/csrc/lud.cu) perform, in the same order, so
 * the results agree bit for bit.  The internal update is split over threads
 * by rows (rows are independent). */
#define LUD_BS 16

__attribute__((target("fma"))) static float fma_hw(float a, float b, float c) { return __builtin_fmaf(a, b, c); }
static float fma_sw(float a, float b, float c) { return fmaf(a, b, c); }
static float (*lud_fma)(float, float, float) = fma_sw;

typedef struct {
  float *a;
  int64_t n, o, r0, r1;
} lud_job;

/* Per row r: sums[c] = fma(L[r][k], U[k][c], sums[c]) for k = 0..15 (the
 * per-element order of the GPU kernel, vectorised across c), then
 * a[r][c] -= sums[c]. */
#define LUD_ROWS_BODY(FMA)                                                   \
  lud_job *j = (lud_job *)p;                                                 \
  float *a = j->a;                                                           \
  const int64_t n = j->n, o = j->o, w = n - o - LUD_BS;                      \
  float *sums = (float *)malloc(sizeof(float) * (size_t)(w > 0 ? w : 1));    \
  for (int64_t r = j->r0; r < j->r1; ++r) {                                  \
    float *ar = a + r * n + o + LUD_BS;                                      \
    for (int64_t c = 0; c < w; ++c) sums[c] = 0.f;                           \
    for (int k = 0; k < LUD_BS; ++k) {                                       \
      const float l = a[r * n + o + k];                                      \
      const float *u = a + (o + k) * n + o + LUD_BS;                         \
      for (int64_t c = 0; c < w; ++c) sums[c] = FMA(l, u[c], sums[c]);       \
    }                                                                        \
    for (int64_t c = 0; c < w; ++c) ar[c] = ar[c] - sums[c];                 \
  }                                                                          \
  free(sums);                                                                \
  return NULL;

__attribute__((target("fma"))) static void *lud_internal_rows_fma(void *p) { LUD_ROWS_BODY(__builtin_fmaf) }
static void *lud_internal_rows_sw(void *p) { LUD_ROWS_BODY(fmaf) }

int oracle_lud(float *a, int64_t n, int threads) {
  if (n < LUD_BS || n % LUD_BS) return 2;
  lud_fma = __builtin_cpu_supports("fma") ? fma_hw : fma_sw;
  if (threads < 1) threads = 1;
  if (threads > 256) threads = 256;
  for (int64_t o = 0; o < n; o += LUD_BS) {
    float *d = a + o * n + o;
    /* diagonal: column i of L, then row i+1 of U */
    for (int i = 0; i < LUD_BS - 1; ++i) {
      for (int r = i + 1; r < LUD_BS; ++r) {
        float x = d[r * n + i];
        for (int j = 0; j < i; ++j) x = lud_fma(-d[r * n + j], d[j * n + i], x);
        d[r * n + i] = x / d[i * n + i];
      }
      for (int c = i + 1; c < LUD_BS; ++c) {
        float x = d[(i + 1) * n + c];
        for (int j = 0; j < i + 1; ++j) x = lud_fma(-d[(i + 1) * n + j], d[j * n + c], x);
        d[(i + 1) * n + c] = x;
      }
    }
    if (o + LUD_BS >= n) break;
    /* perimeter: U12 = L11^-1 A12 (forward substitution per column) */
    for (int64_t c = o + LUD_BS; c < n; ++c)
      for (int i = 1; i < LUD_BS; ++i) {
        float x = a[(o + i) * n + c];
        for (int j = 0; j < i; ++j) x = lud_fma(-d[i * n + j], a[(o + j) * n + c], x);
        a[(o + i) * n + c] = x;
      }
    /* perimeter: L21 = A21 U11^-1 (per row) */
    for (int64_t r = o + LUD_BS; r < n; ++r)
      for (int i = 0; i < LUD_BS; ++i) {
        float x = a[r * n + o + i];
        for (int j = 0; j < i; ++j) x = lud_fma(-a[r * n + o + j], d[j * n + i], x);
        a[r * n + o + i] = x / d[i * n + i];
      }
    /* internal: A22 -= L21 U12, sum over k = 0..15 then one subtraction */
    const int64_t rows = n - o - LUD_BS;
    int t = (int)(rows < threads ? rows : threads);
    if (rows * (n - o) < (1 << 16)) t = 1;
    pthread_t tid[256];
    lud_job jobs[256];
    void *(*rows_fn)(void *) = lud_fma == fma_hw ? lud_internal_rows_fma : lud_internal_rows_sw;
    for (int q = 0; q < t; ++q) {
      jobs[q].a = a;
      jobs[q].n = n;
      jobs[q].o = o;
      jobs[q].r0 = o + LUD_BS + rows * q / t;
      jobs[q].r1 = o + LUD_BS + rows * (q + 1) / t;
      if (t > 1)
        pthread_create(&tid[q], NULL, rows_fn, &jobs[q]);
      else
        rows_fn(&jobs[q]);
    }
    if (t > 1)
      for (int q = 0; q < t; ++q) pthread_join(tid[q], NULL);
  }
  return 0;
}

/* ------------------------------------------------------------ SRAD
 * Rodinia SRAD restated (no reference code), in exactly
 * the operation order of csrc/srad.cu (compiled there with -fmad=false; this
 * file with -ffp-contract=off).  ROI statistics: per ROI row and 128-column
 * warp group, each lane's 4 columns summed in order, then the 32-lane fp64
 * xor-butterfly the kernel performs (lane 0's result), then rows and groups
 * folded in order. */
static int clampi_(int v, int lo, int hi) { return v < lo ? lo : (v > hi ? hi : v); }

static float srad_c(float jc, float n, float s, float w, float e, float q0sqr, float q0den) {
  const float dN = n - jc, dS = s - jc, dW = w - jc, dE = e - jc;
  const float g2 = (((dN * dN + dS * dS) + dW * dW) + dE * dE) / (jc * jc);
  const float l = (((dN + dS) + dW) + dE) / jc;
  const float num = (0.5f * g2) - ((1.0f / 16.0f) * (l * l));
  float den = 1.0f + (0.25f * l);
  const float qsqr = num / (den * den);
  den = (qsqr - q0sqr) / q0den;
  float c = 1.0f / (1.0f + den);
  if (c < 0.0f) c = 0.0f;            /* R_D */
  else if (c > 1.0f) c = 1.0f;
  return c;
}

static float srad_q0(const float *J, int64_t cols, const int *roi) {
  const int w0 = roi[2] / 128, groups = roi[3] / 128 - w0 + 1;
  double s = 0.0, s2 = 0.0;
  for (int g = roi[0]; g <= roi[1]; ++g)
    for (int w = w0; w < w0 + groups; ++w) {
      double a[32], b[32];
      for (int L = 0; L < 32; ++L) {   /* lane L: its 4 columns in order */
        double sa = 0.0, sb = 0.0;
        for (int k = 0; k < 4; ++k) {
          const int64_t j = (int64_t)w * 128 + 4 * L + k;
          const int in = j < cols && j >= roi[2] && j <= roi[3];
          const double v = in ? (double)J[g * cols + j] : 0.0;
          sa += v;
          sb += v * v;
        }
        a[L] = sa;
        b[L] = sb;
      }
      for (int o = 16; o > 0; o >>= 1) {
        double na[32], nb[32];
        for (int L = 0; L < 32; ++L) {
          na[L] = a[L] + a[L ^ o];
          nb[L] = b[L] + b[L ^ o];
        }
        memcpy(a, na, sizeof a);
        memcpy(b, nb, sizeof b);
      }
      s += a[0];
      s2 += b[0];
    }
  const double npix = (double)(roi[1] - roi[0] + 1) * (double)(roi[3] - roi[2] + 1);
  const double mean = s / npix;
  const double var = s2 / npix - mean * mean;
  return (float)(var / (mean * mean));
}

typedef struct {
  const float *J;
  float *C, *out;
  int64_t rows, cols, r0, r1;
  float q0sqr, q0den, lq;
  int phase;
} srad_job;

static void *srad_rows(void *p) {
  srad_job *t = (srad_job *)p;
  const float *J = t->J;
  const int64_t R = t->rows, C = t->cols;
  for (int64_t i = t->r0; i < t->r1; ++i)
    for (int64_t j = 0; j < C; ++j) {
      const float jc = J[i * C + j];
      const float n = J[clampi_((int)i - 1, 0, (int)R - 1) * C + j];
      const float s = J[clampi_((int)i + 1, 0, (int)R - 1) * C + j];
      const float w = J[i * C + clampi_((int)j - 1, 0, (int)C - 1)];
      const float e = J[i * C + clampi_((int)j + 1, 0, (int)C - 1)];
      if (t->phase == 0) {
        t->C[i * C + j] = srad_c(jc, n, s, w, e, t->q0sqr, t->q0den);
      } else {
        const float c0 = t->C[i * C + j];
        const float c1 = t->C[clampi_((int)i + 1, 0, (int)R - 1) * C + j];
        const float ce = t->C[i * C + clampi_((int)j + 1, 0, (int)C - 1)];
        const float dN = n - jc, dS = s - jc, dW = w - jc, dE = e - jc;
        const float d = ((c0 * dN + c1 * dS) + c0 * dW) + ce * dE;
        t->out[i * C + j] = jc + t->lq * d;
      }
    }
  return NULL;
}

int oracle_srad(float *J, int64_t rows, int64_t cols, int iters, float lambda, const int *roi, int threads) {
  if (rows < 1 || cols < 2 || iters < 0) return 2;
  if (threads < 1) threads = 1;
  if (threads > 256) threads = 256;
  float *Cb = (float *)malloc(sizeof(float) * (size_t)(rows * cols));
  float *Jn = (float *)malloc(sizeof(float) * (size_t)(rows * cols));
  if (!Cb || !Jn) return 3;
  const float lq = 0.25f * lambda;
  for (int it = 0; it < iters; ++it) {
    const float q0sqr = srad_q0(J, cols, roi);
    const float q0den = q0sqr * (1.0f + q0sqr);
    for (int phase = 0; phase < 2; ++phase) {
      int t = (int)(rows < threads ? rows : threads);
      pthread_t tid[256];
      srad_job jobs[256];
      for (int q = 0; q < t; ++q) {
        srad_job jb = {J, Cb, Jn, rows, cols, rows * q / t, rows * (q + 1) / t, q0sqr, q0den, lq, phase};
        jobs[q] = jb;
        if (t > 1)
          pthread_create(&tid[q], NULL, srad_rows, &jobs[q]);
        else
          srad_rows(&jobs[q]);
      }
      if (t > 1)
        for (int q = 0; q < t; ++q) pthread_join(tid[q], NULL);
    }
    memcpy(J, Jn, sizeof(float) * (size_t)(rows * cols));
  }
  free(Cb);
  free(Jn);
  return 0;
}
