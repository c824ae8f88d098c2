/*
 * darm_oracle.h — CPU restatement of the reference's runtime path for the
 * corpus kernels.  TEST INFRASTRUCTURE ONLY: loaded by tests/, by
 * __graft_entry__.smoke() and by bench.py's cpu_baseline leg as the checker;
 * the product (paper_2107_05681_b200/) never links or calls it.
 *
 * Pinned against the reference itself: tests/test_oracle.py checks every
 * function here against tests/golden/ (JSON), which oracle/gen_golden.py
 * produced by running the unmodified reference (oracle/_ref/libdarm_ref.so:
 * executeWarp / makeRandomInput / runDarm) — see DESIGN.md §Oracle.
 */
#ifndef DARM_ORACLE_H
#define DARM_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* std::mt19937_64 (used by makeRandomInput, fixtures.cpp:87), restated. */
typedef struct oracle_mt64 {
  uint64_t mt[312];
  int idx;
} oracle_mt64;
void oracle_mt64_seed(oracle_mt64 *g, uint64_t seed);
uint64_t oracle_mt64_next(oracle_mt64 *g);

/* makeRandomInput (fixtures.cpp:82-108) for one warp.  param_kinds[p] is 1
 * when the parameter name starts with 'j' or 'k'.  mem_sizes lists the
 * declared sizes of the globals then the shared decls; mem_words receives
 * them concatenated in that order. */
void oracle_make_random_input(int n_params, const uint8_t *param_kinds, int n_mem,
                              const int64_t *mem_sizes, int warp, uint64_t seed,
                              int32_t *args, int32_t *mem_words);

/* executeWarp (interp.cpp:332-381) restated per corpus kernel as closed-form
 * lane semantics of the IR, batched over n_warps warps in the layout of
 * darm_gpu_execute_warps (globals concatenated, each n_warps x gstride words,
 * lane t of warp w at w*gstride + t; shared n_warps x declared size).
 * Returns 0, or 2 for an unknown kernel / bad arguments. */
int oracle_execute_warps(const char *kernel, int warp, int64_t n_warps, const int32_t *args,
                         int64_t acount, int32_t *globals, int64_t gstride,
                         const int32_t *shared, int32_t *faults);

/* Chain of bitonic.ir steps over every stage (dir = 2..B, k = dir/2..1) of
 * each B-key bucket (B power of two). */
int oracle_bitonic_sort(int32_t *keys, int64_t n, int bucket);

/* Batcher odd-even merge sort of each B-key bucket (PCM; the chain of
 * ir/oddeven_step.ir steps p = 1..B/2, k = p..1). */
int oracle_oddeven_sort(int32_t *keys, int64_t n, int bucket);

/* Bottom-up merge sort of keys[0..n) (MS; the loop of ir/merge_step.ir). */
int oracle_merge_sort(int32_t *keys, int64_t n);

/* N-Queens (no reference code; recursive restatement).  Prefixes: valid
 * placements of rows 0..base-1, lowest free column first, index i kept when
 * i % world == rank, written as {cols, d1, d2} triples (up to cap).  Returns the
 * number kept.  oracle_nqueens_count returns the total solutions below the
 * prefixes, per-prefix counts, and the placements made below them (`nodes`). */
int64_t oracle_nqueens_prefixes(int n, int base, int rank, int world, uint32_t *out, int64_t cap);
int64_t oracle_nqueens_prefixes_ex(int n, int base, int rank, int world, int mirror, uint32_t *out, int64_t cap);
uint64_t oracle_nqueens_count(int n, int base, const uint32_t *states, int64_t count, uint32_t *per_prefix,
                              uint64_t *nodes);

/* LUD (no reference code): blocked LU without pivoting, BLOCK = 16, in
 * place, in exactly the floating-point operation order of csrc/lud.cu.
 * threads > 1 splits the internal update by rows (pthreads). */
int oracle_lud(float *a, int64_t n, int threads);

/* SRAD (no reference code): `iters` iterations on a rows x cols fp32 image,
 * in place, ROI {r1, r2, c1, c2}, in exactly csrc/srad.cu's operation order. */
int oracle_srad(float *J, int64_t rows, int64_t cols, int iters, float lambda, const int *roi, int threads);

#ifdef __cplusplus
}
#endif

#endif
