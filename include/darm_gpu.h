/*
 * darm_gpu.h — C-ABI of libdarm_gpu.so, the B200 (sm_100a) runtime path for the
 * DARM corpus kernels (arXiv 2107.05681).
 *
 * This header is the drop-in boundary.  Every entry point replaces one reference
 * interface on the runtime path; the reference citation is given
 * per function as /root/reference/proj/<file>:<line>.
 *
 * Conventions (SURVEY.md §8b "Errors"):
 *   - return DARM_OK (0), DARM_USER_ERROR (2: bad kernel name, sizes, arguments,
 *     device index) or DARM_INTERNAL_ERROR (3: CUDA failure), mirroring the CLI's
 *     exit codes (tools/darm_cli.cpp:25-27).  No C++ exception crosses the ABI.
 *   - err/errlen: optional buffer that receives a one-line message on failure.
 *   - mem: DARM_MEM_HOST -> every data pointer is host memory; the library stages
 *     it through its own cached device buffers with H2D/D2H copies on `stream`
 *     (pinned host memory gives full PCIe/C2C speed).  DARM_MEM_DEVICE -> every
 *     data pointer is device memory on the current device; nothing is copied.
 *   - stream: a cudaStream_t (NULL = legacy default stream).  HOST calls return
 *     after the D2H copy completed; DEVICE calls are asynchronous on `stream`.
 *   - Thread safety: calls from several host threads are serialised per device
 *     (one lock per device guards the cached buffers and graphs).  The cached
 *     device work areas (HOST staging buffers, LUD's diagonal scratch and
 *     tile counters, SRAD's ping-pong image) are per device, not per stream:
 *     two asynchronous calls of the same entry point on different streams must
 *     be ordered by the caller (an event), or run on one stream.
 *   - There is no CPU fallback: without a usable sm_100 device every compute
 *     entry point fails with DARM_INTERNAL_ERROR.
 */
#ifndef DARM_GPU_H
#define DARM_GPU_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define DARM_GPU_ABI_VERSION 1

#define DARM_OK 0
#define DARM_USER_ERROR 2
#define DARM_INTERNAL_ERROR 3

/* Kernel forms (north star: "each kernel ... in two forms"), plus two
 * reference columns where the comparison needs them. */
#define DARM_UNMELDED 0 /* original CFG, IPDOM reconvergence kept: every arm is
                           a real divergent branch in SASS (BSSY/@P BRA/BSYNC) */
#define DARM_MELDED 1   /* control flow emitted by runDarm   */
#define DARM_PREDICATED 2 /* original CFG as ptxas compiles it (short arms
                           if-converted into predicated runs): corpus kernels,
                           bitonic and PCM sorts                               */
#define DARM_MELDED_LITERAL 3 /* bitonic sorts only: SURVEY App. A.2 as printed
                           (select chain on `up`, one store), next to
                           DARM_MELDED's order-flip form                        */

#define DARM_MEM_HOST 0
#define DARM_MEM_DEVICE 1

typedef struct darm_gpu_stats {
  double kernel_ms;      /* device time of this call's kernel launches        */
  double h2d_ms;         /* HOST mode: host->device copies                     */
  double d2h_ms;         /* HOST mode: device->host copies                     */
  double total_ms;       /* first event to last event on `stream`              */
  uint64_t h2d_bytes;
  uint64_t d2h_bytes;
  uint64_t algorithmic_bytes; /* minimal HBM bytes the kernels must move      */
  int32_t launches;      /* kernels launched by this call                      */
  int32_t reserved;      /* call-specific (bitonic: keys per thread used)      */
} darm_gpu_stats;

/* ---- runtime ------------------------------------------------------------ */

/* Number of visible CUDA devices; fails with DARM_INTERNAL_ERROR when the
 * driver has no device (there is no CPU fallback). */
int darm_gpu_init(int *n_devices, char *err, size_t errlen);

int darm_gpu_abi_version(void);

/* Releases cached device buffers on every device. */
void darm_gpu_shutdown(void);

/* ---- corpus metadata ---------------------------------------------------- */

/* Kernel declaration as written in proj/corpus/<kernel>.ir: parameters
 * (fn <name>(%p, ...)), globals (global <name>[size]) and shared decls
 * (shared <name>[size]).  Writes JSON
 *   {"name":..,"params":[..],"globals":[[name,size],..],"shared":[[name,size],..]}
 * Returns the length needed including the terminator (0 = unknown kernel). */
size_t darm_gpu_kernel_info(const char *kernel, char *out, size_t outlen);

/* Comma-separated list of kernels darm_gpu_execute_warps accepts. */
const char *darm_gpu_kernel_list(void);

/* ---- fixtures: replaces makeRandomInput (include/darm/fixtures.hpp:28-29,
 *      src/fixtures.cpp:82-108) for n_warps consecutive seeds --------------
 * Warp w gets exactly makeRandomInput(module, fn, warp, seed0 + w) (mt19937_64,
 * params named j*|k* -> power of two <= warp, others -> [0, 2*warp), memory
 * words -> rng() % 257 - 128), laid out for darm_gpu_execute_warps:
 *   args[p * n_warps + w]               (n_params x n_warps)
 *   globals[g][w * gstride + i], i < gstride <= declared size (the rest of
 *                                        the declared words is generated and
 *                                        dropped, keeping the stream aligned)
 *   shared[s][w * size_s + i]           (declared size; NULL pointers skip)
 * Host memory only; multi-threaded over warps. */
int darm_gpu_make_random_input(const char *kernel, int warp, int64_t n_warps,
                               uint64_t seed0, int32_t *args,
                               int32_t *const *globals, int64_t gstride,
                               int32_t *const *shared, char *err, size_t errlen);

/* ---- replaces executeWarp (include/darm/interp.hpp:57-58,
 *      src/interp.cpp:332-381) for a batch of independent warps ----------
 * Runs `n_warps` warps of `warp` lanes (1..64) of corpus kernel `kernel` in
 * the given form.  Lane t of warp w is global lane g = w*warp + t; `tid`
 * returns t (interp.cpp:206-208).
 *   args:    n_params x acount int32; acount = 1 (broadcast, interp.cpp:346-354),
 *            n_warps (one value per warp) or n_warps*warp (per lane).
 *   globals: one array per declared global, in declaration order, each
 *            n_warps*warp words: word g is element t of warp w's array (every
 *            corpus kernel indexes its globals by %t).  In/out: the final
 *            contents are written back (WarpResult::globalFinal).
 *   shared:  one array per shared decl, n_warps*declared-size words (shared
 *            initialisers, WarpInput::sharedInit); NULL = zero-filled.
 *            Not written back (compareRuns ignores shared memory,
 *            interp.cpp:415-424).
 *   faults:  n_warps int32 (may be NULL): lanes that faulted (out-of-bounds
 *            shared access; WarpResult::faults.size()).
 * Corpus kernels return void, so WarpResult::returns is all-nullopt. */
int darm_gpu_execute_warps(const char *kernel, int variant, int warp,
                           int64_t n_warps, const int32_t *args, int64_t acount,
                           int32_t *const *globals, int n_globals,
                           const int32_t *const *shared, int n_shared,
                           int32_t *faults, int mem, void *stream,
                           darm_gpu_stats *stats, char *err, size_t errlen);

/* ---- bitonic sort: the corpus compare-exchange step (corpus/bitonic.ir:6-43)
 *      chained over every stage dir = 2..bucket and stride k = dir/2..1 -------
 * Sorts each of the n/bucket consecutive buckets ascending, in place.
 * bucket: power of two in [2, 4096]; n % bucket == 0.  The chained-step
 * semantics equal the reference driver's executeWarp chain for bucket <= 64
 * (oracle: oracle/ref_shim.cpp ref_bitonic_sort); larger buckets are pinned by
 * sortedness and the C restatement. */
int darm_gpu_bitonic_sort(int variant, int32_t *keys, int64_t n, int bucket,
                          int mem, void *stream, darm_gpu_stats *stats,
                          char *err, size_t errlen);

/* Same, choosing how many IR lanes (keys) one hardware thread carries:
 *   1        one key per thread: an IR warp of `bucket` lanes is `bucket`
 *            threads (the shape the reference interpreter runs; bucket <= 1024);
 *   4, 8, 16 register-blocked: a thread holds that many consecutive keys of a
 *            bucket, strides below it are exchanged inside the thread, across
 *            threads of a warp by shuffles, across warps (buckets over
 *            32 * keys_per_thread) through shared memory (needs
 *            bucket / keys_per_thread <= 256, 16-byte aligned keys);
 *   0        the fastest supported (what darm_gpu_bitonic_sort uses).
 * stats->reserved receives the keys per thread used.
 * HOST mode with n >= 2^22 keys pipelines 2^21-key chunks over three internal
 * streams (copy in / sort / copy out overlap); then h2d_ms is the time to the
 * first chunk's sort, kernel_ms the span of the sorts, d2h_ms the rest. */
int darm_gpu_bitonic_sort_ex(int variant, int32_t *keys, int64_t n, int bucket,
                             int keys_per_thread, int mem, void *stream,
                             darm_gpu_stats *stats, char *err, size_t errlen);

/* ---- PCM: Batcher odd-even merge sort of buckets (the
 *      reference has no PCM code) — paper_2107_05681_b200/ir/oddeven_step.ir
 *      chained over p = 1..bucket/2, k = p..1 ----------------------------------
 * Sorts each of the n/bucket consecutive buckets ascending, in place; the
 * arguments, shapes (keys_per_thread), HOST-mode pipelining and stats are those
 * of darm_gpu_bitonic_sort_ex, with bucket <= 1024 and
 * bucket / keys_per_thread <= 32 (a bucket stays inside a warp).  The chained-step semantics equal the
 * reference interpreter's executeWarp chain of the IR step for bucket <= 64
 * (oracle: oracle/ref_shim.cpp ref_chain_sort). */
int darm_gpu_oddeven_sort(int variant, int32_t *keys, int64_t n, int bucket,
                          int keys_per_thread, int mem, void *stream,
                          darm_gpu_stats *stats, char *err, size_t errlen);

/* ---- MS: bottom-up merge sort of the whole array (the
 *      reference has no MS code) — the merge loop of
 *      paper_2107_05681_b200/ir/merge_step.ir, passes w = 1, 2, 4, .. < n ----
 * Sorts keys[0..n) ascending in place (0 <= n < 2^30).  The chained-step
 * semantics equal the reference interpreter running the IR loop to a fixpoint
 * per pass for n <= 1024 (oracle: tests/golden/merge_sort.json).  The pass
 * sequence is recorded once per (keys, n, variant) as a CUDA graph. */
int darm_gpu_merge_sort(int variant, int32_t *keys, int64_t n, int mem,
                        void *stream, darm_gpu_stats *stats, char *err,
                        size_t errlen);

/* ---- N-Queens (NQU; the reference has no code for it):
 *      paper_2107_05681_b200/ir/nqueens_sym.ir run to completion per thread -
 * Counts the placements of n non-attacking queens on an n x n board (2 <= n
 * <= 31).  The search space is split into the valid placements of the first
 * prefix_rows rows (1 <= prefix_rows <= n-1), enumerated lowest free column
 * first; this call solves the prefixes i with i % world == rank (one rank per
 * GPU; the caller sums `solutions` over ranks).  per_prefix (optional, host,
 * >= *n_prefixes entries) receives each prefix's count in enumeration order.
 * Host-in/host-out; the call returns after the result is on the host. */
int64_t darm_gpu_nqueens_prefix_count(int n, int prefix_rows, int rank, int world); /* -1: bad args */

int darm_gpu_nqueens(int variant, int n, int prefix_rows, int rank, int world,
                     uint64_t *solutions, uint32_t *per_prefix, int64_t per_prefix_len,
                     int64_t *n_prefixes, void *stream, darm_gpu_stats *stats,
                     char *err, size_t errlen);

/* Same, with flags: DARM_NQ_MIRROR counts by mirror symmetry — the row-0 queen
 * only in columns < ceil(n/2), those left of the middle counted twice — which
 * halves the search; the prefix set (and per_prefix) is then the reduced one. */
#define DARM_NQ_MIRROR 1
/* DARM_NQ_PAPER_SHAPE runs the search loop in the shape the paper names
 * (ir/nqueens_step.ir: pop / count a leaf / push, an if-then-elseif-then
 * section that runDarm melds by region replication — two block-region melds)
 * instead of the symmetric push/pop encoding (ir/nqueens_sym.ir); n <= 16.
 * Same counts, per prefix and in total. */
#define DARM_NQ_PAPER_SHAPE 2
int darm_gpu_nqueens_ex(int variant, int n, int prefix_rows, int rank, int world,
                        int flags, uint64_t *solutions, uint32_t *per_prefix,
                        int64_t per_prefix_len, int64_t *n_prefixes, void *stream,
                        darm_gpu_stats *stats, char *err, size_t errlen);
int64_t darm_gpu_nqueens_prefix_count_ex(int n, int prefix_rows, int rank, int world,
                                         int flags);

/* ---- LUD (Rodinia lud, no reference code): blocked LU
 *      decomposition without pivoting, BLOCK = 16, in place ----------------
 * a: n x n row-major fp32 (n % 16 == 0, 16 <= n <= 46336); on return the
 * strictly lower part holds L (unit diagonal implied) and the upper part U.
 * Diagonal, perimeter (the melded kernel) and internal launches for every
 * 16-column step are replayed from a cached CUDA graph.  DEVICE pointers must
 * be 16-byte aligned.  Operation order is fixed, so the
 * result is identical for both forms and across runs. */
int darm_gpu_lud(int variant, float *a, int64_t n, int mem, void *stream,
                 darm_gpu_stats *stats, char *err, size_t errlen);

/* ---- SRAD (Rodinia SRAD, no reference code) -------------
 * Speckle reducing anisotropic diffusion of a rows x cols fp32 image J for
 * `iters` iterations with step lambda; q0sqr of every iteration comes from the
 * ROI roi = {r1, r2, c1, c2} (inclusive, at most 4096 rows).  Per-pixel
 * operations are fixed and deterministic.  One fused kernel
 * per iteration (8 B/px of HBM traffic), all iterations in one cached graph.
 * J is updated in place (HOST: copied in/out; DEVICE: device pointer). */
/* SRAD only: OR into `variant` to compute the five divisions per pixel as
 * reciprocal-multiplies and contract the sums of products into FMAs; the
 * image then agrees with the IEEE path (and the oracle) within 1e-5
 * relative, the tolerance BASELINE.json's north star states for SRAD, instead
 * of bit for bit. */
#define DARM_FAST_MATH 0x100
int darm_gpu_srad(int variant, float *j, int64_t rows, int64_t cols, int iters,
                  float lambda, const int *roi, int mem, void *stream,
                  darm_gpu_stats *stats, char *err, size_t errlen);

/* Row-tiled SRAD for one rank of a multi-GPU run (device pointers only).
 * A tile holds global rows [r0, r0 + tile_rows) at local rows 1..tile_rows of
 * a (tile_rows + 3) x pitch float buffer (pitch >= cols, a multiple of 4;
 * 16-byte aligned): local row 0 is the halo row r0 - 1 and local rows
 * tile_rows+1, tile_rows+2 the halo rows below (needed only where they exist
 * in the image; the caller exchanges them between ranks).
 * ROI partial sums: darm_gpu_srad_roi_words() doubles per buffer; a tile
 * writes the entries of the ROI rows it owns, so summing the buffers of all
 * ranks (e.g. an all-reduce) gives the full statistics.
 * tile_roi() fills roi_out for the initial image; tile_step() runs one
 * iteration tile_in -> tile_out using roi_in and writes the next roi_out.
 * `part` splits an iteration so the halo exchange overlaps compute:
 * DARM_SRAD_INTERIOR_ROWS (rows 2 .. tile_rows-2, which read no halo row;
 * also computes q0sqr into q0_scratch) while the halos are in flight, then
 * DARM_SRAD_EDGE_ROWS (rows 1 and tile_rows-1 .. tile_rows) once they landed;
 * DARM_SRAD_ALL_ROWS does both at once.  q0_scratch: one device float. */
#define DARM_SRAD_ALL_ROWS 0
#define DARM_SRAD_INTERIOR_ROWS 1
#define DARM_SRAD_EDGE_ROWS 2
int64_t darm_gpu_srad_pitch(int64_t cols);
int64_t darm_gpu_srad_roi_words(int64_t cols, const int *roi);
int darm_gpu_srad_tile_roi(const float *tile, int64_t cols, int64_t pitch,
                           int64_t tile_rows, int64_t r0, int64_t rows,
                           const int *roi, double *roi_out, void *stream,
                           char *err, size_t errlen);
int darm_gpu_srad_tile_step(int variant, const float *tile_in, float *tile_out,
                            int64_t cols, int64_t pitch, int64_t tile_rows,
                            int64_t r0, int64_t rows, float lambda,
                            const int *roi, const double *roi_in,
                            double *roi_out, float *q0_scratch, int part,
                            void *stream, char *err, size_t errlen);

/* Peer-memory row-tiled SRAD: the multi-GPU product path (one process per
 * GPU, one group per rank).  Instead of a collective library, a rank reads its
 * halo rows and the ROI partial sums straight out of its neighbours' memory
 * (CUDA IPC mappings over NVLink / NVSwitch) and the ranks keep phase with
 * flags in device memory: after the load and after every iteration a rank
 * publishes its phase count into every rank's flag array; before a phase it
 * waits on the GPU until all peers reached its own count.  An iteration is:
 * wait, halo pull (side stream) beside the interior rows, edge rows, signal —
 * all `iters` iterations one cached CUDA graph.  Results are bit-identical to
 * darm_gpu_srad() on the whole image.
 *   create:  allocate this rank's tile (global rows split as evenly as in
 *            paper_2107_05681_b200.srad_tiles.split_rows) and write its
 *            DARM_SRAD_HANDLE_BYTES-byte handle;
 *   connect: give every rank's handle (rank order); peers in another process
 *            are opened by CUDA IPC, in this process used directly;
 *   load:    this rank's rows (tile_rows x cols, row-major) -> the tile;
 *   run:     `iters` iterations (asynchronous on `stream`);
 *   read:    the tile's rows out; returns 3 if a peer never arrived (a device
 *            wait gives up after DARM_PEER_TIMEOUT_S seconds, default 60).
 * Every rank must call load / run with the same sequence of arguments. */
#define DARM_SRAD_HANDLE_BYTES 128
typedef struct darm_gpu_srad_group darm_gpu_srad_group;
int darm_gpu_srad_group_create(int variant, int64_t rows, int64_t cols, float lambda,
                               const int *roi, int rank, int world,
                               darm_gpu_srad_group **out, void *handle_out,
                               char *err, size_t errlen);
int darm_gpu_srad_group_connect(darm_gpu_srad_group *group, const void *handles,
                                char *err, size_t errlen);
int darm_gpu_srad_group_load(darm_gpu_srad_group *group, const float *tile, int mem,
                             void *stream, char *err, size_t errlen);
int darm_gpu_srad_group_run(darm_gpu_srad_group *group, int iters, void *stream,
                            darm_gpu_stats *stats, char *err, size_t errlen);
int darm_gpu_srad_group_read(darm_gpu_srad_group *group, float *tile, int mem,
                             void *stream, char *err, size_t errlen);
/* this rank's first global row and row count */
int darm_gpu_srad_group_rows(const darm_gpu_srad_group *group, int64_t *r0,
                             int64_t *tile_rows);
void darm_gpu_srad_group_free(darm_gpu_srad_group *group);

/* ---- GPU executeWarp for arbitrary mini-IR -------
 * executeWarp (include/darm/interp.hpp:57-58, src/interp.cpp:332-381) for a
 * batch of warps of ANY function in the reference's textual IR (SPEC.md:
 * 111-121): the library parses and lowers the first function of `ir_text`
 * (its own reader; the reference's pass output prints in the same grammar),
 * one CUDA warp interprets one IR warp, and every result field equals the
 * reference interpreter's: per-lane returns, final global / shared memory,
 * fault counts, and the WarpExecStats counters (latencies: the reference's
 * defaults, ir.cpp:235-244, or `latency`, 28 entries in the opcode order of
 * ir.hpp:17-46).  Limits: 256 values per function, 16 phis per block, SIMT
 * stack depth 48.
 *
 * Buffers (HOST or DEVICE per `mem`):
 *   args     n_params x acount, acount = 1 (broadcast), n_warps or n_warps*warp
 *   globals  n_warps x global_words (in/out): warp w's globals in declaration
 *            order (darm_gpu_program_memory gives each array's offset / size)
 *   shared   n_warps x shared_words (in/out; NULL: zero-initialised scratch)
 *   returns / ret_valid  n_warps x warp (may be NULL): a lane's return value
 *            and whether it returned one (WarpResult::returns)
 *   faults   n_warps (may be NULL): faulted lanes (WarpResult::faults.size())
 *   stats    n_warps x 8 int64 (may be NULL): issuedInstructions, threadCycles,
 *            usefulThreadCycles, serializedCycles, divergentBranchCount,
 *            sharedMemIssues, globalMemIssues, flags (bit 0 nonTerminated,
 *            bit 1 taintedObservable)
 * max_steps <= 0 means executeWarp's default budget (10^7 issues).
 * Returns 2 for malformed IR and for the reference's execution errors (a phi
 * without an incoming for the lane's predecessor, a divergent branch without
 * a reconvergence point). */
typedef struct darm_gpu_program darm_gpu_program;
int darm_gpu_program_load(const char *ir_text, const int64_t *latency,
                          darm_gpu_program **out, char *err, size_t errlen);
void darm_gpu_program_free(darm_gpu_program *program);
int darm_gpu_program_shape(const darm_gpu_program *program, int *n_params,
                           int *n_globals, int *n_shared, int64_t *global_words,
                           int64_t *shared_words);
/* memory `index` (globals, then shared arrays): name, or NULL past the end */
const char *darm_gpu_program_memory(const darm_gpu_program *program, int index,
                                    int64_t *size, int64_t *offset, int *is_shared);
const char *darm_gpu_program_param(const darm_gpu_program *program, int index);
int darm_gpu_program_execute(darm_gpu_program *program, int warp, int64_t n_warps,
                             const int32_t *args, int64_t acount,
                             int32_t *globals, int32_t *shared,
                             int32_t *returns, uint8_t *ret_valid,
                             int32_t *faults, int64_t *stats_out,
                             int64_t max_steps, int mem, void *stream,
                             darm_gpu_stats *stats, char *err, size_t errlen);

#ifdef __cplusplus
}
#endif

#endif /* DARM_GPU_H */
