// kernels.h — internal registry between the C-ABI (runtime.cu) and the kernel
// translation units.  Not part of the public boundary (include/darm_gpu.h).
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace darm_gpu {

struct CorpusParams;

struct MemDeclDesc {
  const char *name;
  int size;  // declared words (global <name>[size] / shared <name>[size])
};

using CorpusLaunch = cudaError_t (*)(int variant, int arg_mode, const CorpusParams &P, int sms,
                                     cudaStream_t s);

struct CorpusKernelDesc {
  const char *name;
  const char *params[4];
  int n_params;
  MemDeclDesc globals[4];
  int n_globals;
  MemDeclDesc shared[1];
  int n_shared;
  int lane_bytes;  // minimal global bytes per lane (algorithmic traffic)
  CorpusLaunch launch;
};

extern const CorpusKernelDesc kCorpus[];
extern const int kCorpusCount;

// bitonic_sort.cu
bool bitonic_sort_supported(int bucket);
// resolves keys_per_thread (0 = auto) for this bucket / pointer, at most
// max_threads threads per bucket; -1 = unsupported
int bitonic_keys_per_thread(int bucket, int keys_per_thread, const void *keys, int max_threads);
cudaError_t launch_bitonic_sort(int variant, int32_t *keys, int64_t n, int bucket, int keys_per_thread,
                                cudaStream_t s, int *launches);

// oddeven_sort.cu (PCM): keys_per_thread already resolved by bitonic_keys_per_thread
cudaError_t launch_oddeven_sort(int variant, int32_t *keys, int64_t n, int bucket, int keys_per_thread,
                                cudaStream_t s, int *launches);

// merge_sort.cu (MS): bottom-up merge sort of keys[0..n) (tmp: n-key scratch)
cudaError_t record_merge_sort(int variant, int32_t *keys, int32_t *tmp, int64_t n, cudaStream_t s, int *launches);
int merge_sort_passes(int64_t n);   // global passes over the array, incl. the tile pass

// interp.cu: the GPU executeWarp over a lowered mini-IR program (ir_program.h)
struct InterpLaunch {
  const void *blocks, *insts, *phis, *phi_ins;   // device copies of the IrProgram arrays
  const int64_t *mem_off, *mem_size;
  const uint8_t *mem_shared;
  int64_t latency[28];
  int n_params, n_regs, entry, ret_block;
  int64_t gwords, swords;
  int W;
  int64_t n_warps;
  int am;
  const int32_t *args;
  int64_t acount;
  int32_t *globals, *shared;
  uint8_t *taint;
  int32_t *returns;
  uint8_t *ret_valid;
  int32_t *faults;
  int64_t *stats;
  int32_t *errors;
  int64_t max_steps;
  int sms;
};
cudaError_t launch_ir_interp(const InterpLaunch &L, cudaStream_t s);
int ir_interp_max_regs();
int ir_interp_max_phis();

// nqueens.cu
cudaError_t launch_nqueens(int variant, const uint32_t *prefix, uint32_t n_prefix, uint32_t n_double, int n, int base,
                           uint32_t *per_prefix, unsigned long long *total, unsigned int *counter,
                           int sms, cudaStream_t s, bool paper_shape = false);

// lud.cu: records the launches of one decomposition on `s`; dscr: 256-float
// device scratch for the factored diagonal block
cudaError_t record_lud(int variant, float *a, int n, float *dscr, int *counters, cudaStream_t s, int *launches);
int lud_counter_words(int n);   // ints of `counters` record_lud uses

// srad.cu
struct SradRoi {
  int r1, r2, c1, c2;   // inclusive ROI rectangle (global rows / columns)
  int w0, groups;       // warp column groups (128 columns each) covering [c1, c2]
  int rows;             // r2 - r1 + 1
};
// own rows (0-based, within a tile) one sweep launch computes: [lo0, hi0) then [lo1, hi1)
struct SradRange {
  int lo0, hi0, lo1, hi1;
};
SradRoi srad_roi_layout(int cols, int r1, int r2, int c1, int c2);
int srad_pitch(int cols);   // row pitch (floats) of the library's own buffers: a multiple of 4
cudaError_t launch_srad_roi(const float *jin, int cols, int pitch, int r0, int tile_rows, const SradRoi &roi,
                            double *roi_out, cudaStream_t s);
// One SRAD iteration over `range` of a tile: every warp derives q0sqr from the
// ROI partials of J (roi_in; or, multi-GPU, roi_parts[roi_owner[row]] per ROI
// row), computes J -> J' and the ROI partials of J' (roi_out, may be null);
// q0_out (optional) receives q0sqr.
cudaError_t launch_srad_sweep(int variant, const float *jin, float *jout, const double *roi_in, float *q0_out,
                              double *roi_out, int cols, int pitch, int tile_rows, int r0, int R, float lambda,
                              const SradRoi &roi, const SradRange &range, cudaStream_t s,
                              const double *const *roi_parts = nullptr, const int *roi_owner = nullptr);
// peer-memory row tiles (darm_gpu_srad_group_*): phase barrier, phase signal, halo pull
cudaError_t launch_srad_peer_wait(const unsigned *flags, const unsigned *seq, int rank, int world,
                                  unsigned long long timeout_ns, int *status, cudaStream_t s);
cudaError_t launch_srad_peer_signal(unsigned *const *peer_flags, unsigned *seq, int rank, int world, cudaStream_t s);
cudaError_t launch_srad_peer_halo(float *dst, const float *up, int up_rows, const float *down, int n, int pitch,
                                  cudaStream_t s);

}  // namespace darm_gpu
