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
cudaError_t launch_bitonic_sort(int variant, int32_t *keys, int64_t n, int bucket, cudaStream_t s,
                                int *launches);

// nqueens.cu
cudaError_t launch_nqueens(int variant, const uint32_t *prefix, uint32_t n_prefix, int n, int base,
                           uint32_t *per_prefix, unsigned long long *total, unsigned int *counter,
                           int sms, cudaStream_t s);

// lud.cu: records the 3 x n/16 launches of one decomposition on `s`
cudaError_t record_lud(int variant, float *a, int n, cudaStream_t s, int *launches);

}  // namespace darm_gpu
