// corpus.cu — batched executeWarp for the corpus kernels on sm_100a.
//
// Replaces the reference runtime path executeWarp (interp.cpp:332-381) for the
// corpus kernels: instead of interpreting the IR lane by lane, every IR lane is
// one hardware thread and every IR warp of W=32 lanes is exactly one hardware
// warp, so the divergence the interpreter models (IPDOM reconvergence,
// interp.cpp:285-308) is the divergence the SM executes.
#include "corpus.cuh"
#include "kernels.h"

namespace darm_gpu {

// ------------------------------------------------------------------ lanes
// Grid-stride over lanes.  AM = argument mode: 0 broadcast, 1 per warp,
// 2 per lane (interp.cpp:346-354 allows 1 or warpSize values per parameter;
// batching adds the per-warp case).
template <class K, int F, int WT, int AM>
__global__ void __launch_bounds__(256) corpus_lanes(CorpusParams P) {
  const uint32_t stride = gridDim.x * blockDim.x;
  for (uint32_t g = blockIdx.x * blockDim.x + threadIdx.x; g < P.total; g += stride) {
    uint32_t w;
    int t;
    LaneSplit<WT>::split(g, P.warp, w, t);
    int32_t a[K::kParams];
#pragma unroll
    for (int p = 0; p < K::kParams; ++p)
      a[p] = AM == 0 ? P.argv[p] : (AM == 1 ? __ldg(P.argp[p] + w) : __ldg(P.argp[p] + g));
    K::template lane<F>(P, g, t, a);
  }
}

// ------------------------------------------------------------------ bitonic step
// bitonic.ir:6-43 with `buf` in shared memory exactly as the IR declares it
// (shared buf[64] per warp): each CTA holds `wpc` IR warps, stages their
// shared initialisers with coalesced loads, runs one step, writes res[t].
// A lane whose partner index t^k falls outside buf faults (interp.cpp:251-256)
// and does nothing else.  The barrier between the partner loads and the
// divergent stores restores the interpreter's lockstep order.
template <int F, int WT, int AM>
__global__ void __launch_bounds__(256) bitonic_step_kernel(CorpusParams P) {
  constexpr bool M = F == kMelded;
  extern __shared__ int32_t smem[];
  const uint32_t W = WT > 0 ? uint32_t(WT) : P.warp;
  const uint32_t S = P.shared_size;
  const uint32_t wpc = blockDim.x / W;
  int32_t *__restrict__ res = P.gl[0];
  for (uint32_t w0 = blockIdx.x * wpc; w0 < P.n_warps; w0 += gridDim.x * wpc) {
    const uint32_t nw = min(wpc, P.n_warps - w0);
    for (uint32_t i = threadIdx.x; i < nw * S; i += blockDim.x)
      smem[i] = P.sh ? P.sh[size_t(w0) * S + i] : 0;
    __syncthreads();
    uint32_t lw;
    int t;
    LaneSplit<WT>::split(threadIdx.x, W, lw, t);
    const uint32_t w = w0 + lw;
    const bool live = lw < nw;
    const uint32_t g = w * W + uint32_t(t);
    int32_t *buf = smem + lw * S;
    int32_t k = 0, dir = 0;
    if (live) {
      k = AM == 0 ? P.argv[0] : (AM == 1 ? P.argp[0][w] : P.argp[0][g]);
      dir = AM == 0 ? P.argv[1] : (AM == 1 ? P.argp[1][w] : P.argp[1][g]);
    }
    // ^a :7-14
    const int32_t j = t ^ k;
    const bool fault = live && uint32_t(j) >= S;
    const bool run = live && !fault;
    int32_t b0 = run ? buf[j] : 0;
    if (fault && P.faults) atomicAdd(P.faults + w, 1);
    const bool keep = t < j;
    const bool up = (t & dir) == 0;
    int32_t cv = 0;
    if constexpr (M) cv = run ? buf[t] : 0;                // melded ^a hoists load.shared buf %t
    __syncthreads();
    if (run) {
      if constexpr (!M) {
        if (up) {                                          // ^b condbr %up ^c ^d
          DARM_ARM_F(F, "bstep.c");
          int32_t c0 = buf[t];                             // ^c load.shared buf %t
          bool need1 = keep ? (c0 > b0) : (c0 < b0);
          if (need1) {
            DARM_ARM_F(F, "bstep.e");
            buf[t] = b0;                                   // ^e store.shared
          }
          DARM_ARM("bstep.x1");
        } else {
          DARM_ARM_F(F, "bstep.d");
          int32_t dv = buf[t];                             // ^d load.shared buf %t
          bool need2 = keep ? (dv < b0) : (dv > b0);
          if (need2) {
            DARM_ARM_F(F, "bstep.f");
            buf[t] = b0;                                   // ^f store.shared
          }
          DARM_ARM("bstep.x2");
        }
      } else {
        bool lt2 = false, lt1 = false;
        if (!up) lt2 = cv < b0;
        bool gt1 = cv > b0;
        if (up) lt1 = cv < b0;
        bool need1 = keep ? (up ? gt1 : lt2) : (up ? lt1 : gt1);
        if (need1) buf[t] = b0;                            // ^e.m single melded store
      }
      res[g] = buf[t];                                     // ^g :39-42
    }
    __syncthreads();
  }
}

// ------------------------------------------------------------------ dispatch
namespace {

int grid_for(uint64_t work, int per_cta, int sms) {
  uint64_t ctas = (work + per_cta - 1) / per_cta;
  uint64_t cap = uint64_t(sms) * 8;  // 8 x 256-thread CTAs = 2048 threads per SM
  if (ctas > cap) ctas = cap;
  return int(ctas < 1 ? 1 : ctas);
}

template <class K, int F, int WT>
cudaError_t launch_lanes_am(int am, const CorpusParams &P, int sms, cudaStream_t s) {
  // One thread per lane: every lane's loads are in flight at once (the kernels
  // are latency/HBM-bound and a lane does a handful of instructions).
  (void)sms;
  const int grid = int((uint64_t(P.total) + 255) / 256);
  switch (am) {
    case 0: corpus_lanes<K, F, WT, 0><<<grid, 256, 0, s>>>(P); break;
    case 1: corpus_lanes<K, F, WT, 1><<<grid, 256, 0, s>>>(P); break;
    default: corpus_lanes<K, F, WT, 2><<<grid, 256, 0, s>>>(P); break;
  }
  return cudaGetLastError();
}

template <class K, int F>
cudaError_t launch_lanes_w(int am, const CorpusParams &P, int sms, cudaStream_t s) {
  switch (P.warp) {
    case 32: return launch_lanes_am<K, F, 32>(am, P, sms, s);
    case 64: return launch_lanes_am<K, F, 64>(am, P, sms, s);
    default: return launch_lanes_am<K, F, 0>(am, P, sms, s);
  }
}

template <class K>
cudaError_t launch_lanes(int variant, int am, const CorpusParams &P, int sms, cudaStream_t s) {
  switch (variant) {
    case kUnmelded: return launch_lanes_w<K, kUnmelded>(am, P, sms, s);
    case kMelded: return launch_lanes_w<K, kMelded>(am, P, sms, s);
    default: return launch_lanes_w<K, kPredicated>(am, P, sms, s);
  }
}

template <int F, int WT>
cudaError_t launch_bstep_am(int am, const CorpusParams &P, int sms, cudaStream_t s) {
  // IR warps per CTA: up to 256 lanes, and at most 48 KB of shared `buf`
  // slices (the default dynamic shared-memory limit).
  uint32_t wpc = P.warp >= 256 ? 1 : 256 / P.warp;
  const uint32_t cap = (48u << 10) / (4u * (P.shared_size ? P.shared_size : 1));
  if (wpc > cap) wpc = cap;
  const int block = int(wpc * P.warp);
  const int grid = grid_for(P.n_warps, int(wpc), sms);
  const size_t shm = size_t(wpc) * P.shared_size * sizeof(int32_t);
  switch (am) {
    case 0: bitonic_step_kernel<F, WT, 0><<<grid, block, shm, s>>>(P); break;
    case 1: bitonic_step_kernel<F, WT, 1><<<grid, block, shm, s>>>(P); break;
    default: bitonic_step_kernel<F, WT, 2><<<grid, block, shm, s>>>(P); break;
  }
  return cudaGetLastError();
}

template <int F>
cudaError_t launch_bstep_w(int am, const CorpusParams &P, int sms, cudaStream_t s) {
  switch (P.warp) {
    case 32: return launch_bstep_am<F, 32>(am, P, sms, s);
    case 64: return launch_bstep_am<F, 64>(am, P, sms, s);
    default: return launch_bstep_am<F, 0>(am, P, sms, s);
  }
}

cudaError_t launch_bstep(int variant, int am, const CorpusParams &P, int sms, cudaStream_t s) {
  switch (variant) {
    case kUnmelded: return launch_bstep_w<kUnmelded>(am, P, sms, s);
    case kMelded: return launch_bstep_w<kMelded>(am, P, sms, s);
    default: return launch_bstep_w<kPredicated>(am, P, sms, s);
  }
}

}  // namespace

// Declarations mirror /root/reference/proj/corpus/*.ir headers.
const CorpusKernelDesc kCorpus[] = {
    {"sb1", {"n"}, 1, {{"in", 64}, {"aux2", 64}, {"aux3", 64}, {"out", 64}}, 4, {}, 0, 12, &launch_lanes<Sb1>},
    {"sb1r", {"n"}, 1, {{"in", 64}, {"out", 64}}, 2, {}, 0, 8, &launch_lanes<Sb1r>},
    {"sb2", {"n"}, 1, {{"in", 64}, {"out", 64}}, 2, {}, 0, 8, &launch_lanes<Sb2>},
    {"sb2r", {"n"}, 1, {{"in", 64}, {"out", 64}}, 2, {}, 0, 8, &launch_lanes<Sb2r>},
    {"sb3", {"n"}, 1, {{"in", 64}, {"in2", 64}, {"out", 64}, {"out2", 64}}, 4, {}, 0, 16, &launch_lanes<Sb3>},
    {"sb3r", {"n"}, 1, {{"in", 64}, {"in2", 64}, {"out", 64}, {"out2", 64}}, 4, {}, 0, 16, &launch_lanes<Sb3r>},
    {"sb4", {"h", "q"}, 2, {{"in", 64}, {"out", 64}}, 2, {}, 0, 8, &launch_lanes<Sb4>},
    {"sb4r", {"h", "q"}, 2, {{"in", 64}, {"out", 64}}, 2, {}, 0, 8, &launch_lanes<Sb4r>},
    {"nested", {"n"}, 1, {{"in", 64}, {"out", 64}}, 2, {}, 0, 8, &launch_lanes<Nested>},
    {"bitonic", {"k", "dir"}, 2, {{"res", 64}}, 1, {{"buf", 64}}, 1, 4, &launch_bstep},
};
const int kCorpusCount = int(sizeof(kCorpus) / sizeof(kCorpus[0]));

}  // namespace darm_gpu
