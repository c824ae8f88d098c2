// bitonic_sort.cu — batched bucket sort built from the corpus compare-exchange
// step (corpus/bitonic.ir:6-43), in its unmelded and melded forms.
//
// The reference sorts a bucket by chaining executeWarp over the step kernel:
// one warp of B lanes, lane t owns buf[t], reads its partner buf[t^k], and keeps
// the smaller/larger key depending on keep = t < t^k and up = (t & dir) == 0,
// for dir = 2..B and k = dir/2..1 (oracle/ref_shim.cpp ref_bitonic_sort).
//
// On sm_100a each bucket is B consecutive threads and lane t's slot lives in a
// register for the whole network:
//   - partner read  k <  32: __shfl_xor_sync (the partner is in the same warp)
//                   k >= 32: one exchange through double-buffered shared memory
//                            (one __syncthreads per exchange)
//   - the divergent `if (up)` of the step (bitonic.ir:16) is a real branch in
//     the unmelded form and the select chain of SURVEY App. A.2 in the melded
//     form (bitonic_exchange in corpus.cuh).
// HBM traffic is one coalesced read and one coalesced write per key (8 B/key);
// CTAs are persistent and prefetch their next tile while running the network.
#include <climits>

#include "corpus.cuh"
#include "kernels.h"

namespace darm_gpu {

template <int B>
struct Network {
  static constexpr int kSteps = __builtin_ctz(B) * (__builtin_ctz(B) + 1) / 2;
  static_assert(kSteps <= 64, "step masks are 64-bit");
};

template <bool M, int B, int CTA, int U>
__global__ void __launch_bounds__(CTA) bitonic_sort_kernel(int32_t *__restrict__ keys, uint32_t n) {
  constexpr int LB = __builtin_ctz(B);
  constexpr bool kNeedSmem = B > 32;
  __shared__ int32_t xch[kNeedSmem ? 2 : 1][U][kNeedSmem ? CTA : 1];
  const uint32_t tiles = (n + CTA - 1) / CTA;
  const int t = int(threadIdx.x) & (B - 1);
  // Lane-invariant bits of t (loop-invariant across tiles, kept in predicate
  // registers): keep = icmp.lt %t %j <=> !bit[log k], up = icmp.eq (and %t
  // %dir) 0 <=> !bit[log dir].
  bool bit[LB > 0 ? LB : 1];
#pragma unroll
  for (int i = 0; i < LB; ++i) bit[i] = (t >> i) & 1;
  // U independent tiles per iteration (tile, tile + G, ...): their
  // shuffle -> compare -> select chains interleave and hide each other's latency.
  const uint32_t G = gridDim.x;
  uint32_t tile = blockIdx.x;
  int32_t next[U];
#pragma unroll
  for (int u = 0; u < U; ++u) {
    const uint32_t tt = tile + u * G, id = tt * CTA + threadIdx.x;
    next[u] = (tt < tiles && id < n) ? keys[id] : INT_MAX;
  }
  for (; tile < tiles; tile += U * G) {
    int32_t v[U];
    uint32_t my[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      v[u] = next[u];
      my[u] = (tile + u * G) * CTA + threadIdx.x;
      const uint32_t tn = tile + (U + u) * G, id = tn * CTA + threadIdx.x;
      if (tn < tiles) next[u] = id < n ? keys[id] : INT_MAX;   // prefetch
    }
    int par = 0;
    int32_t neg = 0;   // melded: lanes of a descending half work on ~v (order reversal)
#pragma unroll
    for (int d = 1; d <= LB; ++d) {
      if constexpr (M) {
        // melded `select %up`: within stage dir = 2^d the !up lanes flip their
        // keys' order once (bitwise not), so every lane's exchange is the up-form
        const int32_t m = (d < LB && bit[d]) ? -1 : 0;
#pragma unroll
        for (int u = 0; u < U; ++u) v[u] ^= m ^ neg;
        neg = m;
      }
#pragma unroll
      for (int kb = d - 1; kb >= 0; --kb) {
        const int k = 1 << kb;
        int32_t b0[U];
        if (k < 32) {
#pragma unroll
          for (int u = 0; u < U; ++u) b0[u] = __shfl_xor_sync(0xffffffffu, v[u], k);   // load.shared buf %j
        } else {
#pragma unroll
          for (int u = 0; u < U; ++u) xch[par][u][threadIdx.x] = v[u];
          __syncthreads();
#pragma unroll
          for (int u = 0; u < U; ++u) b0[u] = xch[par][u][threadIdx.x ^ k];
          par ^= 1;
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
          if constexpr (!M) {
            v[u] = bitonic_exchange<false>(v[u], b0[u], !bit[kb], d >= LB ? true : !bit[d], false);
          } else {
            // need1 = (keep == up) ? cv > b0 : cv < b0 with up folded into the data:
            // take the partner's key iff (b0 < cv) xor !keep   (equal keys: either)
            const bool take = (b0[u] < v[u]) ^ bit[kb];
            v[u] = take ? b0[u] : v[u];                       // ^e.m: the single melded store
          }
        }
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if constexpr (M) v[u] ^= neg;
      if (tile + u * G < tiles && my[u] < n) keys[my[u]] = v[u];
    }
  }
}

namespace {

int g_sms = 0;

template <bool M, int B>
cudaError_t launch_b(int32_t *keys, int64_t n, cudaStream_t s) {
  constexpr int CTA = B > 256 ? B : 256;
  if (!g_sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_sms, cudaDevAttrMultiProcessorCount, dev);
    if (g_sms <= 0) g_sms = 148;
  }
  constexpr int U = B <= 256 ? 2 : 1;
  const int64_t tiles = (n + CTA - 1) / CTA;
  const int per_sm = 2048 / CTA;
  int64_t grid = int64_t(g_sms) * per_sm;
  if (grid > (tiles + U - 1) / U) grid = (tiles + U - 1) / U;
  if (grid < 1) grid = 1;
  bitonic_sort_kernel<M, B, CTA, U><<<int(grid), CTA, 0, s>>>(keys, uint32_t(n));
  return cudaGetLastError();
}

template <bool M>
cudaError_t launch_m(int32_t *keys, int64_t n, int bucket, cudaStream_t s) {
  switch (bucket) {
    case 2: return launch_b<M, 2>(keys, n, s);
    case 4: return launch_b<M, 4>(keys, n, s);
    case 8: return launch_b<M, 8>(keys, n, s);
    case 16: return launch_b<M, 16>(keys, n, s);
    case 32: return launch_b<M, 32>(keys, n, s);
    case 64: return launch_b<M, 64>(keys, n, s);
    case 128: return launch_b<M, 128>(keys, n, s);
    case 256: return launch_b<M, 256>(keys, n, s);
    case 512: return launch_b<M, 512>(keys, n, s);
    case 1024: return launch_b<M, 1024>(keys, n, s);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace

bool bitonic_sort_supported(int bucket) {
  return bucket >= 2 && bucket <= 1024 && (bucket & (bucket - 1)) == 0;
}

cudaError_t launch_bitonic_sort(int variant, int32_t *keys, int64_t n, int bucket, cudaStream_t s,
                                int *launches) {
  if (n == 0) return cudaSuccess;
  if (launches) *launches += 1;
  return variant ? launch_m<true>(keys, n, bucket, s) : launch_m<false>(keys, n, bucket, s);
}

}  // namespace darm_gpu
