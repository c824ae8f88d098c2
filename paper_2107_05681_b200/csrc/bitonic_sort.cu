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

// Order flip x ^ m for m in {0, -1} written as x * (1 + 2m) + m: one IMAD on
// the FMA pipe instead of a LOP3 on the ALU pipe, which the compare-exchanges
// (VIMNMX) saturate.
__device__ __forceinline__ int32_t flip_fma(int32_t x, int32_t m) {
  return int32_t(uint32_t(x) * uint32_t(1 + 2 * m) + uint32_t(m));
}

// bit ? max(v, b) : min(v, b) issued as a complementary predicated pair; for
// the plain select ptxas emits min; @P max (a write-after-write on one
// register in every serial step of the one-key network).
__device__ __forceinline__ int32_t select_maxmin(int32_t v, int32_t b, bool bit) {
  asm("{\n .reg .pred p;\n setp.ne.b32 p, %1, 0;\n @p max.s32 %0, %0, %2;\n @!p min.s32 %0, %0, %2;\n}"
      : "+r"(v)
      : "r"(int(bit)), "r"(b));
  return v;
}

template <int B>
struct Network {
  static constexpr int kSteps = __builtin_ctz(B) * (__builtin_ctz(B) + 1) / 2;
  static_assert(kSteps <= 64, "step masks are 64-bit");
};

template <int F, int B, int CTA, int U>
__global__ void __launch_bounds__(CTA) bitonic_sort_kernel(int32_t *__restrict__ keys, uint32_t n) {
  constexpr bool M = F == kMelded;
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
  // exchange-buffer parity runs on across tiles: a write goes to the buffer
  // the previous exchange did not read, whose last reads precede that
  // exchange's barrier (an odd exchange count per tile otherwise lets a fast
  // warp overwrite a slot a slow warp still reads)
  int par = 0;
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
    int32_t neg = 0;   // melded: lanes of a descending half work on ~v (order reversal)
#pragma unroll
    for (int d = 1; d <= LB; ++d) {
      if constexpr (M) {
        // melded `select %up`: within stage dir = 2^d the !up lanes flip their
        // keys' order once (bitwise not), so every lane's exchange is the up-form
        const int32_t m = (d < LB && bit[d]) ? -1 : 0;
#pragma unroll
        for (int u = 0; u < U; ++u) v[u] = flip_fma(v[u], m ^ neg);
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
          bucket_sync<B, CTA>();                           // the bucket's own warps only
#pragma unroll
          for (int u = 0; u < U; ++u) b0[u] = xch[par][u][threadIdx.x ^ k];
          par ^= 1;
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
          if constexpr (F == kLiteral) {
            // App. A.2 select chain, issued as the melded form's predicated pair
            const bool up = d >= LB ? true : !bit[d];
            v[u] = select_maxmin(v[u], b0[u], bit[kb] == up);
          } else if constexpr (!M) {
            v[u] = bitonic_exchange<F>(v[u], b0[u], !bit[kb], d >= LB ? true : !bit[d]);
          } else {
            // need1 = (keep == up) ? cv > b0 : cv < b0 with up folded into the data:
            // need1 = (keep == up) ? gt : lt with up folded into the data: the
            // lower slot keeps the smaller key — one predicated min/max
            v[u] = select_maxmin(v[u], b0[u], bit[kb]);   // ^e.m: the single melded store
          }
        }
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if constexpr (M) v[u] = flip_fma(v[u], neg);
      if (tile + u * G < tiles && my[u] < n) keys[my[u]] = v[u];
    }
  }
}

// ---------------------------------------------------------------------------
// Register-blocked form: each thread carries R consecutive keys of a bucket
// (R lanes of the IR warp; B/R <= 32 threads per bucket, so a bucket never
// leaves its warp).  Steps with stride k < R compare-exchange two registers of
// the same thread (min + max); steps with k >= R exchange with the thread
// lane ^ k/R (__shfl_xor_sync) and keep min or max, as the one-key form does.
// The divergent `if (up)` of the step (bitonic.ir:16) exists where up depends
// on the thread: stages dir >= R below the last one.  There the unmelded
// form branches once per step (both arms of the R-key step under the branch)
// and the melded form folds up into the data as in the one-key form (the !up
// threads flip their keys' order once per stage, so every exchange is the
// up-form).  Stages dir < R have a compile-time up per register pair: no
// branch in either form.  Loads and stores are 16-byte vectors; each warp
// sorts 32*R keys per iteration and walks the array with a grid stride, the
// next tile's keys in flight (PF) while the network runs on the current one.
// The network is bound by the ALU pipe (VIMNMX, half a warp-instruction per
// cycle per SMSP), so the melded form's order flips are IMADs (flip_fma).
template <int R>
__device__ __forceinline__ void load_keys(int32_t (&v)[R], const int32_t *__restrict__ keys, uint32_t base, uint32_t n) {
  if (base < n) {                                         // whole bucket in or out (n % B == 0)
    const int4 *src = reinterpret_cast<const int4 *>(keys + base);
    if (R % 8 == 0 && aligned32(keys)) {
#pragma unroll
      for (int q = 0; q < R / 8; ++q) ld_v8(keys + base + 8 * q, &v[8 * q]);
      return;
    }
#pragma unroll
    for (int q = 0; q < R / 4; ++q) {
      const int4 x = src[q];
      v[4 * q] = x.x;
      v[4 * q + 1] = x.y;
      v[4 * q + 2] = x.z;
      v[4 * q + 3] = x.w;
    }
  } else {
#pragma unroll
    for (int j = 0; j < R; ++j) v[j] = INT_MAX;
  }
}

template <int F, int B, int R, bool PF>
__global__ void __launch_bounds__(256, PF ? DARM_BITONIC_MIN_CTAS : 1) bitonic_sort_reg_kernel(int32_t *__restrict__ keys, uint32_t n) {
  constexpr bool M = F == kMelded;
  constexpr int LB = __builtin_ctz(B), LR = __builtin_ctz(R), P = B / R;
  static_assert(R >= 4 && R <= B && P <= 256, "R keys per thread, at most 256 threads per bucket");
  // kCta: a bucket spans warps (B > 32 R, up to 4096 keys): the CTA walks
  // 256 R-key tiles and strides k >= 32 R exchange through shared memory
  constexpr bool kCta = P > 32;
  // The CTA walks 256 R-key tiles (CTA-uniform loop: ptxas knows every shuffle
  // runs converged, no WARPSYNC around them).
  constexpr uint32_t kTile = 256u * R;
  __shared__ int32_t xch[kCta ? 2 : 1][kCta ? R : 1][kCta ? 256 : 1];   // [buffer][register][thread]: conflict-free
  const int tid = int(threadIdx.x);                     // thread index within the tile
  const int tib = tid & (P - 1);                        // thread index within the bucket
  const uint32_t units = gridDim.x;
  const uint32_t tiles = (n + kTile - 1) / kTile;
  uint32_t tile = blockIdx.x;
  int par = 0;
  const uint32_t one = gridDim.y, mone = 0u - one;   // 1 and -1, opaque (cx_pair)
  // the FMA-pipe maxima need registers the unmelded 4096-key form does not
  // have under the 64-register cap (64 B of stack: 180 -> 1490 us): at 4096
  // keys every form keeps both halves of every pair on the ALU pipe, so the
  // forms differ in control flow only
  constexpr bool kCxFma = B < 4096;
  constexpr int kCxMod = M ? DARM_CX_FMA_MOD_MELDED : DARM_CX_FMA_MOD;
  int32_t nxt[R];
  if (PF && tile < tiles) load_keys<R>(nxt, keys, tile * kTile + uint32_t(tid) * R, n);
  for (; tile < tiles; tile += units) {
    const uint32_t base = tile * kTile + uint32_t(tid) * R;
    const bool live = base < n;
    int32_t v[R];
    if constexpr (PF) {
#pragma unroll
      for (int j = 0; j < R; ++j) v[j] = nxt[j];
      if (tile + units < tiles) load_keys<R>(nxt, keys, base + units * kTile, n);   // next tile in flight
    } else {
      load_keys<R>(v, keys, base, n);
    }
    int32_t neg = 0;                                      // melded: current order flip of this thread
#pragma unroll
    for (int d = 1; d <= LB; ++d) {
      const bool thread_up = d >= LR && d < LB;           // up depends on the thread (runtime)
      const bool upT = d >= LB ? true : !((tib >> (d > LR ? d - LR : 0)) & 1);
      if constexpr (M) {
        const int32_t m = (thread_up && !upT) ? -1 : 0;
#pragma unroll
        for (int j = 0; j < R; ++j) v[j] = flip_fma(v[j], m ^ neg);
        neg = m;
      }
#pragma unroll
      for (int kb = d - 1; kb >= 0; --kb) {
        const int k = 1 << kb;
        if (k < R) {
          // in-register compare-exchange of the pairs (j, j | k)
          if (!thread_up || M) {
#pragma unroll
            for (int j = 0; j < R; ++j) {
              if (j & k) continue;
              const bool up = d < LR ? !((j >> d) & 1) : true;   // compile-time (or folded) direction
              int32_t lo, hi;
              cx_pair(kCxFma && cx_on_fma(j, kCxMod), v[j], v[j | k], lo, hi, one, mone);
              v[j] = up ? lo : hi;
              v[j | k] = up ? hi : lo;
            }
          } else if constexpr (F == kLiteral) {
            // App. A.2: the compare-exchange hoisted out of both arms, the
            // slot each key goes to chosen by `select %up`
#pragma unroll
            for (int j = 0; j < R; ++j) {
              if (j & k) continue;
              int32_t lo, hi;
              cx_pair(kCxFma && cx_on_fma(j, kCxMod), v[j], v[j | k], lo, hi, one, mone);
              v[j] = upT ? lo : hi;
              v[j | k] = upT ? hi : lo;
            }
          } else {
            if (upT) {                                    // condbr %up ^c ^d
              DARM_ARM_F(F, "bitonic.reg.up");
#pragma unroll
              for (int j = 0; j < R; ++j) {
                if (j & k) continue;
                int32_t lo, hi;
                cx_pair(kCxFma && cx_on_fma(j, kCxMod), v[j], v[j | k], lo, hi, one, mone);
                v[j] = lo;
                v[j | k] = hi;
              }
              DARM_ARM("bitonic.reg.up.end");
            } else {
              DARM_ARM_F(F, "bitonic.reg.down");
#pragma unroll
              for (int j = 0; j < R; ++j) {
                if (j & k) continue;
                int32_t lo, hi;
                cx_pair(kCxFma && cx_on_fma(j, kCxMod), v[j], v[j | k], lo, hi, one, mone);
                v[j] = hi;
                v[j | k] = lo;
              }
              DARM_ARM("bitonic.reg.down.end");
            }
          }
        } else {
          // partner thread tib ^ k/R holds the partner keys in the same registers
          const int pk = k / R;
          const bool keep = !(tib & pk);                  // icmp.lt %t %j
          int32_t b0[R];
          if (pk < 32) {
#pragma unroll
            for (int j = 0; j < R; ++j) b0[j] = __shfl_xor_sync(0xffffffffu, v[j], pk);   // load.shared buf %j
          } else if constexpr (kCta) {
            // another warp: one exchange through double-buffered shared memory
#pragma unroll
            for (int j = 0; j < R; ++j) xch[par][j][threadIdx.x] = v[j];
            bucket_sync<P, 256>();                         // the bucket's own warps only
#pragma unroll
            for (int j = 0; j < R; ++j) b0[j] = xch[par][j][threadIdx.x ^ pk];
            par ^= 1;
          }
          if constexpr (M) {
#pragma unroll
            for (int j = 0; j < R; ++j) {
              // need1 with up folded into the data: one predicated min/max
              v[j] = keep ? min(v[j], b0[j]) : max(v[j], b0[j]);   // ^e.m: the single melded store
            }
          } else if (!thread_up) {
#pragma unroll
            for (int j = 0; j < R; ++j) v[j] = keep ? min(v[j], b0[j]) : max(v[j], b0[j]);
          } else if constexpr (F == kLiteral) {
#pragma unroll
            for (int j = 0; j < R; ++j) v[j] = bitonic_exchange<kLiteral>(v[j], b0[j], keep, upT);
          } else {
            if (upT) {                                    // condbr %up ^c ^d
              DARM_ARM_F(F, "bitonic.xr.up");
#pragma unroll
              for (int j = 0; j < R; ++j) v[j] = keep ? min(v[j], b0[j]) : max(v[j], b0[j]);
              DARM_ARM("bitonic.xr.up.end");
            } else {
              DARM_ARM_F(F, "bitonic.xr.down");
#pragma unroll
              for (int j = 0; j < R; ++j) v[j] = keep ? max(v[j], b0[j]) : min(v[j], b0[j]);
              DARM_ARM("bitonic.xr.down.end");
            }
          }
        }
      }
    }
    if (live && R % 8 == 0 && aligned32(keys)) {
#pragma unroll
      for (int j = 0; j < R; ++j) v[j] = flip_fma(v[j], neg);
#pragma unroll
      for (int q = 0; q < R / 8; ++q) st_v8(keys + base + 8 * q, &v[8 * q]);
    } else if (live) {
      int4 *dst = reinterpret_cast<int4 *>(keys + base);
#pragma unroll
      for (int q = 0; q < R / 4; ++q)
        dst[q] = make_int4(flip_fma(v[4 * q], neg), flip_fma(v[4 * q + 1], neg), flip_fma(v[4 * q + 2], neg),
                           flip_fma(v[4 * q + 3], neg));
    }
  }
}

namespace {

int g_sms = 0;
int sm_count();

template <int F, int B>
cudaError_t launch_b(int32_t *keys, int64_t n, cudaStream_t s) {
  constexpr int CTA = B > 256 ? B : 256;
  sm_count();
  constexpr int U = B <= 256 ? 2 : 1;
  const int64_t tiles = (n + CTA - 1) / CTA;
  const int per_sm = 2048 / CTA;
  int64_t grid = int64_t(g_sms) * per_sm;
  if (grid > (tiles + U - 1) / U) grid = (tiles + U - 1) / U;
  if (grid < 1) grid = 1;
  bitonic_sort_kernel<F, B, CTA, U><<<int(grid), CTA, 0, s>>>(keys, uint32_t(n));
  return cudaGetLastError();
}

int sm_count() {
  if (!g_sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_sms, cudaDevAttrMultiProcessorCount, dev);
    if (g_sms <= 0) g_sms = 148;
  }
  return g_sms;
}

// Register-blocked launch: warps walk 32*R-key tiles with a grid stride.  The
// grid is sized so every warp gets the same number of tiles (up to one): with
// I = ceil(tiles / max resident warps) iterations, only ceil(tiles / I) warps
// are launched, spread evenly over the SMs.
template <int F, int B, int R, bool PF>
cudaError_t launch_reg_pf(int32_t *keys, int64_t n, cudaStream_t s) {
  constexpr int CTA = 256;
  static int per_sm = 0;                          // resident CTAs per SM (registers bound it)
  if (!per_sm) {
    cudaError_t e =
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, bitonic_sort_reg_kernel<F, B, R, PF>, CTA, 0);
    if (e != cudaSuccess || per_sm < 1) per_sm = 1;
  }
  const int64_t tiles = (n + CTA * R - 1) / (CTA * R);
  const int64_t max_ctas = int64_t(sm_count()) * per_sm;
  const int64_t iters = (tiles + max_ctas - 1) / max_ctas;
  int64_t grid = (tiles + iters - 1) / iters;
  if (grid < 1) grid = 1;
  bitonic_sort_reg_kernel<F, B, R, PF><<<int(grid), CTA, 0, s>>>(keys, uint32_t(n));
  return cudaGetLastError();
}

// Buckets that span warps: CTAs walk 256*R-key tiles, as many CTAs as fit
// (each with the same tile count, up to one).
template <int F, int B, int R>
cudaError_t launch_reg_cta(int32_t *keys, int64_t n, cudaStream_t s) {
  static int per_sm = 0;
  if (!per_sm) {
    cudaError_t e =
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, bitonic_sort_reg_kernel<F, B, R, true>, 256, 0);
    if (e != cudaSuccess || per_sm < 1) per_sm = 1;
  }
  const int64_t tiles = (n + 256 * R - 1) / (256 * R);
  const int64_t max_ctas = int64_t(sm_count()) * per_sm;
  const int64_t iters = (tiles + max_ctas - 1) / max_ctas;
  int64_t grid = (tiles + iters - 1) / iters;
  if (grid < 1) grid = 1;
  bitonic_sort_reg_kernel<F, B, R, true><<<int(grid), 256, 0, s>>>(keys, uint32_t(n));
  return cudaGetLastError();
}

template <int F, int B, int R>
cudaError_t launch_reg(int32_t *keys, int64_t n, cudaStream_t s) {
  if constexpr (B / R > 32) return launch_reg_cta<F, B, R>(keys, n, s);
  else return launch_reg_pf<F, B, R, true>(keys, n, s);
}

template <int F, int B>
cudaError_t launch_r(int32_t *keys, int64_t n, int r, cudaStream_t s) {
  if constexpr (B >= 4 && B / 4 <= 256) {
    if (r == 4) return launch_reg<F, B, 4>(keys, n, s);
  }
  if constexpr (B >= 8 && B / 8 <= 256) {
    if (r == 8) return launch_reg<F, B, 8>(keys, n, s);
  }
  if constexpr (B >= 16 && B / 16 <= 256) {
    if (r == 16) return launch_reg<F, B, 16>(keys, n, s);
  }
  if constexpr (B <= 1024) {
    if (r == 1) return launch_b<F, B>(keys, n, s);
  }
  return cudaErrorInvalidValue;
}

template <int F>
cudaError_t launch_m(int32_t *keys, int64_t n, int bucket, int r, cudaStream_t s) {
  switch (bucket) {
    case 2: return launch_r<F, 2>(keys, n, r, s);
    case 4: return launch_r<F, 4>(keys, n, r, s);
    case 8: return launch_r<F, 8>(keys, n, r, s);
    case 16: return launch_r<F, 16>(keys, n, r, s);
    case 32: return launch_r<F, 32>(keys, n, r, s);
    case 64: return launch_r<F, 64>(keys, n, r, s);
    case 128: return launch_r<F, 128>(keys, n, r, s);
    case 256: return launch_r<F, 256>(keys, n, r, s);
    case 512: return launch_r<F, 512>(keys, n, r, s);
    case 1024: return launch_r<F, 1024>(keys, n, r, s);
    case 2048: return launch_r<F, 2048>(keys, n, r, s);
    case 4096: return launch_r<F, 4096>(keys, n, r, s);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace

bool bitonic_sort_supported(int bucket) {
  return bucket >= 2 && bucket <= 4096 && (bucket & (bucket - 1)) == 0;
}

// keys_per_thread: 1 = one key per thread (the IR warp shape, buckets up to
// 1024), 4 / 8 / 16 = register-blocked (needs 16-byte aligned keys and
// bucket / r <= max_threads: 256 for bitonic, 32 for PCM), 0 = the fastest
// supported: 16 where bucket / 16 fits, the bucket itself for 4..16, else 1.
// -1: not supported.
int bitonic_keys_per_thread(int bucket, int keys_per_thread, const void *keys, int max_threads) {
  const bool aligned = (reinterpret_cast<uintptr_t>(keys) & 15) == 0;
  if (keys_per_thread == 0) {
    if (bucket >= 32 && bucket / 16 <= max_threads && aligned) return 16;
    if (bucket >= 4 && bucket <= 16 && aligned) return bucket;
    return bucket <= 1024 ? 1 : -1;
  }
  if (keys_per_thread == 1) return bucket <= 1024 ? 1 : -1;
  if (keys_per_thread != 4 && keys_per_thread != 8 && keys_per_thread != 16) return -1;
  if (!aligned || keys_per_thread > bucket || bucket / keys_per_thread > max_threads) return -1;
  return keys_per_thread;
}

cudaError_t launch_bitonic_sort(int variant, int32_t *keys, int64_t n, int bucket, int keys_per_thread,
                                cudaStream_t s, int *launches) {
  if (n == 0) return cudaSuccess;
  if (launches) *launches += 1;
  switch (variant) {
    case kUnmelded: return launch_m<kUnmelded>(keys, n, bucket, keys_per_thread, s);
    case kMelded: return launch_m<kMelded>(keys, n, bucket, keys_per_thread, s);
    case kPredicated: return launch_m<kPredicated>(keys, n, bucket, keys_per_thread, s);
    default: return launch_m<kLiteral>(keys, n, bucket, keys_per_thread, s);
  }
}

}  // namespace darm_gpu
