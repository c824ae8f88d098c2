// oddeven_sort.cu — PCM: Batcher odd-even merge sort of
// independent buckets, built from the step of paper_2107_05681_b200/ir/
// oddeven_step.ir in its unmelded and melded forms.  The reference has no PCM
// code; the step is written in the reference's mini-IR and the melded form is
// what runDarm emits for it (one region-region meld, as for bitonic.ir: the
// partner compare is melded and one select picks gt / lt by the role).
//
// Step (p, k) over a B-key bucket: comparators (x, x + k) for every x with
// x >= k % p, (x - k % p) mod 2k < k, x + k < B and x, x + k in the same 2p
// block; the lower end keeps the smaller key, the upper end the larger, other
// lanes are idle (their own partner).  Steps: p = 1, 2, .., B/2; k = p, .., 1.
//
// Two shapes, as for the bitonic sort (bitonic_sort.cu):
//   one key per thread (the IR warp shape): partner by __shfl_sync inside a
//     warp, through shared memory when it may sit in another warp; the
//     divergent branch is the lower / not-lower role of every lane;
//   R keys per thread: strides below R pair registers of one thread
//     (compile-time roles) or the top k registers of a thread with the bottom
//     k of the next (one shuffle each way), strides k >= R pair whole threads
//     (role per thread, the divergent branch).
// Unmelded: `if (lower) keep min else keep max`, both arms fenced (DARM_ARM).
// Melded:   the select of SURVEY App. A.2's shape: v = lower ? min : max.
#include <climits>

#include "common.cuh"
#include "kernels.h"

namespace darm_gpu {

namespace {

// Roles of key x in step (p, k) as bit tests (compile-time powers of two
// k <= p, 2p <= B; the general test is oracle_oddeven_sort's):
//   k == p: x pairs with x ^ k (lower iff bit k clear);
//   k <  p: lower iff bit k set and x mod 2p < 2p - k; upper iff bit k clear
//           and x mod 2p >= k.
template <int p, int k>
__device__ __forceinline__ bool oe_is_lower(int x) {
  if constexpr (k == p) return !(x & k);
  else return (x & k) && (x & (2 * p - 1)) < 2 * p - k;
}
template <int p, int k>
__device__ __forceinline__ bool oe_is_upper(int x) {
  if constexpr (k == p) return x & k;
  else return !(x & k) && (x & (2 * p - 1)) >= k;
}

// lower ? min(v, b) : max(v, b) issued as a complementary predicated pair:
// for the plain select ptxas emits min; @!P max, whose write-after-write on
// one register stalls every serial step.
__device__ __forceinline__ int32_t oe_select_minmax(int32_t v, int32_t b, bool lower) {
  asm("{\n .reg .pred p;\n setp.ne.b32 p, %1, 0;\n @p min.s32 %0, %0, %2;\n @!p max.s32 %0, %0, %2;\n}"
      : "+r"(v)
      : "r"(int(lower)), "r"(b));
  return v;
}

template <int F>
__device__ __forceinline__ int32_t oe_exchange_unmelded(int32_t v, int32_t b0, bool lower) {
  if (lower) {                                             // condbr %lower ^lo ^up
    DARM_ARM_F(F, "oddeven.lo");
    v = min(v, b0);                                        // ^lo: cv > b0 -> store b0
    DARM_ARM("oddeven.lo.end");
  } else {
    DARM_ARM_F(F, "oddeven.up");
    v = max(v, b0);                                        // ^up: cv < b0 -> store b0
    DARM_ARM("oddeven.up.end");
  }
  return v;
}

}  // namespace

// ------------------------------------------------------------ one key per thread
// The lane roles depend on t only, so they are computed once per thread as
// bit masks over the step index s (bit s of lo / up) outside the tile loop.
template <int B, int p, int k, int s>
__device__ __forceinline__ void oe_roles(int t, uint64_t &lo, uint64_t &up) {
  if constexpr (p < B) {
    lo |= uint64_t(oe_is_lower<p, k>(t)) << s;
    up |= uint64_t(oe_is_upper<p, k>(t)) << s;
    if constexpr (k > 1)
      oe_roles<B, p, k / 2, s + 1>(t, lo, up);
    else
      oe_roles<B, 2 * p, 2 * p, s + 1>(t, lo, up);
  }
}

template <int F, int CTA, int p, int k, int s>
__device__ __forceinline__ int32_t oe_one_step(int32_t v, int lane, uint64_t lo, uint64_t up, int32_t (*xch)[CTA],
                                               int &par) {
  const bool lower = (lo >> s) & 1u;
  const bool upper = (up >> s) & 1u;
  int32_t b0;                                              // load.shared buf %j (partner, or own slot)
  // x + k stays in x's warp unless k >= 32 or (k < p) the add carries across
  // a 32-key boundary inside a 2p > 32 block
  if constexpr (k < 32 && (k == p || 2 * p <= 32)) {
    const int src = lower ? lane + k : (upper ? lane - k : lane);
    b0 = __shfl_sync(0xffffffffu, v, src);
  } else {
    xch[par][threadIdx.x] = v;
    __syncthreads();
    b0 = xch[par][lower ? threadIdx.x + k : (upper ? threadIdx.x - k : threadIdx.x)];
    par ^= 1;
  }
  if constexpr (F == kMelded)
    return oe_select_minmax(v, b0, lower);   // %sel = select %lower %g1 %g2; one store
  else
    return oe_exchange_unmelded<F>(v, b0, lower);
}

template <int F, int B, int CTA, int p, int k, int s>
__device__ __forceinline__ int32_t oe_one_network(int32_t v, int lane, uint64_t lo, uint64_t up,
                                                  int32_t (*xch)[CTA], int &par) {
  if constexpr (p < B) {
    v = oe_one_step<F, CTA, p, k, s>(v, lane, lo, up, xch, par);
    if constexpr (k > 1)
      return oe_one_network<F, B, CTA, p, k / 2, s + 1>(v, lane, lo, up, xch, par);
    else
      return oe_one_network<F, B, CTA, 2 * p, 2 * p, s + 1>(v, lane, lo, up, xch, par);
  }
  return v;
}

template <int F, int B, int CTA>
__global__ void __launch_bounds__(CTA) oddeven_sort_kernel(int32_t *__restrict__ keys, uint32_t n) {
  static_assert(__builtin_ctz(B) * (__builtin_ctz(B) + 1) / 2 <= 64, "step masks are 64-bit");
  __shared__ int32_t xch[2][CTA];
  const int t = int(threadIdx.x) & (B - 1);
  const int lane = int(threadIdx.x) & 31;
  uint64_t lo = 0, up = 0;
  oe_roles<B, 1, 1, 0>(t, lo, up);
  const uint32_t tiles = (n + CTA - 1) / CTA;
  for (uint32_t tile = blockIdx.x; tile < tiles; tile += gridDim.x) {
    const uint32_t id = tile * CTA + threadIdx.x;
    int32_t v = id < n ? keys[id] : INT_MAX;
    int par = 0;
    v = oe_one_network<F, B, CTA, 1, 1, 0>(v, lane, lo, up, xch, par);
    if (id < n) keys[id] = v;
  }
}

// ------------------------------------------------------------ R keys per thread
// One step (p, k) on the R registers of a thread; p and k are template
// parameters so every register index and role test is resolved at compile time.
template <int F, int B, int R, int p, int k>
__device__ __forceinline__ void oe_reg_step(int32_t (&v)[R], int lane, int tib, int x0) {
  constexpr int P = B / R;
  if constexpr (k >= R) {
    // whole threads pair up: partner lane +- k/R, same register; role per thread
    const bool lower = oe_is_lower<p, k>(x0);
    const bool upper = oe_is_upper<p, k>(x0);
    const int src = lower ? lane + k / R : (upper ? lane - k / R : lane);
    int32_t b0[R];
#pragma unroll
    for (int j = 0; j < R; ++j) b0[j] = __shfl_sync(0xffffffffu, v[j], src);
    if constexpr (F == kMelded) {
      // the select as a complementary predicated pair (see oe_one_step) from 8
      // keys per thread up; at 4 the plain select schedules better (57 vs 63 µs)
#pragma unroll
      for (int j = 0; j < R; ++j)
        v[j] = R >= 8 ? oe_select_minmax(v[j], b0[j], lower) : (lower ? min(v[j], b0[j]) : max(v[j], b0[j]));
    } else {
      if (lower) {                                         // condbr %lower ^lo ^up
        DARM_ARM_F(F, "oddeven.reg.lo");
#pragma unroll
        for (int j = 0; j < R; ++j) v[j] = min(v[j], b0[j]);
        DARM_ARM("oddeven.reg.lo.end");
      } else {
        DARM_ARM_F(F, "oddeven.reg.up");
#pragma unroll
        for (int j = 0; j < R; ++j) v[j] = max(v[j], b0[j]);
        DARM_ARM("oddeven.reg.up.end");
      }
    }
  } else if constexpr (2 * p <= R) {
    // the whole 2p block sits in this thread: compile-time comparators
#pragma unroll
    for (int j = 0; j + k < R; ++j) {
      constexpr int kp = k == p ? 0 : k;
      const int y = j % (2 * p);
      if (!(y >= kp && ((y - kp) & k) == 0 && y + k < 2 * p)) continue;
      int32_t lo, hi;
      cx_pair(cx_on_fma(j), v[j], v[j + k], lo, hi, gridDim.y, 0u - gridDim.y);   // half the maxima on the FMA pipe
      v[j] = lo;
      v[j + k] = hi;
    }
  } else {
    // k < R < 2p: kp = k, lower ends have bit k set.  Pairs inside the thread,
    // and the top k registers with the next thread's bottom k when both
    // threads lie in one 2p block (one shuffle each way per pair).
    int32_t dn[k], up[k];
#pragma unroll
    for (int q = 0; q < k; ++q) {
      dn[q] = __shfl_down_sync(0xffffffffu, v[q], 1);           // next thread's register q
      up[q] = __shfl_up_sync(0xffffffffu, v[R - k + q], 1);     // previous thread's register R-k+q
    }
    const bool act_dn = tib + 1 < P && ((x0 + R) % (2 * p)) != 0;
    const bool act_up = tib > 0 && (x0 % (2 * p)) != 0;
#pragma unroll
    for (int j = 0; j + k < R; ++j) {
      if (!(j & k)) continue;
      int32_t lo, hi;
      cx_pair(cx_on_fma(j), v[j], v[j + k], lo, hi, gridDim.y, 0u - gridDim.y);
      v[j] = lo;
      v[j + k] = hi;
    }
#pragma unroll
    for (int q = 0; q < k; ++q) {
      v[R - k + q] = act_dn ? min(v[R - k + q], dn[q]) : v[R - k + q];
      v[q] = act_up ? max(v[q], up[q]) : v[q];
    }
  }
}

// steps k = K, K/2, .., 1 of stage p, then the next stage
template <int F, int B, int R, int p, int k>
__device__ __forceinline__ void oe_reg_network(int32_t (&v)[R], int lane, int tib, int x0) {
  if constexpr (p < B) {
    oe_reg_step<F, B, R, p, k>(v, lane, tib, x0);
    if constexpr (k > 1)
      oe_reg_network<F, B, R, p, k / 2>(v, lane, tib, x0);
    else
      oe_reg_network<F, B, R, 2 * p, 2 * p>(v, lane, tib, x0);
  }
}

// R consecutive keys of one thread (INT_MAX past the end; n % B == 0)
template <int R>
__device__ __forceinline__ void oe_load_keys(int32_t (&v)[R], const int32_t *__restrict__ keys, uint32_t base, uint32_t n) {
  if (base < n && R % 8 == 0 && aligned32(keys)) {         // whole sectors per warp instruction
#pragma unroll
    for (int q = 0; q < R / 8; ++q) ld_v8(keys + base + 8 * q, &v[8 * q]);
  } else if (base < n) {
    const int4 *src = reinterpret_cast<const int4 *>(keys + base);
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

template <int F, int B, int R>
__global__ void __launch_bounds__(256, 4) oddeven_sort_reg_kernel(int32_t *__restrict__ keys, uint32_t n) {
  constexpr int P = B / R;
  static_assert(R >= 4 && R <= B && P <= 32, "R keys per thread, at most 32 threads per bucket");
  // CTA-uniform walk over 256 R-key tiles: ptxas sees every shuffle converged
  constexpr uint32_t kTile = 256u * R;
  const int lane = int(threadIdx.x) & 31;
  const int tib = lane & (P - 1);
  const int x0 = tib * R;                                  // bucket index of register 0
  const uint32_t tiles = (n + kTile - 1) / kTile;
  int32_t nxt[R];                                          // the next tile's keys, in flight
  uint32_t tile = blockIdx.x;
  if (tile < tiles) oe_load_keys<R>(nxt, keys, tile * kTile + uint32_t(threadIdx.x) * R, n);
  for (; tile < tiles; tile += gridDim.x) {
    const uint32_t base = tile * kTile + uint32_t(threadIdx.x) * R;
    int32_t v[R];
#pragma unroll
    for (int j = 0; j < R; ++j) v[j] = nxt[j];
    if (tile + gridDim.x < tiles) oe_load_keys<R>(nxt, keys, base + gridDim.x * kTile, n);
    oe_reg_network<F, B, R, 1, 1>(v, lane, tib, x0);
    if (base < n && R % 8 == 0 && aligned32(keys)) {
#pragma unroll
      for (int q = 0; q < R / 8; ++q) st_v8(keys + base + 8 * q, &v[8 * q]);
    } else if (base < n) {
      int4 *dst = reinterpret_cast<int4 *>(keys + base);
#pragma unroll
      for (int q = 0; q < R / 4; ++q) dst[q] = make_int4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
    }
  }
}

namespace {

int g_sms_oe = 0;

int sms() {
  if (!g_sms_oe) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_sms_oe, cudaDevAttrMultiProcessorCount, dev);
    if (g_sms_oe <= 0) g_sms_oe = 148;
  }
  return g_sms_oe;
}

template <int F, int B>
cudaError_t launch_one(int32_t *keys, int64_t n, cudaStream_t s) {
  constexpr int CTA = B > 256 ? B : 256;
  const int64_t tiles = (n + CTA - 1) / CTA;
  int64_t grid = int64_t(sms()) * (2048 / CTA);
  if (grid > tiles) grid = tiles;
  if (grid < 1) grid = 1;
  oddeven_sort_kernel<F, B, CTA><<<int(grid), CTA, 0, s>>>(keys, uint32_t(n));
  return cudaGetLastError();
}

template <int F, int B, int R>
cudaError_t launch_reg(int32_t *keys, int64_t n, cudaStream_t s) {
  constexpr int CTA = 256;
  static int per_sm = 0;
  if (!per_sm) {
    cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, oddeven_sort_reg_kernel<F, B, R>, CTA, 0);
    if (e != cudaSuccess || per_sm < 1) per_sm = 1;
  }
  const int64_t tiles = (n + CTA * R - 1) / (CTA * R);
  const int64_t max_ctas = int64_t(sms()) * per_sm;
  const int64_t iters = (tiles + max_ctas - 1) / max_ctas;
  int64_t grid = (tiles + iters - 1) / iters;
  if (grid < 1) grid = 1;
  oddeven_sort_reg_kernel<F, B, R><<<int(grid), CTA, 0, s>>>(keys, uint32_t(n));
  return cudaGetLastError();
}

template <int F, int B>
cudaError_t launch_r(int32_t *keys, int64_t n, int r, cudaStream_t s) {
  if constexpr (B >= 4 && B / 4 <= 32) {
    if (r == 4) return launch_reg<F, B, 4>(keys, n, s);
  }
  if constexpr (B >= 8 && B / 8 <= 32) {
    if (r == 8) return launch_reg<F, B, 8>(keys, n, s);
  }
  if constexpr (B >= 16 && B / 16 <= 32) {
    if (r == 16) return launch_reg<F, B, 16>(keys, n, s);
  }
  if (r == 1) return launch_one<F, B>(keys, n, s);
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
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace

cudaError_t launch_oddeven_sort(int variant, int32_t *keys, int64_t n, int bucket, int keys_per_thread,
                                cudaStream_t s, int *launches) {
  if (n == 0) return cudaSuccess;
  if (launches) *launches += 1;
  switch (variant) {
    case kUnmelded: return launch_m<kUnmelded>(keys, n, bucket, keys_per_thread, s);
    case kMelded: return launch_m<kMelded>(keys, n, bucket, keys_per_thread, s);
    default: return launch_m<kPredicated>(keys, n, bucket, keys_per_thread, s);
  }
}

}  // namespace darm_gpu
