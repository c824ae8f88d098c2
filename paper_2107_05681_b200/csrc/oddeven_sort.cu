// oddeven_sort.cu — PCM: Batcher odd-even merge sort of
// independent buckets, built from the step of paper_2107_05681_b200/ir/
// oddeven_step.ir in three forms.  The reference has no PCM code; the step is
// written in the reference's mini-IR and the melded form is what runDarm emits
// for it: a block-region meld of the upper comparator
// region with the idle block (region replication), then a region-region meld
// of the lower region with the result.
//
// Step (p, k) over a B-key bucket: comparators (x, x + k) for every x with
// x >= k % p, (x - k % p) mod 2k < k, x + k < B and x, x + k in the same 2p
// block; the lower end keeps the smaller key, the upper end the larger, other
// lanes are idle.  Steps: p = 1, 2, .., B/2; k = p, .., 1.
//
// The IR's step reads the bucket from shared memory inside the divergent
// region — three-way, lower / upper / idle — and each comparator arm holds a
// nested data-dependent if-then ("loops with nested data-dependent branches",
// PAPER.md:753; "complex control-flow regions with shared memory
// instructions", :835-836):
//   lower: x0 = buf[t+k]; cv = buf[t]; res[t] = cv; if (cv > x0) res[t] = x0
//   upper: x1 = buf[t-k]; dv = buf[t]; res[t] = dv; if (dv < x1) res[t] = x1
//   idle:  res[t] = buf[t]
// Forms:
//   unmelded   that CFG with its IPDOM reconvergence: the role branch and the
//              nested data-dependent branches are real divergent branches
//              (DARM_IPDOM), the shared loads inside the arms;
//   predicated the same CFG as ptxas compiles it (short arms if-converted);
//   melded     runDarm's output: the partner and own loads hoisted and melded
//              (one load at a selected address), the comparison direction and
//              the stored value as selects, one store.
// Two shapes, as for the bitonic sort (bitonic_sort.cu):
//   one key per thread (the IR warp shape): the bucket staged in shared
//     memory every step (double-buffered), the roles per lane;
//   R keys per thread: strides below R pair registers of one thread
//     (compile-time roles, no divergence in any form) or the top k registers
//     of a thread with the bottom k of the next; strides k >= R pair whole
//     threads: the R keys are staged in shared memory ([R/4][thread] int4s,
//     conflict-free) and the role is per thread — the divergent region, with
//     one nested data-dependent branch per key.
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

// One comparator region of the IR for one key: own key cv, partner key xp
// (read inside the arm by the caller), role lower / upper / idle.
//   F == kUnmelded: res = cv; if (out of order) res = xp — behind a real branch.
template <int F>
__device__ __forceinline__ int32_t oe_arm_lower(int32_t cv, int32_t xp) {
  int32_t r = cv;                                          // store.global res %t %cv
  if (cv > xp) {                                           // condbr %g1 ^ls ^lx
    DARM_ARM_F(F, "oddeven.ls");
    r = xp;                                                // ^ls: store.global res %t %x0
  }
  return r;
}
template <int F>
__device__ __forceinline__ int32_t oe_arm_upper(int32_t dv, int32_t xp) {
  int32_t r = dv;                                          // store.global res %t %dv
  if (dv < xp) {                                           // condbr %g2 ^us ^ux
    DARM_ARM_F(F, "oddeven.us");
    r = xp;                                                // ^us: store.global res %t %x1
  }
  return r;
}
// melded: out of order = lower ? cv > xp : upper ? cv < xp : false, one
// store.  The melded load gives an idle lane its own key as the partner
// (xp == cv), so the stored value is `lower ? min(cv, xp) : max(cv, xp)` for
// every role: one predicated VIMNMX (min or max by the role predicate), as
// the bitonic melded exchange.
__device__ __forceinline__ int32_t oe_melded(int32_t cv, int32_t xp, bool lower) {
  return lower ? min(cv, xp) : max(cv, xp);
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

template <int F, int B, int CTA, int p, int k, int s>
__device__ __forceinline__ int32_t oe_one_step(int32_t v, uint64_t lo, uint64_t up, int32_t (*buf)[CTA], int &par) {
  const bool lower = (lo >> s) & 1u;
  const bool upper = (up >> s) & 1u;
  const int t = int(threadIdx.x);
  int32_t *b = buf[par];
  b[t] = v;                                                // the bucket in shared buf
  if constexpr (B <= 32) __syncwarp();                     // a bucket never spans warps
  else __syncthreads();                                    // (per-bucket named barriers measured slower here:
                                                           //  B = 64 melded 190 -> 227 us)
  par ^= 1;                                                // double buffer: no barrier before the next write
  if constexpr (F == kMelded) {
    // the hoisted, melded loads: partner at a selected address, own key
    const int32_t xp = b[lower ? t + k : (upper ? t - k : t)];
    const int32_t cv = b[t];
    return oe_melded(cv, xp, lower);
  } else {
    int32_t r;
    if (lower) {                                           // condbr %lower ^lo ^nl
      DARM_ARM_F(F, "oddeven.lo");
      r = oe_arm_lower<F>(b[t], b[t + k]);                 // ^lo: load.shared buf %t, buf %tk
    } else if (upper) {                                    // ^nl: condbr %upper ^up ^id
      DARM_ARM_F(F, "oddeven.up");
      r = oe_arm_upper<F>(b[t], b[t - k]);                 // ^up: load.shared buf %t, buf %s
    } else {
      DARM_ARM_F(F, "oddeven.id");
      r = b[t];                                            // ^id: load.shared buf %t
    }
    return r;
  }
}

template <int F, int B, int CTA, int p, int k, int s>
__device__ __forceinline__ int32_t oe_one_network(int32_t v, uint64_t lo, uint64_t up, int32_t (*buf)[CTA],
                                                  int &par) {
  if constexpr (p < B) {
    v = oe_one_step<F, B, CTA, p, k, s>(v, lo, up, buf, par);
    if constexpr (k > 1)
      return oe_one_network<F, B, CTA, p, k / 2, s + 1>(v, lo, up, buf, par);
    else
      return oe_one_network<F, B, CTA, 2 * p, 2 * p, s + 1>(v, lo, up, buf, par);
  }
  return v;
}

template <int F, int B, int CTA>
__global__ void __launch_bounds__(CTA) oddeven_sort_kernel(int32_t *__restrict__ keys, uint32_t n) {
  static_assert(__builtin_ctz(B) * (__builtin_ctz(B) + 1) / 2 <= 64, "step masks are 64-bit");
  __shared__ int32_t buf[2][CTA];
  const int t = int(threadIdx.x) & (B - 1);
  uint64_t lo = 0, up = 0;
  oe_roles<B, 1, 1, 0>(t, lo, up);
  const uint32_t tiles = (n + CTA - 1) / CTA;
  // buffer parity runs on across tiles (21 steps at B = 64: reset per tile,
  // the next tile's first write would hit the buffer the last step reads)
  int par = 0;
  for (uint32_t tile = blockIdx.x; tile < tiles; tile += gridDim.x) {
    const uint32_t id = tile * CTA + threadIdx.x;
    int32_t v = id < n ? keys[id] : INT_MAX;
    v = oe_one_network<F, B, CTA, 1, 1, 0>(v, lo, up, buf, par);
    if (id < n) keys[id] = v;
  }
}

// ------------------------------------------------------------ R keys per thread
// One step (p, k) on the R registers of a thread; p and k are template
// parameters so every register index and role test is resolved at compile time.
template <int F, int B, int R, int p, int k>
__device__ __forceinline__ void oe_reg_step(int32_t (&v)[R], int lane, int tib, int x0, int4 (*xs)[256]) {
  constexpr int P = B / R;
  if constexpr (k >= R) {
    // whole threads pair up: partner thread +- k/R, same register; role per
    // thread.  The R keys go through shared memory (the IR's buf): written by
    // every thread, read by its partner inside the divergent region.
    const bool lower = oe_is_lower<p, k>(x0);
    const bool upper = oe_is_upper<p, k>(x0);
    const int t = int(threadIdx.x);
    __syncwarp();                                          // the previous step's reads are done
#pragma unroll
    for (int q = 0; q < R / 4; ++q) xs[q][t] = make_int4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
    __syncwarp();
    auto partner = [&](int src, int32_t (&xp)[R]) {       // load.shared buf %tk / %s
#pragma unroll
      for (int q = 0; q < R / 4; ++q) {
        const int4 x = xs[q][src];
        xp[4 * q] = x.x;
        xp[4 * q + 1] = x.y;
        xp[4 * q + 2] = x.z;
        xp[4 * q + 3] = x.w;
      }
    };
    if constexpr (F == kMelded) {
      int32_t xp[R];
      partner(lower ? t + k / R : (upper ? t - k / R : t), xp);   // one load, selected address
#pragma unroll
      for (int j = 0; j < R; ++j) v[j] = oe_melded(v[j], xp[j], lower);
    } else {
      if (lower) {                                         // condbr %lower ^lo ^nl
        DARM_ARM_F(F, "oddeven.reg.lo");
        int32_t xp[R];
        partner(t + k / R, xp);
#pragma unroll
        for (int j = 0; j < R; ++j) v[j] = oe_arm_lower<F>(v[j], xp[j]);
      } else if (upper) {                                  // ^nl: condbr %upper ^up ^id
        DARM_ARM_F(F, "oddeven.reg.up");
        int32_t xp[R];
        partner(t - k / R, xp);
#pragma unroll
        for (int j = 0; j < R; ++j) v[j] = oe_arm_upper<F>(v[j], xp[j]);
      } else {
        DARM_ARM_F(F, "oddeven.reg.id");                   // ^id: the own keys stay
      }
    }
    (void)lane;
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
__device__ __forceinline__ void oe_reg_network(int32_t (&v)[R], int lane, int tib, int x0, int4 (*xs)[256]) {
  if constexpr (p < B) {
    oe_reg_step<F, B, R, p, k>(v, lane, tib, x0, xs);
    if constexpr (k > 1)
      oe_reg_network<F, B, R, p, k / 2>(v, lane, tib, x0, xs);
    else
      oe_reg_network<F, B, R, 2 * p, 2 * p>(v, lane, tib, x0, xs);
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
  __shared__ int4 xs[R / 4][256];                          // the cross-thread steps' buf
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
    oe_reg_network<F, B, R, 1, 1>(v, lane, tib, x0, xs);
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
