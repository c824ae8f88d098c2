// merge_sort.cu — MS: parallel bottom-up merge sort of the
// whole array, in the unmelded and melded forms of the merge step of
// paper_2107_05681_b200/ir/merge_step.ir.  The reference has no MS code; the
// merge loop is written in the reference's mini-IR and the melded form is what
// runDarm emits for it (one block-block meld of the take-left / take-right
// arms, MP 0.5: one select of the run index, one load, one store, and the two
// index updates as unpredicated runs).
//
// Pass w merges the sorted runs [a, a+w) and [a+w, a+2w) (clipped to n) of
// src into dst, for w = 1, 2, 4, .. < n.  Every thread produces E = 16
// consecutive outputs of one pass: it finds where its first output lies on the
// merge path of its pair (binary search on the diagonal, ties to the left run:
// a stable merge), then runs the IR loop E times — emit the smaller head,
// advance that run — the data-dependent divergent branch.
//   passes w < 4096: one CTA per 4096-key tile, all those passes in shared
//     memory (ping-pong buffers, skewed addresses against bank conflicts);
//   passes w >= 4096: a CTA produces 4096 outputs of one merge; warps 0 and 1
//     find the CTA's two merge-path boundaries with a 32-way ballot search
//     (__ballot_sync), the CTA stages its slices of both runs in shared
//     memory with coalesced loads, merges there and stores coalesced.
// Unmelded: `if (take_left) {emit a; load next a} else {emit b; load next b}`
// (two loads, both arms fenced).  Melded: out = take ? a : b; one load at the
// selected run's next index; the index / head updates are selects.
#include <climits>

#include "common.cuh"
#include "kernels.h"

namespace darm_gpu {

namespace {

constexpr int kThreads = 256;
constexpr int kE = 16;                     // outputs per thread per pass
constexpr int kTile = kThreads * kE;       // 4096 keys

// shared-memory slot of element k: one pad word per 32 so that threads
// writing E-strided outputs hit distinct banks
__device__ __forceinline__ int sk(int k) { return k + (k >> 5); }
constexpr int kSmemWords = kTile + kTile / 32;

// merge path: number of elements taken from A among the first d outputs of
// merge(A[0..na), B[0..nb)), ties to A.  A, B read through `at`.
template <class FA, class FB>
__device__ __forceinline__ int merge_path(FA at_a, FB at_b, int na, int nb, int d) {
  int lo = d > nb ? d - nb : 0, hi = d < na ? d : na;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (at_a(mid) <= at_b(d - 1 - mid))
      lo = mid + 1;
    else
      hi = mid;
  }
  return lo;
}

// NE steps of the IR merge loop over shared memory: inputs s[i..iend) and
// s[j..jend) (logical indices, skewed with sk), outputs emitted to out[0..NE).
template <bool M, int NE>
__device__ __forceinline__ void merge_steps(const int32_t *s, int i, int iend, int j, int jend, int32_t *out) {
  int32_t ah = i < iend ? s[sk(i)] : 0, bh = j < jend ? s[sk(j)] : 0;
#pragma unroll
  for (int e = 0; e < NE; ++e) {
    const bool take = j >= jend || (i < iend && ah <= bh);   // %take
    if constexpr (!M) {
      if (take) {                                             // condbr %take ^ta ^tb
        DARM_ARM("merge.ta");
        out[e] = ah;                                          // store.global dst %k %va
        ++i;                                                  // %i1 = add %i 1
        if (i < iend) ah = s[sk(i)];                          // next head of the left run
        DARM_ARM("merge.ta.end");
      } else {
        DARM_ARM("merge.tb");
        out[e] = bh;
        ++j;
        if (j < jend) bh = s[sk(j)];
        DARM_ARM("merge.tb.end");
      }
    } else {
      // runDarm: %sel = select %take %i %j; one load; one store; %i1 = add %sel 1
      out[e] = take ? ah : bh;
      const int nx = (take ? i : j) + 1;
      const int lim = take ? iend : jend;
      const int32_t nv = nx < lim ? s[sk(nx)] : 0;
      if (take) {                                             // the two unpredicated runs
        i = nx;
        ah = nv;
      } else {
        j = nx;
        bh = nv;
      }
    }
  }
}

}  // namespace

// ------------------------------------------------------------ passes w < kTile
// pass of width W on the tile in buf[cur] -> buf[cur ^ 1]; W is a template
// parameter so the small widths (several whole pairs per thread) unroll.
template <bool M, int W>
__device__ __forceinline__ void tile_pass(int32_t (*buf)[kSmemWords], int cur, int k0) {
  const int32_t *s = buf[cur];
  int32_t o[kE];
  if constexpr (2 * W < kE) {
    // kE / 2W whole pairs per thread, merged one after another
#pragma unroll
    for (int q = 0; q < kE / (2 * W); ++q) {
      const int a = k0 + 2 * W * q;
      merge_steps<M, 2 * W>(s, a, a + W, a + W, a + 2 * W, o + 2 * W * q);
    }
  } else {
    // this thread's outputs lie in one pair; start on its merge path
    const int a = k0 & ~(2 * W - 1);
    const int d = k0 - a;
    const int x = merge_path([&](int q) { return s[sk(a + q)]; }, [&](int q) { return s[sk(a + W + q)]; }, W, W, d);
    merge_steps<M, kE>(s, a + x, a + W, a + W + (d - x), a + 2 * W, o);
  }
  int32_t *d = buf[cur ^ 1];
#pragma unroll
  for (int e = 0; e < kE; ++e) d[sk(k0 + e)] = o[e];
}

template <bool M, int W>
__device__ __forceinline__ int tile_passes(int32_t (*buf)[kSmemWords], int cur, int k0) {
  if constexpr (W < kTile) {
    tile_pass<M, W>(buf, cur, k0);
    __syncthreads();
    return tile_passes<M, 2 * W>(buf, cur ^ 1, k0);
  }
  return cur;
}

template <bool M>
__global__ void __launch_bounds__(kThreads) merge_sort_tile_kernel(const int32_t *__restrict__ in,
                                                                   int32_t *__restrict__ out, int n) {
  __shared__ int32_t buf[2][kSmemWords];
  const int base = blockIdx.x * kTile;
  const int cnt = min(kTile, n - base);
  for (int e = threadIdx.x; e < kTile; e += kThreads) buf[0][sk(e)] = e < cnt ? in[base + e] : INT_MAX;
  __syncthreads();
  const int cur = tile_passes<M, 1>(buf, 0, threadIdx.x * kE);
  for (int e = threadIdx.x; e < cnt; e += kThreads) out[base + e] = buf[cur][sk(e)];
}

// ------------------------------------------------------------ passes w >= kTile
// 32-way ballot search of the merge path (ties to A): the number of elements
// of A among the first d outputs; every lane of the warp returns it.
__device__ __forceinline__ int warp_merge_path(const int32_t *A, int na, const int32_t *B, int nb, int d) {
  const int lane = threadIdx.x & 31;
  int lo = d > nb ? d - nb : 0, hi = d < na ? d : na;        // the answer x* lies in [lo, hi]
  while (lo < hi) {
    // probe x = lo + (lane+1)*step - 1: "A[x] <= B[d-1-x]" holds exactly for x < x*
    const int step = (hi - lo + 31) >> 5;
    const int x = lo + (lane + 1) * step - 1;
    const bool p = x < hi && __ldg(A + x) <= __ldg(B + (d - 1 - x));
    const int c = __popc(__ballot_sync(0xffffffffu, p));   // true probes form a prefix
    const int nlo = lo + c * step;                           // probe c-1 true:  x* >= nlo
    hi = min(hi, nlo + step - 1);                            // probe c false:   x* <= nlo + step - 1
    lo = nlo;
  }
  return lo;
}

template <bool M>
__global__ void __launch_bounds__(kThreads, 7) merge_sort_pass_kernel(const int32_t *__restrict__ src,
                                                                   int32_t *__restrict__ dst, int n, int w) {
  __shared__ int32_t s[kSmemWords];
  __shared__ int bounds[2];
  const int K0 = blockIdx.x * kTile;
  const int cnt = min(kTile, n - K0);
  const int a = K0 & ~(2 * w - 1);                            // pair base (2w >= 2 kTile, aligned)
  const int na = max(0, min(w, n - a)), nb = max(0, min(w, n - a - w));
  const int32_t *A = src + a, *B = src + a + na;
  const int warp = threadIdx.x >> 5;
  if (warp < 2) {
    const int d = warp == 0 ? K0 - a : K0 - a + cnt;
    const int x = warp_merge_path(A, na, B, nb, d);
    if ((threadIdx.x & 31) == 0) bounds[warp] = x;
  }
  __syncthreads();
  const int i0 = bounds[0], i1 = bounds[1];
  const int j0 = (K0 - a) - i0, j1 = (K0 - a + cnt) - i1;
  const int la = i1 - i0, lb = j1 - j0;                       // la + lb == cnt
  for (int e = threadIdx.x; e < cnt; e += kThreads) s[sk(e)] = e < la ? A[i0 + e] : B[j0 + e - la];
  __syncthreads();
  const int k0 = threadIdx.x * kE;
  int32_t o[kE];
  if (k0 < cnt) {
    const int x = merge_path([&](int q) { return s[sk(q)]; }, [&](int q) { return s[sk(la + q)]; }, la, lb, k0);
    merge_steps<M, kE>(s, x, la, la + (k0 - x), la + lb, o);
  }
  __syncthreads();
  if (k0 < cnt) {
#pragma unroll
    for (int e = 0; e < kE; ++e) s[sk(k0 + e)] = o[e];
  }
  __syncthreads();
  for (int e = threadIdx.x; e < cnt; e += kThreads) dst[K0 + e] = s[sk(e)];
}

int merge_sort_passes(int64_t n) {
  if (n < 2) return 0;
  int p = 1;
  for (int64_t w = kTile; w < n; w <<= 1) ++p;
  return p;
}

// The launches of one sort: keys -> (tile passes) -> ping-pong through tmp;
// the result ends in keys (a copy when the pass count leaves it in tmp).
cudaError_t record_merge_sort(int variant, int32_t *keys, int32_t *tmp, int64_t n, cudaStream_t s, int *launches) {
  if (n <= 1) return cudaSuccess;
  const int N = int(n);
  const int tiles = (N + kTile - 1) / kTile;
  int32_t *cur = tmp, *other = keys;
  if (variant)
    merge_sort_tile_kernel<true><<<tiles, kThreads, 0, s>>>(keys, tmp, N);
  else
    merge_sort_tile_kernel<false><<<tiles, kThreads, 0, s>>>(keys, tmp, N);
  ++*launches;
  for (int64_t w = kTile; w < n; w <<= 1) {
    if (variant)
      merge_sort_pass_kernel<true><<<tiles, kThreads, 0, s>>>(cur, other, N, int(w));
    else
      merge_sort_pass_kernel<false><<<tiles, kThreads, 0, s>>>(cur, other, N, int(w));
    ++*launches;
    int32_t *t = cur;
    cur = other;
    other = t;
  }
  if (cur != keys) {
    cudaError_t e = cudaMemcpyAsync(keys, cur, size_t(n) * 4, cudaMemcpyDeviceToDevice, s);
    if (e != cudaSuccess) return e;
  }
  return cudaGetLastError();
}

}  // namespace darm_gpu
