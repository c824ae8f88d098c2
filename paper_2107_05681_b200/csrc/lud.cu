// lud.cu — blocked LU decomposition without pivoting (LUD, PAPER.md:765-768,
// 839), BLOCK = 16, fp32, in place: the unit-lower L below the diagonal and U
// on and above it.  The reference has no LUD code; the algorithm is Rodinia's
// three-kernel blocked scheme restated and the CPU oracle
// (oracle/darm_oracle.c, oracle_lud) performs the same floating-point
// operations in the same order, so GPU and CPU results agree bit for bit.
//
// Per 16-column step at offset o (two launches):
//   panel      factor A[o:o+16, o:o+16] (every CTA, in shared memory), then
//              U12 = L11^-1 A12 for every block right of the diagonal and
//              L21 = A21 U11^-1 for every block below it          (melded kernel)
//   update     A22 -= L21 U12, 16-term fp32 FMA chains             (64x64 tiles)
// with a look-ahead: four steps form a super-step and the far trailing block
// takes their four updates in one pass (same per-element operation order).
// The perimeter kernel is the paper's melding target: each warp owns one
// block pair, lanes 0-15 the row block and lanes 16-31 the column block, so
// the thread-ID test `lane < 16` splits every warp in half (divergent on a
// 32-wide warp only at BLOCK = 16).
//   unmelded: two arms (load / triangular solve / store), one per role;
//   melded:   hand-melded as the paper did for LUD: one load,
//             one solve and one store sequence whose addresses, shared-memory
//             operands and the role-only division are chosen per lane.
// The 2 x (n/16) launches are recorded once into a CUDA graph per (n, form,
// buffer) and replayed.
#include <cstdint>

#include "common.cuh"
#include "kernels.h"

namespace darm_gpu {

namespace {
constexpr int BS = 16;

// Two fp32 FMAs in one instruction (sm_100 FFMA2, fma.rn.f32x2): each half is
// an IEEE fma with one rounding, so the results equal two fmaf calls bit for
// bit; the FMA pipe issues half as many instructions.
__device__ __forceinline__ float2 fma2(float2 a, float2 b, float2 c) {
  unsigned long long ra, rb, rc, rd;
  asm("mov.b64 %0, {%1, %2};" : "=l"(ra) : "f"(a.x), "f"(a.y));
  asm("mov.b64 %0, {%1, %2};" : "=l"(rb) : "f"(b.x), "f"(b.y));
  asm("mov.b64 %0, {%1, %2};" : "=l"(rc) : "f"(c.x), "f"(c.y));
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(rd) : "l"(ra), "l"(rb), "l"(rc));
  float2 d;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(d.x), "=f"(d.y) : "l"(rd));
  return d;
}
constexpr int LD = BS + 1;  // padded shared row: conflict-free column walks
}  // namespace

// ------------------------------------------------------------------ panel
// One launch per 16-column step: every warp solves one perimeter block pair p
// (row block right of the diagonal, column block below it).  Latency first:
//   1. the pair's two 16x16 blocks are requested from HBM at kernel entry
//      (coalesced float4 loads into registers), and so is the diagonal block;
//   2. while they are in flight every warp factors the diagonal block in
//      registers (lane r holds row r; right-looking, U row k broadcast by
//      __shfl_sync) — per element the same fmaf(-L, U, x) sequence in
//      ascending k and the same division as the restatement's left-looking
//      Doolittle (oracle_lud), so the bits agree — and keeps a private
//      shared copy of it (no block barrier anywhere);
//   3. the blocks are staged in shared memory (the column block transposed),
//      so lane t of either role reads its 16 values at [i][t];
//   4. the divergent solve: lanes 0-15 U12 = L11^-1 A12 (one column each),
//      lanes 16-31 L21 = A21 U11^-1 (one row each) — the thread-ID split
//      `lane < 16` of the paper's perimeter kernel (divergent on a 32-wide
//      warp only at BLOCK = 16);
//   5. results go back through shared memory as coalesced float4 stores.
// The factored diagonal block goes to `dst` (CTA 0, row stride `dstride`):
// a scratch block while CTAs of this launch may still be reading the
// unfactored block from `a` (the next launch, lud_update_kernel, moves it
// into place), or straight into `a` for the last block (one CTA).
constexpr int kPairs = 4;

template <bool M>
__global__ void __launch_bounds__(32 * kPairs) lud_panel_kernel(float *__restrict__ a, int n, int o, int npairs,
                                                               float *__restrict__ dst, int dstride) {
  __shared__ float dia[kPairs][BS][LD];
  __shared__ float diaT[kPairs][BS][LD];      // diaT[i][j] = dia[j][i]
  __shared__ float blk[kPairs][2][BS][LD];    // [0] row block R[i][c]; [1] column block transposed C[i][r]
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int p = blockIdx.x * kPairs + warp;
  const bool have = p < npairs;                             // warp-uniform
  const size_t cb = size_t(o) + size_t(BS) * (p + 1);       // column of the row block = row of the column block
  // 1. requests in flight: the pair (2 float4 per lane per block) and the diagonal row of lane r
  float4 rv[2], cv[2];
  if (have) {
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int q = lane + 32 * h, i = q >> 2, c4 = q & 3;
      rv[h] = *reinterpret_cast<const float4 *>(a + (size_t(o) + i) * n + cb + 4 * c4);
      cv[h] = *reinterpret_cast<const float4 *>(a + (cb + i) * n + o + 4 * c4);
    }
  }
  const int r = lane & (BS - 1);
  float v[BS];
  {
    const float4 *src = reinterpret_cast<const float4 *>(a + (size_t(o) + r) * n + o);
#pragma unroll
    for (int q = 0; q < BS / 4; ++q) {
      const float4 t = src[q];
      v[4 * q] = t.x;
      v[4 * q + 1] = t.y;
      v[4 * q + 2] = t.z;
      v[4 * q + 3] = t.w;
    }
  }
  // 2. diagonal factorisation in registers
#pragma unroll
  for (int k = 0; k < BS - 1; ++k) {
    const float ukk = __shfl_sync(0xffffffffu, v[k], k);
    if (r > k) v[k] = v[k] / ukk;                           // L[r][k]
#pragma unroll
    for (int c = k + 1; c < BS; ++c) {
      const float ukc = __shfl_sync(0xffffffffu, v[c], k);  // U[k][c]
      if (r > k) v[c] = fmaf(-v[k], ukc, v[c]);
    }
  }
  if (lane < BS) {
#pragma unroll
    for (int c = 0; c < BS; ++c) {
      dia[warp][r][c] = v[c];
      diaT[warp][c][r] = v[c];
    }
    if (blockIdx.x == 0 && warp == 0) {
      float4 *d4 = reinterpret_cast<float4 *>(dst + size_t(r) * dstride);
#pragma unroll
      for (int q = 0; q < BS / 4; ++q) d4[q] = make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
    }
  }
  if (!have) return;                                        // warp-uniform
  // 3. stage the pair
  float(*R)[LD] = blk[warp][0];
  float(*C)[LD] = blk[warp][1];
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int q = lane + 32 * h, i = q >> 2, c = 4 * (q & 3);
    R[i][c] = rv[h].x;
    R[i][c + 1] = rv[h].y;
    R[i][c + 2] = rv[h].z;
    R[i][c + 3] = rv[h].w;
    C[c][i] = cv[h].x;
    C[c + 1][i] = cv[h].y;
    C[c + 2][i] = cv[h].z;
    C[c + 3][i] = cv[h].w;
  }
  __syncwarp();
  const float(*Dg)[LD] = dia[warp];
  // 4. the perimeter solve
  if constexpr (!M) {
    if (lane < BS) {                                        // U12 = L11^-1 A12, column idx
      DARM_ARM("lud.row");
      const int idx = lane;
      float x[BS];
#pragma unroll
      for (int i = 0; i < BS; ++i) x[i] = R[i][idx];
#pragma unroll
      for (int i = 1; i < BS; ++i)
#pragma unroll
        for (int j = 0; j < i; ++j) x[i] = fmaf(-Dg[i][j], x[j], x[i]);
#pragma unroll
      for (int i = 1; i < BS; ++i) R[i][idx] = x[i];
      DARM_ARM("lud.row.end");
    } else {                                                // L21 = A21 U11^-1, row idx
      DARM_ARM("lud.col");
      const int idx = lane - BS;
      float y[BS];
#pragma unroll
      for (int i = 0; i < BS; ++i) y[i] = C[i][idx];
#pragma unroll
      for (int i = 0; i < BS; ++i) {
#pragma unroll
        for (int j = 0; j < i; ++j) y[i] = fmaf(-y[j], Dg[j][i], y[i]);
        y[i] = y[i] / Dg[i][i];
      }
#pragma unroll
      for (int i = 0; i < BS; ++i) C[i][idx] = y[i];
      DARM_ARM("lud.col.end");
    }
  } else {
    // Melded (by hand, as the paper did for LUD): one
    // load / solve / store sequence.  The role picks the staged block (both
    // read [i][idx]) and the diagonal operand (dia or its transpose, so both
    // read D[i][j]); fmaf(a,b,c) == fmaf(b,a,c), so -x[j] * D[i][j] is the same
    // operation as either arm's.  The column role's division is the only
    // one-sided run.
    const bool col = lane >= BS;
    const int idx = lane & (BS - 1);
    float(*S)[LD] = col ? C : R;
    const float(*D)[LD] = col ? diaT[warp] : dia[warp];
    float x[BS];
#pragma unroll
    for (int i = 0; i < BS; ++i) x[i] = S[i][idx];
#pragma unroll
    for (int i = 0; i < BS; ++i) {
#pragma unroll
      for (int j = 0; j < i; ++j) x[i] = fmaf(-x[j], D[i][j], x[i]);
      if (col) x[i] = x[i] / D[i][i];
    }
#pragma unroll
    for (int i = 0; i < BS; ++i) S[i][idx] = x[i];
  }
  __syncwarp();
  // 5. coalesced write-back of both blocks
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int q = lane + 32 * h, i = q >> 2, c = 4 * (q & 3);
    if (i > 0) *reinterpret_cast<float4 *>(a + (size_t(o) + i) * n + cb + c) = make_float4(R[i][c], R[i][c + 1], R[i][c + 2], R[i][c + 3]);
    *reinterpret_cast<float4 *>(a + (cb + i) * n + o + c) = make_float4(C[c][i], C[c + 1][i], C[c + 2][i], C[c + 3][i]);
  }
}

// ------------------------------------------------------------------ update
// Trailing updates A[r][c] -= sum_k L_t[r][k] U_t[k][c] for the T consecutive
// 16-column steps t at offsets o + 16t, applied in step order to every element
// of up to two rectangles (rows [r_lo, r_hi) x cols [c_lo, c_hi), multiples of
// 16): per element and step, sum = fma(L[r][k], U[k][c], sum) for k = 0..15
// and then a = a - sum — exactly the per-element sequence of one
// 16-column step after another, so deferring the far trailing block's T
// updates into one pass over it (look-ahead) leaves every bit unchanged while
// the trailing matrix crosses HBM once per 64 columns instead of once per 16.
// 64x64 tile per CTA, L (transposed) and U panels staged in shared memory;
// thread (tx, ty) owns the 4x4 micro-tile rows 4ty.., columns 4tx.., so each
// k costs two 16-byte shared loads for 16 FMAs; the element stays in registers
// across t.  CTA (0,0,0) also moves the previous panel launch's factored
// diagonal block from `dsrc` into place (nothing this launch touches reads it).
constexpr int kLook = 4;   // steps per look-ahead super-step

struct Rect {
  int r_lo, r_hi, c_lo, c_hi;
};

__global__ void __launch_bounds__(256) lud_update_kernel(float *__restrict__ a, int n, int o, int T, Rect R0,
                                                         Rect R1, const float *__restrict__ dsrc, int dofs) {
  __shared__ __align__(16) float lt[kLook * BS][64 + 4];      // lt[(t,k)][r] = L_t[r][k]
  __shared__ __align__(16) float up[kLook * BS][64 + 4];      // up[(t,k)][c] = U_t[k][c]
  if (dsrc && blockIdx.x == 0 && blockIdx.y == 0 && blockIdx.z == 0) {
    const int e = threadIdx.x;                                  // 256 = 16 x 16
    a[size_t(dofs + e / BS) * n + dofs + e % BS] = dsrc[e];
  }
  const Rect R = blockIdx.z ? R1 : R0;
  const int r0 = R.r_lo + 64 * int(blockIdx.y), c0 = R.c_lo + 64 * int(blockIdx.x);
  if (r0 >= R.r_hi || c0 >= R.c_hi) return;                    // CTA-uniform
  const int nr = min(64, R.r_hi - r0), nc = min(64, R.c_hi - c0);
  const int K = T * BS, K4 = K / 4;
  // L: float4 along k from row r (lanes walk rows: conflict-free transposed stores)
  for (int e = threadIdx.x; e < 64 * K4; e += 256) {
    const int rr = e & 63, k4 = e >> 6;
    float4 l = make_float4(0.f, 0.f, 0.f, 0.f);
    if (rr < nr) l = *reinterpret_cast<const float4 *>(a + size_t(r0 + rr) * n + o + 4 * k4);
    lt[4 * k4][rr] = l.x;
    lt[4 * k4 + 1][rr] = l.y;
    lt[4 * k4 + 2][rr] = l.z;
    lt[4 * k4 + 3][rr] = l.w;
  }
  // U: float4 along c
  for (int e = threadIdx.x; e < K * 16; e += 256) {
    const int kk = e >> 4, c4 = e & 15;
    float4 u = make_float4(0.f, 0.f, 0.f, 0.f);
    if (4 * c4 < nc) u = *reinterpret_cast<const float4 *>(a + size_t(o + kk) * n + c0 + 4 * c4);
    *reinterpret_cast<float4 *>(&up[kk][4 * c4]) = u;
  }
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  const int c = 4 * tx, rb = 4 * ty;
  const bool live = c < nc && rb < nr;
  float4 v[4];
  if (live) {
#pragma unroll
    for (int i = 0; i < 4; ++i) v[i] = *reinterpret_cast<const float4 *>(a + size_t(r0 + rb + i) * n + c0 + c);
  }
  __syncthreads();
  if (!live) return;
  for (int t = 0; t < T; ++t) {
    float acc[4][4];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int q = 0; q < 4; ++q) acc[i][q] = 0.f;
#pragma unroll
    for (int k = 0; k < BS; ++k) {
      const float4 u = *reinterpret_cast<const float4 *>(&up[t * BS + k][c]);
      const float4 l = *reinterpret_cast<const float4 *>(&lt[t * BS + k][rb]);
      const float lv[4] = {l.x, l.y, l.z, l.w};
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        acc[i][0] = fmaf(lv[i], u.x, acc[i][0]);
        acc[i][1] = fmaf(lv[i], u.y, acc[i][1]);
        acc[i][2] = fmaf(lv[i], u.z, acc[i][2]);
        acc[i][3] = fmaf(lv[i], u.w, acc[i][3]);
      }
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      v[i].x -= acc[i][0];
      v[i].y -= acc[i][1];
      v[i].z -= acc[i][2];
      v[i].w -= acc[i][3];
    }
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) *reinterpret_cast<float4 *>(a + size_t(r0 + rb + i) * n + c0 + c) = v[i];
}

constexpr int kFarRows = 128, kFarCols = 64;   // far-update tile

// The far trailing block's T-step update (the bulk of the FLOPs), persistent:
// one CTA per SM walks the 128x64 tiles
// of the far block; every tile's L rows (non-transposed, 16-byte chunks along
// k), U rows and the tile of A itself are brought into shared memory with
// cp.async while the previous tile computes (two stages).  Per 4 k's a thread
// reads 8 float4 of L (its 8 rows) and 4 float4 of U (its 4 columns) for 64
// FFMA2.  Same per-element operation sequence as lud_update_kernel.
constexpr int kPipeK = kLook * BS;                 // 64
constexpr int kLdL = kPipeK + 4;                   // lp[r][k] row pitch
constexpr int kLdU = kFarCols + 4;                 // up[k][c]
constexpr int kLdV = kFarCols + 4;                 // vt[r][c]
constexpr int kStageWords = kFarRows * kLdL + kPipeK * kLdU + kFarRows * kLdV;

__device__ __forceinline__ void cp_async16(void *smem, const void *gmem, bool valid) {
  const unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  const int bytes = valid ? 16 : 0;                // 0: zero-fill
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(sa), "l"(gmem), "r"(bytes) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory"); }

__global__ void __launch_bounds__(256, 1) lud_far_pipe_kernel(float *__restrict__ a, int n, int o, int T, int lo) {
  extern __shared__ __align__(16) float psm[];
  const int m = n - lo;
  const int tiles_c = (m + kFarCols - 1) / kFarCols, tiles_r = (m + kFarRows - 1) / kFarRows;
  const int tiles = tiles_c * tiles_r;
  const int K = T * BS, K4 = K / 4;
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  const int c = 4 * tx, rb = 8 * ty;
  auto stage_ptr = [&](int st) { return psm + size_t(st) * kStageWords; };
  auto issue = [&](int tile, int st) {
    float *lp = stage_ptr(st), *up = lp + kFarRows * kLdL, *vt = up + kPipeK * kLdU;
    const int r0 = lo + kFarRows * (tile / tiles_c), c0 = lo + kFarCols * (tile % tiles_c);
    const int nr = min(kFarRows, n - r0), nc = min(kFarCols, n - c0);
    for (int e = threadIdx.x; e < kFarRows * K4; e += 256) {          // L rows of the tile, k along
      const int r = e / K4, k4 = e % K4;
      const bool ok = r < nr;
      cp_async16(lp + r * kLdL + 4 * k4, a + size_t(ok ? r0 + r : r0) * n + o + 4 * k4, ok);
    }
    for (int e = threadIdx.x; e < K * (kFarCols / 4); e += 256) {      // U rows, columns of the tile
      const int kk = e / (kFarCols / 4), c4 = e % (kFarCols / 4);
      const bool ok = 4 * c4 < nc;
      cp_async16(up + kk * kLdU + 4 * c4, a + size_t(o + kk) * n + (ok ? c0 + 4 * c4 : c0), ok);
    }
    for (int e = threadIdx.x; e < kFarRows * (kFarCols / 4); e += 256) {   // the tile of A
      const int r = e / (kFarCols / 4), c4 = e % (kFarCols / 4);
      const bool ok = r < nr && 4 * c4 < nc;
      cp_async16(vt + r * kLdV + 4 * c4, a + size_t(ok ? r0 + r : r0) * n + (ok ? c0 + 4 * c4 : c0), ok);
    }
    cp_async_commit();
  };
  int tile = blockIdx.x;
  if (tile < tiles) issue(tile, 0);
  for (int it = 0; tile < tiles; tile += gridDim.x, ++it) {
    const int st = it & 1;
    const int next = tile + gridDim.x;
    if (next < tiles) {
      issue(next, st ^ 1);
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();
    const float *lp = stage_ptr(st), *up = lp + kFarRows * kLdL, *vt = up + kPipeK * kLdU;
    const int r0 = lo + kFarRows * (tile / tiles_c), c0 = lo + kFarCols * (tile % tiles_c);
    const int nr = min(kFarRows, n - r0), nc = min(kFarCols, n - c0);
    float4 v[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) v[i] = *reinterpret_cast<const float4 *>(vt + (rb + i) * kLdV + c);
    for (int t = 0; t < T; ++t) {
      float2 acc[8][2];
#pragma unroll
      for (int i = 0; i < 8; ++i) acc[i][0] = acc[i][1] = make_float2(0.f, 0.f);
#pragma unroll
      for (int k4 = 0; k4 < BS / 4; ++k4) {
        const int kb = t * BS + 4 * k4;
        float4 l[8], u[4];
#pragma unroll
        for (int i = 0; i < 8; ++i) l[i] = *reinterpret_cast<const float4 *>(lp + (rb + i) * kLdL + kb);
#pragma unroll
        for (int q = 0; q < 4; ++q) u[q] = *reinterpret_cast<const float4 *>(up + (kb + q) * kLdU + c);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const float2 u01 = make_float2(u[q].x, u[q].y), u23 = make_float2(u[q].z, u[q].w);
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const float li = q == 0 ? l[i].x : q == 1 ? l[i].y : q == 2 ? l[i].z : l[i].w;
            const float2 ll = make_float2(li, li);
            acc[i][0] = fma2(ll, u01, acc[i][0]);
            acc[i][1] = fma2(ll, u23, acc[i][1]);
          }
        }
      }
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        v[i].x -= acc[i][0].x;
        v[i].y -= acc[i][0].y;
        v[i].z -= acc[i][1].x;
        v[i].w -= acc[i][1].y;
      }
    }
    if (c < nc) {
#pragma unroll
      for (int i = 0; i < 8; ++i)
        if (rb + i < nr) *reinterpret_cast<float4 *>(a + size_t(r0 + rb + i) * n + c0 + c) = v[i];
    }
    __syncthreads();   // this stage is refilled by the next iteration's issue
  }
}

namespace {
cudaError_t launch_update(float *a, int n, int o, int T, Rect R0, Rect R1, const float *dsrc, int dofs,
                          cudaStream_t s) {
  auto tiles = [](int lo, int hi) { return hi > lo ? (hi - lo + 63) / 64 : 0; };
  int gx = max(tiles(R0.c_lo, R0.c_hi), tiles(R1.c_lo, R1.c_hi));
  int gy = max(tiles(R0.r_lo, R0.r_hi), tiles(R1.r_lo, R1.r_hi));
  const int gz = (R1.r_hi > R1.r_lo && R1.c_hi > R1.c_lo) ? 2 : 1;
  if (gx == 0 || gy == 0) {
    if (!dsrc) return cudaSuccess;
    gx = gy = 1;                                   // still move the diagonal block
  }
  lud_update_kernel<<<dim3(gx, gy, gz), 256, 0, s>>>(a, n, o, T, R0, R1, dsrc, dofs);
  return cudaGetLastError();
}
}  // namespace

// ------------------------------------------------------------------ driver
// Super-steps of kLook 16-column steps at offset O.  For each step t in the
// super-step: the panel kernel (diagonal + perimeter over everything right of
// / below the diagonal block), then step t's update restricted to what the
// later steps of the super-step read — the panel columns [o_t+16, O+64) for
// all rows below, and the super-row rows [o_t+16, O+64) for all columns to
// the right.  The far trailing block [O+64, n)^2 then takes the super-step's
// kLook updates in one pass (lud_update_kernel with T = kLook).
cudaError_t record_lud(int variant, float *a, int n, float *dscr, cudaStream_t s, int *launches) {
  const int nb = n / BS;
  for (int O = 0; O < n; O += kLook * BS) {
    const int T = min(kLook, (n - O) / BS);
    const int E = O + T * BS;   // end of the super-step's columns / rows
    for (int t = 0; t < T; ++t) {
      const int o = O + t * BS;
      const int m = nb - o / BS - 1;   // blocks right of / below the diagonal
      const int grid = m > 0 ? (m + kPairs - 1) / kPairs : 1;
      // the last diagonal block has no other reader: factor it in place
      float *dst = m > 0 ? dscr : a + size_t(o) * n + o;
      const int dstride = m > 0 ? BS : n;
      if (variant)
        lud_panel_kernel<true><<<grid, 32 * kPairs, 0, s>>>(a, n, o, m, dst, dstride);
      else
        lud_panel_kernel<false><<<grid, 32 * kPairs, 0, s>>>(a, n, o, m, dst, dstride);
      ++*launches;
      if (m == 0) break;
      const Rect panel_cols{o + BS, n, o + BS, E};   // rows below, panel columns
      const Rect super_row{o + BS, E, E, n};         // super-row rows, columns right
      cudaError_t e = launch_update(a, n, o, 1, panel_cols, super_row, dscr, o, s);
      if (e != cudaSuccess) return e;
      ++*launches;
    }
    if (E < n) {
      // the far trailing block [E, n)^2 takes the super-step's T updates
      const int m = n - E;
      const size_t shm = 2 * size_t(kStageWords) * sizeof(float);
      static int sms = 0;
      if (!sms) {
        cudaError_t e = cudaFuncSetAttribute(lud_far_pipe_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             int(shm));
        if (e != cudaSuccess) return e;
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        if (sms <= 0) sms = 148;
      }
      const int tiles = ((m + kFarCols - 1) / kFarCols) * ((m + kFarRows - 1) / kFarRows);
      lud_far_pipe_kernel<<<min(tiles, sms), 256, shm, s>>>(a, n, O, T, E);
      cudaError_t e = cudaGetLastError();
      if (e != cudaSuccess) return e;
      ++*launches;
    }
  }
  return cudaGetLastError();
}

}  // namespace darm_gpu
