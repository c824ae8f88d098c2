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
constexpr int LD = BS + 1;  // padded shared row: conflict-free column walks
}  // namespace

// ------------------------------------------------------------------ panel
// One launch per 16-column step: every CTA factors the 16x16 diagonal block
// (Doolittle: column i of L, then row i+1 of U — warp 0, lanes 0..15) into
// shared memory, CTA 0 writes it back, and each warp then solves one
// perimeter block pair p (row block right of the diagonal, column block below
// it) with the pair's 16 values per lane in registers.  Redundant diagonal
// factorisations replace a separate launch and a global round trip.
constexpr int kPairs = 4;

template <bool M>
__global__ void __launch_bounds__(32 * kPairs) lud_panel_kernel(float *__restrict__ a, int n, int o, int npairs) {
  __shared__ float dia[BS][LD];
  __shared__ float diaT[BS][LD];   // diaT[i][j] = dia[j][i]
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int e = threadIdx.x; e < BS * BS; e += blockDim.x)
    dia[e / BS][e % BS] = a[(size_t(o) + e / BS) * n + o + e % BS];
  __syncthreads();
  if (warp == 0) {
    const int tx = lane;
    for (int i = 0; i < BS - 1; ++i) {
      if (tx > i && tx < BS) {
        float x = dia[tx][i];
        for (int j = 0; j < i; ++j) x = fmaf(-dia[tx][j], dia[j][i], x);
        dia[tx][i] = x / dia[i][i];
      }
      __syncwarp();
      if (tx > i && tx < BS) {
        float x = dia[i + 1][tx];
        for (int j = 0; j < i + 1; ++j) x = fmaf(-dia[i + 1][j], dia[j][tx], x);
        dia[i + 1][tx] = x;
      }
      __syncwarp();
    }
  }
  __syncthreads();
  for (int e = threadIdx.x; e < BS * BS; e += blockDim.x) {
    diaT[e % BS][e / BS] = dia[e / BS][e % BS];
    if (blockIdx.x == 0 && e >= BS) a[(size_t(o) + e / BS) * n + o + e % BS] = dia[e / BS][e % BS];
  }
  __syncthreads();
  const int p = blockIdx.x * kPairs + warp;
  if (p >= npairs) return;                                 // warp-uniform
  const size_t cb = size_t(o) + size_t(BS) * (p + 1);      // column of the row block
  const size_t rb = cb;                                    // row of the column block
  if constexpr (!M) {
    if (lane < BS) {                                       // U12 = L11^-1 A12, column idx
      DARM_ARM("lud.row");
      const int idx = lane;
      float x[BS];
#pragma unroll
      for (int i = 0; i < BS; ++i) x[i] = a[(size_t(o) + i) * n + cb + idx];
#pragma unroll
      for (int i = 1; i < BS; ++i)
#pragma unroll
        for (int j = 0; j < i; ++j) x[i] = fmaf(-dia[i][j], x[j], x[i]);
#pragma unroll
      for (int i = 1; i < BS; ++i) a[(size_t(o) + i) * n + cb + idx] = x[i];
      DARM_ARM("lud.row.end");
    } else {                                               // L21 = A21 U11^-1, row idx
      DARM_ARM("lud.col");
      const int idx = lane - BS;
      float y[BS];
      const float4 *src = reinterpret_cast<const float4 *>(a + (rb + idx) * n + o);
#pragma unroll
      for (int q = 0; q < BS / 4; ++q) {
        const float4 v = src[q];
        y[4 * q] = v.x;
        y[4 * q + 1] = v.y;
        y[4 * q + 2] = v.z;
        y[4 * q + 3] = v.w;
      }
#pragma unroll
      for (int i = 0; i < BS; ++i) {
#pragma unroll
        for (int j = 0; j < i; ++j) y[i] = fmaf(-y[j], dia[j][i], y[i]);
        y[i] = y[i] / dia[i][i];
      }
      float4 *dst = reinterpret_cast<float4 *>(a + (rb + idx) * n + o);
#pragma unroll
      for (int q = 0; q < BS / 4; ++q) dst[q] = make_float4(y[4 * q], y[4 * q + 1], y[4 * q + 2], y[4 * q + 3]);
      DARM_ARM("lud.col.end");
    }
  } else {
    // Melded (by hand, as the paper did for LUD): one load / solve / store
    // sequence.  The role picks the global addresses (row role: column idx of
    // the row block, stride n; column role: row idx of the column block,
    // stride 1) and the diagonal operand (dia or its transpose, so both read
    // D[i][j]); fmaf(a,b,c) == fmaf(b,a,c), so -x[j] * D[i][j] is the same
    // operation as either arm's.  The column role's division is the only
    // one-sided run.
    const bool col = lane >= BS;
    const int idx = lane & (BS - 1);
    const float(*D)[LD] = col ? diaT : dia;
    const size_t g0 = col ? (rb + idx) * n + o : size_t(o) * n + cb + idx;
    const size_t gs = col ? 1 : size_t(n);
    float x[BS];
#pragma unroll
    for (int i = 0; i < BS; ++i) x[i] = a[g0 + i * gs];
#pragma unroll
    for (int i = 0; i < BS; ++i) {
#pragma unroll
      for (int j = 0; j < i; ++j) x[i] = fmaf(-x[j], D[i][j], x[i]);
      if (col) x[i] = x[i] / D[i][i];
    }
#pragma unroll
    for (int i = 0; i < BS; ++i)
      if (i > 0 || col) a[g0 + i * gs] = x[i];
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
// 64x64 tile per CTA; thread (tx, ty) owns rows ty + 16r (r < 4) and the 4
// consecutive columns 4tx..4tx+3; the element stays in registers across t.
constexpr int kLook = 4;   // steps per look-ahead super-step

struct Rect {
  int r_lo, r_hi, c_lo, c_hi;
};

__global__ void __launch_bounds__(256) lud_update_kernel(float *__restrict__ a, int n, int o, int T, Rect R0,
                                                         Rect R1) {
  __shared__ float colp[64][kLook * BS + 1];                   // L rows of the tile, (t,k)
  __shared__ __align__(16) float rowp[kLook * BS][64 + 4];     // U (t,k), columns of the tile
  const Rect R = blockIdx.z ? R1 : R0;
  const int r0 = R.r_lo + 64 * int(blockIdx.y), c0 = R.c_lo + 64 * int(blockIdx.x);
  if (r0 >= R.r_hi || c0 >= R.c_hi) return;                    // CTA-uniform
  const int nr = min(64, R.r_hi - r0), nc = min(64, R.c_hi - c0);
  const int K = T * BS;
  for (int e = threadIdx.x; e < 64 * K; e += 256) {
    const int r = e / K, k = e % K;
    colp[r][k] = r < nr ? a[size_t(r0 + r) * n + o + k] : 0.f;
    const int kk = e >> 6, c = e & 63;
    rowp[kk][c] = c < nc ? a[size_t(o + kk) * n + c0 + c] : 0.f;
  }
  __syncthreads();
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  const int c = 4 * tx;
  if (c >= nc) return;
  float4 v[4];
#pragma unroll
  for (int r = 0; r < 4; ++r)
    if (ty + 16 * r < nr) v[r] = *reinterpret_cast<const float4 *>(a + size_t(r0 + ty + 16 * r) * n + c0 + c);
  for (int t = 0; t < T; ++t) {
    float acc[4][4];
#pragma unroll
    for (int r = 0; r < 4; ++r)
#pragma unroll
      for (int q = 0; q < 4; ++q) acc[r][q] = 0.f;
#pragma unroll
    for (int k = 0; k < BS; ++k) {
      const float4 u = *reinterpret_cast<const float4 *>(&rowp[t * BS + k][c]);
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        const float l = colp[ty + 16 * r][t * BS + k];
        acc[r][0] = fmaf(l, u.x, acc[r][0]);
        acc[r][1] = fmaf(l, u.y, acc[r][1]);
        acc[r][2] = fmaf(l, u.z, acc[r][2]);
        acc[r][3] = fmaf(l, u.w, acc[r][3]);
      }
    }
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      v[r].x -= acc[r][0];
      v[r].y -= acc[r][1];
      v[r].z -= acc[r][2];
      v[r].w -= acc[r][3];
    }
  }
#pragma unroll
  for (int r = 0; r < 4; ++r)
    if (ty + 16 * r < nr) *reinterpret_cast<float4 *>(a + size_t(r0 + ty + 16 * r) * n + c0 + c) = v[r];
}

namespace {
cudaError_t launch_update(float *a, int n, int o, int T, Rect R0, Rect R1, cudaStream_t s) {
  auto tiles = [](int lo, int hi) { return hi > lo ? (hi - lo + 63) / 64 : 0; };
  const int gx = max(tiles(R0.c_lo, R0.c_hi), tiles(R1.c_lo, R1.c_hi));
  const int gy = max(tiles(R0.r_lo, R0.r_hi), tiles(R1.r_lo, R1.r_hi));
  const int gz = (R1.r_hi > R1.r_lo && R1.c_hi > R1.c_lo) ? 2 : 1;
  if (gx == 0 || gy == 0) return cudaSuccess;
  lud_update_kernel<<<dim3(gx, gy, gz), 256, 0, s>>>(a, n, o, T, R0, R1);
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
cudaError_t record_lud(int variant, float *a, int n, cudaStream_t s, int *launches) {
  const int nb = n / BS;
  for (int O = 0; O < n; O += kLook * BS) {
    const int T = min(kLook, (n - O) / BS);
    const int E = O + T * BS;   // end of the super-step's columns / rows
    for (int t = 0; t < T; ++t) {
      const int o = O + t * BS;
      const int m = nb - o / BS - 1;   // blocks right of / below the diagonal
      const int grid = m > 0 ? (m + kPairs - 1) / kPairs : 1;
      if (variant)
        lud_panel_kernel<true><<<grid, 32 * kPairs, 0, s>>>(a, n, o, m);
      else
        lud_panel_kernel<false><<<grid, 32 * kPairs, 0, s>>>(a, n, o, m);
      ++*launches;
      if (m == 0) break;
      const Rect panel_cols{o + BS, n, o + BS, E};   // rows below, panel columns
      const Rect super_row{o + BS, E, E, n};         // super-row rows, columns right
      cudaError_t e = launch_update(a, n, o, 1, panel_cols, super_row, s);
      if (e != cudaSuccess) return e;
      ++*launches;
    }
    if (E < n) {
      const Rect far{E, n, E, n};
      cudaError_t e = launch_update(a, n, O, T, far, Rect{0, 0, 0, 0}, s);
      if (e != cudaSuccess) return e;
      ++*launches;
    }
  }
  return cudaGetLastError();
}

}  // namespace darm_gpu
