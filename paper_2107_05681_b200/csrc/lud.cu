// lud.cu — blocked LU decomposition without pivoting (LUD, PAPER.md:765-768,
// 839), BLOCK = 16, fp32, in place: the unit-lower L below the diagonal and U
// on and above it.  The reference has no LUD code; the algorithm is Rodinia's
// three-kernel blocked scheme restated and the CPU oracle
// (oracle/darm_oracle.c, oracle_lud) performs the same floating-point
// operations in the same order, so GPU and CPU results agree bit for bit.
//
// Per 16-column step at offset o:
//   diagonal   factor A[o:o+16, o:o+16]                          (1 CTA)
//   perimeter  U12 = L11^-1 A12 for every block right of the diagonal and
//              L21 = A21 U11^-1 for every block below it          (melded kernel)
//   internal   A22 -= L21 U12, 16-term fp32 FMA chains             (64x64 tiles)
// The perimeter kernel is the paper's melding target: each warp owns one
// block pair, lanes 0-15 the row block and lanes 16-31 the column block, so
// the thread-ID test `lane < 16` splits every warp in half (divergent on a
// 32-wide warp only at BLOCK = 16).
//   unmelded: two arms (load / triangular solve / store), one per role;
//   melded:   hand-melded as the paper did for LUD: one load,
//             one solve and one store sequence whose addresses, shared-memory
//             operands and the role-only division are chosen per lane.
// The 3 x (n/16) launches are recorded once into a CUDA graph per (n, form,
// buffer) and replayed.
#include <cstdint>

#include "common.cuh"
#include "kernels.h"

namespace darm_gpu {

namespace {
constexpr int BS = 16;
constexpr int LD = BS + 1;  // padded shared row: conflict-free column walks
}  // namespace

// ------------------------------------------------------------------ diagonal
// Doolittle on the 16x16 diagonal block; column i of L then row i+1 of U.
__global__ void __launch_bounds__(BS) lud_diagonal_kernel(float *__restrict__ a, int n, int o) {
  __shared__ float s[BS][LD];
  const int tx = threadIdx.x;
  const float *blk = a + size_t(o) * n + o;
  for (int i = 0; i < BS; ++i) s[i][tx] = blk[size_t(i) * n + tx];
  __syncthreads();
  for (int i = 0; i < BS - 1; ++i) {
    if (tx > i) {
      float x = s[tx][i];
      for (int j = 0; j < i; ++j) x = fmaf(-s[tx][j], s[j][i], x);
      s[tx][i] = x / s[i][i];
    }
    __syncthreads();
    if (tx > i) {
      float x = s[i + 1][tx];
      for (int j = 0; j < i + 1; ++j) x = fmaf(-s[i + 1][j], s[j][tx], x);
      s[i + 1][tx] = x;
    }
    __syncthreads();
  }
  float *out = a + size_t(o) * n + o;
  for (int i = 1; i < BS; ++i) out[size_t(i) * n + tx] = s[i][tx];
}

// ------------------------------------------------------------------ perimeter
// One warp per block pair p (row block right of the diagonal, column block
// below it); kPairs warps per CTA share the diagonal block.
constexpr int kPairs = 4;

template <bool M>
__global__ void __launch_bounds__(32 * kPairs) lud_perimeter_kernel(float *__restrict__ a, int n, int o,
                                                                   int npairs) {
  __shared__ float dia[BS][LD];
  __shared__ float peri_row[kPairs][BS][LD];   // [pair][i][idx]  = A[o+i][cb+idx]
  __shared__ float peri_col[kPairs][BS][LD];   // [pair][i][idx]  = A[rb+i][o+idx]
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int p = blockIdx.x * kPairs + warp;   // pair index; block column/row (p+1)
  const bool live = p < npairs;
  const size_t cb = size_t(o) + size_t(BS) * (p + 1);   // column of the row block
  const size_t rb = cb;                                   // row of the column block
  // diagonal block, shared by the CTA's warps
  for (int e = threadIdx.x; e < BS * BS; e += blockDim.x)
    dia[e / BS][e % BS] = a[(size_t(o) + e / BS) * n + o + e % BS];
  float(*prow)[LD] = peri_row[warp];
  float(*pcol)[LD] = peri_col[warp];
  if constexpr (!M) {
    if (live) {
      if (lane < BS) {                                   // row role
        DARM_ARM("lud.row.load");
        const int idx = lane;
        for (int i = 0; i < BS; ++i) prow[i][idx] = a[(size_t(o) + i) * n + cb + idx];
        DARM_ARM("lud.row.load.end");
      } else {                                           // column role
        DARM_ARM("lud.col.load");
        const int idx = lane - BS;
        for (int i = 0; i < BS; ++i) pcol[i][idx] = a[(rb + i) * n + o + idx];
        DARM_ARM("lud.col.load.end");
      }
    }
    __syncthreads();
    if (live) {
      if (lane < BS) {                                   // U12 = L11^-1 A12
        DARM_ARM("lud.row.solve");
        const int idx = lane;
        for (int i = 1; i < BS; ++i) {
          float x = prow[i][idx];
          for (int j = 0; j < i; ++j) x = fmaf(-dia[i][j], prow[j][idx], x);
          prow[i][idx] = x;
        }
        DARM_ARM("lud.row.solve.end");
      } else {                                           // L21 = A21 U11^-1
        DARM_ARM("lud.col.solve");
        const int idx = lane - BS;
        for (int i = 0; i < BS; ++i) {
          float x = pcol[idx][i];
          for (int j = 0; j < i; ++j) x = fmaf(-pcol[idx][j], dia[j][i], x);
          pcol[idx][i] = x / dia[i][i];
        }
        DARM_ARM("lud.col.solve.end");
      }
    }
    __syncwarp();
    if (live) {
      if (lane < BS) {
        DARM_ARM("lud.row.store");
        const int idx = lane;
        for (int i = 1; i < BS; ++i) a[(size_t(o) + i) * n + cb + idx] = prow[i][idx];
        DARM_ARM("lud.row.store.end");
      } else {
        DARM_ARM("lud.col.store");
        const int idx = lane - BS;
        for (int i = 0; i < BS; ++i) a[(rb + i) * n + o + idx] = pcol[i][idx];
        DARM_ARM("lud.col.store.end");
      }
    }
  } else {
    // Melded: lane role r = lane >= 16 selects addresses; the loops, loads,
    // FMAs and stores are shared.  The row solve runs i = 0..15 with an empty
    // i = 0 step (j < 0); fmaf(a,b,c) == fmaf(b,a,c), so the column role's
    // pcol[idx][j] * dia[j][i] is the same operation as -X(j) * D(i,j) with
    // D the role-transposed diagonal access.
    const bool col = lane >= BS;
    const int idx = lane & (BS - 1);
    float *X = col ? &pcol[idx][0] : &prow[0][idx];       // X(i) = X[i * xs]
    const int xs = col ? 1 : LD;
    float *L = col ? &pcol[0][idx] : &prow[0][idx];       // load/store slots [i*LD]
    const size_t g0 = col ? rb * n + o + idx : size_t(o) * n + cb + idx;
    const int di = col ? 1 : LD, dj = col ? LD : 1;       // D(i,j) = dia[i*di + j*dj]
    const float *D = &dia[0][0];
    if (live)
      for (int i = 0; i < BS; ++i) L[i * LD] = a[g0 + size_t(i) * n];
    __syncthreads();
    if (live) {
      for (int i = 0; i < BS; ++i) {
        float x = X[i * xs];
        for (int j = 0; j < i; ++j) x = fmaf(-X[j * xs], D[i * di + j * dj], x);
        if (col) x = x / D[i * LD + i];                  // column-role-only run
        X[i * xs] = x;
      }
    }
    __syncwarp();
    if (live)
      for (int i = col ? 0 : 1; i < BS; ++i) a[g0 + size_t(i) * n] = L[i * LD];
  }
}

// ------------------------------------------------------------------ internal
// A22 -= L21 U12 over 64x64 tiles (4x4 blocks); thread (tx, ty) owns rows
// ty + 16r (r < 4) and the 4 consecutive columns 4tx..4tx+3 of its tile.
// Per element: sum = fma(L[r][k], U[k][c], sum) for k = 0..15, then a -= sum.
__global__ void __launch_bounds__(256) lud_internal_kernel(float *__restrict__ a, int n, int o, int mb) {
  __shared__ float colp[64][LD];                   // L21 rows of the tile, k
  __shared__ __align__(16) float rowp[BS][64 + 4]; // U12 k, columns of the tile
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  const int bi = blockIdx.y * 4, bj = blockIdx.x * 4;   // first 16-block of the tile
  const int nbr = min(4, mb - bi), nbc = min(4, mb - bj);
  const size_t r0 = size_t(o) + BS * (1 + bi), c0 = size_t(o) + BS * (1 + bj);
  for (int e = threadIdx.x; e < 64 * BS; e += 256) {
    const int r = e >> 4, k = e & 15;
    colp[r][k] = (r < nbr * BS) ? a[(r0 + r) * n + o + k] : 0.f;
    const int kk = e >> 6, c = e & 63;
    rowp[kk][c] = (c < nbc * BS) ? a[(size_t(o) + kk) * n + c0 + c] : 0.f;
  }
  __syncthreads();
  const int c = 4 * tx;
  if (c >= nbc * BS) return;
  float acc[4][4];
#pragma unroll
  for (int r = 0; r < 4; ++r)
#pragma unroll
    for (int q = 0; q < 4; ++q) acc[r][q] = 0.f;
#pragma unroll
  for (int k = 0; k < BS; ++k) {
    const float4 u = *reinterpret_cast<const float4 *>(&rowp[k][c]);
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const float l = colp[ty + 16 * r][k];
      acc[r][0] = fmaf(l, u.x, acc[r][0]);
      acc[r][1] = fmaf(l, u.y, acc[r][1]);
      acc[r][2] = fmaf(l, u.z, acc[r][2]);
      acc[r][3] = fmaf(l, u.w, acc[r][3]);
    }
  }
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    const int rr = ty + 16 * r;
    if (rr < nbr * BS) {
      float4 *pa = reinterpret_cast<float4 *>(a + (r0 + rr) * n + c0 + c);
      float4 v = *pa;
      v.x -= acc[r][0];
      v.y -= acc[r][1];
      v.z -= acc[r][2];
      v.w -= acc[r][3];
      *pa = v;
    }
  }
}

// ------------------------------------------------------------------ driver
cudaError_t record_lud(int variant, float *a, int n, cudaStream_t s, int *launches) {
  const int nb = n / BS;
  for (int step = 0; step < nb; ++step) {
    const int o = step * BS;
    lud_diagonal_kernel<<<1, BS, 0, s>>>(a, n, o);
    ++*launches;
    const int m = nb - step - 1;   // trailing blocks
    if (m == 0) break;
    const int grid = (m + kPairs - 1) / kPairs;
    if (variant)
      lud_perimeter_kernel<true><<<grid, 32 * kPairs, 0, s>>>(a, n, o, m);
    else
      lud_perimeter_kernel<false><<<grid, 32 * kPairs, 0, s>>>(a, n, o, m);
    const int t = (m + 3) / 4;
    lud_internal_kernel<<<dim3(t, t), 256, 0, s>>>(a, n, o, m);
    *launches += 2;
  }
  return cudaGetLastError();
}

}  // namespace darm_gpu
