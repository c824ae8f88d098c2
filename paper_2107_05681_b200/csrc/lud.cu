// lud.cu — blocked LU decomposition without pivoting (LUD, PAPER.md:765-768,
// 839), BLOCK = 16, fp32, in place: the unit-lower L below the diagonal and U
// on and above it.  The reference has no LUD code; the algorithm is Rodinia's
// three-kernel blocked scheme restated and the CPU oracle
// (oracle/darm_oracle.c, oracle_lud) performs the same floating-point
// operations in the same order, so GPU and CPU results agree bit for bit.
//
// Per 16-column step at offset o, one panel launch: apply the step's pending
// updates to the blocks it reads, factor A[o:o+16, o:o+16] (every warp, in
// registers), then U12 = L11^-1 A12 for every block right of the diagonal and
// L21 = A21 U11^-1 for every block below it (the melded kernel).  Four steps
// form a super-step; the trailing matrix takes their four updates in one
// pass (A22 -= L21 U12 as 16-term fp32 FMA chains, same per-element operation
// order): the 64-wide band the next super-step's panels read, followed by
// those panels on a side stream, beside the far block (record_lud).
// The perimeter kernel is the paper's melding target: each warp owns one
// block pair, lanes 0-15 the row block and lanes 16-31 the column block, so
// the thread-ID test `lane < 16` splits every warp in half (divergent on a
// 32-wide warp only at BLOCK = 16).
//   unmelded: two arms (load / triangular solve / store), one per role;
//   melded:   hand-melded as the paper did for LUD: one load,
//             one solve and one store sequence whose addresses, shared-memory
//             operands and the role-only division are chosen per lane.
// The n/16 + 2 n/64 + 1 launches are recorded once into a CUDA graph per (n,
// form, buffer) and replayed.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cstdint>

#include "common.cuh"
#include "kernels.h"

namespace darm_gpu {

namespace {
constexpr int BS = 16;
constexpr int kLook = 4;   // steps per look-ahead super-step

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
// a scratch slot while CTAs of this launch may still be reading the
// unfactored block from `a` (lud_scatter_diag_kernel moves them all into place
// at the end; no later kernel reads a factored diagonal block), or straight
// into `a` for the last block (one CTA).
constexpr int kPairs = 4;

// Pending updates (left-looking inside a super-step): the blocks a panel
// reads still lack the updates of the earlier steps O, O+16, .., o-16 of its
// super-step; the panel applies them itself, per element in step order as
// sum = fma(L, U, sum) over k = 0..15 then a -= sum — the per-element sequence
// of the separate update kernel it replaces.  L / U come from the earlier
// steps' column / row blocks, already final.  Shared layout (dynamic):
//   Lp[16][kLdP]   rows o..o+15, columns O..o   (the diagonal rows' L)
//   UdT[16][kLdP]  U above the diagonal block, transposed: UdT[c][k] = U[O+k][o+c]
//   per warp UrT[16][kLdP] (U above its row block, transposed) and Lc[16][kLdP]
//   (its column block's L)
// Every operand row is contiguous along k, so the sums read float4s.
constexpr int kMaxPend = kLook - 1;
constexpr int kLdP = kMaxPend * BS + 4;   // 52: float4 rows, 16 rows on distinct bank quads but for pairs
constexpr int kPendFloats = 2 * BS * kLdP + kPairs * 2 * BS * kLdP;

template <bool M, int P>   // P: pending steps of the super-step (0..kLook-1), compile-time
__global__ void __launch_bounds__(32 * kPairs) lud_panel_kernel(float *__restrict__ a, int n, int o, int npairs, int O,
                                                               float *__restrict__ dst, int dstride) {
  __shared__ float dia[BS][LD];               // the factored diagonal block (warp 0 of the CTA)
  __shared__ float diaT[BS][LD];              // diaT[i][j] = dia[j][i]
  __shared__ float blk[kPairs][2][BS][LD];    // [0] row block R[i][c]; [1] column block transposed C[i][r]
  // pending-update operands, static (sized for kMaxPend): the compiler then
  // addresses them in the shared window directly instead of re-deriving a
  // generic base for a dynamic array at every access
  __shared__ __align__(16) float pend[kPendFloats];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int p = blockIdx.x * kPairs + warp;
  const bool have = p < npairs;                             // warp-uniform
  const size_t cb = size_t(o) + size_t(BS) * (p + 1);       // column of the row block = row of the column block
  float(*Lp)[kLdP] = reinterpret_cast<float(*)[kLdP]>(pend);
  float(*UdT)[kLdP] = reinterpret_cast<float(*)[kLdP]>(pend + BS * kLdP);
  float(*UrT)[kLdP] = reinterpret_cast<float(*)[kLdP]>(pend + 2 * BS * kLdP + warp * 2 * BS * kLdP);
  float(*Lc)[kLdP] = reinterpret_cast<float(*)[kLdP]>(pend + 3 * BS * kLdP + warp * 2 * BS * kLdP);
  // 1. every global read of the launch in flight at once (one memory round
  //    trip): the pair (2 float4 per lane per block), the diagonal row of lane
  //    r, and the pending updates' L and U (float4 chunks, fixed counts)
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
  if (warp == 0) {
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
  if constexpr (P > 0) {
    constexpr int K = P * BS, K4 = K / 4, NT = 32 * kPairs;
    constexpr int nL = BS * K4, nU = K * (BS / 4);            // float4 chunks of Lp / Ud (CTA-wide)
    constexpr int nW = K * (BS / 4) / 32;                     // chunks of Ur and of Lc per lane
    static_assert(nW * 32 == K * (BS / 4) && BS * K4 == K * (BS / 4), "chunk counts");
    float4 lb[(nL + NT - 1) / NT], ub[(nU + NT - 1) / NT], urb[nW], lcb[nW];
#pragma unroll
    for (int j = 0; j < (nL + NT - 1) / NT; ++j) {
      const int e = int(threadIdx.x) + NT * j;
      if (e < nL) lb[j] = *reinterpret_cast<const float4 *>(a + (size_t(o) + e / K4) * n + O + 4 * (e % K4));
    }
#pragma unroll
    for (int j = 0; j < (nU + NT - 1) / NT; ++j) {
      const int e = int(threadIdx.x) + NT * j;
      if (e < nU) ub[j] = *reinterpret_cast<const float4 *>(a + (size_t(O) + e / 4) * n + o + 4 * (e % 4));
    }
    if (have) {
#pragma unroll
      for (int j = 0; j < nW; ++j) {
        const int e = lane + 32 * j;
        urb[j] = *reinterpret_cast<const float4 *>(a + (size_t(O) + e / 4) * n + cb + 4 * (e % 4));
        lcb[j] = *reinterpret_cast<const float4 *>(a + (cb + e / K4) * n + O + 4 * (e % K4));
      }
    }
    auto put = [](float *d, float4 x) { *reinterpret_cast<float4 *>(d) = x; };
    auto put_t = [](float (*d)[kLdP], int c, int k, float4 x) {   // d[c + i][k] = x[i]
      d[c][k] = x.x;
      d[c + 1][k] = x.y;
      d[c + 2][k] = x.z;
      d[c + 3][k] = x.w;
    };
#pragma unroll
    for (int j = 0; j < (nL + NT - 1) / NT; ++j) {
      const int e = int(threadIdx.x) + NT * j;
      if (e < nL) put(&Lp[e / K4][4 * (e % K4)], lb[j]);
    }
#pragma unroll
    for (int j = 0; j < (nU + NT - 1) / NT; ++j) {
      const int e = int(threadIdx.x) + NT * j;
      if (e < nU) put_t(UdT, 4 * (e % 4), e / 4, ub[j]);
    }
    if (have) {
#pragma unroll
      for (int j = 0; j < nW; ++j) {
        const int e = lane + 32 * j;
        put_t(UrT, 4 * (e % 4), e / 4, urb[j]);
        put(&Lc[e / K4][4 * (e % K4)], lcb[j]);
      }
    }
    __syncthreads();
  }
  // 2. warp 0: the diagonal block's pending updates (lane r holds row r) and
  //    its factorisation in registers, into shared memory for the CTA;
  //    meanwhile the other warps stage their pairs and apply theirs
  if (warp == 0) {
    for (int st = 0; st < P; ++st) {
      float l[BS];                                          // L[o+r][O+16st+k], k ascending
#pragma unroll
      for (int q = 0; q < BS / 4; ++q) {
        const float4 t = *reinterpret_cast<const float4 *>(&Lp[r][st * BS + 4 * q]);
        l[4 * q] = t.x;
        l[4 * q + 1] = t.y;
        l[4 * q + 2] = t.z;
        l[4 * q + 3] = t.w;
      }
#pragma unroll
      for (int c = 0; c < BS; ++c) {
        float sum = 0.f;
#pragma unroll
        for (int q = 0; q < BS / 4; ++q) {
          const float4 u = *reinterpret_cast<const float4 *>(&UdT[c][st * BS + 4 * q]);   // broadcast
          sum = fmaf(l[4 * q], u.x, sum);
          sum = fmaf(l[4 * q + 1], u.y, sum);
          sum = fmaf(l[4 * q + 2], u.z, sum);
          sum = fmaf(l[4 * q + 3], u.w, sum);
        }
        v[c] = v[c] - sum;
      }
    }
#pragma unroll
    for (int k = 0; k < BS - 1; ++k) {
      const float ukk = __shfl_sync(0xffffffffu, v[k], k);
      const float lk = v[k] / ukk;                            // L[r][k] (rows r > k keep it;
      v[k] = r > k ? lk : v[k];                               //  a select, not a guarded division)
#pragma unroll
      for (int c = k + 1; c < BS; ++c) {
        const float ukc = __shfl_sync(0xffffffffu, v[c], k);  // U[k][c]
        if (r > k) v[c] = fmaf(-v[k], ukc, v[c]);
      }
    }
    if (lane < BS) {
#pragma unroll
      for (int c = 0; c < BS; ++c) {
        dia[r][c] = v[c];
        diaT[c][r] = v[c];
      }
      if (blockIdx.x == 0) {
        float4 *d4 = reinterpret_cast<float4 *>(dst + size_t(r) * dstride);
#pragma unroll
        for (int q = 0; q < BS / 4; ++q) d4[q] = make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
      }
    }
  }
  // 3. stage the pair
  float(*R)[LD] = blk[warp][0];
  float(*C)[LD] = blk[warp][1];
  if (have) {
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
    // the pair's pending updates: R[i][c] (row block) and C[j][rr] (column block)
    const int x = lane & (BS - 1);
    for (int st = 0; st < P; ++st) {
      float ur[BS], lc[BS];                                 // U[O+16st+k][cb+x], L[cb+x][O+16st+k]
#pragma unroll
      for (int q = 0; q < BS / 4; ++q) {
        const float4 t = *reinterpret_cast<const float4 *>(&UrT[x][st * BS + 4 * q]);
        const float4 w = *reinterpret_cast<const float4 *>(&Lc[x][st * BS + 4 * q]);
        ur[4 * q] = t.x;
        ur[4 * q + 1] = t.y;
        ur[4 * q + 2] = t.z;
        ur[4 * q + 3] = t.w;
        lc[4 * q] = w.x;
        lc[4 * q + 1] = w.y;
        lc[4 * q + 2] = w.z;
        lc[4 * q + 3] = w.w;
      }
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const int y = (lane >> 4) + 2 * q;
        float sr = 0.f, sc = 0.f;
#pragma unroll
        for (int k4 = 0; k4 < BS / 4; ++k4) {
          const float4 lp = *reinterpret_cast<const float4 *>(&Lp[y][st * BS + 4 * k4]);   // L[o+y][..]
          const float4 ud = *reinterpret_cast<const float4 *>(&UdT[y][st * BS + 4 * k4]);  // U[..][o+y]
          sr = fmaf(lp.x, ur[4 * k4], sr);
          sc = fmaf(lc[4 * k4], ud.x, sc);
          sr = fmaf(lp.y, ur[4 * k4 + 1], sr);
          sc = fmaf(lc[4 * k4 + 1], ud.y, sc);
          sr = fmaf(lp.z, ur[4 * k4 + 2], sr);
          sc = fmaf(lc[4 * k4 + 2], ud.z, sc);
          sr = fmaf(lp.w, ur[4 * k4 + 3], sr);
          sc = fmaf(lc[4 * k4 + 3], ud.w, sc);
        }
        R[y][x] = R[y][x] - sr;
        C[y][x] = C[y][x] - sc;
      }
    }
  }
  __syncthreads();                                          // the diagonal block is in dia / diaT
  if (!have) return;                                        // warp-uniform
  const float(*Dg)[LD] = dia;
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
    // one-sided run: all lanes divide and a select keeps it for the column
    // role (a guarded division would branch around the IEEE sequence 16 times).
    const bool col = lane >= BS;
    const int idx = lane & (BS - 1);
    float(*S)[LD] = col ? C : R;
    const float(*D)[LD] = col ? diaT : dia;
    float x[BS];
#pragma unroll
    for (int i = 0; i < BS; ++i) x[i] = S[i][idx];
#pragma unroll
    for (int i = 0; i < BS; ++i) {
#pragma unroll
      for (int j = 0; j < i; ++j) x[i] = fmaf(-x[j], D[i][j], x[i]);
      const float q = x[i] / D[i][i];                     // every lane divides; the row role
      x[i] = col ? q : x[i];                                // discards it (select, no branch)
    }
#pragma unroll
    for (int i = 0; i < BS; ++i) S[i][idx] = x[i];
  }
  __syncwarp();
  // 5. coalesced write-back of both blocks
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int q = lane + 32 * h, i = q >> 2, c = 4 * (q & 3);
    *reinterpret_cast<float4 *>(a + (size_t(o) + i) * n + cb + c) = make_float4(R[i][c], R[i][c + 1], R[i][c + 2], R[i][c + 3]);
    *reinterpret_cast<float4 *>(a + (cb + i) * n + o + c) = make_float4(C[c][i], C[c + 1][i], C[c + 2][i], C[c + 3][i]);
  }
}

// ------------------------------------------------------------------ update
// Trailing update of the far block [O+64, n)^2 by the T steps of a super-step:
// per element and step, sum = fma(L[r][k], U[k][c], sum) for k = 0..15 and then
// a = a - sum, in step order — exactly the per-element sequence of one
// 16-column step after another (and of the restatement), so deferring the far
// block's T updates into one pass over it leaves every bit unchanged while the
// trailing matrix crosses HBM once per 64 columns instead of once per 16.
constexpr int kFarRows = 128, kFarCols = 128;  // far-update tile
constexpr int kFarThreads = 256;               // thread = 8 rows x 8 columns of the tile

// The far trailing block's T-step update (the bulk of the FLOPs), persistent:
// one 256-thread CTA per SM walks the 128x128 tiles of its region.  A tile's
// L rows (k along, 16-byte chunks) and U rows go to shared memory with
// cp.async while the previous tile computes (two stages), and so does the
// tile of A (one buffer: copied to registers at the tile's start, then
// refilled with the next tile's).  Thread (tx, ty) owns rows ty + 16 i (i < 8) and
// columns 4 tx .. +3 and 64 + 4 tx .. +3: a warp's L reads are two rows 68
// words apart (one wavefront), its U reads 256 contiguous bytes per half.
// Per 4 k's a thread reads 8 float4 of L and 8 of U for 128 FFMA2 (the L
// operand broadcast to both halves); the accumulators and the tile take 128
// registers.  Band tiles (64 rows or 64 columns) run a half-size variant.
// Per element the operation sequence above; the step's subtraction as FADD2
// (sub.rn.f32x2: both halves IEEE subtractions, half the FMA-pipe issues).
constexpr int kPipeK = kLook * BS;                 // 64
// dense tiles as the tensor memory accelerator writes them (no padding)
constexpr int kLdL = kPipeK;                       // lp[r][k] row pitch
constexpr int kLdU = kFarCols;                     // up[k][c]
constexpr int kStageWords = kFarRows * kLdL + kPipeK * kLdU;
constexpr int kLdA = kFarCols;                     // the A tile's buffer (single)
constexpr int kFarSmemWords = 2 * kStageWords + kFarRows * kLdA;   // 192 KB
constexpr unsigned kStageBytes = unsigned(kStageWords) * 4, kTileABytes = unsigned(kFarRows * kLdA) * 4;

// TMA (cp.async.bulk.tensor); the mbarrier primitives are in common.cuh
__device__ __forceinline__ void tma_load_2d(float *dst, const CUtensorMap *map, int x, int y, uint64_t *bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
          smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ float2 sub2(float2 a, float2 b) {   // sub.rn.f32x2: two IEEE subtractions (FADD2)
  unsigned long long ra, rb, rd;
  asm("mov.b64 %0, {%1, %2};" : "=l"(ra) : "f"(a.x), "f"(a.y));
  asm("mov.b64 %0, {%1, %2};" : "=l"(rb) : "f"(b.x), "f"(b.y));
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(rd) : "l"(ra), "l"(rb));
  float2 d;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(d.x), "=f"(d.y) : "l"(rd));
  return d;
}

// T steps on one tile: NI row groups (of 16 rows: 8 = all, 4 = a 64-row band)
// and NH column halves (2 = all, 1 = a 64-column band).
template <int T, int NI, int NH>
__device__ __forceinline__ void far_tile(const float *__restrict__ lp, const float *__restrict__ up, float4 (&v)[8][2],
                                         int ty, int c1) {
#pragma unroll 1
  for (int t = 0; t < T; ++t) {
    float2 acc[NI][2 * NH];
#pragma unroll
    for (int i = 0; i < NI; ++i)
#pragma unroll
      for (int j = 0; j < 2 * NH; ++j) acc[i][j] = make_float2(0.f, 0.f);
#pragma unroll
    for (int k4 = 0; k4 < BS / 4; ++k4) {
      const int kb = t * BS + 4 * k4;
      float4 l[NI];
#pragma unroll
      for (int i = 0; i < NI; ++i) l[i] = *reinterpret_cast<const float4 *>(lp + (ty + 16 * i) * kLdL + kb);
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        float4 u[NH];
#pragma unroll
        for (int h = 0; h < NH; ++h) u[h] = *reinterpret_cast<const float4 *>(up + (kb + q) * kLdU + c1 + 64 * h);
#pragma unroll
        for (int i = 0; i < NI; ++i) {
          const float li = q == 0 ? l[i].x : q == 1 ? l[i].y : q == 2 ? l[i].z : l[i].w;
          const float2 ll = make_float2(li, li);
#pragma unroll
          for (int h = 0; h < NH; ++h) {
            acc[i][2 * h] = fma2(ll, make_float2(u[h].x, u[h].y), acc[i][2 * h]);
            acc[i][2 * h + 1] = fma2(ll, make_float2(u[h].z, u[h].w), acc[i][2 * h + 1]);
          }
        }
      }
    }
#pragma unroll
    for (int i = 0; i < NI; ++i)
#pragma unroll
      for (int h = 0; h < NH; ++h) {
        const float2 lo = sub2(make_float2(v[i][h].x, v[i][h].y), acc[i][2 * h]);
        const float2 hi = sub2(make_float2(v[i][h].z, v[i][h].w), acc[i][2 * h + 1]);
        v[i][h] = make_float4(lo.x, lo.y, hi.x, hi.y);
      }
  }
}

// The region a launch updates: up to two rectangles of the trailing matrix
// (the look-ahead strips, or the far block), tiles numbered rectangle by
// rectangle, row-major inside each.
struct FarRects {
  int rlo[2], rhi[2], clo[2], chi[2];
  int tiles_c[2], first[2];   // tiles per row of tiles; first tile index of each rectangle
  int tiles;
};

static FarRects far_rects(int n_rects, const int (*r)[4]) {
  FarRects f{};
  f.tiles = 0;
  for (int i = 0; i < 2; ++i) {
    const bool on = i < n_rects && r[i][1] > r[i][0] && r[i][3] > r[i][2];
    f.rlo[i] = on ? r[i][0] : 0;
    f.rhi[i] = on ? r[i][1] : 0;
    f.clo[i] = on ? r[i][2] : 0;
    f.chi[i] = on ? r[i][3] : 0;
    f.tiles_c[i] = on ? (f.chi[i] - f.clo[i] + kFarCols - 1) / kFarCols : 1;
    f.first[i] = f.tiles;
    if (on) f.tiles += f.tiles_c[i] * ((f.rhi[i] - f.rlo[i] + kFarRows - 1) / kFarRows);
  }
  return f;
}

struct FarMaps {                 // tensor maps of A (n x n fp32, row-major): three box shapes
  CUtensorMap l, u, t;           // L rows (64 x 128), U rows (128 x 64), the tile (128 x 128)
};

template <int T>   // steps in the super-step (kLook but for the last one)
__global__ void __launch_bounds__(kFarThreads, 1) lud_far_pipe_kernel(float *__restrict__ a, int n, int o, FarRects R,
                                                                      const __grid_constant__ FarMaps maps,
                                                                      int *__restrict__ next_tile) {
  extern __shared__ __align__(128) float psm[];
  __shared__ __align__(8) uint64_t bar[3];   // stage 0 / stage 1 (L, U) landed; the A tile landed
  __shared__ int s_tile[2];                  // tiles handed out by the launch's counter (double-buffered)
  const int tiles = R.tiles;
  // tile -> its origin (r0, c0) and extent (nr, nc)
  auto place = [&](int tile, int &r0, int &c0, int &nr, int &nc) {
    // selects, not an indexed parameter array (which would go to local memory)
    const bool second = tile >= R.first[1] && R.first[1] < R.tiles;
    const unsigned t = unsigned(tile - (second ? R.first[1] : 0));
    const unsigned tc = unsigned(second ? R.tiles_c[1] : R.tiles_c[0]);
    const unsigned q = t / tc;
    r0 = (second ? R.rlo[1] : R.rlo[0]) + kFarRows * int(q);
    c0 = (second ? R.clo[1] : R.clo[0]) + kFarCols * int(t - q * tc);
    nr = min(kFarRows, (second ? R.rhi[1] : R.rhi[0]) - r0);
    nc = min(kFarCols, (second ? R.chi[1] : R.chi[0]) - c0);
  };
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  const int c1 = 4 * tx;
  auto stage_ptr = [&](int st) { return psm + size_t(st) * kStageWords; };
  float *const ap = psm + 2 * size_t(kStageWords);
  // one thread issues a tile's three boxes: L (rows r0.., columns o..o+63), U
  // (rows o..o+63, columns c0..), A (rows r0.., columns c0..).  Box parts past
  // the region (a band's edge) load neighbouring data that is computed on but
  // never stored; parts past the matrix are zero-filled.
  auto issue = [&](int tile, int st) {
    int r0, c0, nr, nc;
    place(tile, r0, c0, nr, nc);
    float *lp = stage_ptr(st), *up = lp + kFarRows * kLdL;
    mbar_expect_tx(&bar[st], kStageBytes);
    tma_load_2d(lp, &maps.l, o, r0, &bar[st]);
    tma_load_2d(up, &maps.u, c0, o, &bar[st]);
    mbar_expect_tx(&bar[2], kTileABytes);
    tma_load_2d(ap, &maps.t, c0, r0, &bar[2]);
  };
  // Tiles are handed out dynamically (one atomic per tile on the launch's
  // zeroed counter): a CTA that starts late — the band kernel beside this one
  // holds SMs for its first microseconds — simply takes fewer tiles.
  if (threadIdx.x == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    mbar_init(&bar[2], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    s_tile[0] = atomicAdd(next_tile, 1);
  }
  __syncthreads();
  int tile = s_tile[0];
  if (threadIdx.x == 0 && tile < tiles) issue(tile, 0);
  for (int it = 0; tile < tiles; ++it) {
    const int st = it & 1;
    int r0, c0, nr, nc;
    place(tile, r0, c0, nr, nc);
    mbar_wait(&bar[st], unsigned(it >> 1) & 1u);
    mbar_wait(&bar[2], unsigned(it) & 1u);
    // the tile of A into registers; then the buffer and the other stage take the next tile's
    float4 v[8][2];
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
      for (int h = 0; h < 2; ++h) v[i][h] = *reinterpret_cast<const float4 *>(ap + (ty + 16 * i) * kLdA + c1 + 64 * h);
    if (threadIdx.x == 0) s_tile[(it + 1) & 1] = atomicAdd(next_tile, 1);
    __syncthreads();
    const int next = s_tile[(it + 1) & 1];
    if (threadIdx.x == 0 && next < tiles) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // generic reads before async writes
      issue(next, st ^ 1);
    }
    const float *lp = stage_ptr(st), *up = lp + kFarRows * kLdL;
    // nr, nc are multiples of 16: rows ty + 16 i are in the tile iff i < nr / 16
    if (nr > 64) {
      if (nc > 64) far_tile<T, 8, 2>(lp, up, v, ty, c1);
      else far_tile<T, 8, 1>(lp, up, v, ty, c1);
    } else {
      if (nc > 64) far_tile<T, 4, 2>(lp, up, v, ty, c1);
      else far_tile<T, 4, 1>(lp, up, v, ty, c1);
    }
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int r = ty + 16 * i, c = c1 + 64 * h;
        if (r < nr && c < nc) *reinterpret_cast<float4 *>(a + size_t(r0 + r) * n + c0 + c) = v[i][h];
      }
    tile = next;
  }
}


// ------------------------------------------------------------------ driver
// Super-steps of kLook 16-column steps at offset O.  For each step t in the
// super-step one panel launch: it first applies to the blocks it reads the
// updates of the steps O..o-16 before it (left-looking inside the
// super-step), then factors the diagonal block and solves the perimeter.  The
// trailing matrix then takes the super-step's kLook updates in one pass
// (lud_far_pipe_kernel: the band, then the far block); the factored diagonal
// blocks are scattered into place at the end.
// Scatter of the factored diagonal blocks (kept in scratch while later steps
// may still read the unfactored blocks) into the matrix: block j of dscr to
// a[16j.., 16j..].
__global__ void lud_scatter_diag_kernel(float *__restrict__ a, int n, const float *__restrict__ dscr) {
  const int j = blockIdx.x, e = threadIdx.x;   // 256 threads
  a[size_t(BS * j + e / BS) * n + BS * j + e % BS] = dscr[size_t(j) * BS * BS + e];
}

namespace {

template <bool M>
void launch_panel(float *a, int n, int o, int O, float *dscr, cudaStream_t s) {
  const int nb = n / BS;
  const int m = nb - o / BS - 1;   // blocks right of / below the diagonal
  const int grid = m > 0 ? (m + kPairs - 1) / kPairs : 1;
  // the factored diagonal block goes to scratch slot o/16 (CTAs of this launch
  // still read the unfactored one); the last one, with no other reader, in place
  float *dst = m > 0 ? dscr + size_t(o / BS) * BS * BS : a + size_t(o) * n + o;
  const int dstride = m > 0 ? BS : n;
  const size_t shm = 0;
  switch ((o - O) / BS) {
    case 0: lud_panel_kernel<M, 0><<<grid, 32 * kPairs, shm, s>>>(a, n, o, m, O, dst, dstride); break;
    case 1: lud_panel_kernel<M, 1><<<grid, 32 * kPairs, shm, s>>>(a, n, o, m, O, dst, dstride); break;
    case 2: lud_panel_kernel<M, 2><<<grid, 32 * kPairs, shm, s>>>(a, n, o, m, O, dst, dstride); break;
    default: lud_panel_kernel<M, 3><<<grid, 32 * kPairs, shm, s>>>(a, n, o, m, O, dst, dstride); break;
  }
}

// The panel launches of the super-step at O (T steps).
void launch_panels(int variant, float *a, int n, int O, float *dscr, cudaStream_t s, int *launches) {
  const int T = min(kLook, (n - O) / BS);
  for (int t = 0; t < T; ++t) {
    const int o = O + t * BS;
    if (variant)
      launch_panel<true>(a, n, o, O, dscr, s);
    else
      launch_panel<false>(a, n, o, O, dscr, s);
    ++*launches;
  }
}

// The three tensor maps of the matrix (host-encoded through the driver entry point).
cudaError_t far_maps(float *a, int n, FarMaps &m) {
  static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
  if (!encode) {
    cudaDriverEntryPointQueryResult q;
    cudaError_t e = cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", reinterpret_cast<void **>(&encode),
                                            cudaEnableDefault, &q);
    if (e != cudaSuccess || q != cudaDriverEntryPointSuccess || !encode) return cudaErrorNotSupported;
  }
  const cuuint64_t dims[2] = {cuuint64_t(n), cuuint64_t(n)};
  const cuuint64_t strides[1] = {cuuint64_t(n) * sizeof(float)};
  const cuuint32_t es[2] = {1, 1};
  auto one = [&](CUtensorMap &t, unsigned bx, unsigned by) {
    const cuuint32_t box[2] = {bx, by};
    return encode(&t, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, a, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                  CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  };
  if (one(m.l, kPipeK, kFarRows) != CUDA_SUCCESS || one(m.u, kFarCols, kPipeK) != CUDA_SUCCESS ||
      one(m.t, kFarCols, kFarRows) != CUDA_SUCCESS)
    return cudaErrorInvalidValue;
  return cudaSuccess;
}

cudaError_t launch_far(float *a, int n, int O, int T, const FarRects &R, const FarMaps &maps, int grid,
                       int *counter, cudaStream_t s) {
  if (R.tiles == 0) return cudaSuccess;
  const size_t shm = size_t(kFarSmemWords) * sizeof(float);
  grid = max(1, min(grid, R.tiles));
  switch (T) {
    case 1: lud_far_pipe_kernel<1><<<grid, kFarThreads, shm, s>>>(a, n, O, R, maps, counter); break;
    case 2: lud_far_pipe_kernel<2><<<grid, kFarThreads, shm, s>>>(a, n, O, R, maps, counter); break;
    case 3: lud_far_pipe_kernel<3><<<grid, kFarThreads, shm, s>>>(a, n, O, R, maps, counter); break;
    default: lud_far_pipe_kernel<4><<<grid, kFarThreads, shm, s>>>(a, n, O, R, maps, counter); break;
  }
  return cudaGetLastError();
}

struct LudSide {       // per device: the panel stream of the look-ahead and its fork / join events
  cudaStream_t s = nullptr;
  cudaEvent_t fork = nullptr, join = nullptr;
};

}  // namespace

// Tile counters record_lud needs (two trailing-update launches per super-step).
int lud_counter_words(int n) { return 2 * (n / (kLook * BS) + 2); }

// Look-ahead across super-steps (two streams inside the captured graph):
//   main   ... far block(g-1) -> [fork] -> far block(g) -> [join] -> ...
//   panel       [fork] -> band(g) -> panels(g+1) (4 launches) -> join
// The band is the 64-wide L-shaped strip at E = end of super-step g — the
// rows and columns the next super-step's panels read; it needs super-step
// g's panels and the far block of g-1, exactly like the far block of g, and
// the two regions are disjoint, so the band runs beside the far block on the
// high-priority panel stream (its CTAs are dispatched first; the far block's
// tiles are handed out dynamically, so its late-starting CTAs take fewer)
// and the next panels follow it there while the far block [E+64, n)^2 takes
// super-step g's update on all but kPanelSMs SMs.  Every element still
// receives its updates in step order.  The critical path per super-step is
// max(far block, band + panel chain) instead of band + max(far block, panel
// chain).
// SMs the far block leaves to the concurrent panels (round 2, band beside the far
// block, at 8192: 4 -> 10.66 ms, 6 -> 10.57, 8 -> 10.42, 10 -> 10.44, 12 -> 10.45;
// round 1 schedule:
// 0 -> 15.65 ms, 4 -> 14.98, 8 -> 14.72, 16 -> 14.89, 32 -> 16.13)
#ifndef DARM_LUD_PANEL_SMS
#define DARM_LUD_PANEL_SMS 8
#endif
constexpr int kPanelSMs = DARM_LUD_PANEL_SMS;
#ifndef DARM_LUD_PANEL_ADAPT_M
#define DARM_LUD_PANEL_ADAPT_M 6144   // swept at 8192^2: 0 -> 10.49 ms, 3072 -> 10.49, 5120 -> 10.42, 6144 -> 10.40, 7168 -> 10.52, 8192 -> 10.74
#endif

cudaError_t record_lud(int variant, float *a, int n, float *dscr, int *counters, cudaStream_t s, int *launches) {
  // per device: kernel attributes, SM count, the panel stream (callers hold
  // the device's lock)
  struct LudDevice {
    bool attr = false;
    int sms = 0;
    LudSide side;
  };
  static LudDevice devs[64];
  int dev = 0;
  cudaGetDevice(&dev);
  LudDevice &D = devs[dev & 63];
  if (!D.attr) {
    const int shm = int(size_t(kFarSmemWords) * sizeof(float));
    for (auto k : {lud_far_pipe_kernel<1>, lud_far_pipe_kernel<2>, lud_far_pipe_kernel<3>, lud_far_pipe_kernel<4>}) {
      cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, shm);
      if (e != cudaSuccess) return e;
    }
    cudaDeviceGetAttribute(&D.sms, cudaDevAttrMultiProcessorCount, dev);
    if (D.sms <= 0) D.sms = 148;
    D.attr = true;
  }
  const int sms = D.sms;
  LudSide &sd = D.side;
  if (!sd.s) {
    int lo = 0, hi = 0;
    cudaDeviceGetStreamPriorityRange(&lo, &hi);
    cudaError_t e = cudaStreamCreateWithPriority(&sd.s, cudaStreamNonBlocking, hi);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&sd.fork, cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&sd.join, cudaEventDisableTiming);
    if (e != cudaSuccess) return e;
  }
  const int nb = n / BS;
  const int G = kLook * BS;
  FarMaps maps;
  if (n > G) {
    cudaError_t e = far_maps(a, n, maps);
    if (e != cudaSuccess) return e;
  }
  // one tile counter per trailing-update launch, zeroed at the graph's start
  if (n > G) {
    cudaError_t e = cudaMemsetAsync(counters, 0, size_t(lud_counter_words(n)) * sizeof(int), s);
    if (e != cudaSuccess) return e;
  }
  int *ctr = counters;
  launch_panels(variant, a, n, 0, dscr, s, launches);   // super-step 0: nothing to overlap with
  for (int O = 0; O < n; O += G) {
    const int T = min(kLook, (n - O) / BS);
    const int E = O + T * BS;
    if (E >= n) break;
    const int Tn = min(kLook, (n - E) / BS);   // the next super-step's steps
    const int F = E + Tn * BS;                  // end of its band
    // the band the next panels read: rows [E, F) x cols [E, n), rows [F, n) x cols [E, F)
    const int band[2][4] = {{E, F, E, n}, {F, n, E, F}};
    cudaError_t e;
    if (F < n) {
      e = cudaEventRecord(sd.fork, s);
      if (e == cudaSuccess) e = cudaStreamWaitEvent(sd.s, sd.fork, 0);
      if (e == cudaSuccess) e = launch_far(a, n, O, T, far_rects(2, band), maps, sms, ctr++, sd.s);
      if (e != cudaSuccess) return e;
      ++*launches;
      launch_panels(variant, a, n, E, dscr, sd.s, launches);
      e = cudaEventRecord(sd.join, sd.s);
      if (e != cudaSuccess) return e;
      const int far[1][4] = {{F, n, F, n}};
      // SMs left to the panels beside the far block: kPanelSMs while the far
      // block dominates; once it is small (m <= DARM_LUD_PANEL_ADAPT_M) enough
      // for the next panels' CTAs to run in one wave (six per SM)
      int reserve = kPanelSMs;
      const int m_far = n - F, pairs = (n - E) / BS - 1;
      if (m_far <= DARM_LUD_PANEL_ADAPT_M) reserve = max(kPanelSMs, min(32, ((pairs + kPairs - 1) / kPairs + 5) / 6));
      e = launch_far(a, n, O, T, far_rects(1, far), maps, sms - reserve, ctr++, s);
      if (e != cudaSuccess) return e;
      ++*launches;
      e = cudaStreamWaitEvent(s, sd.join, 0);
      if (e != cudaSuccess) return e;
    } else {
      // the last super-step: no far block left
      e = launch_far(a, n, O, T, far_rects(2, band), maps, sms, ctr++, s);
      if (e != cudaSuccess) return e;
      ++*launches;
      launch_panels(variant, a, n, E, dscr, s, launches);
    }
  }
  if (nb > 1) {
    lud_scatter_diag_kernel<<<nb - 1, BS * BS, 0, s>>>(a, n, dscr);
    ++*launches;
  }
  return cudaGetLastError();
}

}  // namespace darm_gpu
