// srad.cu — Speckle Reducing Anisotropic Diffusion (SRAD, PAPER.md:778-781,
// 842-851), fp32, unmelded and melded forms.  The reference has no SRAD code;
// the per-pixel mathematics is Rodinia's SRAD restated and the
// CPU oracle (oracle/darm_oracle.c, oracle_srad) performs the same fp32 / fp64
// operations in the same order.  This translation unit is compiled with
// -fmad=false so no multiply-add is contracted in the IEEE path (the oracle is
// compiled with -ffp-contract=off): GPU and CPU agree bit for bit.
//
// Per iteration, with q0sqr from the ROI statistics of the current image J:
//   c(i,j)  = clamp01( 1 / (1 + (q(i,j) - q0sqr) / (q0sqr (1 + q0sqr))) )
//   J'(i,j) = J + (lambda/4) (c(i,j) dN + c(i+1,j) dS + c(i,j) dW + c(i,j+1) dE)
// with dN..dE the differences to the 4 neighbours (image borders clamp).
//
// B200 layout (round 2): one fused sweep per iteration, 8 B of HBM traffic per
// pixel (one read of J, one write of J').  A thread owns 4 consecutive columns
// (16-byte row loads and stores), a warp 128 columns; the warp slides down a
// segment of rows two rows at a time, keeping the vertical window
// J(i-1 .. i+3) and c(i) in registers, the arithmetic of the two rows in f32x2
// pairs.  West / east neighbours inside a thread are registers; across threads
// one __shfl_up / __shfl_down per row; at the warp's edges lane 0 loads the
// west halo column c0-1 and lane 31 the east halo columns c0+128, c0+129 (one
// predicated scalar load each), and lane 31 computes c for column c0+128 as a
// fifth column (its east c).  Row pointers are 64-bit (one addressing path).
// The pitch of a row buffer is a multiple of 4 floats (16-byte rows).
//
// The divergent regions are
//   R_B  border handling: the west / east neighbour of the warp's edge lanes
//        (halo vs shuffle: thread-position dependent) and, in the warp holding
//        the image's last column, the clamped east neighbour;
//   R_D  the data-dependent three-way clamp of c (c < 0 / c > 1 / else).
// unmelded: if / else-if arms behind real divergent branches (DARM_IPDOM);
// melded: select chains.
//
// ROI statistics are reduced deterministically: per ROI row and 128-column
// warp group, each lane sums its 4 in-ROI values of J' in fp64 in column
// order, then a 32-lane xor butterfly; lane 0 writes one partial per (row,
// group); every warp folds the partials rows-then-groups in order at its start
// (srad_q0_warp: lanes load, the sum runs in index order).  For
// row-tiled multi-GPU runs every partial is written by the one rank owning
// its row.
//
// Row ranges: a launch computes own rows [lo0, hi0) and [lo1, hi1) of a tile
// (segments of `rs` rows each), so a multi-GPU rank runs its interior rows
// while the halo rows are in flight and the two edge bands after they land.
#include <cstdint>

#include "common.cuh"
#include "kernels.h"

namespace darm_gpu {

constexpr int kSradWarpCols = 128;   // 32 lanes x 4 columns
constexpr unsigned kFull = 0xffffffffu;

struct SradParams {
  const float *jin;      // (tile_rows + 3) x pitch, local row 0 = global row r0 - 1
  float *jout;           // same layout; local rows 1..tile_rows written
  const double *roi_in;  // [roi_rows][roi_groups][2] partial sums of J (this iteration's statistics)
  const double *const *roi_parts;   // multi-GPU: per rank partial buffer (null: roi_in) ...
  const int *roi_owner;             // ... and the rank owning each ROI row
  float *q0_out;         // optional: q0sqr written by the first warp
  double npix;           // ROI pixel count
  double *roi_out;       // [roi_rows][roi_groups][2] partial sums of J' (may be null)
  int cols, pitch, tile_rows, r0, R;
  int lo0, hi0, lo1, hi1;   // own rows (0-based) computed: [lo0, hi0) then [lo1, hi1)
  int rs, nseg0;            // rows per segment; segments of range 0
  float lq;                 // lambda / 4
  float nz;                 // -0.0f (opaque to ptxas: see mulx)
  int roi_r1, roi_r2, roi_c1, roi_c2, roi_w0, roi_groups;
};

__device__ __forceinline__ int clampi(int v, int lo, int hi) { return v < lo ? lo : (v > hi ? hi : v); }

__device__ __forceinline__ float rcp_approx(float b) {
  float r;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(b));
  return r;
}

// ---- f32x2 pairs (sm_100): two rows of one column per instruction.  Every
// half is the IEEE operation of the scalar code.  ptxas (12.9) contracts a
// mul.rn.f32x2 feeding an add.rn.f32x2 into FFMA2 even under -fmad=false, so
// exact products are formed as mulx = fma(a, b, z) with z = -0.0f from a
// kernel parameter (a*b + -0 == a*b exactly, and not foldable).
__device__ __forceinline__ unsigned long long pk(float2 a) {
  unsigned long long r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a.x), "f"(a.y));
  return r;
}
__device__ __forceinline__ float2 upk(unsigned long long r) {
  float2 a;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(a.x), "=f"(a.y) : "l"(r));
  return a;
}
#define DARM_F2(NAME, OP)                                                                     \
  __device__ __forceinline__ float2 NAME(float2 a, float2 b) {                                \
    unsigned long long r;                                                                     \
    asm(OP ".rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(pk(a)), "l"(pk(b)));                       \
    return upk(r);                                                                            \
  }
DARM_F2(add2, "add")
DARM_F2(sub2, "sub")
DARM_F2(mul2, "mul")
#undef DARM_F2
__device__ __forceinline__ float2 fma2(float2 a, float2 b, float2 c) {
  unsigned long long r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(pk(a)), "l"(pk(b)), "l"(pk(c)));
  return upk(r);
}
__device__ __forceinline__ float2 f2(float x) { return make_float2(x, x); }
__device__ __forceinline__ float2 mk(float a, float b) { return make_float2(a, b); }

// R_D: the three-way clamp of c, one pixel.
template <bool M>
__device__ __forceinline__ float clamp_rd(float c) {
  if constexpr (!M) {
    if (c < 0.0f) {
      DARM_IPDOM("srad.rd.lo");
      c = 0.0f;
    } else if (c > 1.0f) {
      DARM_IPDOM("srad.rd.hi");
      c = 1.0f;
    }
    return c;
  } else {
    return fminf(fmaxf(c, 0.0f), 1.0f);   // the select chain c < 0 ? 0 : (c > 1 ? 1 : c), as two FMNMX
  }
}

// ---- per-pixel mathematics on column pairs (two adjacent columns of one row).
// Inputs per pixel: centre C, the vertical differences vn = J(i) - J(i-1) and
// vs = J(i+1) - J(i) (so dN = -vn, dS = vs: IEEE subtraction is symmetric, so
// these are the restatement's dN, dS bit for bit), and dW = W - C, dE = E - C.
struct SradQ {
  float q0sqr, q0den;   // IEEE: q0sqr and q0sqr (1 + q0sqr)
  float nk1, nk2;       // FAST: -16 q0den and -16 q0sqr^2
};

// IEEE: the restatement's operations in its order (oracle srad_c / the update),
// one pixel; the clamp is R_D.
template <bool M>
__device__ __forceinline__ float coeff_ieee(float jc, float vn, float vs, float dW, float dE, const SradQ &q) {
  const float dN = -vn, dS = vs;
  const float g2 = (((dN * dN + dS * dS) + dW * dW) + dE * dE) / (jc * jc);
  const float l = (((dN + dS) + dW) + dE) / jc;
  const float num = (0.5f * g2) - ((1.0f / 16.0f) * (l * l));
  float den = 1.0f + (0.25f * l);
  const float qsqr = num / (den * den);
  den = (qsqr - q.q0sqr) / q.q0den;
  return clamp_rd<M>(1.0f / (1.0f + den));
}
__device__ __forceinline__ float update_ieee(float jc, float vn, float vs, float dW, float dE, float c0, float c1,
                                             float ce, float lq) {
  const float dN = -vn, dS = vs;
  const float d = ((c0 * dN + c1 * dS) + c0 * dW) + ce * dE;
  return jc + lq * d;
}

// FAST (DARM_FAST_MATH): no division at all but one reciprocal.  With
// s = dN + dS + dW + dE and Q = dN^2 + dS^2 + dW^2 + dE^2, Rodinia's
//   q^2 = (Q/2 - s^2/16) / (jc (1 + s/(4 jc)))^2 ... c = 1 / (1 + (q^2 - q0sqr) / q0den)
// is, multiplying through by 16 jc^2 (V = (jc + s/4)^2, U = 8Q - s^2 >= 4Q >= 0
// by Cauchy-Schwarz, so nothing cancels),
//   c = 16 q0den V / (U + 16 q0sqr^2 V)
// computed as (-16 q0den) V / (s^2 - 8Q - 16 q0sqr^2 V).  Within the north
// star's 1e-5 relative of the IEEE path after 100 iterations (tests/test_srad.py).
template <bool M>
__device__ __forceinline__ float2 coeff_fast2(float2 C, float2 vn, float2 vs, float2 dW, float2 dE, const SradQ &q) {
  const float2 s = add2(add2(sub2(vs, vn), dW), dE);
  const float2 Q = fma2(dE, dE, fma2(dW, dW, fma2(vs, vs, mul2(vn, vn))));
  const float2 un = fma2(s, s, mul2(Q, f2(-8.0f)));            // -U
  const float2 m = fma2(f2(0.25f), s, C);
  const float2 V = mul2(m, m);
  const float2 tn = fma2(f2(q.nk2), V, un);                     // -(U + 16 q0sqr^2 V)
  const float2 c = mul2(mul2(V, f2(q.nk1)), mk(rcp_approx(tn.x), rcp_approx(tn.y)));
  return mk(clamp_rd<M>(c.x), clamp_rd<M>(c.y));
}
// the same operations on one pixel (the gathered fifth column)
template <bool M>
__device__ __forceinline__ float coeff_fast1(float C, float vn, float vs, float dW, float dE, const SradQ &q) {
  return coeff_fast2<M>(f2(C), f2(vn), f2(vs), f2(dW), f2(dE), q).x;
}
__device__ __forceinline__ float2 update_fast2(float2 C, float2 vn, float2 vs, float2 dW, float2 dE, float2 cv,
                                               float2 cs, float2 ce, float lq) {
  const float2 d = fma2(ce, dE, fma2(cs, vs, mul2(cv, sub2(dW, vn))));   // c dN + c dW = c (dW - vn)
  return fma2(f2(lq), d, C);
}

template <bool M, bool FAST>
__device__ __forceinline__ float2 coeff2(float2 C, float2 vn, float2 vs, float2 dW, float2 dE, const SradQ &q) {
  if constexpr (FAST) return coeff_fast2<M>(C, vn, vs, dW, dE, q);
  else
    return mk(coeff_ieee<M>(C.x, vn.x, vs.x, dW.x, dE.x, q), coeff_ieee<M>(C.y, vn.y, vs.y, dW.y, dE.y, q));
}
template <bool M, bool FAST>
__device__ __forceinline__ float coeff1(float C, float vn, float vs, float dW, float dE, const SradQ &q) {
  if constexpr (FAST) return coeff_fast1<M>(C, vn, vs, dW, dE, q);
  else return coeff_ieee<M>(C, vn, vs, dW, dE, q);
}
template <bool FAST>
__device__ __forceinline__ float2 update2(float2 C, float2 vn, float2 vs, float2 dW, float2 dE, float2 cv, float2 cs,
                                          float2 ce, float lq) {
  if constexpr (FAST) return update_fast2(C, vn, vs, dW, dE, cv, cs, ce, lq);
  else
    return mk(update_ieee(C.x, vn.x, vs.x, dW.x, dE.x, cv.x, cs.x, ce.x, lq),
              update_ieee(C.y, vn.y, vs.y, dW.y, dE.y, cv.y, cs.y, ce.y, lq));
}

// One row of a thread: its 4 columns as two column pairs (the 16-byte load's
// registers) and the halo value (lane 0: J(., c0-1); lane 31: J(., c0+128)).
struct SradRow {
  float2 a, b;
  float h;
};

// R_B for one row: west / east neighbour of the thread's first / last column.
template <bool M>
__device__ __forceinline__ void west_east(const SradRow &r, int lane, float &w, float &e) {
  const float sw = __shfl_up_sync(kFull, r.b.y, 1);
  const float se = __shfl_down_sync(kFull, r.a.x, 1);
  if constexpr (!M) {
    if (lane == 0) {
      DARM_IPDOM("srad.rb.w0");
      w = r.h;
    } else {
      DARM_IPDOM("srad.rb.w");
      w = sw;
    }
    if (lane == 31) {
      DARM_IPDOM("srad.rb.e31");
      e = r.h;
    } else {
      DARM_IPDOM("srad.rb.e");
      e = se;
    }
  } else {
    w = lane == 0 ? r.h : sw;
    e = lane == 31 ? r.h : se;
  }
}

// east c of the thread's last column: the next lane's first, or (lane 31) the
// fifth column's.  R_B as above.
template <bool M>
__device__ __forceinline__ float east_c(float c_first, float c5, int lane) {
  const float s = __shfl_down_sync(kFull, c_first, 1);
  if constexpr (!M) {
    float r;
    if (lane == 31) {
      DARM_IPDOM("srad.rb.c31");
      r = c5;
    } else {
      DARM_IPDOM("srad.rb.c");
      r = s;
    }
    return r;
  } else {
    return lane == 31 ? c5 : s;
  }
}

// ROI partial of one output row (global row g): this lane's 4 values in column
// order, then the warp butterfly; lane 0 writes.
__device__ __forceinline__ void roi_row(const SradParams &P, int g, int wcol, int col, int lane, float2 ja,
                                        float2 jb) {
  const float jn[4] = {ja.x, ja.y, jb.x, jb.y};
  double s = 0.0, s2 = 0.0;
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const int j = col + k;
    const bool in = j >= P.roi_c1 && j <= P.roi_c2 && j < P.cols;
    const double v = in ? double(jn[k]) : 0.0;
    s += v;
    s2 += v * v;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    s += __shfl_xor_sync(kFull, s, o);
    s2 += __shfl_xor_sync(kFull, s2, o);
  }
  if (lane == 0) {
    double *dst = P.roi_out + 2 * (size_t(g - P.roi_r1) * P.roi_groups + (wcol - P.roi_w0));
    dst[0] = s;
    dst[1] = s2;
  }
}

// q0sqr from the ROI partials: entries in index order (rows, then groups),
// summed in fp64 by every lane (lanes load 32 entries at a time, shuffles
// hand them over in order), then the restatement's mean / variance.
__device__ __forceinline__ float srad_q0_warp(const SradParams &P, int lane) {
  const int n = (P.roi_r2 - P.roi_r1 + 1) * P.roi_groups;
  double s = 0.0, s2 = 0.0;
  for (int base = 0; base < n; base += 32) {
    double a = 0.0, b = 0.0;
    const int e = base + lane;
    if (e < n) {
      if (P.roi_parts) {   // a peer's buffer over NVLink: never a stale cached line
        const double *src = P.roi_parts[P.roi_owner[e / P.roi_groups]];
        a = __ldcv(src + 2 * e);
        b = __ldcv(src + 2 * e + 1);
      } else {
        a = P.roi_in[2 * e];
        b = P.roi_in[2 * e + 1];
      }
    }
    const int m = min(32, n - base);
    for (int l = 0; l < m; ++l) {
      s += __shfl_sync(kFull, a, l);
      s2 += __shfl_sync(kFull, b, l);
    }
  }
  const double mean = s / P.npix;
  const double var = s2 / P.npix - mean * mean;
  return float(var / (mean * mean));
}

// Per-row derived state of the sweep: differences and c of the own columns.
struct SradDiff {
  float2 dWa, dWb, dEa, dEb;   // dW, dE of column pairs a = (0,1), b = (2,3)
};

// One warp's segment [seg0, seg1) of own rows: a CTA is one warp (every
// branch that depends on the warp's position is then CTA-uniform, so ptxas
// needs no WARPSYNC around the shuffles).  EDGE: this warp holds the image's
// last column, whose east neighbour (J and c) is itself.
// Row ring: rows of a warp's strip staged in shared memory by 1-D TMA bulk
// copies (columns c0-4 .. c0+131: the own 128 and both halo columns), kSradStages
// rows ahead of the register window, so a warp keeps ~8 rows of loads in
// flight without holding registers for them (the sweep was bound by load
// latency at 2 rows in flight: 55% issue, 50% DRAM).
#ifndef DARM_SRAD_STAGES
#define DARM_SRAD_STAGES 8
#endif
constexpr int kSradStages = DARM_SRAD_STAGES;   // a power of two
constexpr int kSradRowF = kSradWarpCols + 8;    // floats per staged row
struct SradRing {
  float row[kSradStages][kSradRowF];
  uint64_t bar[kSradStages];
};

template <bool M, bool FAST, bool EDGE>
__device__ __forceinline__ void srad_segment(const SradParams &P, int seg0, int seg1, int wcol, int lane,
                                             SradRing &ring) {
  const int wc0 = wcol * kSradWarpCols;   // the warp's first column
  const int col = wc0 + 4 * lane;
  const int lcol = min(col, P.pitch - 4);   // stays inside the row (columns >= cols are never stored)
  const int gmax = P.R - 1;
  const int glim = min(gmax, P.r0 + P.tile_rows + 1);
  const int hcol = lane == 0 ? max(wc0 - 1, 0) : min(wc0 + kSradWarpCols, P.cols - 1);
  const bool hl = lane == 0 || lane == 31;
  SradQ q;
  q.q0sqr = srad_q0_warp(P, lane);
  q.q0den = q.q0sqr * (1.0f + q.q0sqr);
  q.nk1 = -16.0f * q.q0den;
  q.nk2 = -16.0f * (q.q0sqr * q.q0sqr);
  const size_t pitch = size_t(P.pitch);
  auto rowp = [&](int g) { return P.jin + size_t(min(clampi(g, 0, gmax), glim) - P.r0 + 1) * pitch; };
  auto last = [&](int k) { return EDGE && col + k == P.cols - 1; };
  // dW / dE of a row (west / east neighbour values w, e of the thread's ends)
  auto diffs = [&](const SradRow &r, float w, float e, SradDiff &d) {
    const float2 mid = mk(r.a.y, r.b.x);                       // columns 1, 2
    d.dWa = sub2(mk(w, r.a.x), r.a);
    d.dWb = sub2(mid, r.b);
    d.dEa = sub2(mid, r.a);
    d.dEb = sub2(mk(r.b.y, e), r.b);
    if constexpr (EDGE) {   // R_B: the image's last column (dE = 0)
      if constexpr (!M) {
        if (last(0)) { DARM_IPDOM("srad.rb.l0"); d.dEa.x = 0.0f; }
        if (last(1)) { DARM_IPDOM("srad.rb.l1"); d.dEa.y = 0.0f; }
        if (last(2)) { DARM_IPDOM("srad.rb.l2"); d.dEb.x = 0.0f; }
        if (last(3)) { DARM_IPDOM("srad.rb.l3"); d.dEb.y = 0.0f; }
      } else {
        d.dEa = mk(last(0) ? 0.0f : d.dEa.x, last(1) ? 0.0f : d.dEa.y);
        d.dEb = mk(last(2) ? 0.0f : d.dEb.x, last(3) ? 0.0f : d.dEb.y);
      }
    }
  };
  const bool roi_warp = P.roi_out && wcol >= P.roi_w0 && wcol < P.roi_w0 + P.roi_groups;

  // c of the fifth column (c0 + 128) for 32 rows starting at g: lane l -> row g + l
  // (five gathered loads per 32 rows instead of a fifth column per row)
  const int x5 = min(wc0 + kSradWarpCols, P.cols - 1);
  struct G5 {
    float jc, n, s, w, e;
  };
  auto gather_load = [&](int g, G5 &x) {
    const float *p = rowp(g + lane);
    x.jc = __ldg(p + x5);
    x.n = __ldg(rowp(g + lane - 1) + x5);
    x.s = __ldg(rowp(g + lane + 1) + x5);
    x.w = __ldg(p + min(wc0 + kSradWarpCols - 1, P.cols - 1));
    x.e = __ldg(p + min(wc0 + kSradWarpCols + 1, P.cols - 1));
  };
  // (rows below the image never reach a stored pixel: their c is left as computed)
  auto gather_c5 = [&](const G5 &x) { return coeff1<M, FAST>(x.jc, x.jc - x.n, x.s - x.jc, x.w - x.jc, x.e - x.jc, q); };


  // ---- the ring.  Ring index k = row - (g0 - 1); stage k % 8, phase k / 8.
  // The prologue consumes k = 0..4 (rows g0-1 .. g0+3), loop iteration `it`
  // consumes k = 5 + 8 it + u (u = 0..7): every stage index and phase is a
  // compile-time function of u and the parity of it.  A stage is refilled
  // with k + 8 once consumed, four stages per batch.
  static_assert(kSradStages == 8, "the unrolled sweep assumes an 8-row ring");
  const int g0 = P.r0 + seg0;
  const int iters = (seg1 - seg0 + 7) / 8;
  const int kend = 5 + 8 * iters;                      // ring indices the sweep consumes
  const int lo = max(wc0 - 4, 0), hi = min(wc0 + kSradWarpCols + 4, P.pitch);
  const unsigned bytes = unsigned(hi - lo) * 4u;
  const int soff = lo - (wc0 - 4);                       // 0, or 4 for the first strip
  auto issue = [&](int k) {                              // lane 0
    const int st = k & (kSradStages - 1);
    mbar_expect_tx(&ring.bar[st], bytes);
    tma_load_1d(&ring.row[st][soff], rowp(g0 - 1 + k) + lo, bytes, &ring.bar[st]);
  };
  auto refill = [&](int k0, int n) {   // after the warp's reads of stages k0 .. k0+n-1
    __syncwarp();
    if (lane == 0) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
#pragma unroll
      for (int u = 0; u < n; ++u)
        if (k0 + u + kSradStages < kend) issue(k0 + u + kSradStages);
    }
  };
  if (lane == 0) {
#pragma unroll
    for (int st = 0; st < kSradStages; ++st) mbar_init(&ring.bar[st], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
#pragma unroll
    for (int k = 0; k < kSradStages; ++k)
      if (k < kend) issue(k);
  }
  __syncwarp();
  const int io = lcol - (wc0 - 4), ih = hcol - (wc0 - 4);
  auto consume = [&](int st, unsigned parity, SradRow &r) {
    mbar_wait(&ring.bar[st], parity);
    const float4 x = *reinterpret_cast<const float4 *>(&ring.row[st][io]);
    r.a = mk(x.x, x.y);
    r.b = mk(x.z, x.w);
    r.h = hl ? ring.row[st][ih] : 0.0f;
  };
  SradRow jm, j0, j1, j2, j3;
  consume(0, 0, jm);
  consume(1, 0, j0);
  consume(2, 0, j1);
  consume(3, 0, j2);
  consume(4, 0, j3);
  refill(0, 5);
  float w0, e0;
  west_east<M>(j0, lane, w0, e0);
  SradDiff d0;
  diffs(j0, w0, e0, d0);
  float2 vn0a = sub2(j0.a, jm.a), vn0b = sub2(j0.b, jm.b);     // J(g0) - J(g0-1)
  float2 vs0a = sub2(j1.a, j0.a), vs0b = sub2(j1.b, j0.b);     // J(g0+1) - J(g0)
  float2 c0a = coeff2<M, FAST>(j0.a, vn0a, vs0a, d0.dWa, d0.dEa, q);
  float2 c0b = coeff2<M, FAST>(j0.b, vn0b, vs0b, d0.dWb, d0.dEb, q);
  G5 gx;
  gather_load(g0, gx);
  float c5v = gather_c5(gx);
  float *outp = P.jout + size_t(seg0 + 1) * pitch + col;

  // One output row i (global g): c(g+1) from rows g .. g+2 (jc = row g+1,
  // jn = row g+2), then J'(g).  State in: vn / vs / c / differences of row g;
  // out: row g+1's.  Below the image's last row J clamps, so dS = 0 there and
  // c(g+1) multiplies zero (the restatement's clamped c changes no bit).
  auto step = [&](int i, int r5, const SradRow &jc, const SradRow &jn, float2 &vna, float2 &vnb, float2 &vsa,
                  float2 &vsb, float2 &ca, float2 &cb, SradDiff &d, const SradRow &jg) {
    const int g = P.r0 + i;
    float w1, e1;
    west_east<M>(jc, lane, w1, e1);
    SradDiff d1;
    diffs(jc, w1, e1, d1);
    const float2 vs1a = sub2(jn.a, jc.a), vs1b = sub2(jn.b, jc.b);   // J(g+2) - J(g+1)
    const float2 c1a = coeff2<M, FAST>(jc.a, vsa, vs1a, d1.dWa, d1.dEa, q);
    const float2 c1b = coeff2<M, FAST>(jc.b, vsb, vs1b, d1.dWb, d1.dEb, q);
    // east c of row g: in-thread neighbours, the next lane, or the fifth column
    const float c5 = __shfl_sync(kFull, c5v, r5);
    const float cE = east_c<M>(ca.x, c5, lane);
    float2 cea = mk(ca.y, cb.x), ceb = mk(cb.y, cE);
    if constexpr (EDGE) {   // R_B: the image's last column (its own c)
      if constexpr (!M) {
        if (last(0)) { DARM_IPDOM("srad.rb.m0"); cea.x = ca.x; }
        if (last(1)) { DARM_IPDOM("srad.rb.m1"); cea.y = ca.y; }
        if (last(2)) { DARM_IPDOM("srad.rb.m2"); ceb.x = cb.x; }
        if (last(3)) { DARM_IPDOM("srad.rb.m3"); ceb.y = cb.y; }
      } else {
        cea = mk(last(0) ? ca.x : cea.x, last(1) ? ca.y : cea.y);
        ceb = mk(last(2) ? cb.x : ceb.x, last(3) ? cb.y : ceb.y);
      }
    }
    const float2 ja = update2<FAST>(jg.a, vna, vsa, d.dWa, d.dEa, ca, c1a, cea, P.lq);
    const float2 jb = update2<FAST>(jg.b, vnb, vsb, d.dWb, d.dEb, cb, c1b, ceb, P.lq);
    if (i < seg1) {
      if constexpr (!EDGE) {
        *reinterpret_cast<float4 *>(outp) = make_float4(ja.x, ja.y, jb.x, jb.y);
      } else {
        const float v[4] = {ja.x, ja.y, jb.x, jb.y};
#pragma unroll
        for (int k = 0; k < 4; ++k)
          if (col + k < P.cols) outp[k] = v[k];
      }
      if (roi_warp && unsigned(g - P.roi_r1) <= unsigned(P.roi_r2 - P.roi_r1)) roi_row(P, g, wcol, col, lane, ja, jb);
    }
    outp += pitch;
    vna = vsa;
    vnb = vsb;
    vsa = vs1a;
    vsb = vs1b;
    ca = c1a;
    cb = c1b;
    d = d1;
  };
  // eight rows per iteration: rows g .. g+3 in registers, the next rows
  // consumed from the ring two at a time (all register rotations have period
  // 2, so the unrolled body renames them)
#pragma unroll 1
  for (int it = 0; it < iters; ++it) {
    const unsigned p0 = unsigned(it) & 1u, p1 = p0 ^ 1u;
    const int ib = seg0 + 8 * it;
    const int rb = 8 * (it & 3);                 // (row - seg0) mod 32 of the iteration's first row
#pragma unroll
    for (int t = 0; t < 8; t += 2) {
      SradRow j4, j5;
      consume((5 + t) & 7, 5 + t >= 8 ? p1 : p0, j4);
      consume((6 + t) & 7, 6 + t >= 8 ? p1 : p0, j5);
      if (t == 2 || t == 6) refill(5 + 8 * it + t - 2, 4);
      step(ib + t, rb + t, j1, j2, vn0a, vn0b, vs0a, vs0b, c0a, c0b, d0, j0);
      step(ib + t + 1, rb + t + 1, j2, j3, vn0a, vn0b, vs0a, vs0b, c0a, c0b, d0, j1);
      j0 = j2;
      j1 = j3;
      j2 = j4;
      j3 = j5;
    }
    if ((it & 3) == 3) {   // the next 32 rows' fifth column (warp-uniform)
      gather_load(P.r0 + ib + 8, gx);   // (loading one block ahead measured slower: 45.5 -> 57 ms)
      c5v = gather_c5(gx);
    }
  }
}

// resident CTAs (one warp each) per SM the sweep is built for (register cap)
#ifndef DARM_SRAD_MINB
#define DARM_SRAD_MINB 20
#endif
template <bool M, bool FAST>
__global__ void __launch_bounds__(32, DARM_SRAD_MINB) srad_sweep_kernel(SradParams P) {
  const int lane = threadIdx.x;
  const int wcol = blockIdx.x;
  int seg0, seg1;
  if (int(blockIdx.y) < P.nseg0) {
    seg0 = P.lo0 + int(blockIdx.y) * P.rs;
    seg1 = min(seg0 + P.rs, P.hi0);
  } else {
    seg0 = P.lo1 + (int(blockIdx.y) - P.nseg0) * P.rs;
    seg1 = min(seg0 + P.rs, P.hi1);
  }
  if (seg0 >= seg1) return;
  if (P.q0_out && blockIdx.x == 0 && blockIdx.y == 0) {
    const float q0 = srad_q0_warp(P, lane);
    if (lane == 0) *P.q0_out = q0;
  }
  __shared__ __align__(128) SradRing ring;
  if ((wcol + 1) * kSradWarpCols >= P.cols)
    srad_segment<M, FAST, true>(P, seg0, seg1, wcol, lane, ring);
  else
    srad_segment<M, FAST, false>(P, seg0, seg1, wcol, lane, ring);
}

// ROI partials of an existing image (the first iteration's statistics).
__global__ void srad_roi_kernel(const float *jin, int cols, int pitch, int r0, int tile_rows, int roi_r1, int roi_r2,
                                int roi_c1, int roi_c2, int roi_w0, int roi_groups, double *roi_out) {
  const int lane = threadIdx.x & 31;
  const int wcol = roi_w0 + blockIdx.x * 8 + (threadIdx.x >> 5);
  if (wcol >= roi_w0 + roi_groups) return;
  const int col = wcol * kSradWarpCols + 4 * lane;
  for (int g = max(roi_r1, r0); g <= min(roi_r2, r0 + tile_rows - 1); ++g) {
    const float *p = jin + size_t(g - r0 + 1) * size_t(pitch);
    double s = 0.0, s2 = 0.0;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int j = col + k;
      const bool in = j >= roi_c1 && j <= roi_c2 && j < cols;
      const double v = in ? double(p[j]) : 0.0;
      s += v;
      s2 += v * v;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      s += __shfl_xor_sync(kFull, s, o);
      s2 += __shfl_xor_sync(kFull, s2, o);
    }
    if (lane == 0) {
      double *dst = roi_out + 2 * (size_t(g - roi_r1) * roi_groups + (wcol - roi_w0));
      dst[0] = s;
      dst[1] = s2;
    }
  }
}

SradRoi srad_roi_layout(int cols, int r1, int r2, int c1, int c2) {
  SradRoi R;
  R.r1 = r1;
  R.r2 = r2;
  R.c1 = c1;
  R.c2 = c2;
  // warp column groups covering output columns [c1, c2]: group w covers 128w .. 128w+127
  R.w0 = c1 / kSradWarpCols;
  R.groups = c2 / kSradWarpCols - R.w0 + 1;
  R.rows = r2 - r1 + 1;
  (void)cols;
  return R;
}

int srad_pitch(int cols) { return (cols + 3) & ~3; }

cudaError_t launch_srad_roi(const float *jin, int cols, int pitch, int r0, int tile_rows, const SradRoi &roi,
                            double *roi_out, cudaStream_t s) {
  const int grid = (roi.groups + 7) / 8;
  srad_roi_kernel<<<grid, 256, 0, s>>>(jin, cols, pitch, r0, tile_rows, roi.r1, roi.r2, roi.c1, roi.c2, roi.w0,
                                       roi.groups, roi_out);
  return cudaGetLastError();
}

template <bool M, bool FAST>
static int srad_resident_ctas() {
  static int n = [] {
    int dev = 0, sms = 148, per = 1;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, srad_sweep_kernel<M, FAST>, 32, 0);
    return sms * (per > 0 ? per : 1);
  }();
  return n;
}

cudaError_t launch_srad_sweep(int variant, const float *jin, float *jout, const double *roi_in, float *q0_out,
                              double *roi_out, int cols, int pitch, int tile_rows, int r0, int R, float lambda,
                              const SradRoi &roi, const SradRange &range, cudaStream_t s,
                              const double *const *roi_parts, const int *roi_owner) {
  SradParams P;
  P.jin = jin;
  P.jout = jout;
  P.roi_in = roi_in;
  P.roi_parts = roi_parts;
  P.roi_owner = roi_owner;
  P.q0_out = q0_out;
  P.npix = double(roi.rows) * double(roi.c2 - roi.c1 + 1);
  P.roi_out = roi_out;
  P.cols = cols;
  P.pitch = pitch;
  P.tile_rows = tile_rows;
  P.r0 = r0;
  P.R = R;
  P.lo0 = range.lo0;
  P.hi0 = range.hi0;
  P.lo1 = range.lo1;
  P.hi1 = range.hi1;
  P.lq = 0.25f * lambda;
  P.nz = -0.0f;
  P.roi_r1 = roi.r1;
  P.roi_r2 = roi.r2;
  P.roi_c1 = roi.c1;
  P.roi_c2 = roi.c2;
  P.roi_w0 = roi.w0;
  P.roi_groups = roi.groups;
  const int n0 = max(0, range.hi0 - range.lo0), n1 = max(0, range.hi1 - range.lo1);
  if (n0 + n1 == 0) return cudaSuccess;
  const bool fast = variant & 0x100;   // DARM_FAST_MATH
  const bool melded = variant & 1;
  const int resident = melded ? (fast ? srad_resident_ctas<true, true>() : srad_resident_ctas<true, false>())
                              : (fast ? srad_resident_ctas<false, true>() : srad_resident_ctas<false, false>());
  const int gx = (cols + kSradWarpCols - 1) / kSradWarpCols;   // one warp (CTA) per 128 columns
  // Segments: one wave of resident CTAs when the rows allow (every warp one
  // long segment; the 5-row window start is re-read per segment), at least
  // 32 rows per segment.
  const int want_y = max(1, resident / gx);
  int rs = (n0 + n1 + want_y - 1) / want_y;
  rs = max(32, rs);
  P.rs = rs;
  P.nseg0 = (n0 + rs - 1) / rs;
  const int nseg1 = (n1 + rs - 1) / rs;
  dim3 grid(gx, P.nseg0 + nseg1);
  if (melded)
    fast ? srad_sweep_kernel<true, true><<<grid, 32, 0, s>>>(P) : srad_sweep_kernel<true, false><<<grid, 32, 0, s>>>(P);
  else
    fast ? srad_sweep_kernel<false, true><<<grid, 32, 0, s>>>(P)
         : srad_sweep_kernel<false, false><<<grid, 32, 0, s>>>(P);
  return cudaGetLastError();
}

// ---- peer-memory row tiles (multi-GPU SRAD without a collective library).
// Every rank's flags[world] live in its own memory; after a phase (the load,
// or one iteration) rank r stores its phase count into flags[r] of every rank.
// Before a phase a rank waits until every peer's flag has reached its own
// count: all peers finished the previous phase (so their J / ROI partials of
// it are complete, and they are done reading this rank's buffers of the phase
// before).  The counts live in device memory, so a captured graph of N
// iterations is reusable across runs.

// one warp: lane k spins on flags[k] (k != rank) until >= *seq; gives up after
// `timeout_ns` and records the failure in *status (never hangs the GPU)
__global__ void srad_peer_wait_kernel(const unsigned *flags, const unsigned *seq, int rank, int world,
                                      unsigned long long timeout_ns, int *status) {
  const int k = threadIdx.x;
  if (k >= world || k == rank) return;
  const unsigned want = *seq;
  unsigned long long t0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  while (true) {
    unsigned v;
    asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(flags + k) : "memory");
    if (int(v - want) >= 0) break;
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    if (t - t0 > timeout_ns) {
      atomicExch(status, 1);
      break;
    }
    __nanosleep(200);
  }
}

// one warp: ++*seq, then lane k stores it into peer k's flags[rank] (release,
// system scope: every write of this rank's earlier kernels is visible first)
__global__ void srad_peer_signal_kernel(unsigned *const *peer_flags, unsigned *seq, int rank, int world) {
  __shared__ unsigned v;
  if (threadIdx.x == 0) {
    v = *seq + 1;
    *seq = v;
  }
  __syncwarp();
  __threadfence_system();
  const int k = threadIdx.x;
  if (k < world) {
    unsigned *dst = peer_flags[k] + rank;
    asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(dst), "r"(v) : "memory");
  }
}

// halo rows: dst local row 0 <- the upper neighbour's last own row, dst local
// rows n+1, n+2 <- the lower neighbour's first two own rows (peer loads over
// NVLink, 16 bytes per thread, volatile: the neighbour wrote them this phase)
__global__ void srad_peer_halo_kernel(float *dst, const float *up, int up_rows, const float *down, int n,
                                      int pitch) {
  const int v4 = pitch / 4;
  const int r = blockIdx.y;   // 0: top halo, 1, 2: bottom halos
  const float4 *src = nullptr;
  float4 *out = nullptr;
  if (r == 0 && up) {
    src = reinterpret_cast<const float4 *>(up + size_t(up_rows) * pitch);
    out = reinterpret_cast<float4 *>(dst);
  } else if (r > 0 && down) {
    src = reinterpret_cast<const float4 *>(down + size_t(r) * pitch);
    out = reinterpret_cast<float4 *>(dst + size_t(n + r) * pitch);
  }
  if (!src) return;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < v4; i += gridDim.x * blockDim.x) out[i] = __ldcv(src + i);
}

cudaError_t launch_srad_peer_wait(const unsigned *flags, const unsigned *seq, int rank, int world,
                                  unsigned long long timeout_ns, int *status, cudaStream_t s) {
  srad_peer_wait_kernel<<<1, 32, 0, s>>>(flags, seq, rank, world, timeout_ns, status);
  return cudaGetLastError();
}
cudaError_t launch_srad_peer_signal(unsigned *const *peer_flags, unsigned *seq, int rank, int world, cudaStream_t s) {
  srad_peer_signal_kernel<<<1, 32, 0, s>>>(peer_flags, seq, rank, world);
  return cudaGetLastError();
}
cudaError_t launch_srad_peer_halo(float *dst, const float *up, int up_rows, const float *down, int n, int pitch,
                                  cudaStream_t s) {
  const int v4 = pitch / 4;
  dim3 grid((v4 + 255) / 256 < 16 ? (v4 + 255) / 256 : 16, 3);
  srad_peer_halo_kernel<<<grid, 256, 0, s>>>(dst, up, up_rows, down, n, pitch);
  return cudaGetLastError();
}

}  // namespace darm_gpu
