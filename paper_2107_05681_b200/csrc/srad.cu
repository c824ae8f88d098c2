// srad.cu — Speckle Reducing Anisotropic Diffusion (SRAD, PAPER.md:778-781,
// 842-851), fp32, unmelded and melded forms.  The reference has no SRAD code;
// the per-pixel mathematics is Rodinia's SRAD restated and
// the CPU oracle (oracle/darm_oracle.c, oracle_srad) performs the same fp32 /
// fp64 operations in the same order.  This translation unit is compiled with
// -fmad=false so no multiply-add is contracted (the oracle is compiled with
// -ffp-contract=off): GPU and CPU agree bit for bit.
//
// Per iteration, with q0sqr from the ROI statistics of the current image J:
//   c(i,j)  = clamp01( 1 / (1 + (q(i,j) - q0sqr) / (q0sqr (1 + q0sqr))) )
//   J'(i,j) = J + (lambda/4) (c(i,j) dN + c(i+1,j) dS + c(i,j) dW + c(i,j+1) dE)
// with dN..dE the differences to the 4 neighbours (image borders clamp).
//
// B200 layout: one fused kernel per iteration.  Each warp owns 30 output
// columns (lanes 1..30; lanes 0 and 31 are halo lanes that only supply
// neighbour values) and sweeps a segment of rows top to bottom, keeping the
// vertical window J(i-1..i+2) and c(i), c(i+1) in registers and exchanging
// west/east neighbours with __shfl_sync.  HBM traffic is one read of J and
// one write of J' per pixel (8 B/px/iteration; the Rodinia layout moves
// ~52 B/px).  J is double-buffered (J -> J').
//
// The divergent regions are
//   R_B  border handling: west/east neighbours at the image's first/last
//        column (thread-position dependent), and lane 31's own east value;
//   R_D  the data-dependent three-way clamp of c (c < 0 / c > 1 / else).
// unmelded: if / else-if chains (fenced arms); melded: select chains.
//
// ROI statistics are reduced deterministically: each warp sums the ROI part
// of its 30 columns of J' in fp64 with a shuffle butterfly, writing one
// partial per (row, warp column group); srad_q0_kernel folds the partials in a
// fixed order.  For row-tiled multi-GPU runs the partial buffer is summed
// across ranks (each entry is owned by exactly one rank, so the sum is exact).
#include <cstdint>

#include "common.cuh"
#include "kernels.h"

namespace darm_gpu {

struct SradParams {
  const float *jin;      // (tile_rows + 3) x cols, local row 0 = global row r0 - 1
  float *jout;           // same layout; local rows 1..tile_rows written
  const float *q0;       // q0sqr of this iteration (device scalar)
  double *roi_out;       // [roi_rows][roi_groups][2] partial sums of J' (may be null)
  int cols, tile_rows, r0, R, rs;
  float lq;              // lambda / 4
  float nz;              // -0.0f (opaque to ptxas: see mulx)
  int roi_r1, roi_r2, roi_c1, roi_c2, roi_w0, roi_groups;
};

__device__ __forceinline__ int clampi(int v, int lo, int hi) { return v < lo ? lo : (v > hi ? hi : v); }

// c for one pixel from its centre and 4 neighbour values (Rodinia SRAD,
// restated).  R_D is the clamp.
// FAST (DARM_FAST_MATH): the five divisions as a multiply by the MUFU
// reciprocal (rcp.approx.ftz: no range fix-up, the operands here are normal
// numbers of moderate size) and the sums of products contracted to FMAs; the
// result stays within the north star's 1e-5 relative tolerance of the IEEE
// path (tests/test_srad.py) instead of matching it bit for bit.
__device__ __forceinline__ float rcp_approx(float b) {
  float r;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(b));
  return r;
}

template <bool FAST>
__device__ __forceinline__ float sdiv(float a, float b) {
  if constexpr (FAST) return a * rcp_approx(b);
  else return a / b;
}

template <bool M, bool FAST>
__device__ __forceinline__ float srad_coeff(float jc, float n, float s, float w, float e, float q0sqr,
                                            float q0den) {
  const float dN = n - jc, dS = s - jc, dW = w - jc, dE = e - jc;
  float g2, l, num, den;
  if constexpr (FAST) {
    g2 = sdiv<FAST>(__fmaf_rn(dE, dE, __fmaf_rn(dW, dW, __fmaf_rn(dS, dS, dN * dN))), jc * jc);
    l = sdiv<FAST>(((dN + dS) + dW) + dE, jc);
    num = __fmaf_rn(-1.0f / 16.0f, l * l, 0.5f * g2);
    den = __fmaf_rn(0.25f, l, 1.0f);
  } else {
    g2 = (((dN * dN + dS * dS) + dW * dW) + dE * dE) / (jc * jc);
    l = (((dN + dS) + dW) + dE) / jc;
    num = (0.5f * g2) - ((1.0f / 16.0f) * (l * l));
    den = 1.0f + (0.25f * l);
  }
  const float qsqr = sdiv<FAST>(num, den * den);
  den = sdiv<FAST>(qsqr - q0sqr, q0den);
  float c = FAST ? rcp_approx(1.0f + den) : 1.0f / (1.0f + den);
  if constexpr (!M) {
    if (c < 0.0f) {                      // R_D: three-way, data dependent
      DARM_ARM("srad.rd.lo");
      c = 0.0f;
    } else if (c > 1.0f) {
      DARM_ARM("srad.rd.hi");
      c = 1.0f;
    }
  } else {
    c = c < 0.0f ? 0.0f : (c > 1.0f ? 1.0f : c);
  }
  return c;
}

// ---- two pixels per instruction: packed fp32 pairs (sm_100 f32x2).  Every
// half is the IEEE operation of the scalar code.  ptxas (12.9) contracts a
// mul.rn.f32x2 feeding an add.rn.f32x2 into FFMA2 even under -fmad=false, so
// the IEEE path forms products as mulx = fma(a, b, z) with z = -0.0f from a
// kernel parameter (exact: a*b + -0 == a*b, and not foldable).
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

__device__ __forceinline__ float2 mulx(float2 a, float2 b, float2 z) { return fma2(a, b, z); }
// (the fast form's product feeds a subtraction / addition: mulx, not mul2)
template <bool FAST>
__device__ __forceinline__ float2 sdiv2(float2 a, float2 b, float2 z) {
  if constexpr (FAST) return mulx(a, make_float2(rcp_approx(b.x), rcp_approx(b.y)), z);
  else return make_float2(a.x / b.x, a.y / b.y);
}

// R_D for one pixel of a pair (same arms as srad_coeff's)
template <bool M>
__device__ __forceinline__ float clamp_rd(float c) {
  if constexpr (!M) {
    if (c < 0.0f) {
      DARM_ARM("srad.rd2.lo");
      c = 0.0f;
    } else if (c > 1.0f) {
      DARM_ARM("srad.rd2.hi");
      c = 1.0f;
    }
    return c;
  } else {
    return c < 0.0f ? 0.0f : (c > 1.0f ? 1.0f : c);
  }
}

// srad_coeff for two pixels at once (rows i and i+1 of one column)
template <bool M, bool FAST, bool PACK>
__device__ __forceinline__ float2 srad_coeff2(float2 jc, float2 n, float2 s, float2 w, float2 e, float q0sqr,
                                              float q0den, float2 z) {
  if constexpr (!PACK)
    return make_float2(srad_coeff<M, FAST>(jc.x, n.x, s.x, w.x, e.x, q0sqr, q0den),
                       srad_coeff<M, FAST>(jc.y, n.y, s.y, w.y, e.y, q0sqr, q0den));
  const float2 dN = sub2(n, jc), dS = sub2(s, jc), dW = sub2(w, jc), dE = sub2(e, jc);
  float2 g2, l, num, den, qsqr;
  if constexpr (FAST) {
    g2 = sdiv2<FAST>(fma2(dE, dE, fma2(dW, dW, fma2(dS, dS, mul2(dN, dN)))), mul2(jc, jc), z);
    l = sdiv2<FAST>(add2(add2(add2(dN, dS), dW), dE), jc, z);
    num = fma2(f2(-1.0f / 16.0f), mul2(l, l), mul2(f2(0.5f), g2));
    den = fma2(f2(0.25f), l, f2(1.0f));
    qsqr = sdiv2<FAST>(num, mul2(den, den), z);
  } else {
    g2 = sdiv2<FAST>(add2(add2(add2(mulx(dN, dN, z), mulx(dS, dS, z)), mulx(dW, dW, z)), mulx(dE, dE, z)),
                     mulx(jc, jc, z), z);
    l = sdiv2<FAST>(add2(add2(add2(dN, dS), dW), dE), jc, z);
    num = sub2(mulx(f2(0.5f), g2, z), mulx(f2(1.0f / 16.0f), mulx(l, l, z), z));
    den = add2(f2(1.0f), mulx(f2(0.25f), l, z));
    qsqr = sdiv2<FAST>(num, mulx(den, den, z), z);
  }
  den = sdiv2<FAST>(sub2(qsqr, f2(q0sqr)), f2(q0den), z);
  const float2 one_den = add2(f2(1.0f), den);
  float2 c;
  if constexpr (FAST)
    c = make_float2(rcp_approx(one_den.x), rcp_approx(one_den.y));
  else
    c = make_float2(1.0f / one_den.x, 1.0f / one_den.y);
  return make_float2(clamp_rd<M>(c.x), clamp_rd<M>(c.y));
}

// CTAs per SM, each form at its best (16384^2 x 100): 5 (48 registers, a
// small spill) for the IEEE forms (unmelded 169.6 -> 160.6 ms, melded 157.5 ->
// 151.0) and the unmelded fast form (126.7 -> 121.1); the melded fast form
// keeps the compiler's 63 registers and 4 CTAs (102.9 ms; bounded to 5: 105.5)
template <bool M, bool FAST, bool PACK, bool IDX32>
__global__ void __launch_bounds__(256, (FAST && M) ? 0 : 5) srad_sweep_kernel(SradParams P) {
  const int lane = threadIdx.x & 31;
  const int wcol = blockIdx.x * 8 + (threadIdx.x >> 5);   // warp column group
  const int j = wcol * 30 + lane - 1;                      // this lane's column
  const int jc = clampi(j, 0, P.cols - 1);
  const bool out_lane = lane >= 1 && lane <= 30 && j < P.cols;
  const int seg0 = blockIdx.y * P.rs;                      // first local own row (0-based)
  if (seg0 >= P.tile_rows) return;
  const int seg1 = min(seg0 + P.rs, P.tile_rows);
  const float q0sqr = *P.q0;
  const float q0den = q0sqr * (1.0f + q0sqr);
  const int cols = P.cols;
  const int gmax = P.R - 1;
  // global row g -> pointer to its (clamped) row in the tile buffer
  auto row = [&](int g) { return P.jin + size_t(clampi(g, 0, gmax) - P.r0 + 1) * cols; };
  // R_B: the west/east neighbour of this lane at image borders and lane 31's
  // east value (no lane to its right).
  auto west_east = [&](const float *rp, float v, float &w, float &e) {   // rp -> (row, jc)
    const float sw = __shfl_up_sync(0xffffffffu, v, 1);
    const float se = __shfl_down_sync(0xffffffffu, v, 1);
    if constexpr (!M) {
      if (j == 0) {
        DARM_ARM("srad.rb.west");
        w = v;
        e = se;
      } else if (lane == 31 || j == cols - 1) {
        DARM_ARM("srad.rb.east");
        w = sw;
        e = j >= cols - 1 ? v : rp[1];                     // j < cols - 1: jc + 1 is in the row
      } else {
        DARM_ARM("srad.rb.mid");
        w = sw;
        e = se;
      }
    } else {
      const bool edge_e = lane == 31 || j >= cols - 1;
      float ee = v;
      if (lane == 31 && j < cols - 1) ee = rp[1];         // the only one-sided run
      w = j == 0 ? v : sw;
      e = edge_e ? ee : se;
    }
  };
  const int g0 = P.r0 + seg0;
  const bool roi_warp = P.roi_out && wcol >= P.roi_w0 && wcol < P.roi_w0 + P.roi_groups;
  auto roi_row = [&](int g, float jn) {
    if (roi_warp && g >= P.roi_r1 && g <= P.roi_r2) {
      const bool in = out_lane && j >= P.roi_c1 && j <= P.roi_c2;
      double s = in ? double(jn) : 0.0, s2 = in ? double(jn) * double(jn) : 0.0;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        s += __shfl_xor_sync(0xffffffffu, s, o);
        s2 += __shfl_xor_sync(0xffffffffu, s2, o);
      }
      if (lane == 0) {
        double *dst = P.roi_out + 2 * (size_t(g - P.roi_r1) * P.roi_groups + (wcol - P.roi_w0));
        dst[0] = s;
        dst[1] = s2;
      }
    }
  };
  // rows past the image clamp to its last row; the buffer holds rows up to glim
  const int glim = min(gmax, P.r0 + P.tile_rows + 1);
  auto rowc = [&](int g) { return row(min(g, glim)); };
  // window at the segment start: rows g0-1 .. g0+3, c and west / east of row g0
  float jm1 = row(g0 - 1)[jc], j0 = row(g0)[jc], jp1 = rowc(g0 + 1)[jc], jp2 = rowc(g0 + 2)[jc];
  float jp3 = rowc(g0 + 3)[jc];
  float w0, e0;
  west_east(row(g0) + jc, j0, w0, e0);
  float c0 = srad_coeff<M, FAST>(j0, jm1, jp1, w0, e0, q0sqr, q0den);
  float *outp = P.jout + size_t(seg0 + 1) * cols + j;
  const float2 z = f2(P.nz);
  // Row addressing in the two-row loop (rows g+1, g+2 for lane 31's east
  // values, g+4, g+5 for the prefetch): tiles under 2^31 elements use 32-bit
  // element indices (clamp + multiply-add, one wide multiply-add for the
  // address: 16384^2 x 100 IEEE melded 147.4 -> 135.2 ms, fast melded 101.3 ->
  // 92.6); larger tiles slide 64-bit row pointers two rows per iteration
  // (clamping through rowc for a tile's last iterations)
  const size_t cs = size_t(cols);
  const float *pg = row(g0) + jc;
  const int off32 = (1 - P.r0) * cols + jc;                  // IDX32: row g's element index = g * cols + off32
  int i = seg0;
  // two rows (g, g+1) per iteration, their arithmetic in f32x2 pairs
  // unrolled twice for the unmelded fast form only (108.7 -> 104.9 ms; the
  // other forms lose: IEEE melded 135 -> 140, fast melded 93 -> 112 at 80
  // registers) — each form at its best
  constexpr int kUnroll = (FAST && !M) ? 2 : 1;
#pragma unroll kUnroll
  for (; i + 1 < seg1; i += 2) {
    const int g = P.r0 + i;
    const float *p1, *p2, *p4, *p5;
    if constexpr (IDX32) {
      // the tile buffer has < 2^31 elements: a 32-bit element index per row
      // (clamp, multiply-add) and one wide multiply-add for the address
      auto at = [&](int gg) { return P.jin + (min(gg, glim) * cols + off32); };
      p1 = at(g + 1);
      p2 = at(g + 2);
      p4 = at(g + 4);
      p5 = at(g + 5);
    } else if (!(FAST && M) && g + 5 <= glim) {   // (no register room in the melded fast form)
      p1 = pg + cs;
      p2 = p1 + cs;
      p4 = p2 + 2 * cs;
      p5 = p4 + cs;
    } else {
      p1 = rowc(g + 1) + jc;
      p2 = rowc(g + 2) + jc;
      p4 = rowc(g + 4) + jc;
      p5 = rowc(g + 5) + jc;
    }
    if constexpr (!IDX32) pg += 2 * cs;
    const float q4 = *p4, q5 = *p5;                         // next iteration's rows, in flight
    float w1, e1, w2, e2;
    west_east(p1, jp1, w1, e1);
    west_east(p2, jp2, w2, e2);
    const float2 cc = srad_coeff2<M, FAST, PACK>(make_float2(jp1, jp2), make_float2(j0, jp1), make_float2(jp2, jp3),
                                           make_float2(w1, w2), make_float2(e1, e2), q0sqr, q0den, z);
    const float c1 = (g + 1 <= gmax) ? cc.x : c0;           // c at the rows below (clamped at the bottom)
    const float c2 = (g + 2 <= gmax) ? cc.y : c1;
    float ce0 = __shfl_down_sync(0xffffffffu, c0, 1), ce1 = __shfl_down_sync(0xffffffffu, c1, 1);
    if (j >= cols - 1) {
      ce0 = c0;
      ce1 = c1;
    }
    const float2 jv = make_float2(j0, jp1), cv = make_float2(c0, c1), cs = make_float2(c1, c2);
    const float2 dN = sub2(make_float2(jm1, j0), jv), dS = sub2(make_float2(jp1, jp2), jv);
    const float2 dW = sub2(make_float2(w0, w1), jv), dE = sub2(make_float2(e0, e1), jv);
    const float2 ce = make_float2(ce0, ce1);
    float2 jn;
    if constexpr (!PACK) {
      if constexpr (FAST) {
        const float dx = __fmaf_rn(ce.x, dE.x, __fmaf_rn(cv.x, dW.x, __fmaf_rn(cs.x, dS.x, cv.x * dN.x)));
        const float dy = __fmaf_rn(ce.y, dE.y, __fmaf_rn(cv.y, dW.y, __fmaf_rn(cs.y, dS.y, cv.y * dN.y)));
        jn = make_float2(__fmaf_rn(P.lq, dx, jv.x), __fmaf_rn(P.lq, dy, jv.y));
      } else {
        const float dx = ((cv.x * dN.x + cs.x * dS.x) + cv.x * dW.x) + ce.x * dE.x;
        const float dy = ((cv.y * dN.y + cs.y * dS.y) + cv.y * dW.y) + ce.y * dE.y;
        jn = make_float2(jv.x + P.lq * dx, jv.y + P.lq * dy);
      }
    } else if constexpr (FAST) {
      const float2 d = fma2(ce, dE, fma2(cv, dW, fma2(cs, dS, mul2(cv, dN))));
      jn = fma2(f2(P.lq), d, jv);
    } else {
      const float2 d = add2(add2(add2(mulx(cv, dN, z), mulx(cs, dS, z)), mulx(cv, dW, z)), mulx(ce, dE, z));
      jn = add2(jv, mulx(f2(P.lq), d, z));
    }
    if (out_lane) {
      outp[0] = jn.x;
      outp[cols] = jn.y;
    }
    outp += 2 * cols;
    roi_row(g, jn.x);
    roi_row(g + 1, jn.y);
    // slide by two rows
    jm1 = jp1;
    j0 = jp2;
    jp1 = jp3;
    jp2 = q4;
    jp3 = q5;
    w0 = w2;
    e0 = e2;
    c0 = c2;
  }
  if (i < seg1) {   // an odd last row
    const int g = P.r0 + i;
    float w1, e1;
    west_east(rowc(g + 1) + jc, jp1, w1, e1);
    const float c1 = (g + 1 <= gmax) ? srad_coeff<M, FAST>(jp1, j0, jp2, w1, e1, q0sqr, q0den) : c0;
    float ce = __shfl_down_sync(0xffffffffu, c0, 1);
    if (j >= cols - 1) ce = c0;
    const float dN = jm1 - j0, dS = jp1 - j0, dW = w0 - j0, dE = e0 - j0;
    float d, jn;
    if constexpr (FAST) {
      d = __fmaf_rn(ce, dE, __fmaf_rn(c0, dW, __fmaf_rn(c1, dS, c0 * dN)));
      jn = __fmaf_rn(P.lq, d, j0);
    } else {
      d = ((c0 * dN + c1 * dS) + c0 * dW) + ce * dE;
      jn = j0 + P.lq * d;
    }
    if (out_lane) *outp = jn;
    roi_row(g, jn);
  }
}

// q0sqr from the ROI partials: rows in order, groups in order, fp64.
__global__ void srad_q0_kernel(const double *roi, int rows, int groups, double npix, float *q0) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  double s = 0.0, s2 = 0.0;
  for (int r = 0; r < rows; ++r)
    for (int g = 0; g < groups; ++g) {
      s += roi[2 * (size_t(r) * groups + g)];
      s2 += roi[2 * (size_t(r) * groups + g) + 1];
    }
  const double mean = s / npix;
  const double var = s2 / npix - mean * mean;
  *q0 = float(var / (mean * mean));
}

// ROI partials of an existing image (the first iteration's statistics).
__global__ void srad_roi_kernel(const float *jin, int cols, int r0, int tile_rows, int roi_r1, int roi_r2,
                                int roi_c1, int roi_c2, int roi_w0, int roi_groups, double *roi_out) {
  const int lane = threadIdx.x & 31;
  const int wcol = roi_w0 + blockIdx.x * 8 + (threadIdx.x >> 5);
  if (wcol >= roi_w0 + roi_groups) return;
  const int j = wcol * 30 + lane - 1;
  const bool in = lane >= 1 && lane <= 30 && j < cols && j >= roi_c1 && j <= roi_c2;
  for (int g = max(roi_r1, r0); g <= min(roi_r2, r0 + tile_rows - 1); ++g) {
    const float v = in ? jin[size_t(g - r0 + 1) * cols + j] : 0.f;
    double s = in ? double(v) : 0.0, s2 = in ? double(v) * double(v) : 0.0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      s += __shfl_xor_sync(0xffffffffu, s, o);
      s2 += __shfl_xor_sync(0xffffffffu, s2, o);
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
  // warp column groups covering output columns [c1, c2]: group w covers 30w .. 30w+29
  R.w0 = c1 / 30;
  R.groups = c2 / 30 - R.w0 + 1;
  R.rows = r2 - r1 + 1;
  (void)cols;
  return R;
}

cudaError_t launch_srad_roi(const float *jin, int cols, int r0, int tile_rows, const SradRoi &roi, double *roi_out,
                            cudaStream_t s) {
  const int grid = (roi.groups + 7) / 8;
  srad_roi_kernel<<<grid, 256, 0, s>>>(jin, cols, r0, tile_rows, roi.r1, roi.r2, roi.c1, roi.c2, roi.w0,
                                       roi.groups, roi_out);
  return cudaGetLastError();
}

cudaError_t launch_srad_q0(const double *roi_in, const SradRoi &roi, float *q0, cudaStream_t s) {
  const double npix = double(roi.rows) * double(roi.c2 - roi.c1 + 1);
  srad_q0_kernel<<<1, 32, 0, s>>>(roi_in, roi.rows, roi.groups, npix, q0);
  return cudaGetLastError();
}

cudaError_t launch_srad_sweep(int variant, const float *jin, float *jout, const float *q0, double *roi_out,
                              int cols, int tile_rows, int r0, int R, float lambda, const SradRoi &roi,
                              cudaStream_t s) {
  SradParams P;
  P.jin = jin;
  P.jout = jout;
  P.q0 = q0;
  P.roi_out = roi_out;
  P.cols = cols;
  P.tile_rows = tile_rows;
  P.r0 = r0;
  P.R = R;
  P.rs = 128;
  P.lq = 0.25f * lambda;
  P.nz = -0.0f;
  P.roi_r1 = roi.r1;
  P.roi_r2 = roi.r2;
  P.roi_c1 = roi.c1;
  P.roi_c2 = roi.c2;
  P.roi_w0 = roi.w0;
  P.roi_groups = roi.groups;
  const int wgroups = (cols + 29) / 30;
  dim3 grid((wgroups + 7) / 8, (tile_rows + P.rs - 1) / P.rs);
  const bool fast = variant & 0x100;   // DARM_FAST_MATH
  // f32x2 pairs only where they pay (measured, 16384^2 x 100): the melded
  // fast path (105.2 -> 101.8 ms).  The unmelded form's per-pixel R_D branches
  // split every pair (126 -> 147 ms) and the IEEE path's scalar divisions
  // around packed products lose too (157 -> 184 ms): both run two rows per
  // iteration in scalar code.
  // 32-bit element indices while the tile buffer (tile_rows + 3 rows) has
  // fewer than 2^31 elements (16384^2 on one GPU: 2.7e8)
  const bool idx32 = int64_t(tile_rows + 3) * cols < (int64_t(1) << 31) && !(variant & 0x200);   // DARM_SRAD_INDEX64
#define SRAD_L(Mm, F, PK)                                                                                   \
  (idx32 ? srad_sweep_kernel<Mm, F, PK, true><<<grid, 256, 0, s>>>(P)                                    \
         : srad_sweep_kernel<Mm, F, PK, false><<<grid, 256, 0, s>>>(P))
  if (variant & 1)
    fast ? SRAD_L(true, true, true) : SRAD_L(true, false, false);
  else
    fast ? SRAD_L(false, true, false) : SRAD_L(false, false, false);
#undef SRAD_L
  return cudaGetLastError();
}

}  // namespace darm_gpu
