// corpus.cuh — lane bodies of the DARM corpus kernels, one struct per
// /root/reference/proj/corpus/<name>.ir, each in two forms:
//
//   F = kUnmelded   : the original CFG.  Every divergent branch of the IR is a
//                    real branch: each arm starts with DARM_IPDOM (NVVM cannot
//                    hoist/sink/merge across it, ptxas cannot if-convert an arm
//                    holding it), so the hardware runs the arms one after the
//                    other and reconverges at the immediate post-dominator
//                    (BSSY/@P BRA/BSYNC in SASS, checked by tests/test_abi.py).
//   F = kPredicated : the same source with NVVM-only fences (DARM_ARM): what
//                    ptxas makes of the original CFG — it if-converts short
//                    arms into complementary predicated runs (both arms still
//                    issue one after the other, without the branch).
//   F = kMelded     : the control flow runDarm emits for the kernel
//                    (melding_driver.cpp:54-100, threshold 0.2; printed IR in
//                    SURVEY.md Appendix A and DESIGN.md §Melded forms):
//                    common instructions hoisted once, select-based operand
//                    choice, one-sided tails kept as guarded ("unpredicated")
//                    runs.
//
// Read-only inputs are loaded with __ldg in every form (LDG.E.CONSTANT), so the
// forms differ in control flow, not in load class.
// Every global is indexed by %t in the corpus, so arrays are stored compact:
// word g = w*warp + t is element t of warp w's copy (see darm_gpu.h).
// `undef` incomings of the melded phis are materialised as 0; they are never
// selected (interp.cpp:165-171 propagates only the chosen side).
#pragma once

#include "common.cuh"

namespace darm_gpu {

struct CorpusParams {
  int32_t argv[4];           // broadcast argument values
  const int32_t *argp[4];    // per-warp / per-lane argument arrays
  int32_t *gl[4];            // globals, declaration order, compact layout
  const int32_t *sh;         // shared initialiser (n_warps x shared size)
  int32_t *faults;           // per-warp fault counters (may be null)
  uint32_t warp;             // logical warp size W (1..64)
  uint32_t total;            // n_warps * W lanes
  uint32_t n_warps;
  uint32_t shared_size;      // declared shared words per warp
};

// ---------------------------------------------------------------- sb1
// sb1.ir:7-28  out[t] = in[t]*3 + (t < n ? aux2[t] : aux3[t])
struct Sb1 {
  static constexpr int kParams = 1;
  template <int F>
  __device__ __forceinline__ static void lane(const CorpusParams &P, uint32_t g, int t, const int32_t *a) {
    constexpr bool M = F == kMelded;
    const int32_t *__restrict__ in = P.gl[0];
    const int32_t *__restrict__ aux2 = P.gl[1];
    const int32_t *__restrict__ aux3 = P.gl[2];
    int32_t *__restrict__ out = P.gl[3];
    const int32_t n = a[0];
    const bool c = t < n;                                  // ^a1 sb1.ir:9-10
    if constexpr (!M) {
      if (c) {                                             // condbr %c ^a2 ^a3 (:11)
        DARM_ARM_F(F, "sb1.a2");                                // ^a2 :12-18
        int32_t v2 = __ldg(in + g);
        int32_t m2 = ir_mul(v2, 3);
        int32_t e2 = __ldg(aux2 + g);
        out[g] = ir_add(m2, e2);
        DARM_ARM("sb1.a2.end");
      } else {
        DARM_ARM_F(F, "sb1.a3");                                // ^a3 :19-25
        int32_t v3 = __ldg(in + g);
        int32_t m3 = ir_mul(v3, 3);
        int32_t e3 = __ldg(aux3 + g);
        out[g] = ir_add(m3, e3);
        DARM_ARM("sb1.a3.end");
      }
    } else {
      int32_t v2 = __ldg(in + g);                                  // hoisted common
      int32_t m2 = ir_mul(v2, 3);
      int32_t e3 = 0, e2 = 0;
      if (!c) e3 = __ldg(aux3 + g);                                // ^a2.m.g  (false-only run)
      if (c) e2 = __ldg(aux2 + g);                                 // ^a2.m.g1 (true-only run)
      int32_t sel = c ? e2 : e3;                           // ^a2.m.u1 select
      out[g] = ir_add(m2, sel);
    }
  }
};

// ---------------------------------------------------------------- sb1r
// sb1r.ir:5-26  arms differ except the memory accesses
struct Sb1r {
  static constexpr int kParams = 1;
  template <int F>
  __device__ __forceinline__ static void lane(const CorpusParams &P, uint32_t g, int t, const int32_t *a) {
    constexpr bool M = F == kMelded;
    const int32_t *__restrict__ in = P.gl[0];
    int32_t *__restrict__ out = P.gl[1];
    const int32_t n = a[0];
    const bool c = t < n;
    if constexpr (!M) {
      if (c) {
        DARM_ARM_F(F, "sb1r.a2");                               // :10-16
        int32_t v2 = __ldg(in + g);
        int32_t m2 = ir_mul(v2, 3);
        int32_t y2 = ir_add(m2, n);
        int32_t z2 = ir_shl(y2, 1);
        out[g] = z2;
        DARM_ARM("sb1r.a2.end");
      } else {
        DARM_ARM_F(F, "sb1r.a3");                               // :17-23
        int32_t v3 = __ldg(in + g);
        int32_t x3 = ir_xor(v3, n);
        int32_t s3 = ir_sub(x3, 7);
        int32_t y3 = ir_add(s3, 2);
        out[g] = y3;
        DARM_ARM("sb1r.a3.end");
      }
    } else {                                               // runDarm: block-block, 3 selects, 3 runs
      int32_t v2 = __ldg(in + g);
      int32_t s3 = 0, m2 = 0, z2 = 0;
      if (!c) {                                            // ^a2.m.g
        int32_t x3 = ir_xor(v2, n);
        s3 = ir_sub(x3, 7);
      }
      if (c) m2 = ir_mul(v2, 3);                           // ^a2.m.g1
      int32_t sel = c ? m2 : s3;
      int32_t sel1 = c ? n : 2;
      int32_t y2 = ir_add(sel, sel1);
      if (c) z2 = ir_shl(y2, 1);                           // ^a2.m.g2
      int32_t sel2 = c ? z2 : y2;
      out[g] = sel2;
    }
  }
};

// ---------------------------------------------------------------- sb2 / sb2r
// sb2.ir:5-36 / sb2r.ir:5-36  one if-then region per side
template <bool R>
struct Sb2T {
  static constexpr int kParams = 1;
  template <int F>
  __device__ __forceinline__ static void lane(const CorpusParams &P, uint32_t g, int t, const int32_t *a) {
    constexpr bool M = F == kMelded;
    const int32_t *__restrict__ in = P.gl[0];
    int32_t *__restrict__ out = P.gl[1];
    const int32_t n = a[0];
    const bool c = t < n;
    if constexpr (!M) {
      if (c) {
        DARM_ARM_F(F, "sb2.b2");                                // ^b2 :10-21
        int32_t v2 = __ldg(in + g);
        bool g2 = v2 > n;
        int32_t p2 = v2;
        if (g2) {
          DARM_ARM_F(F, "sb2.b2a");
          p2 = ir_add(ir_mul(v2, 2), 1);
        }
        DARM_ARM("sb2.b2m");
        out[g] = p2;
      } else {
        DARM_ARM_F(F, "sb2.b3");                                // ^b3 :22-33
        int32_t v3 = __ldg(in + g);
        bool g3 = v3 > n;
        int32_t p3 = v3;
        if (g3) {
          DARM_ARM_F(F, "sb2.b3a");
          p3 = R ? ir_sub(ir_xor(v3, n), 3) : ir_add(ir_mul(v3, 2), 1);
        }
        DARM_ARM("sb2.b3m");
        out[g] = p3;
      }
    } else if constexpr (!R) {                             // sb2: region-region, MP 0.5, 1 select
      int32_t v2 = __ldg(in + g);
      bool g2 = v2 > n;
      int32_t p2 = v2;
      if (g2) p2 = ir_add(ir_mul(v2, 2), 1);               // ^b2a.m
      out[g] = c ? p2 : p2;                                // %sel = select %c %p2 %p2
    } else {                                               // sb2r: region-region, 1 select, 2 runs
      int32_t v2 = __ldg(in + g);
      bool g2 = v2 > n;
      int32_t u3 = 0, u2 = 0;
      if (g2) {                                            // ^b2a.m
        if (!c) u3 = ir_sub(ir_xor(v2, n), 3);             // ^b2a.m.g
        if (c) u2 = ir_add(ir_mul(v2, 2), 1);              // ^b2a.m.g1
      }
      int32_t p2 = g2 ? u2 : v2;                           // ^b2m.m phis
      int32_t p3 = g2 ? u3 : v2;
      out[g] = c ? p2 : p3;
    }
  }
};
using Sb2 = Sb2T<false>;
using Sb2r = Sb2T<true>;

// ---------------------------------------------------------------- sb3 / sb3r
// sb3.ir:7-58 / sb3r.ir:7-58  two sequential if-then regions per side
template <bool R>
struct Sb3T {
  static constexpr int kParams = 1;
  template <int F>
  __device__ __forceinline__ static void lane(const CorpusParams &P, uint32_t g, int t, const int32_t *a) {
    constexpr bool M = F == kMelded;
    const int32_t *__restrict__ in = P.gl[0];
    const int32_t *__restrict__ in2 = P.gl[1];
    int32_t *__restrict__ out = P.gl[2];
    int32_t *__restrict__ out2 = P.gl[3];
    const int32_t n = a[0];
    const bool c = t < n;
    if constexpr (!M) {
      if (c) {
        DARM_ARM_F(F, "sb3.c2");                                // ^c2..^c3m :12-33
        int32_t v1 = __ldg(in + g);
        int32_t p1 = v1;
        if (v1 > n) {
          DARM_ARM_F(F, "sb3.c2a");
          p1 = ir_mul(v1, 2);
        }
        DARM_ARM("sb3.c2m");
        out[g] = p1;
        int32_t v2 = __ldg(in2 + g);
        int32_t p2 = v2;
        if (v2 > n) {
          DARM_ARM_F(F, "sb3.c3a");
          p2 = ir_add(v2, 7);
        }
        DARM_ARM("sb3.c3m");
        out2[g] = p2;
      } else {
        DARM_ARM_F(F, "sb3.c5");                                // ^c5..^c6m :34-55
        int32_t v5 = __ldg(in + g);
        int32_t p5 = v5;
        if (v5 > n) {
          DARM_ARM_F(F, "sb3.c5a");
          p5 = R ? ir_xor(v5, 9) : ir_mul(v5, 2);
        }
        DARM_ARM("sb3.c5m");
        out[g] = p5;
        int32_t v6 = __ldg(in2 + g);
        int32_t p6 = v6;
        if (v6 > n) {
          DARM_ARM_F(F, "sb3.c6a");
          p6 = R ? ir_sub(v6, 5) : ir_add(v6, 7);
        }
        DARM_ARM("sb3.c6m");
        out2[g] = p6;
      }
    } else if constexpr (!R) {                             // sb3: 2 region-region melds
      int32_t v1 = __ldg(in + g);
      int32_t p1 = v1;
      if (v1 > n) p1 = ir_mul(v1, 2);                      // ^c2a.m
      out[g] = c ? p1 : p1;
      int32_t v2 = __ldg(in2 + g);
      int32_t p2 = v2;
      if (v2 > n) p2 = ir_add(v2, 7);                      // ^c3a.m
      out2[g] = c ? p2 : p2;
    } else {                                               // sb3r: 2 melds, 2 runs each
      int32_t v1 = __ldg(in + g);
      bool g1 = v1 > n;
      int32_t w5 = 0, w1 = 0;
      if (g1) {                                            // ^c2a.m
        if (!c) w5 = ir_xor(v1, 9);
        if (c) w1 = ir_mul(v1, 2);
      }
      int32_t p1 = g1 ? w1 : v1, p5 = g1 ? w5 : v1;
      out[g] = c ? p1 : p5;
      int32_t v2 = __ldg(in2 + g);
      bool g2 = v2 > n;
      int32_t w6 = 0, w2 = 0;
      if (g2) {                                            // ^c3a.m
        if (!c) w6 = ir_sub(v2, 5);
        if (c) w2 = ir_add(v2, 7);
      }
      int32_t p2 = g2 ? w2 : v2, p6 = g2 ? w6 : v2;
      out2[g] = c ? p2 : p6;
    }
  }
};
using Sb3 = Sb3T<false>;
using Sb3r = Sb3T<true>;

// ---------------------------------------------------------------- sb4 / sb4r
// sb4.ir:5-30 / sb4r.ir:5-30  if / else-if / else
template <bool R>
struct Sb4T {
  static constexpr int kParams = 2;
  template <int F>
  __device__ __forceinline__ static void lane(const CorpusParams &P, uint32_t g, int t, const int32_t *a) {
    constexpr bool M = F == kMelded;
    const int32_t *__restrict__ in = P.gl[0];
    int32_t *__restrict__ out = P.gl[1];
    const int32_t h = a[0], q = a[1];
    const bool c1 = t < h;                                 // ^d1 :7-8
    if constexpr (!M) {
      if (c1) {
        DARM_ARM_F(F, "sb4.d2");                                // ^d2 :10-14
        out[g] = ir_add(__ldg(in + g), 1);
        DARM_ARM("sb4.d2.end");
      } else {
        DARM_ARM_F(F, "sb4.d3");                                // ^d3 :15-17
        const bool c2 = t < q;
        if (c2) {
          DARM_ARM_F(F, "sb4.d4");                              // ^d4 :18-22
          int32_t v4 = __ldg(in + g);
          out[g] = R ? ir_mul(v4, 3) : ir_add(v4, 1);
          DARM_ARM("sb4.d4.end");
        } else {
          DARM_ARM_F(F, "sb4.d5");                              // ^d5 :23-27
          int32_t v5 = __ldg(in + g);
          out[g] = R ? ir_xor(v5, 7) : ir_add(v5, 1);
          DARM_ARM("sb4.d5.end");
        }
      }
    } else if constexpr (!R) {                             // sb4: block-region then block-block
      const bool c2 = t < q;
      const bool sel = c1 ? true : c2;
      int32_t w2 = ir_add(__ldg(in + g), 1);
      int32_t pred = 0;
      if (!sel) {                                          // ^d4.r.m.m.g: predicated store
        int32_t old = out[g];
        pred = c1 ? old : w2;
      }
      out[g] = sel ? w2 : pred;
    } else {                                               // sb4r: two block-region melds
      const bool c2 = t < q;
      const bool sel = c1 ? true : c2;
      int32_t w4u = 0, v2e = 0;
      if (sel) {                                           // ^d4.r.m
        int32_t v2 = __ldg(in + g);
        if (!c1) w4u = ir_mul(v2, 3);                      // ^d4.r.m.g
        v2e = v2;
      }
      const bool sel2 = sel ? c1 : true;
      int32_t w2u = 0;
      if (sel2) w2u = ir_add(v2e, 1);                      // ^d4.r.m.g1.m
      int32_t w5u = 0;
      if (!sel) {                                          // ^d4.r.m.u1.m.g
        int32_t v5 = __ldg(in + g);
        w5u = ir_xor(v5, 7);
        // runDarm's block also loads out[t] (the predicated store's old value)
        // for sel3 = select sel w2 old; that value reaches the store only when
        // c1, where sel is true, so it is dead.  The reference's dead-code pass
        // keeps it because an IR load may fault (post_opt.cpp:209-220); here
        // t < warp <= the declared size, so it cannot, and it is not issued.
      }
      int32_t sel3 = w2u;                                  // select sel w2 old, sel true where used
      int32_t sel4 = sel ? w4u : w5u;
      out[g] = c1 ? sel3 : sel4;
    }
  }
};
using Sb4 = Sb4T<false>;
using Sb4r = Sb4T<true>;

// ---------------------------------------------------------------- nested
// nested.ir:6-41  divergent diamond whose arms are data-dependent diamonds
struct Nested {
  static constexpr int kParams = 1;
  template <int F>
  __device__ __forceinline__ static void lane(const CorpusParams &P, uint32_t g, int t, const int32_t *a) {
    constexpr bool M = F == kMelded;
    const int32_t *__restrict__ in = P.gl[0];
    int32_t *__restrict__ out = P.gl[1];
    const int32_t n = a[0];
    const bool c = t < n;
    if constexpr (!M) {
      if (c) {
        DARM_ARM_F(F, "nested.l");                              // ^l..^lm :11-24
        int32_t lv = __ldg(in + g);
        int32_t lp;
        if (lv > n) {
          DARM_ARM_F(F, "nested.la");
          lp = ir_mul(lv, 2);
        } else {
          DARM_ARM_F(F, "nested.lb");
          lp = ir_add(lv, 9);
        }
        DARM_ARM("nested.lm");
        out[g] = lp;
      } else {
        DARM_ARM_F(F, "nested.r");                              // ^r..^rm :25-38
        int32_t rv = __ldg(in + g);
        int32_t rp;
        if (rv > n) {
          DARM_ARM_F(F, "nested.ra");
          rp = ir_mul(rv, 2);
        } else {
          DARM_ARM_F(F, "nested.rb");
          rp = ir_add(rv, 9);
        }
        DARM_ARM("nested.rm");
        out[g] = rp;
      }
    } else {                                               // region-region then block-block
      int32_t lv = __ldg(in + g);
      bool lc = lv > n;
      int32_t ly = 0, lx = 0;
      if (!lc) ly = ir_add(lv, 9);                         // ^la.m.m.g
      if (lc) lx = ir_mul(lv, 2);                          // ^la.m.m.g1
      int32_t lp = lc ? lx : ly;                           // ^p phi
      out[g] = c ? lp : lp;
    }
  }
};

// ---------------------------------------------------------------- bitonic step
// bitonic.ir:6-43, one compare-exchange step with the lane's own slot buf[t]
// held in a register (`cv`); `b0` is the partner's slot buf[t^k] read before
// any store (:10).  Returns what the lane leaves in buf[t].
//
// In both forms the IR's "compare, then conditionally store b0" pairs are
// written as the min/max they compute (`need1 = keep ? cv>b0 : cv<b0;
// if (need1) buf[t] = b0` == `keep ? min(cv,b0) : max(cv,b0)`), so the two
// unmelded forms differ from each other only in control flow.
// Forms (F, darm_gpu.h variant codes):
//   kUnmelded / kPredicated: the divergent `condbr %up ^c ^d` (:16) with each
//     arm's compares/select/store (^c :17-27, ^d :28-38); kUnmelded leads each
//     arm with DARM_IPDOM so ptxas keeps the branch, kPredicated lets ptxas
//     if-convert the two one-instruction arms;
//   kLiteral: SURVEY App. A.2's melded control flow: gt1 hoisted, the lt
//     compare of the two guarded runs (same operands, so one compare),
//     sel = select up gt1 lt2, sel1 = select up lt1 gt1, need1 = select keep
//     sel sel1, one store of b0.  The chain folds to need1 = (keep == up) ?
//     gt1 : lt, and "store b0 if need1" to (keep == up) ? min(cv, b0) :
//     max(cv, b0) — the same min/max the unmelded arms are written with, so
//     the forms differ in control flow only;
//   kMelded is not handled here: the sorts fold `up` into the data (order
//     flips) and issue one predicated min/max (bitonic_sort.cu).
template <int F>
__device__ __forceinline__ int32_t bitonic_exchange(int32_t cv, int32_t b0, bool keep, bool up) {
  static_assert(F != kMelded, "the order-flip melded form lives in the sorts");
  if constexpr (F == kLiteral) {
    const bool need_lt = keep == up;                       // need1 = select keep (select up ..) (select up ..)
    return need_lt ? min(cv, b0) : max(cv, b0);            // ^e.m: the single store of b0
  } else {
    if (up) {                                              // condbr %up ^c ^d (:16)
      DARM_ARM_F(F, "bitonic.c");                          // ^c/^e: keep ? (cv>b0) : (cv<b0)
      cv = keep ? min(cv, b0) : max(cv, b0);
      DARM_ARM("bitonic.x1");
    } else {
      DARM_ARM_F(F, "bitonic.d");                          // ^d/^f: keep ? (cv<b0) : (cv>b0)
      cv = keep ? max(cv, b0) : min(cv, b0);
      DARM_ARM("bitonic.x2");
    }
    return cv;
  }
}

}  // namespace darm_gpu
