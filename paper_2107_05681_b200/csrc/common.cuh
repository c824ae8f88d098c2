// common.cuh — shared helpers for the sm_100a corpus kernels.
//
// IR semantics (from /root/reference/proj/src/interp.cpp):
//   add/sub/mul/and/or/xor wrap as uint32 (interp.cpp:118-130)
//   shl/shr mask the amount with 31; shr is logical (interp.cpp:126-127)
//   icmp.* are signed and produce 0/1 (interp.cpp:145-164)
//   select takes c != 0 (interp.cpp:165-171)
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace darm_gpu {

__device__ __forceinline__ int32_t ir_add(int32_t a, int32_t b) { return int32_t(uint32_t(a) + uint32_t(b)); }
__device__ __forceinline__ int32_t ir_sub(int32_t a, int32_t b) { return int32_t(uint32_t(a) - uint32_t(b)); }
__device__ __forceinline__ int32_t ir_mul(int32_t a, int32_t b) { return int32_t(uint32_t(a) * uint32_t(b)); }
__device__ __forceinline__ int32_t ir_xor(int32_t a, int32_t b) { return a ^ b; }
__device__ __forceinline__ int32_t ir_and(int32_t a, int32_t b) { return a & b; }
__device__ __forceinline__ int32_t ir_shl(int32_t a, int32_t b) { return int32_t(uint32_t(a) << (uint32_t(b) & 31u)); }
__device__ __forceinline__ int32_t ir_shr(int32_t a, int32_t b) { return int32_t(uint32_t(a) >> (uint32_t(b) & 31u)); }

// Forms of a kernel: the `variant` codes of darm_gpu.h.
enum : int {
  kUnmelded = 0,    // original CFG, IPDOM reconvergence kept (real branches in SASS)
  kMelded = 1,      // the control flow runDarm emits
  kPredicated = 2,  // original CFG as ptxas compiles it (short arms if-converted)
  kLiteral = 3,     // bitonic sorts: App. A.2's select chain on `up` as printed
};

// Arm fences.  Without them LLVM's SimplifyCFG hoists the
// identical leading instructions of two arms (`load in; mul 3` in sb1) and
// sinks the identical tails (`add; store out`): the compiler would meld the
// "unmelded" kernel itself.
//   DARM_ARM:   a volatile asm with a distinct text per arm: never identical
//               across arms and not speculatable, so NVVM cannot hoist, sink
//               or merge across it.  It emits no SASS and has no memory
//               clobber (both forms keep the same load classes, e.g.
//               LDG.E.CONSTANT for read-only __restrict__ inputs).
//   DARM_IPDOM: DARM_ARM plus one PMTRIG (`pmevent`, a performance-monitor
//               trigger with no architectural effect): ptxas does not
//               if-convert a block holding it, so the arm stays behind a real
//               divergent branch (BSSY / @P BRA / BSYNC) — the IPDOM
//               reconvergence of interp.cpp:298-306.  Cost: one issue slot
//               per arm executed.
//   DARM_ARM_F: DARM_IPDOM in the kUnmelded form, DARM_ARM otherwise.
#define DARM_ARM(tag) asm volatile("// arm " tag)
#define DARM_IPDOM(tag) asm volatile("pmevent 0; // arm " tag)
#define DARM_ARM_F(F, tag)        \
  do {                            \
    if constexpr ((F) == kUnmelded) \
      DARM_IPDOM(tag);            \
    else                          \
      DARM_ARM(tag);              \
  } while (0)

// 32-byte vectors (LDG/STG.E.ENL2.256): with R >= 8 consecutive keys per thread
// each warp instruction covers whole sectors; 16-byte vectors at a 64-byte
// thread stride touch every sector twice (2x the L1 sector traffic).
__device__ __forceinline__ bool aligned32(const void *p) { return (reinterpret_cast<uintptr_t>(p) & 31) == 0; }
__device__ __forceinline__ void ld_v8(const int32_t *p, int32_t *v) {
  asm("ld.global.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
      : "l"(p));
}
__device__ __forceinline__ void st_v8(int32_t *p, const int32_t *v) {
  asm volatile("st.global.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p), "r"(v[0]), "r"(v[1]), "r"(v[2]),
               "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7])
               : "memory");
}

// In-register compare-exchange (lo, hi) = (min, max) of (a, b).  For the pairs
// with f set the larger key is rebuilt on the FMA pipe as a + b - lo (exact in
// wrapping 32-bit arithmetic): two IMADs by the runtime unit `one` / `mone`
// (gridDim.y = 1, opaque to both compilers) replace one VIMNMX on the ALU pipe,
// which the compare-exchanges saturate.  DARM_CX_FMA_MOD = 0 turns it off.
// resident 256-thread CTAs per SM the prefetching register kernel is built for
#ifndef DARM_BITONIC_MIN_CTAS
#define DARM_BITONIC_MIN_CTAS 4
#endif
#ifndef DARM_CX_FMA_MOD
#define DARM_CX_FMA_MOD 2
#endif
__device__ __forceinline__ void cx_pair(bool f, int32_t a, int32_t b, int32_t &lo, int32_t &hi, uint32_t one,
                                        uint32_t mone) {
  lo = min(a, b);
  if (f) {   // compile-time after unrolling
    uint32_t s, h;
    asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(s) : "r"(a), "r"(one), "r"(b));
    asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(h) : "r"(lo), "r"(mone), "r"(s));
    hi = int32_t(h);
  } else {
    hi = max(a, b);
  }
}
__host__ __device__ constexpr bool cx_on_fma(int j, int mod = DARM_CX_FMA_MOD) { return mod > 0 && j % (mod > 0 ? mod : 1) == 0; }
// the melded bitonic register kernel (issue-bound rather than ALU-bound)
#ifndef DARM_CX_FMA_MOD_MELDED
#define DARM_CX_FMA_MOD_MELDED DARM_CX_FMA_MOD
#endif

// Barrier over the B threads of one bucket (B a power of two, CTA a multiple
// of B): a warp for B <= 32, a named barrier per bucket (ids 1 .. CTA/B) for
// buckets spanning warps, the whole CTA only when the bucket is the CTA.
// Buckets never exchange keys with each other, so a bucket waits only for
// its own warps.
template <int B, int CTA>
__device__ __forceinline__ void bucket_sync() {
  if constexpr (B >= CTA) {
    __syncthreads();
  } else if constexpr (B <= 32) {
    __syncwarp();
  } else {
    static_assert(CTA / B <= 15, "named barriers 1..15");
    asm volatile("bar.sync %0, %1;" ::"r"(1 + int(threadIdx.x) / B), "n"(B) : "memory");
  }
}

// mbarrier primitives (TMA completion): init, producer arrive + expected
// bytes, consumer wait on a phase parity.
__device__ __forceinline__ unsigned smem_u32(const void *p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t *bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, unsigned parity) {
  asm volatile(
      "{\n .reg .pred P1;\n WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      " @!P1 bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
// 1-D TMA bulk copy global -> shared (16-byte aligned, size a multiple of 16),
// completing on `bar`.
__device__ __forceinline__ void tma_load_1d(void *dst, const void *src, unsigned bytes, uint64_t *bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}

// Lane -> (warp, tid) split for a logical warp of W lanes (1..64).  WT is the
// compile-time warp size when it is a power of two, 0 for a runtime W.
template <int WT>
struct LaneSplit {
  __device__ __forceinline__ static void split(uint32_t g, uint32_t W, uint32_t &w, int &t) {
    if constexpr (WT > 0) {
      constexpr int sh = __builtin_ctz(WT);
      w = g >> sh;
      t = int(g & (WT - 1));
    } else {
      w = g / W;
      t = int(g - w * W);
    }
  }
};

}  // namespace darm_gpu
