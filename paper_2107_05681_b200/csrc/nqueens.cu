// nqueens.cu — N-Queens solution count (NQU) in
// the unmelded and melded forms of paper_2107_05681_b200/ir/nqueens_step.ir.
//
// The reference has no NQU code; the search loop is written in the reference's
// mini-IR (ir/nqueens_step.ir: one iteration = pop / count a solution / push,
// the paper's "if-then-elseif-then") and the melded form below mirrors what the
// reference pass emits for it (runDarm, threshold 0.2: two block-region melds,
// 12 selects, 7 unpredicated runs — DESIGN.md §NQU).  The reference interpreter
// runs the same IR as the oracle (tests/golden/nqueens_chain.json).
//
// Work decomposition: the host enumerates every valid placement of the first
// `base` rows (lowest free column first, so prefix i is deterministic) and
// deals prefix i to rank i % world.  On the GPU every thread runs the IR loop
// on one prefix at a time, fetching the next from a global counter when its
// subtree is exhausted (row < base, the IR's ^s %done test).  Thread state
// (row, cols, d1, d2, av, sol) lives in registers — the IR's st_* globals —
// and the per-row stack (the IR's sk_* shared arrays) in shared memory at
// [array][row - base + 1][thread], conflict-free.
#include <cstdint>

#include "common.cuh"
#include "kernels.h"

namespace darm_gpu {

struct NqParams {
  const uint32_t *prefix;          // n_prefix x {cols, d1, d2}
  uint32_t n_prefix;
  uint32_t *per_prefix;            // solutions per prefix (may be null)
  unsigned long long *total;       // sum of solutions
  unsigned int *next;              // work counter
  int n, base, levels;
  uint32_t mask;
};

template <bool M>
__global__ void __launch_bounds__(256) nqueens_kernel(NqParams P) {
  extern __shared__ uint32_t sk[];
  const int T = blockDim.x;
  const int L = P.levels;
  uint32_t *sk_cols = sk, *sk_d1 = sk + L * T, *sk_d2 = sk + 2 * L * T, *sk_av = sk + 3 * L * T;
  const int lane_off = int(threadIdx.x) - (P.base - 1) * T;  // slot(row) = row*T + lane_off
  const int n1 = P.n - 1;
  int row = P.base - 1;
  uint32_t cols = 0, d1 = 0, d2 = 0, av = 0, sol = 0;
  uint32_t pidx = 0xffffffffu;
  unsigned long long acc = 0;
  for (;;) {
    if (row < P.base) {                                    // ^s: %done
      if (pidx != 0xffffffffu) {
        if (P.per_prefix) P.per_prefix[pidx] = sol;
        acc += sol;
      }
      pidx = atomicAdd(P.next, 1u);
      if (pidx >= P.n_prefix) break;
      cols = __ldg(P.prefix + 3 * pidx);
      d1 = __ldg(P.prefix + 3 * pidx + 1);
      d2 = __ldg(P.prefix + 3 * pidx + 2);
      av = ~(cols | d1 | d2) & P.mask;
      row = P.base;
      sol = 0;
    }
    if constexpr (!M) {
      // ^e: condbr %z ^pop ^nz ; ^nz: condbr %last ^leaf ^push
      if (av == 0) {
        DARM_ARM("nq.pop");                                // ^pop
        const int r1 = row - 1;
        const int ix1 = r1 * T + lane_off;
        cols = sk_cols[ix1];
        d1 = sk_d1[ix1];
        d2 = sk_d2[ix1];
        av = sk_av[ix1];
        row = r1;
        DARM_ARM("nq.pop.end");
      } else if (row == n1) {
        DARM_ARM("nq.leaf");                               // ^leaf
        const uint32_t b1 = av & (0u - av);
        av = av ^ b1;
        sol += 1;
        DARM_ARM("nq.leaf.end");
      } else {
        DARM_ARM("nq.push");                               // ^push
        const uint32_t b2 = av & (0u - av);
        const uint32_t rem2 = av ^ b2;
        const int ix2 = row * T + lane_off;
        sk_av[ix2] = rem2;
        sk_cols[ix2] = cols;
        sk_d1[ix2] = d1;
        sk_d2[ix2] = d2;
        cols = cols | b2;
        d1 = (d1 | b2) << 1;
        d2 = (d2 | b2) >> 1;
        av = ~(cols | d1 | d2) & P.mask;
        row = row + 1;
        DARM_ARM("nq.push.end");
      }
    } else {
      // runDarm output: block-region melds of ^pop and ^leaf
      // into the ^push region.
      const bool z = av == 0;
      const bool last = row == n1;
      const bool sel = z ? false : last;                   // the ^leaf lanes
      const int r1 = (z ? row : 0) - (z ? 1 : int(av));    // melded sub: row-1 | 0-av
      uint32_t b2 = 0, rem2 = 0;
      if (!sel && !z) {                                    // ^push.r.m.g
        b2 = av & uint32_t(r1);
        rem2 = av ^ b2;
      }
      const int sel3 = z ? r1 : row;                       // stack row: pop row-1 | push row
      const int ix1 = sel3 * T + lane_off;
      const bool sel9 = sel ? false : z;                   // the ^pop lanes
      uint32_t c2 = 0, f1 = 0, f2 = 0, b1 = 0;
      if (!sel9) {
        uint32_t u3 = 0, ng1 = 0;
        if (!sel) {                                        // ^push.r.m.g1.r.m.g
          sk_av[ix1] = rem2;
          sk_cols[ix1] = cols;
          sk_d1[ix1] = d1;
          sk_d2[ix1] = d2;
          c2 = cols | b2;
          f1 = (d1 | b2) << 1;
          f2 = (d2 | b2) >> 1;
          u3 = ~(c2 | f1 | f2);
        }
        if (sel) ng1 = 0u - av;                            // ^push.r.m.g1.r.m.g1
        b1 = (sel ? av : u3) & (sel ? ng1 : P.mask);       // melded and: bit | new av
        if (sel) {                                         // ^push.r.m.g1.r.m.g2
          av = av ^ b1;
          sol += 1;
        }
      }
      if (!sel) {                                          // ^push.r.m.u1
        uint32_t pc = 0, pd1 = 0, pd2 = 0, pav = 0;
        if (z) {                                           // ^push.r.m.g2
          pc = sk_cols[ix1];
          pd1 = sk_d1[ix1];
          pd2 = sk_d2[ix1];
          pav = sk_av[ix1];
        }
        cols = z ? pc : c2;
        d1 = z ? pd1 : f1;
        d2 = z ? pd2 : f2;
        av = z ? pav : b1;
        int r2 = 0;
        if (!z) r2 = row + 1;                              // ^push.r.m.g3
        row = z ? r1 : r2;
      }
    }
  }
  // every lane has left the loop: reduce the warp's solution counts
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0 && acc) atomicAdd(P.total, acc);
}

cudaError_t launch_nqueens(int variant, const uint32_t *prefix, uint32_t n_prefix, int n, int base,
                           uint32_t *per_prefix, unsigned long long *total, unsigned int *counter,
                           int sms, cudaStream_t s) {
  NqParams P;
  P.prefix = prefix;
  P.n_prefix = n_prefix;
  P.per_prefix = per_prefix;
  P.total = total;
  P.next = counter;
  P.n = n;
  P.base = base;
  P.levels = n - base + 1;
  P.mask = n >= 32 ? 0xffffffffu : ((1u << n) - 1u);
  const int T = 256;
  const size_t shm = size_t(4) * P.levels * T * sizeof(uint32_t);
  auto kern = variant ? nqueens_kernel<true> : nqueens_kernel<false>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(shm));
  if (e != cudaSuccess) return e;
  int per_sm = 0;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, T, shm);
  if (e != cudaSuccess) return e;
  if (per_sm < 1) return cudaErrorInvalidConfiguration;
  uint64_t grid = uint64_t(sms) * per_sm;
  const uint64_t need = (uint64_t(n_prefix) + T - 1) / T;
  if (grid > need) grid = need;
  if (grid < 1) grid = 1;
  kern<<<unsigned(grid), T, shm, s>>>(P);
  return cudaGetLastError();
}

}  // namespace darm_gpu
