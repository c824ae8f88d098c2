// nqueens.cu — N-Queens solution count (NQU) in
// the unmelded and melded forms of paper_2107_05681_b200/ir/nqueens_sym.ir.
//
// The reference has no NQU code; the search loop is written in the reference's
// mini-IR (ir/nqueens_sym.ir: one iteration = push a queen or pop one, the
// paper's divergent search-loop branch) and the melded form below mirrors what
// the reference pass emits for it (runDarm, threshold 0.2: one block-block
// meld of ^pop and ^push, MP 0.435, 7 selects, 6 unpredicated runs —
// DESIGN.md §NQU).  The reference interpreter runs the same IR as the oracle
// (tests/golden/nqueens_chain.json).
//
// Formulation (ir/nqueens_sym.ir header): the diagonals are kept in board
// coordinates (d1 bit r + c, d2 bit c - r + n - 1), the per-row stack holds
// only the column bit placed at that row, and a pop takes that bit back.  Push
// and pop then toggle the same three words with b shifted by the same row, so
// the two arms are one chain in mirror image.  A solution is a push that
// reaches row n.  The words are 32-bit for n <= 16 and 64-bit up to n = 31.
//
// Work decomposition: the host enumerates every valid placement of the first
// `base` rows (lowest free column first, so prefix i is deterministic) and
// deals prefix i to rank i % world.  On the GPU every thread runs the IR loop
// on one prefix at a time; a lane whose subtree is exhausted (row < base, the
// IR's ^s %done test) takes the next prefix, the lanes of a warp that need one
// in the same iteration claiming consecutive prefixes with one atomic
// (__activemask / __popc / __shfl_sync).  Thread state (row, cols, d1, d2, av,
// sol) lives in registers — the IR's st_* globals — and the one-word-per-row
// stack (the IR's sk_b) in shared memory at [row - base + 1][thread],
// conflict-free.
#include <cstdint>

#include "common.cuh"
#include "kernels.h"

namespace darm_gpu {

struct NqParams {
  const uint32_t *prefix;          // n_prefix x {cols, d1, d2} (row-relative, as enumerated)
  uint32_t n_prefix;
  uint32_t n_double;               // prefixes [0, n_double) count twice (mirror symmetry)
  uint32_t *per_prefix;            // solutions per prefix (may be null)
  unsigned long long *total;       // sum of solutions
  unsigned int *next;              // work counter
  int n, base, levels;
  uint32_t mask;
};

template <bool M, typename W>
__global__ void __launch_bounds__(256) nqueens_kernel(NqParams P) {
  extern __shared__ uint32_t sk_b[];
  constexpr int kShift = 8 * sizeof(W) - 1;   // shift amounts wrap like the IR's (interp.cpp:126-127)
  const int T = blockDim.x;
  const int lane = int(threadIdx.x) & 31;
  uint32_t *const stk = sk_b + (int(threadIdx.x) - (P.base - 1) * T);  // row r's slot: stk[r * T]
  // the same slot as a 32-bit shared-window address (row r: sa0 + r * 4T), so
  // the loop does not re-derive the generic window base every iteration
  const uint32_t sa0 = static_cast<uint32_t>(__cvta_generic_to_shared(stk));
  const uint32_t sstride = 4u * uint32_t(T);
  auto ld_stk = [&](int r) {
    uint32_t v;
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(sa0 + uint32_t(r) * sstride) : "memory");
    return v;
  };
  auto st_stk = [&](int r, uint32_t v) {
    asm volatile("st.shared.u32 [%0], %1;" ::"r"(sa0 + uint32_t(r) * sstride), "r"(v) : "memory");
  };
  const int n = P.n, nm1 = P.n - 1;
  const uint32_t mask = P.mask;
  int row = P.base - 1;
  uint32_t cols = 0, av = 0, sol = 0;
  W d1 = 0, d2 = 0;
  uint32_t pidx = 0xffffffffu;
  unsigned long long acc = 0;
  for (;;) {
    if (row < P.base) {                                    // ^s: %done
      if (pidx != 0xffffffffu) {
        if (P.per_prefix) P.per_prefix[pidx] = sol;
        acc += pidx < P.n_double ? 2ull * sol : sol;
      }
      // the lanes refilling in this iteration take consecutive prefixes
      const unsigned act = __activemask();
      const int leader = __ffs(act) - 1;
      unsigned first = 0;
      if (lane == leader) first = atomicAdd(P.next, unsigned(__popc(act)));
      first = __shfl_sync(act, first, leader);
      pidx = first + __popc(act & ((1u << lane) - 1u));
      if (pidx >= P.n_prefix) break;
      const uint32_t pc = __ldg(P.prefix + 3 * pidx);
      const uint32_t p1 = __ldg(P.prefix + 3 * pidx + 1);
      const uint32_t p2 = __ldg(P.prefix + 3 * pidx + 2);
      // row-relative prefix diagonals -> board coordinates at row `base`
      cols = pc;
      d1 = W(p2) << P.base;                                // anti-diagonals r + c
      d2 = W(p1 & mask) << (nm1 - P.base);                 // diagonals c - r + n - 1
      av = ~(pc | p1 | p2) & mask;
      row = P.base;
      sol = 0;
    }
    if constexpr (!M) {
      // ^e: condbr %z ^pop ^push
      if (av == 0) {
        DARM_ARM("nq.pop");                                // ^pop
        const int r1 = row - 1;
        const uint32_t b1 = ld_stk(r1);
        cols ^= b1;
        d1 ^= W(b1) << r1;
        const int k1 = nm1 - r1;
        d2 ^= W(b1) << k1;
        const uint32_t a1 = ~(cols | uint32_t(d1 >> r1) | uint32_t(d2 >> k1)) & mask;
        av = a1 & (0u - (b1 << 1));                        // the free columns above b1
        row = r1;
        DARM_ARM("nq.pop.end");
      } else {
        DARM_ARM("nq.push");                               // ^push
        const uint32_t b2 = av & (0u - av);
        st_stk(row, b2);
        cols ^= b2;
        d1 ^= W(b2) << row;
        const int k2 = nm1 - row;
        d2 ^= W(b2) << k2;
        const int r2 = row + 1;
        const int k3 = (k2 - 1) & kShift;
        av = ~(cols | uint32_t(d1 >> r2) | uint32_t(d2 >> k3)) & mask;
        sol += r2 == n;
        row = r2;
        DARM_ARM("nq.push.end");
      }
    } else {
      // runDarm output: ^pop and ^push melded block-block.
      const bool z = av == 0;
      const int r1 = (z ? row : 0) - (z ? 1 : int(av));   // melded sub: row - 1 | 0 - av
      uint32_t b2 = 0;
      if (!z) b2 = av & uint32_t(r1);                      // ^pop.m.g
      const int rr = z ? r1 : row;                         // the stack row both arms touch
      const uint32_t slot = sa0 + uint32_t(rr) * sstride;
      uint32_t b1 = 0;
      // ^pop.m.g1: if (!z) slot = b2;  ^pop.m.g2: if (z) b1 = slot  (predicated)
      asm volatile(
          "{\n .reg .pred p, q;\n setp.ne.b32 p, %2, 0;\n setp.eq.b32 q, %2, 0;\n"
          " @q st.shared.u32 [%1], %3;\n @p ld.shared.u32 %0, [%1];\n}"
          : "+r"(b1)
          : "r"(slot), "r"(int(z)), "r"(b2)
          : "memory");
      const uint32_t b = z ? b1 : b2;                      // %sel3
      cols ^= b;
      d1 ^= W(b) << rr;
      const int k1 = nm1 - rr;
      d2 ^= W(b) << k1;
      int r2 = 0, k3 = 0;
      if (!z) {                                            // ^pop.m.g3
        r2 = row + 1;
        k3 = (nm1 - r2) & kShift;
      }
      const int rn = z ? r1 : r2;                          // %sel4
      const int kn = z ? k1 : k3;                          // %sel5
      const uint32_t a1 = ~(cols | uint32_t(d1 >> rn) | uint32_t(d2 >> kn)) & mask;
      if (!z) sol += r2 == n;                              // ^pop.m.g4
      uint32_t na1 = 0;
      if (z) na1 = a1 & (0u - (b1 << 1));                  // ^pop.m.g5
      av = z ? na1 : a1;                                   // %sel6
      row = rn;
    }
  }
  // every lane has left the loop: reduce the warp's solution counts
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if (lane == 0 && acc) atomicAdd(P.total, acc);
}

// ------------------------------------------------------------------ the paper's shape
// ir/nqueens_step.ir: one iteration = pop / count a leaf / push — the
// "if-then-elseif-then" section of the paper's NQU loop,
// which runDarm melds by region replication: two block-region melds (^pop and
// ^leaf into the ^push region; MP 0.283 and 0.335, 12 selects, 7 unpredicated
// runs).  The diagonals are row-relative (shifted every row, as enumerated on
// the host) and the stack keeps the whole row state (cols, d1, d2, av) at
// [array][row - base + 1][thread].  32-bit words: n <= 16.  Kept beside the
// symmetric encoding above so the two can be compared on the same search: this
// is the shape the paper names (melded: 0.83x of unmelded on the B200), the
// symmetric one the shape where melding pays.
template <bool M>
__global__ void __launch_bounds__(256) nqueens_step_kernel(NqParams P) {
  extern __shared__ uint32_t sk[];
  const int T = blockDim.x;
  const int L = P.levels;
  const int lane = int(threadIdx.x) & 31;
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
        acc += pidx < P.n_double ? 2ull * sol : sol;
      }
      // the lanes refilling in this iteration take consecutive prefixes
      const unsigned act = __activemask();
      const int leader = __ffs(act) - 1;
      unsigned first = 0;
      if (lane == leader) first = atomicAdd(P.next, unsigned(__popc(act)));
      first = __shfl_sync(act, first, leader);
      pidx = first + __popc(act & ((1u << lane) - 1u));
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
        DARM_ARM("nqs.pop");                               // ^pop
        const int r1 = row - 1;
        const int ix1 = r1 * T + lane_off;
        cols = sk_cols[ix1];
        d1 = sk_d1[ix1];
        d2 = sk_d2[ix1];
        av = sk_av[ix1];
        row = r1;
        DARM_ARM("nqs.pop.end");
      } else if (row == n1) {
        DARM_ARM("nqs.leaf");                              // ^leaf
        const uint32_t b1 = av & (0u - av);
        av = av ^ b1;
        sol += 1;
        DARM_ARM("nqs.leaf.end");
      } else {
        DARM_ARM("nqs.push");                              // ^push
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
        DARM_ARM("nqs.push.end");
      }
    } else {
      // runDarm output: block-region melds of ^pop and ^leaf into the ^push
      // region.  The replicated region's guarded runs (^push.r.m.g*) are
      // issued as predicated code, not as branches around each run: the
      // arithmetic of every run is computed by every lane and selected, the
      // push's four stack stores are predicated stores, the pop's four stack
      // loads read the melded slot (a valid stack row for every lane).
      const bool z = av == 0;
      const bool last = row == n1;
      const bool sel = z ? false : last;                   // the ^leaf lanes
      const bool push = !z && !sel;                        // the ^push lanes
      const int r1 = (z ? row : 0) - (z ? 1 : int(av));    // melded sub: row-1 | 0-av
      const uint32_t b2 = push ? (av & uint32_t(r1)) : 0u; // ^push.r.m.g
      const uint32_t rem2 = av ^ b2;
      const int sel3 = z ? r1 : row;                       // stack row: pop row-1 | push row
      const int ix1 = sel3 * T + lane_off;
      // ^push.r.m.g1.r.m.g: the push's stores (predicated)
      asm volatile(
          "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
          " @p st.shared.u32 [%0], %5;\n @p st.shared.u32 [%1], %6;\n"
          " @p st.shared.u32 [%2], %7;\n @p st.shared.u32 [%3], %8;\n}"
          ::"r"(smem_u32(sk_av + ix1)), "r"(smem_u32(sk_cols + ix1)), "r"(smem_u32(sk_d1 + ix1)),
          "r"(smem_u32(sk_d2 + ix1)), "r"(int(push)), "r"(rem2),
          "r"(cols), "r"(d1), "r"(d2)
          : "memory");
      const uint32_t c2 = cols | b2;
      const uint32_t f1 = (d1 | b2) << 1;
      const uint32_t f2 = (d2 | b2) >> 1;
      const uint32_t u3 = ~(c2 | f1 | f2);
      const uint32_t ng1 = 0u - av;                        // ^push.r.m.g1.r.m.g1
      const uint32_t b1 = (sel ? av : u3) & (sel ? ng1 : P.mask);   // melded and: bit | new av
      // ^push.r.m.g2: the pop's loads (the melded slot, read by every lane)
      const uint32_t pc = sk_cols[ix1], pd1 = sk_d1[ix1], pd2 = sk_d2[ix1], pav = sk_av[ix1];
      sol += sel ? 1u : 0u;                                // ^push.r.m.g1.r.m.g2
      cols = z ? pc : (sel ? cols : c2);
      d1 = z ? pd1 : (sel ? d1 : f1);
      d2 = z ? pd2 : (sel ? d2 : f2);
      av = z ? pav : (sel ? (av ^ b1) : b1);
      row = z ? r1 : (sel ? row : row + 1);                // ^push.r.m.g3
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if (lane == 0 && acc) atomicAdd(P.total, acc);
}

namespace {
template <bool M, typename W>
cudaError_t launch_form(const NqParams &P, int sms, cudaStream_t s) {
  const int T = 256;
  const size_t shm = size_t(P.levels) * T * sizeof(uint32_t);
  auto kern = nqueens_kernel<M, W>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(shm));
  if (e != cudaSuccess) return e;
  int per_sm = 0;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, T, shm);
  if (e != cudaSuccess) return e;
  if (per_sm < 1) return cudaErrorInvalidConfiguration;
  uint64_t grid = uint64_t(sms) * per_sm;
  const uint64_t need = (uint64_t(P.n_prefix) + T - 1) / T;
  if (grid > need) grid = need;
  if (grid < 1) grid = 1;
  kern<<<unsigned(grid), T, shm, s>>>(P);
  return cudaGetLastError();
}
}  // namespace

namespace {
template <bool M>
cudaError_t launch_step_form(const NqParams &P, int sms, cudaStream_t s) {
  const int T = 256;
  const size_t shm = size_t(4) * P.levels * T * sizeof(uint32_t);
  auto kern = nqueens_step_kernel<M>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(shm));
  if (e != cudaSuccess) return e;
  int per_sm = 0;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, T, shm);
  if (e != cudaSuccess) return e;
  if (per_sm < 1) return cudaErrorInvalidConfiguration;
  uint64_t grid = uint64_t(sms) * per_sm;
  const uint64_t need = (uint64_t(P.n_prefix) + T - 1) / T;
  if (grid > need) grid = need;
  if (grid < 1) grid = 1;
  kern<<<unsigned(grid), T, shm, s>>>(P);
  return cudaGetLastError();
}
}  // namespace

cudaError_t launch_nqueens(int variant, const uint32_t *prefix, uint32_t n_prefix, uint32_t n_double, int n, int base,
                           uint32_t *per_prefix, unsigned long long *total, unsigned int *counter,
                           int sms, cudaStream_t s, bool paper_shape) {
  NqParams P;
  P.prefix = prefix;
  P.n_prefix = n_prefix;
  P.n_double = n_double;
  P.per_prefix = per_prefix;
  P.total = total;
  P.next = counter;
  P.n = n;
  P.base = base;
  P.levels = n - base + 1;
  P.mask = n >= 32 ? 0xffffffffu : ((1u << n) - 1u);
  if (paper_shape) return variant ? launch_step_form<true>(P, sms, s) : launch_step_form<false>(P, sms, s);
  if (n <= 16)
    return variant ? launch_form<true, uint32_t>(P, sms, s) : launch_form<false, uint32_t>(P, sms, s);
  return variant ? launch_form<true, uint64_t>(P, sms, s) : launch_form<false, uint64_t>(P, sms, s);
}

}  // namespace darm_gpu
