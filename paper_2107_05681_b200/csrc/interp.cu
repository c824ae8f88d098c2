// interp.cu — a GPU executeWarp for arbitrary mini-IR.
//
// The reference runs one warp of an IR function at a time on the CPU
// (executeWarp, proj/src/interp.cpp:332-381: lockstep lanes, the IPDOM
// reconvergence of execPath :254-314, per-lane fault capture, undef taint,
// issue statistics).  Here one CUDA warp runs one IR warp and a batch of IR
// warps runs as one launch; IR lane l lives on thread l % 32 of the warp (a
// 64-lane IR warp puts two lanes on every thread).  The semantics follow
// interp.cpp instruction for instruction so that returns, final memories,
// fault counts, the taint / non-termination flags and every WarpExecStats
// counter equal the reference's:
//   * active masks are 64-bit; a branch condition becomes a mask with two
//     __ballot_sync (lanes 0-31, 32-63);
//   * execPath's recursion is an explicit stack of (block, mask, stop)
//     frames: a divergent condbr leaves its frame parked at the immediate
//     post-dominator and pushes the false then the true path, so the true
//     path runs first (interp.cpp:301-306);
//   * a store instruction applies its lanes in ascending lane order: lanes
//     storing to the same cell are grouped with __match_any_sync and only the
//     highest lane of a group writes (lanes 32-63 after lanes 0-31);
//   * registers (value + taint) are per-lane local arrays; memories are the
//     warp's slice of the caller's global / shared buffers plus a taint byte
//     per cell;
//   * the counters are warp-uniform and computed redundantly by every thread.
// The programs come from ir_program.cu; the control flow of the interpreter is
// uniform across the warp by construction (every branch depends on masks).
#include <cstdint>

#include "ir_program.h"
#include "kernels.h"

namespace darm_gpu {

constexpr int kMaxRegs = 256;      // values per function (registers per lane)
constexpr int kMaxPhis = 16;       // phis per block
constexpr int kMaxDepth = 48;      // SIMT stack frames
constexpr int kWarpsPerCta = 4;

struct InterpArgs {
  const IrBlock *blocks;
  const IrInst *insts;
  const IrPhi *phis;
  const IrPhiIn *phi_ins;
  const int64_t *mem_off;      // per memory: word offset in its class
  const int64_t *mem_size;
  const uint8_t *mem_shared;
  int64_t latency[kNumOps];
  int n_params, n_regs, entry, ret_block;
  int64_t gwords, swords;
  int W;
  int64_t n_warps;
  int am;                      // args: 0 broadcast, 1 per warp, 2 per lane
  const int32_t *args;         // n_params x acount
  int64_t acount;
  int32_t *globals;            // n_warps x gwords
  int32_t *shared;             // n_warps x swords
  uint8_t *taint;              // n_warps x (gwords + swords)
  int32_t *returns;            // n_warps x W (may be null)
  uint8_t *ret_valid;          // n_warps x W (may be null)
  int32_t *faults;             // n_warps (may be null)
  int64_t *stats;              // n_warps x 8 (may be null)
  int32_t *errors;             // n_warps
  int64_t max_steps;
};

// stats slots
enum { kIssued, kThread, kUseful, kSerialized, kDivergent, kSharedIss, kGlobalIss, kFlags };
// error codes (reference runtime_error cases)
enum { kErrNone = 0, kErrPhi = 1, kErrReconv = 2, kErrDepth = 3 };

struct Frame {
  int block, stop;
  uint64_t mask;
};

__device__ __forceinline__ uint64_t ballot64(bool a, bool b) {
  return uint64_t(__ballot_sync(0xffffffffu, a)) | (uint64_t(__ballot_sync(0xffffffffu, b)) << 32);
}

__global__ void __launch_bounds__(32 * kWarpsPerCta) ir_interp_kernel(InterpArgs A) {
  const int t = threadIdx.x & 31;
  const int W = A.W;
  const uint64_t all = W == 64 ? ~uint64_t(0) : ((uint64_t(1) << W) - 1);
  int32_t rv[2][kMaxRegs];
  uint8_t rt[2][kMaxRegs];
  Frame stk[kMaxDepth];
  const int64_t warps = int64_t(gridDim.x) * kWarpsPerCta;
  for (int64_t w = int64_t(blockIdx.x) * kWarpsPerCta + (threadIdx.x >> 5); w < A.n_warps; w += warps) {
    int32_t *G = A.globals + w * A.gwords;
    int32_t *S = A.shared + w * A.swords;
    uint8_t *TG = A.taint + w * (A.gwords + A.swords);
    uint8_t *TS = TG + A.gwords;
    // registers: an unassigned value evaluates to {0, taint} (interp.cpp:83-85)
    int prev[2] = {-1, -1};
    int32_t retv[2] = {0, 0};
    bool retok[2] = {false, false};
    for (int s = 0; s < 2; ++s)
      for (int r = 0; r < A.n_regs; ++r) {
        rv[s][r] = 0;
        rt[s][r] = 1;
      }
    for (int s = 0; s < 2; ++s) {
      const int lane = t + 32 * s;
      if (lane >= W) continue;
      for (int p = 0; p < A.n_params; ++p) {
        const int64_t ai = A.am == 0 ? 0 : (A.am == 1 ? w : w * W + lane);
        rv[s][p] = A.args[int64_t(p) * A.acount + ai];
        rt[s][p] = 0;
      }
    }
    uint64_t dead = 0, finished = 0;
    int64_t st[7] = {0, 0, 0, 0, 0, 0, 0};
    int64_t steps = A.max_steps;
    bool nonterm = false, tainted = false;
    int err = kErrNone;
    int32_t nfaults = 0;

    auto issue = [&](int op, uint64_t active) {
      const int64_t lat = A.latency[op];
      st[kIssued] += 1;
      st[kThread] += lat * W;
      st[kUseful] += lat * __popcll(active);
      if (op == kLoadShared || op == kStoreShared) st[kSharedIss] += 1;
      if (op == kLoadGlobal || op == kStoreGlobal) st[kGlobalIss] += 1;
      if (--steps < 0) nonterm = true;
    };
    auto eval = [&](int s, const IrOperand &o, int32_t &v, bool &ta) {
      if (o.kind == kOpndReg) {
        v = rv[s][o.v];
        ta = rt[s][o.v];
      } else if (o.kind == kOpndImm) {
        v = o.v;
        ta = false;
      } else {   // undef
        v = 0;
        ta = true;
      }
    };

    for (int phase = 0; phase < 2 && !nonterm && err == kErrNone; ++phase) {
      // execPath(entry, all, ret), then the ret block itself (interp.cpp:356-360)
      if (phase == 1 && (all & ~dead & ~finished) == 0) break;
      int sp = 1;
      stk[0].block = phase == 0 ? A.entry : A.ret_block;
      stk[0].stop = phase == 0 ? A.ret_block : -1;
      stk[0].mask = all;
      while (sp > 0 && !nonterm && err == kErrNone) {
        Frame &F = stk[sp - 1];
        if (F.block == F.stop) {
          --sp;
          continue;
        }
        uint64_t active = F.mask & ~dead & ~finished;
        if (!active) {
          --sp;
          continue;
        }
        const IrBlock B = A.blocks[F.block];
        // ---- phis: parallel copy by each lane's predecessor (interp.cpp:221-245)
        if (B.n_phi) {
          int32_t sv[2][kMaxPhis];
          uint8_t sa[2][kMaxPhis];
          bool missing = false;
          for (int p = 0; p < B.n_phi; ++p) {
            const IrPhi ph = A.phis[B.first_phi + p];
            for (int s = 0; s < 2; ++s) {
              const int lane = t + 32 * s;
              if (lane >= W || !(active >> lane & 1)) continue;
              int found = -1;
              for (int q = 0; q < ph.count; ++q)
                if (A.phi_ins[ph.first + q].pred == prev[s]) found = q;
              if (found < 0) {
                missing = true;
                continue;
              }
              int32_t v;
              bool ta;
              eval(s, A.phi_ins[ph.first + found].val, v, ta);
              sv[s][p] = v;
              sa[s][p] = ta;
            }
          }
          if (__any_sync(0xffffffffu, missing)) {
            err = kErrPhi;
            break;
          }
          for (int p = 0; p < B.n_phi; ++p) {
            issue(kPhi, active);
            if (nonterm) break;
            const int d = A.phis[B.first_phi + p].dst;
            for (int s = 0; s < 2; ++s) {
              const int lane = t + 32 * s;
              if (lane < W && (active >> lane & 1)) {
                rv[s][d] = sv[s][p];
                rt[s][d] = sa[s][p];
              }
            }
          }
          if (nonterm) break;
        }
        // ---- body (interp.cpp:102-219)
        bool left = false;
        for (int k = 0; k < B.n_inst; ++k) {
          const IrInst I = A.insts[B.first_inst + k];
          issue(I.op, active);
          if (nonterm) break;
          bool fl[2] = {false, false}, th[2] = {false, false};
          if (I.op == kStoreShared || I.op == kStoreGlobal) {
            const bool sh = I.op == kStoreShared;
            const int64_t size = A.mem_size[I.mem], off = A.mem_off[I.mem];
            for (int s = 0; s < 2; ++s) {
              const int lane = t + 32 * s;
              bool doit = false;
              int32_t idx = 0, val = 0;
              bool vt = false;
              if (lane < W && (active >> lane & 1)) {
                bool it;
                eval(s, I.a[0], idx, it);
                eval(s, I.a[1], val, vt);
                th[s] = it || vt;
                if (!it) {
                  if (idx < 0 || int64_t(idx) >= size)
                    fl[s] = true;
                  else
                    doit = true;
                }
              }
              // lanes of this half storing to the same cell: the highest writes
              const unsigned long long key =
                  doit ? (uint64_t(I.mem) << 32 | uint32_t(idx)) : (0xffffffff00000000ull | uint64_t(t));
              const unsigned peers = __match_any_sync(0xffffffffu, key);
              if (doit && 31 - __clz(peers) == t) {
                (sh ? S : G)[off + idx] = val;
                (sh ? TS : TG)[off + idx] = vt;
              }
              __syncwarp();
            }
          } else {
            for (int s = 0; s < 2; ++s) {
              const int lane = t + 32 * s;
              if (lane >= W || !(active >> lane & 1)) continue;
              int32_t x = 0, y = 0, r = 0;
              bool xt = false, yt = false, rtt = false;
              switch (I.op) {
                case kAdd: case kSub: case kMul: case kAnd: case kOr: case kXor: case kShl: case kShr: {
                  eval(s, I.a[0], x, xt);
                  eval(s, I.a[1], y, yt);
                  const uint32_t ux = uint32_t(x), uy = uint32_t(y);
                  uint32_t uv = 0;
                  switch (I.op) {
                    case kAdd: uv = ux + uy; break;
                    case kSub: uv = ux - uy; break;
                    case kMul: uv = ux * uy; break;
                    case kAnd: uv = ux & uy; break;
                    case kOr: uv = ux | uy; break;
                    case kXor: uv = ux ^ uy; break;
                    case kShl: uv = ux << (uy & 31u); break;
                    default: uv = ux >> (uy & 31u); break;
                  }
                  r = int32_t(uv);
                  rtt = xt || yt;
                  break;
                }
                case kDiv: case kRem: {
                  eval(s, I.a[0], x, xt);
                  eval(s, I.a[1], y, yt);
                  if (y == 0) {
                    fl[s] = true;
                    continue;
                  }
                  const int64_t q = I.op == kDiv ? int64_t(x) / y : int64_t(x) % y;
                  r = int32_t(q);
                  rtt = xt || yt;
                  break;
                }
                case kIcmpEq: case kIcmpNe: case kIcmpLt: case kIcmpGt: case kIcmpLe: case kIcmpGe: {
                  eval(s, I.a[0], x, xt);
                  eval(s, I.a[1], y, yt);
                  bool c;
                  switch (I.op) {
                    case kIcmpEq: c = x == y; break;
                    case kIcmpNe: c = x != y; break;
                    case kIcmpLt: c = x < y; break;
                    case kIcmpGt: c = x > y; break;
                    case kIcmpLe: c = x <= y; break;
                    default: c = x >= y; break;
                  }
                  r = c ? 1 : 0;
                  rtt = xt || yt;
                  break;
                }
                case kSelect: {
                  int32_t c;
                  bool ct;
                  eval(s, I.a[0], c, ct);
                  eval(s, c != 0 ? I.a[1] : I.a[2], r, rtt);   // only the chosen side's taint
                  rtt = rtt || ct;
                  break;
                }
                case kLoadShared: case kLoadGlobal: {
                  const bool sh = I.op == kLoadShared;
                  eval(s, I.a[0], x, xt);
                  if (xt) {
                    r = 0;
                    rtt = true;
                    break;
                  }
                  if (x < 0 || int64_t(x) >= A.mem_size[I.mem]) {
                    fl[s] = true;
                    continue;
                  }
                  const int64_t a = A.mem_off[I.mem] + x;
                  r = (sh ? S : G)[a];
                  rtt = (sh ? TS : TG)[a];
                  break;
                }
                case kTid:
                  r = lane;
                  rtt = false;
                  break;
                case kConst:
                  eval(s, I.a[0], r, rtt);
                  break;
                default:   // barrier: a whole-warp no-op in lockstep execution
                  continue;
              }
              if (I.dst >= 0) {
                rv[s][I.dst] = r;
                rt[s][I.dst] = rtt;
              }
            }
          }
          const uint64_t f = ballot64(fl[0], fl[1]);
          if (f) {
            dead |= f;
            nfaults += __popcll(f);
          }
          if (__any_sync(0xffffffffu, th[0] || th[1])) tainted = true;
          active = F.mask & ~dead & ~finished;
          if (!active) {
            left = true;
            break;
          }
        }
        if (nonterm) break;
        if (left) {
          --sp;
          continue;
        }
        // ---- terminator (interp.cpp:266-312)
        issue(B.term, active);
        if (nonterm) break;
        if (B.term == kBr) {
          for (int s = 0; s < 2; ++s)
            if (t + 32 * s < W && (active >> (t + 32 * s) & 1)) prev[s] = F.block;
          F.block = B.succ[0];
        } else if (B.term == kRet) {
          bool th = false;
          for (int s = 0; s < 2; ++s) {
            const int lane = t + 32 * s;
            if (lane >= W || !(active >> lane & 1) || B.cond.kind == kOpndNone) continue;
            int32_t v;
            bool ta;
            eval(s, B.cond, v, ta);
            th = th || ta;
            retv[s] = v;
            retok[s] = true;
          }
          if (__any_sync(0xffffffffu, th)) tainted = true;
          finished |= active;
          --sp;
        } else {   // condbr
          bool c[2] = {false, false}, th = false;
          for (int s = 0; s < 2; ++s) {
            const int lane = t + 32 * s;
            if (lane >= W || !(active >> lane & 1)) continue;
            int32_t v;
            bool ta;
            eval(s, B.cond, v, ta);
            th = th || ta;
            c[s] = v != 0;
          }
          if (__any_sync(0xffffffffu, th)) tainted = true;
          const uint64_t t1 = ballot64(c[0], c[1]) & active, f1 = active & ~t1;
          for (int s = 0; s < 2; ++s)
            if (t + 32 * s < W && (active >> (t + 32 * s) & 1)) prev[s] = F.block;
          if (!f1) {
            F.block = B.succ[0];
          } else if (!t1) {
            F.block = B.succ[1];
          } else {
            st[kDivergent] += 1;
            if (B.ipdom < 0) {
              err = kErrReconv;
              break;
            }
            if (sp + 2 > kMaxDepth) {
              err = kErrDepth;
              break;
            }
            const int reconv = B.ipdom;
            F.block = reconv;
            stk[sp] = Frame{B.succ[1], reconv, f1};
            stk[sp + 1] = Frame{B.succ[0], reconv, t1};
            sp += 2;
          }
        }
      }
    }
    // ---- results
    for (int s = 0; s < 2; ++s) {
      const int lane = t + 32 * s;
      if (lane >= W) continue;
      if (A.returns) A.returns[w * W + lane] = retok[s] ? retv[s] : 0;
      if (A.ret_valid) A.ret_valid[w * W + lane] = retok[s];
    }
    if (t == 0) {
      if (A.faults) A.faults[w] = nfaults;
      A.errors[w] = err;
      if (A.stats) {
        int64_t *o = A.stats + w * 8;
        for (int k = 0; k < 7; ++k) o[k] = st[k];
        o[kSerialized] = st[kThread] - st[kUseful];
        o[kFlags] = (nonterm ? 1 : 0) | (tainted ? 2 : 0);
      }
    }
    __syncwarp();
  }
}

cudaError_t launch_ir_interp(const InterpLaunch &L, cudaStream_t s) {
  InterpArgs A;
  A.blocks = static_cast<const IrBlock *>(L.blocks);
  A.insts = static_cast<const IrInst *>(L.insts);
  A.phis = static_cast<const IrPhi *>(L.phis);
  A.phi_ins = static_cast<const IrPhiIn *>(L.phi_ins);
  A.mem_off = L.mem_off;
  A.mem_size = L.mem_size;
  A.mem_shared = L.mem_shared;
  for (int k = 0; k < kNumOps; ++k) A.latency[k] = L.latency[k];
  A.n_params = L.n_params;
  A.n_regs = L.n_regs;
  A.entry = L.entry;
  A.ret_block = L.ret_block;
  A.gwords = L.gwords;
  A.swords = L.swords;
  A.W = L.W;
  A.n_warps = L.n_warps;
  A.am = L.am;
  A.args = L.args;
  A.acount = L.acount;
  A.globals = L.globals;
  A.shared = L.shared;
  A.taint = L.taint;
  A.returns = L.returns;
  A.ret_valid = L.ret_valid;
  A.faults = L.faults;
  A.stats = L.stats;
  A.errors = L.errors;
  A.max_steps = L.max_steps;
  if (L.n_warps == 0) return cudaSuccess;
  int64_t grid = (L.n_warps + kWarpsPerCta - 1) / kWarpsPerCta;
  const int64_t cap = int64_t(L.sms) * 16;
  if (grid > cap) grid = cap;
  ir_interp_kernel<<<unsigned(grid), 32 * kWarpsPerCta, 0, s>>>(A);
  return cudaGetLastError();
}

int ir_interp_max_regs() { return kMaxRegs; }
int ir_interp_max_phis() { return kMaxPhis; }

}  // namespace darm_gpu
