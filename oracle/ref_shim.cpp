// ref_shim.cpp — C-ABI over the UNMODIFIED reference library (TEST INFRASTRUCTURE).
//
// Compiled together with /root/reference/proj/src/*.cpp into oracle/_ref/libdarm_ref.so
// by oracle/Makefile.  Only tests/, __graft_entry__.smoke() and bench.py's CPU legs
// load it; the product (paper_2107_05681_b200/) never does.
//
// Every entry point is a thin batching loop around the reference's own API:
//   parseModule            parser.hpp:25-30        (parser.cpp:465)
//   runDarm                melding.hpp:162         (melding_driver.cpp:54-100)
//   makeRandomInput        fixtures.hpp:28-29      (fixtures.cpp:82-108)
//   executeWarp            interp.hpp:57-58        (interp.cpp:332-381)
//   compareRuns            interp.hpp:67           (interp.cpp:383-426)
//   statsToJson/reportJson fixtures.cpp:51-60, darm_cli.cpp:53-68
// The worker pool mirrors cmdBench (darm_cli.cpp:295-318): an atomic job index
// shared by T std::threads.
#include <array>
#include <atomic>
#include <cstdint>
#include <cstring>
#include <exception>
#include <string>
#include <thread>
#include <vector>

#include "darm/fixtures.hpp"
#include "darm/interp.hpp"
#include "darm/melding.hpp"
#include "darm/parser.hpp"
#include "darm/verifier.hpp"

using namespace darm;

struct ref_module {
  Module m;
  MeldReport report;
  bool melded = false;
};

namespace {

int fail(char *err, size_t errlen, const std::string &msg, int code) {
  if (err && errlen) {
    std::strncpy(err, msg.c_str(), errlen - 1);
    err[errlen - 1] = 0;
  }
  return code;
}

size_t putText(const std::string &s, char *out, size_t outlen) {
  if (out && outlen) {
    size_t n = std::min(outlen - 1, s.size());
    std::memcpy(out, s.data(), n);
    out[n] = 0;
  }
  return s.size() + 1;
}

LatencyModel pickLatency(int unit) {
  LatencyModel lm = LatencyModel::defaults();
  if (unit) {
    // Every opcode at latency 1 => utilization == SIMT lane efficiency
    // (the survey's "unit-latency" model; same effect as a fromFile with all 1s).
    for (int op = int(Opcode::Add); op <= int(Opcode::Barrier); ++op)
      lm.set(Opcode(op), 1);
  }
  return lm;
}

template <class F>
void parallelFor(int64_t n, int threads, F &&body) {
  std::atomic<int64_t> next{0};
  auto work = [&] {
    for (;;) {
      int64_t i = next.fetch_add(1);
      if (i >= n) return;
      body(i);
    }
  };
  if (threads < 1) threads = 1;
  if (threads > n) threads = int(std::max<int64_t>(1, n));
  std::vector<std::thread> pool;
  for (int i = 1; i < threads; ++i) pool.emplace_back(work);
  work();
  for (auto &t : pool) t.join();
}

}  // namespace

extern "C" {

// meld: 0 = original, 1 = DARM (runDarm), 2 = branch fusion only.
int ref_load(const char *ir_text, int meld, double threshold, ref_module **out,
             char *err, size_t errlen) {
  try {
    auto *h = new ref_module;
    h->m = parseModule(ir_text);
    auto viol = verifyModule(h->m);
    if (!viol.empty()) {
      std::string msg = "^" + viol.front().block + ": " + viol.front().message;
      delete h;
      return fail(err, errlen, msg, 2);
    }
    if (meld) {
      MeldConfig cfg;
      cfg.threshold = threshold;
      cfg.branchFusionOnly = meld == 2;
      h->report = runDarm(h->m.functions.front(), cfg, LatencyModel::defaults());
      h->melded = true;
    }
    *out = h;
    return 0;
  } catch (const std::logic_error &e) {
    return fail(err, errlen, e.what(), 3);
  } catch (const std::exception &e) {
    return fail(err, errlen, e.what(), 2);
  }
}

void ref_free(ref_module *h) { delete h; }

// Corpus kernels embedded at build time (oracle/embed_corpus.py), so the
// library works where /root/reference is absent (the GPU box).
extern const char *const ref_corpus_names[];
extern const char *const ref_corpus_texts[];

int ref_load_corpus(const char *name, int meld, double threshold, ref_module **out,
                    char *err, size_t errlen) {
  for (int i = 0; ref_corpus_names[i]; ++i)
    if (std::strcmp(ref_corpus_names[i], name) == 0)
      return ref_load(ref_corpus_texts[i], meld, threshold, out, err, errlen);
  return fail(err, errlen, std::string("no corpus kernel '") + name + "'", 2);
}

const char *ref_corpus_text(const char *name) {
  for (int i = 0; ref_corpus_names[i]; ++i)
    if (std::strcmp(ref_corpus_names[i], name) == 0) return ref_corpus_texts[i];
  return nullptr;
}

size_t ref_print(const ref_module *h, char *out, size_t outlen) {
  return putText(printModule(h->m), out, outlen);
}

// {"params":[..],"globals":[[name,size],..],"shared":[[name,size],..],"melds":[..]}
size_t ref_layout(const ref_module *h, char *out, size_t outlen) {
  const Function &f = h->m.functions.front();
  nlohmann::json j;
  j["function"] = f.name;
  j["params"] = f.params;
  j["globals"] = nlohmann::json::array();
  for (const auto &g : h->m.globals) j["globals"].push_back({g.name, g.size});
  j["shared"] = nlohmann::json::array();
  for (const auto &s : f.sharedDecls) j["shared"].push_back({s.name, s.size});
  j["melds"] = nlohmann::json::array();
  for (const auto &a : h->report.melds)
    j["melds"].push_back({{"regionEntry", a.regionEntry},
                          {"regionExit", a.regionExit},
                          {"kind", a.kind},
                          {"mpScore", a.mpScore},
                          {"selectsInserted", a.selectsInserted},
                          {"unpredicatedRuns", a.unpredicatedRuns}});
  return putText(j.dump(), out, outlen);
}

// makeRandomInput (fixtures.cpp:82-108) flattened: args[n_params],
// globals = declared-size arrays in declaration order, shared likewise.
int ref_make_random_input(const ref_module *h, int warp, uint64_t seed,
                          int32_t *args, int32_t *globals, int32_t *shared) {
  const Function &f = h->m.functions.front();
  WarpInput in = makeRandomInput(h->m, f, warp, seed);
  for (size_t p = 0; p < in.args.size(); ++p) args[p] = in.args[p][0];
  size_t off = 0;
  for (const auto &g : h->m.globals) {
    const auto &v = in.globalInit.at(g.name);
    std::memcpy(globals + off, v.data(), v.size() * 4);
    off += size_t(g.size);
  }
  off = 0;
  for (const auto &s : f.sharedDecls) {
    const auto &v = in.sharedInit.at(s.name);
    std::memcpy(shared + off, v.data(), v.size() * 4);
    off += size_t(s.size);
  }
  return 0;
}

// Batched executeWarp over n_warps independent warp slices.
//   args:    n_params x acount int32, acount in {1, n_warps, n_warps*warp}
//   globals: per declared global (in order) n_warps x gstride words; slice w
//            initialises words [0,gstride) of that warp's array (rest 0) and
//            receives words [0,gstride) of globalFinal back.
//   shared:  per shared decl n_warps x declared-size words (may be NULL => 0).
//   returns/has_ret: n_warps*warp (may be NULL); faults: n_warps (may be NULL)
//   stats:   n_warps x 8 int64 {issued, threadCycles, useful, serialized,
//            divergentBranches, sharedIssues, globalIssues, flags}
//            flags bit0 = nonTerminated, bit1 = taintedObservable (may be NULL)
int ref_execute_warps(const ref_module *h, int warp, int64_t n_warps,
                      const int32_t *args, int64_t acount, int32_t *globals,
                      int64_t gstride, const int32_t *shared, int unit_latency,
                      int64_t max_steps, int threads, int32_t *returns,
                      uint8_t *has_ret, int32_t *faults, int64_t *stats,
                      char *err, size_t errlen) {
  const Function &f = h->m.functions.front();
  const size_t np = f.params.size();
  if (acount != 1 && acount != n_warps && acount != n_warps * warp)
    return fail(err, errlen, "bad argument count", 2);
  LatencyModel lm = pickLatency(unit_latency);
  std::vector<std::string> errors(1);
  std::atomic<bool> bad{false};
  int64_t sharedWords = 0;
  for (const auto &s : f.sharedDecls) sharedWords += s.size;
  parallelFor(n_warps, threads, [&](int64_t w) {
    if (bad.load()) return;
    try {
      WarpInput in;
      in.warpSize = warp;
      for (size_t p = 0; p < np; ++p) {
        const int32_t *a = args + p * acount;
        if (acount == 1)
          in.args.push_back({a[0]});
        else if (acount == n_warps)
          in.args.push_back({a[w]});
        else
          in.args.push_back(std::vector<int32_t>(a + w * warp, a + (w + 1) * warp));
      }
      size_t goff = 0;
      for (const auto &g : h->m.globals) {
        const int32_t *src = globals + goff + size_t(w) * gstride;
        in.globalInit[g.name] = std::vector<int32_t>(src, src + gstride);
        goff += size_t(n_warps) * gstride;
      }
      if (shared) {
        size_t soff = 0;
        for (const auto &s : f.sharedDecls) {
          const int32_t *src = shared + soff + size_t(w) * s.size;
          in.sharedInit[s.name] = std::vector<int32_t>(src, src + s.size);
          soff += size_t(n_warps) * s.size;
        }
      }
      WarpResult r = executeWarp(h->m, f, in, lm, max_steps);
      goff = 0;
      for (const auto &g : h->m.globals) {
        const auto &v = r.globalFinal.at(g.name);
        std::memcpy(globals + goff + size_t(w) * gstride, v.data(), gstride * 4);
        goff += size_t(n_warps) * gstride;
      }
      if (returns)
        for (int l = 0; l < warp; ++l) {
          returns[w * warp + l] = r.returns[l].value_or(0);
          if (has_ret) has_ret[w * warp + l] = r.returns[l].has_value();
        }
      if (faults) faults[w] = int32_t(r.faults.size());
      if (stats) {
        int64_t *s = stats + w * 8;
        s[0] = r.stats.issuedInstructions;
        s[1] = r.stats.threadCycles;
        s[2] = r.stats.usefulThreadCycles;
        s[3] = r.stats.serializedCycles;
        s[4] = r.stats.divergentBranchCount;
        s[5] = r.stats.sharedMemIssues;
        s[6] = r.stats.globalMemIssues;
        s[7] = (r.nonTerminated ? 1 : 0) | (r.taintedObservable ? 2 : 0);
      }
    } catch (const std::exception &e) {
      if (!bad.exchange(true)) errors[0] = e.what();
    }
  });
  (void)sharedWords;
  if (bad) return fail(err, errlen, errors[0], 2);
  return 0;
}

// The reference's own compareRuns (interp.cpp:383-426) applied slice by slice to
// two batched results in the ref_execute_warps layout.  Returns the first
// differing warp index, or -1 when every slice compares equal; diff gets the
// reference's message.
int64_t ref_compare_warps(const ref_module *h, int warp, int64_t n_warps,
                          int64_t gstride, const int32_t *globals_a,
                          const int32_t *returns_a, const uint8_t *has_a,
                          const int32_t *faults_a, const int32_t *globals_b,
                          const int32_t *returns_b, const uint8_t *has_b,
                          const int32_t *faults_b, char *diff, size_t difflen) {
  auto build = [&](int64_t w, const int32_t *g, const int32_t *r,
                   const uint8_t *hr, const int32_t *fc) {
    WarpResult res;
    res.returns.assign(size_t(warp), std::nullopt);
    if (r)
      for (int l = 0; l < warp; ++l)
        if (!hr || hr[w * warp + l]) res.returns[size_t(l)] = r[w * warp + l];
    size_t goff = 0;
    for (const auto &gd : h->m.globals) {
      const int32_t *src = g + goff + size_t(w) * gstride;
      res.globalFinal[gd.name] = std::vector<int32_t>(src, src + gstride);
      goff += size_t(n_warps) * gstride;
    }
    if (fc) res.faults.resize(size_t(fc[w]));
    return res;
  };
  for (int64_t w = 0; w < n_warps; ++w) {
    CompareVerdict v = compareRuns(build(w, globals_a, returns_a, has_a, faults_a),
                                   build(w, globals_b, returns_b, has_b, faults_b));
    if (!v.equal) {
      putText(v.diff, diff, difflen);
      return w;
    }
  }
  return -1;
}

// Chains executeWarp over one warp until a step changes neither global nor
// shared memory (a fixpoint), feeding globalFinal/sharedFinal of each step into
// the next — the loop a per-iteration step kernel such as
// paper_2107_05681_b200/ir/nqueens_sym.ir stands for.  globals/shared are the
// declared-size arrays in declaration order (in/out).  stats_sum (7 counters)
// accumulates every step that changed state; *rounds receives their number.
int ref_run_to_fixpoint(const ref_module *h, int warp, const int32_t *args, int32_t *globals,
                        int32_t *shared, int64_t max_rounds, int unit_latency,
                        int64_t *stats_sum, int64_t *rounds, char *err, size_t errlen) {
  try {
    const Function &f = h->m.functions.front();
    LatencyModel lm = pickLatency(unit_latency);
    WarpInput in;
    in.warpSize = warp;
    for (size_t p = 0; p < f.params.size(); ++p) in.args.push_back({args[p]});
    auto load = [&] {
      size_t off = 0;
      for (const auto &g : h->m.globals) {
        in.globalInit[g.name] = std::vector<int32_t>(globals + off, globals + off + g.size);
        off += size_t(g.size);
      }
      off = 0;
      for (const auto &s : f.sharedDecls) {
        in.sharedInit[s.name] = std::vector<int32_t>(shared + off, shared + off + s.size);
        off += size_t(s.size);
      }
    };
    if (stats_sum)
      for (int i = 0; i < 7; ++i) stats_sum[i] = 0;
    int64_t r = 0;
    for (; r < max_rounds; ++r) {
      load();
      WarpResult res = executeWarp(h->m, f, in, lm);
      if (res.nonTerminated || !res.faults.empty() || res.taintedObservable)
        return fail(err, errlen, "chain step " + std::to_string(r) + " faulted or observed undef", 2);
      bool same = res.globalFinal == in.globalInit && res.sharedFinal == in.sharedInit;
      if (same) break;
      size_t off = 0;
      for (const auto &g : h->m.globals) {
        const auto &v = res.globalFinal.at(g.name);
        std::copy(v.begin(), v.end(), globals + off);
        off += size_t(g.size);
      }
      off = 0;
      for (const auto &s : f.sharedDecls) {
        const auto &v = res.sharedFinal.at(s.name);
        std::copy(v.begin(), v.end(), shared + off);
        off += size_t(s.size);
      }
      if (stats_sum) {
        stats_sum[0] += res.stats.issuedInstructions;
        stats_sum[1] += res.stats.threadCycles;
        stats_sum[2] += res.stats.usefulThreadCycles;
        stats_sum[3] += res.stats.serializedCycles;
        stats_sum[4] += res.stats.divergentBranchCount;
        stats_sum[5] += res.stats.sharedMemIssues;
        stats_sum[6] += res.stats.globalMemIssues;
      }
    }
    if (rounds) *rounds = r;
    if (r == max_rounds) return fail(err, errlen, "no fixpoint within max_rounds", 2);
    return 0;
  } catch (const std::exception &e) {
    return fail(err, errlen, e.what(), 2);
  }
}

// Full bitonic sort of independent B-key buckets by chaining the corpus
// compare-exchange step (bitonic.ir:6-43) through executeWarp: for every stage
// dir = 2..B and stride k = dir/2..1 one warp of B lanes runs with the bucket in
// shared `buf` and the step's `res` becomes the next step's `buf`.
// B must be a power of two <= 64 (warp limit, interp.cpp:334-335).
// stats_sum (may be NULL) accumulates the 7 counters over every step.
int ref_bitonic_sort(const ref_module *h, int32_t *keys, int64_t n, int B,
                     int threads, int unit_latency, int64_t *stats_sum,
                     char *err, size_t errlen) {
  if (B < 2 || B > 64 || (B & (B - 1)) || n % B)
    return fail(err, errlen, "bucket must be a power of two in [2,64] dividing n", 2);
  const Function &f = h->m.functions.front();
  if (f.params.size() != 2 || f.sharedDecls.size() != 1 || h->m.globals.size() != 1)
    return fail(err, errlen, "module is not the bitonic step kernel", 2);
  const std::string bufName = f.sharedDecls[0].name;
  const int64_t bufSize = f.sharedDecls[0].size;
  const std::string resName = h->m.globals[0].name;
  LatencyModel lm = pickLatency(unit_latency);
  int64_t nb = n / B;
  std::vector<std::array<int64_t, 7>> per(size_t(stats_sum ? nb : 0));
  std::vector<std::string> errors(1);
  std::atomic<bool> bad{false};
  parallelFor(nb, threads, [&](int64_t b) {
    if (bad.load()) return;
    try {
      std::vector<int32_t> cur(keys + b * B, keys + (b + 1) * B);
      std::array<int64_t, 7> acc{};
      for (int dir = 2; dir <= B; dir <<= 1)
        for (int k = dir >> 1; k >= 1; k >>= 1) {
          WarpInput in;
          in.warpSize = B;
          in.args = {{k}, {dir}};
          std::vector<int32_t> buf(size_t(bufSize), 0);
          std::copy(cur.begin(), cur.end(), buf.begin());
          in.sharedInit[bufName] = buf;
          WarpResult r = executeWarp(h->m, f, in, lm);
          if (r.nonTerminated || !r.faults.empty())
            throw std::runtime_error("bitonic step faulted");
          const auto &res = r.globalFinal.at(resName);
          std::copy(res.begin(), res.begin() + B, cur.begin());
          acc[0] += r.stats.issuedInstructions;
          acc[1] += r.stats.threadCycles;
          acc[2] += r.stats.usefulThreadCycles;
          acc[3] += r.stats.serializedCycles;
          acc[4] += r.stats.divergentBranchCount;
          acc[5] += r.stats.sharedMemIssues;
          acc[6] += r.stats.globalMemIssues;
        }
      std::copy(cur.begin(), cur.end(), keys + b * B);
      if (stats_sum) per[size_t(b)] = acc;
    } catch (const std::exception &e) {
      if (!bad.exchange(true)) errors[0] = e.what();
    }
  });
  if (bad) return fail(err, errlen, errors[0], 2);
  if (stats_sum) {
    for (int i = 0; i < 7; ++i) stats_sum[i] = 0;
    for (const auto &a : per)
      for (int i = 0; i < 7; ++i) stats_sum[i] += a[size_t(i)];
  }
  return 0;
}

// Generic chain of a one-warp sorting-network step kernel over B-key buckets:
// step s runs with the params step_args[s*arity .. s*arity+arity-1], the
// bucket in the step's shared array and its global `res` as the next step's
// input (the loop a network driver runs; used for ir/oddeven_step.ir, PCM).
// B <= 64 (warp limit, interp.cpp:334-335).  stats_sum as ref_bitonic_sort.
int ref_chain_sort(const ref_module *h, int32_t *keys, int64_t n, int B, const int32_t *step_args,
                   int nsteps, int arity, int threads, int unit_latency, int64_t *stats_sum,
                   char *err, size_t errlen) {
  if (B < 2 || B > 64 || n % B) return fail(err, errlen, "bucket must be in [2,64] and divide n", 2);
  const Function &f = h->m.functions.front();
  if (int(f.params.size()) != arity || f.sharedDecls.size() != 1 || h->m.globals.size() != 1)
    return fail(err, errlen, "module is not a one-buffer network step kernel of this arity", 2);
  const std::string bufName = f.sharedDecls[0].name;
  const int64_t bufSize = f.sharedDecls[0].size;
  const std::string resName = h->m.globals[0].name;
  LatencyModel lm = pickLatency(unit_latency);
  const int64_t nb = n / B;
  std::vector<std::array<int64_t, 7>> per(size_t(stats_sum ? nb : 0));
  std::vector<std::string> errors(1);
  std::atomic<bool> bad{false};
  parallelFor(nb, threads, [&](int64_t b) {
    if (bad.load()) return;
    try {
      std::vector<int32_t> cur(keys + b * B, keys + (b + 1) * B);
      std::array<int64_t, 7> acc{};
      for (int st = 0; st < nsteps; ++st) {
        WarpInput in;
        in.warpSize = B;
        for (int a = 0; a < arity; ++a) in.args.push_back({step_args[st * arity + a]});
        std::vector<int32_t> buf(size_t(bufSize), 0);
        std::copy(cur.begin(), cur.end(), buf.begin());
        in.sharedInit[bufName] = buf;
        WarpResult r = executeWarp(h->m, f, in, lm);
        if (r.nonTerminated || !r.faults.empty()) throw std::runtime_error("network step faulted");
        const auto &res = r.globalFinal.at(resName);
        std::copy(res.begin(), res.begin() + B, cur.begin());
        acc[0] += r.stats.issuedInstructions;
        acc[1] += r.stats.threadCycles;
        acc[2] += r.stats.usefulThreadCycles;
        acc[3] += r.stats.serializedCycles;
        acc[4] += r.stats.divergentBranchCount;
        acc[5] += r.stats.sharedMemIssues;
        acc[6] += r.stats.globalMemIssues;
      }
      std::copy(cur.begin(), cur.end(), keys + b * B);
      if (stats_sum) per[size_t(b)] = acc;
    } catch (const std::exception &e) {
      if (!bad.exchange(true)) errors[0] = e.what();
    }
  });
  if (bad) return fail(err, errlen, errors[0], 2);
  if (stats_sum) {
    for (int i = 0; i < 7; ++i) stats_sum[i] = 0;
    for (const auto &a : per)
      for (int i = 0; i < 7; ++i) stats_sum[i] += a[size_t(i)];
  }
  return 0;
}

// executeWarp over a batch in the GPU program layout (darm_gpu_program_execute):
// globals n_warps x (all globals, declaration order), shared n_warps x (all
// shared arrays) in/out (NULL: zero init, not returned), returns / has_ret
// n_warps x warp, faults n_warps, stats n_warps x 8 (ref_execute_warps' slots).
// latency: 28 entries in opcode order, or NULL for the defaults.
int ref_execute_program(const ref_module *h, int warp, int64_t n_warps, const int32_t *args, int64_t acount,
                        int32_t *globals, int32_t *shared, const int64_t *latency, int64_t max_steps,
                        int threads, int32_t *returns, uint8_t *has_ret, int32_t *faults, int64_t *stats,
                        char *err, size_t errlen) {
  const Function &f = h->m.functions.front();
  const size_t np = f.params.size();
  if (np && acount != 1 && acount != n_warps && acount != n_warps * warp)
    return fail(err, errlen, "bad argument count", 2);
  LatencyModel lm = LatencyModel::defaults();
  if (latency)
    for (int k = 0; k <= int(Opcode::Barrier); ++k) lm.set(Opcode(k), latency[k]);
  int64_t gw = 0, sw = 0;
  for (const auto &g : h->m.globals) gw += g.size;
  for (const auto &s : f.sharedDecls) sw += s.size;
  std::vector<std::string> errors(1);
  std::atomic<bool> bad{false};
  parallelFor(n_warps, threads, [&](int64_t w) {
    if (bad.load()) return;
    try {
      WarpInput in;
      in.warpSize = warp;
      for (size_t p = 0; p < np; ++p) {
        const int32_t *a = args + p * acount;
        if (acount == 1)
          in.args.push_back({a[0]});
        else if (acount == n_warps)
          in.args.push_back({a[w]});
        else
          in.args.push_back(std::vector<int32_t>(a + w * warp, a + (w + 1) * warp));
      }
      int64_t off = 0;
      for (const auto &g : h->m.globals) {
        const int32_t *src = globals + w * gw + off;
        in.globalInit[g.name] = std::vector<int32_t>(src, src + g.size);
        off += g.size;
      }
      off = 0;
      for (const auto &s : f.sharedDecls) {
        if (shared) {
          const int32_t *src = shared + w * sw + off;
          in.sharedInit[s.name] = std::vector<int32_t>(src, src + s.size);
        }
        off += s.size;
      }
      WarpResult r = executeWarp(h->m, f, in, lm, max_steps);
      off = 0;
      for (const auto &g : h->m.globals) {
        const auto &v = r.globalFinal.at(g.name);
        std::memcpy(globals + w * gw + off, v.data(), size_t(g.size) * 4);
        off += g.size;
      }
      off = 0;
      for (const auto &s : f.sharedDecls) {
        if (shared) {
          const auto &v = r.sharedFinal.at(s.name);
          std::memcpy(shared + w * sw + off, v.data(), size_t(s.size) * 4);
        }
        off += s.size;
      }
      if (returns)
        for (int l = 0; l < warp; ++l) {
          returns[w * warp + l] = r.returns[l].value_or(0);
          if (has_ret) has_ret[w * warp + l] = r.returns[l].has_value();
        }
      if (faults) faults[w] = int32_t(r.faults.size());
      if (stats) {
        int64_t *o = stats + w * 8;
        o[0] = r.stats.issuedInstructions;
        o[1] = r.stats.threadCycles;
        o[2] = r.stats.usefulThreadCycles;
        o[3] = r.stats.serializedCycles;
        o[4] = r.stats.divergentBranchCount;
        o[5] = r.stats.sharedMemIssues;
        o[6] = r.stats.globalMemIssues;
        o[7] = (r.nonTerminated ? 1 : 0) | (r.taintedObservable ? 2 : 0);
      }
    } catch (const std::exception &e) {
      if (!bad.exchange(true)) errors[0] = e.what();
    }
  });
  if (bad) return fail(err, errlen, errors[0], 2);
  return 0;
}

}  // extern "C"
