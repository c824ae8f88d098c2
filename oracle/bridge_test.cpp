// bridge_test.cpp — the reference's acceptance criterion 1 run against the GPU
// through the reference-side binding (include/darm_gpu.hpp).  TEST
// INFRASTRUCTURE: built by oracle/Makefile (target `bridge`) from the unmodified
// reference objects plus libdarm_gpu.so; tests/test_bridge.py runs it on a B200.
//
// For every positive corpus kernel (helpers.hpp:27-32), warp sizes {4, 8, 32,
// 64} and `fixtures` makeRandomInput fixtures (acceptance.cpp:101-119 uses 100
// fixtures x {4, 8, 32}):
//   a = executeWarp(original module)            the reference interpreter
//   b = executeWarp(runDarm(module))            the reference's melded IR
//   c = darm::gpu::executeWarps(..., Unmelded)  sm_100a unmelded form
//   d = darm::gpu::executeWarps(..., Melded)    sm_100a melded form
// and compareRuns(a, b), compareRuns(a, c), compareRuns(a, d) must all be equal.
// Then acceptance criteria 5 and 6 (acceptance.cpp:243-310) with every
// executeWarp replaced by darm::gpu::executeWarpsIR (the GPU warp
// interpreter): serialized cycles drop on the structured kernels at a
// half-warp split (sb3 / sb4 more than sb1, sb3 with >= 2 melds) and bitonic
// issues fewer shared-memory accesses after melding; the GPU's statistics are
// also checked equal to the reference interpreter's on every fixture.
// Exit 0 on success, 1 on the first mismatch (with the reference's diff).
#include <cstdio>
#include <cstdlib>
#include <map>
#include <string>
#include <vector>

#include "darm/fixtures.hpp"
#include "darm/interp.hpp"
#include "darm/melding.hpp"
#include "darm/parser.hpp"
#include "darm_gpu.hpp"

using namespace darm;

// corpus kernels embedded at build time (oracle/embed_corpus.py)
extern "C" const char *const ref_corpus_names[];
extern "C" const char *const ref_corpus_texts[];

static const char *corpus_text(const char *k) {
  for (int i = 0; ref_corpus_names[i]; ++i)
    if (std::string(ref_corpus_names[i]) == k) return ref_corpus_texts[i];
  return nullptr;
}

// Sum of one WarpExecStats counter over `seeds` fixtures, on the GPU
// interpreter; every fixture's counters must equal the reference's.
template <class Get>
static bool gpu_stat_sum(const Module &m, std::vector<WarpInput> ins, Get get, int64_t &sum) {
  const Function &f = m.functions[0];
  const LatencyModel lm = LatencyModel::defaults();
  auto g = gpu::executeWarpsIR(m, f, ins, lm);
  sum = 0;
  for (size_t i = 0; i < ins.size(); ++i) {
    WarpResult c = executeWarp(m, f, ins[i], lm);
    if (get(g[i].stats) != get(c.stats) || g[i].stats.serializedCycles != c.stats.serializedCycles ||
        g[i].stats.sharedMemIssues != c.stats.sharedMemIssues) {
      std::printf("MISMATCH stats fixture %zu\n", i);
      return false;
    }
    sum += get(g[i].stats);
  }
  return true;
}

static bool criteria5and6() {
  const LatencyModel lm = LatencyModel::defaults();
  std::map<std::string, double> rel;
  std::map<std::string, size_t> melds;
  for (const char *k : {"sb1", "sb1r", "sb2", "sb2r", "sb3", "sb3r", "sb4", "sb4r"}) {
    Module pre = parseModule(corpus_text(k));
    Module post = pre;
    melds[k] = runDarm(post.functions[0], MeldConfig{}, lm).melds.size();
    std::vector<WarpInput> ins;
    for (uint64_t s = 0; s < 10; ++s) {
      WarpInput in = makeRandomInput(pre, pre.functions[0], 32, 3000 + s);
      in.args[0] = {16};                                   // half-warp split (acceptance.cpp:251-257)
      if (in.args.size() > 1) in.args[1] = {24};
      ins.push_back(in);
    }
    int64_t before = 0, after = 0;
    auto ser = [](const WarpExecStats &st) { return st.serializedCycles; };
    if (!gpu_stat_sum(pre, ins, ser, before) || !gpu_stat_sum(post, ins, ser, after)) return false;
    if (before <= 0 || after >= before) {
      std::printf("C5 FAIL %s: serialized %lld -> %lld\n", k, (long long)before, (long long)after);
      return false;
    }
    rel[k] = double(before - after) / double(before);
  }
  if (melds["sb3"] < 2 || rel["sb3"] <= rel["sb1"] || rel["sb4"] <= rel["sb1"]) {
    std::printf("C5 FAIL: sb3 melds %zu, reductions sb1 %.3f sb3 %.3f sb4 %.3f\n", melds["sb3"], rel["sb1"],
                rel["sb3"], rel["sb4"]);
    return false;
  }
  std::printf("C5 (GPU interpreter): ok, serialized-cycle reduction sb1 %.3f sb3 %.3f sb4 %.3f\n", rel["sb1"],
              rel["sb3"], rel["sb4"]);
  Module pre = parseModule(corpus_text("bitonic"));
  Module post = pre;
  runDarm(post.functions[0], MeldConfig{}, lm);
  std::vector<WarpInput> ins;
  for (uint64_t s = 0; s < 10; ++s) ins.push_back(makeRandomInput(pre, pre.functions[0], 32, 5000 + s));
  int64_t before = 0, after = 0;
  auto shm = [](const WarpExecStats &st) { return st.sharedMemIssues; };
  if (!gpu_stat_sum(pre, ins, shm, before) || !gpu_stat_sum(post, ins, shm, after)) return false;
  if (after >= before) {
    std::printf("C6 FAIL: shared-memory issues %lld -> %lld\n", (long long)before, (long long)after);
    return false;
  }
  std::printf("C6 (GPU interpreter): ok, bitonic shared-memory issues %lld -> %lld\n", (long long)before,
              (long long)after);
  return true;
}

// The reference's testing::oracleCompare (helpers.hpp:156-174), the result
// oracle of criterion 1 and test_pipeline, run on the GPU
// (darm::gpu::oracleCompare): every positive kernel against its runDarm
// output, 100 fixtures x warps {4, 8, 32} -> no diff; and a mutated melded
// sb1 (`mul %v 3` -> `mul %v 4`) -> the same first diff the CPU oracle reports.
static std::string cpu_oracle(const Module &m1, const Function &f1, const Module &m2, const Function &f2,
                              int fixtures, uint64_t seed) {
  for (int w : {4, 8, 32})
    for (int i = 0; i < fixtures; ++i) {
      WarpInput in = makeRandomInput(m1, f1, w, seed + uint64_t(i));
      CompareVerdict v = compareRuns(executeWarp(m1, f1, in, LatencyModel::defaults()),
                                     executeWarp(m2, f2, in, LatencyModel::defaults()));
      if (!v.equal) return f1.name + " warp " + std::to_string(w) + " fixture " + std::to_string(i) + ": " + v.diff;
    }
  return "";
}

static bool gpu_oracle() {
  for (const char *k : {"sb1", "sb1r", "sb2", "sb2r", "sb3", "sb3r", "sb4", "sb4r", "bitonic", "nested"}) {
    Module orig = parseModule(corpus_text(k));
    Module melded = orig;
    runDarm(melded.functions[0], MeldConfig{}, LatencyModel::defaults());
    const std::string d = gpu::oracleCompare(orig, orig.functions[0], melded, melded.functions[0], 100, 7000);
    if (!d.empty()) {
      std::printf("GPU oracle MISMATCH %s: %s\n", k, d.c_str());
      return false;
    }
  }
  std::string text = corpus_text("sb1");
  Module orig = parseModule(text);
  Module melded = orig;
  runDarm(melded.functions[0], MeldConfig{}, LatencyModel::defaults());
  std::string mt = printModule(melded);
  const size_t at = mt.find("mul ");
  if (at == std::string::npos) return false;
  const size_t three = mt.find(" 3", at);
  if (three == std::string::npos) return false;
  mt.replace(three, 2, " 4");
  Module bad = parseModule(mt);
  const std::string g = gpu::oracleCompare(orig, orig.functions[0], bad, bad.functions[0], 20, 7000);
  const std::string c = cpu_oracle(orig, orig.functions[0], bad, bad.functions[0], 20, 7000);
  if (g.empty() || g != c) {
    std::printf("GPU oracle on a mutated kernel: gpu '%s' cpu '%s'\n", g.c_str(), c.c_str());
    return false;
  }
  std::printf("GPU oracle (oracleCompare on executeWarpsIR): ok, 10 kernels x 300 fixtures equal; mutated sb1 "
              "caught with the CPU oracle's diff\n");
  return true;
}

int main(int argc, char **argv) {
  const int fixtures = argc > 1 ? std::atoi(argv[1]) : 100;
  const char *kernels[] = {"sb1", "sb1r", "sb2", "sb2r", "sb3", "sb3r", "sb4", "sb4r", "bitonic", "nested"};
  int n_devices = 0;
  char err[256];
  if (darm_gpu_init(&n_devices, err, sizeof err) != DARM_OK) {
    std::fprintf(stderr, "no GPU: %s\n", err);
    return 2;
  }
  long long compared = 0;
  for (const char *k : kernels) {
    const char *text = nullptr;
    for (int i = 0; ref_corpus_names[i]; ++i)
      if (std::string(ref_corpus_names[i]) == k) text = ref_corpus_texts[i];
    if (!text) {
      std::fprintf(stderr, "corpus kernel %s not embedded\n", k);
      return 2;
    }
    Module orig = parseModule(text);
    Module melded = orig;
    runDarm(melded.functions[0], MeldConfig{}, LatencyModel::defaults());
    const Function &f = orig.functions[0];
    for (int warp : {4, 8, 32, 64}) {
      std::vector<WarpInput> ins;
      for (int i = 0; i < fixtures; ++i) ins.push_back(makeRandomInput(orig, f, warp, 1000 + uint64_t(i)));
      auto gu = gpu::executeWarps(orig, f, ins, gpu::Form::Unmelded);
      auto gm = gpu::executeWarps(orig, f, ins, gpu::Form::Melded);
      for (int i = 0; i < fixtures; ++i) {
        WarpResult a = executeWarp(orig, f, ins[size_t(i)], LatencyModel::defaults());
        WarpResult b = executeWarp(melded, melded.functions[0], ins[size_t(i)], LatencyModel::defaults());
        for (const auto *other : {&b, &gu[size_t(i)], &gm[size_t(i)]}) {
          CompareVerdict v = compareRuns(a, *other);
          ++compared;
          if (!v.equal) {
            std::printf("MISMATCH %s warp %d fixture %d: %s\n", k, warp, i, v.diff.c_str());
            return 1;
          }
        }
      }
    }
    std::printf("%s: ok\n", k);
  }
  std::printf("bridge: %lld compareRuns verdicts equal\n", compared);
  return criteria5and6() && gpu_oracle() ? 0 : 1;
}
