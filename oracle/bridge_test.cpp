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
// Exit 0 on success, 1 on the first mismatch (with the reference's diff).
#include <cstdio>
#include <cstdlib>
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
  return 0;
}
