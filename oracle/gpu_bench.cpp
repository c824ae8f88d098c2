// gpu_bench.cpp — the reference's `darm bench` rows with GPU columns: the stats
// wire format of SURVEY.md §8(f) rank 2.  A reference-side driver (built by
// oracle/Makefile target `gpubench` from the unmodified reference objects plus
// libdarm_gpu.so, like bridge_test.cpp); TEST / INTEGRATION INFRASTRUCTURE, not
// part of the product path.
//
// For every positive corpus kernel it computes the reference's BenchRow
// (tools/darm_cli.cpp:193-269: runDarm at the threshold, `fixtures`
// makeRandomInput fixtures, executeWarp before / after, compareRuns, mean
// serialized cycles and utilisation) and adds, from the GPU through
// include/darm_gpu.hpp and the C-ABI:
//   gpuOracleOk      compareRuns(reference before, GPU unmelded / melded) on the
//                    same fixtures (acceptance criterion 1's check)
//   gpuLanes         lanes of the timed batch (warp x warps, config 1 shape)
//   gpuUnmeldedUs / gpuMeldedUs / gpuSpeedup   kernel time per launch: mean
//                    of `launches` back-to-back DEVICE-mode launches over 8
//                    device copies of the batch (CUDA events), best of `reps`
//   gpuSimEqual      the simulator run on the GPU interpreter
//                    (darm::gpu::executeWarpsIR, before and after the pass)
//                    produced exactly the CPU interpreter's WarpResults,
//                    statistics included; cpuSimMs / gpuSimMs time both
// The JSON keys are the reference's (darm_cli.cpp:343-358) plus the gpu* keys,
// so consumers of the reference's bench JSON read both side by side; the table
// prints the reference's columns followed by the GPU ones.
//
//   darm_gpu_bench [--fixtures N] [--warp W] [--threshold T] [--gpu-warps G]
//                  [--reps R] [--launches L] [--seed S] [--json PATH] [--no-gpu]
// Exit codes as the reference CLI (darm_cli.cpp:25-27): 0 ok, 2 usage,
// 3 oracle failure or internal error.
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <string>
#include <vector>

#include <cuda_runtime.h>

#include "darm/fixtures.hpp"
#include "darm/interp.hpp"
#include "darm/melding.hpp"
#include "darm/parser.hpp"
#include "darm/verifier.hpp"
#include "darm_gpu.hpp"
#include "json.hpp"

using namespace darm;
using json = nlohmann::json;

extern "C" const char *const ref_corpus_names[];
extern "C" const char *const ref_corpus_texts[];

namespace {

struct Row {
  std::string kernel, mode = "darm";
  double threshold = 0.2;
  bool rejected = false, oracleOk = true, converged = true;
  std::string oracleDiff;
  int melds = 0;
  std::vector<double> mpScores;
  double serBefore = 0, serAfter = 0, utilBefore = 1, utilAfter = 1;
  // GPU columns
  bool gpu = false, gpuOracleOk = true, gpuSimEqual = true;
  double cpuSimMs = 0, gpuSimMs = 0;
  std::string gpuOracleDiff;
  long long gpuLanes = 0;
  double gpuUnmeldedUs = 0, gpuMeldedUs = 0;
};

double reduction(double b, double a) { return b <= 0 ? 0.0 : 100.0 * (b - a) / b; }

// Kernel time of one batch through the C-ABI, DEVICE-resident buffers: the
// batch is uploaded once into kCopies device copies (together larger than the
// 126 MB L2 at the config 1 shape, so consecutive launches read from HBM),
// then `launches` launches rotate over the copies between two CUDA events on
// the stream they run on; the figure is the per-launch mean, best of `reps`
// such batches after one untimed batch.  (Round 1 timed single HOST-mode
// launches, whose launch overhead and first-touch effects swamped the
// 7-16 us kernels.)
constexpr int kCopies = 8;

void cuda_ok(cudaError_t e, const char *what) {
  if (e != cudaSuccess) throw std::runtime_error(std::string(what) + ": " + cudaGetErrorString(e));
}

double gpu_kernel_us(const Module &m, const Function &f, const std::vector<WarpInput> &ins, int form, int reps,
                     int launches) {
  const int W = ins[0].warpSize;
  const int64_t n = int64_t(ins.size());
  const size_t np = f.params.size();
  std::vector<int32_t> args(np * size_t(n) * W);
  for (int64_t w = 0; w < n; ++w)
    for (size_t p = 0; p < np; ++p)
      for (int l = 0; l < W; ++l) {
        const auto &v = ins[size_t(w)].args[p];
        args[p * n * W + w * W + l] = v.size() == 1 ? v[0] : v.at(size_t(l));
      }
  std::vector<std::vector<int32_t>> gl(m.globals.size(), std::vector<int32_t>(size_t(n) * W, 0));
  for (size_t g = 0; g < m.globals.size(); ++g)
    for (int64_t w = 0; w < n; ++w) {
      auto it = ins[size_t(w)].globalInit.find(m.globals[g].name);
      if (it != ins[size_t(w)].globalInit.end())
        for (int l = 0; l < W && size_t(l) < it->second.size(); ++l) gl[g][size_t(w) * W + l] = it->second[size_t(l)];
    }
  std::vector<std::vector<int32_t>> sh(f.sharedDecls.size());
  for (size_t s = 0; s < f.sharedDecls.size(); ++s) {
    const size_t size = size_t(f.sharedDecls[s].size);
    sh[s].assign(size_t(n) * size, 0);
    for (int64_t w = 0; w < n; ++w) {
      auto it = ins[size_t(w)].sharedInit.find(f.sharedDecls[s].name);
      if (it != ins[size_t(w)].sharedInit.end())
        std::copy_n(it->second.begin(), std::min(size, it->second.size()), sh[s].begin() + size_t(w) * size);
    }
  }
  // device copies: args, globals and shared initialisers per copy
  std::vector<void *> owned;
  auto upload = [&](const std::vector<int32_t> &v) {
    void *d = nullptr;
    cuda_ok(cudaMalloc(&d, std::max<size_t>(4, v.size() * 4)), "cudaMalloc");
    owned.push_back(d);
    if (!v.empty()) cuda_ok(cudaMemcpy(d, v.data(), v.size() * 4, cudaMemcpyHostToDevice), "cudaMemcpy");
    return static_cast<int32_t *>(d);
  };
  struct Copy {
    int32_t *args;
    std::vector<int32_t *> g;
    std::vector<const int32_t *> s;
  };
  std::vector<Copy> copies(kCopies);
  for (auto &c : copies) {
    c.args = upload(args);
    for (auto &v : gl) c.g.push_back(upload(v));
    for (auto &v : sh) c.s.push_back(upload(v));
  }
  cudaStream_t stream;
  cudaEvent_t e0, e1;
  cuda_ok(cudaStreamCreateWithFlags(&stream, cudaStreamNonBlocking), "cudaStreamCreate");
  cuda_ok(cudaEventCreate(&e0), "cudaEventCreate");
  cuda_ok(cudaEventCreate(&e1), "cudaEventCreate");
  auto launch = [&](const Copy &c) {
    char err[512] = {0};
    int rc = darm_gpu_execute_warps(f.name.c_str(), form, W, n, c.args, n * W,
                                    c.g.data(), int(c.g.size()), c.s.empty() ? nullptr : c.s.data(), int(c.s.size()),
                                    nullptr, DARM_MEM_DEVICE, stream, nullptr, err, sizeof err);
    if (rc != DARM_OK) throw std::runtime_error(std::string("darm_gpu: ") + err);
  };
  double best = 1e30;
  for (int r = 0; r <= reps; ++r) {
    cuda_ok(cudaStreamSynchronize(stream), "sync");
    cuda_ok(cudaEventRecord(e0, stream), "record");
    for (int i = 0; i < launches; ++i) launch(copies[size_t(i % kCopies)]);
    cuda_ok(cudaEventRecord(e1, stream), "record");
    cuda_ok(cudaEventSynchronize(e1), "sync");
    float ms = 0;
    cuda_ok(cudaEventElapsedTime(&ms, e0, e1), "elapsed");
    if (r > 0) best = std::min(best, 1e3 * double(ms) / launches);   // batch 0 is the warm-up
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaStreamDestroy(stream);
  for (void *d : owned) cudaFree(d);
  return best;
}

Row bench_one(const std::string &kernel, const char *text, const Row &opts, int fixtures, int warp,
              uint64_t seed, bool use_gpu, int gpu_warps, int reps, int launches) {
  Row row = opts;
  row.kernel = kernel;
  Module m = parseModule(text);
  Module melded = m;
  MeldConfig cfg;
  cfg.threshold = row.threshold;
  const LatencyModel lm = LatencyModel::defaults();
  try {
    for (auto &f : melded.functions) {
      MeldReport rep = runDarm(f, cfg, lm);
      row.melds += int(rep.melds.size());
      row.converged = row.converged && rep.converged;
      for (const auto &a : rep.melds) row.mpScores.push_back(a.mpScore);
      auto viol = verifySsa(f);
      if (!viol.empty()) throw std::logic_error("transform broke SSA in " + f.name);
    }
  } catch (const std::logic_error &) {
    throw;
  } catch (const std::exception &) {
    row.rejected = true;
    return row;
  }
  const Function &f0 = m.functions.front();
  const Function &f1 = melded.functions.front();
  std::vector<WarpInput> ins;
  for (int i = 0; i < fixtures; ++i) ins.push_back(makeRandomInput(m, f0, warp, seed + uint64_t(i)));
  std::vector<WarpResult> gu, gm;
  if (use_gpu) {
    gu = gpu::executeWarps(m, f0, ins, gpu::Form::Unmelded);
    gm = gpu::executeWarps(m, f0, ins, gpu::Form::Melded);
  }
  // the simulator itself on the GPU interpreter (executeWarpsIR): same stats?
  std::vector<WarpResult> sim_b, sim_a;
  if (use_gpu) {
    const auto t0 = std::chrono::steady_clock::now();
    sim_b = gpu::executeWarpsIR(m, f0, ins, lm);
    sim_a = gpu::executeWarpsIR(melded, f1, ins, lm);
    row.gpuSimMs = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  }
  double sb = 0, sa = 0, ub = 0, ua = 0;
  const auto c0 = std::chrono::steady_clock::now();
  std::vector<WarpResult> cpu_b, cpu_a;
  for (int i = 0; i < fixtures; ++i) {
    cpu_b.push_back(executeWarp(m, f0, ins[size_t(i)], lm));
    cpu_a.push_back(executeWarp(melded, f1, ins[size_t(i)], lm));
  }
  row.cpuSimMs = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - c0).count();
  auto same_stats = [](const WarpResult &x, const WarpResult &y) {
    return x.stats.issuedInstructions == y.stats.issuedInstructions && x.stats.threadCycles == y.stats.threadCycles &&
           x.stats.usefulThreadCycles == y.stats.usefulThreadCycles &&
           x.stats.serializedCycles == y.stats.serializedCycles &&
           x.stats.divergentBranchCount == y.stats.divergentBranchCount &&
           x.stats.sharedMemIssues == y.stats.sharedMemIssues && x.stats.globalMemIssues == y.stats.globalMemIssues &&
           x.returns == y.returns && x.globalFinal == y.globalFinal && x.sharedFinal == y.sharedFinal &&
           x.faults.size() == y.faults.size() && x.nonTerminated == y.nonTerminated &&
           x.taintedObservable == y.taintedObservable;
  };
  for (int i = 0; i < fixtures; ++i) {
    const WarpResult &before = cpu_b[size_t(i)];
    const WarpResult &after = cpu_a[size_t(i)];
    if (use_gpu && !(same_stats(before, sim_b[size_t(i)]) && same_stats(after, sim_a[size_t(i)])))
      row.gpuSimEqual = false;
    CompareVerdict v = compareRuns(before, after);
    if (!v.equal && row.oracleOk) {
      row.oracleOk = false;
      row.oracleDiff = v.diff;
    }
    if (use_gpu)
      for (const auto *g : {&gu[size_t(i)], &gm[size_t(i)]}) {
        CompareVerdict gv = compareRuns(before, *g);
        if (!gv.equal && row.gpuOracleOk) {
          row.gpuOracleOk = false;
          row.gpuOracleDiff = gv.diff;
        }
      }
    sb += double(before.stats.serializedCycles);
    sa += double(after.stats.serializedCycles);
    ub += before.stats.utilization;
    ua += after.stats.utilization;
  }
  row.serBefore = sb / fixtures;
  row.serAfter = sa / fixtures;
  row.utilBefore = ub / fixtures;
  row.utilAfter = ua / fixtures;
  if (use_gpu) {
    // the timed batch: gpu_warps makeRandomInput fixtures at warp 32, half-warp
    // split (the config 1 shape, acceptance.cpp:251-257: n = 16, h = 16, q = 24)
    std::vector<WarpInput> big;
    big.reserve(size_t(gpu_warps));
    for (int i = 0; i < gpu_warps; ++i) {
      WarpInput in = makeRandomInput(m, f0, 32, seed + 100000 + uint64_t(i));
      for (size_t p = 0; p < f0.params.size(); ++p) {
        const std::string &pn = f0.params[p];
        if (pn == "%n" || pn == "n" || pn == "%h" || pn == "h") in.args[p] = {16};
        if (pn == "%q" || pn == "q") in.args[p] = {24};
      }
      big.push_back(std::move(in));
    }
    row.gpu = true;
    row.gpuLanes = 32LL * gpu_warps;
    row.gpuUnmeldedUs = gpu_kernel_us(m, f0, big, DARM_UNMELDED, reps, launches);
    row.gpuMeldedUs = gpu_kernel_us(m, f0, big, DARM_MELDED, reps, launches);
  }
  return row;
}

json to_json(const Row &r) {
  json j = {{"kernel", r.kernel},
            {"mode", r.mode},
            {"threshold", r.threshold},
            {"rejected", r.rejected},
            {"melded", r.melds > 0},
            {"melds", r.melds},
            {"converged", r.converged},
            {"mpScores", r.mpScores},
            {"oracleOk", r.oracleOk},
            {"oracleDiff", r.oracleDiff},
            {"serializedBefore", r.serBefore},
            {"serializedAfter", r.serAfter},
            {"serializedReductionPercent", reduction(r.serBefore, r.serAfter)},
            {"utilizationBefore", r.utilBefore},
            {"utilizationAfter", r.utilAfter}};
  if (r.gpu) {
    j["gpuOracleOk"] = r.gpuOracleOk;
    j["gpuOracleDiff"] = r.gpuOracleDiff;
    j["gpuLanes"] = r.gpuLanes;
    j["gpuUnmeldedUs"] = r.gpuUnmeldedUs;
    j["gpuMeldedUs"] = r.gpuMeldedUs;
    j["gpuSpeedup"] = r.gpuMeldedUs > 0 ? r.gpuUnmeldedUs / r.gpuMeldedUs : 0.0;
    j["gpuSimEqual"] = r.gpuSimEqual;
    j["cpuSimMs"] = r.cpuSimMs;
    j["gpuSimMs"] = r.gpuSimMs;
  } else {
    for (const char *k : {"gpuOracleOk", "gpuOracleDiff", "gpuLanes", "gpuUnmeldedUs", "gpuMeldedUs", "gpuSpeedup",
                          "gpuSimEqual", "cpuSimMs", "gpuSimMs"})
      j[k] = nullptr;
  }
  return j;
}

}  // namespace

int main(int argc, char **argv) {
  int fixtures = 10, warp = 32, gpu_warps = 1 << 15, reps = 5, launches = 50;
  uint64_t seed = 3000;
  Row opts;
  std::string json_path;
  bool use_gpu = true;
  for (int i = 1; i < argc; ++i) {
    const std::string a = argv[i];
    auto next = [&]() -> const char * {
      if (i + 1 >= argc) {
        std::fprintf(stderr, "missing value for %s\n", a.c_str());
        std::exit(2);
      }
      return argv[++i];
    };
    if (a == "--fixtures") fixtures = std::atoi(next());
    else if (a == "--warp") warp = std::atoi(next());
    else if (a == "--threshold") opts.threshold = std::atof(next());
    else if (a == "--gpu-warps") gpu_warps = std::atoi(next());
    else if (a == "--reps") reps = std::atoi(next());
    else if (a == "--launches") launches = std::atoi(next());
    else if (a == "--seed") seed = std::strtoull(next(), nullptr, 10);
    else if (a == "--json") json_path = next();
    else if (a == "--no-gpu") use_gpu = false;
    else {
      std::fprintf(stderr, "usage: darm_gpu_bench [--fixtures N] [--warp W] [--threshold T] [--gpu-warps G] "
                           "[--reps R] [--launches L] [--seed S] [--json PATH] [--no-gpu]\n");
      return 2;
    }
  }
  if (fixtures < 1 || warp < 1 || warp > 64 || gpu_warps < 1 || reps < 1 || launches < 1) {
    std::fprintf(stderr, "bad arguments\n");
    return 2;
  }
  if (use_gpu) {
    int n = 0;
    char err[256];
    if (darm_gpu_init(&n, err, sizeof err) != DARM_OK) {
      std::fprintf(stderr, "no GPU: %s\n", err);
      return 3;
    }
  }
  const char *kernels[] = {"sb1", "sb1r", "sb2", "sb2r", "sb3", "sb3r", "sb4", "sb4r", "nested", "bitonic"};
  json out = json::array();
  bool failed = false;
  std::printf("%-14s %-13s %5s  %-8s %5s  %9s %9s %7s  %5s %5s  %-6s %9s %9s %6s\n", "kernel", "mode", "thr",
              "status", "melds", "ser.pre", "ser.post", "red%", "u.pre", "u.post", "gpu", "gpu.un.us", "gpu.me.us",
              "gpu.x");
  try {
    for (const char *k : kernels) {
      const char *text = nullptr;
      for (int i = 0; ref_corpus_names[i]; ++i)
        if (std::string(ref_corpus_names[i]) == k) text = ref_corpus_texts[i];
      if (!text) throw std::runtime_error(std::string("corpus kernel not embedded: ") + k);
      Row r = bench_one(k, text, opts, fixtures, warp, seed, use_gpu, gpu_warps, reps, launches);
      std::string status = r.rejected ? "rejected" : (r.melds > 0 ? "melded" : "no-meld");
      if (!r.oracleOk) status = "ORACLE-FAIL";
      const char *gst = !r.gpu ? "-" : (r.gpuOracleOk && r.gpuSimEqual ? "ok" : "FAIL");
      failed = failed || !r.oracleOk || (r.gpu && (!r.gpuOracleOk || !r.gpuSimEqual));
      std::printf("%-14s %-13s %5.2f  %-8s %5d  %9.1f %9.1f %6.1f%%  %5.3f %5.3f  %-6s %9.2f %9.2f %6.3f\n",
                  r.kernel.c_str(), r.mode.c_str(), r.threshold, status.c_str(), r.melds, r.serBefore, r.serAfter,
                  reduction(r.serBefore, r.serAfter), r.utilBefore, r.utilAfter, gst, r.gpuUnmeldedUs,
                  r.gpuMeldedUs, r.gpuMeldedUs > 0 ? r.gpuUnmeldedUs / r.gpuMeldedUs : 0.0);
      out.push_back(to_json(r));
    }
  } catch (const std::exception &e) {
    std::fprintf(stderr, "internal error: %s\n", e.what());
    return 3;
  }
  if (!json_path.empty()) {
    std::ofstream os(json_path);
    os << out.dump(2) << "\n";
  }
  return failed ? 3 : 0;
}
