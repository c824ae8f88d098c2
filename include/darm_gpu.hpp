// darm_gpu.hpp — reference-side C++ binding of the C-ABI (header-only).
//
// This is the adapter a maintainer of the reference adds to call the B200
// kernels from code that already speaks darm::Module / WarpInput / WarpResult
// (/root/reference/proj/include/darm/interp.hpp:14-53).  It replaces, for the
// corpus kernels, the per-warp interpreter call
//
//     WarpResult executeWarp(const Module&, const Function&, const WarpInput&,
//                            const LatencyModel&, int64_t)          // interp.hpp:57
//
// with one batched GPU launch, and returns WarpResults that the reference's own
// compareRuns (interp.hpp:67, interp.cpp:383-426) accepts unchanged:
//   returns      all nullopt (corpus kernels `ret` void)
//   globalFinal  every declared word; words >= warpSize keep their initial
//                value (corpus kernels index their globals by %t only)
//   faults       one LaneFault per faulted lane (lane -1: the GPU reports
//                counts; compareRuns compares counts, interp.cpp:411-414)
//   stats        zero (SIMT utilisation comes from ncu on the GPU)
// Used by oracle/bridge_test.cpp, which runs the reference's acceptance
// criterion 1 (acceptance.cpp:101-119) against the GPU.
#pragma once

#include <stdexcept>
#include <string>
#include <vector>

#include "darm/fixtures.hpp"
#include "darm/interp.hpp"
#include "darm/parser.hpp"
#include "darm_gpu.h"

namespace darm {
namespace gpu {

enum class Form { Unmelded = DARM_UNMELDED, Melded = DARM_MELDED };

inline std::vector<WarpResult> executeWarps(const Module &m, const Function &f,
                                            const std::vector<WarpInput> &ins, Form form) {
  std::vector<WarpResult> out(ins.size());
  if (ins.empty()) return out;
  const int W = ins[0].warpSize;
  const int64_t n = int64_t(ins.size());
  for (const auto &in : ins)
    if (in.warpSize != W) throw std::runtime_error("darm::gpu::executeWarps: mixed warp sizes");
  // arguments: per lane (acount = n*W) covers broadcast and per-lane vectors
  const size_t np = f.params.size();
  std::vector<int32_t> args(np * size_t(n) * W);
  for (int64_t w = 0; w < n; ++w) {
    if (ins[w].args.size() != np) throw std::runtime_error("argument count mismatch");
    for (size_t p = 0; p < np; ++p)
      for (int l = 0; l < W; ++l) {
        const auto &v = ins[w].args[p];
        args[p * n * W + w * W + l] = v.size() == 1 ? v[0] : v.at(size_t(l));
      }
  }
  // globals: compact, W words per warp
  std::vector<std::vector<int32_t>> gl(m.globals.size(), std::vector<int32_t>(size_t(n) * W, 0));
  for (size_t g = 0; g < m.globals.size(); ++g)
    for (int64_t w = 0; w < n; ++w) {
      auto it = ins[w].globalInit.find(m.globals[g].name);
      if (it == ins[w].globalInit.end()) continue;
      for (int l = 0; l < W && size_t(l) < it->second.size(); ++l) gl[g][size_t(w) * W + l] = it->second[l];
    }
  std::vector<std::vector<int32_t>> sh(f.sharedDecls.size());
  for (size_t s = 0; s < f.sharedDecls.size(); ++s) {
    const auto size = size_t(f.sharedDecls[s].size);
    sh[s].assign(size_t(n) * size, 0);
    for (int64_t w = 0; w < n; ++w) {
      auto it = ins[w].sharedInit.find(f.sharedDecls[s].name);
      if (it != ins[w].sharedInit.end())
        for (size_t i = 0; i < it->second.size() && i < size; ++i) sh[s][size_t(w) * size + i] = it->second[i];
    }
  }
  std::vector<int32_t *> gp;
  for (auto &v : gl) gp.push_back(v.data());
  std::vector<const int32_t *> sp;
  for (auto &v : sh) sp.push_back(v.data());
  std::vector<int32_t> faults(size_t(n), 0);
  char err[512] = {0};
  int rc = darm_gpu_execute_warps(f.name.c_str(), int(form), W, n, args.data(), n * W, gp.data(),
                                  int(gp.size()), sp.empty() ? nullptr : sp.data(), int(sp.size()),
                                  faults.data(), DARM_MEM_HOST, nullptr, nullptr, err, sizeof err);
  if (rc == DARM_USER_ERROR) throw std::runtime_error(std::string("darm_gpu: ") + err);
  if (rc != DARM_OK) throw std::logic_error(std::string("darm_gpu: ") + err);
  for (int64_t w = 0; w < n; ++w) {
    WarpResult &r = out[size_t(w)];
    r.returns.assign(size_t(W), std::nullopt);
    for (size_t g = 0; g < m.globals.size(); ++g) {
      const auto &decl = m.globals[g];
      std::vector<int32_t> v(size_t(decl.size), 0);
      auto it = ins[w].globalInit.find(decl.name);
      if (it != ins[w].globalInit.end())
        for (size_t i = 0; i < it->second.size() && i < v.size(); ++i) v[i] = it->second[i];
      for (int l = 0; l < W && l < decl.size; ++l) v[size_t(l)] = gl[g][size_t(w) * W + l];
      r.globalFinal[decl.name] = std::move(v);
    }
    for (int i = 0; i < faults[size_t(w)]; ++i) r.faults.push_back({-1, "", "fault on the GPU"});
  }
  return out;
}

// executeWarp for a batch of warps of ANY function on the GPU interpreter
// (darm_gpu_program_*): the module is printed with the reference's printModule
// (parser.hpp) and lowered by the library; the WarpResults carry everything
// executeWarp fills — returns, globalFinal, sharedFinal, stats (incl.
// serializedCycles / utilization), fault count (lanes -1) and the
// nonTerminated / taintedObservable flags — so compareRuns and the bench
// statistics work unchanged.  `lm` supplies the 28 opcode latencies.
inline std::vector<WarpResult> executeWarpsIR(const Module &m, const Function &f,
                                              const std::vector<WarpInput> &ins, const LatencyModel &lm,
                                              int64_t maxSteps = 10000000) {
  std::vector<WarpResult> out(ins.size());
  if (ins.empty()) return out;
  Module one;
  one.globals = m.globals;
  one.functions.push_back(f);
  const std::string text = printModule(one);
  int64_t lat[28];
  for (int k = 0; k <= int(Opcode::Barrier); ++k) lat[k] = lm.latency(Opcode(k));
  darm_gpu_program *p = nullptr;
  char err[512] = {0};
  if (darm_gpu_program_load(text.c_str(), lat, &p, err, sizeof err) != DARM_OK)
    throw std::runtime_error(std::string("darm_gpu: ") + err);
  const int W = ins[0].warpSize;
  const int64_t n = int64_t(ins.size());
  int64_t gw = 0, sw = 0;
  darm_gpu_program_shape(p, nullptr, nullptr, nullptr, &gw, &sw);
  const size_t np = f.params.size();
  std::vector<int32_t> args(np * size_t(n) * W);
  std::vector<int32_t> gl(size_t(n * gw), 0), sh(size_t(n * sw), 0);
  for (int64_t w = 0; w < n; ++w) {
    const WarpInput &in = ins[size_t(w)];
    if (in.warpSize != W) throw std::runtime_error("darm::gpu::executeWarpsIR: mixed warp sizes");
    for (size_t q = 0; q < np; ++q)
      for (int l = 0; l < W; ++l) args[q * n * W + w * W + l] = in.args[q].size() == 1 ? in.args[q][0] : in.args[q].at(size_t(l));
    int64_t off = 0;
    for (const auto &g : m.globals) {
      auto it = in.globalInit.find(g.name);
      if (it != in.globalInit.end()) std::copy(it->second.begin(), it->second.end(), gl.begin() + w * gw + off);
      off += g.size;
    }
    off = 0;
    for (const auto &s : f.sharedDecls) {
      auto it = in.sharedInit.find(s.name);
      if (it != in.sharedInit.end()) std::copy(it->second.begin(), it->second.end(), sh.begin() + w * sw + off);
      off += s.size;
    }
  }
  std::vector<int32_t> rets(static_cast<size_t>(n * W)), faults(static_cast<size_t>(n));
  std::vector<uint8_t> valid(static_cast<size_t>(n * W));
  std::vector<int64_t> st(static_cast<size_t>(n * 8));
  const int rc = darm_gpu_program_execute(p, W, n, args.data(), n * W, gl.data(), sw ? sh.data() : nullptr,
                                          rets.data(), valid.data(), faults.data(), st.data(), maxSteps,
                                          DARM_MEM_HOST, nullptr, nullptr, err, sizeof err);
  darm_gpu_program_free(p);
  if (rc == DARM_USER_ERROR) throw std::runtime_error(std::string("darm_gpu: ") + err);
  if (rc != DARM_OK) throw std::logic_error(std::string("darm_gpu: ") + err);
  for (int64_t w = 0; w < n; ++w) {
    WarpResult &r = out[size_t(w)];
    r.returns.assign(size_t(W), std::nullopt);
    for (int l = 0; l < W; ++l)
      if (valid[size_t(w * W + l)]) r.returns[size_t(l)] = rets[size_t(w * W + l)];
    int64_t off = 0;
    for (const auto &g : m.globals) {
      r.globalFinal[g.name] = std::vector<int32_t>(gl.begin() + w * gw + off, gl.begin() + w * gw + off + g.size);
      off += g.size;
    }
    off = 0;
    for (const auto &s : f.sharedDecls) {
      r.sharedFinal[s.name] = std::vector<int32_t>(sh.begin() + w * sw + off, sh.begin() + w * sw + off + s.size);
      off += s.size;
    }
    for (int i = 0; i < faults[size_t(w)]; ++i) r.faults.push_back({-1, "", "fault on the GPU"});
    const int64_t *s8 = st.data() + w * 8;
    r.stats.issuedInstructions = s8[0];
    r.stats.threadCycles = s8[1];
    r.stats.usefulThreadCycles = s8[2];
    r.stats.serializedCycles = s8[3];
    r.stats.divergentBranchCount = s8[4];
    r.stats.sharedMemIssues = s8[5];
    r.stats.globalMemIssues = s8[6];
    r.stats.utilization = s8[1] == 0 ? 1.0 : double(s8[2]) / double(s8[1]);
    r.nonTerminated = s8[7] & 1;
    r.taintedObservable = (s8[7] & 2) != 0;
    if (r.taintedObservable) r.taintNote = "undef-derived value observed (GPU interpreter)";
  }
  return out;
}

// The result oracle on the GPU: the reference's testing::oracleCompare
// (tests/helpers.hpp:156-174) — makeRandomInput fixtures seed .. seed +
// fixtures - 1 at each warp size, both functions run, compareRuns per fixture —
// with the two executeWarp loops replaced by one executeWarpsIR batch each.
// Returns "" when every verdict is equal, else the first diff as the
// reference formats it.
inline std::string oracleCompare(const Module &m1, const Function &f1, const Module &m2, const Function &f2,
                                 int fixtures, uint64_t seed, const std::vector<int> &warps = {4, 8, 32}) {
  const LatencyModel lm = LatencyModel::defaults();
  for (int w : warps) {
    std::vector<WarpInput> ins;
    for (int i = 0; i < fixtures; ++i) ins.push_back(makeRandomInput(m1, f1, w, seed + uint64_t(i)));
    auto a = executeWarpsIR(m1, f1, ins, lm);
    auto b = executeWarpsIR(m2, f2, ins, lm);
    for (int i = 0; i < fixtures; ++i) {
      CompareVerdict v = compareRuns(a[size_t(i)], b[size_t(i)]);
      if (!v.equal) return f1.name + " warp " + std::to_string(w) + " fixture " + std::to_string(i) + ": " + v.diff;
    }
  }
  return "";
}

}  // namespace gpu
}  // namespace darm
