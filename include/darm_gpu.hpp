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

#include "darm/interp.hpp"
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

}  // namespace gpu
}  // namespace darm
