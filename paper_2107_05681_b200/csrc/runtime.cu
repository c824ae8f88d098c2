// runtime.cu — the C-ABI of libdarm_gpu.so (include/darm_gpu.h).
//
// Replaces the runtime path of the reference: executeWarp's
// memory initialisation (interp.cpp:342-354) becomes H2D staging into cached
// device buffers, the per-lane interpreter loop (interp.cpp:254-314) becomes a
// kernel launch, and the gather of globalFinal (interp.cpp:366-374) becomes a
// D2H copy.  Errors follow the CLI's exit codes (darm_cli.cpp:25-27).
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <mutex>
#include <random>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include <unistd.h>

#include "../../include/darm_gpu.h"
#include "corpus.cuh"
#include "ir_program.h"
#include "kernels.h"

namespace darm_gpu {
namespace {

struct Error {
  int code;
  std::string msg;
};

[[noreturn]] void user_error(const std::string &m) { throw Error{DARM_USER_ERROR, m}; }

#define DARM_CUDA(x)                                                                       \
  do {                                                                                     \
    cudaError_t e_ = (x);                                                                  \
    if (e_ != cudaSuccess)                                                                 \
      throw ::darm_gpu::Error{DARM_INTERNAL_ERROR, std::string(#x) + ": " + cudaGetErrorString(e_)}; \
  } while (0)

int report(const Error &e, char *err, size_t errlen) {
  if (err && errlen) {
    std::strncpy(err, e.msg.c_str(), errlen - 1);
    err[errlen - 1] = 0;
  }
  return e.code;
}

template <class F>
int guarded(char *err, size_t errlen, F &&f) {
  try {
    f();
    return DARM_OK;
  } catch (const Error &e) {
    return report(e, err, errlen);
  } catch (const std::exception &e) {
    return report(Error{DARM_INTERNAL_ERROR, e.what()}, err, errlen);
  } catch (...) {
    return report(Error{DARM_INTERNAL_ERROR, "unknown exception"}, err, errlen);
  }
}

// ---------------------------------------------------------------- devices
struct GraphEntry {
  int kind, variant;
  const void *ptr;
  int64_t n;
  std::vector<int64_t> params;    // every other recorded parameter, compared exactly
  cudaGraphExec_t exec;
  int launches;
};

struct GraphEntry;
struct DeviceState {
  std::mutex mu;
  int sms = 0;
  std::vector<std::pair<void *, size_t>> slots;  // cached staging buffers
  std::vector<GraphEntry> graphs;                // instantiated launch sequences
  cudaStream_t capture = nullptr;                // private stream for graph capture
  cudaStream_t pipe[3] = {nullptr, nullptr, nullptr};  // HOST-mode pipeline: copy in, compute, copy out
  std::vector<cudaEvent_t> events;               // pipeline events (timing disabled)
};

// HOST-mode pipeline streams and >= count sync events of a device.
void pipeline_resources(DeviceState &st, size_t count) {
  for (auto &p : st.pipe)
    if (!p) DARM_CUDA(cudaStreamCreateWithFlags(&p, cudaStreamNonBlocking));
  while (st.events.size() < count) {
    cudaEvent_t e = nullptr;
    DARM_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    st.events.push_back(e);
  }
}

std::mutex g_mu;
std::vector<DeviceState *> g_devices;

DeviceState &device_state(int *dev_out) {
  int dev = 0;
  DARM_CUDA(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lk(g_mu);
  if (g_devices.empty()) {
    int n = 0;
    DARM_CUDA(cudaGetDeviceCount(&n));
    g_devices.assign(size_t(n), nullptr);
  }
  if (dev >= int(g_devices.size())) throw Error{DARM_INTERNAL_ERROR, "device index out of range"};
  if (!g_devices[dev]) {
    cudaDeviceProp prop{};
    DARM_CUDA(cudaGetDeviceProperties(&prop, dev));
    if (prop.major != 10)
      throw Error{DARM_INTERNAL_ERROR, std::string("device ") + prop.name +
                                           " is not sm_100 (libdarm_gpu is built for sm_100a only)"};
    auto *st = new DeviceState;
    st->sms = prop.multiProcessorCount;
    g_devices[dev] = st;
  }
  if (dev_out) *dev_out = dev;
  return *g_devices[dev];
}

// Staging buffer `slot` of at least `bytes` on the current device.  Callers hold
// st.mu for the duration of the call that uses the slots.
void *slot(DeviceState &st, size_t i, size_t bytes) {
  if (st.slots.size() <= i) st.slots.resize(i + 1, {nullptr, 0});
  auto &s = st.slots[i];
  if (s.second < bytes) {
    // cached graphs may hold the old pointer: drop them all
    for (auto &g : st.graphs) cudaGraphExecDestroy(g.exec);
    st.graphs.clear();
    if (s.first) DARM_CUDA(cudaFree(s.first));
    s.first = nullptr;
    s.second = 0;
    size_t want = bytes < 256 ? 256 : bytes;
    DARM_CUDA(cudaMalloc(&s.first, want));
    s.second = want;
  }
  return s.first;
}

// Event bracket for darm_gpu_stats: t0 | H2D | t1 | kernels | t2 | D2H | t3.
struct Timeline {
  cudaEvent_t ev[4] = {nullptr, nullptr, nullptr, nullptr};
  cudaStream_t s;
  bool on;
  Timeline(cudaStream_t st, bool enabled) : s(st), on(enabled) {
    if (on)
      for (auto &e : ev) DARM_CUDA(cudaEventCreate(&e));
  }
  ~Timeline() {
    for (auto &e : ev)
      if (e) cudaEventDestroy(e);
  }
  void mark(int i) {
    if (on) DARM_CUDA(cudaEventRecord(ev[i], s));
  }
  void mark_on(int i, cudaStream_t other) {
    if (on) DARM_CUDA(cudaEventRecord(ev[i], other));
  }
  void fill(darm_gpu_stats *st) {
    if (!on || !st) return;
    DARM_CUDA(cudaEventSynchronize(ev[3]));
    float a = 0, b = 0, c = 0, d = 0;
    DARM_CUDA(cudaEventElapsedTime(&a, ev[0], ev[1]));
    DARM_CUDA(cudaEventElapsedTime(&b, ev[1], ev[2]));
    DARM_CUDA(cudaEventElapsedTime(&c, ev[2], ev[3]));
    DARM_CUDA(cudaEventElapsedTime(&d, ev[0], ev[3]));
    st->h2d_ms = a;
    st->kernel_ms = b;
    st->d2h_ms = c;
    st->total_ms = d;
  }
};

// Returns the cached executable graph for (kind, variant, ptr, n), recording
// it with `record` on the device's private capture stream the first time.
template <class Rec>
GraphEntry &cached_graph(DeviceState &st, int kind, int variant, const void *ptr, int64_t n, Rec &&record,
                         std::vector<int64_t> params = {}) {
  for (auto &g : st.graphs)
    if (g.kind == kind && g.variant == variant && g.ptr == ptr && g.n == n && g.params == params) return g;
  if (!st.capture) DARM_CUDA(cudaStreamCreateWithFlags(&st.capture, cudaStreamNonBlocking));
  cudaGraph_t graph = nullptr;
  int launches = 0;
  DARM_CUDA(cudaStreamBeginCapture(st.capture, cudaStreamCaptureModeThreadLocal));
  cudaError_t rec = record(st.capture, &launches);
  cudaError_t end = cudaStreamEndCapture(st.capture, &graph);
  DARM_CUDA(rec);
  DARM_CUDA(end);
  cudaGraphExec_t exec = nullptr;
  cudaError_t inst = cudaGraphInstantiate(&exec, graph, 0);
  cudaGraphDestroy(graph);
  DARM_CUDA(inst);
  st.graphs.push_back({kind, variant, ptr, n, std::move(params), exec, launches});
  return st.graphs.back();
}

const CorpusKernelDesc *find_kernel(const char *name) {
  if (!name) return nullptr;
  for (int i = 0; i < kCorpusCount; ++i)
    if (std::strcmp(kCorpus[i].name, name) == 0) return &kCorpus[i];
  return nullptr;
}

}  // namespace
}  // namespace darm_gpu

using namespace darm_gpu;

extern "C" {

int darm_gpu_abi_version(void) { return DARM_GPU_ABI_VERSION; }

int darm_gpu_init(int *n_devices, char *err, size_t errlen) {
  return guarded(err, errlen, [&] {
    int n = 0;
    cudaError_t e = cudaGetDeviceCount(&n);
    if (e != cudaSuccess || n == 0)
      throw Error{DARM_INTERNAL_ERROR, std::string("no CUDA device: ") + cudaGetErrorString(e)};
    if (n_devices) *n_devices = n;
    device_state(nullptr);
  });
}

void darm_gpu_shutdown(void) {
  std::lock_guard<std::mutex> lk(g_mu);
  int cur = 0;
  cudaGetDevice(&cur);
  for (size_t d = 0; d < g_devices.size(); ++d) {
    if (!g_devices[d]) continue;
    cudaSetDevice(int(d));
    for (auto &s : g_devices[d]->slots)
      if (s.first) cudaFree(s.first);
    for (auto &g : g_devices[d]->graphs) cudaGraphExecDestroy(g.exec);
    if (g_devices[d]->capture) cudaStreamDestroy(g_devices[d]->capture);
    delete g_devices[d];
    g_devices[d] = nullptr;
  }
  cudaSetDevice(cur);
}

const char *darm_gpu_kernel_list(void) {
  static std::string list = [] {
    std::string s;
    for (int i = 0; i < kCorpusCount; ++i) {
      if (i) s += ",";
      s += kCorpus[i].name;
    }
    return s;
  }();
  return list.c_str();
}

size_t darm_gpu_kernel_info(const char *kernel, char *out, size_t outlen) {
  const CorpusKernelDesc *d = find_kernel(kernel);
  if (!d) return 0;
  std::string j = std::string("{\"name\":\"") + d->name + "\",\"params\":[";
  for (int p = 0; p < d->n_params; ++p) j += std::string(p ? "," : "") + "\"" + d->params[p] + "\"";
  j += "],\"globals\":[";
  for (int g = 0; g < d->n_globals; ++g)
    j += std::string(g ? "," : "") + "[\"" + d->globals[g].name + "\"," + std::to_string(d->globals[g].size) + "]";
  j += "],\"shared\":[";
  for (int s = 0; s < d->n_shared; ++s)
    j += std::string(s ? "," : "") + "[\"" + d->shared[s].name + "\"," + std::to_string(d->shared[s].size) + "]";
  j += "],\"lane_bytes\":" + std::to_string(d->lane_bytes) + "}";
  if (out && outlen) {
    size_t n = j.size() < outlen - 1 ? j.size() : outlen - 1;
    std::memcpy(out, j.data(), n);
    out[n] = 0;
  }
  return j.size() + 1;
}

// makeRandomInput (fixtures.cpp:82-108), one std::mt19937_64 stream per warp.
int darm_gpu_make_random_input(const char *kernel, int warp, int64_t n_warps, uint64_t seed0,
                               int32_t *args, int32_t *const *globals, int64_t gstride,
                               int32_t *const *shared, char *err, size_t errlen) {
  return guarded(err, errlen, [&] {
    const CorpusKernelDesc *d = find_kernel(kernel);
    if (!d) user_error(std::string("unknown kernel '") + (kernel ? kernel : "") + "'");
    if (warp < 1 || warp > 64) user_error("warp size must be in [1, 64]");
    if (n_warps < 0) user_error("n_warps must be >= 0");
    for (int g = 0; g < d->n_globals; ++g)
      if (gstride < 0 || gstride > d->globals[g].size) user_error("gstride exceeds a declared global size");
    auto work = [&](int64_t lo, int64_t hi) {
      for (int64_t w = lo; w < hi; ++w) {
        std::mt19937_64 rng(seed0 + uint64_t(w));
        auto word = [&] { return int32_t(rng() % 257) - 128; };
        for (int p = 0; p < d->n_params; ++p) {
          const char c = d->params[p][0];
          int32_t v;
          if (c == 'j' || c == 'k') {
            int maxShift = 0;
            while ((1 << (maxShift + 1)) <= warp) ++maxShift;
            v = 1 << int(rng() % uint64_t(maxShift + 1));
          } else {
            v = int32_t(rng() % uint64_t(2 * warp));
          }
          if (args) args[p * n_warps + w] = v;
        }
        for (int g = 0; g < d->n_globals; ++g)
          for (int i = 0; i < d->globals[g].size; ++i) {
            int32_t v = word();
            if (i < gstride && globals && globals[g]) globals[g][w * gstride + i] = v;
          }
        for (int s = 0; s < d->n_shared; ++s)
          for (int i = 0; i < d->shared[s].size; ++i) {
            int32_t v = word();
            if (shared && shared[s]) shared[s][w * d->shared[s].size + i] = v;
          }
      }
    };
    unsigned hw = std::thread::hardware_concurrency();
    int64_t nt = hw ? hw : 1;
    if (n_warps < 4096) nt = 1;
    std::vector<std::thread> pool;
    int64_t chunk = (n_warps + nt - 1) / (nt ? nt : 1);
    for (int64_t i = 1; i < nt; ++i) {
      int64_t lo = i * chunk, hi = std::min<int64_t>(n_warps, lo + chunk);
      if (lo < hi) pool.emplace_back(work, lo, hi);
    }
    work(0, std::min<int64_t>(n_warps, chunk));
    for (auto &t : pool) t.join();
  });
}

int darm_gpu_execute_warps(const char *kernel, int variant, int warp, int64_t n_warps,
                           const int32_t *args, int64_t acount, int32_t *const *globals,
                           int n_globals, const int32_t *const *shared, int n_shared,
                           int32_t *faults, int mem, void *stream, darm_gpu_stats *stats,
                           char *err, size_t errlen) {
  return guarded(err, errlen, [&] {
    const CorpusKernelDesc *d = find_kernel(kernel);
    if (!d) user_error(std::string("unknown kernel '") + (kernel ? kernel : "") + "'");
    if (variant != DARM_UNMELDED && variant != DARM_MELDED && variant != DARM_PREDICATED)
      user_error("variant must be 0 (unmelded), 1 (melded) or 2 (predicated)");
    if (warp < 1 || warp > 64) user_error("warp size must be in [1, 64]");  // interp.cpp:334-335
    if (n_warps < 0) user_error("n_warps must be >= 0");
    if (n_warps * int64_t(warp) >= (int64_t(1) << 31)) user_error("too many lanes (limit 2^31)");
    if (n_globals != d->n_globals)
      user_error("expected " + std::to_string(d->n_globals) + " global arrays, got " + std::to_string(n_globals));
    if (shared && n_shared != d->n_shared)
      user_error("expected " + std::to_string(d->n_shared) + " shared arrays, got " + std::to_string(n_shared));
    const int64_t lanes = n_warps * warp;
    int am;
    if (acount == 1) am = 0;
    else if (acount == n_warps) am = 1;
    else if (acount == lanes) am = 2;
    else user_error("argument count must be 1, n_warps or n_warps*warp");  // interp.cpp:348-350
    if (d->n_params && !args) user_error("args is NULL");
    if (mem != DARM_MEM_HOST && mem != DARM_MEM_DEVICE) user_error("mem must be HOST or DEVICE");
    for (int g = 0; g < n_globals; ++g)
      if (!globals || !globals[g]) user_error("global array is NULL");
    if (stats) std::memset(stats, 0, sizeof(*stats));

    DeviceState &st = device_state(nullptr);
    std::lock_guard<std::mutex> lk(st.mu);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    Timeline tl(s, stats != nullptr);
    tl.mark(0);

    CorpusParams P{};
    P.warp = uint32_t(warp);
    P.total = uint32_t(lanes);
    P.n_warps = uint32_t(n_warps);
    P.shared_size = d->n_shared ? uint32_t(d->shared[0].size) : 0;
    const size_t gbytes = size_t(lanes) * 4;
    const size_t sbytes = size_t(n_warps) * P.shared_size * 4;
    uint64_t h2d = 0, d2h = 0;
    size_t si = 0;
    if (am == 0) {
      for (int p = 0; p < d->n_params; ++p) P.argv[p] = args[p];  // broadcast: host scalars
    } else if (mem == DARM_MEM_HOST) {
      auto *dev = static_cast<int32_t *>(slot(st, si++, size_t(acount) * d->n_params * 4));
      DARM_CUDA(cudaMemcpyAsync(dev, args, size_t(acount) * d->n_params * 4, cudaMemcpyHostToDevice, s));
      h2d += size_t(acount) * d->n_params * 4;
      for (int p = 0; p < d->n_params; ++p) P.argp[p] = dev + size_t(p) * acount;
    } else {
      for (int p = 0; p < d->n_params; ++p) P.argp[p] = args + size_t(p) * acount;
    }
    for (int g = 0; g < n_globals; ++g) {
      if (mem == DARM_MEM_HOST) {
        P.gl[g] = static_cast<int32_t *>(slot(st, si++, gbytes));
        if (gbytes) DARM_CUDA(cudaMemcpyAsync(P.gl[g], globals[g], gbytes, cudaMemcpyHostToDevice, s));
        h2d += gbytes;
      } else {
        P.gl[g] = globals[g];
      }
    }
    if (d->n_shared && shared && shared[0]) {
      if (mem == DARM_MEM_HOST) {
        auto *dev = static_cast<int32_t *>(slot(st, si++, sbytes));
        if (sbytes) DARM_CUDA(cudaMemcpyAsync(dev, shared[0], sbytes, cudaMemcpyHostToDevice, s));
        h2d += sbytes;
        P.sh = dev;
      } else {
        P.sh = shared[0];
      }
    }
    int32_t *dfaults = nullptr;
    if (faults || d->n_shared) {
      dfaults = (mem == DARM_MEM_DEVICE && faults) ? faults
                                                   : static_cast<int32_t *>(slot(st, si++, size_t(n_warps) * 4));
      if (n_warps) DARM_CUDA(cudaMemsetAsync(dfaults, 0, size_t(n_warps) * 4, s));
    }
    P.faults = dfaults;
    tl.mark(1);
    if (lanes) {
      DARM_CUDA(d->launch(variant, am, P, st.sms, s));
      if (stats) stats->launches = 1;
    }
    tl.mark(2);
    if (mem == DARM_MEM_HOST) {
      for (int g = 0; g < n_globals; ++g) {
        if (gbytes) DARM_CUDA(cudaMemcpyAsync(globals[g], P.gl[g], gbytes, cudaMemcpyDeviceToHost, s));
        d2h += gbytes;
      }
      if (faults && n_warps) {
        DARM_CUDA(cudaMemcpyAsync(faults, dfaults, size_t(n_warps) * 4, cudaMemcpyDeviceToHost, s));
        d2h += size_t(n_warps) * 4;
      }
    }
    tl.mark(3);
    if (mem == DARM_MEM_HOST) DARM_CUDA(cudaStreamSynchronize(s));
    if (stats) {
      tl.fill(stats);
      stats->h2d_bytes = h2d;
      stats->d2h_bytes = d2h;
      stats->algorithmic_bytes = uint64_t(lanes) * d->lane_bytes + sbytes;
    }
  });
}

int darm_gpu_bitonic_sort(int variant, int32_t *keys, int64_t n, int bucket, int mem, void *stream,
                          darm_gpu_stats *stats, char *err, size_t errlen) {
  return darm_gpu_bitonic_sort_ex(variant, keys, n, bucket, 0, mem, stream, stats, err, errlen);
}

using NetworkLaunch = cudaError_t (*)(int, int32_t *, int64_t, int, int, cudaStream_t, int *);

// Bucket sorts built from a one-warp network step (bitonic.ir, oddeven_step.ir):
// argument checks, HOST-mode staging (pipelined for large inputs), stats.
// max_bucket / max_threads: the largest bucket and threads per bucket the
// network's kernels take (bitonic 4096 / 256: buckets may span warps; PCM
// 1024 / 32).
static int network_sort(NetworkLaunch launch, int max_bucket, int max_threads, int max_variant, int variant,
                        int32_t *keys,
                        int64_t n, int bucket, int keys_per_thread, int mem, void *stream, darm_gpu_stats *stats,
                        char *err, size_t errlen) {
  return guarded(err, errlen, [&] {
    if (variant < DARM_UNMELDED || variant > max_variant)
      user_error("variant must be 0 (unmelded), 1 (melded), 2 (predicated)" +
                 std::string(max_variant >= DARM_MELDED_LITERAL ? " or 3 (melded literal)" : ""));
    if (!bitonic_sort_supported(bucket) || bucket > max_bucket)
      user_error("bucket must be a power of two in [2, " + std::to_string(max_bucket) + "]");
    if (n < 0 || n % bucket) user_error("n must be a non-negative multiple of the bucket size");
    if (n >= (int64_t(1) << 31)) user_error("too many keys (limit 2^31 - 1)");
    if (n && !keys) user_error("keys is NULL");
    if (mem != DARM_MEM_HOST && mem != DARM_MEM_DEVICE) user_error("mem must be HOST or DEVICE");
    // HOST mode stages through a cudaMalloc'd (aligned) buffer
    const int kpt =
        bitonic_keys_per_thread(bucket, keys_per_thread, mem == DARM_MEM_DEVICE ? keys : nullptr, max_threads);
    if (kpt < 0)
      user_error("keys_per_thread must be 0, 1 (bucket <= 1024), 4, 8 or 16, with bucket / keys_per_thread <= " +
                 std::to_string(max_threads) + " and 16-byte aligned keys");
    if (stats) std::memset(stats, 0, sizeof(*stats));
    DeviceState &st = device_state(nullptr);
    std::lock_guard<std::mutex> lk(st.mu);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    Timeline tl(s, stats != nullptr);
    const size_t bytes = size_t(n) * 4;
    int32_t *dk = keys;
    int launches = 0;
    // HOST mode, large inputs: chunks pipelined over three streams so the
    // host->device copy of chunk i+1, the sort of chunk i and the
    // device->host copy of chunk i-1 overlap (the buckets are independent).
    const int64_t chunk = int64_t(1) << 21;   // keys (8 MiB), a multiple of every bucket and warp tile
    if (mem == DARM_MEM_HOST && n >= 2 * chunk) {
      dk = static_cast<int32_t *>(slot(st, 0, bytes));
      const int64_t nc = (n + chunk - 1) / chunk;
      pipeline_resources(st, size_t(2 * nc + 2));
      cudaStream_t in = st.pipe[0], comp = st.pipe[1], out = st.pipe[2];
      cudaEvent_t start = st.events[0], done = st.events[1];
      tl.mark(0);
      DARM_CUDA(cudaEventRecord(start, s));                 // after the caller's prior work on s
      DARM_CUDA(cudaStreamWaitEvent(in, start, 0));
      DARM_CUDA(cudaStreamWaitEvent(comp, start, 0));
      DARM_CUDA(cudaStreamWaitEvent(out, start, 0));
      for (int64_t c = 0; c < nc; ++c) {
        const int64_t off = c * chunk, len = std::min(chunk, n - off);
        cudaEvent_t copied = st.events[2 + 2 * c], sorted = st.events[3 + 2 * c];
        DARM_CUDA(cudaMemcpyAsync(dk + off, keys + off, size_t(len) * 4, cudaMemcpyHostToDevice, in));
        DARM_CUDA(cudaEventRecord(copied, in));
        DARM_CUDA(cudaStreamWaitEvent(comp, copied, 0));
        if (c == 0) tl.mark_on(1, comp);
        DARM_CUDA(launch(variant, dk + off, len, bucket, kpt, comp, &launches));
        DARM_CUDA(cudaEventRecord(sorted, comp));
        if (c == nc - 1) tl.mark_on(2, comp);
        DARM_CUDA(cudaStreamWaitEvent(out, sorted, 0));
        DARM_CUDA(cudaMemcpyAsync(keys + off, dk + off, size_t(len) * 4, cudaMemcpyDeviceToHost, out));
      }
      DARM_CUDA(cudaEventRecord(done, out));
      DARM_CUDA(cudaStreamWaitEvent(s, done, 0));
      tl.mark(3);
      DARM_CUDA(cudaStreamSynchronize(s));
    } else {
      tl.mark(0);
      if (mem == DARM_MEM_HOST) {
        dk = static_cast<int32_t *>(slot(st, 0, bytes));
        if (bytes) DARM_CUDA(cudaMemcpyAsync(dk, keys, bytes, cudaMemcpyHostToDevice, s));
      }
      tl.mark(1);
      DARM_CUDA(launch(variant, dk, n, bucket, kpt, s, &launches));
      tl.mark(2);
      if (mem == DARM_MEM_HOST && bytes) DARM_CUDA(cudaMemcpyAsync(keys, dk, bytes, cudaMemcpyDeviceToHost, s));
      tl.mark(3);
      if (mem == DARM_MEM_HOST) DARM_CUDA(cudaStreamSynchronize(s));
    }
    if (stats) {
      tl.fill(stats);
      stats->launches = launches;
      stats->h2d_bytes = mem == DARM_MEM_HOST ? bytes : 0;
      stats->d2h_bytes = mem == DARM_MEM_HOST ? bytes : 0;
      stats->algorithmic_bytes = 2 * bytes;
      stats->reserved = kpt;
    }
  });
}

int darm_gpu_bitonic_sort_ex(int variant, int32_t *keys, int64_t n, int bucket, int keys_per_thread, int mem,
                             void *stream, darm_gpu_stats *stats, char *err, size_t errlen) {
  return network_sort(launch_bitonic_sort, 4096, 256, DARM_MELDED_LITERAL, variant, keys, n, bucket, keys_per_thread, mem, stream, stats, err,
                      errlen);
}

int darm_gpu_oddeven_sort(int variant, int32_t *keys, int64_t n, int bucket, int keys_per_thread, int mem,
                          void *stream, darm_gpu_stats *stats, char *err, size_t errlen) {
  return network_sort(launch_oddeven_sort, 1024, 32, DARM_PREDICATED, variant, keys, n, bucket, keys_per_thread, mem, stream, stats, err,
                      errlen);
}

int darm_gpu_merge_sort(int variant, int32_t *keys, int64_t n, int mem, void *stream, darm_gpu_stats *stats,
                        char *err, size_t errlen) {
  return guarded(err, errlen, [&] {
    if (variant != DARM_UNMELDED && variant != DARM_MELDED) user_error("variant must be 0 (unmelded) or 1 (melded)");
    if (n < 0 || n >= (int64_t(1) << 30)) user_error("n must be in [0, 2^30)");
    if (n && !keys) user_error("keys is NULL");
    if (mem != DARM_MEM_HOST && mem != DARM_MEM_DEVICE) user_error("mem must be HOST or DEVICE");
    if (stats) std::memset(stats, 0, sizeof(*stats));
    DeviceState &st = device_state(nullptr);
    std::lock_guard<std::mutex> lk(st.mu);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const size_t bytes = size_t(n) * 4;
    Timeline tl(s, stats != nullptr);
    tl.mark(0);
    int32_t *dk = keys;
    if (mem == DARM_MEM_HOST) {
      dk = static_cast<int32_t *>(slot(st, 0, bytes));
      if (bytes) DARM_CUDA(cudaMemcpyAsync(dk, keys, bytes, cudaMemcpyHostToDevice, s));
    }
    auto *tmp = static_cast<int32_t *>(slot(st, 8, bytes));
    int launches = 0;
    tl.mark(1);
    if (n > 1) {
      GraphEntry &g = cached_graph(st, 4, variant, dk, n, [&](cudaStream_t cs, int *l) {
        return record_merge_sort(variant, dk, tmp, n, cs, l);
      });
      DARM_CUDA(cudaGraphLaunch(g.exec, s));
      launches = g.launches;
    }
    tl.mark(2);
    if (mem == DARM_MEM_HOST && bytes) DARM_CUDA(cudaMemcpyAsync(keys, dk, bytes, cudaMemcpyDeviceToHost, s));
    tl.mark(3);
    if (mem == DARM_MEM_HOST) DARM_CUDA(cudaStreamSynchronize(s));
    if (stats) {
      tl.fill(stats);
      stats->launches = launches;
      stats->h2d_bytes = mem == DARM_MEM_HOST ? bytes : 0;
      stats->d2h_bytes = mem == DARM_MEM_HOST ? bytes : 0;
      stats->algorithmic_bytes = uint64_t(merge_sort_passes(n)) * 2 * bytes;
    }
  });
}

// N-Queens prefixes: every valid placement of the first `base` rows, lowest
// free column first; prefix i goes to rank i % world.
// symmetric: row 0 only in the columns < ceil(n/2) (mirror symmetry; the
// placements with the row-0 queen left of the middle count twice, the middle
// column of an odd n once); *n_double receives how many of the kept prefixes
// (they come first) carry the factor 2.
static void nqueens_prefixes(int n, int base, int rank, int world, std::vector<uint32_t> &out,
                             bool symmetric = false, int64_t *n_double = nullptr) {
  const uint32_t mask = n >= 32 ? 0xffffffffu : ((1u << n) - 1u);
  uint32_t cols[32], d1[32], d2[32], av[32];
  int row = 0;
  cols[0] = d1[0] = d2[0] = 0;
  av[0] = symmetric ? ((1u << ((n + 1) / 2)) - 1u) : mask;
  const uint32_t left = (1u << (n / 2)) - 1u;   // row-0 columns that count twice
  int64_t dbl = 0;
  uint32_t first = 0;                           // the row-0 queen
  uint64_t idx = 0;
  while (row >= 0) {
    if (av[row] == 0) {
      --row;
      continue;
    }
    const uint32_t bit = av[row] & (0u - av[row]);
    av[row] ^= bit;
    if (row == 0) first = bit;
    const uint32_t c = cols[row] | bit, e1 = (d1[row] | bit) << 1, e2 = (d2[row] | bit) >> 1;
    if (row + 1 == base) {
      if (int(idx % uint64_t(world)) == rank) {
        out.push_back(c);
        out.push_back(e1);
        out.push_back(e2);
        if (symmetric && (first & left)) ++dbl;
      }
      ++idx;
      continue;
    }
    ++row;
    cols[row] = c;
    d1[row] = e1;
    d2[row] = e2;
    av[row] = ~(c | e1 | e2) & mask;
  }
  if (n_double) *n_double = dbl;
}

int64_t darm_gpu_nqueens_prefix_count(int n, int prefix_rows, int rank, int world) {
  return darm_gpu_nqueens_prefix_count_ex(n, prefix_rows, rank, world, 0);
}

int64_t darm_gpu_nqueens_prefix_count_ex(int n, int prefix_rows, int rank, int world, int flags) {
  if (n < 2 || n > 31 || prefix_rows < 1 || prefix_rows > n - 1 || world < 1 || rank < 0 || rank >= world ||
      (flags & ~(DARM_NQ_MIRROR | DARM_NQ_PAPER_SHAPE)))
    return -1;
  std::vector<uint32_t> pre;
  nqueens_prefixes(n, prefix_rows, rank, world, pre, (flags & DARM_NQ_MIRROR) != 0);
  return int64_t(pre.size() / 3);
}

int darm_gpu_nqueens(int variant, int n, int prefix_rows, int rank, int world, uint64_t *solutions,
                     uint32_t *per_prefix, int64_t per_prefix_len, int64_t *n_prefixes, void *stream,
                     darm_gpu_stats *stats, char *err, size_t errlen) {
  return darm_gpu_nqueens_ex(variant, n, prefix_rows, rank, world, 0, solutions, per_prefix, per_prefix_len,
                             n_prefixes, stream, stats, err, errlen);
}

int darm_gpu_nqueens_ex(int variant, int n, int prefix_rows, int rank, int world, int flags, uint64_t *solutions,
                        uint32_t *per_prefix, int64_t per_prefix_len, int64_t *n_prefixes, void *stream,
                        darm_gpu_stats *stats, char *err, size_t errlen) {
  return guarded(err, errlen, [&] {
    if (flags & ~(DARM_NQ_MIRROR | DARM_NQ_PAPER_SHAPE)) user_error("unknown n-queens flags");
    const bool paper_shape = (flags & DARM_NQ_PAPER_SHAPE) != 0;
    if (paper_shape && n > 16) user_error("the paper-shaped encoding (DARM_NQ_PAPER_SHAPE) takes n <= 16");
    if (variant != DARM_UNMELDED && variant != DARM_MELDED) user_error("variant must be 0 (unmelded) or 1 (melded)");
    if (n < 2 || n > 31) user_error("n must be in [2, 31]");
    if (prefix_rows < 1 || prefix_rows > n - 1) user_error("prefix_rows must be in [1, n-1]");
    if (world < 1 || rank < 0 || rank >= world) user_error("need 0 <= rank < world");
    if (!solutions) user_error("solutions is NULL");
    if (stats) std::memset(stats, 0, sizeof(*stats));
    std::vector<uint32_t> pre;
    int64_t n_double = 0;
    nqueens_prefixes(n, prefix_rows, rank, world, pre, (flags & DARM_NQ_MIRROR) != 0, &n_double);
    const int64_t np = int64_t(pre.size() / 3);
    if (n_prefixes) *n_prefixes = np;
    if (np >= (int64_t(1) << 32) - 1) user_error("too many prefixes; lower prefix_rows");
    if (per_prefix && per_prefix_len < np) user_error("per_prefix buffer too small");
    DeviceState &st = device_state(nullptr);
    std::lock_guard<std::mutex> lk(st.mu);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    Timeline tl(s, stats != nullptr);
    tl.mark(0);
    auto *dpre = static_cast<uint32_t *>(slot(st, 0, pre.size() * 4));
    auto *dctl = static_cast<unsigned long long *>(slot(st, 1, 16));
    uint32_t *dper = per_prefix ? static_cast<uint32_t *>(slot(st, 2, size_t(np) * 4)) : nullptr;
    if (!pre.empty()) DARM_CUDA(cudaMemcpyAsync(dpre, pre.data(), pre.size() * 4, cudaMemcpyHostToDevice, s));
    DARM_CUDA(cudaMemsetAsync(dctl, 0, 16, s));
    tl.mark(1);
    if (np) DARM_CUDA(launch_nqueens(variant, dpre, uint32_t(np), uint32_t(n_double), n, prefix_rows, dper, dctl,
                                     reinterpret_cast<unsigned int *>(dctl + 1), st.sms, s, paper_shape));
    tl.mark(2);
    unsigned long long total = 0;
    DARM_CUDA(cudaMemcpyAsync(&total, dctl, 8, cudaMemcpyDeviceToHost, s));
    if (per_prefix && np) DARM_CUDA(cudaMemcpyAsync(per_prefix, dper, size_t(np) * 4, cudaMemcpyDeviceToHost, s));
    tl.mark(3);
    DARM_CUDA(cudaStreamSynchronize(s));
    *solutions = total;
    if (stats) {
      tl.fill(stats);
      stats->launches = np ? 1 : 0;
      stats->h2d_bytes = pre.size() * 4;
      stats->d2h_bytes = 8 + (per_prefix ? uint64_t(np) * 4 : 0);
      stats->algorithmic_bytes = pre.size() * 4 + (per_prefix ? uint64_t(np) * 4 : 0);
    }
  });
}

int darm_gpu_lud(int variant, float *a, int64_t n, int mem, void *stream, darm_gpu_stats *stats, char *err,
                 size_t errlen) {
  return guarded(err, errlen, [&] {
    if (variant != DARM_UNMELDED && variant != DARM_MELDED) user_error("variant must be 0 (unmelded) or 1 (melded)");
    if (n < 16 || n % 16 || n > 46336) user_error("n must be a multiple of 16 in [16, 46336]");
    if (!a) user_error("matrix is NULL");
    if (mem != DARM_MEM_HOST && mem != DARM_MEM_DEVICE) user_error("mem must be HOST or DEVICE");
    if (mem == DARM_MEM_DEVICE && (reinterpret_cast<uintptr_t>(a) & 15)) user_error("device matrix must be 16-byte aligned");
    if (stats) std::memset(stats, 0, sizeof(*stats));
    DeviceState &st = device_state(nullptr);
    std::lock_guard<std::mutex> lk(st.mu);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const size_t bytes = size_t(n) * size_t(n) * 4;
    Timeline tl(s, stats != nullptr);
    tl.mark(0);
    float *d = a;
    if (mem == DARM_MEM_HOST) {
      d = static_cast<float *>(slot(st, 0, bytes));
      DARM_CUDA(cudaMemcpyAsync(d, a, bytes, cudaMemcpyHostToDevice, s));
    }
    // factored diagonals, then the trailing-update launches' tile counters
    const size_t diag_words = size_t(n / 16) * 256;
    auto *dscr = static_cast<float *>(
        slot(st, 7, (diag_words + size_t(darm_gpu::lud_counter_words(int(n)))) * sizeof(float)));
    int *counters = reinterpret_cast<int *>(dscr + diag_words);
    GraphEntry &g = cached_graph(st, 1, variant, d, n, [&](cudaStream_t cs, int *launches) {
      return record_lud(variant, d, int(n), dscr, counters, cs, launches);
    });
    tl.mark(1);
    DARM_CUDA(cudaGraphLaunch(g.exec, s));
    tl.mark(2);
    if (mem == DARM_MEM_HOST) DARM_CUDA(cudaMemcpyAsync(a, d, bytes, cudaMemcpyDeviceToHost, s));
    tl.mark(3);
    if (mem == DARM_MEM_HOST) DARM_CUDA(cudaStreamSynchronize(s));
    if (stats) {
      tl.fill(stats);
      stats->launches = g.launches;
      stats->h2d_bytes = mem == DARM_MEM_HOST ? bytes : 0;
      stats->d2h_bytes = mem == DARM_MEM_HOST ? bytes : 0;
      // internal update reads + writes the trailing matrix once per step
      double nb = double(n) / 16.0, tb = 0;
      for (double m = nb - 1; m > 0; m -= 1) tb += m * m;
      stats->algorithmic_bytes = uint64_t(tb * 16.0 * 16.0 * 8.0);
    }
  });
}

static uint32_t float_bits(float f) {
  uint32_t u;
  std::memcpy(&u, &f, 4);
  return u;
}

static void check_srad_args(int64_t rows, int64_t cols, const int *roi, float lambda) {
  if (rows < 1 || cols < 2 || rows > (1 << 20) || cols > (1 << 20) || rows * cols > (int64_t(1) << 34))
    user_error("image must be rows x cols with rows >= 1, cols >= 2");
  if (!roi) user_error("roi is NULL");
  if (roi[0] < 0 || roi[1] < roi[0] || roi[1] >= rows || roi[2] < 0 || roi[3] < roi[2] || roi[3] >= cols)
    user_error("roi must be {r1, r2, c1, c2} inside the image with r1 <= r2, c1 <= c2");
  if (roi[1] - roi[0] + 1 > 4096) user_error("roi spans more than 4096 rows");
  if (!(lambda > 0.0f) || !(lambda <= 1.0f)) user_error("lambda must be in (0, 1]");
}

int64_t darm_gpu_srad_roi_words(int64_t cols, const int *roi) {
  if (!roi || cols < 1) return -1;
  SradRoi R = srad_roi_layout(int(cols), roi[0], roi[1], roi[2], roi[3]);
  return int64_t(R.rows) * R.groups * 2;
}

static void check_srad_variant(int variant) {
  if ((variant & ~DARM_FAST_MATH) != DARM_UNMELDED && (variant & ~DARM_FAST_MATH) != DARM_MELDED)
    user_error("variant must be 0 (unmelded) or 1 (melded), optionally | DARM_FAST_MATH");
}

int darm_gpu_srad(int variant, float *j, int64_t rows, int64_t cols, int iters, float lambda, const int *roi,
                  int mem, void *stream, darm_gpu_stats *stats, char *err, size_t errlen) {
  return guarded(err, errlen, [&] {
    check_srad_variant(variant);
    check_srad_args(rows, cols, roi, lambda);
    if (iters < 0) user_error("iters must be >= 0");
    if (!j) user_error("image is NULL");
    if (mem != DARM_MEM_HOST && mem != DARM_MEM_DEVICE) user_error("mem must be HOST or DEVICE");
    if (stats) std::memset(stats, 0, sizeof(*stats));
    DeviceState &st = device_state(nullptr);
    std::lock_guard<std::mutex> lk(st.mu);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const SradRoi R = srad_roi_layout(int(cols), roi[0], roi[1], roi[2], roi[3]);
    const int pitch = srad_pitch(int(cols));
    const size_t img = size_t(rows) * size_t(cols) * 4;
    const size_t buf = size_t(rows + 3) * size_t(pitch) * 4;   // 1 halo row above, 2 below
    const size_t roi_bytes = size_t(R.rows) * R.groups * 2 * 8;
    auto *b0 = static_cast<float *>(slot(st, 0, buf));
    auto *b1 = static_cast<float *>(slot(st, 1, buf));
    auto *ctl = static_cast<char *>(slot(st, 2, 2 * roi_bytes + 256));
    double *roiA = reinterpret_cast<double *>(ctl + 256), *roiB = roiA + roi_bytes / 8;
    Timeline tl(s, stats != nullptr);
    tl.mark(0);
    if (pitch != cols) {   // defined pad columns (never stored to the image, but read as neighbours' lanes)
      DARM_CUDA(cudaMemsetAsync(b0, 0, buf, s));
      DARM_CUDA(cudaMemsetAsync(b1, 0, buf, s));
    }
    const cudaMemcpyKind kin = mem == DARM_MEM_HOST ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice;
    DARM_CUDA(cudaMemcpy2DAsync(b0 + pitch, size_t(pitch) * 4, j, size_t(cols) * 4, size_t(cols) * 4, size_t(rows),
                                kin, s));
    tl.mark(1);
    const int it = iters;
    const SradRange all{0, int(rows), 0, 0};
    GraphEntry &g = cached_graph(st, 16, variant, b0, it, [&](cudaStream_t cs, int *launches) {
      cudaError_t e = launch_srad_roi(b0, int(cols), pitch, 0, int(rows), R, roiA, cs);
      ++*launches;
      float *in = b0, *out = b1;
      double *ri = roiA, *ro = roiB;
      for (int t = 0; t < it && e == cudaSuccess; ++t) {
        e = launch_srad_sweep(variant, in, out, ri, nullptr, ro, int(cols), pitch, int(rows), 0, int(rows), lambda, R,
                              all, cs);
        ++*launches;
        std::swap(in, out);
        std::swap(ri, ro);
      }
      return e;
    }, {rows, cols, roi[0], roi[1], roi[2], roi[3], int64_t(float_bits(lambda))});
    DARM_CUDA(cudaGraphLaunch(g.exec, s));
    tl.mark(2);
    float *res = (iters % 2 == 0) ? b0 : b1;
    const cudaMemcpyKind kout = mem == DARM_MEM_HOST ? cudaMemcpyDeviceToHost : cudaMemcpyDeviceToDevice;
    DARM_CUDA(cudaMemcpy2DAsync(j, size_t(cols) * 4, res + pitch, size_t(pitch) * 4, size_t(cols) * 4,
                                size_t(rows), kout, s));
    tl.mark(3);
    if (mem == DARM_MEM_HOST) DARM_CUDA(cudaStreamSynchronize(s));
    if (stats) {
      tl.fill(stats);
      stats->launches = g.launches;
      stats->h2d_bytes = mem == DARM_MEM_HOST ? img : 0;
      stats->d2h_bytes = mem == DARM_MEM_HOST ? img : 0;
      stats->algorithmic_bytes = uint64_t(iters) * uint64_t(rows) * uint64_t(cols) * 8;
    }
  });
}

static void check_srad_tile(int64_t rows, int64_t cols, int64_t pitch, int64_t tile_rows, int64_t r0) {
  if (tile_rows < 1 || r0 < 0 || r0 + tile_rows > rows) user_error("tile outside the image");
  if (pitch < cols || pitch % 4) user_error("pitch must be >= cols and a multiple of 4 floats");
  if ((tile_rows + 3) * pitch >= (int64_t(1) << 40)) user_error("tile too large");
}

int64_t darm_gpu_srad_pitch(int64_t cols) { return cols < 1 ? -1 : int64_t(srad_pitch(int(cols))); }

int darm_gpu_srad_tile_roi(const float *tile, int64_t cols, int64_t pitch, int64_t tile_rows, int64_t r0,
                           int64_t rows, const int *roi, double *roi_out, void *stream, char *err, size_t errlen) {
  return guarded(err, errlen, [&] {
    check_srad_args(rows, cols, roi, 0.5f);
    check_srad_tile(rows, cols, pitch, tile_rows, r0);
    if (!tile || !roi_out) user_error("NULL buffer");
    if (reinterpret_cast<uintptr_t>(tile) & 15) user_error("tile must be 16-byte aligned");
    device_state(nullptr);
    const SradRoi R = srad_roi_layout(int(cols), roi[0], roi[1], roi[2], roi[3]);
    DARM_CUDA(cudaMemsetAsync(roi_out, 0, size_t(R.rows) * R.groups * 2 * sizeof(double),
                              static_cast<cudaStream_t>(stream)));
    DARM_CUDA(launch_srad_roi(tile, int(cols), int(pitch), int(r0), int(tile_rows), R, roi_out,
                              static_cast<cudaStream_t>(stream)));
  });
}

// own rows that need no halo row: [1, tile_rows - 2) (output row i reads rows i-1 .. i+2)
static SradRange srad_part_range(int part, int n) {
  if (part == DARM_SRAD_ALL_ROWS || n <= 3) {
    if (part == DARM_SRAD_INTERIOR_ROWS) return SradRange{0, 0, 0, 0};
    return SradRange{0, n, 0, 0};
  }
  if (part == DARM_SRAD_INTERIOR_ROWS) return SradRange{1, n - 2, 0, 0};
  return SradRange{0, 1, n - 2, n};   // DARM_SRAD_EDGE_ROWS
}

int darm_gpu_srad_tile_step(int variant, const float *tile_in, float *tile_out, int64_t cols, int64_t pitch,
                            int64_t tile_rows, int64_t r0, int64_t rows, float lambda, const int *roi,
                            const double *roi_in, double *roi_out, float *q0_scratch, int part, void *stream,
                            char *err, size_t errlen) {
  return guarded(err, errlen, [&] {
    check_srad_variant(variant);
    check_srad_args(rows, cols, roi, lambda);
    check_srad_tile(rows, cols, pitch, tile_rows, r0);
    if (part != DARM_SRAD_ALL_ROWS && part != DARM_SRAD_INTERIOR_ROWS && part != DARM_SRAD_EDGE_ROWS)
      user_error("part must be DARM_SRAD_ALL_ROWS, DARM_SRAD_INTERIOR_ROWS or DARM_SRAD_EDGE_ROWS");
    if (!tile_in || !tile_out || !roi_in || !q0_scratch) user_error("NULL buffer");
    if ((reinterpret_cast<uintptr_t>(tile_in) | reinterpret_cast<uintptr_t>(tile_out)) & 15)
      user_error("tiles must be 16-byte aligned");
    device_state(nullptr);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const SradRoi R = srad_roi_layout(int(cols), roi[0], roi[1], roi[2], roi[3]);
    if (part != DARM_SRAD_EDGE_ROWS && roi_out)   // the first (or only) launch of the iteration
      DARM_CUDA(cudaMemsetAsync(roi_out, 0, size_t(R.rows) * R.groups * 2 * sizeof(double), s));
    DARM_CUDA(launch_srad_sweep(variant, tile_in, tile_out, roi_in, part != DARM_SRAD_EDGE_ROWS ? q0_scratch : nullptr,
                                roi_out, int(cols), int(pitch), int(tile_rows), int(r0), int(rows), lambda, R,
                                srad_part_range(part, int(tile_rows)), s));
  });
}


// ---------------------------------------------------------------- peer-memory SRAD tiles
namespace darm_gpu {
namespace {
struct SradHandle {   // DARM_SRAD_HANDLE_BYTES bytes on the wire
  uint32_t magic;
  int32_t pid, dev, world;
  uint64_t ptr;
  cudaIpcMemHandle_t ipc;
};
static_assert(sizeof(SradHandle) <= DARM_SRAD_HANDLE_BYTES, "handle size");
constexpr uint32_t kSradMagic = 0x53524144u;   // "SRAD"

size_t align256(size_t b) { return (b + 255) & ~size_t(255); }

// every rank's allocation: flags[world] | ROI partials x2 | tile x2
struct SradLayout {
  size_t roi, tile[2], tile_bytes, roi_bytes, total;
};
SradLayout srad_layout(int world, const SradRoi &R, int n, int pitch) {
  SradLayout L;
  L.roi_bytes = align256(size_t(R.rows) * R.groups * 2 * sizeof(double));
  L.tile_bytes = align256(size_t(n + 3) * size_t(pitch) * sizeof(float));
  L.roi = align256(size_t(world) * sizeof(unsigned));
  L.tile[0] = L.roi + 2 * L.roi_bytes;
  L.tile[1] = L.tile[0] + L.tile_bytes;
  L.total = L.tile[1] + L.tile_bytes;
  return L;
}
}  // namespace
}  // namespace darm_gpu

struct darm_gpu_srad_group {
  int variant = 0, rank = 0, world = 1, dev = 0, pitch = 0, cur = 0;
  int64_t rows = 0, cols = 0;
  float lambda = 0.5f;
  int roi[4] = {0, 0, 0, 0};
  darm_gpu::SradRoi R{};
  std::vector<std::pair<int, int>> split;   // (r0, n) per rank
  std::vector<char *> base;                 // every rank's allocation as mapped here
  std::vector<bool> opened;                 // opened through CUDA IPC (closed on free)
  char *own = nullptr;
  // device control block: seq, status, peer flag pointers, ROI partial pointers x2, ROI row owners
  char *ctl = nullptr;
  unsigned *seq = nullptr;
  int *status = nullptr;
  unsigned **peer_flags = nullptr;
  const double **parts[2] = {nullptr, nullptr};
  int *owner = nullptr;
  cudaStream_t capture = nullptr, side = nullptr;
  cudaEvent_t fork = nullptr, join = nullptr;
  struct G {
    int iters, cur;
    cudaGraphExec_t exec;
  };
  std::vector<G> graphs;
  unsigned long long timeout_ns = 60ull * 1000000000ull;
  bool connected = false;

  darm_gpu::SradLayout layout(int k) const { return darm_gpu::srad_layout(world, R, split[k].second, pitch); }
  float *tile(int k, int which) const { return reinterpret_cast<float *>(base[k] + layout(k).tile[which]); }
  double *roi_buf(int k, int which) const {
    const auto L = layout(k);
    return reinterpret_cast<double *>(base[k] + L.roi + size_t(which) * L.roi_bytes);
  }
  unsigned *flags(int k) const { return reinterpret_cast<unsigned *>(base[k]); }
};

using darm_gpu::srad_layout;

int darm_gpu_srad_group_create(int variant, int64_t rows, int64_t cols, float lambda, const int *roi, int rank,
                               int world, darm_gpu_srad_group **out, void *handle_out, char *err, size_t errlen) {
  return guarded(err, errlen, [&] {
    check_srad_variant(variant);
    check_srad_args(rows, cols, roi, lambda);
    if (!out || !handle_out) user_error("out / handle_out is NULL");
    if (world < 1 || world > 64 || rank < 0 || rank >= world) user_error("need 0 <= rank < world <= 64");
    auto g = std::make_unique<darm_gpu_srad_group>();
    g->variant = variant;
    g->rank = rank;
    g->world = world;
    g->rows = rows;
    g->cols = cols;
    g->lambda = lambda;
    std::memcpy(g->roi, roi, sizeof(g->roi));
    g->R = srad_roi_layout(int(cols), roi[0], roi[1], roi[2], roi[3]);
    g->pitch = srad_pitch(int(cols));
    int64_t r0 = 0;
    for (int k = 0; k < world; ++k) {   // as srad_tiles.split_rows
      const int64_t n = rows / world + (k < rows % world ? 1 : 0);
      if (n < 2) user_error("every rank needs at least 2 image rows");
      g->split.emplace_back(int(r0), int(n));
      r0 += n;
    }
    if (const char *t = std::getenv("DARM_PEER_TIMEOUT_S")) g->timeout_ns = (unsigned long long)(std::atof(t) * 1e9);
    device_state(&g->dev);
    DARM_CUDA(cudaGetDevice(&g->dev));
    const auto L = g->layout(rank);
    DARM_CUDA(cudaMalloc(&g->own, L.total));
    DARM_CUDA(cudaMemset(g->own, 0, L.total));   // flags, partials, halo and pad columns defined
    const size_t ctl_bytes = 256 + size_t(world) * sizeof(void *) * 3 + size_t(g->R.rows) * sizeof(int);
    DARM_CUDA(cudaMalloc(&g->ctl, ctl_bytes));
    DARM_CUDA(cudaMemset(g->ctl, 0, ctl_bytes));
    g->seq = reinterpret_cast<unsigned *>(g->ctl);
    g->status = reinterpret_cast<int *>(g->ctl + 16);
    g->peer_flags = reinterpret_cast<unsigned **>(g->ctl + 256);
    g->parts[0] = reinterpret_cast<const double **>(g->ctl + 256 + size_t(world) * sizeof(void *));
    g->parts[1] = g->parts[0] + world;
    g->owner = reinterpret_cast<int *>(g->ctl + 256 + size_t(world) * sizeof(void *) * 3);
    SradHandle h{};
    h.magic = kSradMagic;
    h.pid = int32_t(getpid());
    h.dev = g->dev;
    h.world = world;
    h.ptr = reinterpret_cast<uint64_t>(g->own);
    DARM_CUDA(cudaIpcGetMemHandle(&h.ipc, g->own));
    std::memset(handle_out, 0, DARM_SRAD_HANDLE_BYTES);
    std::memcpy(handle_out, &h, sizeof(h));
    *out = g.release();
  });
}

int darm_gpu_srad_group_connect(darm_gpu_srad_group *g, const void *handles, char *err, size_t errlen) {
  return guarded(err, errlen, [&] {
    if (!g || !handles) user_error("group / handles is NULL");
    if (g->connected) user_error("group already connected");
    DARM_CUDA(cudaSetDevice(g->dev));
    g->base.assign(size_t(g->world), nullptr);
    g->opened.assign(size_t(g->world), false);
    const char *hb = static_cast<const char *>(handles);
    for (int k = 0; k < g->world; ++k) {
      SradHandle h;
      std::memcpy(&h, hb + size_t(k) * DARM_SRAD_HANDLE_BYTES, sizeof(h));
      if (h.magic != kSradMagic || h.world != g->world) user_error("handle " + std::to_string(k) + " is not a SRAD group handle of this world");
      if (k == g->rank) {
        g->base[k] = g->own;
      } else if (h.pid == int32_t(getpid())) {   // a rank in this process: its pointer as is
        if (h.dev != g->dev) {
          cudaError_t e = cudaDeviceEnablePeerAccess(h.dev, 0);
          if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) DARM_CUDA(e);
          cudaGetLastError();
        }
        g->base[k] = reinterpret_cast<char *>(h.ptr);
      } else {
        void *p = nullptr;
        DARM_CUDA(cudaIpcOpenMemHandle(&p, h.ipc, cudaIpcMemLazyEnablePeerAccess));
        g->base[k] = static_cast<char *>(p);
        g->opened[k] = true;
      }
    }
    std::vector<unsigned *> pf(size_t(g->world));
    std::vector<const double *> parts(2 * size_t(g->world));
    for (int k = 0; k < g->world; ++k) {
      pf[k] = g->flags(k);
      parts[k] = g->roi_buf(k, 0);
      parts[g->world + k] = g->roi_buf(k, 1);
    }
    std::vector<int> owner(size_t(g->R.rows));
    for (int r = 0; r < g->R.rows; ++r) {
      const int row = g->R.r1 + r;
      for (int k = 0; k < g->world; ++k)
        if (row >= g->split[k].first && row < g->split[k].first + g->split[k].second) owner[r] = k;
    }
    DARM_CUDA(cudaMemcpy(g->peer_flags, pf.data(), pf.size() * sizeof(void *), cudaMemcpyHostToDevice));
    DARM_CUDA(cudaMemcpy(g->parts[0], parts.data(), parts.size() * sizeof(void *), cudaMemcpyHostToDevice));
    DARM_CUDA(cudaMemcpy(g->owner, owner.data(), owner.size() * sizeof(int), cudaMemcpyHostToDevice));
    DARM_CUDA(cudaStreamCreateWithFlags(&g->capture, cudaStreamNonBlocking));
    DARM_CUDA(cudaStreamCreateWithFlags(&g->side, cudaStreamNonBlocking));
    DARM_CUDA(cudaEventCreateWithFlags(&g->fork, cudaEventDisableTiming));
    DARM_CUDA(cudaEventCreateWithFlags(&g->join, cudaEventDisableTiming));
    g->connected = true;
  });
}

static void srad_group_ready(const darm_gpu_srad_group *g) {
  if (!g) user_error("group is NULL");
  if (!g->connected) user_error("group not connected");
  DARM_CUDA(cudaSetDevice(g->dev));
}

int darm_gpu_srad_group_load(darm_gpu_srad_group *g, const float *tile, int mem, void *stream, char *err,
                             size_t errlen) {
  return guarded(err, errlen, [&] {
    srad_group_ready(g);
    if (!tile) user_error("tile is NULL");
    if (mem != DARM_MEM_HOST && mem != DARM_MEM_DEVICE) user_error("mem must be HOST or DEVICE");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const int r0 = g->split[g->rank].first, n = g->split[g->rank].second;
    DARM_CUDA(launch_srad_peer_wait(g->flags(g->rank), g->seq, g->rank, g->world, g->timeout_ns, g->status, s));
    float *t = g->tile(g->rank, 0);
    DARM_CUDA(cudaMemcpy2DAsync(t + g->pitch, size_t(g->pitch) * 4, tile, size_t(g->cols) * 4, size_t(g->cols) * 4,
                                size_t(n), mem == DARM_MEM_HOST ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice,
                                s));
    DARM_CUDA(cudaMemsetAsync(g->roi_buf(g->rank, 0), 0, g->layout(g->rank).roi_bytes, s));
    DARM_CUDA(launch_srad_roi(t, int(g->cols), g->pitch, r0, n, g->R, g->roi_buf(g->rank, 0), s));
    DARM_CUDA(launch_srad_peer_signal(g->peer_flags, g->seq, g->rank, g->world, s));
    g->cur = 0;
    if (mem == DARM_MEM_HOST) DARM_CUDA(cudaStreamSynchronize(s));
  });
}

// one iteration from tile buffer `cur` into 1 - cur, recorded on g->capture
static cudaError_t record_srad_group_iteration(darm_gpu_srad_group *g, int cur, int *launches) {
  using namespace darm_gpu;
  cudaStream_t s = g->capture;
  const int r0 = g->split[g->rank].first, n = g->split[g->rank].second;
  const int k = g->rank;
  cudaError_t e = launch_srad_peer_wait(g->flags(k), g->seq, k, g->world, g->timeout_ns, g->status, s);
  if (e != cudaSuccess) return e;
  const bool halo = g->world > 1;
  if (halo) {   // the halo rows come over NVLink while the interior rows run
    if ((e = cudaEventRecord(g->fork, s)) != cudaSuccess) return e;
    if ((e = cudaStreamWaitEvent(g->side, g->fork, 0)) != cudaSuccess) return e;
    const float *up = k > 0 ? g->tile(k - 1, cur) : nullptr;
    const float *down = k + 1 < g->world ? g->tile(k + 1, cur) : nullptr;
    const int up_rows = k > 0 ? g->split[k - 1].second : 0;
    if ((e = launch_srad_peer_halo(g->tile(k, cur), up, up_rows, down, n, g->pitch, g->side)) != cudaSuccess) return e;
    if ((e = cudaEventRecord(g->join, g->side)) != cudaSuccess) return e;
  }
  auto sweep = [&](SradRange range) {
    return launch_srad_sweep(g->variant, g->tile(k, cur), g->tile(k, 1 - cur), nullptr, nullptr,
                             g->roi_buf(k, 1 - cur), int(g->cols), g->pitch, n, r0, int(g->rows), g->lambda, g->R,
                             range, s, g->parts[cur], g->owner);
  };
  const bool split = halo && n > 3;
  if ((e = sweep(split ? SradRange{1, n - 2, 0, 0} : SradRange{0, 0, 0, 0})) != cudaSuccess) return e;
  if (halo && (e = cudaStreamWaitEvent(s, g->join, 0)) != cudaSuccess) return e;
  if ((e = sweep(split ? SradRange{0, 1, n - 2, n} : SradRange{0, n, 0, 0})) != cudaSuccess) return e;
  e = launch_srad_peer_signal(g->peer_flags, g->seq, k, g->world, s);
  *launches += halo ? 5 : 4;
  return e;
}

int darm_gpu_srad_group_run(darm_gpu_srad_group *g, int iters, void *stream, darm_gpu_stats *stats, char *err,
                            size_t errlen) {
  return guarded(err, errlen, [&] {
    srad_group_ready(g);
    if (iters < 0) user_error("iters must be >= 0");
    if (stats) std::memset(stats, 0, sizeof(*stats));
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    darm_gpu_srad_group::G *gr = nullptr;
    for (auto &x : g->graphs)
      if (x.iters == iters && x.cur == g->cur) gr = &x;
    int launches = 0;
    if (!gr) {
      cudaGraph_t graph = nullptr;
      DARM_CUDA(cudaStreamBeginCapture(g->capture, cudaStreamCaptureModeThreadLocal));
      cudaError_t rec = cudaSuccess;
      for (int t = 0, cur = g->cur; t < iters && rec == cudaSuccess; ++t, cur = 1 - cur)
        rec = record_srad_group_iteration(g, cur, &launches);
      cudaError_t end = cudaStreamEndCapture(g->capture, &graph);
      DARM_CUDA(rec);
      DARM_CUDA(end);
      cudaGraphExec_t exec = nullptr;
      cudaError_t inst = cudaGraphInstantiate(&exec, graph, 0);
      cudaGraphDestroy(graph);
      DARM_CUDA(inst);
      g->graphs.push_back({iters, g->cur, exec});
      gr = &g->graphs.back();
    } else {
      launches = iters * (g->world > 1 ? 5 : 4);
    }
    Timeline tl(s, stats != nullptr);
    tl.mark(0);
    tl.mark(1);
    DARM_CUDA(cudaGraphLaunch(gr->exec, s));
    tl.mark(2);
    tl.mark(3);
    g->cur = (g->cur + iters) & 1;
    if (stats) {
      tl.fill(stats);
      stats->launches = launches;
      stats->algorithmic_bytes = uint64_t(iters) * uint64_t(g->split[g->rank].second) * uint64_t(g->cols) * 8;
    }
  });
}

int darm_gpu_srad_group_read(darm_gpu_srad_group *g, float *tile, int mem, void *stream, char *err, size_t errlen) {
  return guarded(err, errlen, [&] {
    srad_group_ready(g);
    if (!tile) user_error("tile is NULL");
    if (mem != DARM_MEM_HOST && mem != DARM_MEM_DEVICE) user_error("mem must be HOST or DEVICE");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const int n = g->split[g->rank].second;
    DARM_CUDA(cudaMemcpy2DAsync(tile, size_t(g->cols) * 4, g->tile(g->rank, g->cur) + g->pitch, size_t(g->pitch) * 4,
                                size_t(g->cols) * 4, size_t(n),
                                mem == DARM_MEM_HOST ? cudaMemcpyDeviceToHost : cudaMemcpyDeviceToDevice, s));
    int status = 0;
    DARM_CUDA(cudaMemcpyAsync(&status, g->status, sizeof(int), cudaMemcpyDeviceToHost, s));
    DARM_CUDA(cudaStreamSynchronize(s));
    if (status) throw Error{DARM_INTERNAL_ERROR, "a peer rank never reached this phase (device wait timed out)"};
  });
}

int darm_gpu_srad_group_rows(const darm_gpu_srad_group *g, int64_t *r0, int64_t *tile_rows) {
  if (!g || !r0 || !tile_rows) return DARM_USER_ERROR;
  *r0 = g->split[g->rank].first;
  *tile_rows = g->split[g->rank].second;
  return DARM_OK;
}

void darm_gpu_srad_group_free(darm_gpu_srad_group *g) {
  if (!g) return;
  cudaSetDevice(g->dev);
  cudaDeviceSynchronize();
  for (auto &x : g->graphs) cudaGraphExecDestroy(x.exec);
  for (size_t k = 0; k < g->base.size(); ++k)
    if (g->opened[k]) cudaIpcCloseMemHandle(g->base[k]);
  if (g->capture) cudaStreamDestroy(g->capture);
  if (g->side) cudaStreamDestroy(g->side);
  if (g->fork) cudaEventDestroy(g->fork);
  if (g->join) cudaEventDestroy(g->join);
  cudaFree(g->ctl);
  cudaFree(g->own);
  delete g;
}

// ---------------------------------------------------------------- mini-IR programs
struct darm_gpu_program {
  darm_gpu::IrProgram prog;
  int device = -1;
  void *dev = nullptr;            // one allocation: blocks, insts, phis, phi_ins, mem tables
  size_t off_insts = 0, off_phis = 0, off_phi_ins = 0, off_mem_off = 0, off_mem_size = 0, off_mem_sh = 0;
};

int darm_gpu_program_load(const char *ir_text, const int64_t *latency, darm_gpu_program **out, char *err,
                          size_t errlen) {
  return guarded(err, errlen, [&] {
    if (!ir_text || !out) user_error("ir_text / out is NULL");
    *out = nullptr;
    auto *p = new darm_gpu_program;
    try {
      p->prog = compile_ir(ir_text);
    } catch (const std::runtime_error &e) {
      delete p;
      user_error(e.what());
    }
    if (int(p->prog.reg_names.size()) > ir_interp_max_regs()) {
      delete p;
      user_error("the GPU interpreter supports at most " + std::to_string(ir_interp_max_regs()) + " values");
    }
    for (const auto &b : p->prog.blocks)
      if (b.n_phi > ir_interp_max_phis()) {
        delete p;
        user_error("the GPU interpreter supports at most " + std::to_string(ir_interp_max_phis()) +
                   " phis per block");
      }
    if (latency)
      for (int k = 0; k < kNumOps; ++k) {
        if (latency[k] <= 0) {
          delete p;
          user_error("latencies must be positive");
        }
        p->prog.latency[k] = latency[k];
      }
    *out = p;
  });
}

void darm_gpu_program_free(darm_gpu_program *p) {
  if (!p) return;
  if (p->dev) {
    int cur = 0;
    cudaGetDevice(&cur);
    cudaSetDevice(p->device);
    cudaFree(p->dev);
    cudaSetDevice(cur);
  }
  delete p;
}

int darm_gpu_program_shape(const darm_gpu_program *p, int *n_params, int *n_globals, int *n_shared,
                           int64_t *global_words, int64_t *shared_words) {
  if (!p) return DARM_USER_ERROR;
  if (n_params) *n_params = int(p->prog.params.size());
  if (n_globals) *n_globals = p->prog.n_globals;
  if (n_shared) *n_shared = p->prog.n_shared;
  if (global_words) *global_words = p->prog.global_words;
  if (shared_words) *shared_words = p->prog.shared_words;
  return DARM_OK;
}

const char *darm_gpu_program_memory(const darm_gpu_program *p, int index, int64_t *size, int64_t *offset,
                                    int *is_shared) {
  if (!p || index < 0 || index >= int(p->prog.mems.size())) return nullptr;
  const auto &m = p->prog.mems[size_t(index)];
  if (size) *size = m.size;
  if (offset) *offset = m.offset;
  if (is_shared) *is_shared = m.shared ? 1 : 0;
  return m.name.c_str();
}

const char *darm_gpu_program_param(const darm_gpu_program *p, int index) {
  if (!p || index < 0 || index >= int(p->prog.params.size())) return nullptr;
  return p->prog.params[size_t(index)].c_str();
}

int darm_gpu_program_execute(darm_gpu_program *p, int warp, int64_t n_warps, const int32_t *args, int64_t acount,
                             int32_t *globals, int32_t *shared, int32_t *returns, uint8_t *ret_valid,
                             int32_t *faults, int64_t *stats_out, int64_t max_steps, int mem, void *stream,
                             darm_gpu_stats *stats, char *err, size_t errlen) {
  return guarded(err, errlen, [&] {
    if (!p) user_error("program is NULL");
    const IrProgram &P = p->prog;
    if (warp < 1 || warp > 64) user_error("warp size must be in [1, 64]");  // interp.cpp:334-335
    if (n_warps < 0) user_error("n_warps must be >= 0");
    const int np = int(P.params.size());
    int am = 0;
    if (np) {
      if (acount == 1) am = 0;
      else if (acount == n_warps) am = 1;
      else if (acount == n_warps * warp) am = 2;
      else user_error("argument count must be 1, n_warps or n_warps*warp");  // interp.cpp:348-350
      if (!args) user_error("args is NULL");
    }
    if (P.global_words && n_warps && !globals) user_error("globals is NULL");
    if (mem != DARM_MEM_HOST && mem != DARM_MEM_DEVICE) user_error("mem must be HOST or DEVICE");
    if (max_steps <= 0) max_steps = 10000000;   // executeWarp's default (interp.hpp:57-58)
    if (stats) std::memset(stats, 0, sizeof(*stats));
    int dev = 0;
    DARM_CUDA(cudaGetDevice(&dev));
    DeviceState &st = device_state(nullptr);
    std::lock_guard<std::mutex> lk(st.mu);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    // program arrays on this device (uploaded once)
    if (!p->dev || p->device != dev) {
      if (p->dev) {
        cudaSetDevice(p->device);
        cudaFree(p->dev);
        cudaSetDevice(dev);
      }
      auto al = [](size_t x) { return (x + 255) & ~size_t(255); };
      size_t o = 0;
      const size_t ob = o; o = al(o + P.blocks.size() * sizeof(IrBlock));
      p->off_insts = o; o = al(o + P.insts.size() * sizeof(IrInst));
      p->off_phis = o; o = al(o + P.phis.size() * sizeof(IrPhi));
      p->off_phi_ins = o; o = al(o + P.phi_ins.size() * sizeof(IrPhiIn));
      p->off_mem_off = o; o = al(o + P.mems.size() * 8);
      p->off_mem_size = o; o = al(o + P.mems.size() * 8);
      p->off_mem_sh = o; o = al(o + P.mems.size() + 1);
      std::vector<char> host(o, 0);
      std::memcpy(host.data() + ob, P.blocks.data(), P.blocks.size() * sizeof(IrBlock));
      if (!P.insts.empty()) std::memcpy(host.data() + p->off_insts, P.insts.data(), P.insts.size() * sizeof(IrInst));
      if (!P.phis.empty()) std::memcpy(host.data() + p->off_phis, P.phis.data(), P.phis.size() * sizeof(IrPhi));
      if (!P.phi_ins.empty())
        std::memcpy(host.data() + p->off_phi_ins, P.phi_ins.data(), P.phi_ins.size() * sizeof(IrPhiIn));
      for (size_t m = 0; m < P.mems.size(); ++m) {
        reinterpret_cast<int64_t *>(host.data() + p->off_mem_off)[m] = P.mems[m].offset;
        reinterpret_cast<int64_t *>(host.data() + p->off_mem_size)[m] = P.mems[m].size;
        reinterpret_cast<uint8_t *>(host.data() + p->off_mem_sh)[m] = P.mems[m].shared;
      }
      DARM_CUDA(cudaMalloc(&p->dev, o));
      DARM_CUDA(cudaMemcpy(p->dev, host.data(), o, cudaMemcpyHostToDevice));
      p->device = dev;
    }
    Timeline tl(s, stats != nullptr);
    tl.mark(0);
    const int64_t gbytes = n_warps * P.global_words * 4, sbytes = n_warps * P.shared_words * 4;
    const int64_t acnt = np ? acount : 0;
    size_t si = 16;   // slots 16.. (the other entry points use the low ones)
    InterpLaunch L{};
    char *base = static_cast<char *>(p->dev);
    L.blocks = base;
    L.insts = base + p->off_insts;
    L.phis = base + p->off_phis;
    L.phi_ins = base + p->off_phi_ins;
    L.mem_off = reinterpret_cast<const int64_t *>(base + p->off_mem_off);
    L.mem_size = reinterpret_cast<const int64_t *>(base + p->off_mem_size);
    L.mem_shared = reinterpret_cast<const uint8_t *>(base + p->off_mem_sh);
    for (int k = 0; k < kNumOps; ++k) L.latency[k] = P.latency[k];
    L.n_params = np;
    L.n_regs = int(P.reg_names.size());
    L.entry = P.entry;
    L.ret_block = P.ret_block;
    L.gwords = P.global_words;
    L.swords = P.shared_words;
    L.W = warp;
    L.n_warps = n_warps;
    L.am = am;
    L.acount = acnt;
    L.max_steps = max_steps;
    L.sms = st.sms;
    uint64_t h2d = 0, d2h = 0;
    auto stage_in = [&](const void *src, size_t bytes) -> void * {
      void *d = slot(st, si++, bytes ? bytes : 4);
      if (bytes) DARM_CUDA(cudaMemcpyAsync(d, src, bytes, cudaMemcpyHostToDevice, s));
      h2d += bytes;
      return d;
    };
    if (mem == DARM_MEM_HOST) {
      L.args = np ? static_cast<const int32_t *>(stage_in(args, size_t(np) * acnt * 4)) : nullptr;
      L.globals = static_cast<int32_t *>(stage_in(globals, size_t(gbytes)));
      if (shared) {
        L.shared = static_cast<int32_t *>(stage_in(shared, size_t(sbytes)));
      } else {
        L.shared = static_cast<int32_t *>(slot(st, si++, sbytes ? size_t(sbytes) : 4));
        if (sbytes) DARM_CUDA(cudaMemsetAsync(L.shared, 0, size_t(sbytes), s));
      }
      L.returns = returns ? static_cast<int32_t *>(slot(st, si++, size_t(n_warps * warp) * 4 + 4)) : nullptr;
      L.ret_valid = ret_valid ? static_cast<uint8_t *>(slot(st, si++, size_t(n_warps * warp) + 4)) : nullptr;
      L.faults = faults ? static_cast<int32_t *>(slot(st, si++, size_t(n_warps) * 4 + 4)) : nullptr;
      L.stats = stats_out ? static_cast<int64_t *>(slot(st, si++, size_t(n_warps) * 64 + 8)) : nullptr;
    } else {
      L.args = args;
      L.globals = globals;
      if (shared) {
        L.shared = shared;
      } else {
        L.shared = static_cast<int32_t *>(slot(st, si++, sbytes ? size_t(sbytes) : 4));
        if (sbytes) DARM_CUDA(cudaMemsetAsync(L.shared, 0, size_t(sbytes), s));
      }
      L.returns = returns;
      L.ret_valid = ret_valid;
      L.faults = faults;
      L.stats = stats_out;
    }
    const size_t tbytes = size_t(n_warps) * size_t(P.global_words + P.shared_words);
    L.taint = static_cast<uint8_t *>(slot(st, si++, tbytes ? tbytes : 4));
    if (tbytes) DARM_CUDA(cudaMemsetAsync(L.taint, 0, tbytes, s));   // initial cells are untainted
    auto *derr = static_cast<int32_t *>(slot(st, si++, size_t(n_warps) * 4 + 4));
    L.errors = derr;
    tl.mark(1);
    DARM_CUDA(launch_ir_interp(L, s));
    tl.mark(2);
    std::vector<int32_t> herr(static_cast<size_t>(n_warps));
    if (n_warps) DARM_CUDA(cudaMemcpyAsync(herr.data(), derr, size_t(n_warps) * 4, cudaMemcpyDeviceToHost, s));
    if (mem == DARM_MEM_HOST) {
      auto back = [&](void *dst, const void *src, size_t bytes) {
        if (dst && bytes) DARM_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, s));
        if (dst) d2h += bytes;
      };
      back(globals, L.globals, size_t(gbytes));
      back(shared, L.shared, size_t(sbytes));
      back(returns, L.returns, size_t(n_warps * warp) * 4);
      back(ret_valid, L.ret_valid, size_t(n_warps * warp));
      back(faults, L.faults, size_t(n_warps) * 4);
      back(stats_out, L.stats, size_t(n_warps) * 64);
    }
    tl.mark(3);
    DARM_CUDA(cudaStreamSynchronize(s));
    for (int64_t w = 0; w < n_warps; ++w)
      if (herr[size_t(w)]) {
        static const char *const what[] = {"", "a phi has no incoming for the lane's predecessor",
                                           "divergent branch without a reconvergence point",
                                           "SIMT stack deeper than the interpreter supports"};
        const int e = herr[size_t(w)];
        user_error("warp " + std::to_string(w) + ": " + (e >= 1 && e <= 3 ? what[e] : "execution error"));
      }
    if (stats) {
      tl.fill(stats);
      stats->launches = n_warps ? 1 : 0;
      stats->h2d_bytes = h2d;
      stats->d2h_bytes = d2h;
      stats->algorithmic_bytes = uint64_t(2 * (gbytes + sbytes));
    }
  });
}

}  // extern "C"
