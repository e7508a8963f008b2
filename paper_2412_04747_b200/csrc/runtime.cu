// Library runtime: thread-local errors, allocator fallback, launch counting,
// CUDA-event kernel profiling (rgnn_profile_*).
#include <atomic>
#include <cstdio>
#include <cstring>
#include <map>
#include <mutex>

#include "common.cuh"

namespace rgnn {

static thread_local std::string g_last_error;
void set_error(const std::string& m) { g_last_error = m; }
void clear_error() { g_last_error.clear(); }

void* Allocator::get(size_t bytes, cudaStream_t s) const {
  void* p = nullptr;
  if (alloc) {
    p = alloc(bytes, (void*)s, ctx);
    RGNN_CHECK(p != nullptr, RGNN_ERR_OOM, "allocator callback returned NULL for " + std::to_string(bytes) + " bytes");
  } else {
    cudaError_t e = cudaMallocAsync(&p, bytes, s);
    if (e != cudaSuccess) {
      cudaGetLastError();
      RGNN_FAIL(RGNN_ERR_OOM, "cudaMallocAsync(" + std::to_string(bytes) + "): " + cudaGetErrorString(e));
    }
  }
  return p;
}

void Allocator::put(void* p, cudaStream_t s) const {
  if (!p) return;
  if (free_fn) free_fn(p, (void*)s, ctx);
  else cudaFreeAsync(p, s);
}

struct Side {
  cudaStream_t stream = nullptr;
  cudaEvent_t fork = nullptr, join = nullptr;
  int device = -1;
};
static thread_local Side g_side;

cudaStream_t fork_side(cudaStream_t s) {
  int dev = 0;
  RGNN_CUDA(cudaGetDevice(&dev));
  if (g_side.stream == nullptr || g_side.device != dev) {
    RGNN_CUDA(cudaStreamCreateWithFlags(&g_side.stream, cudaStreamNonBlocking));
    RGNN_CUDA(cudaEventCreateWithFlags(&g_side.fork, cudaEventDisableTiming));
    RGNN_CUDA(cudaEventCreateWithFlags(&g_side.join, cudaEventDisableTiming));
    g_side.device = dev;
  }
  RGNN_CUDA(cudaEventRecord(g_side.fork, s));
  RGNN_CUDA(cudaStreamWaitEvent(g_side.stream, g_side.fork, 0));
  return g_side.stream;
}

void join_side(cudaStream_t s) {
  RGNN_CUDA(cudaEventRecord(g_side.join, g_side.stream));
  RGNN_CUDA(cudaStreamWaitEvent(s, g_side.join, 0));
}

const char* intern(const std::string& name) {
  static std::mutex mu;
  static std::map<std::string, std::string> table;
  std::lock_guard<std::mutex> lk(mu);
  auto it = table.find(name);
  if (it == table.end()) it = table.emplace(name, name).first;
  return it->second.c_str();
}

static std::atomic<int64_t> g_launches{0};
void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

struct ProfRec {
  const char* name;
  cudaEvent_t a, b;
};
struct ProfStat {
  int64_t launches = 0;
  double ms = 0.0;
};
static std::mutex g_pmu;
static bool g_prof = false;
static std::vector<ProfRec> g_pending;
static std::vector<cudaEvent_t> g_pool;
static std::map<std::string, ProfStat> g_stats;

static cudaEvent_t take_event() {
  if (!g_pool.empty()) {
    cudaEvent_t e = g_pool.back();
    g_pool.pop_back();
    return e;
  }
  cudaEvent_t e;
  RGNN_CUDA(cudaEventCreate(&e));
  return e;
}

void profile_begin(const char* name, cudaStream_t s, int* slot) {
  if (!g_prof) return;
  std::lock_guard<std::mutex> lk(g_pmu);
  ProfRec r{name, take_event(), take_event()};
  RGNN_CUDA(cudaEventRecord(r.a, s));
  g_pending.push_back(r);
  *slot = (int)g_pending.size() - 1;
}

void profile_end(int slot, cudaStream_t s) {
  if (slot < 0) return;
  std::lock_guard<std::mutex> lk(g_pmu);
  RGNN_CUDA(cudaEventRecord(g_pending[slot].b, s));
}

static void drain_locked() {
  for (auto& r : g_pending) {
    RGNN_CUDA(cudaEventSynchronize(r.b));
    float ms = 0.f;
    RGNN_CUDA(cudaEventElapsedTime(&ms, r.a, r.b));
    auto& st = g_stats[r.name];
    st.launches += 1;
    st.ms += ms;
    g_pool.push_back(r.a);
    g_pool.push_back(r.b);
  }
  g_pending.clear();
}

}  // namespace rgnn

using namespace rgnn;

extern "C" {

const char* rgnn_last_error(void) { return g_last_error.c_str(); }

const char* rgnn_version(void) {
  return "librgnn 0.1 (sm_100a; CUDA " RGNN_STR(__CUDACC_VER_MAJOR__) "." RGNN_STR(__CUDACC_VER_MINOR__) ")";
}

int64_t rgnn_launch_count(void) { return g_launches.load(); }

rgnn_status rgnn_profile_enable(int32_t on) {
  return guarded([&] {
    std::lock_guard<std::mutex> lk(g_pmu);
    if (!on) drain_locked();
    g_prof = on != 0;
  });
}

rgnn_status rgnn_profile_reset(void) {
  return guarded([&] {
    std::lock_guard<std::mutex> lk(g_pmu);
    drain_locked();
    g_stats.clear();
  });
}

rgnn_status rgnn_profile_read(char* buf, size_t len) {
  return guarded([&] {
    RGNN_CHECK(buf && len > 2, RGNN_ERR_INVALID_ARG, "buffer too small");
    std::lock_guard<std::mutex> lk(g_pmu);
    drain_locked();
    std::string out = "{";
    bool first = true;
    for (auto& kv : g_stats) {
      char tmp[256];
      snprintf(tmp, sizeof(tmp), "%s\"%s\": {\"launches\": %lld, \"ms\": %.6f}", first ? "" : ", ", kv.first.c_str(),
               (long long)kv.second.launches, kv.second.ms);
      out += tmp;
      first = false;
    }
    out += "}";
    RGNN_CHECK(out.size() + 1 <= len, RGNN_ERR_INVALID_ARG, "buffer too small for profile JSON");
    memcpy(buf, out.c_str(), out.size() + 1);
  });
}

}  // extern "C"
