// prof.cu — launch counter and optional per-kernel CUDA-event timing (tracing subsystem).
//
// Every kernel launch of libtango goes through a ProfScope: it always increments a global launch
// counter (tango_launch_count) and, when profiling is enabled, brackets the launch with two CUDA
// events on the launching stream.  tango_profile_collect() waits for the recorded events and
// accumulates per-kernel device time; bench.py reads it to compute the live roofline fraction of
// the dominant kernel over the timed region.  With tango_nvtx_enable(1) (or TANGO_NVTX=1) every launch is
// also an NVTX range named after the kernel (header-only NVTX v3), for timeline tools.
#include <atomic>
#include <cstdlib>
#include <nvtx3/nvToolsExt.h>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/tango.h"
#include "kernels.h"

namespace tango {
namespace {
struct Entry { std::string name; double ms = 0.0; int64_t count = 0; };
struct Pending { int entry; cudaEvent_t a, b; };
std::mutex g_mu;
std::vector<Entry> g_entries;
std::vector<Pending> g_pending;
std::vector<cudaEvent_t> g_pool;
std::atomic<bool> g_enabled{false};
std::atomic<int> g_nvtx{-1};   // -1: not yet read from the environment
bool nvtx_on() {
  int v = g_nvtx.load(std::memory_order_relaxed);
  if (v < 0) {
    const char* e = getenv("TANGO_NVTX");
    v = (e && atoi(e)) ? 1 : 0;
    g_nvtx.store(v);
  }
  return v != 0;
}
std::atomic<int64_t> g_launches{0};

cudaEvent_t take_event() {
  if (!g_pool.empty()) { cudaEvent_t e = g_pool.back(); g_pool.pop_back(); return e; }
  cudaEvent_t e = nullptr;
  cudaEventCreate(&e);
  return e;
}
int entry_of(const char* name) {
  for (size_t i = 0; i < g_entries.size(); ++i)
    if (g_entries[i].name == name) return (int)i;
  g_entries.push_back(Entry{name});
  return (int)g_entries.size() - 1;
}
}  // namespace

ProfScope::ProfScope(const char* name, cudaStream_t st) : st_(st) {
  g_launches.fetch_add(1, std::memory_order_relaxed);
  nvtx_ = nvtx_on();
  if (nvtx_) nvtxRangePushA(name);
  on_ = g_enabled.load(std::memory_order_relaxed);
  if (on_) {
    std::lock_guard<std::mutex> lk(g_mu);
    entry_ = entry_of(name);
    a_ = take_event();
    b_ = take_event();
    cudaEventRecord(a_, st_);
  }
}
ProfScope::~ProfScope() {
  if (nvtx_) nvtxRangePop();
  if (on_) {
    cudaEventRecord(b_, st_);
    std::lock_guard<std::mutex> lk(g_mu);
    g_pending.push_back(Pending{entry_, a_, b_});
  }
}

}  // namespace tango

using namespace tango;

extern "C" {

void tango_profile_enable(int32_t on) { g_enabled.store(on != 0); }

void tango_nvtx_enable(int32_t on) { g_nvtx.store(on != 0 ? 1 : 0); }

int64_t tango_launch_count(void) { return g_launches.load(); }

tango_status tango_profile_collect(void) {
  std::lock_guard<std::mutex> lk(g_mu);
  tango_status st = TANGO_OK;
  for (const Pending& p : g_pending) {
    float ms = 0.0f;
    if (cudaEventSynchronize(p.b) != cudaSuccess || cudaEventElapsedTime(&ms, p.a, p.b) != cudaSuccess)
      st = TANGO_ERR_CUDA;
    g_entries[p.entry].ms += ms;
    g_entries[p.entry].count += 1;
    g_pool.push_back(p.a);
    g_pool.push_back(p.b);
  }
  g_pending.clear();
  return st;
}

int32_t tango_profile_num_entries(void) {
  std::lock_guard<std::mutex> lk(g_mu);
  return (int32_t)g_entries.size();
}

tango_status tango_profile_entry(int32_t i, char* name, int32_t name_cap, double* total_ms, int64_t* launches) {
  std::lock_guard<std::mutex> lk(g_mu);
  if (i < 0 || i >= (int32_t)g_entries.size() || !name || name_cap <= 0) return TANGO_ERR_INVALID_ARG;
  strncpy(name, g_entries[i].name.c_str(), (size_t)name_cap - 1);
  name[name_cap - 1] = 0;
  if (total_ms) *total_ms = g_entries[i].ms;
  if (launches) *launches = g_entries[i].count;
  return TANGO_OK;
}

void tango_profile_reset(void) {
  std::lock_guard<std::mutex> lk(g_mu);
  for (Entry& e : g_entries) { e.ms = 0.0; e.count = 0; }
}

}  // extern "C"
