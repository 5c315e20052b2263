// common.cu -- library identity and error bookkeeping for the C ABI.
#include <cstring>

#include "../../include/hull3d_b200.h"
#include "h3d_host.h"

#include <atomic>

static thread_local char g_last_error[256] = "";
static std::atomic<long long> g_launches{0};

void h3d_count_launches(int k) { g_launches.fetch_add(k, std::memory_order_relaxed); }

bool h3d_check(cudaError_t e) {
  if (e == cudaSuccess) return false;
  std::strncpy(g_last_error, cudaGetErrorString(e), sizeof(g_last_error) - 1);
  return true;
}

extern "C" const char *h3d_impl(void) { return "b200"; }
extern "C" const char *h3d_last_error(void) { return g_last_error; }
extern "C" int64_t h3d_launch_count(void) { return g_launches.load(); }

// ------------------------------------------------------------ level profile
#include <mutex>
#include <vector>

namespace {
struct ProfRec {
  int level, pass;
  cudaEvent_t e0, e1;
};
std::mutex g_prof_mu;
bool g_prof_on = false;
std::vector<ProfRec> g_prof;
std::vector<cudaEvent_t> g_ev_free;  // recycled events (creation is not free)

cudaEvent_t ev_get() {
  {
    std::lock_guard<std::mutex> g(g_prof_mu);
    if (!g_ev_free.empty()) {
      cudaEvent_t e = g_ev_free.back();
      g_ev_free.pop_back();
      return e;
    }
  }
  cudaEvent_t e;
  return cudaEventCreate(&e) == cudaSuccess ? e : nullptr;
}
}  // namespace

bool h3d_profiling() { return g_prof_on; }

void *h3d_prof_begin(cudaStream_t s) {
  cudaEvent_t e = ev_get();
  if (e) cudaEventRecord(e, s);
  return e;
}

void h3d_prof_end(void *e0, int level, int pass, cudaStream_t s) {
  if (!e0) return;
  cudaEvent_t e1 = ev_get();
  if (!e1) return;
  cudaEventRecord(e1, s);
  std::lock_guard<std::mutex> g(g_prof_mu);
  g_prof.push_back({level, pass, static_cast<cudaEvent_t>(e0), e1});
}

extern "C" void h3d_profile_enable(int32_t on) {
  std::lock_guard<std::mutex> g(g_prof_mu);
  g_prof_on = on != 0;
}

extern "C" int64_t h3d_profile_collect(int32_t *level, int32_t *pass, float *ms, int64_t max) {
  std::lock_guard<std::mutex> g(g_prof_mu);
  int64_t m = 0;
  // every record is on one stream: waiting for the last end event covers all
  if (!g_prof.empty()) cudaEventSynchronize(g_prof.back().e1);
  for (auto &r : g_prof) {
    if (m < max) {
      float t = 0.f;
      cudaEventElapsedTime(&t, r.e0, r.e1);
      level[m] = r.level;
      pass[m] = r.pass;
      ms[m] = t;
      ++m;
    }
    g_ev_free.push_back(r.e0);
    g_ev_free.push_back(r.e1);
  }
  g_prof.clear();
  return m;
}
