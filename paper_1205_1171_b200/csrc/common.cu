// common.cu -- library identity and error bookkeeping for the C ABI.
#include <cstring>

#include "../../include/hull3d_b200.h"
#include "h3d_host.h"

#include <atomic>

static thread_local char g_last_error[256] = "";
static std::atomic<long long> g_launches{0};

void h3d_count_launches(int k) { g_launches.fetch_add(k, std::memory_order_relaxed); }

static std::atomic<long long> g_syncs{0};
cudaError_t h3d_sync(cudaStream_t s) {
  g_syncs.fetch_add(1, std::memory_order_relaxed);
  return cudaStreamSynchronize(s);
}
extern "C" int64_t h3d_sync_count(void) { return g_syncs.load(); }

bool h3d_check(cudaError_t e) {
  if (e == cudaSuccess) return false;
  std::strncpy(g_last_error, cudaGetErrorString(e), sizeof(g_last_error) - 1);
  return true;
}

extern "C" const char *h3d_impl(void) { return "b200"; }
extern "C" const char *h3d_last_error(void) { return g_last_error; }
extern "C" int64_t h3d_launch_count(void) { return g_launches.load(); }

// ------------------------------------------------------------ level profile
// Per-level CUDA-event profile.  The records and the on/off switch belong to
// the calling THREAD (a hull runs on its caller's thread; two threads driving
// two devices never see each other's records), and recycled events are pooled
// per DEVICE (an event may only be recorded on a stream of its own device).
#include <map>
#include <mutex>
#include <vector>

namespace {
struct ProfRec {
  int level, pass, device;
  cudaEvent_t e0, e1;
};
thread_local bool t_prof_on = false;
thread_local std::vector<ProfRec> t_prof;
thread_local int t_prof_dev = -1;  // device of the pending begin event
std::mutex g_pool_mu;
std::map<int, std::vector<cudaEvent_t>> g_ev_free;  // per device

cudaEvent_t ev_get(int dev) {
  {
    std::lock_guard<std::mutex> g(g_pool_mu);
    auto &v = g_ev_free[dev];
    if (!v.empty()) {
      cudaEvent_t e = v.back();
      v.pop_back();
      return e;
    }
  }
  cudaEvent_t e;
  return cudaEventCreate(&e) == cudaSuccess ? e : nullptr;
}

void ev_put(int dev, cudaEvent_t e) {
  std::lock_guard<std::mutex> g(g_pool_mu);
  g_ev_free[dev].push_back(e);
}
}  // namespace

thread_local int t_prof_mode = 0;
thread_local long long *t_stamps = nullptr;
thread_local int t_routes[H3D_STAMPS];

bool h3d_profiling() { return t_prof_mode == 1; }
bool h3d_prof_kernels() { return t_prof_mode == 2; }
long long *h3d_stamp_buf() { return t_stamps; }
void h3d_stamp_route(int level, int tag) {
  if (t_stamps && level >= 0 && level < H3D_STAMPS) t_routes[level] = tag;
}

__global__ void k_stamp(long long *buf, int slot) {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  buf[slot] = static_cast<long long>(t);
}
void h3d_stamp_now(cudaStream_t s, int slot) {
  if (!t_stamps) return;
  h3d_count_launches(1);
  k_stamp<<<1, 1, 0, s>>>(t_stamps, slot);
}

extern "C" void h3d_profile_stamps(int64_t *dev_buf) {
  t_stamps = reinterpret_cast<long long *>(dev_buf);
  if (dev_buf)  // a new recording starts; switching off keeps the routes for h3d_profile_routes
    for (int &r : t_routes) r = -1;
}
extern "C" int64_t h3d_profile_routes(int32_t *out, int64_t max) {
  int64_t m = 0;
  for (; m < max && m < H3D_STAMPS; ++m) out[m] = t_routes[m];
  return m;
}

void *h3d_prof_begin(cudaStream_t s) {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return nullptr;
  cudaEvent_t e = ev_get(dev);
  if (e) {
    cudaEventRecord(e, s);
    t_prof_dev = dev;
  }
  return e;
}

void h3d_prof_end(void *e0, int level, int pass, cudaStream_t s) {
  if (!e0) return;
  const int dev = t_prof_dev;
  cudaEvent_t e1 = ev_get(dev);
  if (!e1) {
    ev_put(dev, static_cast<cudaEvent_t>(e0));
    return;
  }
  cudaEventRecord(e1, s);
  t_prof.push_back({level, pass, dev, static_cast<cudaEvent_t>(e0), e1});
}

// an interval that turned out empty (the route declined): back to the pool
void h3d_prof_drop(void *e0) {
  if (e0) ev_put(t_prof_dev, static_cast<cudaEvent_t>(e0));
}

extern "C" void h3d_profile_enable(int32_t on) {
  t_prof_on = on != 0;
  t_prof_mode = on < 0 ? 0 : (on > 2 ? 1 : on);
}

extern "C" int64_t h3d_profile_collect(int32_t *level, int32_t *pass, float *ms, int64_t max) {
  int64_t m = 0;
  // the caller's records are stream-ordered on its own stream: waiting for
  // its last end event covers all of them (nothing else is synchronised)
  if (!t_prof.empty()) cudaEventSynchronize(t_prof.back().e1);
  for (auto &r : t_prof) {
    if (m < max) {
      float t = 0.f;
      cudaEventElapsedTime(&t, r.e0, r.e1);
      level[m] = r.level;
      pass[m] = r.pass;
      ms[m] = t;
      ++m;
    }
    ev_put(r.device, r.e0);
    ev_put(r.device, r.e1);
  }
  t_prof.clear();
  return m;
}
