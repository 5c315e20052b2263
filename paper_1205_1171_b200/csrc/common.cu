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
