// h3d_host.h -- host-side helpers shared by the C-ABI translation units.
#pragma once
#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>

// records the error string for h3d_last_error(); returns true on failure
bool h3d_check(cudaError_t e);
// counts this library's own kernel launches (bench.py reports gpu_launches)
void h3d_count_launches(int k);
// every host synchronisation of the library goes through here (counted:
// bench.py reports host_syncs per step)
cudaError_t h3d_sync(cudaStream_t s);
// per-level CUDA-event profile (h3d_profile_enable); no-ops when disabled.
// Mode 1: every level bracketed (measurement + routing + kernels); mode 2:
// only the lane-per-job kernel launches (h3d_prof_kernels()), for bench.py's
// roofline of the dominant kernel.
bool h3d_profiling();
bool h3d_prof_kernels();
void *h3d_prof_begin(cudaStream_t s);
void h3d_prof_end(void *e0, int level, int pass, cudaStream_t s);
void h3d_prof_drop(void *e0);
// per-level DEVICE time stamps (h3d_profile_stamps): the calling thread's
// device buffer of H3D_STAMPS int64 (ns, %globaltimer) or nullptr; slot l =
// start of level l's work, slot H3D_STAMP_END = end of the last level.  The
// level kernels write them (no host work, no event records); the route of
// each level is kept host-side (h3d_stamp_route).
constexpr int H3D_STAMPS = 64;
constexpr int H3D_STAMP_END = 40;
long long *h3d_stamp_buf();
void h3d_stamp_route(int level, int tag);
void h3d_stamp_now(cudaStream_t s, int slot);  // one tiny kernel

inline unsigned h3d_grid(long long work, int block) {
  long long g = (work + block - 1) / block;
  if (g < 1) g = 1;
  if (g > 0x7fffffffll) g = 0x7fffffffll;
  return static_cast<unsigned>(g);
}

// bump allocator over a caller-provided workspace (the library never
// allocates on the fused path); every carve is 256-byte aligned
struct h3d_arena {
  char *base;
  size_t size, used;
  h3d_arena(void *p, size_t n) : base(static_cast<char *>(p)), size(n), used(0) {}
  template <class T>
  T *take(size_t count) {
    size_t bytes = (count * sizeof(T) + 255) & ~size_t(255);
    if (base == nullptr) {  // sizing pass
      used += bytes;
      return nullptr;
    }
    if (used + bytes > size) return nullptr;
    T *p = reinterpret_cast<T *>(base + used);
    used += bytes;
    return p;
  }
};
