// seam.cu -- reference-semantics device kernels behind the kernel-module seam.
//
// Each kernel here reproduces one function of pkg/src/hull3d/_ckernels.pyx on
// the reference data layout in HBM (pts (n,3) f64, links (n,2) i32, slots 2n
// i32), so that a forward replay, the merged logs and the link state are
// bit-identical to the reference.  One thread runs one merge job (the
// reference runs one CPU thread per job span, backends.py:56-101); a whole
// level is one launch with the job tiling computed from the thread index
// (plan_level, parallel.py:49-65) instead of a host-built jobs array.
//
// This is the exact / seam path.  The fused fast path (fast.cu) produces the
// same final logs with warp-cooperative merges over compact groups.
#include <cuda_runtime.h>

#include "h3d_device.cuh"
#include "h3d_host.h"

namespace h3d {

__device__ __forceinline__ int act_g(int *K, long long i) {
  const long long lf = K[2 * i], rt = K[2 * i + 1];
  if (lf == NIL || rt == NIL) return -1;
  if (K[2 * lf + 1] == i) {
    K[2 * lf + 1] = static_cast<int>(rt);
    K[2 * rt] = static_cast<int>(lf);
  } else {
    K[2 * lf + 1] = static_cast<int>(i);
    K[2 * rt] = static_cast<int>(i);
  }
  return 0;
}

// _find_bridge (_ckernels.pyx:63-83)
__device__ long long bridge_g(const RowPts &P, const int *K, long long *pu,
                              long long *pv, long long limit) {
  long long u = *pu, v = *pv, moves = 0;
  for (;;) {
    const long long vn = K[2 * v + 1];
    bool moved = false;
    if (vn != NIL && turn_xy(P.x(u), P.y(u), P.x(v), P.y(v), P.x(vn), P.y(vn)) < 0.0) {
      v = vn;
      moved = true;
    } else {
      const long long up = K[2 * u];
      if (up != NIL && turn_xy(P.x(up), P.y(up), P.x(u), P.y(u), P.x(v), P.y(v)) < 0.0) {
        u = up;
        moved = true;
      }
    }
    if (!moved) {
      *pu = u;
      *pv = v;
      return 0;
    }
    if (++moves > limit) return H3D_E_BRIDGE;
  }
}

// _merge_one (_ckernels.pyx:86-208), reference layout, one thread.
__device__ long long merge_g(const RowPts &P, int *K, const int *in, int *out,
                             long long L, long long M, long long R) {
  const long long cap = 2 * (R - L), base = 2 * L;
  long long u = M - 1, v = M, li = 2 * L, ri = 2 * M, k = 0;
  const long long lend = 2 * M, rend = 2 * R;
  double tcur = -INF;
  if (bridge_g(P, K, &u, &v, R - L) < 0) return H3D_E_BRIDGE;

#define H3D_EMIT(e)                                 \
  do {                                              \
    if (k >= cap - 1) return H3D_E_OVERFLOW;        \
    out[base + k] = static_cast<int>(e);            \
    ++k;                                            \
  } while (0)

  for (;;) {
    if (li >= lend || ri >= rend) return H3D_E_UNTERMINATED;
    const long long el = in[li], er = in[ri];
    const double c0 = (el != NIL) ? P.evt(K[2 * el], el, K[2 * el + 1]) : INF;
    const double c1 = (er != NIL) ? P.evt(K[2 * er], er, K[2 * er + 1]) : INF;
    const double c2 = P.evt(u, K[2 * u + 1], v);
    const double c3 = P.evt(K[2 * u], u, v);
    const double c4 = P.evt(u, v, K[2 * v + 1]);
    const double c5 = P.evt(u, K[2 * v], v);
    double best = INF;
    int which = -1;
    if (c0 > tcur && c0 < best) { best = c0; which = 0; }
    if (c1 > tcur && c1 < best) { best = c1; which = 1; }
    if (c2 > tcur && c2 < best) { best = c2; which = 2; }
    if (c3 > tcur && c3 < best) { best = c3; which = 3; }
    if (c4 > tcur && c4 < best) { best = c4; which = 4; }
    if (c5 > tcur && c5 < best) { best = c5; which = 5; }
    if (which < 0) break;
    switch (which) {
      case 0:
        if (el < u) H3D_EMIT(el);  // x strictly increasing: x[e] < x[u] <=> e < u
        if (act_g(K, el) < 0) return H3D_E_CHAIN;
        ++li;
        break;
      case 1:
        if (er > v) H3D_EMIT(er);
        if (act_g(K, er) < 0) return H3D_E_CHAIN;
        ++ri;
        break;
      case 2:
        u = K[2 * u + 1];
        H3D_EMIT(u);
        break;
      case 3:
        H3D_EMIT(u);
        u = K[2 * u];
        break;
      case 4:
        H3D_EMIT(v);
        v = K[2 * v + 1];
        break;
      default:
        v = K[2 * v];
        H3D_EMIT(v);
        break;
    }
    tcur = best;
  }
#undef H3D_EMIT
  out[base + k] = NIL;
  K[2 * u + 1] = static_cast<int>(v);
  K[2 * v] = static_cast<int>(u);
  for (long long idx = k - 1; idx >= 0; --idx) {
    const long long e = out[base + idx];
    if (e <= u || e >= v) {
      if (act_g(K, e) < 0) return H3D_E_CHAIN;
      if (e == u)
        u = K[2 * u];
      else if (e == v)
        v = K[2 * v + 1];
    } else {
      K[2 * u + 1] = static_cast<int>(e);
      K[2 * e] = static_cast<int>(u);
      K[2 * v] = static_cast<int>(e);
      K[2 * e + 1] = static_cast<int>(v);
      if (e < M)
        u = e;
      else
        v = e;
    }
  }
  return k;
}

__device__ long long copy_log_g(const int *src, int *dst, long long off, long long cap) {
  for (long long idx = 0; idx < cap; ++idx) {
    const int e = src[off + idx];
    dst[off + idx] = e;
    if (e == NIL) return idx;
  }
  return H3D_E_UNTERMINATED;
}

__global__ void k_init_base(int *K, int *slots, long long n) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    reinterpret_cast<int2 *>(K)[i] = make_int2(NIL, NIL);
    slots[2 * i] = NIL;
  }
}

// one level of build_movie: group g is a merge job or the trailing carry
__global__ void k_level_exact(RowPts P, int *K, const int *in, int *out,
                              long long n, int level, long long *err) {
  const long long g = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  const long long size = 1ll << level, half = size >> 1;
  const long long L = g << level;
  if (L >= n) return;
  const long long R = (L + size < n) ? L + size : n;
  long long r;
  if (R - L > half)
    r = merge_g(P, K, in, out, L, L + half, R);
  else
    r = copy_log_g(in, out, 2 * L, 2 * n - 2 * L);
  if (r < 0) raise_err(err, r);
}

__global__ void k_merge_range(RowPts P, int *K, const int *in, int *out,
                              const long long *jobs, long long lo, long long hi,
                              long long *err) {
  const long long j = lo + blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (j >= hi) return;
  const long long r = merge_g(P, K, in, out, jobs[3 * j], jobs[3 * j + 1], jobs[3 * j + 2]);
  if (r < 0) raise_err(err, r);
}

// single-thread seam kernels: result in *res
__global__ void k_act(int *K, long long i, long long *res) {
  *res = (act_g(K, i) < 0) ? H3D_E_CHAIN : 0;
}

__global__ void k_find_bridge(RowPts P, const int *K, long long u, long long v,
                              long long limit, long long *res) {
  const long long r = bridge_g(P, K, &u, &v, limit);
  res[0] = (r < 0) ? NIL : u;
  res[1] = (r < 0) ? NIL : v;
}

__global__ void k_merge_one(RowPts P, int *K, const int *in, int *out, long long L,
                            long long M, long long R, long long *res) {
  *res = merge_g(P, K, in, out, L, M, R);
}

__global__ void k_replay(int *K, const int *slots, long long off, long long count,
                         int backward, long long *res) {
  long long r = 0;
  for (long long s = 0; s < count; ++s) {
    const long long e = slots[off + (backward ? count - 1 - s : s)];
    if (e == NIL) { r = H3D_E_COUNT; break; }
    if (act_g(K, e) < 0) { r = H3D_E_CHAIN; break; }
  }
  *res = r;
}

__global__ void k_extract_exact(int *K, const int *slots, long long off, int *faces,
                                long long limit, long long *res) {
  long long m = 0, r;
  for (long long idx = off;; ++idx) {
    const long long e = slots[idx];
    if (e == NIL) { r = m; break; }
    if (m >= limit) { r = H3D_E_OVERFLOW; break; }
    faces[3 * m] = K[2 * e];
    faces[3 * m + 1] = static_cast<int>(e);
    faces[3 * m + 2] = K[2 * e + 1];
    if (act_g(K, e) < 0) { r = H3D_E_CHAIN; break; }
    ++m;
  }
  *res = r;
}

__global__ void k_log_length(const int *slots, long long off, long long cap, long long *res) {
  long long r = H3D_E_UNTERMINATED;
  for (long long idx = 0; idx < cap; ++idx)
    if (slots[off + idx] == NIL) { r = idx; break; }
  *res = r;
}

__global__ void k_copy_log(const int *src, int *dst, long long off, long long cap,
                           long long *res) {
  *res = copy_log_g(src, dst, off, cap);
}

}  // namespace h3d

using namespace h3d;

// ----------------------------------------------------------------- C ABI

namespace {
// one small device result buffer per call, allocated through the stream's
// pool: the seam is the reference's blocking API, so these calls sync.
struct Res {
  long long *d = nullptr;
  cudaStream_t s;
  explicit Res(void *stream, int words = 2) : s(static_cast<cudaStream_t>(stream)) {
    if (cudaMallocAsync(&d, sizeof(long long) * words, s) == cudaSuccess)
      cudaMemsetAsync(d, 0, sizeof(long long) * words, s);
    else
      d = nullptr;
  }
  ~Res() {
    if (d) cudaFreeAsync(d, s);
  }
  long long get(int words = 1, long long *host = nullptr) {
    long long tmp[2] = {0, 0};
    long long *h = host ? host : tmp;
    if (!d) return H3D_E_CUDA;
    if (h3d_check(cudaMemcpyAsync(h, d, sizeof(long long) * words,
                                  cudaMemcpyDeviceToHost, s)) ||
        h3d_check(h3d_sync(s)))
      return H3D_E_CUDA;
    return h[0];
  }
};
}  // namespace

extern "C" {

int64_t h3d_seam_act(int32_t *links, int64_t i, void *stream) {
  Res r(stream);
  h3d_count_launches(1);
  k_act<<<1, 1, 0, r.s>>>(links, i, r.d);
  return r.get();
}

int64_t h3d_seam_init_base_logs(int32_t *links, int32_t *slots, int64_t n, void *stream) {
  if (n <= 0) return 0;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  h3d_count_launches(1);
  k_init_base<<<h3d_grid(n, 256), 256, 0, s>>>(links, slots, n);
  if (h3d_check(cudaGetLastError()) || h3d_check(h3d_sync(s))) return H3D_E_CUDA;
  return 0;
}

int64_t h3d_seam_find_initial_bridge(const double *pts, const int32_t *links, int64_t u,
                                     int64_t v, int64_t limit, int64_t *uv_out,
                                     void *stream) {
  Res r(stream);
  h3d_count_launches(1);
  k_find_bridge<<<1, 1, 0, r.s>>>(RowPts{pts, 1.0}, links, u, v, limit, r.d);
  long long h[2];
  const long long st = r.get(2, h);
  if (st == H3D_E_CUDA && !r.d) return H3D_E_CUDA;
  uv_out[0] = h[0];
  uv_out[1] = h[1];
  return 0;
}

int64_t h3d_seam_merge_movies(const double *pts, int32_t *links, const int32_t *in_slots,
                              int32_t *out_slots, int64_t L, int64_t M, int64_t R,
                              void *stream) {
  Res r(stream);
  h3d_count_launches(1);
  k_merge_one<<<1, 1, 0, r.s>>>(RowPts{pts, 1.0}, links, in_slots, out_slots, L, M, R, r.d);
  return r.get();
}

int64_t h3d_seam_merge_range(const double *pts, int32_t *links, const int32_t *in_slots,
                             int32_t *out_slots, const int64_t *jobs, int64_t lo,
                             int64_t hi, void *stream) {
  if (hi <= lo) return 0;
  Res r(stream);
  h3d_count_launches(1);
  k_merge_range<<<h3d_grid(hi - lo, 128), 128, 0, r.s>>>(
      RowPts{pts, 1.0}, links, in_slots, out_slots,
      reinterpret_cast<const long long *>(jobs), lo, hi, r.d);
  return r.get();
}

int64_t h3d_seam_replay(int32_t *links, const int32_t *slots, int64_t off, int64_t count,
                        void *stream) {
  Res r(stream);
  h3d_count_launches(1);
  k_replay<<<1, 1, 0, r.s>>>(links, slots, off, count, 0, r.d);
  return r.get();
}

int64_t h3d_seam_rewind_replay(int32_t *links, const int32_t *slots, int64_t off,
                               int64_t count, void *stream) {
  Res r(stream);
  h3d_count_launches(1);
  k_replay<<<1, 1, 0, r.s>>>(links, slots, off, count, 1, r.d);
  return r.get();
}

int64_t h3d_seam_extract_faces(int32_t *links, const int32_t *slots, int64_t off,
                               int32_t *faces, int64_t limit, void *stream) {
  Res r(stream);
  h3d_count_launches(1);
  k_extract_exact<<<1, 1, 0, r.s>>>(links, slots, off, faces, limit, r.d);
  return r.get();
}

int64_t h3d_seam_log_length(const int32_t *slots, int64_t off, int64_t cap, void *stream) {
  Res r(stream);
  h3d_count_launches(1);
  k_log_length<<<1, 1, 0, r.s>>>(slots, off, cap, r.d);
  return r.get();
}

int64_t h3d_seam_copy_log(const int32_t *src, int32_t *dst, int64_t off, int64_t cap,
                          void *stream) {
  Res r(stream);
  h3d_count_launches(1);
  k_copy_log<<<1, 1, 0, r.s>>>(src, dst, off, cap, r.d);
  return r.get();
}

int64_t h3d_seam_run_level(const double *pts, double zsign, int32_t *links,
                           const int32_t *in_slots, int32_t *out_slots, int64_t n,
                           int64_t level, void *stream) {
  if (level < 1 || n < 2) return H3D_E_ARG;
  Res r(stream);
  const long long groups = (n + (1ll << level) - 1) >> level;
  h3d_count_launches(1);
  k_level_exact<<<h3d_grid(groups, 128), 128, 0, r.s>>>(RowPts{pts, zsign}, links, in_slots,
                                                        out_slots, n, (int)level, r.d);
  return r.get();
}

}  // extern "C"
