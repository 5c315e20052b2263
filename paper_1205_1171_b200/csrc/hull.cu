// hull.cu -- the whole device pipeline of convex_hull_3d (api.py:162-284)
// behind ONE C-ABI call: presort + degeneracy scan, both hull passes over all
// merge levels, facet extraction, orientation / remap / vertex compaction,
// and ONE read-back of the results' sizes.
//
// The presort runs optimistically without host synchronisation (the common
// case has no x ties, no long runs of equal keys, finite input and a
// non-degenerate cloud); its flags and the degeneracy scan are judged on the
// device by a gate kernel that writes the level loop's error word, so a rare
// input stops every later launch at once.  After the single read-back an
// input with ties is redone through the exact tie path (h3d_presort, api.py
// :90-110), an error is returned, and a fast-path decline is reported in
// info[0] for the caller's exact engine; the next call of the same size
// then starts on the exact tie path.  Host synchronisations per hull:
// one for a replayed level plan (fast.cu), one per measured level otherwise,
// plus this final one -- counted by h3d_sync_count().
#include <unordered_map>

#include "../../include/hull3d_b200.h"
#include "fast.cuh"
#include "h3d_host.h"

namespace h3d {
int64_t presort_async(const double *pts, int64_t n, double *sorted_pts, int64_t *order, void *workspace,
                      size_t workspace_bytes, long long *err, cudaStream_t s, int *sums_ready);
int64_t presort_ties_async(const double *pts, int64_t n, double *sorted_pts, int64_t *order, void *workspace,
                           size_t workspace_bytes, long long *err, long long *perturbed, cudaStream_t s);
int64_t orient_async(const double *sorted_pts, int64_t n, const int64_t *order, const int32_t *faces_raw,
                     const long long *counts, int64_t cap, int64_t *faces, int32_t *vertex_mark,
                     int64_t *vertices, long long *vcount, void *workspace, size_t workspace_bytes,
                     cudaStream_t s, int sums_ready);
}  // namespace h3d

using namespace h3d;

namespace {

// device state words (int64): err, k_lo, k_up, verify diagnostics, vertex
// count, 3 spare, then the level stamps
constexpr int kStErr = 0, kStCounts = 1, kStVcount = 4, kStPerturbed = 5, kStStamps = 8;

int64_t passes_and_epilogue(const double *sorted_pts, int64_t n, const int64_t *order, void *presort_ws,
                            size_t presort_ws_bytes, void *ws_lower, void *ws_upper, size_t pass_ws_bytes,
                            int32_t *faces_raw, int64_t cap, int64_t *faces, int64_t *vertices,
                            int32_t *vertex_mark, int64_t *state_dev, int32_t verify, int64_t *fin,
                            cudaStream_t s, int sums_ready) {
  long long *st = reinterpret_cast<long long *>(state_dev);
  int levels = 0;
  while ((1ll << levels) < n) ++levels;
  const int64_t r = h3d_fast_passes_range(sorted_pts, n, 0, n, 1, levels, ws_lower, ws_upper, pass_ws_bytes,
                                          state_dev + kStErr, verify, s);
  if (r < 0) return r;
  *fin = r;
  const int64_t e = h3d_fast_extract(ws_lower, ws_upper, n, r, r, faces_raw, cap, state_dev + kStCounts,
                                     state_dev + kStErr, s);
  if (e < 0) return e;
  return orient_async(sorted_pts, n, order, faces_raw, st + kStCounts, cap, faces, vertex_mark, vertices,
                      st + kStVcount, presort_ws, presort_ws_bytes, s, sums_ready);
}

}  // namespace

extern "C" {

int64_t h3d_hull(const double *pts, int64_t n, double *sorted_pts, int64_t *order, void *presort_ws,
                 size_t presort_ws_bytes, void *ws_lower, void *ws_upper, size_t pass_ws_bytes,
                 int32_t *faces_raw, int64_t cap, int64_t *faces, int64_t *vertices, int32_t *vertex_mark,
                 int64_t *state_dev, int32_t flags, int64_t *info, void *stream) {
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (n < 4 || n > (1ll << 30) || cap < 2 * n) return H3D_E_ARG;
  const bool stamps = flags & 1;
  const int32_t verify = (flags & 2) ? 2 : 0;
  long long *st = reinterpret_cast<long long *>(state_dev);
  for (int q = 0; q < H3D_HULL_INFO; ++q) info[q] = 0;
  if (h3d_check(cudaMemsetAsync(state_dev, 0, H3D_HULL_STATE * sizeof(int64_t), s))) return H3D_E_CUDA;
  if (stamps) {
    h3d_profile_stamps(state_dev + kStStamps);
    h3d_stamp_now(s, 0);  // slot 0: the presort's start
  }
  int64_t fin = 0;
  // a call whose previous same-size call had x ties (integer clouds) starts
  // on the tie path (presort_ties_async, also free of host synchronisation):
  // the optimistic attempt would only be redone
  int dev = 0;
  cudaGetDevice(&dev);
  const long long key = (static_cast<long long>(dev) << 40) ^ n;
  thread_local std::unordered_map<long long, bool> ties_last;
  const bool direct = ties_last.count(key) && ties_last[key];
  int sums_ready = 0;  // the optimistic gather made the epilogue's centroid sums
  int64_t rc = direct ? presort_ties_async(pts, n, sorted_pts, order, presort_ws, presort_ws_bytes, st + kStErr,
                                          st + kStPerturbed, s)
                       : presort_async(pts, n, sorted_pts, order, presort_ws, presort_ws_bytes, st + kStErr, s,
                                       &sums_ready);
  if (rc == 0)
    rc = passes_and_epilogue(sorted_pts, n, order, presort_ws, presort_ws_bytes, ws_lower, ws_upper,
                             pass_ws_bytes, faces_raw, cap, faces, vertices, vertex_mark, state_dev, verify,
                             &fin, s, sums_ready);
  // the one read-back (+ the level stamps)
  const int words = stamps ? H3D_HULL_STATE : kStStamps;
  if (rc == 0 && (h3d_check(cudaMemcpyAsync(info + H3D_HULL_INFO - H3D_HULL_STATE, state_dev,
                                            words * sizeof(int64_t), cudaMemcpyDeviceToHost, s)) ||
                  h3d_check(h3d_sync(s))))
    rc = H3D_E_CUDA;
  const int64_t *hs = info + H3D_HULL_INFO - H3D_HULL_STATE;
  int32_t perturbed = direct && rc == 0 ? static_cast<int32_t>(hs[kStPerturbed]) : 0;
  if (rc == 0 && hs[kStErr] == H3D_E_REDO) {
    // x ties or a long run of equal keys: the exact presort (tie path,
    // perturbation, its own checks), then the rest again
    rc = h3d_presort(pts, n, sorted_pts, order, presort_ws, presort_ws_bytes, &perturbed, stream);
    if (rc == 0 && h3d_check(cudaMemsetAsync(state_dev, 0, kStStamps * sizeof(int64_t), s))) rc = H3D_E_CUDA;
    if (rc == 0)
      rc = passes_and_epilogue(sorted_pts, n, order, presort_ws, presort_ws_bytes, ws_lower, ws_upper,
                               pass_ws_bytes, faces_raw, cap, faces, vertices, vertex_mark, state_dev, verify,
                               &fin, s, 0);
    if (rc == 0 && (h3d_check(cudaMemcpyAsync(info + H3D_HULL_INFO - H3D_HULL_STATE, state_dev,
                                              words * sizeof(int64_t), cudaMemcpyDeviceToHost, s)) ||
                    h3d_check(h3d_sync(s))))
      rc = H3D_E_CUDA;
  }
  if (rc == 0) ties_last[key] = perturbed != 0;
  if (stamps) h3d_profile_stamps(nullptr);
  if (rc < 0) return rc;
  const long long err = hs[kStErr];
  // the gate's verdicts are the presort's errors (api.py:106-108, :131-147)
  if (err == H3D_E_NONFINITE || err == H3D_E_TIES || err == H3D_E_COINCIDENT || err == H3D_E_COLLINEAR ||
      err == H3D_E_COPLANAR)
    return err;
  info[0] = err;  // 0, or the fast path's decline: the caller's exact engine takes over
  info[1] = hs[kStCounts];
  info[2] = hs[kStCounts + 1];
  info[3] = err ? 0 : hs[kStCounts] + hs[kStCounts + 1];
  info[4] = err ? 0 : hs[kStVcount];
  info[5] = perturbed;
  info[6] = fin;
  info[7] = hs[3];  // verify diagnostics
  if (err == 0 && info[3] == 0) return H3D_E_NOFACETS;
  return 0;
}

}  // extern "C"
