/*
 * hull3d_b200.h -- C ABI of the B200-native kinetic 3D convex hull.
 *
 * Drop-in boundary for the hot path of the reference package `hull3d`
 * (arxiv/paper_1205_1171).  Two groups of entry points:
 *
 *  1. The kernel-module seam.  The reference selects its hot kernels through
 *     `hull3d.kernels.active()` (pkg/src/hull3d/kernels.py:52-54), a module
 *     exporting the functions of pkg/src/hull3d/_ckernels.pyx:231-375 over
 *     caller-owned buffers that never allocate and report failures as
 *     negative codes.  Each `h3d_seam_*` function below replaces one of them
 *     with the same argument meaning, buffer layout and return convention,
 *     except that every buffer is a DEVICE pointer and a CUDA stream is
 *     passed.  They are synchronous (they read back one result word), like
 *     the reference's blocking calls.  INTEGRATION.md shows the ctypes module
 *     a maintainer would register in kernels._BY_NAME.
 *
 *  2. The fused B200 path used by `paper_1205_1171_b200.convex_hull_3d`
 *     (the reference entry point pkg/src/hull3d/api.py:162-284): device
 *     presort, both passes of all merge levels, facet extraction and the
 *     orientation / remap epilogue, stream-ordered, over caller-provided
 *     fixed-capacity workspace (the library never allocates).
 *
 * Layouts (pkg/src/hull3d/store.py:46-118): pts = n rows of (x,y,z) f64,
 * links = n rows of (prev,next) i32, slots = 2n i32 with the log of group
 * [L,R) at slot 2L, NIL (-1) terminated; jobs = m rows of (L,M,R) i64.
 * No torch types cross this boundary: plain pointers, sizes and a
 * cudaStream_t passed as void*.
 */
#ifndef HULL3D_B200_H
#define HULL3D_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* constants and error codes: pkg/src/hull3d/_ckernels.pyx:19-24 */
#define H3D_NIL (-1)
#define H3D_E_OVERFLOW (-1)      /* MergeOverflowError   (merge.py:33-35)   */
#define H3D_E_BRIDGE (-2)        /* BridgeWalkError      (merge.py:37-39)   */
#define H3D_E_CHAIN (-3)         /* ChainError           (store.py:24-26)   */
#define H3D_E_COUNT (-4)         /* LogError             (store.py:29-30)   */
#define H3D_E_UNTERMINATED (-5)  /* LogError             (store.py:29-30)   */
#define H3D_E_TIES (-6)          /* DegenerateInputError (api.py:106-108)   */
#define H3D_E_COINCIDENT (-7)    /* DegenerateInputError (api.py:131-132)   */
#define H3D_E_COLLINEAR (-8)     /* DegenerateInputError (api.py:138-139)   */
#define H3D_E_COPLANAR (-9)      /* DegenerateInputError (api.py:146-147)   */
#define H3D_E_NOFACETS (-10)     /* DegenerateInputError (api.py:253-256)   */
#define H3D_E_CAPACITY (-11)     /* fast-path fixed capacity exceeded       */
#define H3D_E_NONFINITE (-12)   /* ValueError("coordinates must be finite") */
#define H3D_E_FASTPATH (-13)     /* fast path declined: caller takes the exact route */
#define H3D_E_VERIFY (-14)       /* verify mode: a level wrote an inconsistent group */
#define H3D_E_REDO (-15)         /* h3d_hull internal: the optimistic presort met ties */
#define H3D_E_ARG (-100)         /* bad argument                            */
#define H3D_E_CUDA (-101)        /* CUDA runtime error                      */

/* library identification (the reference's kernel modules export IMPL) */
const char *h3d_impl(void);
/* last CUDA error string seen by the library (diagnostics) */
const char *h3d_last_error(void);
/* number of this library's own kernel launches so far (process-wide) */
int64_t h3d_launch_count(void);
/* number of host synchronisations (stream syncs) the library made so far */
int64_t h3d_sync_count(void);
/* per-level profile of the CALLING THREAD: when enabled (per thread; on = 1),
 * every merge level of h3d_fast_passes* run by this thread is bracketed by
 * CUDA events on its stream (events pooled per device); on = 2 brackets only
 * the lane-per-job kernel launches themselves (the dominant kernel's
 * duration for bench.py's roofline); collect returns this thread's (level,
 * pass, milliseconds) rows, waiting only for its own last event, and clears
 * them */
void h3d_profile_enable(int32_t on);
/* per-level DEVICE time stamps for the calling thread's next
 * h3d_fast_passes* calls: dev_buf = 64 device int64 (or NULL = off).  The
 * level kernels write %globaltimer (ns) at the start of level l into slot l
 * and the end of the last level into slot 40 -- no event records, no host
 * work (HullStats' per-level seconds, api.py:28-44).  routes: the route tag
 * of each stamped slot (1000+l lane-per-job, 3000+B fused leaf levels 1..B,
 * 4000+l time-split pipeline, 5000+l one CTA per job, l warp per job, -1 none). */
void h3d_profile_stamps(int64_t *dev_buf);
int64_t h3d_profile_routes(int32_t *routes, int64_t max);
int64_t h3d_profile_collect(int32_t *level, int32_t *pass, float *ms,
                            int64_t max);

/* ---------------------------------------------------------------------
 * 1. kernel-module seam (pkg/src/hull3d/_ckernels.pyx)
 * ------------------------------------------------------------------- */

/* act(links, i) -> 0 or E_CHAIN                        _ckernels.pyx:231-234 */
int64_t h3d_seam_act(int32_t *links, int64_t i, void *stream);

/* init_base_logs(links, slots, n) -> 0                 _ckernels.pyx:237-245 */
int64_t h3d_seam_init_base_logs(int32_t *links, int32_t *slots, int64_t n,
                                void *stream);

/* find_initial_bridge(pts, links, u, v, limit) -> (u, v) or (NIL, NIL)
 *                                                      _ckernels.pyx:248-255 */
int64_t h3d_seam_find_initial_bridge(const double *pts, const int32_t *links,
                                     int64_t u, int64_t v, int64_t limit,
                                     int64_t *uv_out /* host, 2 */,
                                     void *stream);

/* merge_movies(pts, links, in, out, L, M, R) -> k or code
 *                                                      _ckernels.pyx:258-264 */
int64_t h3d_seam_merge_movies(const double *pts, int32_t *links,
                              const int32_t *in_slots, int32_t *out_slots,
                              int64_t L, int64_t M, int64_t R, void *stream);

/* merge_range(pts, links, in, out, jobs, lo, hi) -> 0 or code
 *                                                      _ckernels.pyx:267-280 */
int64_t h3d_seam_merge_range(const double *pts, int32_t *links,
                             const int32_t *in_slots, int32_t *out_slots,
                             const int64_t *jobs, int64_t lo, int64_t hi,
                             void *stream);

/* replay / rewind_replay(links, slots, off, count) -> 0 or code
 *                                                      _ckernels.pyx:292-321 */
int64_t h3d_seam_replay(int32_t *links, const int32_t *slots, int64_t off,
                        int64_t count, void *stream);
int64_t h3d_seam_rewind_replay(int32_t *links, const int32_t *slots,
                               int64_t off, int64_t count, void *stream);

/* extract_faces(links, slots, off, faces (limit,3) i32) -> m or code
 *                                                      _ckernels.pyx:324-349 */
int64_t h3d_seam_extract_faces(int32_t *links, const int32_t *slots,
                               int64_t off, int32_t *faces, int64_t limit,
                               void *stream);

/* log_length(slots, off, cap) -> k or E_UNTERMINATED   _ckernels.pyx:352-360 */
int64_t h3d_seam_log_length(const int32_t *slots, int64_t off, int64_t cap,
                            void *stream);

/* copy_log(src, dst, off, cap) -> k or E_UNTERMINATED  _ckernels.pyx:363-375 */
int64_t h3d_seam_copy_log(const int32_t *src, int32_t *dst, int64_t off,
                          int64_t cap, void *stream);

/* One whole level of build_movie (pkg/src/hull3d/parallel.py:96-109): every
 * merge job of plan_level(n, level) plus the carry, in one launch, with the
 * reference's exact sequential merge per job.  zsign = -1.0 reads pts with z
 * negated (the upper pass).  Returns 0 or the first error code. */
int64_t h3d_seam_run_level(const double *pts, double zsign, int32_t *links,
                           const int32_t *in_slots, int32_t *out_slots,
                           int64_t n, int64_t level, void *stream);

/* ---------------------------------------------------------------------
 * 2. fused B200 path
 * ------------------------------------------------------------------- */

/* bytes of workspace h3d_presort / h3d_hull need for n points */
size_t h3d_presort_workspace_bytes(int64_t n);

/* Device presort = _sort_and_perturb + _scan_degenerate
 * (pkg/src/hull3d/api.py:61-147): stable radix argsort of x; on any x tie,
 * a stable (x,y,z) lexsort, bit-exact tie perturbation and a stable
 * re-sort.  Writes sorted (n,3) f64 and order (n) i64 (caller -> sorted).
 * *perturbed (host) is set to 0/1.  Returns 0 or H3D_E_NONFINITE / _TIES /
 * _COINCIDENT / _COLLINEAR / _COPLANAR. */
int64_t h3d_presort(const double *pts, int64_t n, double *sorted_pts,
                    int64_t *order, void *workspace, size_t workspace_bytes,
                    int32_t *perturbed, void *stream);

/* Sharded presort (multi-GPU): writes rows [q0, p1) of the global sorted
 * order (sorted_pts[3*q0 ...], order[q0 ...]: only the window's rows are
 * touched, so the caller may pass a window-sized buffer minus q0 rows) from
 * the full input without sorting the rest: 32-bit keys, a radix select of
 * the two window boundaries, exact ranking of the boundary key runs, a sort
 * of the window.  scan != 0 also runs _scan_degenerate over rows [0, p1)
 * (rank 0, q0 = 0).  Workspace: h3d_presort_slab_workspace_bytes(n, p1 - q0)
 * (4 bytes per input point + O(window)).  Returns 0, or H3D_E_FASTPATH
 * whenever the window cannot reproduce h3d_presort on its own (any x tie, a
 * long run of equal keys, non-finite input, a degeneracy not decided inside
 * the window): the caller then runs the replicated h3d_presort.  Needs
 * n >= 2048. */
size_t h3d_presort_slab_workspace_bytes(int64_t n, int64_t m);
int64_t h3d_presort_slab(const double *pts, int64_t n, int64_t q0, int64_t p1,
                         int32_t scan, double *sorted_pts, int64_t *order,
                         void *workspace, size_t workspace_bytes, void *stream);

/* workspace h3d_orient_remap* needs (<= h3d_presort_workspace_bytes(n)) */
size_t h3d_epilogue_workspace_bytes(int64_t n);
/* Epilogue (pkg/src/hull3d/api.py:252-266): faces_raw (F,3) i32 in sorted
 * indices (lower block then upper block) -> faces (F,3) i64 oriented outward
 * against the centroid and mapped through order; vertex_mark (n) i32 scratch;
 * vertices (<= n) i64 = np.unique(faces).  Returns the vertex count. */
int64_t h3d_orient_remap(const double *sorted_pts, int64_t n,
                         const int64_t *order, const int32_t *faces_raw,
                         int64_t nfaces, int64_t *faces, int32_t *vertex_mark,
                         int64_t *vertices, void *workspace,
                         size_t workspace_bytes, void *stream);

/* h3d_orient_remap with the centroid taken over centroid_pts (n rows, any
 * order; nullptr = sorted_pts): the sharded multi-GPU path, whose rank 0
 * holds only the rows its merges touched, passes the caller-order input. */
int64_t h3d_orient_remap_ex(const double *sorted_pts, int64_t n,
                            const int64_t *order, const int32_t *faces_raw,
                            int64_t nfaces, int64_t *faces,
                            int32_t *vertex_mark, int64_t *vertices,
                            const double *centroid_pts, void *workspace,
                            size_t workspace_bytes, void *stream);

/* Routing knobs of the fast path (not a reference interface; used by the
 * tests to drive every kernel route and by tuning sweeps; DESIGN.md §3.2b
 * lists them with their defaults): "big_kin" (time-split pipeline from this
 * merged child log size), "big_total" (or half that log size with this many
 * child events in the level), "big_max_jobs", "leaf_b" (levels 1..B fused: 3
 * or 4; 0-2 = off), "lane" / "lane_max_level" / "lane_xyz_kb" / "lane_stage"
 * / "lane_own" / "lane_pf1" / "lane_pf2" (the lane.cu kernel), "tpj_min_jobs", "tpj_xyz_kb", "tpj_xyz_ctas",
 * "tpj_max_level", "tpj_cap_level" (the 128-register build up to this
 * level), "tpj_split" (split / hybrid lane-per-job levels; 2 = split every
 * level, tests), "mini" (0/1: the one-CTA-per-job merges), "mini_ctas",
 * "mini_one_wave", "mini_tiny_ctas" / "mini_tiny_kin", "mini_huge_ctas" /
 * "mini_huge_kin", "mini_seg", "mini_spec", "plan" (record & replay level
 * plans), "interleave" (the two passes' CTAs adjacent).  value < 0 only
 * queries.  Returns the previous value, or -1 for an unknown name.
 * Environment variables H3D_BIG_KIN, H3D_LEAF_B, ... set the defaults. */
int64_t h3d_tune(const char *name, int64_t value);

/* bytes of workspace one h3d_fast_pass needs for n points (two compact
 * group buffers: headers, int2 links, ids, 16-byte events; HBM scratch of
 * the warp merge; and, in the lower pass's workspace, the scratch of the
 * time-split pipeline for large merge jobs, sized for min(n, max(2^21, n/8)) points
 * per pass -- levels beyond it fall back to the warp merge) */
size_t h3d_fast_pass_workspace_bytes(int64_t n);
/* the upper pass's workspace needs only this much (no big-job scratch; the
 * workspace_bytes argument of the calls below stays the lower pass's) */
size_t h3d_fast_upper_workspace_bytes(int64_t n);

/* Both hull passes (build_movie, pkg/src/hull3d/parallel.py:68-112) over the
 * presorted points, all ceil(log2 n) levels, stream-ordered, no host sync:
 * every level is ONE launch covering the lower (z as is) and the upper pass
 * (z negated on load, api.py:215-216).  ws_lower / ws_upper are two
 * workspaces of h3d_fast_pass_workspace_bytes(n) each.  Errors are recorded
 * into *err_dev (device int64, first error wins; H3D_E_* codes or -13 = the
 * fast path cannot reproduce the reference semantics for this input, rerun
 * the exact seam path).  final_out (host int64[2]) receives which buffer of
 * each workspace holds the final group.  Returns 0 or a negative code. */
int64_t h3d_fast_passes(const double *sorted_pts, int64_t n, void *ws_lower,
                        void *ws_upper, size_t workspace_bytes, int64_t *err_dev,
                        int32_t verify, int64_t *final_out, void *stream);

/* Level range form (multi-GPU x-slabs, pkg/src/hull3d/parallel.py:96-111
 * restricted to the jobs inside one slab): runs levels lv_lo..lv_hi only for
 * the jobs whose point range starts in [p0, p1); lv_lo == 1 also initialises
 * the level-0 groups of [p0, p1).  Level l reads buffer (l-1)&1 and writes
 * buffer l&1 of each workspace.  Returns lv_hi&1 or a negative code. */
int64_t h3d_fast_passes_range(const double *sorted_pts, int64_t n, int64_t p0,
                              int64_t p1, int32_t lv_lo, int32_t lv_hi,
                              void *ws_lower, void *ws_upper,
                              size_t workspace_bytes, int64_t *err_dev,
                              int32_t verify, void *stream);

/* Byte offsets of the compact-group arrays inside one pass workspace:
 * A.hdr, A.lnk, A.gid, A.ev, B.hdr, B.lnk, B.gid, B.ev, seq (host int64[9]).
 * hdr = int2 (nS, k) per group; lnk = int2 (prev, next) group-local ids of
 * each kept point at t = -inf; gid = i32 sorted index of each kept point
 * (coordinates are read from sorted_pts); ev = 16-byte events (t f64, then
 * one u64 word: local ids a | b << 21 | c << 42, kind in bit 63); a group
 * [L, R) at level l has header l, links/ids at
 * [L, L+nS) and events at [2L, 2L+k).  Used to ship groups between GPUs. */
int64_t h3d_fast_layout(int64_t n, int64_t *offsets);

/* Facets of both passes from their final groups (extract_faces,
 * _ckernels.pyx:324-349): faces (cap,3) i32 in sorted indices, lower block
 * then upper block; counts_dev (device int64[2]) = (lower, upper) counts.
 * A total above cap records H3D_E_CAPACITY into err_dev. */
int64_t h3d_fast_extract(void *ws_lower, void *ws_upper, int64_t n,
                         int64_t final_lower, int64_t final_upper,
                         int32_t *faces, int64_t cap, int64_t *counts_dev,
                         int64_t *err_dev, void *stream);

/* ---- the whole convex_hull_3d device pipeline in ONE call (csrc/hull.cu):
 * presort + tie path + degeneracy scan (api.py:90-147), both hull passes over
 * all merge levels (parallel.py:68-112, one launch per level covering both
 * passes), extract_faces (_ckernels.pyx:324-349), orientation / remap /
 * vertex compaction (api.py:252-266), then ONE read-back of the sizes (plus
 * one per measured merge level inside the level loop).
 *   pts        device (n,3) f64, caller order, n >= 4
 *   sorted_pts device (n,3) f64 out; order device int64[n] out (api.py:97)
 *   presort_ws h3d_presort_workspace_bytes(n); ws_lower / ws_upper
 *              h3d_fast_pass_workspace_bytes(n) each
 *   faces_raw  device int32 (cap,3) scratch, cap >= 2n; faces device int64
 *              (cap,3) out (outward, caller indices, lower block then upper
 *              block in log order); vertices device int64[n] out (sorted
 *              unique); vertex_mark device int32[n] scratch
 *   state_dev  device int64[H3D_HULL_STATE] scratch
 *   flags      bit 0: per-level device time stamps; bit 1: verify mode
 *   info       host int64[H3D_HULL_INFO]: [0] 0 or the fast path's decline
 *              code (run the exact engine on sorted_pts), [1] lower events,
 *              [2] upper events, [3] facets, [4] vertices, [5] perturbed,
 *              [6] final buffer, [7] verify diagnostics; info[32 + 8 + l] =
 *              stamp (ns) of level l (0 = presort start, 40 = end).
 * Returns 0 or a negative code: H3D_E_NONFINITE / _TIES / _COINCIDENT /
 * _COLLINEAR / _COPLANAR / _NOFACETS (DegenerateInputError, ValueError),
 * H3D_E_ARG, H3D_E_CUDA. */
#define H3D_HULL_STATE 96
#define H3D_HULL_INFO 128
int64_t h3d_hull(const double *pts, int64_t n, double *sorted_pts, int64_t *order, void *presort_ws,
                 size_t presort_ws_bytes, void *ws_lower, void *ws_upper, size_t pass_ws_bytes,
                 int32_t *faces_raw, int64_t cap, int64_t *faces, int64_t *vertices, int32_t *vertex_mark,
                 int64_t *state_dev, int32_t flags, int64_t *info, void *stream);

/* ---- device-wide primitives (csrc/prims.cuh), hand-written for sm_100a;
 * exported so the parity tests can check them against numpy on their own.
 * All pointers are device pointers; tmp is caller-owned scratch of
 * h3d_prim_temp_bytes(n) bytes. */
size_t h3d_prim_temp_bytes(int64_t n);
/* Stable LSD radix sort of (key, i32 value) pairs by key bits
 * [begin_bit, end_bit) (numpy argsort(kind="stable") semantics, the sort
 * under api.py:97 and :86-87); key_bytes 4 or 8; iota_vals: the input values
 * are 0..n-1 (vals is not read).  The data ping-pong between (keys, vals)
 * and (keys_alt, vals_alt); returns 0 (result in keys/vals), 1 (result in
 * the _alt buffers) or a negative code. */
int64_t h3d_radix_sort_pairs(void *keys, void *keys_alt, int32_t *vals, int32_t *vals_alt, int64_t n,
                             int32_t key_bytes, int32_t begin_bit, int32_t end_bit, int32_t iota_vals,
                             void *tmp, size_t tmp_bytes, void *stream);
/* Inclusive or exclusive scan of int64 with + or max (np.cumsum /
 * np.maximum.accumulate); in == out allowed. */
int64_t h3d_scan_i64(const int64_t *in, int64_t *out, int64_t n, int32_t op_max, int32_t exclusive,
                     void *tmp, size_t tmp_bytes, void *stream);
/* Indices of the nonzero flags in ascending order (np.flatnonzero);
 * *count_dev (device int64) receives how many. */
int64_t h3d_select_flagged(const int32_t *flags, int64_t n, int64_t *out, int64_t *count_dev, void *tmp,
                           size_t tmp_bytes, void *stream);

#ifdef __cplusplus
}
#endif
#endif /* HULL3D_B200_H */
