// fast.cu -- the fused fast path: all merge levels of a pass over compact groups.
//
// Level scheduler (parallel.py:68-112 on the device): one launch of
// k_fast_level per level plus one k_fast_big launch that picks up the jobs
// too big for the level kernel's shared-memory budget and the carry.  No
// host synchronisation inside a pass; a device error word is read once per
// hull.
//
// k_fast_level: one thread per merge job, jobs packed into a CTA's dynamic
// shared memory by a block-wide prefix scan of their footprints (jobs that do
// not fit wait for the next round).  Each warp stages its jobs' contiguous
// child runs (records, events) with coalesced loads, every thread then runs
// its merge (merge_compact, fast.cuh) entirely in shared memory, and the warp
// compacts (ballot/popc prefix scans) and streams each merged group back out.
#include <cub/cub.cuh>

#include "fast.cuh"
#include "h3d_host.h"

namespace h3d {

struct GroupBuf {
  int2 *hdr;
  Rec *rec;
  int *gid;
  Ev *ev;
};

constexpr unsigned FULL = 0xffffffffu;

__device__ __forceinline__ long long align8(long long b) { return (b + 7) & ~7ll; }

// shared-memory footprint of one merge job
__device__ __forceinline__ long long job_bytes(int nS, int kin) {
  return align8(32ll * nS + 24ll * kin + 24ll * (2ll * nS) + 4ll * nS);
}

struct JobView {
  Rec *rec;
  Ev *evL, *evR, *out;
  int *mark;
};

__device__ __forceinline__ JobView carve_job(unsigned char *base, int nS, int kL, int kR) {
  JobView v;
  v.rec = reinterpret_cast<Rec *>(base);
  v.evL = reinterpret_cast<Ev *>(base + 32ll * nS);
  v.evR = v.evL + kL;
  v.out = v.evR + kR;
  v.mark = reinterpret_cast<int *>(v.out + 2 * nS);
  return v;
}

// level 0: every point is a one-point group with an empty log
__global__ void k_fast_init(const double *__restrict__ pts, double zs, long long n, GroupBuf g) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    Rec r;
    r.x = pts[3 * i];
    r.y = pts[3 * i + 1];
    r.z = zs * pts[3 * i + 2];
    r.prev = NIL;
    r.next = NIL;
    g.rec[i] = r;
    g.gid[i] = static_cast<int>(i);
    g.hdr[i] = make_int2(1, 0);
  }
}

// Cooperative (group of `width` lanes, lane index `lane`) staging of one job.
__device__ __forceinline__ void stage_job(const GroupBuf &in, JobView v, long long L, long long M,
                                          int nSL, int nSR, int kL, int kR, int lane, int width) {
  const int nS = nSL + nSR;
  for (int p = lane; p < nS; p += width) {
    Rec r;
    if (p < nSL) {
      r = in.rec[L + p];
    } else {
      r = in.rec[M + (p - nSL)];
      if (r.prev != NIL) r.prev += nSL;
      if (r.next != NIL) r.next += nSL;
    }
    v.rec[p] = r;
    v.mark[p] = 0;
  }
  for (int e = lane; e < kL; e += width) v.evL[e] = in.ev[2 * L + e];
  for (int e = lane; e < kR; e += width) v.evR[e] = in.ev[2 * M + e];
}

// Warp-cooperative compaction + write-out of one merged job (warp-wide call).
// mark[p] != 0 keeps p; afterwards mark[p] holds its new id (or -1).
__device__ void writeout_job_warp(const GroupBuf &in, const GroupBuf &out, JobView v, long long L,
                                  long long M, int nSL, int nS, int k, long long gidx,
                                  long long *err) {
  const int lane = threadIdx.x & 31;
  int base = 0;
  for (int p0 = 0; p0 < nS; p0 += 32) {
    const int p = p0 + lane;
    const bool keep = p < nS && v.mark[p] != 0;
    const unsigned bal = __ballot_sync(FULL, keep);
    if (p < nS) v.mark[p] = keep ? base + __popc(bal & ((1u << lane) - 1)) : -1;
    base += __popc(bal);
  }
  __syncwarp();
  bool bad = false;
  for (int p = lane; p < nS; p += 32) {
    const int id = v.mark[p];
    if (id < 0) continue;
    Rec r = v.rec[p];
    if (r.prev != NIL) {
      r.prev = v.mark[r.prev];
      bad |= r.prev < 0;
    }
    if (r.next != NIL) {
      r.next = v.mark[r.next];
      bad |= r.next < 0;
    }
    out.rec[L + id] = r;
    out.gid[L + id] = in.gid[p < nSL ? L + p : M + (p - nSL)];
  }
  for (int e = lane; e < k; e += 32) {
    Ev o = v.out[e];
    o.a = v.mark[o.a];
    o.b = v.mark[o.b];
    o.c = v.mark[o.c];
    bad |= (o.a < 0) | (o.b < 0) | (o.c < 0);
    out.ev[2 * L + e] = o;
  }
  if (__any_sync(FULL, bad) && lane == 0) raise_err(err, E_FASTPATH);
  if (lane == 0) out.hdr[gidx] = make_int2(base, k);
}

template <int TPB>
__global__ void __launch_bounds__(TPB) k_fast_level(GroupBuf in, GroupBuf out, long long n,
                                                    int level, int *deferred, int *ndeferred,
                                                    long long *err, int verify, int budget) {
  extern __shared__ __align__(16) unsigned char smem[];
  typedef cub::BlockScan<long long, TPB> Scan;
  __shared__ typename Scan::TempStorage scan_tmp;

  const long long size = 1ll << level, half = size >> 1;
  const long long jobs = (n + size - 1) >> level;
  const long long j = blockIdx.x * (long long)TPB + threadIdx.x;
  const long long L = j << level, M = L + half;
  const long long R = (L + size < n) ? L + size : n;
  const bool valid = j < jobs;
  bool pending = valid && (R - L > half);
  int nSL = 0, kL = 0, nSR = 0, kR = 0;
  long long f = 0;
  if (valid) {
    const int2 hl = in.hdr[2 * j];
    nSL = hl.x;
    kL = hl.y;
    if (pending) {
      const int2 hr = in.hdr[2 * j + 1];
      nSR = hr.x;
      kR = hr.y;
      f = job_bytes(nSL + nSR, kL + kR);
    }
    if (!pending || f > budget) {
      // carries and oversize jobs go to k_fast_big
      deferred[atomicAdd(ndeferred, 1)] = static_cast<int>(j);
      pending = false;
    }
  }
  const int lane = threadIdx.x & 31;
  while (__syncthreads_or(pending)) {
    long long off, total;
    Scan(scan_tmp).ExclusiveSum(pending ? f : 0ll, off, total);
    const bool active = pending && off + f <= budget;
    unsigned char *mine = smem + (active ? off : 0);
    // stage: the warp copies each active lane's child runs in turn
    unsigned todo = __ballot_sync(FULL, active);
    while (todo) {
      const int src = __ffs(todo) - 1;
      todo &= todo - 1;
      const long long sL = __shfl_sync(FULL, L, src), sM = __shfl_sync(FULL, M, src);
      const int snSL = __shfl_sync(FULL, nSL, src), snSR = __shfl_sync(FULL, nSR, src);
      const int skL = __shfl_sync(FULL, kL, src), skR = __shfl_sync(FULL, kR, src);
      const long long soff = __shfl_sync(FULL, off, src);
      stage_job(in, carve_job(smem + soff, snSL + snSR, skL, skR), sL, sM, snSL, snSR, skL, skR,
                lane, 32);
    }
    __syncwarp();
    long long k = 0;
    if (active) {
      JobView v = carve_job(mine, nSL + nSR, kL, kR);
      k = merge_compact(v.rec, nSL, nSL + nSR, v.evL, kL, 0, v.evR, kR, nSL, v.out,
                        2 * (nSL + nSR), v.mark, 2 * (R - L), R - L, verify != 0);
      if (k < 0) raise_err(err, k);
    }
    __syncwarp();
    // write-out: the warp compacts and stores each active lane's job in turn
    todo = __ballot_sync(FULL, active && k >= 0);
    while (todo) {
      const int src = __ffs(todo) - 1;
      todo &= todo - 1;
      const long long sL = __shfl_sync(FULL, L, src), sM = __shfl_sync(FULL, M, src);
      const int snSL = __shfl_sync(FULL, nSL, src), snSR = __shfl_sync(FULL, nSR, src);
      const int skL = __shfl_sync(FULL, kL, src), skR = __shfl_sync(FULL, kR, src);
      const long long soff = __shfl_sync(FULL, off, src);
      const int sk = static_cast<int>(__shfl_sync(FULL, k, src));
      const long long sj = __shfl_sync(FULL, j, src);
      writeout_job_warp(in, out, carve_job(smem + soff, snSL + snSR, skL, skR), sL, sM, snSL,
                        snSL + snSR, sk, sj, err);
    }
    pending = pending && !active;
    __syncthreads();
  }
}

// ---------------------------------------------------------------- big jobs
// One CTA per deferred job: carries are copied; merges are staged in this
// CTA's (large) shared memory when they fit, else run in place in global
// memory using the output group's own slot range as scratch.
template <int TPB>
__global__ void __launch_bounds__(TPB) k_fast_big(GroupBuf in, GroupBuf out, long long n,
                                                  int level, const int *deferred,
                                                  const int *ndeferred, long long *err,
                                                  int verify, int budget) {
  extern __shared__ __align__(16) unsigned char smem[];
  typedef cub::BlockScan<int, TPB> Scan;
  __shared__ typename Scan::TempStorage scan_tmp;
  __shared__ long long s_k;
  __shared__ int s_base;
  const int count = *ndeferred;
  const long long size = 1ll << level, half = size >> 1;
  for (int w = blockIdx.x; w < count; w += gridDim.x) {
    const long long j = deferred[w];
    const long long L = j << level, M = L + half;
    const long long R = (L + size < n) ? L + size : n;
    const int2 hl = in.hdr[2 * j];
    const int nSL = hl.x, kL = hl.y;
    if (R - L <= half) {  // carry (copy_log, parallel.py:107-108)
      for (int p = threadIdx.x; p < nSL; p += TPB) {
        out.rec[L + p] = in.rec[L + p];
        out.gid[L + p] = in.gid[L + p];
      }
      for (int e = threadIdx.x; e < kL; e += TPB) out.ev[2 * L + e] = in.ev[2 * L + e];
      if (threadIdx.x == 0) out.hdr[j] = hl;
      __syncthreads();
      continue;
    }
    const int2 hr = in.hdr[2 * j + 1];
    const int nSR = hr.x, kR = hr.y, nS = nSL + nSR;
    const bool in_smem = job_bytes(nS, kL + kR) <= budget;
    JobView v;
    const Ev *evL, *evR;
    if (in_smem) {
      v = carve_job(smem, nS, kL, kR);
      stage_job(in, v, L, M, nSL, nSR, kL, kR, threadIdx.x, TPB);
      evL = v.evL;
      evR = v.evR;
    } else {
      // global scratch inside the output group's slots: records at [L, L+nS)
      // (nS <= R-L), marks in the gid slots, merged events at [2L, 2L+2nS)
      v.rec = out.rec + L;
      v.mark = out.gid + L;
      v.out = out.ev + 2 * L;
      for (int p = threadIdx.x; p < nS; p += TPB) {
        Rec r;
        if (p < nSL) {
          r = in.rec[L + p];
        } else {
          r = in.rec[M + (p - nSL)];
          if (r.prev != NIL) r.prev += nSL;
          if (r.next != NIL) r.next += nSL;
        }
        v.rec[p] = r;
        v.mark[p] = 0;
      }
      evL = in.ev + 2 * L;
      evR = in.ev + 2 * M;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      s_k = merge_compact(v.rec, nSL, nS, evL, kL, 0, evR, kR, nSL, v.out, 2 * nS, v.mark,
                          2 * (R - L), R - L, verify != 0);
      if (s_k < 0) raise_err(err, s_k);
    }
    __syncthreads();
    const long long k = s_k;
    if (k < 0) continue;
    // new ids by a chunked block scan (in order, so in-place is safe)
    if (threadIdx.x == 0) s_base = 0;
    __syncthreads();
    for (int p0 = 0; p0 < nS; p0 += TPB) {
      const int p = p0 + threadIdx.x;
      const int keep = (p < nS && v.mark[p] != 0) ? 1 : 0;
      int pre, tot;
      Scan(scan_tmp).ExclusiveSum(keep, pre, tot);
      const int base = s_base;
      __syncthreads();
      if (p < nS) v.mark[p] = keep ? base + pre : -1;
      if (threadIdx.x == 0) s_base = base + tot;
      __syncthreads();
    }
    const int nKeep = s_base;
    int bad = 0;
    // events first (they read arbitrary marks), in place
    for (long long e = threadIdx.x; e < k; e += TPB) {
      Ev o = v.out[e];
      o.a = v.mark[o.a];
      o.b = v.mark[o.b];
      o.c = v.mark[o.c];
      bad |= (o.a < 0) | (o.b < 0) | (o.c < 0);
      out.ev[2 * L + e] = o;
    }
    // links next (they read arbitrary marks), in place
    for (int p = threadIdx.x; p < nS; p += TPB) {
      if (v.mark[p] < 0) continue;
      Rec &r = v.rec[p];
      if (r.prev != NIL) {
        r.prev = v.mark[r.prev];
        bad |= r.prev < 0;
      }
      if (r.next != NIL) {
        r.next = v.mark[r.next];
        bad |= r.next < 0;
      }
    }
    __syncthreads();
    // records + gids: chunked read-all / sync / write (destinations <= sources,
    // and a gid write only lands on marks already consumed)
    for (int p0 = 0; p0 < nS; p0 += TPB) {
      const int p = p0 + threadIdx.x;
      int id = -1;
      Rec r;
      int g = 0;
      if (p < nS) {
        id = v.mark[p];
        if (id >= 0) {
          r = v.rec[p];
          g = in.gid[p < nSL ? L + p : M + (p - nSL)];
        }
      }
      __syncthreads();
      if (id >= 0) {
        out.rec[L + id] = r;
        out.gid[L + id] = g;
      }
      __syncthreads();
    }
    if (__syncthreads_or(bad) && threadIdx.x == 0) raise_err(err, E_FASTPATH);
    if (threadIdx.x == 0) out.hdr[j] = make_int2(nKeep, static_cast<int>(k));
    __syncthreads();
  }
}

// facets of both passes: lower block then upper block, sorted indices
__global__ void k_fast_extract(GroupBuf lo, GroupBuf up, int *faces, long long cap,
                               long long *counts, long long *err) {
  const int kLo = lo.hdr[0].y, kUp = up.hdr[0].y;
  long long F = (long long)kLo + kUp;
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    counts[0] = kLo;
    counts[1] = kUp;
    if (F > cap) raise_err(err, H3D_E_CAPACITY);
  }
  if (F > cap) F = 0;
  for (long long f = blockIdx.x * (long long)blockDim.x + threadIdx.x; f < F;
       f += (long long)gridDim.x * blockDim.x) {
    const GroupBuf &g = (f < kLo) ? lo : up;
    const Ev e = g.ev[f < kLo ? f : f - kLo];
    faces[3 * f] = g.gid[e.a];
    faces[3 * f + 1] = g.gid[e.b];
    faces[3 * f + 2] = g.gid[e.c];
  }
}

}  // namespace h3d

using namespace h3d;

namespace {

constexpr int kLevelTPB = 128;
constexpr int kBigTPB = 256;
constexpr int kLevelBudget = 96 * 1024;
constexpr int kBigBudget = 200 * 1024;
constexpr int kBigGrid = 296;

struct PassWS {
  GroupBuf A, B;
  int *deferred;
  int *ndeferred;  // one counter per level (64)
};

bool carve_pass(h3d_arena &ar, long long n, PassWS &w) {
  for (GroupBuf *g : {&w.A, &w.B}) {
    g->hdr = ar.take<int2>(n);
    g->rec = ar.take<Rec>(n);
    g->gid = ar.take<int>(n);
    g->ev = ar.take<Ev>(2 * n);
  }
  w.deferred = ar.take<int>(n);
  w.ndeferred = ar.take<int>(64);
  return ar.base == nullptr || w.ndeferred != nullptr;
}

bool g_attr_done = false;

}  // namespace

extern "C" {

size_t h3d_fast_pass_workspace_bytes(int64_t n) {
  if (n < 1) n = 1;
  h3d_arena ar(nullptr, 0);
  PassWS w;
  carve_pass(ar, n, w);
  return ar.used + 4096;
}

int64_t h3d_fast_pass(const double *sorted_pts, int64_t n, double zsign, void *workspace,
                      size_t workspace_bytes, int64_t *err_dev, int32_t verify, void *stream) {
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (n < 2 || n > (1ll << 30)) return H3D_E_ARG;
  h3d_arena ar(workspace, workspace_bytes);
  PassWS w;
  if (!carve_pass(ar, n, w)) return H3D_E_ARG;
  if (!g_attr_done) {
    if (h3d_check(cudaFuncSetAttribute(k_fast_level<kLevelTPB>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, kLevelBudget)) ||
        h3d_check(cudaFuncSetAttribute(k_fast_big<kBigTPB>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, kBigBudget)))
      return H3D_E_CUDA;
    g_attr_done = true;
  }
  long long *err = reinterpret_cast<long long *>(err_dev);
  cudaMemsetAsync(w.ndeferred, 0, sizeof(int) * 64, s);
  h3d_count_launches(1);
  k_fast_init<<<h3d_grid(n, 256) > 8192 ? 8192 : h3d_grid(n, 256), 256, 0, s>>>(sorted_pts, zsign,
                                                                                n, w.A);
  GroupBuf src = w.A, dst = w.B;
  int levels = 0;
  while ((1ll << levels) < n) ++levels;
  for (int lv = 1; lv <= levels; ++lv) {
    const long long jobs = (n + (1ll << lv) - 1) >> lv;
    void *ev = h3d_profiling() ? h3d_prof_begin(s) : nullptr;
    h3d_count_launches(2);
    k_fast_level<kLevelTPB><<<h3d_grid(jobs, kLevelTPB), kLevelTPB, kLevelBudget, s>>>(
        src, dst, n, lv, w.deferred + 0, w.ndeferred + lv, err, verify, kLevelBudget);
    k_fast_big<kBigTPB><<<kBigGrid, kBigTPB, kBigBudget, s>>>(
        src, dst, n, lv, w.deferred, w.ndeferred + lv, err, verify, kBigBudget);
    h3d_prof_end(ev, lv, zsign > 0 ? 0 : 1, s);
    GroupBuf t = src;
    src = dst;
    dst = t;
  }
  if (h3d_check(cudaGetLastError())) return H3D_E_CUDA;
  // the final group lives in `src`; report which buffer (0 = A, 1 = B)
  return (levels & 1) ? 1 : 0;
}

int64_t h3d_fast_extract(void *ws_lower, void *ws_upper, int64_t n, int64_t final_lower,
                         int64_t final_upper, int32_t *faces, int64_t cap, int64_t *counts_dev,
                         int64_t *err_dev, void *stream) {
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  h3d_arena a1(ws_lower, ~size_t(0) >> 1), a2(ws_upper, ~size_t(0) >> 1);
  PassWS w1, w2;
  carve_pass(a1, n, w1);
  carve_pass(a2, n, w2);
  GroupBuf lo = final_lower ? w1.B : w1.A;
  GroupBuf up = final_upper ? w2.B : w2.A;
  h3d_count_launches(1);
  k_fast_extract<<<1184, 256, 0, s>>>(lo, up, faces, cap,
                                      reinterpret_cast<long long *>(counts_dev),
                                      reinterpret_cast<long long *>(err_dev));
  if (h3d_check(cudaGetLastError())) return H3D_E_CUDA;
  return 0;
}

}  // extern "C"
