// fast.cuh -- data layout and merge routines of the fused fast path.
//
// Layout in HBM (per pass, double-buffered A/B):
//   hdr[g]              int2 (nS, k) of group g at the current level
//   lnk[L .. L+nS)      int2 chain links prev/next of each kept point as
//                       GROUP-LOCAL ids (NIL = -1), at the group's
//                       start-of-time (t = -inf) state
//   gid[L .. L+nS)      global sorted index of each kept point: its
//                       coordinates are read from the sorted point array
//                       (never copied between levels)
//   ev[2L .. 2L+k)      EvP (16 B): event time t (f64), the facet (a, b, c)
//                       of the event in group-local ids (21 bits each) and
//                       its kind (insertion / deletion); b is the
//                       reference's log entry
// A group [L, R) keeps only the points that matter above it: its chain at
// t = -inf plus every point its log mentions.  Local ids preserve x order, so
// the reference's x comparisons become integer comparisons (x is strictly
// increasing, store.py:70-71).
#pragma once
#include "h3d_device.cuh"

namespace h3d {

// shared-memory record of the warp-per-job merge: coordinates (z negated on
// the upper pass) and the chain links as group-local ids
struct __align__(8) Rec {
  double x, y, z;
  int prev, next;
};

struct __align__(8) Ev {
  double t;
  int a, b, c, kind;  // kind: 0 = b inserted between a and c, 1 = b deleted
};

static_assert(sizeof(Rec) == 32, "Rec must be one 32-byte sector");
static_assert(sizeof(Ev) == 24, "Ev is 24 bytes");

// Group-local ids in the stored events are < 2^21: a merge whose two children
// keep 2^21 points or more declines (E_FASTPATH, the exact engine takes the
// hull) -- far above every configured cloud's top groups (<= 1.03M kept).
constexpr int kEvIdBits = 21;
constexpr int kEvIdMax = 1 << kEvIdBits;

// An event as stored in the group buffers (HBM): 16 bytes, the time and one
// word with the facet's three local ids (21 bits each) and the kind (bit 63).
// Converts to and from the unpacked Ev the kernels compute with.
struct __align__(16) EvP {
  double t;
  unsigned long long w;
  EvP() = default;
  __host__ __device__ __forceinline__ EvP(const Ev &e)
      : t(e.t),
        w(static_cast<unsigned long long>(static_cast<unsigned>(e.a)) |
          (static_cast<unsigned long long>(static_cast<unsigned>(e.b)) << kEvIdBits) |
          (static_cast<unsigned long long>(static_cast<unsigned>(e.c)) << (2 * kEvIdBits)) |
          (static_cast<unsigned long long>(e.kind & 1) << 63)) {}
  __host__ __device__ __forceinline__ int a() const { return static_cast<int>(w & (kEvIdMax - 1)); }
  __host__ __device__ __forceinline__ int b() const {
    return static_cast<int>((w >> kEvIdBits) & (kEvIdMax - 1));
  }
  __host__ __device__ __forceinline__ int c() const {
    return static_cast<int>((w >> (2 * kEvIdBits)) & (kEvIdMax - 1));
  }
  __host__ __device__ __forceinline__ int kind() const { return static_cast<int>(w >> 63); }
  __host__ __device__ __forceinline__ operator Ev() const {
    Ev e;
    e.t = t;
    e.a = a();
    e.b = b();
    e.c = c();
    e.kind = kind();
    return e;
  }
};
static_assert(sizeof(EvP) == 16, "EvP is 16 bytes");

struct GroupBuf {
  int2 *hdr;  // (nS, k) per group
  int2 *lnk;  // start-of-time links (group-local ids) per kept point
  int *gid;   // global sorted index per kept point
  EvP *ev;    // events, 2 slots per point
};

// both passes of a level in one launch: blockIdx.y = 0 lower, 1 upper
struct Pass2 {
  GroupBuf in0, in1, out0, out1;
};

constexpr unsigned FULL = 0xffffffffu;

// Which pass and which block of jobs a CTA of a level launch covers.  Grid
// (g, 2): blockIdx.y is the pass (all lower-pass CTAs are scheduled before
// the upper-pass ones); grid (2g, 1): the two passes of the same jobs are
// adjacent CTAs, so the rows both read (the same sorted points, z negated on
// the upper pass) are fetched from DRAM once and hit in L2 for the other.
__device__ __forceinline__ int lvl_pass() { return gridDim.y == 2 ? blockIdx.y : (blockIdx.x & 1); }
__device__ __forceinline__ long long lvl_blk() {
  return gridDim.y == 2 ? static_cast<long long>(blockIdx.x) : static_cast<long long>(blockIdx.x >> 1);
}
inline dim3 lvl_grid(unsigned g, bool interleave) { return interleave ? dim3(2 * g, 1) : dim3(g, 2); }
extern int g_interleave;  // H3D_INTERLEAVE: pass-interleaved level grids
constexpr int FIRST_FLAG = 1 << 30;        // "on a child's -inf chain"
constexpr int FIRST_NONE = FIRST_FLAG - 1; // no event yet

__host__ __device__ __forceinline__ long long align8(long long b) { return (b + 7) & ~7ll; }
__host__ __device__ __forceinline__ long long align16(long long b) { return (b + 15) & ~15ll; }

// coordinates of sorted point g; z negated on the upper pass (exact)
struct P3 {
  double x, y, z;
};
__device__ __forceinline__ P3 load_pt(const double *__restrict__ pts, int g, double zs) {
  P3 r;
  r.x = __ldg(pts + 3ll * g);
  r.y = __ldg(pts + 3ll * g + 1);
  r.z = zs * __ldg(pts + 3ll * g + 2);
  return r;
}

__device__ __forceinline__ double evt3(int a, int b, int c, const P3 &A, const P3 &B, const P3 &C) {
  if (a == NIL || b == NIL || c == NIL) return INF;
  return evtime_xyz(A.x, A.y, A.z, B.x, B.y, B.z, C.x, C.y, C.z);
}

constexpr int EV_INS = 0;
constexpr int EV_DEL = 1;

// fast path could not reproduce the reference semantics: rerun exact
constexpr long long E_FASTPATH = -13;

__device__ __forceinline__ double evt_rec(const Rec *R, int a, int b, int c) {
  if (a == NIL || b == NIL || c == NIL) return INF;
  const Rec &A = R[a], &B = R[b], &C = R[c];
  return evtime_xyz(A.x, A.y, A.z, B.x, B.y, B.z, C.x, C.y, C.z);
}

// _act (_ckernels.pyx:49-60) on local links; returns the kind or -1 on a
// NIL neighbour
__device__ __forceinline__ int act_rec(Rec *R, int e) {
  const int p = R[e].prev, q = R[e].next;
  if (p == NIL || q == NIL) return -1;
  if (R[p].next == e) {
    R[p].next = q;
    R[q].prev = p;
    return EV_DEL;
  }
  R[p].next = e;
  R[q].prev = e;
  return EV_INS;
}

// _find_bridge (_ckernels.pyx:63-83) on local ids
__device__ __forceinline__ int bridge_rec(const Rec *R, int *pu, int *pv, long long limit) {
  int u = *pu, v = *pv;
  long long moves = 0;
  for (;;) {
    const int vn = R[v].next;
    bool moved = false;
    if (vn != NIL && turn_xy(R[u].x, R[u].y, R[v].x, R[v].y, R[vn].x, R[vn].y) < 0.0) {
      v = vn;
      moved = true;
    } else {
      const int up = R[u].prev;
      if (up != NIL && turn_xy(R[up].x, R[up].y, R[u].x, R[u].y, R[v].x, R[v].y) < 0.0) {
        u = up;
        moved = true;
      }
    }
    if (!moved) {
      *pu = u;
      *pv = v;
      return 0;
    }
    if (++moves > limit) return -1;
  }
}

// lane-per-job merge (lane.cu): a job's shared-memory slice is
//   [XYZ: x, y, z f64 per point] lk short2, gd int, fi u32 per point,
//   then ot f64 + ow u64 per staged output event (16-byte aligned pieces)
__host__ __device__ __forceinline__ int lane_pt_bytes(bool xyz) { return xyz ? 36 : 12; }
// staged output capacity of a job: its child events plus a margin (a merged
// log is rarely much longer than its children's; the rest spills to HBM)
__host__ __device__ __forceinline__ int lane_ocap(int nS, int kin) { return kin + (nS >> 2) + 4; }
__host__ __device__ __forceinline__ int lane_slice_bytes(int nS, int ocap, bool xyz) {
  return static_cast<int>(align16((long long)lane_pt_bytes(xyz) * nS) + 16ll * ocap);
}

}  // namespace h3d

// ---------------------------------------------------------------- host side
#include "h3d_host.h"

namespace h3d {

struct PassWS {
  GroupBuf A, B;
  Ev *seq;                  // merged child events of HBM-resident warp jobs (2n)
  Rec *rec;                 // records of HBM-resident warp jobs (n)
  unsigned long long *need; // thread-per-job pool sizing (+ the per-CTA need histogram)
  int *ovf;                 // CTAs of a split lane-per-job level left to the big-pool launch
  long long ovf_cap;
};
constexpr int kNeedWords = 48, kNeedHist = 64, kNeedHistBins = 128;  // need[64 .. 192): histogram
// a split lane-per-job level (fast.cu tpj_split): the overflow list, the big
// pool and its launch's grid, and the small pool
struct TpjSplit {
  int *ovf;
  long long cap;
  int pool, grid;
  long long small;
  int mini = -1;  // >= 0: the list goes to this mini variant (one CTA per job) instead
  void *scratch = nullptr;  // the huge variant's global-memory slots
  size_t scratch_bytes = 0;
};

inline bool carve_pass(h3d_arena &ar, long long n, PassWS &w) {
  for (GroupBuf *g : {&w.A, &w.B}) {
    g->hdr = ar.take<int2>(n);
    g->lnk = ar.take<int2>(n);
    g->gid = ar.take<int>(n);
    g->ev = ar.take<EvP>(2 * n);
  }
  w.seq = ar.take<Ev>(2 * n);
  w.rec = ar.take<Rec>(n);
  w.need = ar.take<unsigned long long>(kNeedHist + kNeedHistBins);
  w.ovf_cap = (n >> 4) + 64;
  w.ovf = ar.take<int>(w.ovf_cap + 1);
  return ar.base == nullptr || w.need != nullptr;
}


// Scratch of the time-split pipeline for large merge jobs (big.cu), carved
// from the lower pass's workspace; sized for m points (sum of group sizes
// of a level, both passes) -- levels above that use the warp kernel.
struct BigWS;
size_t big_workspace_bytes(long long m);
long long big_capacity(long long n);
// one merge level of both passes through the pipeline; returns 0, or 1 when
// the level does not fit the scratch (caller falls back), or a negative code
long long big_level(const Pass2 &P, void *big_ws, size_t big_bytes, const double *pts,
                    long long n, int lv, long long j0, long long j1, long long *err,
                    cudaStream_t s, long long kin_total = -1, long long pts_total = -1,
                    long long *spec = nullptr);

// one merge level of both passes, one CTA per job, all in shared memory
// (mini.cu): jobs of at most MINI_N points and MINI_K merged child events
// variant 0: jobs of <= 256 points and 512 child events (~40 KB, several
// CTAs per SM); variant 1: <= 1024 points and 2048 events (~154 KB)
// one level of both passes, one lane per job (lane.cu); need = the level's
// measurement (k_tpj_need); returns 0, 1 (does not fit) or a negative code
// the launch lane_level chose (variant v = 2 * xyz + staged, 32 >> r jobs per
// CTA, pool bytes): recorded in a level plan, replayed with need == nullptr
struct LaneCfg {
  int v, r;
  long long pool;
};
long long lane_level(const Pass2 &P, const double *pts, long long n, int lv, long long j0,
                     long long j1, long long *err, const unsigned long long *need,
                     cudaStream_t s, LaneCfg *cfg = nullptr, long long *spec = nullptr,
                     long long *stamp = nullptr);
extern long long g_lane_xyz_max;  // lane.cu knobs
extern int g_lane_stage;
extern int g_lane_own;
extern int g_lane_pf1, g_lane_pf2;

// variant 3 (huge): <= kMiniHugePoints / kMiniHugeEvents per job, the job's
// arrays in global-memory slots of gscratch (returns 1 when they do not fit)
size_t mini_huge_stride();  // bytes of one huge-variant global-memory slot
long long mini_level(const Pass2 &P, const double *pts, long long n, int lv, long long j0,
                     long long j1, long long *err, cudaStream_t s, int variant,
                     long long *spec = nullptr, long long *stamp = nullptr,
                     void *gscratch = nullptr, size_t gbytes = 0, const int *list = nullptr,
                     int list_grid = 0);
constexpr int kMiniMaxPoints = 1024, kMiniMaxEvents = 2048;
constexpr int kMiniHugePoints = 8192, kMiniHugeEvents = 16384;
constexpr int kMiniSmallPoints = 256, kMiniSmallEvents = 512;
constexpr int kMiniMedPoints = 320, kMiniMedEvents = 640;
constexpr int kMiniL2Points = 640, kMiniL2Events = 1280;
constexpr int kMiniXlPoints = 1152, kMiniXlEvents = 2304;
constexpr int kMiniTinyPoints = 192, kMiniTinyEvents = 320;
extern int g_mini_seglen;  // mini.cu: child events per time segment

}  // namespace h3d
