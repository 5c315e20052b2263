// big.cu -- time-split merge pipeline for levels with large merge jobs.
//
// A merge job of the reference (_merge_one, _ckernels.pyx:86-208) is a
// kinetic sweep over the time-merged child logs.  For a large job almost
// every child event is "passed through": it neither touches the bridge feet
// nor coincides with a bridge move (99.6% at a 2^18 sphere
// top merge), so its fate is decided by the bridge position at its time
// alone.  The pipeline therefore splits a job into
//
//   1. the merged child sequence S (merge path, one thread per element);
//   2. per-point incidence lists: every event of S that names the point as
//      a, b or c, in time order (one stable radix sort of (point, event)
//      pairs for the whole level), with the point's links after each event
//      (one thread per point) -- links of any point at any position of S in
//      one binary search;
//   3. the time axis cut into segments of SEG child events; each segment's
//      start bridge is found by a walk at the segment's start time (the
//      reference's _find_bridge walk with the kinetic turn test at time T,
//      evaluated through the reference's own rounded event times);
//   4. one thread per segment runs the sequential core: only the events of
//      S that touch the current feet (found through the feet's incidence
//      lists) and the bridge events.  Each segment's end bridge must equal
//      the next segment's start bridge, else the input goes to the exact
//      engine;
//   5. every child event is kept or hidden by the bridge at its time (the
//      reference's emission rule), the output log is the time-ordered union
//      with the bridge events (prefix sums + binary searches);
//   6. the merged group's start-of-time links are rebuilt (merged -inf chain
//      + each kept point's first facet) and compacted.
//
// All arrays are compact over the level's jobs of both passes (pass-major),
// so a level costs O(sum of group sizes), not O(n).
#include "fast.cuh"
#include "prims.cuh"

namespace h3d {

constexpr int SEG_MIN = 16;  // child events per time segment: chosen per level, >= SEG_MIN

struct IncE {  // one incidence of a point: event index in S + links after it
  double t;
  int idx;  // position in the job's S
  int prv, nxt;
  int pad;
};

struct BEv {  // a bridge event and the feet after it
  double t;
  int a, b, c, kind;
  int u, v;
};

constexpr unsigned long long LS_MASK = (1ull << 22) - 1;
constexpr unsigned long long LS_HP = 1ull << 44, LS_HN = 1ull << 45, LS_HEAD = 1ull << 46;

__host__ __device__ __forceinline__ unsigned long long ls_pack(int prv, int nxt, bool hp, bool hn,
                                                               bool head) {
  return (static_cast<unsigned long long>(prv) & LS_MASK) |
         ((static_cast<unsigned long long>(nxt) & LS_MASK) << 22) | (hp ? LS_HP : 0ull) |
         (hn ? LS_HN : 0ull) | (head ? LS_HEAD : 0ull);
}

struct LinkScanOp {
  __host__ __device__ __forceinline__ unsigned long long operator()(unsigned long long a,
                                                                    unsigned long long b) const {
    if (b & LS_HEAD) return b;
    unsigned long long r = a;  // keeps a's head flag
    if (b & LS_HP) r = (r & ~LS_MASK) | (b & LS_MASK) | LS_HP;
    if (b & LS_HN) r = (r & ~(LS_MASK << 22)) | (b & (LS_MASK << 22)) | LS_HN;
    return r;
  }
};

struct BigWS {
  // a replayed plan's level-fit flag (nullptr when measured): once set, by
  // this level's total check or an earlier replayed level, every kernel of
  // the pipeline returns at once (the host resumes, measured, from the
  // level that did not fit; its input buffer is intact)
  const long long *spec = nullptr;
  // per job (both passes, pass-major): J2 = 2 * jobs
  int *jkin, *jkinoff;   // child events of S, exclusive scan
  int *jns, *jnsoff;     // points, exclusive scan
  int *jseg, *jsegoff;   // time segments, exclusive scan
  int *jflag;            // 1 = merge job, 0 = carry/empty
  int2 *ju0v0;           // bridge at t = -inf
  int *jkout, *jkoutoff; // merged events, exclusive scan
  // per child event of S (compact)
  Ev *seq;
  int *em, *cpos;
  // incidences (3 per event)
  unsigned *k0, *k1, *v0, *v1;
  IncE *inc;
  unsigned long long *sc0, *sc1;  // segmented link scan (in, out)
  // per point (compact)
  int *ibeg, *iend;
  int *first, *keep, *newid;
  int2 *ltmp;
  int *pjob;   // job of each compact point
  int *gjob;   // job of each compact child event
  // per segment
  int2 *segst;
  int *bcnt, *boff;
  // bridge events: per-segment slabs (sweep) and the compact array
  BEv *slab;
  BEv *bev;
  // scalars: [0] total kin, [1] total points, [2] total segments, [3] total
  // bridge events, [4] total kout
  int *tot;
  void *tmp;
  size_t tmp_bytes;
  long long m;  // capacity in points
};

static bool carve_big(h3d_arena &ar, long long m, BigWS &b) {
  // m points per pass: each group log holds < 2 events per point, so both
  // passes' merged child logs hold < 4m events
  const long long EK = 4 * m + 64;     // child events (both passes)
  const long long EP = 2 * m + 64;     // points (both passes)
  const long long NJ = m + 64;         // jobs (both passes)
  const long long NS = EK / SEG_MIN + NJ;  // segments
  b.m = m;
  b.jkin = ar.take<int>(NJ + 1);
  b.jkinoff = ar.take<int>(NJ + 1);
  b.jns = ar.take<int>(NJ + 1);
  b.jnsoff = ar.take<int>(NJ + 1);
  b.jseg = ar.take<int>(NJ + 1);
  b.jsegoff = ar.take<int>(NJ + 1);
  b.jflag = ar.take<int>(NJ + 1);
  b.ju0v0 = ar.take<int2>(NJ + 1);
  b.jkout = ar.take<int>(NJ + 1);
  b.jkoutoff = ar.take<int>(NJ + 1);
  b.seq = ar.take<Ev>(EK);
  b.em = ar.take<int>(EK + 1);
  b.cpos = ar.take<int>(EK + 1);
  b.k0 = ar.take<unsigned>(3 * EK);
  b.k1 = ar.take<unsigned>(3 * EK);
  b.v0 = ar.take<unsigned>(3 * EK);
  b.v1 = ar.take<unsigned>(3 * EK);
  b.inc = ar.take<IncE>(3 * EK);
  b.sc0 = ar.take<unsigned long long>(3 * EK);
  b.sc1 = ar.take<unsigned long long>(3 * EK);
  b.ibeg = ar.take<int>(EP);
  b.iend = ar.take<int>(EP);
  b.first = ar.take<int>(EP);
  b.keep = ar.take<int>(EP + 1);
  b.newid = ar.take<int>(EP + 1);
  b.ltmp = ar.take<int2>(EP);
  b.pjob = ar.take<int>(EP);
  b.gjob = ar.take<int>(EK);
  b.segst = ar.take<int2>(NS + 1);
  b.bcnt = ar.take<int>(NS + 1);
  b.boff = ar.take<int>(NS + 1);
  b.slab = ar.take<BEv>(2 * EK);  // shared by the level's segments
  b.bev = ar.take<BEv>(EK);
  b.tot = ar.take<int>(16);
  // primitives' temp (prims.cuh): the largest of the sort and the scans
  size_t a = prim::rs_temp_bytes<unsigned>(3 * EK);
  const size_t c = prim::scan_temp_bytes<int>(EK + 1 > 2 * EP ? EK + 1 : 2 * EP);
  const size_t d = prim::scan_temp_bytes<unsigned long long>(3 * EK);
  if (d > a) a = d;
  b.tmp_bytes = (a > c ? a : c) + 256;
  b.tmp = ar.take<unsigned char>(b.tmp_bytes);
  return ar.base == nullptr || b.tmp != nullptr;
}

// points per pass the pipeline's scratch holds (~1.3 KB each): an eighth of
// the cloud, at least 2^21 -- the mid levels of a 2^27 mixed cloud need
// 2^24 (C5 levels 10-12: 22-28 ms on the lane kernel, 4-15 ms here)
long long big_capacity(long long n) {
  long long cap = n / 8 > (1ll << 21) ? n / 8 : (1ll << 21);
  if (const char *e = getenv("H3D_BIG_CAP")) cap = atoll(e);
  return n < cap ? n : cap;
}

size_t big_workspace_bytes(long long m) {
  h3d_arena ar(nullptr, 0);
  BigWS b;
  carve_big(ar, m, b);
  return ar.used + 4096;
}

// ------------------------------------------------------------ job context
struct JobRef {
  GroupBuf in, out;
  long long L, M, R;
  int nSL, nS, kL, kR;
  double zs;
};

__device__ __forceinline__ JobRef job_ref(const Pass2 &P, int jb, long long J, long long j0,
                                          int lv, long long n) {
  JobRef r;
  const int pass = jb >= J ? 1 : 0;
  const long long j = j0 + (jb - pass * J);
  r.in = pass ? P.in1 : P.in0;
  r.out = pass ? P.out1 : P.out0;
  r.zs = pass ? -1.0 : 1.0;
  r.L = j << lv;
  r.M = r.L + (1ll << (lv - 1));
  r.R = (r.L + (1ll << lv) < n) ? r.L + (1ll << lv) : n;
  const int2 hl = r.in.hdr[2 * j];
  r.nSL = hl.x;
  r.kL = hl.y;
  return r;
}

// largest jb with off[jb] <= x (off = exclusive scan, non-decreasing)
__device__ __forceinline__ int find_job(const int *off, int J2, int x) {
  int lo = 0, hi = J2 - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (off[mid] <= x) lo = mid; else hi = mid - 1;
  }
  return lo;
}

__device__ __forceinline__ int gid_of(const JobRef &r, int p) {
  return p < r.nSL ? r.in.gid[r.L + p] : r.in.gid[r.M + (p - r.nSL)];
}

__device__ __forceinline__ int2 minf_links(const JobRef &r, int p) {
  if (p < r.nSL) return r.in.lnk[r.L + p];
  int2 l = r.in.lnk[r.M + (p - r.nSL)];
  if (l.x != NIL) l.x += r.nSL;
  if (l.y != NIL) l.y += r.nSL;
  return l;
}

__device__ __forceinline__ P3 pt_of(const JobRef &r, const double *__restrict__ pts, int p) {
  return load_pt(pts, gid_of(r, p), r.zs);
}

__device__ __forceinline__ double evt_job(const JobRef &r, const double *__restrict__ pts, int a,
                                          int b, int c) {
  if (a == NIL || b == NIL || c == NIL) return INF;
  const P3 A = pt_of(r, pts, a), B = pt_of(r, pts, b), C = pt_of(r, pts, c);
  return evtime_xyz(A.x, A.y, A.z, B.x, B.y, B.z, C.x, C.y, C.z);
}

// ------------------------------------------------------------------ K1 jobs
__global__ void k_big_jobs(Pass2 P, long long n, int lv, long long j0, long long J, BigWS W,
                           long long *err) {
  if (W.spec && *reinterpret_cast<const volatile long long *>(W.spec) != 0) return;
  const long long J2 = 2 * J;
  for (long long jb = blockIdx.x * (long long)blockDim.x + threadIdx.x; jb < J2;
       jb += (long long)gridDim.x * blockDim.x) {
    const int pass = jb >= J ? 1 : 0;
    const long long j = j0 + (jb - pass * J);
    const GroupBuf in = pass ? P.in1 : P.in0;
    const GroupBuf out = pass ? P.out1 : P.out0;
    const long long size = 1ll << lv, half = size >> 1;
    const long long L = j << lv;
    const long long R_ = (L + size < n) ? L + size : n;
    const int2 hl = in.hdr[2 * j];
    int kin = 0, ns = 0, seg = 0, flag = 0;
    if (R_ - L > half) {
      const int2 hr = in.hdr[2 * j + 1];
      kin = hl.y + hr.y;
      ns = hl.x + hr.x;
      flag = 1;
      // stored events carry 21-bit local ids (fast.cuh kEvIdBits)
      if (ns >= kEvIdMax) raise_err(err, E_FASTPATH);
    } else if (L < n) {  // carry (copy_log, parallel.py:107-108)
      for (int p = 0; p < hl.x; ++p) {
        out.lnk[L + p] = in.lnk[L + p];
        out.gid[L + p] = in.gid[L + p];
      }
      for (int e = 0; e < hl.y; ++e) out.ev[2 * L + e] = in.ev[2 * L + e];
      out.hdr[j] = hl;
    }
    W.jkin[jb] = kin;
    W.jns[jb] = ns;
    W.jseg[jb] = seg;
    W.jflag[jb] = flag;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    W.jkin[J2] = 0;
    W.jns[J2] = 0;
    W.jseg[J2] = 0;
  }
}

// segments per job for the level's segment length
__global__ void k_big_segs(long long J, BigWS W, int seg_len) {
  if (W.spec && *reinterpret_cast<const volatile long long *>(W.spec) != 0) return;
  const int J2 = static_cast<int>(2 * J);
  for (int jb = blockIdx.x * blockDim.x + threadIdx.x; jb <= J2; jb += gridDim.x * blockDim.x) {
    int sg = 0;
    if (jb < J2 && W.jflag[jb]) {
      sg = (W.jkin[jb] + seg_len - 1) / seg_len;
      if (sg < 1) sg = 1;
    }
    W.jseg[jb] = sg;
  }
}

// -------------------------------------------- K2 merged child sequence S
// element d of job jb: merge path (left first on equal times), right ids
// shifted by nSL, side in bit 1 of kind; plus its three incidence entries
// (key = compact point index, value = compact event index)
__global__ void k_big_seq(Pass2 P, long long n, int lv, long long j0, long long J, BigWS W) {
  if (W.spec && *reinterpret_cast<const volatile long long *>(W.spec) != 0) return;
  const int J2 = static_cast<int>(2 * J);
  const int total = W.jkinoff[J2];
  for (int g = blockIdx.x * blockDim.x + threadIdx.x; g < total; g += gridDim.x * blockDim.x) {
    const int jb = find_job(W.jkinoff, J2, g);
    W.gjob[g] = jb;
    const JobRef r = job_ref(P, jb, J, j0, lv, n);
    const int d = g - W.jkinoff[jb];
    const int kL = r.kL, kR = W.jkin[jb] - kL;
    const EvP *evL = r.in.ev + 2 * r.L, *evR = r.in.ev + 2 * r.M;
    int lo = d - kR > 0 ? d - kR : 0, hi = d < kL ? d : kL;
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (evL[mid].t <= evR[d - mid - 1].t) lo = mid + 1; else hi = mid;
    }
    const int i = lo, jj = d - lo;
    Ev o;
    if (i < kL && (jj >= kR || evL[i].t <= evR[jj].t)) {
      o = evL[i];
    } else {
      o = evR[jj];
      o.a += r.nSL;
      o.b += r.nSL;
      o.c += r.nSL;
      o.kind |= 2;
    }
    W.seq[g] = o;
    const unsigned pb = static_cast<unsigned>(W.jnsoff[jb]);
    W.k0[3 * g] = pb + o.a;
    W.k0[3 * g + 1] = pb + o.b;
    W.k0[3 * g + 2] = pb + o.c;
    W.v0[3 * g] = W.v0[3 * g + 1] = W.v0[3 * g + 2] = static_cast<unsigned>(g);
  }
}

// job of every compact point (one binary search per point, reused by the
// fill, keep and write kernels)
__global__ void k_big_pjob(long long J, BigWS W) {
  if (W.spec && *reinterpret_cast<const volatile long long *>(W.spec) != 0) return;
  const int J2 = static_cast<int>(2 * J);
  const int total = W.jnsoff[J2];
  for (int x = blockIdx.x * blockDim.x + threadIdx.x; x < total; x += gridDim.x * blockDim.x)
    W.pjob[x] = find_job(W.jnsoff, J2, x);
}

// ------------------------------------------------ K4 incidence list bounds
__global__ void k_big_incidx(const unsigned *__restrict__ key, int E, BigWS W) {
  if (W.spec && *reinterpret_cast<const volatile long long *>(W.spec) != 0) return;
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < E; k += gridDim.x * blockDim.x) {
    const unsigned q = key[k];
    if (k == 0 || key[k - 1] != q) W.ibeg[q] = k;
    if (k == E - 1 || key[k + 1] != q) W.iend[q] = k + 1;
  }
}

// ------------------------------------ K5 links after each incidence (fill)
// A point's links after each of its incidences are a forward fill over its
// list: an event naming it as a sets its next, as c its prev, its own
// insertion sets both (its deletion sets nothing: _act never writes the
// deleted point's links).  One segmented inclusive scan over all lists:
// element = prv (22 bits) | nxt (22 bits) << 22 | has-prv << 44 |
// has-nxt << 45 | list-head << 46.
__global__ void k_big_fill_init(Pass2 P, long long n, int lv, long long j0, long long J, BigWS W,
                                const unsigned *__restrict__ key, const unsigned *__restrict__ val,
                                int E) {
  if (W.spec && *reinterpret_cast<const volatile long long *>(W.spec) != 0) return;
  const int J2 = static_cast<int>(2 * J);
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < E; k += gridDim.x * blockDim.x) {
    const int x = static_cast<int>(key[k]);
    const int jb = W.pjob[x];
    const int p = x - W.jnsoff[jb];
    const Ev e = W.seq[val[k]];
    const bool ins = (e.kind & 1) == EV_INS;
    int prv = 0, nxt = 0;
    bool hp = false, hn = false;
    if (e.a == p) {
      nxt = ins ? e.b : e.c;
      hn = true;
    } else if (e.c == p) {
      prv = ins ? e.b : e.a;
      hp = true;
    } else if (ins) {  // p inserted between a and c
      prv = e.a;
      nxt = e.c;
      hp = hn = true;
    }
    W.sc0[k] = ls_pack(prv, nxt, hp, hn, k == W.ibeg[x]);
  }
}

__global__ void k_big_fill_final(Pass2 P, long long n, int lv, long long j0, long long J, BigWS W,
                                 const unsigned *__restrict__ key, const unsigned *__restrict__ val,
                                 int E) {
  if (W.spec && *reinterpret_cast<const volatile long long *>(W.spec) != 0) return;
  const int J2 = static_cast<int>(2 * J);
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < E; k += gridDim.x * blockDim.x) {
    const int x = static_cast<int>(key[k]);
    const int jb = W.pjob[x];
    const int p = x - W.jnsoff[jb];
    const unsigned long long sv = W.sc1[k];
    int2 l = make_int2(NIL, NIL);
    if (!(sv & LS_HP) || !(sv & LS_HN)) l = minf_links(job_ref(P, jb, J, j0, lv, n), p);
    const int g = static_cast<int>(val[k]);
    IncE o;
    o.t = W.seq[g].t;
    o.idx = g - W.jkinoff[jb];
    o.prv = (sv & LS_HP) ? static_cast<int>(sv & LS_MASK) : l.x;
    o.nxt = (sv & LS_HN) ? static_cast<int>((sv >> 22) & LS_MASK) : l.y;
    W.inc[k] = o;
  }
}

// links of job-local point p after the first `pos` events of S
__device__ __forceinline__ int2 links_at(const JobRef &r, const BigWS &W, int pbase, int p,
                                         int pos) {
  const int b0 = W.ibeg[pbase + p], b1 = W.iend[pbase + p];
  int lo = b0, hi = b1;  // first entry with idx >= pos
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (W.inc[mid].idx < pos) lo = mid + 1; else hi = mid;
  }
  if (lo == b0) return minf_links(r, p);
  const IncE e = W.inc[lo - 1];
  return make_int2(e.prv, e.nxt);
}

__device__ __forceinline__ int first_at(const BigWS &W, int pbase, int p, int pos) {
  int lo = W.ibeg[pbase + p], hi = W.iend[pbase + p];
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (W.inc[mid].idx < pos) lo = mid + 1; else hi = mid;
  }
  return lo;
}

// kinetic turn of (a, b, c) just after time T (the bridge walk's test at
// time T): the sign of the xy determinant flips at the triple's event time,
// the reference's own rounded value (_evtime operand order)
__device__ __forceinline__ bool turn_neg_at(const JobRef &r, const double *__restrict__ pts,
                                            int a, int b, int c, double T) {
  const P3 A = pt_of(r, pts, a), B = pt_of(r, pts, b), C = pt_of(r, pts, c);
  const double den = turn_xy(A.x, A.y, B.x, B.y, C.x, C.y);
  const double tau = evtime_xyz(A.x, A.y, A.z, B.x, B.y, B.z, C.x, C.y, C.z);
  const bool crossed = tau <= T;
  return crossed ? den > 0.0 : den < 0.0;
}

// ------------------------------------------------ K6 segment start bridges
__global__ void k_big_walk(Pass2 P, const double *__restrict__ pts, long long n, int lv, long long j0,
                           long long J, BigWS W, int SEG, long long *err) {
  if (W.spec && *reinterpret_cast<const volatile long long *>(W.spec) != 0) return;
  const int J2 = static_cast<int>(2 * J);
  const int total = W.jsegoff[J2];
  for (int gs = blockIdx.x * blockDim.x + threadIdx.x; gs < total;
       gs += gridDim.x * blockDim.x) {
    const int jb = find_job(W.jsegoff, J2, gs);
    if (!W.jflag[jb]) continue;
    const JobRef r = job_ref(P, jb, J, j0, lv, n);
    const int s = gs - W.jsegoff[jb];
    const int pbase = W.jnsoff[jb], gbase = W.jkinoff[jb];
    const long long limit = W.jns[jb] + 2;
    int u = r.nSL - 1, v = r.nSL;
    long long moves = 0;
    bool bad = false;
    if (s == 0) {  // t = -inf: _find_bridge (_ckernels.pyx:63-83)
      P3 U = pt_of(r, pts, u), V = pt_of(r, pts, v);
      for (;;) {
        const int vn = minf_links(r, v).y;
        if (vn != NIL) {
          const P3 X = pt_of(r, pts, vn);
          if (turn_xy(U.x, U.y, V.x, V.y, X.x, X.y) < 0.0) {
            v = vn;
            V = X;
            if (++moves > limit) { bad = true; break; }
            continue;
          }
        }
        const int up = minf_links(r, u).x;
        if (up != NIL) {
          const P3 X = pt_of(r, pts, up);
          if (turn_xy(X.x, X.y, U.x, U.y, V.x, V.y) < 0.0) {
            u = up;
            U = X;
            if (++moves > limit) { bad = true; break; }
            continue;
          }
        }
        break;
      }
      W.ju0v0[jb] = make_int2(u, v);
    } else {  // just after the last child event before the segment
      // both candidate moves are evaluated every step (the v-advance wins,
      // as in _find_bridge): the lanes' load chains stay converged
      const int pos = s * SEG;
      const double T = W.seq[gbase + pos - 1].t;
      for (;;) {
        const int vn = links_at(r, W, pbase, v, pos).y;
        const int up = links_at(r, W, pbase, u, pos).x;
        const bool mv = vn != NIL && turn_neg_at(r, pts, u, v, vn, T);
        const bool mu = up != NIL && turn_neg_at(r, pts, up, u, v, T);
        if (!mv && !mu) break;
        if (mv) v = vn; else u = up;
        if (++moves > limit) { bad = true; break; }
      }
    }
    if (bad) raise_err(err, E_FASTPATH);
    W.segst[gs] = make_int2(u, v);
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) W.bcnt[total] = 0;
}

// -------------------------------------------- K7 segment sweeps (the core)
// One thread per segment: the reference's sweep restricted to the events
// that can change the bridge -- child events naming a foot (from the feet's
// incidence lists) and the bridge events themselves.  The feet, their four
// neighbours and their coordinates stay in registers.  The 32 segments of a
// warp step together (vote at the loop head) through a branch-light step:
// one shared binary search (the new foot's list: its links and its next
// incidence at once) and two coordinate loads, so the lanes' dependent load
// chains overlap instead of serialising on divergent branches.
//
// MODE 0: every segment; bridge events to its slab of `cap` entries
// (counting on past it); end bridge checked against the next segment's start
// bridge.  MODE 1: only the segments whose slab overflowed, written straight
// to the compact array.
template <int MODE>
__global__ void __launch_bounds__(128) k_big_sweep(Pass2 P, const double *__restrict__ pts,
                                                   long long n, int lv, long long j0, long long J,
                                                   BigWS W, int SEG, int cap, long long *err) {
  if (W.spec && *reinterpret_cast<const volatile long long *>(W.spec) != 0) return;
  const int J2 = static_cast<int>(2 * J);
  const int total = W.jsegoff[J2];
  const int gs = blockIdx.x * blockDim.x + threadIdx.x;
  bool active = gs < total;
  if (MODE == 1 && active && W.bcnt[gs] <= cap) active = false;
  int jb = 0;
  if (active) {
    jb = find_job(W.jsegoff, J2, gs);
    if (!W.jflag[jb]) {
      W.bcnt[gs] = 0;
      active = false;
    }
  }
  const bool valid = active;
  JobRef r;
  int s = 0, nseg = 0, pbase = 0, gbase = 0, pos0 = 0, pos1 = 0;
  double tend = INF, tcur = -INF;
  int u = 0, v = 0;
  if (active) {
    r = job_ref(P, jb, J, j0, lv, n);
    s = gs - W.jsegoff[jb];
    nseg = W.jseg[jb];
    pbase = W.jnsoff[jb];
    gbase = W.jkinoff[jb];
    const int kin = W.jkin[jb];
    pos0 = s * SEG;
    pos1 = (pos0 + SEG < kin) ? pos0 + SEG : kin;
    tend = (s == nseg - 1) ? INF : W.seq[gbase + pos1 - 1].t;
    tcur = (s == 0) ? -INF : W.seq[gbase + pos0 - 1].t;
    const int2 st = W.segst[gs];
    u = st.x;
    v = st.y;
  }
  int pos = pos0;
  int up = NIL, un = NIL, vp = NIL, vn = NIL, cu = 0, cv = 0, eu = 0, ev_ = 0;
  P3 U, V, UN, UP, VN, VP;
  U.x = U.y = U.z = 0.0;
  V = UN = UP = VN = VP = U;
  if (active) {
    const int2 lu = links_at(r, W, pbase, u, pos), lvv = links_at(r, W, pbase, v, pos);
    up = lu.x;
    un = lu.y;
    vp = lvv.x;
    vn = lvv.y;
    cu = first_at(W, pbase, u, pos);
    cv = first_at(W, pbase, v, pos);
    eu = W.iend[pbase + u];
    ev_ = W.iend[pbase + v];
    U = pt_of(r, pts, u);
    V = pt_of(r, pts, v);
    if (un != NIL) UN = pt_of(r, pts, un);
    if (up != NIL) UP = pt_of(r, pts, up);
    if (vn != NIL) VN = pt_of(r, pts, vn);
    if (vp != NIL) VP = pt_of(r, pts, vp);
  }
  double c2 = evt3(u, un, v, U, UN, V), c3 = evt3(up, u, v, UP, U, V);
  double c4 = evt3(u, v, vn, U, V, VN), c5 = evt3(u, vp, v, U, VP, V);
  if (!active) c2 = c3 = c4 = c5 = INF;
  int nb = 0;
  BEv *bout = W.bev;
  if (active) bout = MODE == 0 ? W.slab + static_cast<long long>(gs) * cap : W.bev + W.boff[gs];
  bool bad = false;
  IncE iu, iv;
  iu.t = iv.t = INF;
  iu.idx = iv.idx = 0x7fffffff;
  if (active && cu < eu) iu = W.inc[cu];
  if (active && cv < ev_) iv = W.inc[cv];
  while (__any_sync(FULL, active)) {
    const double tu = (iu.idx < pos1) ? iu.t : INF, tv = (iv.idx < pos1) ? iv.t : INF;
    double best = INF;
    int which = -1;
    if (tu > tcur && tu < best) { best = tu; which = 0; }
    if (tv > tcur && tv < best) { best = tv; which = 1; }
    if (c2 > tcur && c2 < best) { best = c2; which = 2; }
    if (c3 > tcur && c3 < best) { best = c3; which = 3; }
    if (c4 > tcur && c4 < best) { best = c4; which = 4; }
    if (c5 > tcur && c5 < best) { best = c5; which = 5; }
    if (which < 0 || best > tend) active = false;
    // exact ties break the reference's strict `t > oldt` order
    if (active && ((which != 0 && tu == best) || (which != 1 && tv == best) ||
                   (which != 2 && c2 == best) || (which != 3 && c3 == best) ||
                   (which != 4 && c4 == best) || (which != 5 && c5 == best))) {
      bad = true;
      active = false;
    }
    const bool touch = active && which <= 1;
    const bool bridge = active && which >= 2;
    const bool sideU = which == 0 || which == 2 || which == 3;
    // bridge: position after the child events before this time
    if (bridge) {
      int lo = pos, hi = pos1;
      while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (W.seq[gbase + mid].t < best) lo = mid + 1; else hi = mid;
      }
      pos = lo;
    } else if (touch) {
      pos = (sideU ? iu.idx : iv.idx) + 1;
    }
    // the new foot of a bridge move; its list: links now + next incidence
    const int nfoot = which == 2 ? un : which == 3 ? up : which == 4 ? vn : vp;
    int lo = 0, hi = 0;
    if (bridge) {
      lo = W.ibeg[pbase + nfoot];
      hi = W.iend[pbase + nfoot];
    }
    const int b0 = lo, b1 = hi;
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (W.inc[mid].idx < pos) lo = mid + 1; else hi = mid;
    }
    int2 fl = make_int2(NIL, NIL);
    if (bridge) fl = (lo == b0) ? minf_links(r, nfoot) : make_int2(W.inc[lo - 1].prv, W.inc[lo - 1].nxt);
    // register moves; the (at most two) points whose coordinates are new
    int q1 = NIL, q2 = NIL;
    BEv o;
    o.t = best;
    if (touch) {
      const IncE &e = sideU ? iu : iv;
      if (sideU) {
        if (e.nxt != un) { un = e.nxt; q1 = un; }
        if (e.prv != up) { up = e.prv; q2 = up; }
        ++cu;
      } else {
        if (e.nxt != vn) { vn = e.nxt; q1 = vn; }
        if (e.prv != vp) { vp = e.prv; q2 = vp; }
        ++cv;
      }
    } else if (bridge) {
      // the new foot takes both links from its list (the other one is the
      // old foot unless a child event deleted the old foot while it was a
      // foot -- a near-degenerate input)
      if (which == 2) {  // u advances: the new foot enters the merged chain
        o.a = u; o.b = un; o.c = v; o.kind = EV_INS;
        const int of = u;
        up = u; UP = U; u = un; U = UN; un = fl.y; q1 = un;
        if (fl.x != of) { up = fl.x; q2 = up; }
      } else if (which == 3) {  // u leaves the merged chain
        o.a = up; o.b = u; o.c = v; o.kind = EV_DEL;
        const int of = u;
        un = u; UN = U; u = up; U = UP; up = fl.x; q2 = up;
        if (fl.y != of) { un = fl.y; q1 = un; }
      } else if (which == 4) {  // v leaves the merged chain
        o.a = u; o.b = v; o.c = vn; o.kind = EV_DEL;
        const int of = v;
        vp = v; VP = V; v = vn; V = VN; vn = fl.y; q1 = vn;
        if (fl.x != of) { vp = fl.x; q2 = vp; }
      } else {  // v retreats: the new foot enters the merged chain
        o.a = u; o.b = vp; o.c = v; o.kind = EV_INS;
        const int of = v;
        vn = v; VN = V; v = vp; V = VP; vp = fl.x; q2 = vp;
        if (fl.y != of) { vn = fl.y; q1 = vn; }
      }
      if (sideU) {
        cu = lo;
        eu = b1;
      } else {
        cv = lo;
        ev_ = b1;
      }
      o.u = u;
      o.v = v;
      if (MODE == 1 || nb < cap) bout[nb] = o;
      ++nb;
    }
    // coordinates of the new neighbours (both loads issued together)
    P3 Q1 = U, Q2 = U;
    if (q1 != NIL) Q1 = pt_of(r, pts, q1);
    if (q2 != NIL) Q2 = pt_of(r, pts, q2);
    if (q1 != NIL) { if (sideU) UN = Q1; else VN = Q1; }
    if (q2 != NIL) { if (sideU) UP = Q2; else VP = Q2; }
    // the next incidence of the side's foot
    if (active && (touch || bridge)) {
      const int c = sideU ? cu : cv, e = sideU ? eu : ev_;
      IncE nx;
      nx.t = INF;
      nx.idx = 0x7fffffff;
      if (c < e) nx = W.inc[c];
      if (sideU) iu = nx; else iv = nx;
    }
    if (__any_sync(FULL, active)) {
      if (active) {
        c2 = evt3(u, un, v, U, UN, V);
        c3 = evt3(up, u, v, UP, U, V);
        c4 = evt3(u, v, vn, U, V, VN);
        c5 = evt3(u, vp, v, U, VP, V);
        tcur = best;
      }
    }
  }
  if (MODE == 0 && valid) {
    W.bcnt[gs] = nb;
    if (s + 1 < nseg) {
      const int2 nx = W.segst[gs + 1];
      if (nx.x != u || nx.y != v) bad = true;
    }
  }
  if (bad) raise_err(err, E_FASTPATH);
}

// slabs -> one time-ordered array per job (bev2 = compact bridge events)
__global__ void k_big_bcompact(long long J, BigWS W, int cap) {
  if (W.spec && *reinterpret_cast<const volatile long long *>(W.spec) != 0) return;
  const int J2 = static_cast<int>(2 * J);
  const int total = W.jsegoff[J2];
  for (int gs = blockIdx.x; gs < total; gs += gridDim.x) {
    const int nb = W.bcnt[gs];
    if (nb > cap) continue;  // re-swept straight into place
    const int o = W.boff[gs];
    for (int q = threadIdx.x; q < nb; q += blockDim.x)
      W.bev[o + q] = W.slab[static_cast<long long>(gs) * cap + q];
  }
}

// bridge events of job jb: [W.boff[first seg], W.boff[end seg])
__device__ __forceinline__ int2 job_bridges(const BigWS &W, int jb) {
  return make_int2(W.boff[W.jsegoff[jb]], W.boff[W.jsegoff[jb + 1]]);
}

// number of bridge events of [b0, b1) strictly before t
__device__ __forceinline__ int bridges_before(const BigWS &W, int b0, int b1, double t) {
  int lo = b0, hi = b1;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (W.bev[mid].t < t) lo = mid + 1; else hi = mid;
  }
  return lo - b0;
}

// ------------------------------------------ K8 child event kept or hidden
__global__ void k_big_emit(long long J, BigWS W, long long *err) {
  if (W.spec && *reinterpret_cast<const volatile long long *>(W.spec) != 0) return;
  const int J2 = static_cast<int>(2 * J);
  const int total = W.jkinoff[J2];
  for (int g = blockIdx.x * blockDim.x + threadIdx.x; g < total; g += gridDim.x * blockDim.x) {
    const int jb = W.gjob[g];
    const Ev e = W.seq[g];
    const int2 br = job_bridges(W, jb);
    const int nbf = bridges_before(W, br.x, br.y, e.t);
    int u, v;
    if (nbf == 0) {
      const int2 uv = W.ju0v0[jb];
      u = uv.x;
      v = uv.y;
    } else {
      const BEv &bb = W.bev[br.x + nbf - 1];
      u = bb.u;
      v = bb.v;
    }
    bool bad = (br.x + nbf < br.y && W.bev[br.x + nbf].t == e.t);
    if (g > W.jkinoff[jb] && W.seq[g - 1].t == e.t) bad = true;
    if (bad) raise_err(err, E_FASTPATH);
    // _merge_one cases 0/1: emit if outside the bridge (x order = id order)
    W.em[g] = ((e.kind & 2) == 0) ? (e.b < u) : (e.b > v);
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) W.em[total] = 0;
}

// ------------------------------------------- K10 merged output (unmapped)
__global__ void k_big_out(Pass2 P, long long n, int lv, long long j0, long long J, BigWS W, long long *err) {
  if (W.spec && *reinterpret_cast<const volatile long long *>(W.spec) != 0) return;
  const int J2 = static_cast<int>(2 * J);
  const int total = W.jkinoff[J2];
  const int nbtot = W.boff[W.jsegoff[J2]];
  const int stride = gridDim.x * blockDim.x;
  for (int g = blockIdx.x * blockDim.x + threadIdx.x; g < total + nbtot; g += stride) {
    if (g < total) {  // a kept child event
      if (!W.em[g]) continue;
      const int jb = W.gjob[g];
      const JobRef r = job_ref(P, jb, J, j0, lv, n);
      const Ev e = W.seq[g];
      const int2 br = job_bridges(W, jb);
      const int idx = (W.cpos[g] - W.cpos[W.jkinoff[jb]]) + bridges_before(W, br.x, br.y, e.t);
      if (idx > 2 * (r.R - r.L) - 2) {  // the reference's cap (k >= cap - 1)
        raise_err(err, H3D_E_OVERFLOW);
        continue;
      }
      Ev o = e;
      o.kind &= 1;
      r.out.ev[2 * r.L + idx] = o;
      atomicMin(W.first + W.jnsoff[jb] + e.b, idx);
    } else {  // a bridge event
      const int bi = g - total;
      // job of bridge event bi: the job whose bridge range holds it
      int lo = 0, hi = J2 - 1;
      while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (W.boff[W.jsegoff[mid]] <= bi) lo = mid; else hi = mid - 1;
      }
      const int jb = lo;
      const JobRef r = job_ref(P, jb, J, j0, lv, n);
      const BEv b = W.bev[bi];
      const int gbase = W.jkinoff[jb], kin = W.jkin[jb];
      int a = 0, z = kin;  // first child event after b.t
      while (a < z) {
        const int mid = (a + z) >> 1;
        if (W.seq[gbase + mid].t < b.t) a = mid + 1; else z = mid;
      }
      const int idx = (bi - W.boff[W.jsegoff[jb]]) + (W.cpos[gbase + a] - W.cpos[gbase]);
      if (idx > 2 * (r.R - r.L) - 2) {
        raise_err(err, H3D_E_OVERFLOW);
        continue;
      }
      Ev o;
      o.t = b.t;
      o.a = b.a;
      o.b = b.b;
      o.c = b.c;
      o.kind = b.kind;
      r.out.ev[2 * r.L + idx] = o;
      atomicMin(W.first + W.jnsoff[jb] + b.b, idx);
    }
  }
}

// kout per job (kept child + bridge events)
__global__ void k_big_kout(long long J, BigWS W) {
  if (W.spec && *reinterpret_cast<const volatile long long *>(W.spec) != 0) return;
  const int J2 = static_cast<int>(2 * J);
  for (int jb = blockIdx.x * blockDim.x + threadIdx.x; jb < J2; jb += gridDim.x * blockDim.x) {
    const int g0 = W.jkinoff[jb], g1 = W.jkinoff[jb + 1];
    const int2 br = job_bridges(W, jb);
    W.jkout[jb] = W.jflag[jb] ? (W.cpos[g1] - W.cpos[g0]) + (br.y - br.x) : 0;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) W.jkout[J2] = 0;
}

// ------------------------------------------- K11 kept points + old links
__global__ void k_big_keep(Pass2 P, long long n, int lv, long long j0, long long J, BigWS W) {
  if (W.spec && *reinterpret_cast<const volatile long long *>(W.spec) != 0) return;
  const int J2 = static_cast<int>(2 * J);
  const int total = W.jnsoff[J2];
  for (int x = blockIdx.x * blockDim.x + threadIdx.x; x < total; x += gridDim.x * blockDim.x) {
    const int jb = W.pjob[x];
    const JobRef r = job_ref(P, jb, J, j0, lv, n);
    const int p = x - W.jnsoff[jb];
    const int2 uv = W.ju0v0[jb];
    const int2 l = minf_links(r, p);
    bool chain = p == 0 || p == r.nSL;
    if (!chain && l.x != NIL) chain = minf_links(r, l.x).y == p;
    chain = chain && (p < r.nSL ? p <= uv.x : p >= uv.y);
    const int f = W.first[x];
    const bool kept = chain || f != 0x7fffffff;
    int2 o = make_int2(NIL, NIL);
    if (chain) {
      o = l;
      if (p == uv.x) o.y = uv.y;
      if (p == uv.y) o.x = uv.x;
    } else if (kept) {
      const Ev e = r.out.ev[2 * r.L + f];
      o = make_int2(e.a, e.c);
    }
    W.keep[x] = kept ? 1 : 0;
    W.ltmp[x] = o;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) W.keep[total] = 0;
}

// ------------------------------------ K13 compacted links, gids, events
__global__ void k_big_write(Pass2 P, long long n, int lv, long long j0, long long J, BigWS W,
                            long long *err) {
  if (W.spec && *reinterpret_cast<const volatile long long *>(W.spec) != 0) return;
  const int J2 = static_cast<int>(2 * J);
  const int ptot = W.jnsoff[J2];
  const int etot = W.jkoutoff[J2];
  const int stride = gridDim.x * blockDim.x;
  bool bad = false;
  for (int x = blockIdx.x * blockDim.x + threadIdx.x; x < ptot + etot; x += stride) {
    if (x < ptot) {
      if (!W.keep[x]) continue;
      const int jb = W.pjob[x];
      const JobRef r = job_ref(P, jb, J, j0, lv, n);
      const int pb = W.jnsoff[jb], nb = W.newid[pb];
      const int p = x - pb;
      const int2 l = W.ltmp[x];
      int2 o;
      o.x = l.x == NIL ? NIL : W.newid[pb + l.x] - nb;
      o.y = l.y == NIL ? NIL : W.newid[pb + l.y] - nb;
      if ((l.x != NIL && !W.keep[pb + l.x]) || (l.y != NIL && !W.keep[pb + l.y])) bad = true;
      const int id = W.newid[x] - nb;
      r.out.lnk[r.L + id] = o;
      r.out.gid[r.L + id] = gid_of(r, p);
      if (p == 0) {
        const int cnt = W.newid[pb + W.jns[jb]] - nb;
        r.out.hdr[r.L >> lv] = make_int2(cnt, W.jkout[jb]);
      }
    } else {
      const int y = x - ptot;
      const int jb = find_job(W.jkoutoff, J2, y);
      const JobRef r = job_ref(P, jb, J, j0, lv, n);
      const int e = y - W.jkoutoff[jb];
      const int pb = W.jnsoff[jb], nb = W.newid[pb];
      Ev o = r.out.ev[2 * r.L + e];
      if (!W.keep[pb + o.a] || !W.keep[pb + o.b] || !W.keep[pb + o.c]) bad = true;
      o.a = W.newid[pb + o.a] - nb;
      o.b = W.newid[pb + o.b] - nb;
      o.c = W.newid[pb + o.c] - nb;
      r.out.ev[2 * r.L + e] = o;
    }
  }
  if (bad) raise_err(err, E_FASTPATH);
}

__global__ void k_big_fill_first(BigWS W, int total) {
  if (W.spec && *reinterpret_cast<const volatile long long *>(W.spec) != 0) return;
  for (int x = blockIdx.x * blockDim.x + threadIdx.x; x < total; x += gridDim.x * blockDim.x) {
    W.first[x] = 0x7fffffff;
    W.ibeg[x] = 0;
    W.iend[x] = 0;
  }
}

// ------------------------------------------------------------------- host
static unsigned grid_of(long long work) {
  long long g = (work + 255) / 256;
  if (g < 1) g = 1;
  if (g > 148 * 16) g = 148 * 16;
  return static_cast<unsigned>(g);
}

// a replayed level: the totals the plan recorded must be this cloud's
__global__ void k_big_check(const int *kin_dev, const int *pts_dev, long long kin, long long pts, int lv,
                            long long *spec) {
  if (*kin_dev != kin || *pts_dev != pts)
    atomicCAS(reinterpret_cast<unsigned long long *>(spec), 0ull, static_cast<unsigned long long>(lv));
}

// kin_total / pts_total: the level's merged child events and points (both
// passes) from the caller's measurement -- then the level reads nothing back:
// the segment kernels size their grids from an upper bound of the segment
// count and take the exact count from the device scan
long long big_level(const Pass2 &P, void *big_ws, size_t big_bytes, const double *pts,
                    long long n, int lv, long long j0, long long j1, long long *err,
                    cudaStream_t s, long long kin_total, long long pts_total, long long *spec) {
  h3d_arena ar(big_ws, big_bytes);
  BigWS W;
  if (!big_ws || !carve_big(ar, big_capacity(n), W)) return 1;
  W.spec = spec;
  const long long J = j1 - j0;
  const long long J2 = 2 * J;
  if (J2 + 1 > W.m + 64) return 1;
  auto scan = [&](int *in, int *out, long long items) -> bool {
    h3d_count_launches(1);
    return h3d_check(prim::scan<true, int>(W.tmp, W.tmp_bytes, in, out, items, prim::OpSum(), 0, 0, s));
  };
  h3d_count_launches(1);
  k_big_jobs<<<grid_of(J2), 256, 0, s>>>(P, n, lv, j0, J, W, err);
  if (scan(W.jkin, W.jkinoff, J2 + 1) || scan(W.jns, W.jnsoff, J2 + 1)) return H3D_E_CUDA;
  // totals: the level must fit the scratch
  int tot[3] = {0, 0, 0};
  const bool known = kin_total >= 0 && pts_total >= 0;
  if (!known &&
      (h3d_check(cudaMemcpyAsync(&tot[0], W.jkinoff + J2, sizeof(int), cudaMemcpyDeviceToHost, s)) ||
       h3d_check(cudaMemcpyAsync(&tot[1], W.jnsoff + J2, sizeof(int), cudaMemcpyDeviceToHost, s)) ||
       h3d_check(h3d_sync(s))))
    return H3D_E_CUDA;
  const long long kin = known ? kin_total : tot[0], pts_n = known ? pts_total : tot[1];
  if (spec) {  // replayed: this cloud's totals must be the recorded ones
    h3d_count_launches(1);
    k_big_check<<<1, 1, 0, s>>>(W.jkinoff + J2, W.jnsoff + J2, kin, pts_n, lv, spec);
  }
  // segment length: enough segments to give every SM a few warps
  static long long segs_per_sm = -1;
  if (segs_per_sm < 0) {
    segs_per_sm = 512;
    if (const char *e = getenv("H3D_BIG_SEGS")) segs_per_sm = atoll(e);
  }
  long long SEG = kin / (148 * segs_per_sm) + 1;
  if (SEG < SEG_MIN) SEG = SEG_MIN;
  h3d_count_launches(1);
  k_big_segs<<<grid_of(J2 + 1), 256, 0, s>>>(J, W, static_cast<int>(SEG));
  if (scan(W.jseg, W.jsegoff, J2 + 1)) return H3D_E_CUDA;
  // segments: sum over jobs of ceil(kin_j / SEG) (at least one per merge)
  // <= kin / SEG + J2; with the totals known that bound sizes the grids
  // (every segment kernel reads the exact count, jsegoff[J2], on the device)
  long long nseg = kin / SEG + J2;
  if (!known) {
    if (h3d_check(cudaMemcpyAsync(&tot[2], W.jsegoff + J2, sizeof(int), cudaMemcpyDeviceToHost, s)) ||
        h3d_check(h3d_sync(s)))
      return H3D_E_CUDA;
    nseg = tot[2];
  }
  if (kin > 4 * W.m || pts_n > 2 * W.m || nseg > 4 * W.m / SEG_MIN + W.m) {
    // carries were already copied; the caller reruns the level elsewhere
    return 1;
  }
  h3d_count_launches(9);
  k_big_fill_first<<<grid_of(pts_n), 256, 0, s>>>(W, static_cast<int>(pts_n));
  k_big_pjob<<<grid_of(pts_n), 256, 0, s>>>(J, W);
  k_big_seq<<<grid_of(kin), 256, 0, s>>>(P, n, lv, j0, J, W);
  // incidence lists: stable sort of (point, event) pairs by point
  {
    int bits = 1;
    while ((1ll << bits) < pts_n + 1) ++bits;
    bool alt = false;
    h3d_count_launches((bits + 7) / 8 + 1);
    if (h3d_check(prim::rs_sort_pairs<unsigned>(W.tmp, W.tmp_bytes, W.k0, reinterpret_cast<int *>(W.v0), W.k1,
                                                reinterpret_cast<int *>(W.v1), 3 * kin, 0, bits, &alt, s)))
      return H3D_E_CUDA;
    const unsigned *kcur = alt ? W.k1 : W.k0;
    const unsigned *vcur = alt ? W.v1 : W.v0;
    k_big_incidx<<<grid_of(3 * kin), 256, 0, s>>>(kcur, static_cast<int>(3 * kin), W);
    k_big_fill_init<<<grid_of(3 * kin), 256, 0, s>>>(P, n, lv, j0, J, W, kcur, vcur,
                                                    static_cast<int>(3 * kin));
    h3d_count_launches(1);
    if (h3d_check(prim::scan<false, unsigned long long>(W.tmp, W.tmp_bytes, W.sc0, W.sc1, 3 * kin,
                                                        LinkScanOp(), 0ull, 0ull, s)))
      return H3D_E_CUDA;
    k_big_fill_final<<<grid_of(3 * kin), 256, 0, s>>>(P, n, lv, j0, J, W, kcur, vcur,
                                                     static_cast<int>(3 * kin));
  }
  k_big_walk<<<grid_of(nseg), 256, 0, s>>>(P, pts, n, lv, j0, J, W, static_cast<int>(SEG), err);
  {
    // bridge-event slabs: the level's segments share 2*EK entries
    long long cap = (8 * W.m + 128) / (nseg > 0 ? nseg : 1);
    if (cap > 1024) cap = 1024;
    if (cap < 1) cap = 1;
    // the segment count is an upper bound when the totals came from the
    // measurement: counts past the real segments must read as zero in the
    // scan of the slab sizes
    if (known) cudaMemsetAsync(W.bcnt, 0, sizeof(int) * (nseg + 1), s);
    h3d_count_launches(3);
    const unsigned gsw = static_cast<unsigned>((nseg + 127) / 128 > 0 ? (nseg + 127) / 128 : 1);
    k_big_sweep<0><<<gsw, 128, 0, s>>>(P, pts, n, lv, j0, J, W, static_cast<int>(SEG), static_cast<int>(cap), err);
    if (scan(W.bcnt, W.boff, nseg + 1)) return H3D_E_CUDA;
    k_big_sweep<1><<<gsw, 128, 0, s>>>(P, pts, n, lv, j0, J, W, static_cast<int>(SEG), static_cast<int>(cap), err);
    const unsigned gb = nseg < 148 * 32 ? static_cast<unsigned>(nseg > 0 ? nseg : 1) : 148 * 32;
    k_big_bcompact<<<gb, 128, 0, s>>>(J, W, static_cast<int>(cap));
  }
  k_big_emit<<<grid_of(kin), 256, 0, s>>>(J, W, err);
  if (scan(W.em, W.cpos, kin + 1)) return H3D_E_CUDA;
  k_big_out<<<grid_of(kin + kin), 256, 0, s>>>(P, n, lv, j0, J, W, err);
  h3d_count_launches(3);
  k_big_kout<<<grid_of(J2), 256, 0, s>>>(J, W);
  if (scan(W.jkout, W.jkoutoff, J2 + 1)) return H3D_E_CUDA;
  k_big_keep<<<grid_of(pts_n), 256, 0, s>>>(P, n, lv, j0, J, W);
  if (scan(W.keep, W.newid, pts_n + 1)) return H3D_E_CUDA;
  k_big_write<<<grid_of(pts_n + 2 * kin), 256, 0, s>>>(P, n, lv, j0, J, W, err);
  if (h3d_check(cudaGetLastError())) return H3D_E_CUDA;
  return 0;
}

}  // namespace h3d
