// fast.cu -- the fused fast path: all merge levels of a pass over compact groups.
//
// Level scheduler (parallel.py:68-112 on the device), no host synchronisation
// inside a pass; a device error word is read once per hull:
//
//  * k_fast_tpj    one launch per level while jobs are plentiful: one THREAD
//                  per merge job (merge_tpj, the reference's sequential sweep
//                  with cached candidate times), int16 links in a packed
//                  shared-memory slice, coordinates and child events streamed
//                  from HBM, merged events written straight back, and the
//                  start-of-time links rebuilt from the merged -inf chain and
//                  first events (no sequential rewind).
//  * k_fast_warp   one launch per level above the leaf.  One WARP per merge
//                  job (merge_warp): the kinetic sweep advances through the
//                  time-merged child logs 32 events at a time -- every event
//                  that neither touches the bridge feet nor comes after the
//                  next bridge event is retired in parallel (survivor
//                  emission by ballot prefix, link writes resolved
//                  last-writer-wins with __match_any_sync) -- and only foot
//                  events and bridge events are sequential.  The start-of-time
//                  links of the merged group are rebuilt in parallel (merged
//                  -inf chain + each point's first facet) instead of the
//                  reference's sequential rewind.  Jobs are staged in a
//                  shared-memory pool when they fit, else run in place in HBM.
//  * k_fast_extract  facets of both passes straight from the final events.
#include <cstdlib>

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

// both passes of a level in one launch: blockIdx.y = 0 lower, 1 upper
struct Pass2 {
  GroupBuf in0, in1, out0, out1;
};

constexpr unsigned FULL = 0xffffffffu;
constexpr int FIRST_FLAG = 1 << 30;        // "on a child's -inf chain"
constexpr int FIRST_NONE = FIRST_FLAG - 1; // no event yet

__host__ __device__ __forceinline__ long long align8(long long b) { return (b + 7) & ~7ll; }

// --------------------------------------------------------- thread per job
// level 0: every point is a one-point group with an empty log
__global__ void k_fast_init(const double *__restrict__ pts, long long p0, long long p1, Pass2 P) {
  const GroupBuf g = blockIdx.y ? P.in1 : P.in0;
  const double zs = blockIdx.y ? -1.0 : 1.0;
  for (long long i = p0 + blockIdx.x * (long long)blockDim.x + threadIdx.x; i < p1;
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

constexpr unsigned short INFO_CHAIN = 0x8000;  // on its child's -inf chain
constexpr unsigned short INFO_NONE = 0x7fff;   // no merged event yet

// Thread-per-job merge state: the job's records (coordinates + int16 links
// would not save a cycle on the dependency chain, so records stay 32 B) and
// its info table live in this thread's shared-memory slice.
struct TpjJob {
  Rec *R;                 // nS records, left [0,nSL), right [nSL,nS)
  unsigned short *info;   // nS: INFO_CHAIN | first merged event index
  int nSL;
};

// The reference's kinetic sweep (_merge_one phase 1, _ckernels.pyx:86-183)
// for one job on one thread, written branch-free so the 32 lanes of a warp
// (32 different jobs) stay converged: every lane evaluates the quantities of
// all six cases and selects; the four bridge candidates are recomputed every
// step.  Child candidate times are the stored times (the time the facet got
// when it was emitted one level down, same expression, same triple); events
// go straight to HBM with their facet and kind; each point's first merged
// event is recorded for the link rebuild that replaces the rewind.
// Returns k or a negative code.
__device__ long long merge_tpj(TpjJob &J, const Ev *__restrict__ evL, int kL,
                               const Ev *__restrict__ evR, int kR, Ev *out, long long capRef,
                               long long limitRef, int *pu0, int *pv0, unsigned mask) {
  Rec *R = J.R;
  const int nSL = J.nSL;
  int u = nSL - 1, v = nSL;
  const int bst = bridge_rec(R, &u, &v, limitRef);
  __syncwarp(mask);
  if (bst < 0) return H3D_E_BRIDGE;
  *pu0 = u;
  *pv0 = v;
  int i = 0, j = 0, k = 0;
  double tcur = -INF;
  double c0 = INF, c1 = INF;
  int bL = 0, bR = 0;
  Ev nL, nR;  // prefetched next child events
  nL.t = INF;
  nR.t = INF;
  if (kL > 0) {
    c0 = evL[0].t;
    bL = evL[0].b;
    if (kL > 1) nL = evL[1];
  }
  if (kR > 0) {
    c1 = evR[0].t;
    bR = evR[0].b + nSL;
    if (kR > 1) nR = evR[1];
  }
  double c2 = evt_rec(R, u, R[u].next, v);
  double c3 = evt_rec(R, R[u].prev, u, v);
  double c4 = evt_rec(R, u, v, R[v].next);
  double c5 = evt_rec(R, u, R[v].prev, v);
  int err = 0;
  for (;;) {
    double best = INF;
    int which = -1;
    if (c0 > tcur && c0 < best) { best = c0; which = 0; }
    if (c1 > tcur && c1 < best) { best = c1; which = 1; }
    if (c2 > tcur && c2 < best) { best = c2; which = 2; }
    if (c3 > tcur && c3 < best) { best = c3; which = 3; }
    if (c4 > tcur && c4 < best) { best = c4; which = 4; }
    if (c5 > tcur && c5 < best) { best = c5; which = 5; }
    if (which < 0) break;
    const bool left = which == 0, right = which == 1, child = which <= 1;
    const int e = left ? bL : (right ? bR : u);
    const int p = R[e].prev, q = R[e].next;
    const int un = R[u].next, up = R[u].prev, vn = R[v].next, vp = R[v].prev;
    const bool nilnb = (p == NIL) | (q == NIL);
    const int ps = nilnb ? e : p;
    const bool del = R[ps].next == e;
    int ea = u, eb = un, ec = v, ek = EV_INS;  // case 2
    if (child) { ea = p; eb = e; ec = q; ek = del ? EV_DEL : EV_INS; }
    if (which == 3) { ea = up; eb = u; ek = EV_DEL; }
    if (which == 4) { eb = v; ec = vn; ek = EV_DEL; }
    if (which == 5) { eb = vp; }
    const bool emit = child ? (left ? e < u : e > v) : true;
    if (child && nilnb) {
      err = H3D_E_CHAIN;
      break;
    }
    if (emit) {
      if (k >= capRef - 1) {
        err = H3D_E_OVERFLOW;
        break;
      }
      if (k >= 0x4000) {
        err = static_cast<int>(E_FASTPATH);
        break;
      }
      Ev o;
      o.t = best;
      o.a = ea;
      o.b = eb;
      o.c = ec;
      o.kind = ek;
      out[k] = o;
      const unsigned short inf = J.info[eb];
      if ((inf & INFO_NONE) == INFO_NONE)
        J.info[eb] = static_cast<unsigned short>((inf & INFO_CHAIN) | k);
      ++k;
    }
    if (child) {  // _act
      R[p].next = del ? q : e;
      R[q].prev = del ? p : e;
    }
    if (left) {
      ++i;
      c0 = nL.t;
      bL = nL.b;
      if (i + 1 < kL) nL = evL[i + 1]; else nL.t = INF;
    }
    if (right) {
      ++j;
      c1 = nR.t;
      bR = nR.b + nSL;
      if (j + 1 < kR) nR = evR[j + 1]; else nR.t = INF;
    }
    u = (which == 2) ? un : ((which == 3) ? up : u);
    v = (which == 4) ? vn : ((which == 5) ? vp : v);
    c2 = evt_rec(R, u, R[u].next, v);
    c3 = evt_rec(R, R[u].prev, u, v);
    c4 = evt_rec(R, u, v, R[v].next);
    c5 = evt_rec(R, u, R[v].prev, v);
    tcur = best;
  }
  return err ? err : k;
}

constexpr int TPJ_REC_BYTES = 34;

// max over CTAs (chunks of tpb consecutive jobs) of the shared bytes the
// chunk's merges need -- sizes the thread-per-job pool so no CTA needs a
// second round (a round serialises behind the slowest sweep)
__global__ void k_tpj_need(Pass2 P, long long n, int level, long long j0, long long j1, int tpb,
                           unsigned long long *out) {
  const GroupBuf in = blockIdx.y ? P.in1 : P.in0;
  const long long size = 1ll << level, half = size >> 1;
  const long long chunks = (j1 - j0 + tpb - 1) / tpb;
  for (long long c = blockIdx.x * (long long)blockDim.x + threadIdx.x; c < chunks;
       c += (long long)gridDim.x * blockDim.x) {
    unsigned long long tot = 0;
    for (long long j = j0 + c * tpb; j < j0 + (c + 1) * tpb && j < j1; ++j) {
      const long long L = j << level;
      const long long R_ = (L + size < n) ? L + size : n;
      if (R_ - L <= half) continue;
      const int nS = in.hdr[2 * j].x + in.hdr[2 * j + 1].x;
      tot += align8((long long)TPJ_REC_BYTES * nS);
    }
    atomicMax(out, tot);
  }
}  // 32-byte record + 2-byte info per point

// One thread per merge job (levels with many jobs).  Each thread's slice of
// the shared-memory pool holds its job's records and info table; slices are
// packed by a block-wide prefix scan of the actual sizes (jobs that do not
// fit wait for the next round).
template <int TPJ_TPB>
__global__ void __launch_bounds__(TPJ_TPB) k_fast_tpj(Pass2 P, long long n, int level,
                                                     long long j0, long long j1,
                                                     long long *err, int pool) {
  const GroupBuf in = blockIdx.y ? P.in1 : P.in0;
  const GroupBuf out = blockIdx.y ? P.out1 : P.out0;
  extern __shared__ __align__(16) unsigned char smem[];
  typedef cub::BlockScan<int, TPJ_TPB> Scan;
  __shared__ typename Scan::TempStorage scan_tmp;
  const long long size = 1ll << level, half = size >> 1;
  const long long jobs = j1;
  const long long j = j0 + blockIdx.x * (long long)TPJ_TPB + threadIdx.x;
  const long long L = j << level, M = L + half;
  const long long R_ = (L + size < n) ? L + size : n;
  const bool valid = j < jobs;
  int nSL = 0, kL = 0, nSR = 0, kR = 0;
  bool pending = false;
  if (valid) {
    const int2 hl = in.hdr[2 * j];
    nSL = hl.x;
    kL = hl.y;
    if (R_ - L > half) {
      const int2 hr = in.hdr[2 * j + 1];
      nSR = hr.x;
      kR = hr.y;
      pending = true;
    } else {  // carry (copy_log, parallel.py:107-108)
      for (int p = 0; p < nSL; ++p) {
        out.rec[L + p] = in.rec[L + p];
        out.gid[L + p] = in.gid[L + p];
      }
      for (int e = 0; e < kL; ++e) out.ev[2 * L + e] = in.ev[2 * L + e];
      out.hdr[j] = hl;
    }
  }
  const int nS = nSL + nSR;
  const int need = static_cast<int>(align8((long long)TPJ_REC_BYTES * nS));
  if (pending && (need > pool || nS >= 0x4000)) {
    raise_err(err, E_FASTPATH);  // the host never routes such jobs here
    pending = false;
  }
  while (__syncthreads_or(pending)) {
    int off, total;
    Scan(scan_tmp).ExclusiveSum(pending ? need : 0, off, total);
    const bool run = pending && off + need <= pool;
    // the lanes that run this round re-converge at every phase boundary
    // (independent thread scheduling would otherwise let the variable-length
    // staging loops split the warp and run the sweep once per split)
    const unsigned rmask = __ballot_sync(0xffffffffu, run);
    if (run) {
      TpjJob J;
      J.R = reinterpret_cast<Rec *>(smem + off);
      J.info = reinterpret_cast<unsigned short *>(J.R + nS);
      J.nSL = nSL;
      Rec *R = J.R;
      {  // stage: independent loads first, then shared stores
        const Rec *__restrict__ gl = in.rec + L;
        const Rec *__restrict__ gr = in.rec + M;
        int p = 0;
        for (; p + 4 <= nS; p += 4) {
          Rec r0 = p < nSL ? gl[p] : gr[p - nSL];
          Rec r1 = p + 1 < nSL ? gl[p + 1] : gr[p + 1 - nSL];
          Rec r2 = p + 2 < nSL ? gl[p + 2] : gr[p + 2 - nSL];
          Rec r3 = p + 3 < nSL ? gl[p + 3] : gr[p + 3 - nSL];
          R[p] = r0;
          R[p + 1] = r1;
          R[p + 2] = r2;
          R[p + 3] = r3;
        }
        for (; p < nS; ++p) R[p] = p < nSL ? gl[p] : gr[p - nSL];
        for (p = nSL; p < nS; ++p) {
          if (R[p].prev != NIL) R[p].prev += nSL;
          if (R[p].next != NIL) R[p].next += nSL;
        }
      }
      for (int p = 0; p < nS; ++p) {
        const int pr = R[p].prev;
        const bool chain = p == 0 || p == nSL || (pr != NIL && R[pr].next == p);
        J.info[p] = chain ? (INFO_CHAIN | INFO_NONE) : INFO_NONE;
      }
      __syncwarp(rmask);
      int u0 = 0, v0 = 0;
      Ev *evo = out.ev + 2 * L;
      const long long k = merge_tpj(J, in.ev + 2 * L, kL, in.ev + 2 * M, kR, evo, 2 * (R_ - L),
                                    R_ - L, &u0, &v0, rmask);
      __syncwarp(rmask);
      if (k < 0) {
        raise_err(err, k);
      } else {
        // start-of-time links of the merged group (see rebuild_writeout)
        int cnt = 0;
        for (int p = 0; p < nS; ++p) {
          const unsigned short inf = J.info[p];
          const bool chain = (inf & INFO_CHAIN) && (p < nSL ? p <= u0 : p >= v0);
          const int fe = inf & INFO_NONE;
          const bool keep = chain || fe != INFO_NONE;
          int prv = NIL, nxt = NIL;
          if (chain) {
            const Rec &r = p < nSL ? in.rec[L + p] : in.rec[M + (p - nSL)];
            const int o = p < nSL ? 0 : nSL;
            prv = r.prev == NIL ? NIL : r.prev + o;
            nxt = r.next == NIL ? NIL : r.next + o;
            if (p == u0) nxt = v0;
            if (p == v0) prv = u0;
          } else if (keep) {
            prv = evo[fe].a;
            nxt = evo[fe].c;
          }
          R[p].prev = prv;
          R[p].next = nxt;
          J.info[p] = keep ? static_cast<unsigned short>(cnt++) : 0xffff;
        }
        bool bad = false;
        // events first (they read arbitrary new ids), in place in HBM
        for (int e = 0; e < k; ++e) {
          Ev o = evo[e];
          const unsigned short na = J.info[o.a], nb = J.info[o.b], nc = J.info[o.c];
          bad |= (na == 0xffff) | (nb == 0xffff) | (nc == 0xffff);
          o.a = na;
          o.b = nb;
          o.c = nc;
          evo[e] = o;
        }
        for (int p = 0; p < nS; ++p) {
          const unsigned short id = J.info[p];
          if (id == 0xffff) continue;
          Rec r = R[p];
          r.prev = r.prev == NIL ? NIL : J.info[r.prev];
          r.next = r.next == NIL ? NIL : J.info[r.next];
          bad |= (r.prev == 0xffff) | (r.next == 0xffff);
          out.rec[L + id] = r;
          out.gid[L + id] = in.gid[p < nSL ? L + p : M + (p - nSL)];
        }
        if (bad) raise_err(err, E_FASTPATH);
        out.hdr[j] = make_int2(cnt, static_cast<int>(k));
      }
      pending = false;
    }
  }
}

// -------------------------------------------------------------- warp merge
__device__ __forceinline__ void first_event(int *first, int b, int idx) {
  const int cur = *reinterpret_cast<volatile int *>(&first[b]);
  atomicMin(&first[b], (cur & FIRST_FLAG) | idx);
}

// Warp-wide merge path: the child logs evL[0,kL) and evR[0,kR) (each sorted
// by time) merged into seq[0, kL+kR) by time, left first on equal times; the
// right child's ids get +nSL and the side is kept in bit 1 of `kind`.  Each
// lane finds its diagonal split by one binary search, then merges its
// contiguous slice of the output sequentially.
__device__ void merge_logs_warp(const Ev *__restrict__ evL, int kL, const Ev *__restrict__ evR,
                                int kR, int nSL, Ev *seq) {
  const int lane = threadIdx.x & 31;
  const int K = kL + kR;
  const int chunk = (K + 31) / 32;
  const int d0 = min(K, lane * chunk), d1 = min(K, d0 + chunk);
  int lo = max(0, d0 - kR), hi = min(d0, kL);
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (evL[mid].t <= evR[d0 - mid - 1].t) lo = mid + 1; else hi = mid;
  }
  int i = lo, j = d0 - lo;
  for (int d = d0; d < d1; ++d) {
    const bool takeL = i < kL && (j >= kR || evL[i].t <= evR[j].t);
    Ev o;
    if (takeL) {
      o = evL[i++];
    } else {
      o = evR[j++];
      o.a += nSL;
      o.b += nSL;
      o.c += nSL;
      o.kind |= 2;
    }
    seq[d] = o;
  }
  __syncwarp();
}

// The warp-cooperative merge (levels with few, large jobs).  All lanes call
// it; returns k (warp-uniform) or a negative code.
//
// The sweep walks the time-merged child events 32 at a time.  Every event
// before the first one that touches a bridge foot (its facet has u or v as a
// neighbour) and before the next bridge event is retired in parallel:
// survivors (left: b < u, right: b > v -- the reference's emission rule) get
// output slots by a ballot prefix sum, and the link writes of the retired
// events are resolved last-writer-wins with __match_any_sync (an event's
// facet and kind say exactly what act() writes).  A foot-touching event or
// a bridge event is then processed alone, with the four bridge candidates
// recomputed on four lanes.  Decisions are the reference's, step for step,
// as long as no two events share a time (exact ties are outside general
// position and send the job to the exact path).
//
// R[0,nS): records at -inf (left [0,nSL), right [nSL,nS)); seq: merged child
// events; out: merged events (HBM); first[p]: FIRST_FLAG if p is on its
// child's -inf chain, low bits = index of p's first merged event.
__device__ long long merge_warp(Rec *R, int nSL, const Ev *seq, int kin, Ev *out,
                                int *first, long long capRef, long long limitRef, int *pu0,
                                int *pv0) {
  const int lane = threadIdx.x & 31;
  const unsigned ltmask = (1u << lane) - 1;
  int u = nSL - 1, v = nSL, st = 0;
  if (lane == 0) st = bridge_rec(R, &u, &v, limitRef);
  st = __shfl_sync(FULL, st, 0);
  if (st < 0) return H3D_E_BRIDGE;
  u = __shfl_sync(FULL, u, 0);
  v = __shfl_sync(FULL, v, 0);
  *pu0 = u;
  *pv0 = v;
  double c2, c3, c4, c5;
  auto cands = [&]() {
    double c = INF;
    if (lane == 0)
      c = evt_rec(R, u, R[u].next, v);
    else if (lane == 1)
      c = evt_rec(R, R[u].prev, u, v);
    else if (lane == 2)
      c = evt_rec(R, u, v, R[v].next);
    else if (lane == 3)
      c = evt_rec(R, u, R[v].prev, v);
    c2 = __shfl_sync(FULL, c, 0);
    c3 = __shfl_sync(FULL, c, 1);
    c4 = __shfl_sync(FULL, c, 2);
    c5 = __shfl_sync(FULL, c, 3);
  };
  cands();
  int ptr = 0, k = 0, errc = 0;
  double tcur = -INF;
  for (;;) {
    // next bridge event: earliest candidate strictly after tcur, lowest case on ties
    double tb = INF;
    int wb = -1;
    if (c2 > tcur && c2 < tb) { tb = c2; wb = 2; }
    if (c3 > tcur && c3 < tb) { tb = c3; wb = 3; }
    if (c4 > tcur && c4 < tb) { tb = c4; wb = 4; }
    if (c5 > tcur && c5 < tb) { tb = c5; wb = 5; }
    const int rem = kin - ptr;
    bool child_next = false;
    if (rem > 0) {
      const bool valid = lane < rem;
      Ev my;
      my.t = INF;
      if (valid) my = seq[ptr + lane];
      const double tprev = __shfl_up_sync(FULL, my.t, 1);
      // exact ties break the reference's strict `t > oldt` rule: exact path
      if (valid && ((lane > 0 && my.t == tprev) || my.t == tb || my.t <= tcur)) errc = E_FASTPATH;
      const bool touches = valid && (my.a == u || my.a == v || my.c == u || my.c == v);
      const bool stop = !valid || touches || my.t > tb;
      const unsigned sb = __ballot_sync(FULL, stop);
      const int f = sb ? __ffs(sb) - 1 : 32;
      const bool pre = lane < f;
      const bool isL = (my.kind & 2) == 0;
      const int kind = my.kind & 1;
      const bool surv = pre && (isL ? my.b < u : my.b > v);
      const unsigned vs = __ballot_sync(FULL, surv);
      if (surv) {
        const int pos = k + __popc(vs & ltmask);
        if (pos >= capRef - 1) {
          errc = H3D_E_OVERFLOW;
        } else {
          Ev o = my;
          o.kind = kind;
          out[pos] = o;
          first_event(first, my.b, pos);
        }
      }
      k += __popc(vs);
      const int key1 = pre ? my.a : (int)(0x80000000u + lane);
      const int key2 = pre ? my.c : (int)(0x80000000u + lane);
      const unsigned m1 = __match_any_sync(FULL, key1);
      const unsigned m2 = __match_any_sync(FULL, key2);
      if (pre && (31 - __clz(m1)) == lane) R[my.a].next = (kind == EV_INS) ? my.b : my.c;
      if (pre && (31 - __clz(m2)) == lane) R[my.c].prev = (kind == EV_INS) ? my.b : my.a;
      if (f > 0) tcur = __shfl_sync(FULL, my.t, f - 1);
      ptr += f;
      if (f < 32 && f < rem) {
        const double tf = __shfl_sync(FULL, my.t, f);
        child_next = tf < tb;
        if (child_next) {  // a foot-touching child event: process it alone
          const int a = __shfl_sync(FULL, my.a, f), b = __shfl_sync(FULL, my.b, f);
          const int c = __shfl_sync(FULL, my.c, f), kd = __shfl_sync(FULL, my.kind, f);
          const bool sL = (kd & 2) == 0;
          const bool sv = sL ? b < u : b > v;
          __syncwarp();
          if (lane == 0) {
            const int p = R[b].prev, q = R[b].next;
            if (p != a || q != c || p == NIL || q == NIL) {
              errc = E_FASTPATH;
            } else {
              const int kind1 = (R[p].next == b) ? EV_DEL : EV_INS;
              if (kind1 != (kd & 1)) errc = E_FASTPATH;
              if (sv) {
                if (k >= capRef - 1) {
                  errc = H3D_E_OVERFLOW;
                } else {
                  Ev o;
                  o.t = tf;
                  o.a = a;
                  o.b = b;
                  o.c = c;
                  o.kind = kind1;
                  out[k] = o;
                  first_event(first, b, k);
                }
              }
              act_rec(R, b);
            }
          }
          if (sv) ++k;
          ++ptr;
          tcur = tf;
          __syncwarp();
          cands();
        }
      }
      errc = __reduce_min_sync(FULL, errc);
      if (errc < 0) return errc;
      if (child_next) continue;
      if (f == 32 && ptr < kin) continue;  // a full window retired: keep going
      if (wb < 0) continue;                // no bridge event left: drain the logs
    } else if (wb < 0) {
      break;  // nothing left
    }
    // the bridge event comes next
    if (lane == 0) {
      int a, b, c, kind;
      if (wb == 2) {
        a = u; b = R[u].next; c = v; kind = EV_INS; u = b;
      } else if (wb == 3) {
        a = R[u].prev; b = u; c = v; kind = EV_DEL; u = a;
      } else if (wb == 4) {
        a = u; b = v; c = R[v].next; kind = EV_DEL; v = c;
      } else {
        a = u; b = R[v].prev; c = v; kind = EV_INS; v = b;
      }
      if (k >= capRef - 1) {
        errc = H3D_E_OVERFLOW;
      } else {
        Ev o;
        o.t = tb;
        o.a = a;
        o.b = b;
        o.c = c;
        o.kind = kind;
        out[k] = o;
        first_event(first, b, k);
      }
    }
    errc = __shfl_sync(FULL, errc, 0);
    if (errc < 0) return errc;
    u = __shfl_sync(FULL, u, 0);
    v = __shfl_sync(FULL, v, 0);
    ++k;
    tcur = tb;
    __syncwarp();
    cands();
  }
  return k;
}

// Parallel rebuild of the merged group's start-of-time links, compaction and
// write-out (warp-wide).  Kept = merged -inf chain (left chain up to u0, right
// chain from v0) U every point of the merged log.  Links: chain points keep
// their -inf links (u0 -> v0 stitched), the others get the neighbours of
// their first event (an insertion: a point off the -inf chain enters the
// hull once).  These are exactly the links the reference's rewind leaves on
// every kept point.  evo (the merged events, local ids) is out.ev + 2L.
__device__ void rebuild_writeout(const GroupBuf &in, const GroupBuf &out, Rec *R, Ev *evo,
                                 int *first, long long L, long long M, int nSL, int nS, int k,
                                 int u0, int v0, long long gidx, long long *err) {
  const int lane = threadIdx.x & 31;
  bool bad = false;
  // A: final links (local ids) into R, keep flag into first
  for (int p = lane; p < nS; p += 32) {
    const int fp = first[p];
    const bool chain = (fp & FIRST_FLAG) && (p < nSL ? p <= u0 : p >= v0);
    const int fe = fp & FIRST_NONE;
    const bool hasev = fe != FIRST_NONE;
    int prv = NIL, nxt = NIL;
    if (chain) {
      const Rec o = (p < nSL) ? in.rec[L + p] : in.rec[M + (p - nSL)];
      const int off = (p < nSL) ? 0 : nSL;
      prv = (o.prev == NIL) ? NIL : o.prev + off;
      nxt = (o.next == NIL) ? NIL : o.next + off;
      if (p == u0) nxt = v0;
      if (p == v0) prv = u0;
    } else if (hasev) {
      prv = evo[fe].a;
      nxt = evo[fe].c;
    }
    R[p].prev = prv;
    R[p].next = nxt;
    first[p] = (chain || hasev) ? 1 : 0;
  }
  __syncwarp();
  // B: new ids
  int cnt = 0;
  for (int p0 = 0; p0 < nS; p0 += 32) {
    const int p = p0 + lane;
    const bool keep = p < nS && first[p] != 0;
    const unsigned bal = __ballot_sync(FULL, keep);
    if (p < nS) first[p] = keep ? cnt + __popc(bal & ((1u << lane) - 1)) : -1;
    cnt += __popc(bal);
  }
  __syncwarp();
  // C: events, in place
  for (int e = lane; e < k; e += 32) {
    Ev o = evo[e];
    o.a = first[o.a];
    o.b = first[o.b];
    o.c = first[o.c];
    bad |= (o.a < 0) | (o.b < 0) | (o.c < 0);
    evo[e] = o;
  }
  // D: links remapped in place
  for (int p = lane; p < nS; p += 32) {
    if (first[p] < 0) continue;
    Rec &r = R[p];
    if (r.prev != NIL) {
      r.prev = first[r.prev];
      bad |= r.prev < 0;
    }
    if (r.next != NIL) {
      r.next = first[r.next];
      bad |= r.next < 0;
    }
  }
  __syncwarp();
  // E: move records and gids (chunked read-all / write; ids only move left,
  // and a gid write only lands on ids already consumed)
  for (int p0 = 0; p0 < nS; p0 += 32) {
    const int p = p0 + lane;
    int id = -1, g = 0;
    Rec r;
    if (p < nS) {
      id = first[p];
      if (id >= 0) {
        r = R[p];
        g = in.gid[p < nSL ? L + p : M + (p - nSL)];
      }
    }
    __syncwarp();
    if (id >= 0) {
      out.rec[L + id] = r;
      out.gid[L + id] = g;
    }
    __syncwarp();
  }
  if (__any_sync(FULL, bad) && lane == 0) raise_err(err, E_FASTPATH);
  if (lane == 0) out.hdr[gidx] = make_int2(cnt, k);
}

// shared bytes of one warp job: records, first table, merged child events
__device__ __forceinline__ long long warp_job_bytes(int nS, int kin) {
  return align8(32ll * nS + 4ll * nS) + 24ll * kin;
}

// One warp per merge job (levels with few, large jobs).  A job's records,
// first table and time-merged child events are staged in the CTA's shared
// pool when they fit (warps whose jobs do not fit wait a round), else they
// live in HBM scratch inside the job's own output slots (records at
// out.rec[L..], first table in out.gid[L..]) with the merged child events
// in the pass's HBM scratch (PassWS::seq).
template <int WARPS>
__global__ void __launch_bounds__(WARPS * 32) k_fast_warp(Pass2 P, long long n, int level,
                                                          long long j0, long long j1,
                                                          long long *err, int pool,
                                                          Ev *gseq0, Ev *gseq1) {
  const GroupBuf in = blockIdx.y ? P.in1 : P.in0;
  const GroupBuf out = blockIdx.y ? P.out1 : P.out0;
  Ev *gseq = blockIdx.y ? gseq1 : gseq0;
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ long long s_need[WARPS];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const long long size = 1ll << level, half = size >> 1;
  const long long jobs = j1;
  const long long j = j0 + blockIdx.x * (long long)WARPS + warp;
  const long long L = j << level, M = L + half;
  const long long R_ = (L + size < n) ? L + size : n;
  const bool valid = j < jobs;
  int nSL = 0, kL = 0, nSR = 0, kR = 0;
  bool merge = false;
  if (valid) {
    const int2 hl = in.hdr[2 * j];
    nSL = hl.x;
    kL = hl.y;
    merge = R_ - L > half;
    if (merge) {
      const int2 hr = in.hdr[2 * j + 1];
      nSR = hr.x;
      kR = hr.y;
    } else {  // carry (copy_log, parallel.py:107-108)
      for (int p = lane; p < nSL; p += 32) {
        out.rec[L + p] = in.rec[L + p];
        out.gid[L + p] = in.gid[L + p];
      }
      for (int e = lane; e < kL; e += 32) out.ev[2 * L + e] = in.ev[2 * L + e];
      if (lane == 0) out.hdr[j] = hl;
    }
  }
  const int nS = nSL + nSR, kin = kL + kR;
  const long long need = merge ? warp_job_bytes(nS, kin) : 0;
  const bool global_mode = merge && need > pool;
  bool pending = merge && !global_mode;
  auto run_job = [&](Rec *Rr, int *first, Ev *seq) {
    for (int p = lane; p < nS; p += 32) {
      Rec r = (p < nSL) ? in.rec[L + p] : in.rec[M + (p - nSL)];
      if (p >= nSL) {
        if (r.prev != NIL) r.prev += nSL;
        if (r.next != NIL) r.next += nSL;
      }
      Rr[p] = r;
    }
    merge_logs_warp(in.ev + 2 * L, kL, in.ev + 2 * M, kR, nSL, seq);
    for (int p = lane; p < nS; p += 32) {
      const int pr = Rr[p].prev;
      const bool chain = (p == 0 || p == nSL) || (pr != NIL && Rr[pr].next == p);
      first[p] = (chain ? FIRST_FLAG : 0) | FIRST_NONE;
    }
    __syncwarp();
    int u0, v0;
    Ev *evo = out.ev + 2 * L;
    const long long k = merge_warp(Rr, nSL, seq, kin, evo, first, 2 * (R_ - L), R_ - L, &u0, &v0);
    __syncwarp();
    if (k < 0) {
      if (lane == 0) raise_err(err, k);
    } else {
      rebuild_writeout(in, out, Rr, evo, first, L, M, nSL, nS, static_cast<int>(k), u0, v0, j,
                       err);
    }
  };
  if (global_mode) {
    // in HBM: records at out.rec[L..L+nS) (nS <= R-L), first table in
    // out.gid[L..), merged child events in the level scratch at gseq[2L..)
    run_job(out.rec + L, out.gid + L, gseq + 2 * L);
  }
  // shared-memory pool: warps whose jobs fit run together, the rest wait
  for (;;) {
    if (lane == 0) s_need[warp] = pending ? need : 0;
    __syncthreads();
    long long off = 0;
    bool any = false;
    for (int w = 0; w < WARPS; ++w) {
      const long long nw = s_need[w];
      if (nw > 0) any = true;
      if (w < warp) off += nw;
    }
    __syncthreads();
    if (!any) break;
    // a warp runs this round if its prefix fits (the first pending one always does)
    if (pending && off + need <= pool) {
      unsigned char *mine = smem + off;
      Rec *Rr = reinterpret_cast<Rec *>(mine);
      int *first = reinterpret_cast<int *>(Rr + nS);
      Ev *seq = reinterpret_cast<Ev *>(mine + align8(36ll * nS));
      run_job(Rr, first, seq);
      pending = false;
    }
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

constexpr int kWarps = 8;
constexpr int kPool = 64 * 1024;
constexpr int kTpjPool = 200 * 1024;
int kTpjMaxLevel = 9;  // H3D_TPJ_MAX_LEVEL
long long kTpjMinJobs = 16384;  // H3D_TPJ_MIN_JOBS (per pass)

struct PassWS {
  GroupBuf A, B;
  Ev *seq;                  // merged child events of HBM-resident warp jobs (2n)
  unsigned long long *need; // thread-per-job pool sizing
};

bool carve_pass(h3d_arena &ar, long long n, PassWS &w) {
  for (GroupBuf *g : {&w.A, &w.B}) {
    g->hdr = ar.take<int2>(n);
    g->rec = ar.take<Rec>(n);
    g->gid = ar.take<int>(n);
    g->ev = ar.take<Ev>(2 * n);
  }
  w.seq = ar.take<Ev>(2 * n);
  w.need = ar.take<unsigned long long>(4);
  return ar.base == nullptr || w.need != nullptr;
}

bool g_attr_done = false;
// thread-per-job tuning (H3D_TPJ_TPB, H3D_TPJ_FILL, H3D_TPJ_POOL_KB override)
int g_tpj_tpb = 32;
double g_tpj_fill = 0.5;
long long g_tpj_pool = 200 * 1024;
int g_tpj_measure = 1;  // H3D_TPJ_MEASURE=0: size the pool by H3D_TPJ_FILL instead

}  // namespace

extern "C" {

int64_t h3d_fast_layout(int64_t n, int64_t *offsets) {
  // byte offsets of A.hdr, A.rec, A.gid, A.ev, B.hdr, B.rec, B.gid, B.ev, seq
  char *base = reinterpret_cast<char *>(size_t(1) << 40);
  h3d_arena ar(base, ~size_t(0) >> 4);
  PassWS w;
  if (!carve_pass(ar, n, w)) return H3D_E_ARG;
  const void *p[9] = {w.A.hdr, w.A.rec, w.A.gid, w.A.ev, w.B.hdr, w.B.rec, w.B.gid, w.B.ev, w.seq};
  for (int i = 0; i < 9; ++i) offsets[i] = static_cast<const char *>(p[i]) - base;
  return 0;
}

size_t h3d_fast_pass_workspace_bytes(int64_t n) {  // per pass
  if (n < 1) n = 1;
  h3d_arena ar(nullptr, 0);
  PassWS w;
  carve_pass(ar, n, w);
  return ar.used + 4096;
}

int64_t h3d_fast_passes_range(const double *sorted_pts, int64_t n, int64_t p0, int64_t p1,
                              int32_t lv_lo, int32_t lv_hi, void *ws_lower, void *ws_upper,
                              size_t workspace_bytes, int64_t *err_dev, int32_t verify,
                              void *stream) {
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  (void)verify;
  if (n < 2 || n > (1ll << 30) || p0 < 0 || p1 > n || p0 >= p1 || lv_lo < 1) return H3D_E_ARG;
  h3d_arena a0(ws_lower, workspace_bytes), a1(ws_upper, workspace_bytes);
  PassWS w0, w1;
  if (!carve_pass(a0, n, w0) || !carve_pass(a1, n, w1)) return H3D_E_ARG;
  if (!g_attr_done) {
    if (h3d_check(cudaFuncSetAttribute(k_fast_warp<kWarps>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, kPool)) ||
        h3d_check(cudaFuncSetAttribute(k_fast_tpj<32>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       kTpjPool)) ||
        h3d_check(cudaFuncSetAttribute(k_fast_tpj<64>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       kTpjPool)) ||
        h3d_check(cudaFuncSetAttribute(k_fast_tpj<128>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       kTpjPool)))
      return H3D_E_CUDA;
    if (const char *e = getenv("H3D_TPJ_TPB")) g_tpj_tpb = atoi(e);
    if (const char *e = getenv("H3D_TPJ_FILL")) g_tpj_fill = atof(e);
    if (const char *e = getenv("H3D_TPJ_POOL_KB")) g_tpj_pool = atoll(e) * 1024;
    if (const char *e = getenv("H3D_TPJ_MAX_LEVEL")) kTpjMaxLevel = atoi(e);
    if (const char *e = getenv("H3D_TPJ_MEASURE")) g_tpj_measure = atoi(e);
    if (const char *e = getenv("H3D_TPJ_MIN_JOBS")) kTpjMinJobs = atoll(e);
    if (g_tpj_tpb != 32 && g_tpj_tpb != 64) g_tpj_tpb = 128;
    if (g_tpj_pool > kTpjPool) g_tpj_pool = kTpjPool;
    g_attr_done = true;
  }
  long long *err = reinterpret_cast<long long *>(err_dev);
  int levels = 0;
  while ((1ll << levels) < n) ++levels;
  if (lv_hi > levels) lv_hi = levels;
  // level l reads buffer (l-1)&1 and writes buffer l&1 (A = 0, B = 1)
  Pass2 P = (lv_lo & 1) ? Pass2{w0.A, w1.A, w0.B, w1.B} : Pass2{w0.B, w1.B, w0.A, w1.A};
  if (lv_lo == 1) {
    h3d_count_launches(1);
    const long long np = p1 - p0;
    const unsigned gi = h3d_grid(np, 256) > 4096 ? 4096 : h3d_grid(np, 256);
    k_fast_init<<<dim3(gi, 2), 256, 0, s>>>(sorted_pts, p0, p1, P);
  }
  for (int lv = lv_lo; lv <= lv_hi; ++lv) {
    // the jobs of this level inside the point range [p0, p1)
    const long long j0 = p0 >> lv;
    const long long j1 = (p1 + (1ll << lv) - 1) >> lv;
    const long long jobs = j1 - j0;
    void *e0 = h3d_profiling() ? h3d_prof_begin(s) : nullptr;
    h3d_count_launches(1);
    // thread per job while jobs are plentiful and small, warp per job above
    if (jobs >= kTpjMinJobs && lv <= kTpjMaxLevel && ((long long)TPJ_REC_BYTES << lv) <= kTpjPool) {
      // threads per CTA and shared pool per level: the pool is the largest
      // CTA's actual need (one small read-back per level), capped
      const int tpb = g_tpj_tpb;
      long long pool;
      if (g_tpj_measure) {
        cudaMemsetAsync(w0.need, 0, sizeof(unsigned long long), s);
        const long long chunks = (jobs + tpb - 1) / tpb;
        h3d_count_launches(1);
        k_tpj_need<<<dim3(h3d_grid(chunks, 128) > 2048 ? 2048 : h3d_grid(chunks, 128), 2), 128, 0,
                     s>>>(P, n, lv, j0, j1, tpb, w0.need);
        unsigned long long hneed = 0;
        if (h3d_check(cudaMemcpyAsync(&hneed, w0.need, sizeof(hneed), cudaMemcpyDeviceToHost, s)) ||
            h3d_check(cudaStreamSynchronize(s)))
          return H3D_E_CUDA;
        pool = static_cast<long long>(hneed);
      } else {
        pool = (long long)tpb * align8((long long)(TPJ_REC_BYTES * g_tpj_fill * (1ll << lv)));
      }
      if (pool > g_tpj_pool) pool = g_tpj_pool;
      if (pool < (long long)TPJ_REC_BYTES << lv) pool = align8((long long)TPJ_REC_BYTES << lv);
      if (pool < 2048) pool = 2048;
      const dim3 grid(h3d_grid(jobs, tpb), 2);
      if (tpb == 32)
        k_fast_tpj<32><<<grid, 32, pool, s>>>(P, n, lv, j0, j1, err, static_cast<int>(pool));
      else if (tpb == 64)
        k_fast_tpj<64><<<grid, 64, pool, s>>>(P, n, lv, j0, j1, err, static_cast<int>(pool));
      else
        k_fast_tpj<128><<<grid, 128, pool, s>>>(P, n, lv, j0, j1, err, static_cast<int>(pool));
      h3d_prof_end(e0, lv + 1000, 2, s);
    } else {
      k_fast_warp<kWarps><<<dim3(h3d_grid(jobs, kWarps), 2), kWarps * 32, kPool, s>>>(
          P, n, lv, j0, j1, err, kPool, w0.seq, w1.seq);
      h3d_prof_end(e0, lv, 2, s);
    }
    P = Pass2{P.out0, P.out1, P.in0, P.in1};
  }
  if (h3d_check(cudaGetLastError())) return H3D_E_CUDA;
  return lv_hi & 1;  // buffer holding the last level's groups
}

int64_t h3d_fast_passes(const double *sorted_pts, int64_t n, void *ws_lower, void *ws_upper,
                        size_t workspace_bytes, int64_t *err_dev, int32_t verify,
                        int64_t *final_out, void *stream) {
  int levels = 0;
  while ((1ll << levels) < n) ++levels;
  const int64_t r = h3d_fast_passes_range(sorted_pts, n, 0, n, 1, levels, ws_lower, ws_upper,
                                          workspace_bytes, err_dev, verify, stream);
  if (r < 0) return r;
  final_out[0] = r;
  final_out[1] = r;
  return 0;
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
