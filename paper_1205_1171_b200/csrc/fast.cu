// fast.cu -- the fused fast path: all merge levels of a pass over compact groups.
//
// Level scheduler (parallel.py:68-112 on the device); a device error word is
// read once per hull.  Each level is routed from one small measurement (or
// replayed from the previous same-size call's plan) to one of:
//
//  * k_fast_init1  level 1 (pairs of one-point groups) written directly;
//    k_fast_leaf   levels 1..3 fused, one lane per 8-point block.
//  * k_lane (lane.cu, levels <= 5) / k_fast_tpj: one LANE per merge job;
//    a level whose few largest CTAs need far more shared memory than the
//    rest is split (a small pool + an overflow list for a full-pool launch,
//    k_fast_tpj_ovf), and a level of a few large jobs among many small ones
//    runs hybrid (the overflow CTAs' jobs one CTA each on a mini variant).
//  * k_mini (mini.cu): one CTA per job, the time axis split into segments.
//  * big.cu: the time-split pipeline over global memory for huge jobs.
//  * k_fast_tpj    one launch per level while jobs are plentiful: one LANE per
//                  merge job (merge_tpj2, the reference's sequential sweep with
//                  stored child event times and the bridge neighbourhood in
//                  registers); int16 links, gids and first-event info in a
//                  packed shared-memory slice per job (plus coordinates when
//                  they fit), staged and written back warp-cooperatively; the
//                  start-of-time links are rebuilt from the merged -inf chain
//                  and first events (no sequential rewind).
//  * k_fast_warp   one launch per level above.  One WARP per merge job
//                  (merge_warp): the kinetic sweep advances through the
//                  time-merged child logs 32 events at a time -- every event
//                  that neither touches the bridge feet nor comes after the
//                  next bridge event is retired in parallel (survivor
//                  emission by ballot prefix, link writes resolved
//                  last-writer-wins with __match_any_sync) -- and only foot
//                  events and bridge events are sequential.  Jobs are staged
//                  in a shared-memory pool when they fit, else run in HBM.
//  * k_fast_extract  facets of both passes straight from the final events.
//
// Coordinates are never copied between levels: a group stores each kept
// point's gid and kernels read the sorted point array (z negated on the
// upper pass).
#include <cstdlib>
#include <map>
#include <mutex>
#include <string>
#include <type_traits>
#include <vector>


#include "fast.cuh"
#include "h3d_host.h"

namespace h3d {

// ----------------------------------------------------------- level 1 init
// Level 1 merges two one-point groups: the bridge walk stops at once (both
// feet have NIL neighbours), no event can occur and the stitch links the
// pair -- so the level-1 groups are written directly, without reading a
// coordinate: (nS, k) = (2, 0), links 0 <-> 1, or a one-point carry.
__global__ void k_fast_init1(long long n, long long j0, long long j1, Pass2 P) {
  const GroupBuf g = blockIdx.y ? P.out1 : P.out0;
  for (long long j = j0 + blockIdx.x * (long long)blockDim.x + threadIdx.x; j < j1;
       j += (long long)gridDim.x * blockDim.x) {
    const long long L = 2 * j;
    if (L + 1 < n) {
      g.hdr[j] = make_int2(2, 0);
      reinterpret_cast<int4 *>(g.lnk + L)[0] = make_int4(NIL, 1, 0, NIL);
      reinterpret_cast<int2 *>(g.gid + L)[0] = make_int2(static_cast<int>(L), static_cast<int>(L + 1));
    } else {
      g.hdr[j] = make_int2(1, 0);
      g.lnk[L] = make_int2(NIL, NIL);
      g.gid[L] = static_cast<int>(L);
    }
  }
}

// --------------------------------------------------------- thread per job
// One WARP = 32 merge jobs, one per lane (levels with many small jobs).
//
// Each job owns a slice of the CTA's shared memory, packed by a warp prefix
// sum of the slice sizes:
//   [XYZ: x[nS], y[nS], z[nS] f64]  lk[nS] short2 current links
//   gd[nS] int gid                   fi[nS] u32 first-event / chain info
// Staging and write-out are warp-cooperative per job (coalesced); the
// kinetic sweep runs on the job's own lane with the bridge feet, their four
// neighbours, their coordinates and the four bridge candidate times held in
// registers, so one step costs a handful of shared-memory accesses: the two
// link stores of the child event's act, one link load and one coordinate
// fetch for the one point that changes, and the candidates whose inputs
// changed.  Without XYZ staging, coordinates come from the sorted point
// array through the point's gid.
constexpr unsigned FI_CHAIN = 1u << 31;  // on its child's -inf chain
constexpr unsigned FI_EV = 1u << 30;     // has a merged event; bits 0-14 a, 15-29 c

__host__ __device__ __forceinline__ int tpj_slice_bytes(int nS, bool xyz) {
  return static_cast<int>(align16((long long)(xyz ? 36 : 12) * nS));
}

// A job's point table: coordinates (XYZ) or gids, links, first-event info.
// STRIDE = 1: a packed slice (thread-per-job kernel); STRIDE = 32: lane-
// interleaved arrays (leaf kernel, conflict-free whatever the index).
template <bool XYZ, int STRIDE = 1>
struct TpjSlice {
  // the sweep re-reads the bridge neighbourhood's coordinates from shared
  // memory instead of rotating a register copy: a win in the leaf kernel
  // (117 vs 140 registers, -9 %), not in the lane-per-job one (measured)
  static constexpr bool kReload = XYZ && STRIDE == 32;
  // first-event info word: 32 bits with 15-bit ids (lane kernel), 16 bits
  // with 7-bit ids in the leaf's lane-interleaved blocks (<= 16 points), so
  // that 12 leaf CTAs fit an SM
  using FiT = typename std::conditional<STRIDE == 32, unsigned short, unsigned>::type;
  static constexpr unsigned kFiChain = STRIDE == 32 ? (1u << 15) : FI_CHAIN;
  static constexpr unsigned kFiEv = STRIDE == 32 ? (1u << 14) : FI_EV;
  static constexpr int kFiShift = STRIDE == 32 ? 7 : 15;
  static constexpr unsigned kFiMask = STRIDE == 32 ? 0x7fu : 0x7fffu;
  double *x, *y, *z;
  short2 *lk;
  int *gd;
  FiT *fi;
  __device__ __forceinline__ TpjSlice() {}
  __device__ __forceinline__ TpjSlice(unsigned char *base, int nS) {
    unsigned char *p = base;
    if (XYZ) {
      x = reinterpret_cast<double *>(p);
      y = x + nS;
      z = y + nS;
      p += 24ll * nS;
    }
    lk = reinterpret_cast<short2 *>(p);
    gd = reinterpret_cast<int *>(lk + nS);
    fi = reinterpret_cast<FiT *>(gd + nS);
  }
  __device__ __forceinline__ short2 &LK(int p) const { return lk[p * STRIDE]; }
  __device__ __forceinline__ FiT &FI(int p) const { return fi[p * STRIDE]; }
  __device__ __forceinline__ int &GD(int p) const { return gd[p * STRIDE]; }
  __device__ __forceinline__ TpjSlice shifted(int d) const {  // ids relative to point d
    TpjSlice r = *this;
    if (XYZ) {
      r.x += d * STRIDE;
      r.y += d * STRIDE;
      r.z += d * STRIDE;
    }
    r.lk += d * STRIDE;
    if (!XYZ) r.gd += d * STRIDE;
    r.fi += d * STRIDE;
    return r;
  }
  __device__ __forceinline__ P3 pt(int p, const double *__restrict__ pts, double zs) const {
    P3 r;
    if (p == NIL) {
      r.x = r.y = r.z = 0.0;
      return r;
    }
    if (XYZ) {
      r.x = x[p * STRIDE];
      r.y = y[p * STRIDE];
      r.z = z[p * STRIDE];
      return r;
    }
    return load_pt(pts, gd[p * STRIDE], zs);
  }
};

// event streams of the sweep: HBM (16-byte EvP) ...
// The prefetched event stays PACKED (Raw) in registers and is unpacked only
// when it becomes the stream head one consumption later: unpacking at the
// load would put the load's full latency on the step that issued it (47 % of
// the stall samples at C4 level 8, profiles/r2_ncu_lines_tpj.txt).
struct GEvIn {
  static constexpr bool kPrefetch = true;  // HBM: one event of prefetch
  using Raw = EvP;
  const EvP *__restrict__ p;
  __device__ __forceinline__ EvP raw(int i) const {
    EvP r;  // two 64-bit loads: a 128-bit one needs an aligned register quad,
    r.t = __ldg(&p[i].t);  // which the loop-carried prefetch does not get
    r.w = __ldg(&p[i].w);
    return r;
  }
  __device__ __forceinline__ Ev get(int i) const { return p[i]; }
  __device__ __forceinline__ static Ev unpack(const EvP &r) { return r; }
  __device__ __forceinline__ static EvP none() {
    EvP r;
    r.t = INF;
    r.w = 0;
    return r;
  }
};
struct GEvOut {
  EvP *__restrict__ p;
  __device__ __forceinline__ void put(long long k, const Ev &o) const { p[k] = EvP(o); }
};
// ... or lane-interleaved shared memory (leaf kernel): time + one 16-bit
// word with the 4-bit block-local ids a, b, c (blocks of <= 16 points) and
// the kind -- half the bytes of a 32-bit word, so more CTAs fit an SM
struct LEvIn {
  static constexpr bool kPrefetch = false;  // shared memory: read when consumed
  using Raw = Ev;
  __device__ __forceinline__ Ev raw(int i) const { return get(i); }
  __device__ __forceinline__ static Ev unpack(const Ev &r) { return r; }
  __device__ __forceinline__ static Ev none() {
    Ev r;
    r.t = INF;
    r.a = r.b = r.c = r.kind = 0;
    return r;
  }
  // the event time is not stored: it is the canonical time of the facet
  // (evtime of the x-ordered triple, F4), re-derived from the block's
  // coordinates in shared memory -- bit for bit the stored value, and the
  // leaf's shared memory drops to 320 B per lane (16 CTAs per SM, was 12)
  const double *x, *y, *z;  // lane-interleaved block coordinates
  const unsigned short *w;
  __device__ __forceinline__ Ev get(int i) const {
    Ev e;
    const unsigned v = w[i * 32];
    e.a = v & 0xf;
    e.b = (v >> 4) & 0xf;
    e.c = (v >> 8) & 0xf;
    e.kind = v >> 12;
    e.t = evtime_xyz(x[e.a * 32], y[e.a * 32], z[e.a * 32], x[e.b * 32], y[e.b * 32], z[e.b * 32],
                     x[e.c * 32], y[e.c * 32], z[e.c * 32]);
    return e;
  }
};
struct LEvOut {
  unsigned short *w;
  __device__ __forceinline__ void put(long long k, const Ev &o) const {
    w[k * 32] = static_cast<unsigned short>(o.a | (o.b << 4) | (o.c << 8) | (o.kind << 12));
  }
};

// The reference's kinetic sweep (_merge_one phase 1, _ckernels.pyx:86-183)
// for one job on one lane.  Child candidate times are the stored times (the
// time the facet got when it was emitted one level down: same expression,
// same operand order, F4); each child event's stored facet and kind are
// checked against the current links (a mismatch hands the input to the
// exact engine).  Emitted events go straight to HBM with their facet and
// kind; the first merged event of each point is kept for the link rebuild
// that replaces the reference's rewind.  Returns k or a negative code.
// u_init: the left child's last point (its right neighbour is the right
// child's first); roff: added to the right child's event ids.
// CHILD = false: both child logs are empty (level 2: two linked pairs), so
// the child-event machinery compiles away.
template <class SL, class EIN, class EOUT, bool CHILD = true>
__device__ long long merge_tpj2(const SL &S, bool active, int u_init, int roff,
                                const double *__restrict__ pts, double zs, EIN evL, int kL,
                                EIN evR, int kR, EOUT out, long long capRef, long long limitRef,
                                int *pu0, int *pv0) {
  long long err = 0;
  // ---- bridge at t = -inf (_find_bridge, _ckernels.pyx:63-83)
  int u = u_init, v = u_init + 1;
  P3 U, V;
  U.x = U.y = U.z = V.x = V.y = V.z = 0.0;
  if (active) {
    U = S.pt(u, pts, zs);
    V = S.pt(v, pts, zs);
    long long moves = 0;
    for (;;) {
      const int vn = S.LK(v).y;
      if (vn != NIL) {
        const P3 W = S.pt(vn, pts, zs);
        if (turn_xy(U.x, U.y, V.x, V.y, W.x, W.y) < 0.0) {
          v = vn;
          V = W;
          if (++moves > limitRef) break;
          continue;
        }
      }
      const int up = S.LK(u).x;
      if (up != NIL) {
        const P3 W = S.pt(up, pts, zs);
        if (turn_xy(W.x, W.y, U.x, U.y, V.x, V.y) < 0.0) {
          u = up;
          U = W;
          if (++moves > limitRef) break;
          continue;
        }
      }
      break;
    }
    if (moves > limitRef) {
      err = H3D_E_BRIDGE;
      active = false;
    }
  }
  *pu0 = u;
  *pv0 = v;
  int un = NIL, up = NIL, vn = NIL, vp = NIL;
  if (active) {
    un = S.LK(u).y;
    up = S.LK(u).x;
    vn = S.LK(v).y;
    vp = S.LK(v).x;
  }
  P3 UN = S.pt(un, pts, zs), UP = S.pt(up, pts, zs), VN = S.pt(vn, pts, zs),
     VP = S.pt(vp, pts, zs);
  double c2 = evt3(u, un, v, U, UN, V);
  double c3 = evt3(up, u, v, UP, U, V);
  double c4 = evt3(u, v, vn, U, V, VN);
  double c5 = evt3(u, vp, v, U, VP, V);
  // child event streams with one event of prefetch
  int i = 0, j = 0;
  Ev cL, cR;
  typename EIN::Raw nL = EIN::none(), nR = EIN::none();
  cL.t = cR.t = INF;
  if (active) {
    if (kL > 0) cL = evL.get(0);
    if (kR > 0) cR = evR.get(0);
    if (EIN::kPrefetch) {  // HBM streams: one event of prefetch (packed)
      if (kL > 0) nL = evL.raw(kL > 1 ? 1 : 0);
      if (kR > 0) nR = evR.raw(kR > 1 ? 1 : 0);
    }
  }
  long long k = 0;
  double tcur = -INF;
  // Branch-free step: all 32 lanes (32 different jobs) iterate together until
  // every job is done -- the vote at the loop head keeps the warp converged;
  // a finished lane's step is a no-op (every store and load predicated).
  while (__any_sync(FULL, active)) {
    double best = INF;
    int which = -1;
    if (cL.t > tcur && cL.t < best) { best = cL.t; which = 0; }
    if (cR.t > tcur && cR.t < best) { best = cR.t; which = 1; }
    if (c2 > tcur && c2 < best) { best = c2; which = 2; }
    if (c3 > tcur && c3 < best) { best = c3; which = 3; }
    if (c4 > tcur && c4 < best) { best = c4; which = 4; }
    if (c5 > tcur && c5 < best) { best = c5; which = 5; }
    active = active && which >= 0;
    const bool left = CHILD && active && which == 0, right = CHILD && active && which == 1;
    const bool child = left || right;
    const bool b2 = active && which == 2, b3 = active && which == 3;
    const bool b4 = active && which == 4, b5 = active && which == 5;
    const int off = left ? 0 : roff;
    const int Ea = (left ? cL.a : cR.a) + off, Eb = (left ? cL.b : cR.b) + off,
              Ec = (left ? cL.c : cR.c) + off, Ek = left ? cL.kind : cR.kind;
    // the one link word this step reads: the child event's point, or the
    // new bridge foot (whose far neighbour becomes the cached neighbour)
    const int nf = b2 ? un : (b3 ? up : (b4 ? vn : vp));
    const int z = child ? Eb : ((b2 | b3 | b4 | b5) ? nf : 0);
    short2 lz = make_short2(NIL, NIL);
    if (active) lz = S.LK(z);
    const int e = Eb, p = lz.x, q = lz.y;
    bool del = false;
    if (child && p != NIL) del = S.LK(p).y == e;
    if (child && (p != Ea || q != Ec || (del ? EV_DEL : EV_INS) != Ek)) {
      err = E_FASTPATH;
      active = false;
    }
    const bool act = child && active;
    // _act (_ckernels.pyx:49-60) on the child event
    if (act) {
      S.LK(p).y = static_cast<short>(del ? q : e);
      S.LK(q).x = static_cast<short>(del ? p : e);
    }
    // the cached neighbour that changes and its new point
    int slot = -1, newpt = NIL;
    if (act) {
      slot = (p == u) ? 0 : (q == u) ? 1 : (p == v) ? 2 : (q == v) ? 3 : -1;
      newpt = del ? ((slot & 1) ? p : q) : e;
    } else if (active) {
      slot = which - 2;
      newpt = (b2 | b4) ? lz.y : lz.x;
    }
    // emission (old feet), the reference's rules
    bool emit = active && (child ? (left ? e < u : e > v) : true);
    if (emit && k >= capRef - 1) {
      err = H3D_E_OVERFLOW;
      active = emit = false;
      slot = -1;
    }
    const int ea = child ? p : (b3 ? up : u);
    const int eb = child ? e : (b2 ? un : (b3 ? u : (b4 ? v : vp)));
    const int ec = child ? q : (b4 ? vn : v);
    const int ek = child ? Ek : ((b3 | b4) ? EV_DEL : EV_INS);
    if (emit) {
      Ev o;
      o.t = best;
      o.a = ea;
      o.b = eb;
      o.c = ec;
      o.kind = ek;
      out.put(k, o);
      const unsigned f = S.FI(eb);
      if (!(f & SL::kFiEv))
        S.FI(eb) = static_cast<typename SL::FiT>(f | SL::kFiEv | static_cast<unsigned>(ea) |
                                                 (static_cast<unsigned>(ec) << SL::kFiShift));
    }
    k += emit;
    // advance the consumed child stream
    if (left) {
      ++i;
      if (EIN::kPrefetch) {
        // unconditional load straight into the loop-carried register (a
        // predicated one compiles to a register move that waits for the
        // load)
        cL = i < kL ? EIN::unpack(nL) : EIN::unpack(EIN::none());
        nL = evL.raw(min(i + 1, kL - 1));  // clamped: never reads a slot no level wrote
      } else {
        if (i < kL) cL = evL.get(i); else cL.t = INF;
      }
    }
    if (right) {
      ++j;
      if (EIN::kPrefetch) {
        cR = j < kR ? EIN::unpack(nR) : EIN::unpack(EIN::none());
        nR = evR.raw(min(j + 1, kR - 1));
      } else {
        if (j < kR) cR = evR.get(j); else cR.t = INF;
      }
    }
    // rotate the bridge neighbourhood (selects), fetch the one new point
    // A bridge move's new foot takes BOTH its links from its link word: the
    // other one is normally the old foot, but not when a child event has
    // deleted the old foot from its chain while it was still a foot (a
    // near-degenerate input; the reference then reads the current links)
    const bool bm = b2 | b3 | b4 | b5;
    const int oth = bm ? ((b2 | b4) ? lz.x : lz.y) : NIL;
    const int oldfoot = (b2 | b3) ? u : v;
    const bool oth_new = bm && oth != oldfoot;
    const P3 N = S.pt(slot >= 0 ? newpt : NIL, pts, zs);
    const P3 N2 = S.pt(oth_new ? oth : NIL, pts, zs);
    const P3 OF = (b2 | b3) ? U : V;
    const P3 O2 = oth_new ? N2 : OF;
    const int u1 = b2 ? un : (b3 ? up : u), v1 = b4 ? vn : (b5 ? vp : v);
    const P3 U1 = b2 ? UN : (b3 ? UP : U), V1 = b4 ? VN : (b5 ? VP : V);
    const int un1 = (slot == 0) ? newpt : (b3 ? oth : un);
    const int up1 = (slot == 1) ? newpt : (b2 ? oth : up);
    const int vn1 = (slot == 2) ? newpt : (b5 ? oth : vn);
    const int vp1 = (slot == 3) ? newpt : (b4 ? oth : vp);
    const P3 UN1 = (slot == 0) ? N : (b3 ? O2 : UN);
    const P3 UP1 = (slot == 1) ? N : (b2 ? O2 : UP);
    const P3 VN1 = (slot == 2) ? N : (b5 ? O2 : VN);
    const P3 VP1 = (slot == 3) ? N : (b4 ? O2 : VP);
    u = u1; v = v1; un = un1; up = up1; vn = vn1; vp = vp1;
    if (SL::kReload) {
      // coordinates in shared memory: only the ids rotate; the six points
      // are re-read when the candidate times are recomputed (the same
      // values, so the same rounded times)
      if (__any_sync(FULL, slot >= 0)) {
        const P3 Uc = S.pt(u, pts, zs), Vc = S.pt(v, pts, zs), UNc = S.pt(un, pts, zs),
                 UPc = S.pt(up, pts, zs), VNc = S.pt(vn, pts, zs), VPc = S.pt(vp, pts, zs);
        c2 = evt3(u, un, v, Uc, UNc, Vc);
        c3 = evt3(up, u, v, UPc, Uc, Vc);
        c4 = evt3(u, v, vn, Uc, Vc, VNc);
        c5 = evt3(u, vp, v, Uc, VPc, Vc);
      }
    } else {
      U = U1; V = V1; UN = UN1; UP = UP1; VN = VN1; VP = VP1;
      if (__any_sync(FULL, slot >= 0)) {
        c2 = evt3(u, un, v, U, UN, V);
        c3 = evt3(up, u, v, UP, U, V);
        c4 = evt3(u, v, vn, U, V, VN);
        c5 = evt3(u, vp, v, U, VP, V);
      }
    }
    if (active) tcur = best;
  }
  return err ? err : k;
}

// shared bytes of one warp job: records, first table, merged child events
__host__ __device__ __forceinline__ long long warp_job_bytes(int nS, int kin) {
  return align8(32ll * nS + 4ll * nS) + 24ll * kin;
}

// histogram bin of a CTA's point sum (six bins per octave) and the largest
// sum a bin holds
__host__ __device__ __forceinline__ int need_bin(unsigned long long t) {
  const int b = static_cast<int>(6.0 * log2(static_cast<double>(t)));
  return b < 0 ? 0 : (b >= kNeedHistBins ? kNeedHistBins - 1 : b);
}
inline long long need_bin_max(int b) { return static_cast<long long>(floor(exp2((b + 1) / 6.0))); }

// Shared-memory need of the thread-per-job launch, for every jobs-per-CTA
// choice at once: out[r] = max over CTAs of sum(nS) when a CTA takes
// 32 >> r consecutive jobs (r = 0..5); out[6] = largest single nS; out[7] =
// largest shared-memory need of one warp-per-job merge; out[8] = largest
// merged child log of one job; out[9] = all merged child logs.  One warp per 32
// jobs, coalesced header reads.
__global__ void k_tpj_need(Pass2 P, long long n, int level, long long j0, long long j1,
                           unsigned long long *out, const long long *err, long long *stamp) {
  if (stamp && blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x == 0) {  // level start (ns)
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    *stamp = static_cast<long long>(t);
  }
  // out[10] = the error word, read back with the measurement (one copy)
  if (blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x == 0)
    out[10] = static_cast<unsigned long long>(*reinterpret_cast<const volatile long long *>(err));
  const GroupBuf in = blockIdx.y ? P.in1 : P.in0;
  const long long size = 1ll << level, half = size >> 1;
  const int lane = threadIdx.x & 31;
  const long long warps = (long long)gridDim.x * (blockDim.x >> 5);
  const long long chunks = (j1 - j0 + 31) >> 5;
  unsigned long long mx[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
  // lane kernel pools (lane.cu): per jobs-per-CTA choice r and variant
  // v = 2 * xyz + staged events
  unsigned long long lb[24];
#pragma unroll
  for (int q = 0; q < 24; ++q) lb[q] = 0;
  unsigned long long ksum = 0, nssum = 0;  // out[9] merged child events, out[11] points of the merges
  // out[kNeedHist + b]: CTAs (32 jobs) whose point sum falls in bin b
  // (b = floor(6 log2 sum): six bins per octave) -- the host sizes a split
  // level's small pool from it
  __shared__ unsigned s_hist[kNeedHistBins];
  for (int q = threadIdx.x; q < kNeedHistBins; q += blockDim.x) s_hist[q] = 0;
  __syncthreads();
  for (long long c = blockIdx.x * (long long)(blockDim.x >> 5) + (threadIdx.x >> 5); c < chunks;
       c += warps) {
    const long long j = j0 + c * 32 + lane;
    unsigned long long nS = 0, wb = 0, kin = 0, b[4] = {0, 0, 0, 0};
    if (j < j1) {
      const long long L = j << level;
      const long long R_ = (L + size < n) ? L + size : n;
      if (R_ - L > half) {
        const int2 hl = in.hdr[2 * j], hr = in.hdr[2 * j + 1];
        nS = hl.x + hr.x;
        kin = hl.y + hr.y;
        wb = warp_job_bytes(static_cast<int>(nS), hl.y + hr.y);
        if (nS < 0x7fff) {
          const int oc = lane_ocap(static_cast<int>(nS), static_cast<int>(kin));
#pragma unroll
          for (int v = 0; v < 4; ++v)
            b[v] = lane_slice_bytes(static_cast<int>(nS), (v & 1) ? oc : 0, v >= 2);
        } else {
#pragma unroll
          for (int v = 0; v < 4; ++v) b[v] = 1ull << 40;  // never fits a lane pool
        }
      }
    }
#pragma unroll
    for (int v = 0; v < 4; ++v) {
      unsigned long long t = b[v];
      lb[6 * v + 5] = t > lb[6 * v + 5] ? t : lb[6 * v + 5];
#pragma unroll
      for (int r = 4; r >= 0; --r) {  // 2, 4, 8, 16, 32 jobs per CTA
        t += __shfl_xor_sync(FULL, t, 1 << (4 - r));
        lb[6 * v + r] = t > lb[6 * v + r] ? t : lb[6 * v + r];
      }
    }
    mx[6] = nS > mx[6] ? nS : mx[6];
    mx[7] = wb > mx[7] ? wb : mx[7];
    mx[8] = kin > mx[8] ? kin : mx[8];
    ksum += kin;
    nssum += nS;
    unsigned long long t = nS;
    mx[5] = t > mx[5] ? t : mx[5];  // 1 job per CTA
#pragma unroll
    for (int r = 4; r >= 0; --r) {  // 2, 4, 8, 16, 32 jobs per CTA
      t += __shfl_xor_sync(FULL, t, 1 << (4 - r));
      mx[r] = t > mx[r] ? t : mx[r];
    }
    if (lane == 0 && t > 0) atomicAdd(&s_hist[need_bin(t)], 1u);
  }
  // warp, then block reduction; one atomic per value per block
  __shared__ unsigned long long red[32][34];
  const int w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int o = 16; o; o >>= 1) ksum += __shfl_xor_sync(FULL, ksum, o);
  for (int o = 16; o; o >>= 1) nssum += __shfl_xor_sync(FULL, nssum, o);
  if (lane == 0 && nssum) atomicAdd(out + 11, nssum);
#pragma unroll
  for (int r = 0; r < 9; ++r) {
    unsigned long long m = mx[r];
    for (int o = 16; o; o >>= 1) {
      const unsigned long long x = __shfl_xor_sync(FULL, m, o);
      m = x > m ? x : m;
    }
    if (lane == 0) red[w][r] = m;
  }
  if (lane == 0) red[w][9] = ksum;
#pragma unroll
  for (int r = 0; r < 24; ++r) {
    unsigned long long m = lb[r];
    for (int o = 16; o; o >>= 1) {
      const unsigned long long x = __shfl_xor_sync(FULL, m, o);
      m = x > m ? x : m;
    }
    if (lane == 0) red[w][10 + r] = m;
  }
  __syncthreads();
  if (threadIdx.x < 34) {
    unsigned long long m = 0;
    for (int q = 0; q < nw; ++q) {
      const unsigned long long x = red[q][threadIdx.x];
      m = threadIdx.x == 9 ? m + x : (x > m ? x : m);
    }
    // out[16 + 6 v + r]: lane pools of variant v (2 * xyz + staged events)
    const int slot = threadIdx.x < 10 ? threadIdx.x : 6 + threadIdx.x;
    if (m) {
      if (threadIdx.x == 9) atomicAdd(out + 9, m); else atomicMax(out + slot, m);
    }
  }
  for (int q = threadIdx.x; q < kNeedHistBins; q += blockDim.x)
    if (s_hist[q]) atomicAdd(out + kNeedHist + q, static_cast<unsigned long long>(s_hist[q]));
}

// One CTA (32 jobs of pass `pass`, job chunk `blk`).  With ovf (a split
// level): a CTA whose jobs do not fit the pool is appended to the overflow
// list for the big-pool launch instead of failing.
template <bool XYZ>
__device__ __forceinline__ void tpj_body(Pass2 P, const double *__restrict__ pts, long long n, int level,
                                         long long j0, long long j1, long long *err, int pool, int jpc,
                                         int prefetch, long long *spec, long long blk, int pass, int *ovf,
                                         long long ovf_cap) {
  // an earlier level failed, or (a replayed plan, spec) did not fit: stop
  // (warp-uniform; the words it reads may be stale)
  if (__any_sync(0xffffffffu, *reinterpret_cast<volatile long long *>(err) != 0 ||
                                  (spec && *reinterpret_cast<volatile long long *>(spec) != 0)))
    return;
  const GroupBuf in = pass ? P.in1 : P.in0;
  const GroupBuf out = pass ? P.out1 : P.out0;
  const double zs = pass ? -1.0 : 1.0;
  extern __shared__ __align__(16) unsigned char smem[];
  const int lane = threadIdx.x;
  const long long size = 1ll << level, half = size >> 1;
  // jpc (1..32) jobs per CTA: lanes >= jpc idle (large jobs, few per CTA)
  const long long j = j0 + blk * jpc + lane;
  const long long L = j << level, M = L + half;
  const long long R_ = (L + size < n) ? L + size : n;
  int nSL = 0, kL = 0, nSR = 0, kR = 0;
  bool merge = false;
  if (lane < jpc && j < j1) {
    const int2 hl = in.hdr[2 * j];
    nSL = hl.x;
    kL = hl.y;
    if (R_ - L > half) {
      const int2 hr = in.hdr[2 * j + 1];
      nSR = hr.x;
      kR = hr.y;
      merge = true;
    } else {  // carry (copy_log, parallel.py:107-108): the short last group
      for (int p = 0; p < nSL; ++p) {
        out.lnk[L + p] = in.lnk[L + p];
        out.gid[L + p] = in.gid[L + p];
      }
      for (int e = 0; e < kL; ++e) out.ev[2 * L + e] = in.ev[2 * L + e];
      out.hdr[j] = hl;
    }
  }
  const int nS = nSL + nSR;
  if (merge && nS >= 0x7fff) {  // int16 local ids; the host never routes such jobs here ...
    if (spec)  // ... unless it replays a plan: report the level, it is redone measured
      atomicCAS(reinterpret_cast<unsigned long long *>(spec), 0ull, static_cast<unsigned long long>(level));
    else
      raise_err(err, E_FASTPATH);
    merge = false;
  }
  // pack the slices: warp exclusive prefix sum of the slice sizes
  const int bytes = merge ? tpj_slice_bytes(nS, XYZ) : 0;
  int off = bytes;
  for (int o = 1; o < 32; o <<= 1) {
    const int t = __shfl_up_sync(FULL, off, o);
    if (lane >= o) off += t;
  }
  const int total = __shfl_sync(FULL, off, 31);
  off -= bytes;
  if (total > pool) {  // the host sizes the pool from the measured need (or a replayed plan's)
    if (ovf) {  // a split level: the big-pool launch takes this CTA
      if (lane == 0) {
        const int i = atomicAdd(ovf, 1);
        if (i < ovf_cap)
          ovf[1 + i] = static_cast<int>(2 * blk + pass);
        else if (spec)  // a replayed plan's list launch is too small: measured again
          atomicCAS(reinterpret_cast<unsigned long long *>(spec), 0ull, static_cast<unsigned long long>(level));
        else
          raise_err(err, E_FASTPATH);
      }
      return;
    }
    if (lane == 0) {
      if (spec)
        atomicCAS(reinterpret_cast<unsigned long long *>(spec), 0ull, static_cast<unsigned long long>(level));
      else
        raise_err(err, E_FASTPATH);
    }
    return;
  }
  // per-job metadata for the cooperative phases (shared, no shuffles); the
  // cooperative loops run over the concatenated points (events) of the 32
  // jobs, 32 elements per iteration, each lane locating its job by a binary
  // search of the prefix sums
  __shared__ long long s_L[32], s_M[32];
  __shared__ int s_off[32], s_nSL[32], s_pre[33], s_epre[33], s_cnt[32];
  s_L[lane] = L;
  s_M[lane] = M;
  s_off[lane] = off;
  s_nSL[lane] = nSL;
  {
    int c = merge ? nS : 0;
    for (int o = 1; o < 32; o <<= 1) {
      const int t = __shfl_up_sync(FULL, c, o);
      if (lane >= o) c += t;
    }
    s_pre[lane + 1] = c;
    if (lane == 0) s_pre[0] = 0;
  }
  __syncwarp();
  const int tot_pts = s_pre[32];
  auto job_of = [&](const int *pre, int x) {
    int jj = 0;
#pragma unroll
    for (int st = 16; st; st >>= 1)
      if (pre[jj + st] <= x) jj += st;
    return jj;
  };
  // ---- stage (cooperative, coalesced; U elements per lane in flight)
  constexpr int U = 4;
  int js = 0;
  for (int x0 = 0; x0 < tot_pts; x0 += 32 * U) {
    int jj[U], p[U];
    long long src[U];
    int2 l[U];
    int g[U];
#pragma unroll
    for (int q = 0; q < U; ++q) {
      const int x = x0 + q * 32 + lane;
      const int xc = x < tot_pts ? x : tot_pts - 1;
      while (s_pre[js + 1] <= xc) ++js;  // the job index only advances
      jj[q] = js;
      p[q] = x - s_pre[jj[q]];
      const int m_nSL = s_nSL[jj[q]];
      src[q] = p[q] < m_nSL ? s_L[jj[q]] + p[q] : s_M[jj[q]] + (p[q] - m_nSL);
    }
#pragma unroll
    for (int q = 0; q < U; ++q) {
      if (x0 + q * 32 + lane < tot_pts) {
        l[q] = in.lnk[src[q]];
        g[q] = in.gid[src[q]];
      }
    }
    P3 c[U];
    if (XYZ) {
#pragma unroll
      for (int q = 0; q < U; ++q)
        if (x0 + q * 32 + lane < tot_pts) c[q] = load_pt(pts, g[q], zs);
    } else if (prefetch) {
      // the sweep reads these rows through the ids: start them towards L2
      // (pays on the large, DRAM-miss-bound levels; the host decides)
#pragma unroll
      for (int q = 0; q < U; ++q)
        if (x0 + q * 32 + lane < tot_pts)
          asm volatile("prefetch.global.L2 [%0];" ::"l"(pts + 3ll * g[q]));
    }
#pragma unroll
    for (int q = 0; q < U; ++q) {
      if (x0 + q * 32 + lane >= tot_pts) continue;
      const int m_nS = s_pre[jj[q] + 1] - s_pre[jj[q]], m_nSL = s_nSL[jj[q]];
      const TpjSlice<XYZ> S(smem + s_off[jj[q]], m_nS);
      int2 lq = l[q];
      if (p[q] >= m_nSL) {
        if (lq.x != NIL) lq.x += m_nSL;
        if (lq.y != NIL) lq.y += m_nSL;
      }
      S.lk[p[q]] = make_short2(static_cast<short>(lq.x), static_cast<short>(lq.y));
      S.gd[p[q]] = g[q];
      if (XYZ) {
        S.x[p[q]] = c[q].x;
        S.y[p[q]] = c[q].y;
        S.z[p[q]] = c[q].z;
      }
    }
  }
  __syncwarp();
  long long k = 0;
  int u0 = 0, v0 = 0;
  const TpjSlice<XYZ> S(smem + off, nS);
  if (merge) {
    // chain flags: p is on its child's -inf chain iff its prev points back
    for (int p = 0; p < nS; ++p) {
      const int pr = S.lk[p].x;
      const bool chain = p == 0 || p == nSL || (pr != NIL && S.lk[pr].y == p);
      S.fi[p] = chain ? FI_CHAIN : 0u;
    }
  }
  // all 32 lanes enter the sweep together (idle lanes inactive)
  k = merge_tpj2(S, merge, nSL - 1, nSL, pts, zs, GEvIn{in.ev + 2 * L}, kL, GEvIn{in.ev + 2 * M}, kR,
                 GEvOut{out.ev + 2 * L}, 2 * (R_ - L), R_ - L, &u0, &v0);
  if (merge && k < 0) {
    raise_err(err, k);
    merge = false;
  }
  int cnt = 0;
  if (merge) {
    // ---- start-of-time links of the merged group (replaces the rewind,
    // DESIGN.md 3.3): the merged -inf chain is every chain-flagged point
    // left of u0 (inclusive) or right of v0, linked in x order; every other
    // kept point gets the neighbours of its first merged event (its
    // insertion).  fi becomes the old -> new id map.
    int last = NIL;
    for (int p = 0; p < nS; ++p) {
      const unsigned f = S.fi[p];
      const bool chain = (f & FI_CHAIN) && (p < nSL ? p <= u0 : p >= v0);
      if (chain) {
        S.lk[p].x = static_cast<short>(last);
        if (last != NIL) S.lk[last].y = static_cast<short>(p);
        last = p;
      } else if (f & FI_EV) {
        S.lk[p] = make_short2(static_cast<short>(f & 0x7fff), static_cast<short>((f >> 15) & 0x7fff));
      }
      S.fi[p] = (chain || (f & FI_EV)) ? static_cast<unsigned>(cnt++) : FULL;
    }
    if (last != NIL) S.lk[last].y = NIL;
  }
  __syncwarp();
  {  // prefix sums of the surviving jobs' kept points and events
    int c = merge ? nS : 0, e = merge ? static_cast<int>(k) : 0;
    for (int o = 1; o < 32; o <<= 1) {
      const int t = __shfl_up_sync(FULL, c, o), te = __shfl_up_sync(FULL, e, o);
      if (lane >= o) {
        c += t;
        e += te;
      }
    }
    __syncwarp();
    s_pre[lane + 1] = c;
    s_epre[lane + 1] = e;
    if (lane == 0) s_pre[0] = s_epre[0] = 0;
    s_cnt[lane] = cnt;
    if (merge) out.hdr[j] = make_int2(cnt, static_cast<int>(k));
  }
  __syncwarp();
  // ---- write-out (cooperative): links + gids at their new ids, events
  // remapped in place
  bool bad = false;
  const int tot_p2 = s_pre[32], tot_ev = s_epre[32];
  int jw = 0;
  for (int x = lane; x < tot_p2; x += 32) {
    while (s_pre[jw + 1] <= x) ++jw;  // the job index only advances
    const int jj = jw;
    const int p = x - s_pre[jj];
    const TpjSlice<XYZ> T(smem + s_off[jj], s_pre[jj + 1] - s_pre[jj]);
    const unsigned id = T.fi[p];
    if (id == FULL) continue;
    const short2 l = T.lk[p];
    int2 o;
    o.x = l.x == NIL ? NIL : static_cast<int>(T.fi[l.x]);
    o.y = l.y == NIL ? NIL : static_cast<int>(T.fi[l.y]);
    bad |= (o.x == -1 && l.x != NIL) | (o.y == -1 && l.y != NIL);
    out.lnk[s_L[jj] + id] = o;
    out.gid[s_L[jj] + id] = T.gd[p];
  }
  {  // events: 4 read-backs in flight per lane; the job index only advances
    int jj = 0;
    for (int x0 = 0; x0 < tot_ev; x0 += 4 * 32) {
      int jq[4];
      EvP *ptr[4];
      Ev o[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int x = x0 + q * 32 + lane;
        if (x < tot_ev) {
          while (s_epre[jj + 1] <= x) ++jj;
          jq[q] = jj;
          ptr[q] = out.ev + 2 * s_L[jj] + (x - s_epre[jj]);
          o[q] = *ptr[q];
        }
      }
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        if (x0 + q * 32 + lane >= tot_ev) continue;
        const TpjSlice<XYZ> T(smem + s_off[jq[q]], s_pre[jq[q] + 1] - s_pre[jq[q]]);
        const unsigned na = T.fi[o[q].a], nb = T.fi[o[q].b], nc = T.fi[o[q].c];
        bad |= (na == FULL) | (nb == FULL) | (nc == FULL);
        o[q].a = static_cast<int>(na);
        o[q].b = static_cast<int>(nb);
        o[q].c = static_cast<int>(nc);
        *ptr[q] = EvP(o[q]);
      }
    }
  }
  if (__any_sync(FULL, bad) && lane == 0) raise_err(err, E_FASTPATH);
}

// the lane-per-job level kernel.  Two register budgets of the same body: the
// compiler's own (156 registers, 12 warps/SM) and a 128-register cap (16
// warps/SM) that pays at the lower levels, where more resident jobs hide the
// gathers (measured per level, g_tpj_cap_level)
__device__ __forceinline__ void level_stamp(long long *stamp) {
  if (stamp && blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x == 0) {  // level start (ns)
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    *stamp = static_cast<long long>(t);
  }
}
template <bool XYZ>
__global__ void __launch_bounds__(32) k_fast_tpj(Pass2 P, const double *__restrict__ pts, long long n,
                                                 int level, long long j0, long long j1, long long *err,
                                                 int pool, int jpc, int prefetch, long long *spec,
                                                 long long *stamp, int *ovf, long long ovf_cap) {
  level_stamp(stamp);
  tpj_body<XYZ>(P, pts, n, level, j0, j1, err, pool, jpc, prefetch, spec, lvl_blk(), lvl_pass(), ovf, ovf_cap);
}
template <bool XYZ>
__global__ void __launch_bounds__(32, 16) k_fast_tpj_r128(Pass2 P, const double *__restrict__ pts, long long n,
                                                          int level, long long j0, long long j1, long long *err,
                                                          int pool, int jpc, int prefetch, long long *spec,
                                                          long long *stamp, int *ovf, long long ovf_cap) {
  level_stamp(stamp);
  tpj_body<XYZ>(P, pts, n, level, j0, j1, err, pool, jpc, prefetch, spec, lvl_blk(), lvl_pass(), ovf, ovf_cap);
}
// the CTAs a split level's small-pool launch left (the list it wrote),
// with the level's full pool; any grid (a CTA loops over the list)
__global__ void __launch_bounds__(32) k_fast_tpj_ovf(Pass2 P, const double *__restrict__ pts, long long n,
                                                     int level, long long j0, long long j1, long long *err,
                                                     int pool, int jpc, int prefetch, long long *spec,
                                                     const int *ovf) {
  const int cnt = *reinterpret_cast<const volatile int *>(ovf);
  for (int i = blockIdx.x; i < cnt; i += gridDim.x) {
    const int e = ovf[1 + i];
    tpj_body<false>(P, pts, n, level, j0, j1, err, pool, jpc, prefetch, spec, e >> 1, e & 1, nullptr, 0);
    __syncwarp();
  }
}

// ------------------------------------------------------------- leaf levels
// Levels 1..B fused: one LANE owns a block of 2^B consecutive sorted points
// and runs every merge of levels 1..B inside its block (parallel.py's level
// loop restricted to the block: the jobs of a level never cross a 2^B
// boundary), with all state in lane-interleaved shared memory -- points,
// links, first-event info and two event buffers (8-bit block-local ids).
// Nothing touches HBM between levels; groups stay uncompacted inside the
// block (a hidden point is never referenced again), and the level-B group
// is compacted and written in the compact-group format the per-level
// kernels read.  Per lane: 30 B per point + 2 x 2 x 2 B event words.
template <int B>
__host__ __device__ constexpr int leaf_lane_bytes() {
  return (1 << B) * (24 + 4 + 2) + 2 * (2 << B) * 2 + ((1 << B) / 2) * 4;
}

// 20 resident CTAs per SM: 10 KB of shared memory each at B = 3, and the
// register budget that allows it (96; a few spilled words, measured 3.7 %
// faster than 112 registers at 16 CTAs)
template <int B>
__global__ void __launch_bounds__(32, 20) k_fast_leaf(Pass2 P, const double *__restrict__ pts,
                                                  long long n, long long p0, long long p1,
                                                  long long *err) {
  // an earlier level failed: stop (warp-uniform; the words it reads may be stale)
  if (__any_sync(0xffffffffu, *reinterpret_cast<volatile long long *>(err) != 0)) return;
  constexpr int NP = 1 << B;
  const int pass = lvl_pass();
  const GroupBuf out = pass ? P.out1 : P.out0;
  const double zs = pass ? -1.0 : 1.0;
  extern __shared__ __align__(16) unsigned char smem[];
  const int lane = threadIdx.x;
  const long long blk = (p0 >> B) + lvl_blk() * 32 + lane;
  const long long base = blk << B;
  const long long top = p1 < n ? p1 : n;
  const int cnt = base < top ? static_cast<int>((top - base) < NP ? (top - base) : NP) : 0;
  // lane-interleaved arrays: element i of this lane at [i * 32 + lane]
  double *X = reinterpret_cast<double *>(smem) + lane;
  double *Y = X + 32 * NP;
  double *Z = Y + 32 * NP;
  short2 *LK = reinterpret_cast<short2 *>(reinterpret_cast<double *>(smem) + 32 * 3 * NP) + lane;
  unsigned short *FI = reinterpret_cast<unsigned short *>(LK - lane + 32 * NP) + lane;
  constexpr unsigned FULL16 = 0xffffu;  // "not kept" in the 16-bit words
  unsigned short *EW0 = reinterpret_cast<unsigned short *>(FI - lane + 32 * NP) + lane;
  unsigned short *EW1 = EW0 + 32 * 2 * NP;
  int *KG = reinterpret_cast<int *>(EW1 - lane + 32 * 2 * NP);
  for (int p = 0; p < NP; ++p) {
    double x = 0.0, y = 0.0, z = 0.0;
    if (p < cnt) {
      const double *q = pts + 3 * (base + p);
      x = q[0];
      y = q[1];
      z = zs * q[2];
    }
    X[p * 32] = x;
    Y[p * 32] = y;
    Z[p * 32] = z;
    // level 1: pairs linked (a lone last point is a carry)
    const bool has_pair = (p ^ 1) < cnt;
    LK[p * 32] = (p & 1) ? make_short2(has_pair ? p - 1 : NIL, NIL)
                         : make_short2(NIL, has_pair ? p + 1 : NIL);
  }
  for (int g = 0; g < NP / 2; ++g) KG[g * 32 + lane] = 0;
  TpjSlice<true, 32> S;
  S.x = X;
  S.y = Y;
  S.z = Z;
  S.lk = LK;
  S.gd = nullptr;
  S.fi = FI;
  bool ok = true;
  int u0 = 0, v0 = 0;
  long long kfin = 0;
  unsigned short *EWi = EW0, *EWo = EW1;
#pragma unroll 1
  for (int lv = 2; lv <= B; ++lv) {
    const int size = 1 << lv, half = size >> 1;
#pragma unroll 1
    for (int g = 0; g < NP / size; ++g) {
      const int L = g * size, M = L + half, R = (L + size < cnt) ? L + size : cnt;
      const bool merge = ok && R - L > half;
      const int kL = KG[(2 * g) * 32 + lane], kR = KG[(2 * g + 1) * 32 + lane];
      if (!merge && L < cnt) {  // carry (copy_log): the short last group
        for (int e = 0; e < kL; ++e) EWo[(2 * L + e) * 32] = EWi[(2 * L + e) * 32];
      }
      // block-relative ids throughout (links, events, first-event info)
      if (merge) {
        for (int p = L; p < R; ++p) {
          const int pr = S.LK(p).x;
          const bool chain = p == L || p == M || (pr != NIL && S.LK(pr).y == p);
          S.FI(p) = static_cast<unsigned short>(chain ? S.kFiChain : 0u);
        }
      }
      const long long k = merge_tpj2(
          S, merge, M - 1, 0, pts, zs, LEvIn{X, Y, Z, EWi + 2 * L * 32}, kL,
          LEvIn{X, Y, Z, EWi + 2 * M * 32}, kR, LEvOut{EWo + 2 * L * 32},
          2 * (R - L), R - L, &u0, &v0);
      if (merge && k < 0) {
        raise_err(err, k);
        ok = false;
      }
      if (merge && ok) {
        // start-of-time links, no compaction inside the block
        int last = NIL;
        for (int p = L; p < R; ++p) {
          const unsigned f = S.FI(p);
          const bool chain = (f & S.kFiChain) && (p < M ? p <= u0 : p >= v0);
          if (chain) {
            S.LK(p).x = static_cast<short>(last);
            if (last != NIL) S.LK(last).y = static_cast<short>(p);
            last = p;
          } else if (f & S.kFiEv) {
            S.LK(p) = make_short2(static_cast<short>(f & S.kFiMask),
                                  static_cast<short>((f >> S.kFiShift) & S.kFiMask));
          } else {
            // hidden from here on: NIL links, so no later chain test can
            // take a stale link for a chain link (the compact kernels drop
            // such points instead)
            S.LK(p) = make_short2(NIL, NIL);
          }
          if (lv == B) S.FI(p) = (chain || (f & S.kFiEv)) ? 1 : 0;  // keep flag
        }
        if (last != NIL) S.LK(last).y = NIL;
      }
      KG[g * 32 + lane] = merge ? static_cast<int>(k) : (L < cnt ? kL : 0);
      kfin = KG[g * 32 + lane];
    }
    unsigned short *tw = EWi; EWi = EWo; EWo = tw;
    __syncwarp();
  }
  // ---- level-B group: compact (kept = merged -inf chain U logged points)
  // and write it out; a short last block whose top merge was a carry keeps
  // the flags of its last merged level
  if (!ok || cnt == 0) return;
  const bool top_merged = cnt > NP / 2;
  if (!top_merged) {
    // re-derive keep flags: chain membership + logged points of the group
    for (int p = 0; p < cnt; ++p) FI[p * 32] = 0u;
    int p = 0;
    while (p != NIL && p < cnt) {  // -inf chain from point 0
      FI[p * 32] = 1u;
      p = LK[p * 32].y;
    }
    for (int e = 0; e < kfin; ++e) FI[((EWi[e * 32] >> 4) & 0xf) * 32] = 1u;
  }
  int m = 0;
  for (int p = 0; p < cnt; ++p) {
    const bool keep = FI[p * 32] != 0u;
    FI[p * 32] = static_cast<unsigned short>(keep ? m++ : FULL16);
  }
  bool bad = false;
  auto new_id = [&](int q) {  // -1: not kept
    const unsigned v = FI[q * 32];
    return v == FULL16 ? -1 : static_cast<int>(v);
  };
  for (int p = 0; p < cnt; ++p) {
    const unsigned id = FI[p * 32];
    if (id == FULL16) continue;
    const short2 l = LK[p * 32];
    int2 o;
    o.x = l.x == NIL ? NIL : new_id(l.x);
    o.y = l.y == NIL ? NIL : new_id(l.y);
    bad |= (o.x == -1 && l.x != NIL) | (o.y == -1 && l.y != NIL);
    out.lnk[base + id] = o;
    out.gid[base + id] = static_cast<int>(base + p);
  }
  EvP *evo = out.ev + 2 * base;
  for (int e = 0; e < kfin; ++e) {
    const unsigned w = EWi[e * 32];
    Ev o;
    o.t = LEvIn{X, Y, Z, EWi}.get(e).t;  // the canonical time, re-derived
    const unsigned na = FI[(w & 0xf) * 32], nb = FI[((w >> 4) & 0xf) * 32],
                   nc = FI[((w >> 8) & 0xf) * 32];
    bad |= (na == FULL16) | (nb == FULL16) | (nc == FULL16);
    o.a = static_cast<int>(na);
    o.b = static_cast<int>(nb);
    o.c = static_cast<int>(nc);
    o.kind = static_cast<int>(w >> 12);
    evo[e] = EvP(o);
  }
  out.hdr[blk] = make_int2(m, static_cast<int>(kfin));
  if (bad) raise_err(err, E_FASTPATH);
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
__device__ void merge_logs_warp(const EvP *__restrict__ evL, int kL, const EvP *__restrict__ evR,
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
__device__ long long merge_warp(Rec *R, int nSL, const Ev *seq, int kin, EvP *out,
                                int *first, long long capRef, long long limitRef, int *pu0,
                                int *pv0) {
  const int lane = threadIdx.x & 31;
  const unsigned ltmask = (1u << lane) - 1;
  int u = nSL - 1, v = nSL, st = 0;
  if (lane == 0) st = bridge_rec(R, &u, &v, limitRef);
  // lane 0's walk reads R; the window retire below writes it (WAR across
  // lanes): a memory barrier for the warp, not just the shuffle's rendezvous
  __syncwarp();
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
          out[pos] = EvP(o);
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
                  out[k] = EvP(o);
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
        out[k] = EvP(o);
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
__device__ void rebuild_writeout(const GroupBuf &in, const GroupBuf &out, Rec *R, EvP *evo,
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
      const int2 o = (p < nSL) ? in.lnk[L + p] : in.lnk[M + (p - nSL)];
      const int off = (p < nSL) ? 0 : nSL;
      prv = (o.x == NIL) ? NIL : o.x + off;
      nxt = (o.y == NIL) ? NIL : o.y + off;
      if (p == u0) nxt = v0;
      if (p == v0) prv = u0;
    } else if (hasev) {
      prv = evo[fe].a();
      nxt = evo[fe].c();
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
    evo[e] = EvP(o);
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
  // E: move links and gids (chunked read-all / write; ids only move left,
  // and a gid write only lands on ids already consumed)
  for (int p0 = 0; p0 < nS; p0 += 32) {
    const int p = p0 + lane;
    int id = -1, g = 0;
    int2 l;
    if (p < nS) {
      id = first[p];
      if (id >= 0) {
        l = make_int2(R[p].prev, R[p].next);
        g = in.gid[p < nSL ? L + p : M + (p - nSL)];
      }
    }
    __syncwarp();
    if (id >= 0) {
      out.lnk[L + id] = l;
      out.gid[L + id] = g;
    }
    __syncwarp();
  }
  if (__any_sync(FULL, bad) && lane == 0) raise_err(err, E_FASTPATH);
  if (lane == 0) out.hdr[gidx] = make_int2(cnt, k);
}


// One warp per merge job (levels with few, large jobs).  A job's records,
// first table and time-merged child events are staged in the CTA's shared
// pool when they fit (warps whose jobs do not fit wait a round), else they
// live in HBM scratch inside the job's own output slots (records at
// out.rec[L..], first table in out.gid[L..]) with the merged child events
// in the pass's HBM scratch (PassWS::seq).
template <int WARPS>
__global__ void __launch_bounds__(WARPS * 32) k_fast_warp(Pass2 P, const double *__restrict__ pts,
                                                          long long n, int level,
                                                          long long j0, long long j1,
                                                          long long *err, int pool,
                                                          Ev *gseq0, Ev *gseq1, Rec *grec0,
                                                          Rec *grec1) {
  // an earlier level failed: stop (warp-uniform; the words it reads may be stale)
  if (__any_sync(0xffffffffu, *reinterpret_cast<volatile long long *>(err) != 0)) return;
  const GroupBuf in = blockIdx.y ? P.in1 : P.in0;
  const GroupBuf out = blockIdx.y ? P.out1 : P.out0;
  Ev *gseq = blockIdx.y ? gseq1 : gseq0;
  Rec *grec = blockIdx.y ? grec1 : grec0;
  const double zs = blockIdx.y ? -1.0 : 1.0;
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
        out.lnk[L + p] = in.lnk[L + p];
        out.gid[L + p] = in.gid[L + p];
      }
      for (int e = lane; e < kL; e += 32) out.ev[2 * L + e] = in.ev[2 * L + e];
      if (lane == 0) out.hdr[j] = hl;
    }
  }
  const int nS = nSL + nSR, kin = kL + kR;
  if (merge && nS >= kEvIdMax) {  // stored events carry 21-bit local ids
    if (lane == 0) raise_err(err, E_FASTPATH);
    merge = false;
  }
  const long long need = merge ? warp_job_bytes(nS, kin) : 0;
  const bool global_mode = merge && need > pool;
  bool pending = merge && !global_mode;
  auto run_job = [&](Rec *Rr, int *first, Ev *seq) {
    for (int p = lane; p < nS; p += 32) {
      const long long src = (p < nSL) ? L + p : M + (p - nSL);
      const int2 l = in.lnk[src];
      const P3 c = load_pt(pts, in.gid[src], zs);
      Rec r;
      r.x = c.x;
      r.y = c.y;
      r.z = c.z;
      r.prev = l.x;
      r.next = l.y;
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
    EvP *evo = out.ev + 2 * L;
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
    // in HBM: records in the pass's record scratch at grec[L..L+nS) (nS <=
    // R-L), first table in out.gid[L..), merged child events in the level
    // scratch at gseq[2L..)
    run_job(grec + L, out.gid + L, gseq + 2 * L);
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

// verify mode (h3d_fast_passes*(verify = 1)): an independent check of every
// group a level wrote, one warp per group -- the header is in range, the
// kept points' ids are strictly increasing inside the group's point range
// (x order), every link is NIL or a local id, every event's facet is an
// x-ordered triple (a < b < c) of local ids, its stored time equals the
// event time RE-DERIVED from the facet's coordinates (evtime of the x-sorted
// triple, _ckernels.pyx:34-46, bit for bit) and the times strictly increase
// along the log.  A violation records H3D_E_VERIFY.
__global__ void k_verify_level(Pass2 P, const double *__restrict__ pts, long long n, int level,
                               long long j0, long long j1, long long *err, long long *diag,
                               const long long *spec) {
  // a speculative top-level chain (mini.cu) whose level (or an earlier one)
  // did not fit wrote nothing: the loop redoes it, measured, and checks then
  if (spec && *reinterpret_cast<const volatile long long *>(spec) != 0) return;
  const GroupBuf g = blockIdx.y ? P.in1 : P.in0;  // the groups the level wrote
  const double zs = blockIdx.y ? -1.0 : 1.0;
  const int lane = threadIdx.x & 31;
  const long long warps = (long long)gridDim.x * (blockDim.x >> 5);
  for (long long j = j0 + blockIdx.x * (long long)(blockDim.x >> 5) + (threadIdx.x >> 5); j < j1;
       j += warps) {
    const long long L = j << level;
    const long long R_ = (L + (1ll << level) < n) ? L + (1ll << level) : n;
    const int2 h = g.hdr[j];
    const int nS = h.x, k = h.y;
    int why = (nS < 1 || nS > R_ - L || k < 0 || k > 2 * (R_ - L) - 1) ? 1 : 0;
    long long at = 0;
    if (!why) {
      for (int p = lane; p < nS; p += 32) {
        const int gp = g.gid[L + p];
        const int2 l = g.lnk[L + p];
        if (gp < L || gp >= R_ || (p > 0 && g.gid[L + p - 1] >= gp)) why = 2, at = p;
        if (l.x < NIL || l.x >= nS || l.y < NIL || l.y >= nS) why = 3, at = p;
      }
      for (int e = lane; e < k; e += 32) {
        const Ev ev = g.ev[2 * L + e];
        if (ev.a < 0 || ev.a >= ev.b || ev.b >= ev.c || ev.c >= nS) {
          why = 4, at = e;
          continue;
        }
        const P3 A = load_pt(pts, g.gid[L + ev.a], zs), B = load_pt(pts, g.gid[L + ev.b], zs),
                 C = load_pt(pts, g.gid[L + ev.c], zs);
        const double t = evtime_xyz(A.x, A.y, A.z, B.x, B.y, B.z, C.x, C.y, C.z);
        if (__double_as_longlong(t) != __double_as_longlong(ev.t)) why = 5, at = e;
        if (e > 0 && !(g.ev[2 * L + e - 1].t < ev.t)) why = 6, at = e;
      }
    }
    if (why) {
      raise_err(err, H3D_E_VERIFY);
      // first violation: kind | level | pass | group | index (debug aid)
      if (diag)
        atomicCAS(reinterpret_cast<unsigned long long *>(diag), 0ull,
                  (static_cast<unsigned long long>(why) << 60) |
                      (static_cast<unsigned long long>(level) << 54) |
                      (static_cast<unsigned long long>(blockIdx.y) << 53) |
                      (static_cast<unsigned long long>(j & 0xffffffffll) << 20) |
                      static_cast<unsigned long long>(at & 0xfffff));
    }
  }
}

// facets of both passes: lower block then upper block, sorted indices
__global__ void k_fast_extract(GroupBuf lo, GroupBuf up, int *faces, long long cap,
                               long long *counts, long long *err) {
  // a level failed: its buffers hold nothing valid (the caller falls back)
  if (*reinterpret_cast<volatile long long *>(err) != 0) {
    if (blockIdx.x == 0 && threadIdx.x == 0) counts[0] = counts[1] = 0;
    return;
  }
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
    const Ev e = g.ev[f < kLo ? f : f - kLo];  // unpacked
    faces[3 * f] = g.gid[e.a];
    faces[3 * f + 1] = g.gid[e.b];
    faces[3 * f + 2] = g.gid[e.c];
  }
}

}  // namespace h3d

using namespace h3d;

namespace {

constexpr long long kWarpPoolMax = 200 * 1024;
long long kTpjMinTotalJobs = 148 * 32;  // H3D_TPJ_MIN_JOBS (both passes)
constexpr int kTpjPool = 200 * 1024;
int kTpjMaxLevel = 40;          // H3D_TPJ_MAX_LEVEL
long long kTpjXyzMax = 16 * 1024;  // H3D_TPJ_XYZ_KB: stage coordinates when the pool fits
long long kBigKin = 1000;          // H3D_BIG_KIN: time-split pipeline from this job log size
long long kBigTotal = 200000;     // H3D_BIG_TOTAL: ... or half that with this many child events in the level
long long kBigMaxJobs = 1ll << 18;  // H3D_BIG_MAX_JOBS: ... and fewer jobs (both passes) than this

// shared-memory attributes are per device: set once per device used
bool g_attr_done[64] = {};
bool g_env_done = false;
int g_leaf_b = 3;  // H3D_LEAF_B: levels 1..B fused (0 = off)
int g_mini = 1;    // H3D_MINI: few small jobs -> mini.cu (0 = warp kernel)
long long kMiniMaxCtas = 32 * 148;  // H3D_MINI_CTAS
// the tiny mini variant (several CTAs per SM): at most this many CTAs, and
// over the lane-per-job kernel only when the longest merged child log is at
// least kMiniTinyKin events (the lane kernel's serial path then dominates)
long long kMiniTinyCtas = 16384;  // H3D_MINI_TINY_CTAS
long long kMiniTinyKin = 160;    // H3D_MINI_TINY_KIN
// the huge mini variant (global-memory slots): at most this many CTAs, and
// only from this merged child log size (below it the shared-memory ones)
long long kMiniOneWave = 2 * 148;  // mini_one_wave: CTAs up to which the large variant runs
long long kMiniHugeCtas = 32 * 148;  // H3D_MINI_HUGE_CTAS (capped by the workspace slots)
long long kMiniHugeKin = 1000;   // H3D_MINI_HUGE_KIN
// after a level on the large mini variant, launch the remaining levels on it
// without measuring them (no read-back and host sync per level)
int g_mini_spec = 1;  // H3D_MINI_SPEC
int g_trace = 0;      // H3D_TRACE: one stderr line per routed level
long long kTpjXyzCtas = 4 * 148;  // tpj_xyz_ctas: stage coordinates on levels of at most this many CTAs
int g_tpj_split = 1;  // H3D_TPJ_SPLIT: small-pool launch + big-pool launch for levels of a few large CTAs
int g_tpj_cap_level = 6;  // H3D_TPJ_CAP_LEVEL: k_fast_tpj levels <= this at 128 registers
int g_lane = 1;       // H3D_LANE: lane-per-job levels on lane.cu (0 = k_fast_tpj)
// highest level routed to lane.cu; k_fast_tpj above (measured per level, C4:
// lane.cu 2.33 / 1.90 ms at levels 4 / 5 vs 2.60 / 2.13; k_fast_tpj ahead
// from level 6 on, profiles/r2_levels_c4.jsonl)
int g_lane_max_level = 5;  // H3D_LANE_MAX_LEVEL
long long kTpjPrefetchJobs = 1ll << 17;  // H3D_TPJ_PREFETCH: L2 prefetch of rows from this many jobs (2^18 -> 2^17: C4 level 7 -2.3 %)

// leaf kernel depth: 3 or 4 fused levels, anything below 3 = off
int leaf_depth(long long b) { return b >= 4 ? 4 : (b == 3 ? 3 : 0); }

// ---- level plans: record & replay of the routing.  A call that measured
// every level records what it launched (route + launch parameters); the next
// call with the same point range launches that plan WITHOUT the per-level
// measurement and read-back.  Every replayed kernel checks that its jobs fit
// the recorded launch (shared-memory pool, jobs per CTA, job size caps); a
// level that does not fit writes nothing, records its level in a device
// flag, and every later replayed launch exits at once -- after the single
// read-back at the end of the replay the loop resumes, measured, from that
// level (its input buffer is intact).  Results never depend on the plan:
// every route reproduces the reference's logs.
enum { REC_MINI = 0, REC_LANE = 1, REC_TPJ = 2, REC_WARP = 3, REC_BIG = 4 };
struct LevelRec {
  int lv, kind, variant, jpc, prefetch;
  long long pool;
  LaneCfg lane;
  long long pool2 = 0;  // a split lane-per-job level: the big pool (0: not split)
  int ogrid = 0;        // ... and the big-pool (or mini list) launch's grid
  int mini = -1;        // a hybrid level: the mini variant of the large CTAs' jobs
  long long big_kin = -1, big_pts = -1;  // a pipeline level: its measured totals (checked on replay)
};
struct PlanKey {
  int dev;
  long long n, p0, p1;
  int lo, hi;
  bool operator<(const PlanKey &o) const {
    if (dev != o.dev) return dev < o.dev;
    if (n != o.n) return n < o.n;
    if (p0 != o.p0) return p0 < o.p0;
    if (p1 != o.p1) return p1 < o.p1;
    if (lo != o.lo) return lo < o.lo;
    return hi < o.hi;
  }
};
std::mutex g_plan_mu;
std::map<PlanKey, std::vector<LevelRec>> g_plans;
int g_plan = 1;  // H3D_PLAN: replay recorded level plans (0 = measure every level)
}  // namespace
namespace h3d {
int g_interleave = 1;  // H3D_INTERLEAVE: the two passes of the same jobs in adjacent CTAs
}  // namespace h3d
namespace {
void plans_clear() {
  std::lock_guard<std::mutex> g(g_plan_mu);
  g_plans.clear();
}

// tuning knobs from the environment (read once; h3d_tune overrides)
void load_env_once() {
  if (g_env_done) return;
  g_env_done = true;
  if (const char *e = getenv("H3D_TPJ_MAX_LEVEL")) kTpjMaxLevel = atoi(e);
  if (const char *e = getenv("H3D_TPJ_XYZ_KB")) kTpjXyzMax = atoll(e) * 1024;
  if (const char *e = getenv("H3D_TPJ_MIN_JOBS")) kTpjMinTotalJobs = atoll(e);
  if (const char *e = getenv("H3D_LEAF_B")) g_leaf_b = atoi(e);
  if (const char *e = getenv("H3D_BIG_KIN")) kBigKin = atoll(e);
  if (const char *e = getenv("H3D_BIG_TOTAL")) kBigTotal = atoll(e);
  if (const char *e = getenv("H3D_BIG_MAX_JOBS")) kBigMaxJobs = atoll(e);
  if (const char *e = getenv("H3D_MINI")) g_mini = atoi(e);
  if (const char *e = getenv("H3D_MINI_CTAS")) kMiniMaxCtas = atoll(e);
  if (const char *e = getenv("H3D_MINI_TINY_CTAS")) kMiniTinyCtas = atoll(e);
  if (const char *e = getenv("H3D_MINI_TINY_KIN")) kMiniTinyKin = atoll(e);
  if (const char *e = getenv("H3D_MINI_HUGE_CTAS")) kMiniHugeCtas = atoll(e);
  if (const char *e = getenv("H3D_MINI_HUGE_KIN")) kMiniHugeKin = atoll(e);
  if (const char *e = getenv("H3D_MINI_SEG")) g_mini_seglen = atoi(e) < 1 ? 1 : atoi(e);
  if (const char *e = getenv("H3D_MINI_SPEC")) g_mini_spec = atoi(e) ? 1 : 0;
  if (const char *e = getenv("H3D_TRACE")) g_trace = atoi(e);
  if (const char *e = getenv("H3D_LANE")) g_lane = atoi(e);
  if (const char *e = getenv("H3D_LANE_MAX_LEVEL")) g_lane_max_level = atoi(e);
  if (const char *e = getenv("H3D_LANE_XYZ_KB")) g_lane_xyz_max = atoll(e) * 1024;
  if (const char *e = getenv("H3D_LANE_STAGE")) g_lane_stage = atoi(e);
  if (const char *e = getenv("H3D_LANE_OWN")) g_lane_own = atoi(e);
  if (const char *e = getenv("H3D_TPJ_PREFETCH")) kTpjPrefetchJobs = atoll(e);
  if (const char *e = getenv("H3D_PLAN")) g_plan = atoi(e) ? 1 : 0;
  if (const char *e = getenv("H3D_INTERLEAVE")) g_interleave = atoi(e) ? 1 : 0;
  if (const char *e = getenv("H3D_TPJ_CAP_LEVEL")) g_tpj_cap_level = atoi(e);
  if (const char *e = getenv("H3D_TPJ_SPLIT")) g_tpj_split = atoi(e);
  if (const char *e = getenv("H3D_LANE_PF1")) g_lane_pf1 = atoi(e);
  if (const char *e = getenv("H3D_LANE_PF2")) g_lane_pf2 = atoi(e);
  g_leaf_b = leaf_depth(g_leaf_b);
}

template <bool XYZ>
long long launch_tpj(dim3 grid, int pool, int jpc, int prefetch, cudaStream_t s, Pass2 P,
                const double *pts,
                long long n, int lv, long long j0, long long j1, long long *err,
                long long *spec = nullptr, long long *stamp = nullptr, const TpjSplit *sp = nullptr) {
  // a split level: the CTAs that do not fit the small pool go to the list,
  // then to the big-pool launch
  int *ovf = sp ? sp->ovf : nullptr;
  // the mini's list launch has a fixed grid: more large CTAs than it covers
  // fail the level (a replayed plan: measured again)
  const long long cap = sp ? (sp->mini >= 0 && sp->grid < sp->cap ? sp->grid : sp->cap) : 0;
  if (ovf) cudaMemsetAsync(ovf, 0, sizeof(int), s);
  if (lv <= g_tpj_cap_level)
    k_fast_tpj_r128<XYZ><<<grid, 32, pool, s>>>(P, pts, n, lv, j0, j1, err, pool, jpc, prefetch, spec, stamp, ovf,
                                                cap);
  else
    k_fast_tpj<XYZ><<<grid, 32, pool, s>>>(P, pts, n, lv, j0, j1, err, pool, jpc, prefetch, spec, stamp, ovf, cap);
  if (ovf && sp->mini >= 0) {  // hybrid: the large CTAs' jobs one CTA each on a mini variant
    h3d_count_launches(1);
    const long long rm = mini_level(P, pts, n, lv, j0, j1, err, s, sp->mini, spec, nullptr, sp->scratch,
                                    sp->scratch_bytes, ovf, sp->grid);
    if (rm < 0) return rm;
  } else if (ovf) {
    h3d_count_launches(1);
    k_fast_tpj_ovf<<<sp->grid, 32, sp->pool, s>>>(P, pts, n, lv, j0, j1, err, sp->pool, jpc, prefetch, spec,
                                                  ovf);
  }
  return 0;
}

// The hybrid route for a level the time-split pipeline would take because
// of a few large jobs (C5's shell runs): lane per job on a small pool for
// all CTAs but at most an eighth, the large CTAs' jobs one CTA each on the
// smallest mini variant that fits the level's largest job.
// The huge variant (global-memory slots, one per list CTA) when the level's
// largest job needs it and the slots of the large CTAs fit the scratch.
bool tpj_hybrid(const unsigned long long *need, long long maxkin, size_t gbytes, TpjSplit *sp) {
  if (!g_tpj_split) return false;
  const long long np = static_cast<long long>(need[6]);
  int var = -1;
  if (np <= kMiniSmallPoints && maxkin <= kMiniSmallEvents) var = 0;
  else if (np <= kMiniMedPoints && maxkin <= kMiniMedEvents) var = 4;
  else if (np <= kMiniL2Points && maxkin <= kMiniL2Events) var = 5;
  else if (np <= kMiniMaxPoints && maxkin <= kMiniMaxEvents) var = 1;
  else if (np <= kMiniXlPoints && maxkin <= kMiniXlEvents) var = 6;
  else if (np <= kMiniHugePoints && maxkin <= kMiniHugeEvents) var = 3;
  if (var < 0) return false;
  long long C = 0;
  for (int b = 0; b < kNeedHistBins; ++b) C += static_cast<long long>(need[kNeedHist + b]);
  long long cap = C / 8;
  if (var == 3) {
    const long long slots = static_cast<long long>(gbytes / mini_huge_stride()) / 32;
    if (slots < 1) return false;  // not even one list entry's slots
    if (slots < cap) cap = slots;
  }
  long long above = C;
  for (int b = 0; b < kNeedHistBins; ++b) {
    above -= static_cast<long long>(need[kNeedHist + b]);
    if (above > cap) continue;
    long long small = 12 * need_bin_max(b) + 32 * 16;
    if (small < 1024) small = 1024;
    if (small > kTpjPool) return false;
    sp->small = small;
    sp->pool = 0;
    sp->grid = static_cast<int>(above < 1 ? 1 : above);
    sp->mini = var;
    return true;
  }
  return false;
}

// Split a lane-per-job level whose largest CTA needs far more shared memory
// than most (x-extreme runs of hull points, C5's shell): the small pool
// covers all CTAs but at most an eighth, and at most about one wave of the
// big-pool launch, and only when it fits more CTAs per SM.
// need[kNeedHist ..]: the per-CTA histogram of point sums.  tpj_split = 2
// (tests): split at the median, whatever the occupancy.
bool tpj_split(const unsigned long long *need, long long pool, int lv, TpjSplit *sp) {
  if (!g_tpj_split) return false;
  const int regcap = lv <= g_tpj_cap_level ? 16 : 12;
  auto occ = [&](long long P) {
    const long long by_smem = 233472 / (P + 1024);
    return by_smem < regcap ? by_smem : static_cast<long long>(regcap);
  };
  long long C = 0;
  for (int b = 0; b < kNeedHistBins; ++b) C += static_cast<long long>(need[kNeedHist + b]);
  const bool force = g_tpj_split == 2;
  long long allowed = 148 * occ(pool);
  if (allowed > C / 8) allowed = C / 8;
  if (force) allowed = C / 2;
  long long above = C;
  for (int b = 0; b < kNeedHistBins; ++b) {
    above -= static_cast<long long>(need[kNeedHist + b]);
    if (above > allowed) continue;
    long long small = 12 * need_bin_max(b) + 32 * 16;
    if (small < 1024) small = 1024;
    if (small >= pool || (!force && occ(small) <= occ(pool))) return false;
    sp->small = small;
    sp->pool = static_cast<int>(pool);
    sp->grid = static_cast<int>(above < 1 ? 1 : above);
    return true;
  }
  return false;
}

}  // namespace

extern "C" {

int64_t h3d_tune(const char *name, int64_t value) {
  load_env_once();
  const std::string k(name ? name : "");
  long long old = -1;
  if (value >= 0) plans_clear();  // recorded plans follow the knobs they were made with
  if (k == "plan") { old = g_plan; if (value >= 0) g_plan = value ? 1 : 0; }
  if (k == "interleave") { old = g_interleave; if (value >= 0) g_interleave = value ? 1 : 0; }
  else if (k == "tpj_cap_level") { old = g_tpj_cap_level; if (value >= 0) g_tpj_cap_level = value; }
  else if (k == "tpj_xyz_ctas") { old = kTpjXyzCtas; if (value >= 0) kTpjXyzCtas = value; }
  else if (k == "tpj_split") { old = g_tpj_split; if (value >= 0) g_tpj_split = static_cast<int>(value); }
  if (k == "big_kin") { old = kBigKin; if (value >= 0) kBigKin = value; }
  else if (k == "leaf_b") { old = g_leaf_b; if (value >= 0) g_leaf_b = leaf_depth(value); }
  else if (k == "mini") { old = g_mini; if (value >= 0) g_mini = value ? 1 : 0; }
  else if (k == "mini_ctas") { old = kMiniMaxCtas; if (value >= 0) kMiniMaxCtas = value; }
  else if (k == "mini_tiny_ctas") { old = kMiniTinyCtas; if (value >= 0) kMiniTinyCtas = value; }
  else if (k == "mini_tiny_kin") { old = kMiniTinyKin; if (value >= 0) kMiniTinyKin = value; }
  else if (k == "mini_one_wave") { old = kMiniOneWave; if (value >= 0) kMiniOneWave = value; }
  else if (k == "mini_huge_ctas") { old = kMiniHugeCtas; if (value >= 0) kMiniHugeCtas = value; }
  else if (k == "mini_huge_kin") { old = kMiniHugeKin; if (value >= 0) kMiniHugeKin = value; }
  else if (k == "mini_seg") { old = g_mini_seglen; if (value >= 1) g_mini_seglen = static_cast<int>(value); }
  else if (k == "mini_spec") { old = g_mini_spec; if (value >= 0) g_mini_spec = value ? 1 : 0; }
  else if (k == "big_total") { old = kBigTotal; if (value >= 0) kBigTotal = value; }
  else if (k == "big_max_jobs") { old = kBigMaxJobs; if (value >= 0) kBigMaxJobs = value; }
  else if (k == "tpj_min_jobs") { old = kTpjMinTotalJobs; if (value >= 0) kTpjMinTotalJobs = value; }
  else if (k == "tpj_xyz_kb") { old = kTpjXyzMax / 1024; if (value >= 0) kTpjXyzMax = value * 1024; }
  else if (k == "lane") { old = g_lane; if (value >= 0) g_lane = value ? 1 : 0; }
  else if (k == "lane_max_level") { old = g_lane_max_level; if (value >= 0) g_lane_max_level = static_cast<int>(value); }
  else if (k == "lane_xyz_kb") { old = g_lane_xyz_max / 1024; if (value >= 0) g_lane_xyz_max = value * 1024; }
  else if (k == "lane_stage") { old = g_lane_stage; if (value >= 0) g_lane_stage = value ? 1 : 0; }
  else if (k == "lane_own") { old = g_lane_own; if (value >= 0) g_lane_own = static_cast<int>(value); }
  else if (k == "lane_pf1") { old = g_lane_pf1; if (value >= 0) g_lane_pf1 = static_cast<int>(value); }
  else if (k == "lane_pf2") { old = g_lane_pf2; if (value >= 0) g_lane_pf2 = static_cast<int>(value); }
  else if (k == "tpj_max_level") { old = kTpjMaxLevel; if (value >= 0) kTpjMaxLevel = static_cast<int>(value); }
  return old;
}

int64_t h3d_fast_layout(int64_t n, int64_t *offsets) {
  // byte offsets of A.hdr, A.lnk, A.gid, A.ev, B.hdr, B.lnk, B.gid, B.ev, seq
  char *base = reinterpret_cast<char *>(size_t(1) << 40);
  h3d_arena ar(base, ~size_t(0) >> 4);
  PassWS w;
  if (!carve_pass(ar, n, w)) return H3D_E_ARG;
  const void *p[9] = {w.A.hdr, w.A.lnk, w.A.gid, w.A.ev, w.B.hdr, w.B.lnk, w.B.gid, w.B.ev, w.seq};
  for (int i = 0; i < 9; ++i) offsets[i] = static_cast<const char *>(p[i]) - base;
  return 0;
}

static size_t base_pass_bytes(long long n) {
  h3d_arena ar(nullptr, 0);
  PassWS w;
  carve_pass(ar, n, w);
  return (ar.used + 4095) & ~size_t(4095);
}

size_t h3d_fast_pass_workspace_bytes(int64_t n) {  // per pass (+ the big-job scratch)
  if (n < 1) n = 1;
  return base_pass_bytes(n) + big_workspace_bytes(big_capacity(n)) + 4096;
}

size_t h3d_fast_upper_workspace_bytes(int64_t n) {  // the upper pass: no big-job scratch
  if (n < 1) n = 1;
  return base_pass_bytes(n) + 4096;
}

int64_t h3d_fast_passes_range(const double *sorted_pts, int64_t n, int64_t p0, int64_t p1,
                              int32_t lv_lo, int32_t lv_hi, void *ws_lower, void *ws_upper,
                              size_t workspace_bytes, int64_t *err_dev, int32_t verify,
                              void *stream) {
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (n < 2 || n > (1ll << 30) || p0 < 0 || p1 > n || p0 >= p1 || lv_lo < 1) return H3D_E_ARG;
  h3d_arena a0(ws_lower, workspace_bytes), a1(ws_upper, workspace_bytes);
  PassWS w0, w1;
  if (!carve_pass(a0, n, w0) || !carve_pass(a1, n, w1)) return H3D_E_ARG;
  // the big-job scratch lives after the lower pass's arrays
  const size_t bb = base_pass_bytes(n);
  void *big_ws = workspace_bytes > bb ? static_cast<char *>(ws_lower) + bb : nullptr;
  const size_t big_bytes = workspace_bytes > bb ? workspace_bytes - bb : 0;
  int dev_id = 0;
  cudaGetDevice(&dev_id);
  if (dev_id < 0 || dev_id >= 64) return H3D_E_ARG;
  if (!g_attr_done[dev_id]) {
    if (h3d_check(cudaFuncSetAttribute(k_fast_warp<1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(kWarpPoolMax))) ||
        h3d_check(cudaFuncSetAttribute(k_fast_tpj<true>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, kTpjPool)) ||
        h3d_check(cudaFuncSetAttribute(k_fast_tpj<false>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, kTpjPool)) ||
        h3d_check(cudaFuncSetAttribute(k_fast_tpj_ovf, cudaFuncAttributeMaxDynamicSharedMemorySize, kTpjPool)) ||
        h3d_check(cudaFuncSetAttribute(k_fast_tpj_r128<true>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, kTpjPool)) ||
        h3d_check(cudaFuncSetAttribute(k_fast_tpj_r128<false>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, kTpjPool)))
      return H3D_E_CUDA;
    load_env_once();
    if (h3d_check(cudaFuncSetAttribute(k_fast_leaf<3>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       32 * leaf_lane_bytes<3>())) ||
        h3d_check(cudaFuncSetAttribute(k_fast_leaf<4>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       32 * leaf_lane_bytes<4>())))
      return H3D_E_CUDA;
    g_attr_done[dev_id] = true;
  }
  long long *err = reinterpret_cast<long long *>(err_dev);
  // verify mode: check the groups level l wrote (they are Q.in0/Q.in1)
  auto check = [&](const Pass2 &Q, int l, const long long *spec = nullptr) {
    if (!verify) return;
    const long long a = p0 >> l, b = (p1 + (1ll << l) - 1) >> l;
    h3d_count_launches(1);
    const unsigned gv = h3d_grid(b - a, 8) > 4096 ? 4096 : h3d_grid(b - a, 8);
    // verify >= 2: err_dev has 4 words, the first violation goes to err_dev[3]
    k_verify_level<<<dim3(gv, 2), 256, 0, s>>>(Q, sorted_pts, n, l, a, b, err, verify >= 2 ? err + 3 : nullptr,
                                               spec);
  };
  int levels = 0;
  while ((1ll << levels) < n) ++levels;
  if (lv_hi > levels) lv_hi = levels;
  // level l reads buffer (l-1)&1 and writes buffer l&1 (A = 0, B = 1)
  Pass2 P = (lv_lo & 1) ? Pass2{w0.A, w1.A, w0.B, w1.B} : Pass2{w0.B, w1.B, w0.A, w1.A};
  int lv = lv_lo;
  const int NPB = 1 << g_leaf_b;
  if (lv_lo == 1 && g_leaf_b >= 3 && lv_hi >= g_leaf_b && (p0 & (NPB - 1)) == 0) {
    // levels 1..B fused in shared memory, one lane per 2^B-point block
    const long long blocks = (p1 - p0 + NPB - 1) / NPB;
    h3d_stamp_now(s, 1);
    h3d_stamp_route(1, 3000 + g_leaf_b);
    void *e0 = h3d_profiling() ? h3d_prof_begin(s) : nullptr;
    h3d_count_launches(1);
    const dim3 grid = lvl_grid(h3d_grid(blocks, 32), g_interleave != 0);
    // level B's groups go to buffer B&1
    const Pass2 LP = (g_leaf_b & 1) ? Pass2{w0.A, w1.A, w0.B, w1.B} : Pass2{w0.B, w1.B, w0.A, w1.A};
    if (g_leaf_b == 4)
      k_fast_leaf<4><<<grid, 32, 32 * leaf_lane_bytes<4>(), s>>>(LP, sorted_pts, n, p0, p1, err);
    else
      k_fast_leaf<3><<<grid, 32, 32 * leaf_lane_bytes<3>(), s>>>(LP, sorted_pts, n, p0, p1, err);
    h3d_prof_end(e0, 3000 + g_leaf_b, 2, s);
    // the leaf writes level B's groups into buffer B&1
    P = (g_leaf_b & 1) ? Pass2{w0.B, w1.B, w0.A, w1.A} : Pass2{w0.A, w1.A, w0.B, w1.B};
    lv = g_leaf_b + 1;
  } else if (lv_lo == 1) {  // level 1 written directly (no coordinates needed)
    const long long j0 = p0 >> 1, j1 = (p1 + 1) >> 1;
    h3d_stamp_now(s, 1);
    h3d_stamp_route(1, 2001);
    void *e0 = h3d_profiling() ? h3d_prof_begin(s) : nullptr;
    h3d_count_launches(1);
    const unsigned gi = h3d_grid(j1 - j0, 256) > 8192 ? 8192 : h3d_grid(j1 - j0, 256);
    k_fast_init1<<<dim3(gi, 2), 256, 0, s>>>(n, j0, j1, P);
    h3d_prof_end(e0, 1 + 2000, 2, s);
    P = Pass2{P.out0, P.out1, P.in0, P.in1};
    lv = 2;
  }
  // ---- replay the level plan the last call with this point range recorded
  std::vector<LevelRec> rec;  // this call's launches: the next call's plan
  const PlanKey key{dev_id, n, p0, p1, lv_lo, lv_hi};
  if (g_plan && lv <= lv_hi) {
    std::vector<LevelRec> plan;
    {
      std::lock_guard<std::mutex> g(g_plan_mu);
      auto it = g_plans.find(key);
      if (it != g_plans.end()) plan = it->second;
    }
    if (!plan.empty() && plan.front().lv == lv) {
      long long *spec = reinterpret_cast<long long *>(w0.need + 12);
      cudaMemsetAsync(spec, 0, sizeof(long long), s);
      const int lv_start = lv;
      for (const LevelRec &r : plan) {
        if (r.lv != lv || lv > lv_hi) break;
        if (lv > lv_lo) check(P, lv - 1, spec);
        const long long j0 = p0 >> lv, j1 = (p1 + (1ll << lv) - 1) >> lv;
        // the level's first kernel writes its start stamp (no extra launch)
        long long *stp = h3d_stamp_buf() ? h3d_stamp_buf() + lv : nullptr;
        if (r.kind == REC_WARP) h3d_stamp_now(s, lv);
        void *e0 = h3d_profiling() ? h3d_prof_begin(s) : nullptr;
        int tag = lv;
        long long rc = 0;
        if (r.kind == REC_BIG) {
          // the pipeline with the recorded totals (checked on the device);
          // a level that no longer fits the scratch resumes measured
          tag = lv + 4000;
          if (stp) h3d_stamp_now(s, lv);
          rc = big_level(P, big_ws, big_bytes, sorted_pts, n, lv, j0, j1, err, s, r.big_kin, r.big_pts, spec);
          if (rc == 1) {
            h3d_prof_drop(e0);
            break;
          }
        } else if (r.kind == REC_MINI) {
          tag = lv + 5000;
          rc = mini_level(P, sorted_pts, n, lv, j0, j1, err, s, r.variant, spec, stp, big_ws, big_bytes);
        } else if (r.kind == REC_LANE) {
          tag = lv + 1000;
          void *ek = h3d_prof_kernels() ? h3d_prof_begin(s) : nullptr;
          LaneCfg c = r.lane;
          rc = lane_level(P, sorted_pts, n, lv, j0, j1, err, nullptr, s, &c, spec, stp);
          h3d_prof_end(ek, tag, 2, s);
        } else if (r.kind == REC_TPJ) {
          tag = lv + 1000;
          void *ek = h3d_prof_kernels() ? h3d_prof_begin(s) : nullptr;
          h3d_count_launches(1);
          const dim3 grid = lvl_grid(h3d_grid(j1 - j0, r.jpc), g_interleave != 0);
          if (r.variant) {
            launch_tpj<true>(grid, static_cast<int>(r.pool), r.jpc, 0, s, P, sorted_pts, n, lv, j0, j1, err,
                             spec, stp);
          } else {
            TpjSplit sp{w0.ovf, w0.ovf_cap, static_cast<int>(r.pool2), r.ogrid, 0, r.mini, big_ws, big_bytes};
            rc = launch_tpj<false>(grid, static_cast<int>(r.pool), r.jpc, r.prefetch, s, P, sorted_pts, n, lv,
                                   j0, j1, err, spec, stp, (r.pool2 || r.mini >= 0) ? &sp : nullptr);
          }
          h3d_prof_end(ek, tag, 2, s);
        } else {  // REC_WARP: an oversized job runs in HBM mode, always fits
          h3d_count_launches(1);
          k_fast_warp<1><<<dim3(h3d_grid(j1 - j0, 1), 2), 32, r.pool, s>>>(
              P, sorted_pts, n, lv, j0, j1, err, static_cast<int>(r.pool), w0.seq, w1.seq, w0.rec, w1.rec);
        }
        if (rc < 0) return rc;
        h3d_prof_end(e0, tag, 2, s);
        h3d_stamp_route(lv, tag);
        rec.push_back(r);
        P = Pass2{P.out0, P.out1, P.in0, P.in1};
        ++lv;
      }
      // the replay's one read-back: the first level that did not fit, the error word
      long long hv[2] = {0, 0};
      if (h3d_check(cudaMemcpyAsync(&hv[0], spec, sizeof(long long), cudaMemcpyDeviceToHost, s)) ||
          h3d_check(cudaMemcpyAsync(&hv[1], err, sizeof(long long), cudaMemcpyDeviceToHost, s)) ||
          h3d_check(h3d_sync(s)))
        return H3D_E_CUDA;
      if (hv[1] != 0) {
        lv = lv_hi + 2;  // declined: the caller sees the error word
      } else if (hv[0] != 0) {
        // redo from the level that did not fit: it reads buffer (f-1)&1, intact
        const int f = static_cast<int>(hv[0]);
        rec.resize(f - lv_start);
        lv = f;
        P = (f & 1) ? Pass2{w0.A, w1.A, w0.B, w1.B} : Pass2{w0.B, w1.B, w0.A, w1.A};
        if (g_trace) fprintf(stderr, "h3d plan replay: level %d did not fit, measured from there\n", f);
      }
    }
  }
  for (; lv <= lv_hi; ++lv) {
    if (lv > lv_lo) check(P, lv - 1);  // the previous level's groups
    // the jobs of this level inside the point range [p0, p1)
    const long long j0 = p0 >> lv;
    const long long j1 = (p1 + (1ll << lv) - 1) >> lv;
    const long long jobs = j1 - j0;
    void *e0 = h3d_profiling() ? h3d_prof_begin(s) : nullptr;
    // Level routing from the measured group sizes (one small read-back):
    // one lane per job while the level has enough jobs to fill the GPU and
    // they fit a shared-memory slice (int16 local ids); one warp per job
    // (1-warp CTAs, pool = the largest job's need, HBM mode above it) for
    // the few-job levels.
    cudaMemsetAsync(w0.need, 0, (kNeedHist + kNeedHistBins) * sizeof(unsigned long long), s);
    const long long chunks = (jobs + 31) / 32;
    h3d_count_launches(1);
    k_tpj_need<<<dim3(h3d_grid(chunks, 8) > 2 * 148 ? 2 * 148 : h3d_grid(chunks, 8), 2), 256, 0, s>>>(
        P, n, lv, j0, j1, w0.need, err, h3d_stamp_buf() ? h3d_stamp_buf() + lv : nullptr);
    unsigned long long need[kNeedHist + kNeedHistBins];
    if (h3d_check(cudaMemcpyAsync(need, w0.need, sizeof(need), cudaMemcpyDeviceToHost, s)) ||
        h3d_check(h3d_sync(s)))
      return H3D_E_CUDA;
    const long long herr = static_cast<long long>(need[10]);
    // A launch declined the input (or failed): its level wrote nothing, so
    // the groups this level would read are stale -- stop routing; the caller
    // sees the error word and hands the hull to the exact engine.
    if (herr != 0) {
      if (g_trace) fprintf(stderr, "h3d level %d: error %lld set, levels stop\n", lv, herr);
      break;
    }
    const long long maxkin = static_cast<long long>(need[8]), sumkin = static_cast<long long>(need[9]);
    if (g_trace)
      fprintf(stderr, "h3d level %d: jobs %lld max nS %llu max kin %lld sum kin %lld\n", lv, jobs,
              need[6], maxkin, sumkin);
    // few small jobs: the in-shared-memory time-split merge (mini.cu)
    // (154 KB of shared memory per CTA: one CTA per SM, so only for levels of
    // at most a few CTAs per SM)
    const bool mini_small = static_cast<long long>(need[6]) <= kMiniSmallPoints &&
                            maxkin <= kMiniSmallEvents;
    const bool mini_tiny = static_cast<long long>(need[6]) <= kMiniTinyPoints &&
                           maxkin <= kMiniTinyEvents && 2 * jobs <= kMiniTinyCtas &&
                           (2 * jobs < kTpjMinTotalJobs || maxkin >= kMiniTinyKin);
    if (g_mini && mini_tiny) {
      const long long rm = mini_level(P, sorted_pts, n, lv, j0, j1, err, s, 2);
      if (rm < 0) return rm;
      rec.push_back(LevelRec{lv, REC_MINI, 2, 0, 0, 0, LaneCfg{}});
      h3d_prof_end(e0, lv + 5000, 2, s);
      h3d_stamp_route(lv, lv + 5000);
      P = Pass2{P.out0, P.out1, P.in0, P.in1};
      continue;
    }
    if (g_mini && 2 * jobs < kTpjMinTotalJobs &&
        ((mini_small && 2 * jobs <= 4 * kMiniMaxCtas) ||
         (2 * jobs <= kMiniMaxCtas && static_cast<long long>(need[6]) <= kMiniXlPoints &&
          maxkin <= kMiniXlEvents))) {
      // up to two CTAs per SM the large variant (one wave); more jobs take
      // the smallest variant the level's largest job fits (more CTAs per SM)
      const long long np = static_cast<long long>(need[6]);
      const bool one_wave = 2 * jobs <= kMiniOneWave;
      int var = mini_small ? 0
                      : one_wave ? 1
                      : (np <= kMiniMedPoints && maxkin <= kMiniMedEvents)
                          ? 4
                          : (np <= kMiniL2Points && maxkin <= kMiniL2Events) ? 5 : 1;
      if (var == 1 && (np > kMiniMaxPoints || maxkin > kMiniMaxEvents)) var = 6;
      const long long rm = mini_level(P, sorted_pts, n, lv, j0, j1, err, s, var);
      if (rm < 0) return rm;
      rec.push_back(LevelRec{lv, REC_MINI, var, 0, 0, 0, LaneCfg{}});
      h3d_prof_end(e0, lv + 5000, 2, s);
      h3d_stamp_route(lv, lv + 5000);
      P = Pass2{P.out0, P.out1, P.in0, P.in1};
      if (g_mini_spec && var == 1 && one_wave && lv < lv_hi) {
        // the remaining levels have at most half these jobs: launch them all
        // on the large variant unmeasured; a job that does not fit records
        // its level in `spec` (later launches then write nothing) and the
        // loop resumes, measured, from that level
        long long *spec = reinterpret_cast<long long *>(w0.need + 12);
        cudaMemsetAsync(spec, 0, sizeof(long long), s);
        for (int l2 = lv + 1; l2 <= lv_hi; ++l2) {
          void *e2 = h3d_profiling() ? h3d_prof_begin(s) : nullptr;
          const long long rs = mini_level(P, sorted_pts, n, l2, p0 >> l2,
                                          (p1 + (1ll << l2) - 1) >> l2, err, s, 1, spec,
                                          h3d_stamp_buf() ? h3d_stamp_buf() + l2 : nullptr);
          if (rs < 0) return rs;
          rec.push_back(LevelRec{l2, REC_MINI, 1, 0, 0, 0, LaneCfg{}});
          if (g_trace) {
            long long f = 0;
            cudaMemcpyAsync(&f, spec, sizeof(f), cudaMemcpyDeviceToHost, s);
            const cudaError_t ce = h3d_sync(s);
            fprintf(stderr, "h3d level %d speculative: flag %lld (%s)\n", l2, f,
                    cudaGetErrorString(ce));
          }
          h3d_prof_end(e2, l2 + 5000, 2, s);
          h3d_stamp_route(l2, l2 + 5000);
          P = Pass2{P.out0, P.out1, P.in0, P.in1};
          check(P, l2, spec);
        }
        long long failed = 0, serr = 0;
        if (h3d_check(cudaMemcpyAsync(&failed, spec, sizeof(failed), cudaMemcpyDeviceToHost, s)) ||
            h3d_check(cudaMemcpyAsync(&serr, err, sizeof(serr), cudaMemcpyDeviceToHost, s)) ||
            h3d_check(h3d_sync(s)))
          return H3D_E_CUDA;
        if (serr != 0) {
          lv = lv_hi + 2;  // declined: nothing more to check or record
          break;
        }
        if (g_trace)
          fprintf(stderr, "h3d levels %d..%d speculative on the large mini: failed at %lld\n",
                  lv + 1, lv_hi, failed);
        if (failed == 0) {
          lv = lv_hi + 3;  // every level done (each chain level checked above)
          break;
        }
        // redo from the failed level: it reads buffer (f-1)&1, intact
        const int f = static_cast<int>(failed);
        P = (f & 1) ? Pass2{w0.A, w1.A, w0.B, w1.B} : Pass2{w0.B, w1.B, w0.A, w1.A};
        while (!rec.empty() && rec.back().lv >= f) rec.pop_back();
        lv = f - 1;
      }
      continue;
    }
    // few large jobs (the top levels of ball clouds, the mid levels of
    // spheres): one CTA per job with its arrays in global memory (L1/L2)
    if (g_mini && big_ws && 2 * jobs <= kMiniHugeCtas &&
        static_cast<long long>(need[6]) <= kMiniHugePoints && maxkin <= kMiniHugeEvents &&
        maxkin >= kMiniHugeKin) {
      const long long rm = mini_level(P, sorted_pts, n, lv, j0, j1, err, s, 3, nullptr, nullptr,
                                      big_ws, big_bytes);
      if (rm < 0) return rm;
      if (rm == 0) {
        rec.push_back(LevelRec{lv, REC_MINI, 3, 0, 0, 0, LaneCfg{}});
        h3d_prof_end(e0, lv + 5000, 2, s);
        h3d_stamp_route(lv, lv + 5000);
        P = Pass2{P.out0, P.out1, P.in0, P.in1};
        continue;
      }
    }
    // a few large jobs among many small ones: lane per job + mini (hybrid)
    {
      TpjSplit sp{w0.ovf, w0.ovf_cap, 0, 0, 0, -1, big_ws, big_bytes};
      const bool big_wants = big_ws && (maxkin >= kBigKin || (2 * maxkin >= kBigKin && sumkin >= kBigTotal &&
                                                              2 * jobs < kBigMaxJobs));
      if (big_wants && lv <= kTpjMaxLevel && 2 * jobs >= kTpjMinTotalJobs && tpj_hybrid(need, maxkin, big_bytes, &sp)) {
        if (g_trace)
          fprintf(stderr, "h3d level %d: hybrid pool %lld, <= %d large CTAs on mini variant %d\n", lv, sp.small,
                  sp.grid, sp.mini);
        h3d_count_launches(1);
        void *ek = h3d_prof_kernels() ? h3d_prof_begin(s) : nullptr;
        const dim3 grid = lvl_grid(h3d_grid(jobs, 32), g_interleave != 0);
        const int pf = jobs >= kTpjPrefetchJobs ? 1 : 0;
        const long long rt = launch_tpj<false>(grid, static_cast<int>(sp.small), 32, pf, s, P, sorted_pts, n, lv,
                                               j0, j1, err, nullptr, nullptr, &sp);
        if (rt < 0) return rt;
        LevelRec lr{lv, REC_TPJ, 0, 32, pf, sp.small, LaneCfg{}};
        lr.ogrid = sp.grid;
        lr.mini = sp.mini;
        rec.push_back(lr);
        h3d_prof_end(ek, lv + 1000, 2, s);
        h3d_prof_end(e0, lv + 1000, 2, s);
        h3d_stamp_route(lv, lv + 1000);
        P = Pass2{P.out0, P.out1, P.in0, P.in1};
        continue;
      }
    }
    // large merge jobs: the time-split pipeline (big.cu)
    // (its fixed cost, ~25 launches, only pays when the level has work)
    // (many moderate jobs keep the lane kernel busy: the second clause only
    // for levels of fewer jobs)
    if (big_ws && (maxkin >= kBigKin ||
                   (2 * maxkin >= kBigKin && sumkin >= kBigTotal && 2 * jobs < kBigMaxJobs))) {
      const long long rb = big_level(P, big_ws, big_bytes, sorted_pts, n, lv, j0, j1, err, s, sumkin,
                                     static_cast<long long>(need[11]));
      if (rb < 0) return rb;
      if (rb == 0) {
        LevelRec lr{lv, REC_BIG, 0, 0, 0, 0, LaneCfg{}};
        lr.big_kin = sumkin;
        lr.big_pts = static_cast<long long>(need[11]);
        rec.push_back(lr);
        h3d_prof_end(e0, lv + 4000, 2, s);
      h3d_stamp_route(lv, lv + 4000);
        P = Pass2{P.out0, P.out1, P.in0, P.in1};
        continue;
      }
    }
    bool tpj = lv <= kTpjMaxLevel && 2 * jobs >= kTpjMinTotalJobs && need[6] < 0x7fff;
    int jpc = 32;
    bool xyz = false;
    long long pool = 0;
    if (tpj) {
      int r = 0;
      while (r < 5 && 12ll * need[r] + 32 * 16 > kTpjPool) ++r;
      if (12ll * need[r] + 32 * 16 > kTpjPool) {
        tpj = false;
      } else {
        jpc = 32 >> r;
        // stage coordinates when the pool stays small, or when there are
        // too few CTAs for shared memory to limit occupancy
        const long long ctas = 2 * ((jobs + jpc - 1) / jpc);
        xyz = 36ll * need[r] + 32 * 16 <= kTpjXyzMax ||
              (ctas <= kTpjXyzCtas && 36ll * need[r] + 32 * 16 <= kTpjPool);
        pool = (xyz ? 36ll : 12ll) * need[r] + 32 * 16;
        if (pool < 1024) pool = 1024;
      }
    }
    if (tpj && g_lane && lv <= g_lane_max_level) {
      void *ek = h3d_prof_kernels() ? h3d_prof_begin(s) : nullptr;
      LaneCfg lc{};
      const long long rl = lane_level(P, sorted_pts, n, lv, j0, j1, err, need, s, &lc);
      if (rl < 0) return rl;
      if (rl == 0) rec.push_back(LevelRec{lv, REC_LANE, 0, 0, 0, 0, lc});
      if (rl == 0) h3d_prof_end(ek, lv + 1000, 2, s); else h3d_prof_drop(ek);
      if (rl == 0) {
        h3d_prof_end(e0, lv + 1000, 2, s);
      h3d_stamp_route(lv, lv + 1000);
        P = Pass2{P.out0, P.out1, P.in0, P.in1};
        continue;
      }
      tpj = false;
    }
    if (tpj) {
      TpjSplit sp{w0.ovf, w0.ovf_cap, 0, 0, 0};
      const bool split = !xyz && jpc == 32 && tpj_split(need, pool, lv, &sp);
      if (g_trace)
        fprintf(stderr, "h3d level %d: tpj xyz %d jpc %d pool %lld split %lld / %d (%d CTAs)\n", lv, xyz ? 1 : 0,
                jpc, pool, split ? sp.small : 0, split ? sp.pool : 0, split ? sp.grid : 0);
      h3d_count_launches(1);
      void *ek = h3d_prof_kernels() ? h3d_prof_begin(s) : nullptr;
      const dim3 grid = lvl_grid(h3d_grid(jobs, jpc), g_interleave != 0);
      if (xyz)
        launch_tpj<true>(grid, static_cast<int>(pool), jpc, 0, s, P, sorted_pts, n, lv, j0, j1, err);
      else
        launch_tpj<false>(grid, static_cast<int>(split ? sp.small : pool), jpc, jobs >= kTpjPrefetchJobs ? 1 : 0,
                          s, P, sorted_pts, n, lv, j0, j1, err, nullptr, nullptr, split ? &sp : nullptr);
      LevelRec lr{lv, REC_TPJ, xyz ? 1 : 0, jpc, jobs >= kTpjPrefetchJobs ? 1 : 0, split ? sp.small : pool,
                  LaneCfg{}};
      if (split) {
        lr.pool2 = sp.pool;
        lr.ogrid = sp.grid;
      }
      rec.push_back(lr);
      h3d_prof_end(ek, lv + 1000, 2, s);
      h3d_prof_end(e0, lv + 1000, 2, s);
      h3d_stamp_route(lv, lv + 1000);
    } else {
      long long wpool = static_cast<long long>(need[7]);
      if (wpool > kWarpPoolMax) wpool = kWarpPoolMax;
      if (wpool < 1024) wpool = 1024;
      h3d_count_launches(1);
      k_fast_warp<1><<<dim3(h3d_grid(jobs, 1), 2), 32, wpool, s>>>(
          P, sorted_pts, n, lv, j0, j1, err, static_cast<int>(wpool), w0.seq, w1.seq, w0.rec,
          w1.rec);
      rec.push_back(LevelRec{lv, REC_WARP, 0, 0, 0, wpool, LaneCfg{}});
      h3d_prof_end(e0, lv, 2, s);
      h3d_stamp_route(lv, lv);
    }
    P = Pass2{P.out0, P.out1, P.in0, P.in1};
  }
  // lv: lv_hi + 1 = the loop ran every level, lv_hi + 3 = the speculative
  // chain did, lv_hi + 2 = declined, <= lv_hi = a level read an error word
  if (lv == lv_hi + 1 && lv - 1 >= lv_lo) check(P, lv - 1);  // the last level
  h3d_stamp_now(s, H3D_STAMP_END);
  // the next call with this point range replays what this one launched
  // (only a complete record: a declined or failed run records nothing)
  if (g_plan && (lv == lv_hi + 1 || lv == lv_hi + 3) && !rec.empty() && rec.back().lv == lv_hi) {
    std::lock_guard<std::mutex> g(g_plan_mu);
    g_plans[key] = rec;
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
