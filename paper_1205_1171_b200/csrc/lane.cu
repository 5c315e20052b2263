// lane.cu -- one LANE per merge job: the levels with many small jobs.
//
// The reference merges one job per CPU thread with the sequential kinetic
// sweep of _merge_one (_ckernels.pyx:86-208).  Here one warp runs 32 jobs,
// one per lane, and every lane runs the same sweep; the design keeps one
// sweep step as short as the reference's own semantics allow:
//
//  * the bridge neighbourhood (u, v and the four chain neighbours up, un,
//    vp, vn) is cached as ids, the feet's coordinates in registers;
//  * a child event needs two link loads (its point and its left neighbour,
//    for the toggle direction), two link stores, and recomputes at most ONE
//    bridge candidate (the one whose foot neighbour it changed);
//  * a bridge move recomputes three candidates: the fourth is the reversed
//    event just taken, the same three points in the same operand order --
//    the same rounded time -- so it is copied, not recomputed;
//  * candidates are recomputed in one loop over a dirty mask (a warp pays
//    for the largest mask among its lanes, 3 evtimes for a bridge move);
//  * child event times are the stored canonical times; every
//    child event is checked against the current links (facet and toggle
//    direction) so a stored time is used only where the reference would
//    recompute the same value;
//  * merged events are staged in the job's shared-memory slice and written
//    to HBM ONCE, coalesced, with the compacted ids (a job whose log outgrows
//    its staged capacity spills the rest to its own HBM slots, which the
//    write-out then rewrites in place).
//
// Start-of-time links are rebuilt from the merged -inf chain and the first
// merged event of every point -- no sequential rewind.
#include "fast.cuh"

namespace h3d {

namespace {

constexpr unsigned kFiChain = 1u << 31;  // on its child's -inf chain
constexpr unsigned kFiEv = 1u << 30;     // has a merged event; bits 0-14 a, 15-29 c

// staged merged events: packed 15-bit ids (lane jobs have < 2^15 points)
__device__ __forceinline__ unsigned long long pack15(int a, int b, int c, int kind) {
  return static_cast<unsigned long long>(a) | (static_cast<unsigned long long>(b) << 15) |
         (static_cast<unsigned long long>(c) << 30) |
         (static_cast<unsigned long long>(kind) << 45);
}

template <bool XYZ>
struct LSlice {
  double *x, *y, *z;
  short2 *lk;
  int *gd;
  unsigned *fi;
  double *ot;
  unsigned long long *ow;
  __device__ __forceinline__ LSlice(unsigned char *base, int nS) {
    unsigned char *p = base;
    if (XYZ) {
      x = reinterpret_cast<double *>(p);
      y = x + nS;
      z = y + nS;
      p += 24ll * nS;
    }
    lk = reinterpret_cast<short2 *>(p);
    gd = reinterpret_cast<int *>(lk + nS);
    fi = reinterpret_cast<unsigned *>(gd + nS);
    p = base + align16((long long)lane_pt_bytes(XYZ) * nS);
    ot = reinterpret_cast<double *>(p);
  }
  __device__ __forceinline__ void set_ocap(int ocap) {
    ow = reinterpret_cast<unsigned long long *>(ot + ocap);
  }
  __device__ __forceinline__ P3 pt(int p, const double *__restrict__ pts, double zs) const {
    if (XYZ) {
      P3 r;
      r.x = x[p];
      r.y = y[p];
      r.z = z[p];
      return r;
    }
    return load_pt(pts, gd[p], zs);
  }
};

// two 64-bit loads straight into the loop-carried prefetch registers (a
// 128-bit load needs an aligned register quad, and the copy into the
// loop-carried registers then waits for the load)
__device__ __forceinline__ EvP ld_ev(const EvP *__restrict__ p) {
  EvP r;
  r.t = __ldg(&p->t);
  r.w = __ldg(&p->w);
  return r;
}

__device__ __forceinline__ EvP ev_inf() {
  EvP e;
  e.t = INF;
  e.w = 0;
  return e;
}

// The sweep of one job on one lane (_merge_one phase 1, _ckernels.pyx:86-183).
// All 32 lanes call it; a lane with active == false idles through it.
// Returns k (merged events) or a negative code.
template <bool XYZ>
__device__ long long lane_sweep(const LSlice<XYZ> &S, int ocap, bool active, int nSL,
                                const double *__restrict__ pts, double zs,
                                const EvP *__restrict__ evL, int kL,
                                const EvP *__restrict__ evR, int kR, EvP *__restrict__ spill,
                                long long capRef, long long limitRef, int *pu0, int *pv0) {
  long long err = 0;
  // ---- bridge at t = -inf (_find_bridge, _ckernels.pyx:63-83)
  int u = nSL - 1, v = nSL;
  P3 U, V;
  U.x = U.y = U.z = V.x = V.y = V.z = 0.0;
  if (active) {
    U = S.pt(u, pts, zs);
    V = S.pt(v, pts, zs);
    long long moves = 0;
    for (;;) {
      const int vn = S.lk[v].y;
      if (vn != NIL) {
        const P3 W = S.pt(vn, pts, zs);
        if (turn_xy(U.x, U.y, V.x, V.y, W.x, W.y) < 0.0) {
          v = vn;
          V = W;
          if (++moves > limitRef) break;
          continue;
        }
      }
      const int up = S.lk[u].x;
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
  int up = NIL, un = NIL, vp = NIL, vn = NIL;
  if (active) {
    const short2 lu = S.lk[u], lv = S.lk[v];
    up = lu.x;
    un = lu.y;
    vp = lv.x;
    vn = lv.y;
  }
  // candidate times of the four bridge moves (cases 2..5)
  double c2 = INF, c3 = INF, c4 = INF, c5 = INF;
  unsigned dirty = active ? 0xfu : 0u;
  // child streams: head + one event of prefetch (HBM)
  EvP hL = ev_inf(), hR = ev_inf(), nL = ev_inf(), nR = ev_inf();
  if (active) {
    if (kL > 0) hL = evL[0];
    if (kR > 0) hR = evR[0];
    // the prefetch index is clamped to the log (k - 1): reading the stale
    // slot k would be harmless but reads memory no level wrote (initcheck)
    if (kL > 0) nL = ld_ev(evL + (kL > 1 ? 1 : 0));
    if (kR > 0) nR = ld_ev(evR + (kR > 1 ? 1 : 0));
  }
  int i = 0, j = 0, k = 0;
  double tcur = -INF;
  while (__any_sync(FULL, active)) {
    // ---- recompute the candidates whose inputs changed
    // c2 = (u, un, v)  c3 = (up, u, v)  c4 = (u, v, vn)  c5 = (u, vp, v)
    if (XYZ) {
      // coordinates in shared memory: one loop, a warp pays for the largest
      // dirty mask of its lanes
      while (dirty) {
        const int d = __ffs(dirty) - 1;
        dirty &= dirty - 1;
        const int o = d == 0 ? un : (d == 1 ? up : (d == 2 ? vn : vp));
        double t = INF;
        if (o != NIL) {
          const P3 O = S.pt(o, pts, zs);
          const P3 A = d == 1 ? O : U;
          const P3 B = (d == 0 || d == 3) ? O : (d == 1 ? U : V);
          const P3 C = d == 2 ? O : V;
          t = evtime_xyz(A.x, A.y, A.z, B.x, B.y, B.z, C.x, C.y, C.z);
        }
        c2 = d == 0 ? t : c2;
        c3 = d == 1 ? t : c3;
        c4 = d == 2 ? t : c4;
        c5 = d == 3 ? t : c5;
      }
    } else if (__any_sync(FULL, dirty != 0)) {
      // coordinates in HBM/L2: issue every needed row first (one latency),
      // then compute
      const bool d0 = (dirty & 1u) && un != NIL, d1 = (dirty & 2u) && up != NIL;
      const bool d2 = (dirty & 4u) && vn != NIL, d3 = (dirty & 8u) && vp != NIL;
      P3 O0, O1, O2, O3;
      O0.x = O0.y = O0.z = O1.x = O1.y = O1.z = 0.0;
      O2 = O0;
      O3 = O0;
      if (d0) O0 = S.pt(un, pts, zs);
      if (d1) O1 = S.pt(up, pts, zs);
      if (d2) O2 = S.pt(vn, pts, zs);
      if (d3) O3 = S.pt(vp, pts, zs);
      if (dirty & 1u) c2 = d0 ? evtime_xyz(U.x, U.y, U.z, O0.x, O0.y, O0.z, V.x, V.y, V.z) : INF;
      if (dirty & 2u) c3 = d1 ? evtime_xyz(O1.x, O1.y, O1.z, U.x, U.y, U.z, V.x, V.y, V.z) : INF;
      if (dirty & 4u) c4 = d2 ? evtime_xyz(U.x, U.y, U.z, V.x, V.y, V.z, O2.x, O2.y, O2.z) : INF;
      if (dirty & 8u) c5 = d3 ? evtime_xyz(U.x, U.y, U.z, O3.x, O3.y, O3.z, V.x, V.y, V.z) : INF;
      dirty = 0;
    }
    // ---- next event: earliest time strictly after tcur, lowest case on ties
    double best = INF;
    int which = -1;
    if (hL.t > tcur && hL.t < best) { best = hL.t; which = 0; }
    if (hR.t > tcur && hR.t < best) { best = hR.t; which = 1; }
    if (c2 > tcur && c2 < best) { best = c2; which = 2; }
    if (c3 > tcur && c3 < best) { best = c3; which = 3; }
    if (c4 > tcur && c4 < best) { best = c4; which = 4; }
    if (c5 > tcur && c5 < best) { best = c5; which = 5; }
    active = active && which >= 0;
    int ea = 0, eb = 0, ec = 0, ek = 0;
    bool emit = false;
    if (active && which <= 1) {
      // ---- child event: _act (_ckernels.pyx:49-60) + the emission rule
      const bool left = which == 0;
      const EvP ev = left ? hL : hR;
      const int off = left ? 0 : nSL;
      const int e = ev.b() + off;
      const short2 le = S.lk[e];
      const int p = le.x, q = le.y;
      bool ok = p != NIL && q != NIL && p == ev.a() + off && q == ev.c() + off;
      bool del = false;
      if (ok) {
        del = S.lk[p].y == e;
        ok = (del ? EV_DEL : EV_INS) == ev.kind();
      }
      if (!ok) {
        err = E_FASTPATH;
        active = false;
      } else {
        S.lk[p].y = static_cast<short>(del ? q : e);
        S.lk[q].x = static_cast<short>(del ? p : e);
        emit = left ? e < u : e > v;
        ea = p;
        eb = e;
        ec = q;
        ek = del ? EV_DEL : EV_INS;
        // the feet's own links never change here; their neighbours' may
        if (p == u) { un = del ? q : e; dirty |= 1u; }
        if (q == u) { up = del ? p : e; dirty |= 2u; }
        if (p == v) { vn = del ? q : e; dirty |= 4u; }
        if (q == v) { vp = del ? p : e; dirty |= 8u; }
        if (left) {
          ++i;
          hL = i < kL ? nL : ev_inf();
          nL = ld_ev(evL + min(i + 1, kL - 1));
        } else {
          ++j;
          hR = j < kR ? nR : ev_inf();
          nR = ld_ev(evR + min(j + 1, kR - 1));
        }
      }
    } else if (active) {
      // ---- bridge move (cases 2..5, _ckernels.pyx:159-182): emit, move the
      // foot, read the new foot's links
      const bool uside = which <= 3;
      const int nf = which == 2 ? un : (which == 3 ? up : (which == 4 ? vn : vp));
      ea = which == 3 ? up : u;
      eb = which == 2 ? un : (which == 3 ? u : (which == 4 ? v : vp));
      ec = which == 4 ? vn : v;
      ek = (which == 3 || which == 4) ? EV_DEL : EV_INS;
      emit = true;
      const short2 lf = S.lk[nf];
      const P3 F = S.pt(nf, pts, zs);
      if (uside) {
        const int old = u;
        u = nf;
        U = F;
        up = lf.x;
        un = lf.y;
        // the reversed move is the event just taken: same points, same
        // operand order, same rounded time (not eligible again)
        if (which == 2 && up == old) { c3 = best; dirty |= 0xdu; }
        else if (which == 3 && un == old) { c2 = best; dirty |= 0xeu; }
        else dirty |= 0xfu;
      } else {
        const int old = v;
        v = nf;
        V = F;
        vp = lf.x;
        vn = lf.y;
        if (which == 4 && vp == old) { c5 = best; dirty |= 0x7u; }
        else if (which == 5 && vn == old) { c4 = best; dirty |= 0xbu; }
        else dirty |= 0xfu;
      }
    }
    if (emit) {
      if (k >= capRef - 1) {
        err = H3D_E_OVERFLOW;
        active = false;
      } else {
        if (k < ocap) {
          S.ot[k] = best;
          S.ow[k] = pack15(ea, eb, ec, ek);
        } else {
          Ev o;
          o.t = best;
          o.a = ea;
          o.b = eb;
          o.c = ec;
          o.kind = ek;
          spill[k] = EvP(o);
        }
        const unsigned f = S.fi[eb];
        if (!(f & kFiEv))
          S.fi[eb] = f | kFiEv | static_cast<unsigned>(ea) | (static_cast<unsigned>(ec) << 15);
        ++k;
      }
    }
    if (active) tcur = best;
  }
  return err ? err : k;
}

}  // namespace

// One warp = up to 32 merge jobs (jpc per CTA), one per lane.
template <bool XYZ>
#ifdef H3D_LANE_MINB  // register cap experiments (tools/ab_libs.sh); unset by default
__global__ void __launch_bounds__(32, H3D_LANE_MINB) k_lane(
#else
__global__ void __launch_bounds__(32) k_lane(
#endif
Pass2 P, const double *__restrict__ pts, long long n,
                                             int level, long long j0, long long j1,
                                             long long *err, int pool, int jpc, int stage_own,
                                             long long *spec, long long *stamp) {
  // stage_own: bit 0 stage the merged events, bit 1 each lane stages its own job's rows
  const int stage = stage_own & 1, own = (stage_own >> 1) & 1;
  if (stamp && blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x == 0) {  // level start (ns)
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    *stamp = static_cast<long long>(t);
  }
  // an earlier level failed, or (a replayed plan, spec) did not fit: stop
  // (warp-uniform; the words it reads may be stale)
  if (__any_sync(FULL, *reinterpret_cast<volatile long long *>(err) != 0 ||
                           (spec && *reinterpret_cast<volatile long long *>(spec) != 0)))
    return;
  const int pass = lvl_pass();
  const GroupBuf in = pass ? P.in1 : P.in0;
  const GroupBuf out = pass ? P.out1 : P.out0;
  const double zs = pass ? -1.0 : 1.0;
  extern __shared__ __align__(16) unsigned char smem[];
  const int lane = threadIdx.x;
  const long long size = 1ll << level, half = size >> 1;
  const long long j = j0 + lvl_blk() * jpc + lane;
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
  if (merge && (stage_own & 12)) {
    // the job's rows (sorted positions [L, R_)) towards L1 (bit 2) or L2
    // (bit 3) before the staging: the sweep's dependent gathers then hit
    const char *a = reinterpret_cast<const char *>(pts + 3 * L);
    const char *e = reinterpret_cast<const char *>(pts + 3 * R_);
    for (const char *q = reinterpret_cast<const char *>(reinterpret_cast<uintptr_t>(a) & ~uintptr_t(127)); q < e;
         q += 128) {
      if (stage_own & 4)
        asm volatile("prefetch.global.L1 [%0];" ::"l"(q));
      else
        asm volatile("prefetch.global.L2 [%0];" ::"l"(q));
    }
  }
  if (merge && nS >= 0x7fff) {  // int16 local ids; the host never routes such jobs here ...
    if (spec)  // ... unless it replays a plan: report the level, it is redone measured
      atomicCAS(reinterpret_cast<unsigned long long *>(spec), 0ull, static_cast<unsigned long long>(level));
    else
      raise_err(err, E_FASTPATH);
    merge = false;
  }
  const int ocap = (merge && stage) ? lane_ocap(nS, kL + kR) : 0;
  // pack the slices: warp exclusive prefix sum of the slice sizes
  const int bytes = merge ? lane_slice_bytes(nS, ocap, XYZ) : 0;
  int off = bytes;
  for (int o = 1; o < 32; o <<= 1) {
    const int t = __shfl_up_sync(FULL, off, o);
    if (lane >= o) off += t;
  }
  const int total = __shfl_sync(FULL, off, 31);
  off -= bytes;
  if (total > pool) {  // the host sizes the pool from the measured need (or a replayed plan's)
    if (lane == 0) {
      if (spec)
        atomicCAS(reinterpret_cast<unsigned long long *>(spec), 0ull, static_cast<unsigned long long>(level));
      else
        raise_err(err, E_FASTPATH);
    }
    return;
  }
  // per-job metadata for the cooperative phases
  __shared__ long long s_L[32], s_M[32];
  __shared__ int s_off[32], s_nSL[32], s_pre[33], s_epre[33], s_ocap[32];
  s_L[lane] = L;
  s_M[lane] = M;
  s_off[lane] = off;
  s_nSL[lane] = nSL;
  s_ocap[lane] = ocap;
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
  // ---- stage links, gids (+ coordinates): flattened over the 32 jobs'
  // points, coalesced, U elements per lane in flight -- or (own, small jobs
  // without coordinates) every lane its own job's rows, no job-index walk
  constexpr int U = 4;
  int js = 0;
  if (own && !XYZ) {
    if (merge) {
      const LSlice<XYZ> T(smem + off, nS);
      for (int p0 = 0; p0 < nS; p0 += U) {
        int2 l[U];
        int g[U];
#pragma unroll
        for (int q = 0; q < U; ++q) {
          const int p = p0 + q;
          if (p < nS) {
            const long long src = p < nSL ? L + p : M + (p - nSL);
            l[q] = in.lnk[src];
            g[q] = in.gid[src];
          }
        }
#pragma unroll
        for (int q = 0; q < U; ++q) {
          const int p = p0 + q;
          if (p >= nS) break;
          int2 lq = l[q];
          if (p >= nSL) {
            if (lq.x != NIL) lq.x += nSL;
            if (lq.y != NIL) lq.y += nSL;
          }
          T.lk[p] = make_short2(static_cast<short>(lq.x), static_cast<short>(lq.y));
          T.gd[p] = g[q];
        }
      }
    }
  }
  for (int x0 = 0; x0 < (own && !XYZ ? 0 : tot_pts); x0 += 32 * U) {
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
    }
#pragma unroll
    for (int q = 0; q < U; ++q) {
      if (x0 + q * 32 + lane >= tot_pts) continue;
      const int m_nS = s_pre[jj[q] + 1] - s_pre[jj[q]], m_nSL = s_nSL[jj[q]];
      const LSlice<XYZ> T(smem + s_off[jj[q]], m_nS);
      int2 lq = l[q];
      if (p[q] >= m_nSL) {
        if (lq.x != NIL) lq.x += m_nSL;
        if (lq.y != NIL) lq.y += m_nSL;
      }
      T.lk[p[q]] = make_short2(static_cast<short>(lq.x), static_cast<short>(lq.y));
      T.gd[p[q]] = g[q];
      if (XYZ) {
        T.x[p[q]] = c[q].x;
        T.y[p[q]] = c[q].y;
        T.z[p[q]] = c[q].z;
      }
    }
  }
  __syncwarp();
  LSlice<XYZ> S(smem + off, nS);
  S.set_ocap(ocap);
  if (merge) {
    // chain flags: p is on its child's -inf chain iff its prev points back
    for (int p = 0; p < nS; ++p) {
      const int pr = S.lk[p].x;
      const bool chain = p == 0 || p == nSL || (pr != NIL && S.lk[pr].y == p);
      S.fi[p] = chain ? kFiChain : 0u;
    }
  }
  int u0 = 0, v0 = 0;
  long long k = lane_sweep<XYZ>(S, ocap, merge, nSL, pts, zs, in.ev + 2 * L, kL, in.ev + 2 * M, kR,
                                out.ev + 2 * L, 2 * (R_ - L), R_ - L, &u0, &v0);
  if (merge && k < 0) {
    raise_err(err, k);
    merge = false;
  }
  int cnt = 0;
  if (merge) {
    // ---- start-of-time links of the merged group: the
    // merged -inf chain is every chain-flagged point left of u0 (inclusive)
    // or right of v0, linked in x order; every other kept point gets the
    // neighbours of its first merged event (its insertion).  fi becomes
    // the old -> new id map.
    int last = NIL;
    for (int p = 0; p < nS; ++p) {
      const unsigned f = S.fi[p];
      const bool chain = (f & kFiChain) && (p < nSL ? p <= u0 : p >= v0);
      if (chain) {
        S.lk[p].x = static_cast<short>(last);
        if (last != NIL) S.lk[last].y = static_cast<short>(p);
        last = p;
      } else if (f & kFiEv) {
        S.lk[p] = make_short2(static_cast<short>(f & 0x7fff), static_cast<short>((f >> 15) & 0x7fff));
      }
      S.fi[p] = (chain || (f & kFiEv)) ? static_cast<unsigned>(cnt++) : FULL;
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
    if (merge) out.hdr[j] = make_int2(cnt, static_cast<int>(k));
  }
  __syncwarp();
  // ---- write-out (cooperative, coalesced): links + gids at their new ids
  // (own: every lane its own job, no job-index walk)
  bool bad = false;
  const int tot_p2 = own ? 0 : s_pre[32], tot_ev = own ? 0 : s_epre[32];
  if (own && merge) {
    for (int p = 0; p < nS; ++p) {
      const unsigned id = S.fi[p];
      if (id == FULL) continue;
      const short2 l = S.lk[p];
      int2 o;
      o.x = l.x == NIL ? NIL : static_cast<int>(S.fi[l.x]);
      o.y = l.y == NIL ? NIL : static_cast<int>(S.fi[l.y]);
      bad |= (o.x == -1 && l.x != NIL) | (o.y == -1 && l.y != NIL);
      out.lnk[L + id] = o;
      out.gid[L + id] = S.gd[p];
    }
    for (int e = 0; e < static_cast<int>(k); ++e) {
      EvP *dst = out.ev + 2 * L + e;
      Ev o;
      if (e < ocap) {
        const unsigned long long w = S.ow[e];
        o.t = S.ot[e];
        o.a = static_cast<int>(w & 0x7fff);
        o.b = static_cast<int>((w >> 15) & 0x7fff);
        o.c = static_cast<int>((w >> 30) & 0x7fff);
        o.kind = static_cast<int>(w >> 45);
      } else {
        o = *dst;
      }
      const unsigned na = S.fi[o.a], nb = S.fi[o.b], nc = S.fi[o.c];
      bad |= (na == FULL) | (nb == FULL) | (nc == FULL);
      o.a = static_cast<int>(na);
      o.b = static_cast<int>(nb);
      o.c = static_cast<int>(nc);
      *dst = EvP(o);
    }
  }
  int jw = 0;
  for (int x = lane; x < tot_p2; x += 32) {
    while (s_pre[jw + 1] <= x) ++jw;  // the job index only advances
    const int jj = jw;
    const int p = x - s_pre[jj];
    const LSlice<XYZ> T(smem + s_off[jj], s_pre[jj + 1] - s_pre[jj]);
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
  // ---- events: once, with the new ids (staged ones from shared memory,
  // spilled ones read back from their own slots)
  jw = 0;
  for (int x = lane; x < tot_ev; x += 32) {
    while (s_epre[jw + 1] <= x) ++jw;
    const int jj = jw;
    const int e = x - s_epre[jj];
    LSlice<XYZ> T(smem + s_off[jj], s_pre[jj + 1] - s_pre[jj]);
    const int oc = s_ocap[jj];
    T.set_ocap(oc);
    EvP *dst = out.ev + 2 * s_L[jj] + e;
    Ev o;
    if (e < oc) {
      const unsigned long long w = T.ow[e];
      o.t = T.ot[e];
      o.a = static_cast<int>(w & 0x7fff);
      o.b = static_cast<int>((w >> 15) & 0x7fff);
      o.c = static_cast<int>((w >> 30) & 0x7fff);
      o.kind = static_cast<int>(w >> 45);
    } else {
      o = *dst;
    }
    const unsigned na = T.fi[o.a], nb = T.fi[o.b], nc = T.fi[o.c];
    bad |= (na == FULL) | (nb == FULL) | (nc == FULL);
    o.a = static_cast<int>(na);
    o.b = static_cast<int>(nb);
    o.c = static_cast<int>(nc);
    *dst = EvP(o);
  }
  if (__any_sync(FULL, bad) && lane == 0) raise_err(err, E_FASTPATH);
}

namespace {
bool g_lane_attr[64] = {};
}

// lane-kernel variant knobs (h3d_tune / environment, fast.cu)
// (defaults measured on C4/C2/C3: staging either costs more occupancy than
// it saves, profiles/r2_levels_c4.jsonl)
long long g_lane_xyz_max = 0;  // H3D_LANE_XYZ_KB: stage coordinates up to this pool
int g_lane_stage = 0;          // H3D_LANE_STAGE: stage merged events (0 = never)
// H3D_LANE_PF1 / _PF2: lane.cu levels up to which each job's rows are
// prefetched to L1 / L2 before the staging (C4 level 4 -1.5 %, level 5 -2.8 %)
int g_lane_pf1 = 4, g_lane_pf2 = 5;
int g_lane_own = 4;            // H3D_LANE_OWN: up to this level each lane stages and writes its own job (C4 level 4 -3 %)

// Host side: choose the variant (coordinates / merged events staged in
// shared memory) and jobs per CTA from the level's measured shared-memory
// need (k_tpj_need: need[16 + 6 v + r] = largest CTA pool of variant
// v = 2 * xyz + staged for 32 >> r jobs per CTA), and launch.  Returns 0,
// 1 (does not fit: the caller routes the level elsewhere) or a negative code.
long long lane_level(const Pass2 &P, const double *pts, long long n, int lv, long long j0,
                     long long j1, long long *err, const unsigned long long *need,
                     cudaStream_t s, LaneCfg *cfg, long long *spec, long long *stamp) {
  constexpr int kPool = 200 * 1024;
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) return H3D_E_ARG;
  if (!g_lane_attr[dev]) {
    if (h3d_check(cudaFuncSetAttribute(k_lane<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, kPool)) ||
        h3d_check(cudaFuncSetAttribute(k_lane<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, kPool)))
      return H3D_E_CUDA;
    g_lane_attr[dev] = true;
  }
  const long long jobs = j1 - j0;
  if (!need) {  // a replayed plan: the recorded variant, jobs per CTA and pool
    const int jpc = 32 >> cfg->r;
    h3d_count_launches(1);
    const dim3 grid = lvl_grid(h3d_grid(jobs, jpc), g_interleave != 0);
    const int pool = static_cast<int>(cfg->pool);
    if (cfg->v >= 2)
      k_lane<true><<<grid, 32, pool, s>>>(P, pts, n, lv, j0, j1, err, pool, jpc, (cfg->v & 1) | ((lv <= g_lane_own ? 1 : 0) << 1) | (lv <= g_lane_pf1 ? 4 : (lv <= g_lane_pf2 ? 8 : 0)),
                                          spec, stamp);
    else
      k_lane<false><<<grid, 32, pool, s>>>(P, pts, n, lv, j0, j1, err, pool, jpc, (cfg->v & 1) | ((lv <= g_lane_own ? 1 : 0) << 1) | (lv <= g_lane_pf1 ? 4 : (lv <= g_lane_pf2 ? 8 : 0)),
                                           spec, stamp);
    return 0;
  }
  auto pick = [&](int v, int *jr) {  // fewest-lanes-idle jobs per CTA that fits
    int r = 0;
    while (r < 5 && static_cast<long long>(need[16 + 6 * v + r]) > kPool) ++r;
    *jr = r;
    return static_cast<long long>(need[16 + 6 * v + r]);
  };
  int r = 0, v = -1;
  long long pool = 0;
  for (int xyz = 1; xyz >= 0 && v < 0; --xyz) {
    for (int st = g_lane_stage ? 1 : 0; st >= 0 && v < 0; --st) {
      int rr;
      const long long p = pick(2 * xyz + st, &rr);
      if (p > kPool || (xyz && p > g_lane_xyz_max)) continue;
      // staged events only while they cost no jobs per CTA
      if (st) {
        int r0;
        pick(2 * xyz, &r0);
        if (rr != r0) continue;
      }
      v = 2 * xyz + st;
      r = rr;
      pool = p;
    }
  }
  if (v < 0) return 1;
  const int jpc = 32 >> r;
  if (pool < 1024) pool = 1024;
  h3d_count_launches(1);
  const dim3 grid = lvl_grid(h3d_grid(jobs, jpc), g_interleave != 0);
  if (v >= 2)
    k_lane<true><<<grid, 32, pool, s>>>(P, pts, n, lv, j0, j1, err, static_cast<int>(pool), jpc,
                                       (v & 1) | ((lv <= g_lane_own ? 1 : 0) << 1) | (lv <= g_lane_pf1 ? 4 : (lv <= g_lane_pf2 ? 8 : 0)), spec, stamp);
  else
    k_lane<false><<<grid, 32, pool, s>>>(P, pts, n, lv, j0, j1, err, static_cast<int>(pool), jpc,
                                        (v & 1) | ((lv <= g_lane_own ? 1 : 0) << 1) | (lv <= g_lane_pf1 ? 4 : (lv <= g_lane_pf2 ? 8 : 0)), spec, stamp);
  if (cfg) *cfg = LaneCfg{v, r, pool};
  return 0;
}

}  // namespace h3d
