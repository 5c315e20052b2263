// fast.cuh -- data layout and the compact-group merge of the fused fast path.
//
// Layout in HBM (per pass, double-buffered A/B):
//   hdr[g]              int2 (nS, k) of group g at the current level
//   rec[L .. L+nS)      Rec: x, y, z (f64, z negated on the upper pass) and the
//                       chain links prev/next as GROUP-LOCAL ids (NIL = -1)
//   gid[L .. L+nS)      global sorted index of each record
//   ev[2L .. 2L+k)      Ev: event time t (f64) and the facet (a, b, c) of the
//                       event, group-local ids; b is the reference's log entry
// A group [L, R) keeps only the points that matter above it: its chain at
// t = -inf plus every point its log mentions (S = -inf chain U log).  Local
// ids preserve x order, so the reference's x comparisons become integer
// comparisons (x is strictly increasing, store.py:70-71).
#pragma once
#include "h3d_device.cuh"

namespace h3d {

struct __align__(8) Rec {
  double x, y, z;
  int prev, next;
};

struct __align__(8) Ev {
  double t;
  int a, b, c, pad;
};

static_assert(sizeof(Rec) == 32, "Rec must be one 32-byte sector");
static_assert(sizeof(Ev) == 24, "Ev is 24 bytes");

// fast path could not reproduce the reference semantics: rerun exact
constexpr long long E_FASTPATH = -13;

__device__ __forceinline__ double evt_rec(const Rec *R, int a, int b, int c) {
  if (a == NIL || b == NIL || c == NIL) return INF;
  const Rec &A = R[a], &B = R[b], &C = R[c];
  return evtime_xyz(A.x, A.y, A.z, B.x, B.y, B.z, C.x, C.y, C.z);
}

// _act (_ckernels.pyx:49-60) on local links; returns -1 on a NIL neighbour
__device__ __forceinline__ int act_rec(Rec *R, int e, int *p_out, int *q_out) {
  const int p = R[e].prev, q = R[e].next;
  *p_out = p;
  *q_out = q;
  if (p == NIL || q == NIL) return -1;
  if (R[p].next == e) {
    R[p].next = q;
    R[q].prev = p;
  } else {
    R[p].next = e;
    R[q].prev = e;
  }
  return 0;
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

// One pairwise merge on a compact group pair: records R[0, nS) with the left
// group at [0, nSL) and the right at [nSL, nS) (links already in this id
// space); child logs evL[0,kL) and evR[0,kR) whose ids get +offL/+offR.
// Semantics are _merge_one's (_ckernels.pyx:86-208) with three changes that
// do not alter any decision: (1) a child event's candidate time is its
// stored time (the time its facet got when it was emitted one level down,
// computed by the same expression on the same triple); (2) the four bridge
// candidates are recomputed only when a foot or a foot's neighbour changed;
// (3) every emitted event records its facet (a, b, c) and time.  The rewind
// is the reference's.  mark[p] |= 1 for every emitted point.
// Returns k >= 0, or a negative code.
__device__ long long merge_compact(Rec *R, int nSL, int nS, const Ev *evL, int kL, int offL,
                                   const Ev *evR, int kR, int offR, Ev *out, int capO,
                                   int *mark, long long capRef, long long limitRef,
                                   bool verify) {
  int u = nSL - 1, v = nSL;
  if (bridge_rec(R, &u, &v, limitRef) < 0) return H3D_E_BRIDGE;
  int i = 0, j = 0, k = 0;
  double tcur = -INF;
  double c0 = (kL > 0) ? evL[0].t : INF;
  double c1 = (kR > 0) ? evR[0].t : INF;
  double c2, c3, c4, c5;
#define H3D_BRIDGE_CANDS()                      \
  do {                                          \
    c2 = evt_rec(R, u, R[u].next, v);           \
    c3 = evt_rec(R, R[u].prev, u, v);           \
    c4 = evt_rec(R, u, v, R[v].next);           \
    c5 = evt_rec(R, u, R[v].prev, v);           \
  } while (0)
#define H3D_EMIT(A_, B_, C_, T_)                        \
  do {                                                  \
    if (k >= capRef - 1) return H3D_E_OVERFLOW;         \
    if (k >= capO) return E_FASTPATH;                   \
    Ev &o_ = out[k];                                    \
    o_.t = (T_);                                        \
    o_.a = (A_);                                        \
    o_.b = (B_);                                        \
    o_.c = (C_);                                        \
    mark[B_] |= 1;                                      \
    ++k;                                                \
  } while (0)
  H3D_BRIDGE_CANDS();
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
    if (which <= 1) {
      const Ev &ce = (which == 0) ? evL[i] : evR[j];
      const int e = ce.b + (which == 0 ? offL : offR);
      if (verify) {
        // the stored time must be what the reference computes from the links
        const double tl = evt_rec(R, R[e].prev, e, R[e].next);
        if (!(tl == best)) return E_FASTPATH;
      }
      const bool outside = (which == 0) ? (e < u) : (e > v);
      if (outside) H3D_EMIT(R[e].prev, e, R[e].next, best);
      int p, q;
      if (act_rec(R, e, &p, &q) < 0) return H3D_E_CHAIN;
      if (which == 0) {
        ++i;
        c0 = (i < kL) ? evL[i].t : INF;
      } else {
        ++j;
        c1 = (j < kR) ? evR[j].t : INF;
      }
      if (p == u || q == u || p == v || q == v) H3D_BRIDGE_CANDS();
    } else {
      switch (which) {
        case 2: {
          const int un = R[u].next;
          H3D_EMIT(u, un, v, best);
          u = un;
          break;
        }
        case 3:
          H3D_EMIT(R[u].prev, u, v, best);
          u = R[u].prev;
          break;
        case 4:
          H3D_EMIT(u, v, R[v].next, best);
          v = R[v].next;
          break;
        default: {
          const int vp = R[v].prev;
          H3D_EMIT(u, vp, v, best);
          v = vp;
          break;
        }
      }
      H3D_BRIDGE_CANDS();
    }
    tcur = best;
  }
#undef H3D_EMIT
#undef H3D_BRIDGE_CANDS
  // stitch the final bridge, then rewind to the merged start-of-time chain
  R[u].next = v;
  R[v].prev = u;
  for (int idx = k - 1; idx >= 0; --idx) {
    const int e = out[idx].b;
    if (e <= u || e >= v) {
      int p, q;
      if (act_rec(R, e, &p, &q) < 0) return H3D_E_CHAIN;
      if (e == u)
        u = R[u].prev;
      else if (e == v)
        v = R[v].next;
    } else {
      R[u].next = e;
      R[e].prev = u;
      R[v].prev = e;
      R[e].next = v;
      if (e < nSL)
        u = e;
      else
        v = e;
    }
  }
  // the merged -inf chain (always kept): walk from the leftmost point
  int steps = 0;
  for (int p = 0; p != NIL; p = R[p].next) {
    mark[p] |= 2;
    if (++steps > nS) return E_FASTPATH;
  }
  (void)nS;
  return k;
}

}  // namespace h3d
