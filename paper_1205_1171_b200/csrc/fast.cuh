// fast.cuh -- data layout and merge routines of the fused fast path.
//
// Layout in HBM (per pass, double-buffered A/B):
//   hdr[g]              int2 (nS, k) of group g at the current level
//   rec[L .. L+nS)      Rec: x, y, z (f64, z negated on the upper pass) and the
//                       chain links prev/next as GROUP-LOCAL ids (NIL = -1),
//                       at the group's start-of-time (t = -inf) state
//   gid[L .. L+nS)      global sorted index of each record
//   ev[2L .. 2L+k)      Ev: event time t (f64), the facet (a, b, c) of the
//                       event in group-local ids, and its kind (insertion /
//                       deletion); b is the reference's log entry
// A group [L, R) keeps only the points that matter above it: its chain at
// t = -inf plus every point its log mentions.  Local ids preserve x order, so
// the reference's x comparisons become integer comparisons (x is strictly
// increasing, store.py:70-71).
#pragma once
#include "h3d_device.cuh"

namespace h3d {

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

// Sequential merge (one thread) of ids [lo, mid) and [mid, hi) of R.  The
// semantics are _merge_one's (_ckernels.pyx:86-208) with changes that do not
// alter any decision: a child event's candidate time is its stored time (the
// time its facet got when it was emitted one level down, by the same
// expression on the same triple); the four bridge candidates are recomputed
// only when a foot or a foot's neighbour changed; every emitted event records
// its facet, kind and time.  The rewind is the reference's, so the links end
// exactly as the reference leaves them.  mark[p] = 1 for every emitted p.
// Returns k >= 0 or a negative code.
__device__ long long merge_seq(Rec *R, int lo, int mid, const Ev *evL, int kL, const Ev *evR,
                               int kR, Ev *out, int capO, int *mark, long long capRef,
                               long long limitRef, bool verify) {
  int u = mid - 1, v = mid;
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
#define H3D_EMIT(A_, B_, C_, T_, K_)                    \
  do {                                                  \
    if (k >= capRef - 1) return H3D_E_OVERFLOW;         \
    if (k >= capO) return E_FASTPATH;                   \
    Ev &o_ = out[k];                                    \
    o_.t = (T_);                                        \
    o_.a = (A_);                                        \
    o_.b = (B_);                                        \
    o_.c = (C_);                                        \
    o_.kind = (K_);                                     \
    mark[B_] = 1;                                       \
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
      const int e = (which == 0) ? evL[i].b : evR[j].b;
      const int p = R[e].prev, q = R[e].next;
      if (verify && !(evt_rec(R, p, e, q) == best)) return E_FASTPATH;
      if (p == NIL || q == NIL) return H3D_E_CHAIN;
      const int kind = (R[p].next == e) ? EV_DEL : EV_INS;
      if ((which == 0) ? (e < u) : (e > v)) H3D_EMIT(p, e, q, best, kind);
      act_rec(R, e);
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
        case 2: {  // u advances: the new foot enters the merged chain
          const int un = R[u].next;
          H3D_EMIT(u, un, v, best, EV_INS);
          u = un;
          break;
        }
        case 3:  // u leaves the merged chain
          H3D_EMIT(R[u].prev, u, v, best, EV_DEL);
          u = R[u].prev;
          break;
        case 4:  // v leaves the merged chain
          H3D_EMIT(u, v, R[v].next, best, EV_DEL);
          v = R[v].next;
          break;
        default: {  // v retreats: the new foot enters the merged chain
          const int vp = R[v].prev;
          H3D_EMIT(u, vp, v, best, EV_INS);
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
      if (act_rec(R, e) < 0) return H3D_E_CHAIN;
      if (e == u)
        u = R[u].prev;
      else if (e == v)
        v = R[v].next;
    } else {
      R[u].next = e;
      R[e].prev = u;
      R[v].prev = e;
      R[e].next = v;
      if (e < mid)
        u = e;
      else
        v = e;
    }
  }
  return k;
}

}  // namespace h3d
