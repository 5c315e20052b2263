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

}  // namespace h3d
