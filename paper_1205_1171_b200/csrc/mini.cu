// mini.cu -- the time-split merge (big.cu) for SMALL jobs, one CTA per job,
// everything in shared memory.
//
// Levels with few jobs whose merged child log is a few hundred to two
// thousand events (the top levels of cube/ball clouds) are sequential
// chains: ~800 dependent steps per job whatever the kernel.  Here the same
// decomposition as big.cu runs inside one CTA: merged child sequence S,
// per-point incidence lists (counting sort + per-list insertion sort), links
// after each incidence, segment start bridges by walks at the segment time,
// segment sweeps over only the foot-touching events and the bridge events,
// classification of every child event by the bridge at its time, and the
// start-of-time link rebuild + compaction -- with shared-memory latencies
// instead of HBM ones, and one launch per level.
#include <type_traits>


#include "fast.cuh"

namespace h3d {

#ifdef H3D_MINI_PROF
// phase clocks of CTA (0, 0) per level (profiling builds only)
__device__ long long g_mini_prof[64][16];
#define MINI_TICK(i) \
  do { if (tid == 0 && blockIdx.x == 0 && blockIdx.y == 0) g_mini_prof[lv][i] = clock64(); } while (0)
#else
#define MINI_TICK(i) do {} while (0)
#endif

constexpr int MINI_S = 256;    // largest number of time segments
constexpr int MINI_NIL = -1;

// MINI_T threads per CTA (one job), MINI_K largest merged child log,
// MINI_N largest job (points), MINI_B largest number of bridge events
// facet words: a | b << S | c << 2S | kind << 3S | side << 3S+1, with
// S = 10 in 32-bit words (jobs of <= 1024 points) and S = 16 in 64-bit words
// (the huge variant in global memory)
template <int MINI_N>
using MiniWord = typename std::conditional<(MINI_N <= 1024), unsigned, unsigned long long>::type;

template <class W>
__device__ __forceinline__ constexpr int wsh() {
  return sizeof(W) == 4 ? 10 : 16;
}
template <class W>
__device__ __forceinline__ W wpack(int a, int b, int c, int kind, int side) {
  constexpr int S = wsh<W>();
  return static_cast<W>(a) | (static_cast<W>(b) << S) | (static_cast<W>(c) << (2 * S)) |
         (static_cast<W>(kind & 1) << (3 * S)) | (static_cast<W>(side & 1) << (3 * S + 1));
}

template <int MINI_T, int MINI_K, int MINI_N>
struct MiniSmem {
  static constexpr int MINI_B = MINI_K;
  using W = MiniWord<MINI_N>;
  double st[MINI_K];            // S: event times
  W sw[MINI_K];                 // S: facet words (a, b, c, kind, side)
  double X[MINI_N], Y[MINI_N], Z[MINI_N];
  short2 LN[MINI_N];            // links at t = -inf (job-local)

  int ib[MINI_N + 1];           // incidence list bounds (exclusive scan)
  short ei[3 * MINI_K];         // incidence: event index (each list in event order);
                                // the rebuild's links KL live here (dead after the sweeps)
  short2 el[3 * MINI_K];        // incidence: links after the event
  double bt[MINI_B];            // bridge events: time
  W bw[MINI_B];                 //   facet word (side 0)
  short2 buv[MINI_B];           //   feet after
  // per-segment slabs of the sweep (then compacted); the incidence
  // scatter's temporary (eo: 3K shorts, dead before the sweeps) lives in
  // slt: the smaller footprint lets the tiny variant fit 7 CTAs per SM
  static_assert(3 * MINI_K * sizeof(short) <= MINI_B * sizeof(double), "eo must fit slt");
  double slt[MINI_B];
  W slw[MINI_B];
  short2 sluv[MINI_B];
  static constexpr int NSEG = MINI_T < MINI_S ? MINI_T : MINI_S;  // segments <= threads
  short2 sst[NSEG];             // segment start bridges
  int sbn[NSEG + 1];            // bridge events per segment, then offsets
  int flag, nb, kept;
  __device__ __forceinline__ short *eo() { return reinterpret_cast<short *>(slt); }
  static_assert(MINI_N * sizeof(short2) <= 3 * MINI_K * sizeof(short), "KL must fit ei");
  __device__ __forceinline__ short2 *KL() { return reinterpret_cast<short2 *>(ei); }
  // after the sweeps the incidence arrays are dead: the kept-child-event
  // positions live in el, the new point ids in ib
  static_assert((MINI_K + 1) * sizeof(int) <= 3 * MINI_K * sizeof(short2), "cpos must fit el");
  __device__ __forceinline__ int *cpos() { return reinterpret_cast<int *>(el); }
  __device__ __forceinline__ int *nid() { return ib; }
  // the per-point counts / scatter cursors (phase 2) and first output
  // events (after the compaction) live in the sweep slab's word array, dead
  // in both phases
  static_assert(MINI_N * sizeof(int) <= MINI_B * sizeof(W), "cur must fit slw");
  __device__ __forceinline__ int *cur() { return reinterpret_cast<int *>(slw); }
};

template <class W>
__device__ __forceinline__ int swa(W w) {
  return static_cast<int>(w & ((W(1) << wsh<W>()) - 1));
}
template <class W>
__device__ __forceinline__ int swb(W w) {
  return static_cast<int>((w >> wsh<W>()) & ((W(1) << wsh<W>()) - 1));
}
template <class W>
__device__ __forceinline__ int swc(W w) {
  return static_cast<int>((w >> (2 * wsh<W>())) & ((W(1) << wsh<W>()) - 1));
}
template <class W>
__device__ __forceinline__ int swk(W w) {
  return static_cast<int>((w >> (3 * wsh<W>())) & 1u);
}
template <class W>
__device__ __forceinline__ int sws(W w) {
  return static_cast<int>((w >> (3 * wsh<W>() + 1)) & 1u);
}

// exclusive prefix sum of one value per thread over a T-thread block
template <int T>
__device__ __forceinline__ int mini_excl_sum(int v, int *s_w) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  int x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int t = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += t;
  }
  if (lane == 31) s_w[w] = x;
  __syncthreads();
  int pre = 0;
#pragma unroll
  for (int q = 0; q < T / 32; ++q) pre += q < w ? s_w[q] : 0;
  __syncthreads();
  return pre + x - v;
}

template <class MS>
__device__ __forceinline__ P3 mpt(const MS &m, int p) {
  P3 r;
  if (p == MINI_NIL) {
    r.x = r.y = r.z = 0.0;
    return r;
  }
  r.x = m.X[p];
  r.y = m.Y[p];
  r.z = m.Z[p];
  return r;
}

template <class MS>
__device__ __forceinline__ double mevt(const MS &m, int a, int b, int c) {
  if (a == MINI_NIL || b == MINI_NIL || c == MINI_NIL) return INF;
  return evtime_xyz(m.X[a], m.Y[a], m.Z[a], m.X[b], m.Y[b], m.Z[b], m.X[c], m.Y[c], m.Z[c]);
}

// links of p after the first `pos` events of S; *first = its first
// incidence at or after pos
template <class MS>
__device__ __forceinline__ short2 mlinks(const MS &m, int p, int pos, int *first) {
  int lo = m.ib[p], hi = m.ib[p + 1];
  const int b0 = lo;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (m.ei[mid] < pos) lo = mid + 1; else hi = mid;
  }
  *first = lo;
  return lo == b0 ? m.LN[p] : m.el[lo - 1];
}

template <class MS>
__device__ __forceinline__ bool mturn_neg_at(const MS &m, int a, int b, int c, double T) {
  const double den = turn_xy(m.X[a], m.Y[a], m.X[b], m.Y[b], m.X[c], m.Y[c]);
  const double tau = mevt(m, a, b, c);
  return tau <= T ? den > 0.0 : den < 0.0;
}

// the sequential core of one segment (see big.cu k_big_sweep); MODE 0
// counts, MODE 1 writes.  Returns false on an exact tie.  Converged: every
// step is one predicated body (touch or bridge), so the segments of a warp
// never serialise on their event kinds; `active` lanes step, the others
// idle through the loop until the whole warp is done.
template <int MODE, class MS>
__device__ bool mini_sweep(MS &m, bool active, int s, int nseg, int seg, int kin, int cap,
                           int *nb_out, int2 *end_uv) {
  const int pos0 = s * seg, pos1 = (pos0 + seg < kin) ? pos0 + seg : kin;
  const double tend = (!active || s == nseg - 1) ? INF : m.st[pos1 - 1];
  double tcur = (!active || s == 0) ? -INF : m.st[pos0 - 1];
  int u = 0, v = 0, cu = 0, cv = 0, eu = 0, ev = 0;
  int up = MINI_NIL, un = MINI_NIL, vp = MINI_NIL, vn = MINI_NIL;
  int pos = pos0;
  if (active) {
    u = m.sst[s].x;
    v = m.sst[s].y;
    const short2 lu = mlinks(m, u, pos, &cu), lw = mlinks(m, v, pos, &cv);
    up = lu.x; un = lu.y; vp = lw.x; vn = lw.y;
    eu = m.ib[u + 1];
    ev = m.ib[v + 1];
  }
  double c2 = INF, c3 = INF, c4 = INF, c5 = INF;
  if (active) {
    c2 = mevt(m, u, un, v);
    c3 = mevt(m, up, u, v);
    c4 = mevt(m, u, v, vn);
    c5 = mevt(m, u, vp, v);
  }
  int nb = 0;
  bool ok = true;
  const int base = (MODE == 1) ? (active ? m.sbn[s] : 0) : s * cap;
  while (__any_sync(0xffffffffu, active)) {
    double tu = INF, tv = INF;
    if (active && cu < eu && m.ei[cu] < pos1) tu = m.st[m.ei[cu]];
    if (active && cv < ev && m.ei[cv] < pos1) tv = m.st[m.ei[cv]];
    double best = INF;
    int which = -1;
    if (tu > tcur && tu < best) { best = tu; which = 0; }
    if (tv > tcur && tv < best) { best = tv; which = 1; }
    if (c2 > tcur && c2 < best) { best = c2; which = 2; }
    if (c3 > tcur && c3 < best) { best = c3; which = 3; }
    if (c4 > tcur && c4 < best) { best = c4; which = 4; }
    if (c5 > tcur && c5 < best) { best = c5; which = 5; }
    if (which < 0 || best > tend) active = false;
    if (active && ((which != 0 && tu == best) || (which != 1 && tv == best) ||
                   (which != 2 && c2 == best) || (which != 3 && c3 == best) ||
                   (which != 4 && c4 == best) || (which != 5 && c5 == best))) {
      ok = false;
      active = false;
    }
    const bool touch = active && which <= 1, bridge = active && which >= 2;
    const bool sideU = which == 0 || which == 2 || which == 3;
    // position after the child events before this time: the touched event
    // itself, or a search of the segment for a bridge event
    if (touch) pos = m.ei[sideU ? cu : cv] + 1;
    {
      int lo = bridge ? pos : 0, hi = bridge ? pos1 : 0;
      while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (m.st[mid] < best) lo = mid + 1; else hi = mid;
      }
      if (bridge) pos = lo;
    }
    // the facet of a bridge move and the foot that moves
    int a = u, b = un, c = v, kind = EV_INS, nfoot = un;
    if (which == 3) { a = up; b = u; c = v; kind = EV_DEL; nfoot = up; }
    if (which == 4) { a = u; b = v; c = vn; kind = EV_DEL; nfoot = vn; }
    if (which == 5) { a = u; b = vp; c = v; kind = EV_INS; nfoot = vp; }
    // links of the point whose links change: the touched foot (the
    // event's links) or the new foot (its list at pos) -- one lookup
    int first = 0;
    short2 l = make_short2(MINI_NIL, MINI_NIL);
    if (touch) l = m.el[sideU ? cu : cv];
    {
      const int q = bridge ? nfoot : 0;
      int lo = bridge ? m.ib[q] : 0, hi = bridge ? m.ib[q + 1] : 0;
      const int b0 = lo;
      while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (m.ei[mid] < pos) lo = mid + 1; else hi = mid;
      }
      first = lo;
      if (bridge) l = lo == b0 ? m.LN[q] : m.el[lo - 1];
    }
    if (bridge) {
      if (sideU) { u = nfoot; cu = first; eu = m.ib[u + 1]; }
      else { v = nfoot; cv = first; ev = m.ib[v + 1]; }
      const typename MS::W bw = wpack<typename MS::W>(a, b, c, kind, 0);
      if (MODE == 1 && base + nb < MS::MINI_B) {
        m.bt[base + nb] = best;
        m.bw[base + nb] = bw;
        m.buv[base + nb] = make_short2(static_cast<short>(u), static_cast<short>(v));
      } else if (MODE == 0 && nb < cap) {
        m.slt[base + nb] = best;
        m.slw[base + nb] = bw;
        m.sluv[base + nb] = make_short2(static_cast<short>(u), static_cast<short>(v));
      }
      ++nb;
    }
    if (touch) {
      if (sideU) ++cu; else ++cv;
    }
    if (active) {
      if (sideU) { up = l.x; un = l.y; } else { vp = l.x; vn = l.y; }
      c2 = mevt(m, u, un, v);
      c3 = mevt(m, up, u, v);
      c4 = mevt(m, u, v, vn);
      c5 = mevt(m, u, vp, v);
      tcur = best;
    }
  }
  *nb_out = nb;
  *end_uv = make_int2(u, v);
  return ok;
}

template <int MINI_T, int MINI_K, int MINI_N>
__global__ void __launch_bounds__(MINI_T) k_mini(Pass2 P, const double *__restrict__ pts,
                                                 long long n, int lv, long long j0, long long j1,
                                                 long long *err, int seglen, long long *spec,
                                                 long long *stamp, unsigned char *gmem,
                                                 size_t gstride, const int *list) {
  if (stamp && blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x == 0) {  // level start (ns)
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    *stamp = static_cast<long long>(t);
  }
  typedef MiniSmem<MINI_T, MINI_K, MINI_N> MS;
  constexpr int MINI_B = MS::MINI_B;
  constexpr int PER = (MINI_K + MINI_T) / MINI_T;  // blocked-scan items per thread
  extern __shared__ __align__(16) unsigned char smem_raw[];
  // the huge variant keeps the job's arrays in a global-memory slot (L1/L2
  // resident; far more than one SM's shared memory), the others in shared
  // memory
  MS &m = *reinterpret_cast<MS *>(
      gmem ? gmem + (static_cast<size_t>(blockIdx.y) * gridDim.x + blockIdx.x) * gstride : smem_raw);
  // the per-point counters / cursors / first output events: in shared
  // memory for the global-memory variant too (its hot atomics), else in the
  // sweep slab's word array
  int *const curp = gmem ? reinterpret_cast<int *>(smem_raw) : m.cur();
  __shared__ int s_scan[MINI_T / 32];  // mini_excl_sum's warp totals
  const int tid = threadIdx.x, T = MINI_T;
  // list mode (a split lane-per-job level's large CTAs): 32 CTAs per list
  // entry (2 * chunk + pass), one per job of the 32-job chunk
  long long j;
  int pass;
  if (list) {
    const int e = static_cast<int>(blockIdx.x >> 5);
    if (e >= *reinterpret_cast<const volatile int *>(list)) return;
    const int v = list[1 + e];
    pass = v & 1;
    j = j0 + static_cast<long long>(v >> 1) * 32 + (blockIdx.x & 31);
  } else {
    j = j0 + lvl_blk();
    pass = lvl_pass();
  }
  if (j >= j1) return;
  // Stop when an earlier launch failed, or (speculative top levels) when a
  // job of an earlier level did not fit, so this level's input is not valid:
  // write nothing, the host redoes from there.  One thread reads the flags
  // and the CTA decides together -- the flags can change while the CTA
  // starts, and a split exit would leave the barriers below short.
  __shared__ int s_stop;
  if (threadIdx.x == 0)
    s_stop = *reinterpret_cast<volatile long long *>(err) != 0 ||
             (spec && *reinterpret_cast<volatile long long *>(spec) != 0);
  __syncthreads();
  if (s_stop) return;
  const GroupBuf in = pass ? P.in1 : P.in0;
  const GroupBuf out = pass ? P.out1 : P.out0;
  const double zs = pass ? -1.0 : 1.0;
  const long long size = 1ll << lv, half = size >> 1;
  const long long L = j << lv, M = L + half;
  const long long R_ = (L + size < n) ? L + size : n;
  const int2 hl = in.hdr[2 * j];
  if (R_ - L <= half) {  // carry (copy_log, parallel.py:107-108)
    for (int p = tid; p < hl.x; p += T) {
      out.lnk[L + p] = in.lnk[L + p];
      out.gid[L + p] = in.gid[L + p];
    }
    for (int e = tid; e < hl.y; e += T) out.ev[2 * L + e] = in.ev[2 * L + e];
    if (tid == 0) out.hdr[j] = hl;
    return;
  }
  const int2 hr = in.hdr[2 * j + 1];
  const int nSL = hl.x, nS = hl.x + hr.x, kL = hl.y, kR = hr.y, kin = kL + kR;
  if (nS > MINI_N || kin > MINI_K) {  // the host routes only fitting levels here ...
    if (tid == 0) {
      if (spec)  // ... or launched it unmeasured: report the level, no fallback
        atomicCAS(reinterpret_cast<unsigned long long *>(spec), 0ull,
                  static_cast<unsigned long long>(lv));
      else
        raise_err(err, E_FASTPATH);
    }
    return;
  }
  if (tid == 0) m.flag = 0;
  MINI_TICK(0);
  // ---- points
  for (int p = tid; p < nS; p += T) {
    const long long src = p < nSL ? L + p : M + (p - nSL);
    int2 l = in.lnk[src];
    if (p >= nSL) {
      if (l.x != NIL) l.x += nSL;
      if (l.y != NIL) l.y += nSL;
    }
    const int g = in.gid[src];
    const P3 c = load_pt(pts, g, zs);
    m.X[p] = c.x;
    m.Y[p] = c.y;
    m.Z[p] = c.z;
    m.LN[p] = make_short2(static_cast<short>(l.x), static_cast<short>(l.y));
    curp[p] = 0;
  }
  MINI_TICK(1);
  // ---- merged child sequence S (merge path, left first on equal times);
  // the child times are staged in shared memory first (the bridge-event
  // arrays are free until the sweeps) so the co-rank searches stay on chip
  const EvP *evL = in.ev + 2 * L, *evR = in.ev + 2 * M;
  double *tL = m.bt, *tR = m.bt + kL;
  for (int d = tid; d < kL; d += T) tL[d] = evL[d].t;
  for (int d = tid; d < kR; d += T) tR[d] = evR[d].t;
  __syncthreads();
  for (int d = tid; d < kin; d += T) {
    int lo = d - kR > 0 ? d - kR : 0, hi = d < kL ? d : kL;
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (tL[mid] <= tR[d - mid - 1]) lo = mid + 1; else hi = mid;
    }
    const int i = lo, jj = d - lo;
    Ev o;
    unsigned side = 0;
    if (i < kL && (jj >= kR || tL[i] <= tR[jj])) {
      o = evL[i];
    } else {
      o = evR[jj];
      o.a += nSL;
      o.b += nSL;
      o.c += nSL;
      side = 1;
    }
    m.st[d] = o.t;
    m.sw[d] = wpack<typename MS::W>(o.a, o.b, o.c, o.kind, static_cast<int>(side));
  }
  __syncthreads();
  MINI_TICK(2);
  // ---- incidence lists: counts, scan, scatter, per-list sort, links after
  for (int d = tid; d < kin; d += T) {
    if (d > 0 && m.st[d] == m.st[d - 1]) m.flag = 1;  // exact tie
    const auto w = m.sw[d];
    atomicAdd(&curp[swa(w)], 1);
    atomicAdd(&curp[swb(w)], 1);
    atomicAdd(&curp[swc(w)], 1);
  }
  __syncthreads();
  {
    const int per = (nS + T) / T;  // blocked scan: `per` consecutive items per thread
    int local[PER];
    int sum = 0;
    for (int q = 0; q < per && q < PER; ++q) {
      const int p = tid * per + q;
      local[q] = p < nS ? curp[p] : 0;
      sum += local[q];
    }
    int off;
    off = mini_excl_sum<MINI_T>(sum, s_scan);
    for (int q = 0; q < per && q < PER; ++q) {
      const int p = tid * per + q;
      if (p <= nS) m.ib[p] = off;
      off += local[q];
    }
  }
  __syncthreads();
  for (int p = tid; p < nS; p += T) curp[p] = m.ib[p];
  __syncthreads();
  // scatter (arbitrary order within a list; the owner kept alongside) ...
  for (int d = tid; d < kin; d += T) {
    const auto w = m.sw[d];
    const int pa = swa(w), pb = swb(w), pc = swc(w);
    int q = atomicAdd(&curp[pa], 1);
    m.eo()[q] = static_cast<short>(d);
    m.el[q].x = static_cast<short>(pa);
    q = atomicAdd(&curp[pb], 1);
    m.eo()[q] = static_cast<short>(d);
    m.el[q].x = static_cast<short>(pb);
    q = atomicAdd(&curp[pc], 1);
    m.eo()[q] = static_cast<short>(d);
    m.el[q].x = static_cast<short>(pc);
  }
  __syncthreads();
  MINI_TICK(3);
  // ... then every entry placed at its rank within its list (event order),
  // all entries in parallel (a list of L entries costs L reads per entry,
  // not a sequential L^2 sort)
  for (int k = tid; k < 3 * kin; k += T) {
    const int p = m.el[k].x, b0 = m.ib[p], b1 = m.ib[p + 1];
    const short x = m.eo()[k];
    int rank = 0;
    for (int q = b0; q < b1; ++q) rank += m.eo()[q] < x;
    m.ei[b0 + rank] = x;
  }
  __syncthreads();
  for (int p = tid; p < nS; p += T) {
    const int b0 = m.ib[p], b1 = m.ib[p + 1];
    short2 l = m.LN[p];
    for (int k = b0; k < b1; ++k) {  // links after each incidence (forward fill)
      const auto w = m.sw[m.ei[k]];
      const bool ins = swk(w) == EV_INS;
      if (swa(w) == p) {
        l.y = static_cast<short>(ins ? swb(w) : swc(w));
      } else if (swc(w) == p) {
        l.x = static_cast<short>(ins ? swb(w) : swa(w));
      } else if (ins) {
        l.x = static_cast<short>(swa(w));
        l.y = static_cast<short>(swc(w));
      }
      m.el[k] = l;
    }
  }
  __syncthreads();
  MINI_TICK(4);
  // ---- segments: start bridges by walks
  int nseg = kin / seglen;
  if (nseg > MS::NSEG) nseg = MS::NSEG;
  if (nseg > T) nseg = T;
  if (nseg < 1) nseg = 1;
  const int seg = (kin + nseg - 1) / nseg > 0 ? (kin + nseg - 1) / nseg : 1;
  nseg = kin > 0 ? (kin + seg - 1) / seg : 1;
  const long long limit = nS + 2;
  if (tid < nseg) {
    const int s = tid;
    int u = nSL - 1, v = nSL;
    long long moves = 0;
    bool bad = false;
    if (s == 0) {  // _find_bridge (_ckernels.pyx:63-83)
      for (;;) {
        const int vn = m.LN[v].y;
        if (vn != NIL && turn_xy(m.X[u], m.Y[u], m.X[v], m.Y[v], m.X[vn], m.Y[vn]) < 0.0) {
          v = vn;
          if (++moves > limit) { bad = true; break; }
          continue;
        }
        const int up = m.LN[u].x;
        if (up != NIL && turn_xy(m.X[up], m.Y[up], m.X[u], m.Y[u], m.X[v], m.Y[v]) < 0.0) {
          u = up;
          if (++moves > limit) { bad = true; break; }
          continue;
        }
        break;
      }
    } else {  // just after the last child event before the segment
      // both candidate moves are evaluated every step (the v-advance wins,
      // as in _find_bridge) so the warp's walks stay converged
      // only the foot that moved needs its links again: one incidence-list
      // search per step, shared by both kinds of move
      const int pos = s * seg;
      const double T0 = m.st[pos - 1];
      int dummy;
      int vn = mlinks(m, v, pos, &dummy).y;
      int up = mlinks(m, u, pos, &dummy).x;
      for (;;) {
        const bool mv = vn != NIL && mturn_neg_at(m, u, v, vn, T0);
        const bool mu = up != NIL && mturn_neg_at(m, up, u, v, T0);
        if (!mv && !mu) break;
        if (mv) v = vn; else u = up;
        const short2 l = mlinks(m, mv ? v : u, pos, &dummy);
        if (mv) vn = l.y; else up = l.x;
        if (++moves > limit) { bad = true; break; }
      }
    }
    if (bad) m.flag = 1;
    m.sst[s] = make_short2(static_cast<short>(u), static_cast<short>(v));
  }
  __syncthreads();
  MINI_TICK(5);
  // ---- segment sweeps (bridge events to per-segment slabs), offsets,
  // compaction; a segment whose slab overflowed is swept again in place
  const int cap = MINI_B / nseg;
  if (tid < ((nseg + 31) & ~31)) {  // whole warps: the sweep votes per warp
    int nb;
    int2 e;
    const bool mine = tid < nseg;
    if (!mini_sweep<0>(m, mine, tid, nseg, seg, kin, cap, &nb, &e)) m.flag = 1;
    if (mine && tid + 1 < nseg && (m.sst[tid + 1].x != e.x || m.sst[tid + 1].y != e.y)) m.flag = 1;
    if (mine) m.sbn[tid] = nb;
  }
  __syncthreads();
  MINI_TICK(10);
  if (tid < 32) {  // exclusive scan of the segments' bridge counts: warp 0,
                   // MINI_S / 32 consecutive segments per lane (a serial loop
                   // here cost ~65 us per level in the global-memory variant)
    constexpr int PL = (MS::NSEG + 31) / 32;
    int c[PL], sum = 0;
#pragma unroll
    for (int q = 0; q < PL; ++q) {
      const int sg = tid * PL + q;
      c[q] = sg < nseg ? m.sbn[sg] : 0;
      sum += c[q];
    }
    int inc = sum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int t = __shfl_up_sync(0xffffffffu, inc, o);
      if (tid >= o) inc += t;
    }
    int o = inc - sum;
#pragma unroll
    for (int q = 0; q < PL; ++q) {
      const int sg = tid * PL + q;
      if (sg < nseg) m.sbn[sg] = o;
      o += c[q];
    }
    if (tid == 31) {
      m.sbn[nseg] = inc;
      m.nb = inc;
      if (inc > MINI_B) m.flag = 1;
    }
  }
  __syncthreads();
  if (m.flag) {  // exact tie, walk/sweep disagreement or capacity: exact engine
    if (tid == 0) raise_err(err, E_FASTPATH);
    return;
  }
  for (int q = tid; q < nseg * cap; q += T) {  // slabs -> compact arrays
    const int sg = q / cap, r = q - sg * cap;
    const int cnt = m.sbn[sg + 1] - m.sbn[sg];
    if (cnt <= cap && r < cnt) {
      m.bt[m.sbn[sg] + r] = m.slt[q];
      m.bw[m.sbn[sg] + r] = m.slw[q];
      m.buv[m.sbn[sg] + r] = m.sluv[q];
    }
  }
  if (tid < ((nseg + 31) & ~31)) {  // overflowed slabs: swept again in place
    int nb;
    int2 e;
    const bool redo = tid < nseg && m.sbn[tid + 1] - m.sbn[tid] > cap;
    if (__any_sync(0xffffffffu, redo)) mini_sweep<1>(m, redo, tid, nseg, seg, kin, cap, &nb, &e);
  }
  __syncthreads();
  MINI_TICK(6);
  const int NB = m.nb;
  const int2 uv0 = make_int2(m.sst[0].x, m.sst[0].y);
  // ---- every child event kept or hidden by the bridge at its time
  auto bridges_before = [&](double t) {
    int lo = 0, hi = NB;
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (m.bt[mid] < t) lo = mid + 1; else hi = mid;
    }
    return lo;
  };
  {
    const int per = (kin + T) / T;
    int local[PER];
    int sum = 0;
    for (int q = 0; q < per && q < PER; ++q) {
      const int d = tid * per + q;
      int keep = 0;
      if (d < kin) {
        const double t = m.st[d];
        const auto w = m.sw[d];
        const int nbf = bridges_before(t);
        if (nbf < NB && m.bt[nbf] == t) m.flag = 1;
        const int u = nbf ? m.buv[nbf - 1].x : uv0.x, v = nbf ? m.buv[nbf - 1].y : uv0.y;
        keep = sws(w) ? (swb(w) > v) : (swb(w) < u);  // _merge_one cases 0/1
      }
      local[q] = keep;
      sum += keep;
    }
    int off;
    off = mini_excl_sum<MINI_T>(sum, s_scan);
    for (int q = 0; q < per && q < PER; ++q) {
      const int d = tid * per + q;
      if (d <= kin) m.cpos()[d] = local[q] ? (off | (1 << 30)) : off;
      off += local[q];
    }
  }
  for (int p = tid; p < nS; p += T) curp[p] = 0x7fffffff;  // first output event
  __syncthreads();
  const int kept = m.cpos()[kin] & ~(1 << 30);
  const int kout = kept + NB;
  if (m.flag || kout > 2 * (R_ - L) - 1) {
    if (tid == 0) raise_err(err, m.flag ? E_FASTPATH : H3D_E_OVERFLOW);
    return;
  }
  MINI_TICK(7);
  // ---- merged log (job-local ids) straight to HBM, first event per point
  EvP *evo = out.ev + 2 * L;
  for (int d = tid; d < kin; d += T) {
    const int cp = m.cpos()[d];
    if (!(cp & (1 << 30))) continue;
    const double t = m.st[d];
    const auto w = m.sw[d];
    const int idx = (cp & ~(1 << 30)) + bridges_before(t);
    Ev o;
    o.t = t;
    o.a = swa(w);
    o.b = swb(w);
    o.c = swc(w);
    o.kind = swk(w);
    evo[idx] = o;
    atomicMin(&curp[o.b], idx);
  }
  for (int i = tid; i < NB; i += T) {
    const double t = m.bt[i];
    int lo = 0, hi = kin;  // first child event after t
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (m.st[mid] < t) lo = mid + 1; else hi = mid;
    }
    const int idx = i + (m.cpos()[lo] & ~(1 << 30));
    const auto w = m.bw[i];
    Ev o;
    o.t = t;
    o.a = swa(w);
    o.b = swb(w);
    o.c = swc(w);
    o.kind = swk(w);
    evo[idx] = o;
    atomicMin(&curp[o.b], idx);
  }
  __syncthreads();
  MINI_TICK(8);
  // ---- start-of-time links + compaction
  {
    const int per = (nS + T) / T;
    int local[PER];
    int sum = 0;
    for (int q = 0; q < per && q < PER; ++q) {
      const int p = tid * per + q;
      int keep = 0;
      if (p < nS) {
        const short2 l = m.LN[p];
        bool chain = p == 0 || p == nSL || (l.x != NIL && m.LN[l.x].y == p);
        chain = chain && (p < nSL ? p <= uv0.x : p >= uv0.y);
        const int f = curp[p];
        keep = chain || f != 0x7fffffff;
        short2 o = make_short2(NIL, NIL);
        if (chain) {
          o = l;
          if (p == uv0.x) o.y = static_cast<short>(uv0.y);
          if (p == uv0.y) o.x = static_cast<short>(uv0.x);
        } else if (keep) {
          const Ev e = evo[f];
          o = make_short2(static_cast<short>(e.a), static_cast<short>(e.c));
        }
        m.KL()[p] = o;
      }
      local[q] = keep;
      sum += keep;
    }
    int off;
    off = mini_excl_sum<MINI_T>(sum, s_scan);
    for (int q = 0; q < per && q < PER; ++q) {
      const int p = tid * per + q;
      if (p <= nS) m.nid()[p] = local[q] ? off : -1;
      off += local[q];
    }
    if (tid == T - 1) m.kept = off;  // kept points
  }
  __syncthreads();
  bool bad = false;
  for (int p = tid; p < nS; p += T) {
    const int id = m.nid()[p];
    if (id < 0) continue;
    const short2 l = m.KL()[p];
    int2 o;
    o.x = l.x == NIL ? NIL : m.nid()[l.x];
    o.y = l.y == NIL ? NIL : m.nid()[l.y];
    bad |= (l.x != NIL && o.x < 0) | (l.y != NIL && o.y < 0);
    out.lnk[L + id] = o;
    out.gid[L + id] = in.gid[p < nSL ? L + p : M + (p - nSL)];  // the gid, re-read (not kept in smem)
  }
  for (int e = tid; e < kout; e += T) {
    Ev o = evo[e];
    o.a = m.nid()[o.a];
    o.b = m.nid()[o.b];
    o.c = m.nid()[o.c];
    bad |= (o.a < 0) | (o.b < 0) | (o.c < 0);
    evo[e] = o;
  }
  if (bad) raise_err(err, E_FASTPATH);
  MINI_TICK(9);
  if (tid == 0) out.hdr[j] = make_int2(m.kept, kout);
}

template <int T, int K, int N>
static long long launch_mini(const Pass2 &P, const double *pts, long long n, int lv, long long j0,
                             long long j1, long long *err, cudaStream_t s, long long *spec,
                             long long *stamp, void *gscratch = nullptr, size_t gbytes = 0,
                             const int *list = nullptr, int list_grid = 0) {
  static bool attr[64] = {};  // the attribute is per device
  int dev_id = 0;
  cudaGetDevice(&dev_id);
  if (dev_id < 0 || dev_id >= 64) return H3D_E_ARG;
  const size_t bytes = sizeof(MiniSmem<T, K, N>);
  const size_t stride = (bytes + 255) & ~size_t(255);
  if (gscratch) {  // global-memory slots, one per CTA
    const size_t ctas = list ? 32 * static_cast<size_t>(list_grid) : 2 * static_cast<size_t>(j1 - j0);
    if (ctas * stride > gbytes) return list ? H3D_E_ARG : 1;  // a list launch was sized to fit
  } else if (!attr[dev_id]) {
    if (h3d_check(cudaFuncSetAttribute(k_mini<T, K, N>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(bytes))))
      return H3D_E_CUDA;
    attr[dev_id] = true;
  }
  h3d_count_launches(1);
  const dim3 grid = list ? dim3(32u * static_cast<unsigned>(list_grid), 1)
                         : lvl_grid(static_cast<unsigned>(j1 - j0), g_interleave != 0);
  k_mini<T, K, N><<<grid, T, gscratch ? N * sizeof(int) : bytes, s>>>(
      P, pts, n, lv, j0, j1, err, g_mini_seglen, spec, stamp, static_cast<unsigned char *>(gscratch),
      stride, list);
  return h3d_check(cudaGetLastError()) ? H3D_E_CUDA : 0;
}

int g_mini_seglen = 3;  // child events per time segment (H3D_MINI_SEG / h3d_tune)

size_t mini_huge_stride() {
  return (sizeof(MiniSmem<1024, kMiniHugeEvents, kMiniHugePoints>) + 255) & ~size_t(255);
}

// list mode (list != nullptr): the jobs of the 32-job chunks in the list
// (count at list[0]; at most list_grid entries) -- shared-memory variants
long long mini_level(const Pass2 &P, const double *pts, long long n, int lv, long long j0,
                     long long j1, long long *err, cudaStream_t s, int variant, long long *spec,
                     long long *stamp, void *gscratch, size_t gbytes, const int *list, int list_grid) {
  if (list) {
    if (variant == 0) return launch_mini<256, 512, 256>(P, pts, n, lv, j0, j1, err, s, spec, stamp, nullptr, 0, list, list_grid);
    if (variant == 4)
      return launch_mini<256, kMiniMedEvents, kMiniMedPoints>(P, pts, n, lv, j0, j1, err, s, spec, stamp, nullptr,
                                                              0, list, list_grid);
    if (variant == 5)
      return launch_mini<512, kMiniL2Events, kMiniL2Points>(P, pts, n, lv, j0, j1, err, s, spec, stamp, nullptr, 0,
                                                            list, list_grid);
    if (variant == 1)
      return launch_mini<1024, 2048, 1024>(P, pts, n, lv, j0, j1, err, s, spec, stamp, nullptr, 0, list, list_grid);
    if (variant == 6)
      return launch_mini<1024, kMiniXlEvents, kMiniXlPoints>(P, pts, n, lv, j0, j1, err, s, spec, stamp, nullptr, 0,
                                                             list, list_grid);
    if (variant == 3)
      return launch_mini<1024, kMiniHugeEvents, kMiniHugePoints>(P, pts, n, lv, j0, j1, err, s, spec, stamp,
                                                                 gscratch, gbytes, list, list_grid);
    return H3D_E_ARG;
  }
  if (variant == 2) return launch_mini<128, 320, 192>(P, pts, n, lv, j0, j1, err, s, spec, stamp);
  if (variant == 0) return launch_mini<256, 512, 256>(P, pts, n, lv, j0, j1, err, s, spec, stamp);
  // medium (50 KB: 4 CTAs per SM) and large2 (100 KB: 2 per SM) for levels of
  // many mid-size jobs (sphere-like clouds keep every point)
  if (variant == 4)
    return launch_mini<256, kMiniMedEvents, kMiniMedPoints>(P, pts, n, lv, j0, j1, err, s, spec, stamp);
  if (variant == 5)
    return launch_mini<512, kMiniL2Events, kMiniL2Points>(P, pts, n, lv, j0, j1, err, s, spec, stamp);
  // xl: a little past the large variant (64-bit facet words), one CTA per SM
  if (variant == 6)
    return launch_mini<1024, kMiniXlEvents, kMiniXlPoints>(P, pts, n, lv, j0, j1, err, s, spec, stamp);
  if (variant == 3)
    return launch_mini<1024, kMiniHugeEvents, kMiniHugePoints>(P, pts, n, lv, j0, j1, err, s, spec, stamp,
                                                               gscratch, gbytes);
  return launch_mini<1024, 2048, 1024>(P, pts, n, lv, j0, j1, err, s, spec, stamp);
}

}  // namespace h3d

#ifdef H3D_MINI_PROF
extern "C" void h3d_mini_prof_read(long long *host) {
  cudaMemcpyFromSymbol(host, h3d::g_mini_prof, sizeof(long long) * 64 * 16);
}
#endif
