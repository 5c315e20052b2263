// presort.cu -- device x-presort, tie perturbation, degeneracy scan, epilogue.
//
// Restates on the GPU the host numpy steps around the engine:
//   _sort_and_perturb / perturb_ties / _lex_order  pkg/src/hull3d/api.py:61-110
//   _scan_degenerate                               pkg/src/hull3d/api.py:113-147
//   orientation, remap, np.unique                  pkg/src/hull3d/api.py:252-266
//
// Sorting: stable LSD radix sort (prims.cuh, hand-written onesweep) of
// order-preserving u64 keys
// of the fp64 coordinates with the row index as payload.  -0.0 is folded
// onto +0.0 first so that the two compare equal, as they do under numpy's
// comparisons.  Stability + index payload reproduces argsort(kind="stable")
// and np.lexsort((z, y, x)) exactly (three stable passes z, y, x).

#include "h3d_device.cuh"
#include "h3d_host.h"
#include "prims.cuh"

namespace h3d {

__device__ __forceinline__ unsigned long long order_key(double d) {
  if (d == 0.0) d = 0.0;  // fold -0.0 onto +0.0
  const unsigned long long b = static_cast<unsigned long long>(__double_as_longlong(d));
  return (b >> 63) ? ~b : (b | (1ull << 63));
}

// keys of column `col` of pts gathered through perm (perm == nullptr: identity)
__global__ void k_keys(const double *__restrict__ pts, const int *__restrict__ perm, int col,
                       long long n, unsigned long long *keys, int *vals) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    const long long r = perm ? perm[i] : i;
    keys[i] = order_key(pts[3 * r + col]);
    vals[i] = static_cast<int>(r);
  }
}

// flag any adjacent equal key (sorted keys are non-decreasing)
__global__ void k_adjacent_tie(const unsigned long long *__restrict__ keys, long long n,
                               int *flag) {
  for (long long i = 1 + blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    if (keys[i] == keys[i - 1]) {
      *flag = 1;
      return;
    }
  }
}

// ---- fast stable argsort of x: 32-bit monotone fixed-point keys (4 radix
// passes instead of 8), then the rare runs of equal 32-bit keys re-sorted by
// the exact 64-bit order key (stable: equal x keep index order).  Any run
// longer than RUN_MAX sends the sort to the 64-bit path.
constexpr int RUN_MAX = 64;

__device__ __forceinline__ double key_to_double(unsigned long long k) {
  const unsigned long long b = (k >> 63) ? (k & ~(1ull << 63)) : ~k;
  return __longlong_as_double(static_cast<long long>(b));
}

__device__ __forceinline__ unsigned fixed_key(double x, double lo, double sc) {
  if (x == 0.0) x = 0.0;
  double f = __dmul_rn(__dsub_rn(x, lo), sc);  // monotone in x
  if (!(f >= 0.0)) f = 0.0;
  if (f > 4294967295.0) f = 4294967295.0;
  return static_cast<unsigned>(f);
}

__global__ void k_keys32(const double *__restrict__ pts, long long n,
                         const unsigned long long *__restrict__ mm, unsigned *keys, int *vals) {
  const double lo = key_to_double(mm[0]), hi = key_to_double(mm[1]);
  const double span = __dsub_rn(hi, lo);
  const double sc = span > 0.0 ? __ddiv_rn(4294967295.0, span) : 0.0;
  const long long stride = (long long)gridDim.x * blockDim.x;
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  for (; i + 3 * stride < n; i += 4 * stride) {  // four loads in flight
    double x[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) x[q] = pts[3 * (i + q * stride)];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      keys[i + q * stride] = fixed_key(x[q], lo, sc);
      if (vals) vals[i + q * stride] = static_cast<int>(i + q * stride);
    }
  }
  for (; i < n; i += stride) {
    keys[i] = fixed_key(pts[3 * i], lo, sc);
    if (vals) vals[i] = static_cast<int>(i);
  }
}

// k_keys32 with the radix sort's four 8-bit digit histograms accumulated on
// the way (block histograms in shared memory, one atomic per bin and block):
// the sort then skips its histogram pass over the keys
__global__ void __launch_bounds__(256) k_keys32_rshist(const double *__restrict__ pts, long long n,
                                                      const unsigned long long *__restrict__ mm, unsigned *keys,
                                                      unsigned *hist) {
  __shared__ unsigned sh[4][256];
  for (int i = threadIdx.x; i < 4 * 256; i += blockDim.x) (&sh[0][0])[i] = 0;
  __syncthreads();
  const double lo = key_to_double(mm[0]), hi = key_to_double(mm[1]);
  const double span = __dsub_rn(hi, lo);
  const double sc = span > 0.0 ? __ddiv_rn(4294967295.0, span) : 0.0;
  const long long stride = (long long)gridDim.x * blockDim.x;
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  for (; i + 3 * stride < n; i += 4 * stride) {  // four loads in flight
    double x[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) x[q] = pts[3 * (i + q * stride)];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const unsigned k = fixed_key(x[q], lo, sc);
      keys[i + q * stride] = k;
#pragma unroll
      for (int p = 0; p < 4; ++p) atomicAdd(&sh[p][(k >> (8 * p)) & 255u], 1u);
    }
  }
  for (; i < n; i += stride) {
    const unsigned k = fixed_key(pts[3 * i], lo, sc);
    keys[i] = k;
#pragma unroll
    for (int p = 0; p < 4; ++p) atomicAdd(&sh[p][(k >> (8 * p)) & 255u], 1u);
  }
  __syncthreads();
  for (int i2 = threadIdx.x; i2 < 4 * 256; i2 += blockDim.x) {
    const unsigned c = (&sh[0][0])[i2];
    if (c) atomicAdd(hist + i2, c);
  }
}

// runs of equal 32-bit keys: insertion sort by (64-bit order key, index)
__global__ void k_tiefix(const double *__restrict__ pts, const unsigned *__restrict__ k32,
                         int *vals, long long n, int *flag) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i + 1 < n;
       i += (long long)gridDim.x * blockDim.x) {
    const unsigned k = k32[i];
    if (k32[i + 1] != k || (i > 0 && k32[i - 1] == k)) continue;  // i: head of a run
    long long e = i + 1;
    while (e < n && k32[e] == k && e - i <= RUN_MAX) ++e;
    if (e - i > RUN_MAX) {
      *flag = 1;  // degenerate distribution: use the 64-bit sort
      continue;
    }
    for (long long a = i + 1; a < e; ++a) {
      const int va = vals[a];
      const unsigned long long ka = order_key(pts[3ll * va]);
      long long b = a - 1;
      while (b >= i) {
        const int vb = vals[b];
        const unsigned long long kb = order_key(pts[3ll * vb]);
        if (kb < ka || (kb == ka && vb < va)) break;
        vals[b + 1] = vb;
        --b;
      }
      vals[b + 1] = va;
    }
  }
}

// one pass over the input: any non-finite coordinate (api.py:192-193), the
// x range (order keys) for the fixed-point sort keys, and max |coordinate|
// (the degeneracy scan's scale, api.py:122; valid while no tie perturbs x)
__global__ void k_scan_input(const double *__restrict__ pts, long long n, int *nonfinite,
                             unsigned long long *mm, unsigned long long *absmax_bits) {
  unsigned long long lo = ~0ull, hi = 0ull;
  double amax = 0.0;
  bool bad = false;
  // the (n,3) rows as a flat array read in 16-byte pairs; element e is an
  // x coordinate iff e % 3 == 0
  const long long m = 3 * n;
  // (a row-offset view is only 8-byte aligned: one element per step then)
  const bool vec = (reinterpret_cast<unsigned long long>(pts) & 15ull) == 0;
  const long long pairs = vec ? (m >> 1) : 0;
  const double2 *p2 = reinterpret_cast<const double2 *>(pts);
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; !vec && e < m;
       e += (long long)gridDim.x * blockDim.x) {
    const double d = pts[e];
    bad |= !isfinite(d);
    amax = fmax(amax, fabs(d));
    if (e % 3 == 0) {
      const unsigned long long k = order_key(d);
      lo = k < lo ? k : lo;
      hi = k > hi ? k : hi;
    }
  }
  const long long j0 = blockIdx.x * (long long)blockDim.x + threadIdx.x,
                  stride = (long long)gridDim.x * blockDim.x;
  const int inc = static_cast<int>((2 * stride) % 3);
  int r0 = static_cast<int>((2 * j0) % 3);  // phase of element 2j, kept incrementally
  auto visit = [&](double d, int r) {
    bad |= !isfinite(d);
    amax = fmax(amax, fabs(d));
    if (r == 0) {
      const unsigned long long k = order_key(d);
      lo = k < lo ? k : lo;
      hi = k > hi ? k : hi;
    }
  };
  auto step = [&](int &r) {
    r += inc;
    if (r >= 3) r -= 3;
  };
  long long j = j0;
  if (vec) {
    // four independent 16-byte loads in flight per thread
    for (; j + 3 * stride < pairs; j += 4 * stride) {
      double2 d[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) d[q] = p2[j + q * stride];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int r1 = r0 == 2 ? 0 : r0 + 1;
        visit(d[q].x, r0);
        visit(d[q].y, r1);
        step(r0);
      }
    }
    for (; j < pairs; j += stride) {
      const double2 d = p2[j];
      visit(d.x, r0);
      visit(d.y, r0 == 2 ? 0 : r0 + 1);
      step(r0);
    }
    if (j == pairs && (m & 1)) visit(pts[m - 1], r0);
  }
  for (int o = 16; o; o >>= 1) {
    const unsigned long long a = __shfl_xor_sync(0xffffffffu, lo, o),
                             b = __shfl_xor_sync(0xffffffffu, hi, o);
    lo = a < lo ? a : lo;
    hi = b > hi ? b : hi;
    amax = fmax(amax, __shfl_xor_sync(0xffffffffu, amax, o));
  }
  bad = __any_sync(0xffffffffu, bad);
  // block reduction, then one atomic of each kind per block
  __shared__ unsigned long long s_lo[32], s_hi[32], s_am[32];
  __shared__ int s_bad;
  const int w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  if (threadIdx.x == 0) s_bad = 0;
  __syncthreads();
  if ((threadIdx.x & 31) == 0) {
    s_lo[w] = lo;
    s_hi[w] = hi;
    s_am[w] = static_cast<unsigned long long>(__double_as_longlong(amax));
    if (bad) s_bad = 1;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long L = s_lo[0], H = s_hi[0], A = s_am[0];
    for (int i = 1; i < nw; ++i) {
      L = s_lo[i] < L ? s_lo[i] : L;
      H = s_hi[i] > H ? s_hi[i] : H;
      A = s_am[i] > A ? s_am[i] : A;  // non-negative doubles order as bits
    }
    atomicMin(mm, L);
    atomicMax(mm + 1, H);
    atomicMax(absmax_bits, A);
    if (s_bad) *nonfinite = 1;
  }
}

__global__ void k_gather_rows(const double *__restrict__ pts, const int *__restrict__ perm,
                              long long n, double *out, long long *order,
                              const int *__restrict__ outer, int *tie = nullptr) {
  // random 24-byte rows: bound by DRAM efficiency of scattered reads (more
  // rows in flight per thread measured no faster)
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    const long long r = perm[i];
    // adjacent equal x in the sorted order (the reference's tie test)
    if (tie && i > 0 && pts[3 * r] == pts[3ll * perm[i - 1]]) *tie = 1;
    out[3 * i] = pts[3 * r];
    out[3 * i + 1] = pts[3 * r + 1];
    out[3 * i + 2] = pts[3 * r + 2];
    if (order) order[i] = outer ? outer[r] : r;
  }
}

// The optimistic presort's gather with the epilogue's centroid column sums
// folded in: the grid and the per-thread row order of k_colsum (kColsumBlocks
// x 256 threads, grid-stride over the sorted rows) and the same block
// reduction, so the partial sums -- and the centroid -- are bit for bit
// k_colsum's; four rows in flight per thread, added in row order.
__global__ void __launch_bounds__(256) k_gather_rows_colsum(const double *__restrict__ pts,
                                                           const int *__restrict__ perm, long long n,
                                                           double *out, long long *order, int *tie,
                                                           double *partial) {
  const long long stride = (long long)gridDim.x * blockDim.x;
  double s0 = 0, s1 = 0, s2 = 0;
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  for (; i < n; i += 4 * stride) {
    long long r[4];
    double x[4], y[4], z[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) r[q] = i + q * stride < n ? perm[i + q * stride] : 0;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      if (i + q * stride < n) {
        x[q] = pts[3 * r[q]];
        y[q] = pts[3 * r[q] + 1];
        z[q] = pts[3 * r[q] + 2];
      }
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const long long k = i + q * stride;
      if (k >= n) break;
      // adjacent equal x in the sorted order (the reference's tie test)
      if (k > 0 && x[q] == pts[3ll * perm[k - 1]]) *tie = 1;
      out[3 * k] = x[q];
      out[3 * k + 1] = y[q];
      out[3 * k + 2] = z[q];
      order[k] = r[q];
      s0 += x[q];
      s1 += y[q];
      s2 += z[q];
    }
  }
  __shared__ double s_warp[8];
  const prim::OpSum add;
  double t = prim::block_reduce256(s0, s_warp, add);
  if (threadIdx.x == 0) partial[3 * blockIdx.x] = t;
  t = prim::block_reduce256(s1, s_warp, add);
  if (threadIdx.x == 0) partial[3 * blockIdx.x + 1] = t;
  t = prim::block_reduce256(s2, s_warp, add);
  if (threadIdx.x == 0) partial[3 * blockIdx.x + 2] = t;
}

// ---- sharded presort (multi-GPU): one rank's window [q0, p1) of the global
// stable x order without sorting the other ranks' points.  The 32-bit keys of
// every point are computed; a 3-pass radix select (11+11+10 bits) finds the
// key K_b of the element at each window boundary b and its rank inside the
// run of equal keys; elements strictly between the two boundary keys are
// compacted, the (short) boundary runs are ranked by (64-bit order key,
// index) exactly as k_tiefix orders them, and only the window is sorted.
struct SelState {
  unsigned pre[2];   // key prefix found so far, per boundary
  long long rem[2];  // rank inside the prefix bucket still to skip
  long long b[2];    // boundary positions (-1: none)
  int count, nrun, bad, pad;
};

constexpr int kSelRunCap = 2 * RUN_MAX;

__device__ __forceinline__ int sel_shift(int pass) { return pass == 0 ? 21 : (pass == 1 ? 10 : 0); }
__device__ __forceinline__ int sel_bits(int pass) { return pass == 2 ? 10 : 11; }

__global__ void k_sel_hist(const unsigned *__restrict__ k32, long long n,
                           const SelState *__restrict__ st, int pass, unsigned *hist) {
  __shared__ unsigned h[2][2048];
  for (int i = threadIdx.x; i < 4096; i += blockDim.x) (&h[0][0])[i] = 0;
  __syncthreads();
  const int sh = sel_shift(pass), hi = sh + sel_bits(pass);
  const unsigned mask = (1u << sel_bits(pass)) - 1u;
  const bool h0 = st->b[0] >= 0, h1 = st->b[1] >= 0;
  const unsigned p0 = st->pre[0], p1 = st->pre[1];
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    const unsigned k = k32[i];
    const unsigned top = hi >= 32 ? 0u : (k >> hi);
    const unsigned d = (k >> sh) & mask;
    if (h0 && top == p0) atomicAdd(&h[0][d], 1u);
    if (h1 && top == p1) atomicAdd(&h[1][d], 1u);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < 4096; i += blockDim.x) {
    const unsigned v = (&h[0][0])[i];
    if (v) atomicAdd(hist + i, v);
  }
}

// one block of 256 threads, 8 bins each: the bucket holding each boundary's rank
__global__ void k_sel_pick(unsigned *hist, SelState *st, int pass) {
  __shared__ long long s_warp[8];
  const int bins = 1 << sel_bits(pass);
  const int t = threadIdx.x;
  for (int b = 0; b < 2; ++b) {
    const bool has = st->b[b] >= 0;
    const long long rem = st->rem[b];
    long long c[8], tot = 0;
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      c[q] = 8 * t + q < bins ? hist[(pass == 0 ? 0 : 2048 * b) + 8 * t + q] : 0;
      tot += c[q];
    }
    long long before = prim::block_excl_sum256(tot, s_warp);
    if (has && rem >= before && rem < before + tot) {
      int d = 0;
      while (rem >= before + c[d]) before += c[d++];
      st->pre[b] = (st->pre[b] << sel_bits(pass)) | static_cast<unsigned>(8 * t + d);
      st->rem[b] = rem - before;
    }
    __syncthreads();
  }
  for (int i = t; i < 4096; i += blockDim.x) hist[i] = 0;
}

// block-aggregated compaction: 8 keys per thread, one atomic per block tile
constexpr int kSelItems = 8;

__global__ void __launch_bounds__(256) k_sel_compact(const unsigned *__restrict__ k32, long long n,
                                                     SelState *st, int *out, int *runs, long long cap) {
  __shared__ int s_warp[8];
  __shared__ int s_base;
  const bool h0 = st->b[0] >= 0, h1 = st->b[1] >= 0;
  const unsigned K0 = st->pre[0], K1 = st->pre[1];
  const long long tile = 256ll * kSelItems;
  for (long long base = blockIdx.x * tile; base < n; base += (long long)gridDim.x * tile) {
    const long long i0 = base + (long long)threadIdx.x * kSelItems;
    unsigned k[kSelItems];
    if (i0 + kSelItems <= n) {
      const uint4 a = *reinterpret_cast<const uint4 *>(k32 + i0);
      const uint4 b = *reinterpret_cast<const uint4 *>(k32 + i0 + 4);
      k[0] = a.x; k[1] = a.y; k[2] = a.z; k[3] = a.w;
      k[4] = b.x; k[5] = b.y; k[6] = b.z; k[7] = b.w;
    } else {
#pragma unroll
      for (int q = 0; q < kSelItems; ++q) k[q] = i0 + q < n ? k32[i0 + q] : 0u;
    }
    int cnt = 0;
    unsigned inm = 0;
#pragma unroll
    for (int q = 0; q < kSelItems; ++q) {
      if (i0 + q >= n) continue;
      const bool in = (!h0 || k[q] > K0) && (!h1 || k[q] < K1);
      const bool run = (h0 && k[q] == K0) || (h1 && k[q] == K1);
      inm |= (in ? 1u : 0u) << q;
      cnt += in;
      if (run) {
        const int r = atomicAdd(&st->nrun, 1);
        if (r < kSelRunCap) runs[r] = static_cast<int>(i0 + q);
        else st->bad = 1;
      }
    }
    int total;
    int off = prim::block_excl_sum256(cnt, s_warp, &total);
    if (threadIdx.x == 0) s_base = total ? atomicAdd(&st->count, total) : 0;
    __syncthreads();
    off += s_base;
    // a bad selection may find more than the window holds: never write past
    // the window buffer (the count check in k_sel_keys rejects it)
#pragma unroll
    for (int q = 0; q < kSelItems; ++q)
      if (inm >> q & 1u) {
        if (off < cap) out[off] = static_cast<int>(i0 + q);
        ++off;
      }
    __syncthreads();
  }
}

// k_keys32 fused with the first select pass (top 11 bits, every key)
__global__ void k_keys32_hist(const double *__restrict__ pts, long long n,
                              const unsigned long long *__restrict__ mm, unsigned *keys,
                              unsigned *hist) {
  __shared__ unsigned h[2048];
  for (int i = threadIdx.x; i < 2048; i += blockDim.x) h[i] = 0;
  __syncthreads();
  const double lo = key_to_double(mm[0]), hi = key_to_double(mm[1]);
  const double span = __dsub_rn(hi, lo);
  const double sc = span > 0.0 ? __ddiv_rn(4294967295.0, span) : 0.0;
  const long long stride = (long long)gridDim.x * blockDim.x;
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  for (; i + 3 * stride < n; i += 4 * stride) {
    double x[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) x[q] = pts[3 * (i + q * stride)];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const unsigned k = fixed_key(x[q], lo, sc);  // the same key as k_keys32
      keys[i + q * stride] = k;
      atomicAdd(&h[k >> 21], 1u);
    }
  }
  for (; i < n; i += stride) {
    const unsigned k = fixed_key(pts[3 * i], lo, sc);
    keys[i] = k;
    atomicAdd(&h[k >> 21], 1u);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < 2048; i += blockDim.x)
    if (h[i]) atomicAdd(hist + i, h[i]);
}

// boundary runs: global position = (b - rem_b) + rank inside the run
__global__ void k_sel_runs(const double *__restrict__ pts, const unsigned *__restrict__ k32,
                           SelState *st, const int *__restrict__ runs, int *out, long long cap) {
  const int nr = min(st->nrun, kSelRunCap);
  const long long q0 = st->b[0] >= 0 ? st->b[0] : 0;
  for (int e = threadIdx.x; e < nr; e += blockDim.x) {
    const int ve = runs[e];
    const unsigned k = k32[ve];
    const unsigned long long ke = order_key(pts[3ll * ve]);
    long long r = 0;
    for (int f = 0; f < nr; ++f) {
      const int vf = runs[f];
      if (vf == ve || k32[vf] != k) continue;
      const unsigned long long kf = order_key(pts[3ll * vf]);
      r += (kf < ke || (kf == ke && vf < ve));
    }
    const int b = (st->b[0] >= 0 && k == st->pre[0]) ? 0 : 1;
    const long long pos = st->b[b] - st->rem[b] + r;
    const long long p1 = st->b[1] >= 0 ? st->b[1] : 0x7fffffffffffffffll;
    if (pos >= q0 && pos < p1) {
      const int at = atomicAdd(&st->count, 1);
      if (at < cap) out[at] = ve;
    }
  }
}

// window keys; a count other than the window size flags the selection
__global__ void k_sel_keys(const unsigned *__restrict__ k32, SelState *st, int *idx,
                           unsigned *keys, long long m) {
  const long long cnt = st->count;
  if (blockIdx.x == 0 && threadIdx.x == 0 && cnt != m) st->bad = 1;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < m;
       i += (long long)gridDim.x * blockDim.x) {
    if (i >= cnt) idx[i] = 0;
    keys[i] = k32[idx[i]];
  }
}

// run start index per row of lex-sorted x (0 where the row continues a run)
// The lexsort of the tie path (api.py:86-87, np.lexsort((z, y, x))) from the
// stable x order already at hand: runs of equal x are contiguous and hold
// the same points in both orders, so only each run is re-ordered, by
// (y, z, index) -- an insertion sort per run (runs longer than RUN_MAX set
// *flag: the caller does the three full stable passes instead).
__global__ void k_lexruns(const double *__restrict__ pts, int *perm, long long n, int *flag) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i + 1 < n;
       i += (long long)gridDim.x * blockDim.x) {
    const double x = pts[3ll * perm[i]];
    if (pts[3ll * perm[i + 1]] != x || (i > 0 && pts[3ll * perm[i - 1]] == x)) continue;  // i: run head
    flag[1] = 1;  // an x tie
    long long e = i + 1;
    while (e < n && pts[3ll * perm[e]] == x && e - i <= RUN_MAX) ++e;
    if (e - i > RUN_MAX) {
      *flag = 1;
      continue;
    }
    for (long long a = i + 1; a < e; ++a) {
      const int va = perm[a];
      const unsigned long long ya = order_key(pts[3ll * va + 1]), za = order_key(pts[3ll * va + 2]);
      long long b = a - 1;
      while (b >= i) {
        const int vb = perm[b];
        const unsigned long long yb = order_key(pts[3ll * vb + 1]), zb = order_key(pts[3ll * vb + 2]);
        if (yb < ya || (yb == ya && (zb < za || (zb == za && vb < va)))) break;
        perm[b + 1] = vb;
        --b;
      }
      perm[b + 1] = va;
    }
  }
}

// After the perturbation: is x still non-decreasing along the lexsorted
// rows (then the reference's stable re-sort, api.py:102-104, is the
// identity)?  flag[3] = a descent (re-sort needed), flag[0] = equal
// neighbours (the ties survived: DegenerateInputError).
__global__ void k_perturbed_order(const double *__restrict__ w, long long n, int *flag) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i + 1 < n;
       i += (long long)gridDim.x * blockDim.x) {
    const double a = w[3 * i], b = w[3 * (i + 1)];
    if (a > b) flag[3] = 1;
    if (a == b) flag[0] = 1;
  }
}

__global__ void k_perm_to_order(const int *__restrict__ perm, long long n, long long *order) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    order[i] = perm[i];
}

__global__ void k_run_heads(const double *__restrict__ w, long long n, long long *head) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    head[i] = (i == 0 || w[3 * i] != w[3 * (i - 1)]) ? i : 0;
}

// perturb_ties (api.py:61-83): x[s+r] = x[s] + r * 16eps*max(1,|x[s]|)
__global__ void k_perturb(double *w, const long long *__restrict__ head, long long n) {
  const double tie_eps = 16.0 * 2.220446049250313080847263336181640625e-16;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    const long long s = head[i];
    const long long rank = i - s;
    if (rank > 0) {
      const double base = w[3 * s];
      const double ab = fabs(base);
      const double step = __dmul_rn(tie_eps, ab > 1.0 ? ab : 1.0);
      w[3 * i] = __dadd_rn(base, __dmul_rn(static_cast<double>(rank), step));
    }
  }
}

// ---------------------------------------------------------- degeneracy scan
// max |coord| (non-negative doubles order like their bit patterns)
__global__ void k_absmax(const double *__restrict__ p, long long m, unsigned long long *out) {
  double best = 0.0;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < m;
       i += (long long)gridDim.x * blockDim.x)
    best = fmax(best, fabs(p[i]));
  __shared__ double s_warp[8];
  const double b = prim::block_reduce256(best, s_warp, [](double a, double c) { return fmax(a, c); });
  if (threadIdx.x == 0) atomicMax(out, static_cast<unsigned long long>(__double_as_longlong(b)));
}

struct ScanState {
  unsigned long long scale_bits;
  long long i, j, k;  // first hits (LLONG_MAX = none)
};

__device__ __forceinline__ double norm3(double a, double b, double c) {
  return sqrt(__dadd_rn(__dadd_rn(__dmul_rn(a, a), __dmul_rn(b, b)), __dmul_rn(c, c)));
}

__device__ __forceinline__ void cross3(double a0, double a1, double a2, double b0, double b1,
                                       double b2, double *c) {
  c[0] = __dsub_rn(__dmul_rn(a1, b2), __dmul_rn(a2, b1));
  c[1] = __dsub_rn(__dmul_rn(a2, b0), __dmul_rn(a0, b2));
  c[2] = __dsub_rn(__dmul_rn(a0, b1), __dmul_rn(a1, b0));
}

// stage 0: first i >= 1 with |p_i - p0| > tol*scale
// stage 1: first j >= 1 with |cross(p_i - p0, p_j - p0)| > tol*scale*scale
// stage 2: first k >= 1 with |(p_k - p0) . normal| > tol*scale*|normal|
__global__ void k_degenerate(const double *__restrict__ P, long long n, ScanState *st,
                             int stage, long long r0, long long r1) {
  const double tol = 1e-9;
  double scale = __longlong_as_double(static_cast<long long>(st->scale_bits));
  if (scale < 1e-30) scale = 1e-30;
  const double x0 = P[0], y0 = P[1], z0 = P[2];
  double di[3] = {0, 0, 0}, nrm[3] = {0, 0, 0}, thr;
  const long long none = 0x7fffffffffffffffll;
  if ((stage >= 1 && st->i == none) || (stage == 2 && st->j == none)) return;
  if (stage >= 1) {
    const long long i = st->i;
    di[0] = __dsub_rn(P[3 * i], x0);
    di[1] = __dsub_rn(P[3 * i + 1], y0);
    di[2] = __dsub_rn(P[3 * i + 2], z0);
  }
  if (stage == 0) {
    thr = __dmul_rn(tol, scale);
  } else if (stage == 1) {
    thr = __dmul_rn(__dmul_rn(tol, scale), scale);
  } else {
    const long long j = st->j;
    cross3(di[0], di[1], di[2], __dsub_rn(P[3 * j], x0), __dsub_rn(P[3 * j + 1], y0),
           __dsub_rn(P[3 * j + 2], z0), nrm);
    thr = __dmul_rn(__dmul_rn(tol, scale), norm3(nrm[0], nrm[1], nrm[2]));
  }
  long long *slot = stage == 0 ? &st->i : (stage == 1 ? &st->j : &st->k);
  // rows [r0, r1): a later range only matters when no earlier row hit
  if (*reinterpret_cast<volatile long long *>(slot) != none) return;
  if (r1 > n) r1 = n;
  for (long long r = r0 + blockIdx.x * (long long)blockDim.x + threadIdx.x; r < r1;
       r += (long long)gridDim.x * blockDim.x) {
    if (r > *reinterpret_cast<volatile long long *>(slot)) return;
    const double dx = __dsub_rn(P[3 * r], x0), dy = __dsub_rn(P[3 * r + 1], y0),
                 dz = __dsub_rn(P[3 * r + 2], z0);
    bool hit;
    if (stage == 0) {
      hit = norm3(dx, dy, dz) > thr;
    } else if (stage == 1) {
      double c[3];
      cross3(di[0], di[1], di[2], dx, dy, dz, c);
      hit = norm3(c[0], c[1], c[2]) > thr;
    } else {
      const double dot =
          __dadd_rn(__dadd_rn(__dmul_rn(dx, nrm[0]), __dmul_rn(dy, nrm[1])), __dmul_rn(dz, nrm[2]));
      hit = fabs(dot) > thr;
    }
    if (hit) {
      atomicMin(reinterpret_cast<unsigned long long *>(slot), static_cast<unsigned long long>(r));
      return;
    }
  }
}

// The three stages over rows [1, r1) in ONE CTA (random inputs hit in the
// first rows): each stage is a block-wide first-hit reduction, so the next
// stage starts from the exact first hit.  The full-range launches above run
// only for a stage this head leaves undecided.
__global__ void __launch_bounds__(1024) k_degenerate_head(const double *__restrict__ P,
                                                          long long n, ScanState *st,
                                                          long long r1) {
  const double tol = 1e-9;
  double scale = __longlong_as_double(static_cast<long long>(st->scale_bits));
  if (scale < 1e-30) scale = 1e-30;
  const double x0 = P[0], y0 = P[1], z0 = P[2];
  const long long none = 0x7fffffffffffffffll;
  if (r1 > n) r1 = n;
  __shared__ long long s_hit;
  double di[3] = {0, 0, 0}, nrm[3] = {0, 0, 0};
  for (int stage = 0; stage < 3; ++stage) {
    if (threadIdx.x == 0) s_hit = none;
    __syncthreads();
    double thr;
    if (stage == 0) {
      thr = __dmul_rn(tol, scale);
    } else if (stage == 1) {
      thr = __dmul_rn(__dmul_rn(tol, scale), scale);
    } else {
      thr = __dmul_rn(__dmul_rn(tol, scale), norm3(nrm[0], nrm[1], nrm[2]));
    }
    for (long long base = 1; base < r1; base += blockDim.x) {
      const long long r = base + threadIdx.x;
      bool hit = false;
      if (r < r1) {
        const double dx = __dsub_rn(P[3 * r], x0), dy = __dsub_rn(P[3 * r + 1], y0),
                     dz = __dsub_rn(P[3 * r + 2], z0);
        if (stage == 0) {
          hit = norm3(dx, dy, dz) > thr;
        } else if (stage == 1) {
          double c[3];
          cross3(di[0], di[1], di[2], dx, dy, dz, c);
          hit = norm3(c[0], c[1], c[2]) > thr;
        } else {
          const double dot = __dadd_rn(__dadd_rn(__dmul_rn(dx, nrm[0]), __dmul_rn(dy, nrm[1])),
                                       __dmul_rn(dz, nrm[2]));
          hit = fabs(dot) > thr;
        }
      }
      if (hit) atomicMin(reinterpret_cast<unsigned long long *>(&s_hit),
                         static_cast<unsigned long long>(r));
      __syncthreads();
      if (s_hit != none) break;  // block-uniform: the first hit is in this chunk
    }
    const long long h = s_hit;
    if (threadIdx.x == 0) (stage == 0 ? st->i : (stage == 1 ? st->j : st->k)) = h;
    if (h == none) return;  // undecided here: the full-range stages take over
    if (stage == 0) {
      di[0] = __dsub_rn(P[3 * h], x0);
      di[1] = __dsub_rn(P[3 * h + 1], y0);
      di[2] = __dsub_rn(P[3 * h + 2], z0);
    } else if (stage == 1) {
      cross3(di[0], di[1], di[2], __dsub_rn(P[3 * h], x0), __dsub_rn(P[3 * h + 1], y0),
             __dsub_rn(P[3 * h + 2], z0), nrm);
    }
    __syncthreads();
  }
}

__global__ void k_scan_init(ScanState *st) {
  st->scale_bits = 0;
  st->i = st->j = st->k = 0x7fffffffffffffffll;
}

// ----------------------------------------------------------------- epilogue
// per-block partial sums of the coordinates (fixed order -> deterministic)
__global__ void k_colsum(const double *__restrict__ P, long long n, double *partial) {
  double s0 = 0, s1 = 0, s2 = 0;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    s0 += P[3 * i];
    s1 += P[3 * i + 1];
    s2 += P[3 * i + 2];
  }
  __shared__ double s_warp[8];
  const prim::OpSum add;
  double r = prim::block_reduce256(s0, s_warp, add);
  if (threadIdx.x == 0) partial[3 * blockIdx.x] = r;
  r = prim::block_reduce256(s1, s_warp, add);
  if (threadIdx.x == 0) partial[3 * blockIdx.x + 1] = r;
  r = prim::block_reduce256(s2, s_warp, add);
  if (threadIdx.x == 0) partial[3 * blockIdx.x + 2] = r;
}

__global__ void k_centroid(const double *partial, int blocks, long long n, double *c) {
  if (threadIdx.x < 3) {
    double s = 0;
    for (int b = 0; b < blocks; ++b) s += partial[3 * b + threadIdx.x];
    c[threadIdx.x] = s / static_cast<double>(n);
  }
}

// orient every facet outward against the centroid, remap, mark vertices
__global__ void k_orient(const double *__restrict__ P, const double *__restrict__ cen,
                         const long long *__restrict__ order, const int *__restrict__ raw,
                         long long F, long long *faces, int *mark,
                         const long long *counts = nullptr) {
  if (counts) F = counts[0] + counts[1];  // F < 0: the facet count is on the device
  const double c0 = cen[0], c1 = cen[1], c2 = cen[2];
  for (long long f = blockIdx.x * (long long)blockDim.x + threadIdx.x; f < F;
       f += (long long)gridDim.x * blockDim.x) {
    const long long a = raw[3 * f], b = raw[3 * f + 1], c = raw[3 * f + 2];
    const double ax = P[3 * a], ay = P[3 * a + 1], az = P[3 * a + 2];
    double nrm[3];
    cross3(__dsub_rn(P[3 * b], ax), __dsub_rn(P[3 * b + 1], ay), __dsub_rn(P[3 * b + 2], az),
           __dsub_rn(P[3 * c], ax), __dsub_rn(P[3 * c + 1], ay), __dsub_rn(P[3 * c + 2], az), nrm);
    const double dot = __dadd_rn(__dadd_rn(__dmul_rn(nrm[0], __dsub_rn(c0, ax)),
                                           __dmul_rn(nrm[1], __dsub_rn(c1, ay))),
                                 __dmul_rn(nrm[2], __dsub_rn(c2, az)));
    const bool flip = dot > 0.0;
    const long long oa = order[a], ob = order[flip ? c : b], oc = order[flip ? b : c];
    faces[3 * f] = oa;
    faces[3 * f + 1] = ob;
    faces[3 * f + 2] = oc;
    mark[oa] = 1;
    mark[ob] = 1;
    mark[oc] = 1;
  }
}

}  // namespace h3d

using namespace h3d;

namespace {

struct PresortWS {
  unsigned long long *k0, *k1;
  int *v0, *v1, *v2;
  double *work;
  long long *head;
  void *prim_tmp;
  size_t prim_bytes;
  int *flag;
  ScanState *scan;
  double *partial;
  double *centroid;
  long long *count;
  unsigned long long *mm;
};

constexpr int kColsumBlocks = 296;

// temporary bytes of the device-wide primitives (prims.cuh) over n items
size_t prim_bytes_for(long long n) {
  size_t m = prim::rs_temp_bytes<unsigned long long>(n);
  const size_t a = prim::rs_temp_bytes<unsigned>(n), b = prim::scan_temp_bytes<long long>(n),
               c = prim::select_temp_bytes(n);
  if (a > m) m = a;
  if (b > m) m = b;
  return m > c ? m : c;
}

bool carve(h3d_arena &ar, long long n, PresortWS &w) {
  w.k0 = ar.take<unsigned long long>(n);
  w.k1 = ar.take<unsigned long long>(n);
  w.v0 = ar.take<int>(n);
  w.v1 = ar.take<int>(n);
  w.v2 = ar.take<int>(n);
  w.work = ar.take<double>(3 * n);
  w.head = ar.take<long long>(n);
  w.prim_bytes = prim_bytes_for(n);
  w.prim_tmp = ar.take<char>(w.prim_bytes);
  w.flag = ar.take<int>(16);
  w.scan = ar.take<ScanState>(1);
  w.partial = ar.take<double>(3 * kColsumBlocks);
  w.centroid = ar.take<double>(4);
  w.count = ar.take<long long>(2);
  w.mm = ar.take<unsigned long long>(2);
  return ar.base == nullptr || w.mm != nullptr;
}

// the epilogue's workspace: centroid partials, the count, the flagged
// select's temp (O(n / 2048)) -- carved from the front of whatever buffer
// the caller passes (a presort workspace, or an epilogue-sized one)
struct EpiWS {
  double *partial, *centroid;
  long long *count;
  void *tmp;
  size_t tmp_bytes;
};

bool carve_epi(h3d_arena &ar, long long n, EpiWS &w) {
  w.partial = ar.take<double>(3 * kColsumBlocks);
  w.centroid = ar.take<double>(4);
  w.count = ar.take<long long>(2);
  w.tmp_bytes = prim::select_temp_bytes(n);
  w.tmp = ar.take<char>(w.tmp_bytes);
  return ar.base == nullptr || w.tmp != nullptr;
}

// the sharded presort's workspace: keys of all n points, everything else
// sized by the window (m rows) -- O(n) 4-byte keys, not O(n) rows
struct SlabWS {
  unsigned *k32, *lk, *lk_alt;
  int *idx, *idx_alt, *runs;
  unsigned *hist;
  SelState *st;
  int *flag;
  ScanState *scan;
  unsigned long long *mm;
  void *tmp;
  size_t tmp_bytes;
};

bool carve_slab(h3d_arena &ar, long long n, long long m, SlabWS &w) {
  w.k32 = ar.take<unsigned>(n);
  w.lk = ar.take<unsigned>(m);
  w.lk_alt = ar.take<unsigned>(m);
  w.idx = ar.take<int>(m);
  w.idx_alt = ar.take<int>(m);
  w.runs = ar.take<int>(kSelRunCap + 64);
  w.hist = ar.take<unsigned>(4096);
  w.st = ar.take<SelState>(1);
  w.flag = ar.take<int>(4);
  w.scan = ar.take<ScanState>(1);
  w.mm = ar.take<unsigned long long>(2);
  w.tmp_bytes = prim::rs_temp_bytes<unsigned>(m);
  w.tmp = ar.take<char>(w.tmp_bytes);
  return ar.base == nullptr || w.tmp != nullptr;
}

// stable sort of (keys, vals) pairs; result in (*ko, *vo)
bool radix(PresortWS &w, unsigned long long *kin, int *vin, unsigned long long *kalt, int *valt,
           long long n, unsigned long long **ko, int **vo, cudaStream_t s) {
  bool alt = false;
  h3d_count_launches(9);
  if (h3d_check(prim::rs_sort_pairs<unsigned long long>(w.prim_tmp, w.prim_bytes, kin, vin, kalt, valt, n, 0,
                                                        64, &alt, s)))
    return false;
  *ko = alt ? kalt : kin;
  *vo = alt ? valt : vin;
  return true;
}

// _scan_degenerate on rows [0, rows) (api.py:113-147): the three stages over
// the first 16K rows in one CTA; only a stage left undecided there scans the
// rest (random inputs stop in the first block, as the reference's block-wise
// scan does).  Reads back the state and the flag words (one sync, two when
// the head is undecided).
bool degenerate_scan(const double *sorted_pts, long long rows, ScanState *wscan, int *wflag, unsigned G,
                     ScanState *hs, int *hflag, int nflag, cudaStream_t s) {
  const long long none = 0x7fffffffffffffffll;
  h3d_count_launches(1);
  k_degenerate_head<<<1, 1024, 0, s>>>(sorted_pts, rows, wscan, 16384);
  if (h3d_check(cudaMemcpyAsync(hs, wscan, sizeof(ScanState), cudaMemcpyDeviceToHost, s)) ||
      h3d_check(cudaMemcpyAsync(hflag, wflag, nflag * sizeof(int), cudaMemcpyDeviceToHost, s)) ||
      h3d_check(h3d_sync(s)))
    return false;
  if (hs->i != none && hs->j != none && hs->k != none) return true;
  h3d_count_launches(3);
  for (int stage = 0; stage < 3; ++stage)
    k_degenerate<<<G, 256, 0, s>>>(sorted_pts, rows, wscan, stage, 1, rows);
  return !h3d_check(cudaMemcpyAsync(hs, wscan, sizeof(ScanState), cudaMemcpyDeviceToHost, s)) &&
         !h3d_check(h3d_sync(s));
}

}  // namespace

namespace h3d {

// Gate of the optimistic presort (h3d_hull): its flags and the degeneracy
// scan decide, on the device, whether the merge levels may run on the sorted
// rows.  A tie or a long run of equal 32-bit keys needs the exact tie path
// (the host redoes the presort), a non-finite coordinate or a degenerate
// input is an error -- either way the error word stops every later launch.
__global__ void k_presort_gate(const int *flag, const ScanState *st, long long *err) {
  const long long none = 0x7fffffffffffffffll;
  long long e = 0;
  if (flag[1]) e = H3D_E_NONFINITE;
  else if (flag[0] || flag[2]) e = H3D_E_REDO;
  else if (st->i == none) e = H3D_E_COINCIDENT;
  else if (st->j == none) e = H3D_E_COLLINEAR;
  else if (st->k == none) e = H3D_E_COPLANAR;
  if (e) raise_err(err, e);
}

// The presort's common path with no host synchronisation: scan, 32-bit keys,
// radix sort, tie fix, row gather (+ adjacent-tie test), degeneracy scan
// (head, then each full stage only if the head left it undecided: the
// stage kernels return at once otherwise), gate.  Returns 0 or a code.
int64_t presort_async(const double *pts, int64_t n, double *sorted_pts, int64_t *order, void *workspace,
                      size_t workspace_bytes, long long *err, cudaStream_t s, int *sums_ready) {
  if (n < 1 || n > (1ll << 30)) return H3D_E_ARG;
  h3d_arena ar(workspace, workspace_bytes);
  PresortWS w;
  if (!carve(ar, n, w)) return H3D_E_ARG;
  const unsigned G = h3d_grid(n, 256) > 4096 ? 4096 : h3d_grid(n, 256);
  long long *ord = reinterpret_cast<long long *>(order);
  cudaMemsetAsync(w.flag, 0, sizeof(int) * 4, s);
  h3d_count_launches(1);
  k_scan_init<<<1, 1, 0, s>>>(w.scan);
  const unsigned long long mm_init[2] = {~0ull, 0ull};
  cudaMemcpyAsync(w.mm, mm_init, sizeof(mm_init), cudaMemcpyHostToDevice, s);
  h3d_count_launches(2);
  k_scan_input<<<G > 1184 ? 1184 : G, 256, 0, s>>>(pts, n, w.flag + 1, w.mm, &w.scan->scale_bits);
  unsigned *k32a = reinterpret_cast<unsigned *>(w.k0), *k32b = reinterpret_cast<unsigned *>(w.k1);
  // the keys with the sort's digit histograms (zeroed with its tickets)
  cudaMemsetAsync(w.prim_tmp, 0, 8 * prim::RS_BINS * sizeof(unsigned) + 256, s);
  k_keys32_rshist<<<G > 1184 ? 1184 : G, 256, 0, s>>>(pts, n, w.mm, k32a, static_cast<unsigned *>(w.prim_tmp));
  bool alt = false;
  h3d_count_launches(4);
  if (h3d_check(prim::rs_sort_pairs<unsigned>(w.prim_tmp, w.prim_bytes, k32a, w.v0, k32b, w.v1, n, 0, 32, &alt,
                                              s, true, true)))
    return H3D_E_CUDA;
  int *vs = alt ? w.v1 : w.v0;
  h3d_count_launches(2);
  k_tiefix<<<G, 256, 0, s>>>(pts, alt ? k32b : k32a, vs, n, w.flag + 2);
  // the epilogue's centroid partial sums land where orient_async carves
  // them: the front of this workspace, inside the keys (dead after the tie
  // fix) when they hold them -- else the epilogue sums the rows itself
  h3d_arena ea(workspace, workspace_bytes);
  EpiWS ew;
  carve_epi(ea, n, ew);
  const bool fuse = reinterpret_cast<char *>(ew.count) <= reinterpret_cast<char *>(w.k1);
  if (fuse)
    k_gather_rows_colsum<<<kColsumBlocks, 256, 0, s>>>(pts, vs, n, sorted_pts, ord, w.flag, ew.partial);
  else
    k_gather_rows<<<G, 256, 0, s>>>(pts, vs, n, sorted_pts, ord, nullptr, w.flag);
  *sums_ready = fuse ? 1 : 0;
  h3d_count_launches(5);
  k_degenerate_head<<<1, 1024, 0, s>>>(sorted_pts, n, w.scan, 16384);
  // (grid-stride: 4 CTAs per SM suffice; a stage the head decided returns at once)
  const unsigned GD = G < 4 * 148 ? G : 4 * 148;
  for (int stage = 0; stage < 3; ++stage) k_degenerate<<<GD, 256, 0, s>>>(sorted_pts, n, w.scan, stage, 1, n);
  k_presort_gate<<<1, 1, 0, s>>>(w.flag, w.scan, err);
  return h3d_check(cudaGetLastError()) ? H3D_E_CUDA : 0;
}

// The exact tie path with no host synchronisation, for a size whose
// previous call had x ties (h3d_hull): the common tie case -- short runs of
// equal x, a perturbation that keeps x non-decreasing (the reference's
// re-sort is then the identity) -- runs through on the device; its gate
// hands anything else (long runs, a re-sort) back to h3d_presort (E_REDO),
// and raises the presort's errors in the reference's order.  flag words:
// [1] non-finite, [2] long run of equal 32-bit keys, [8] long run of equal
// x, [9] an x tie, [12] a tie that survived the perturbation, [15] x
// descended after it.
__global__ void k_ties_gate(const int *flag, const ScanState *st, long long *err, long long *perturbed) {
  const long long none = 0x7fffffffffffffffll;
  const int tie = flag[9];
  long long e = 0;
  if (flag[1]) e = H3D_E_NONFINITE;
  else if (flag[2] || flag[8] || flag[15]) e = H3D_E_REDO;
  else if (tie && flag[12]) e = H3D_E_TIES;
  else if (st->i == none) e = H3D_E_COINCIDENT;
  else if (st->j == none) e = H3D_E_COLLINEAR;
  else if (st->k == none) e = H3D_E_COPLANAR;
  *perturbed = tie;
  if (e) raise_err(err, e);
}

int64_t presort_ties_async(const double *pts, int64_t n, double *sorted_pts, int64_t *order, void *workspace,
                           size_t workspace_bytes, long long *err, long long *perturbed, cudaStream_t s) {
  if (n < 1 || n > (1ll << 30)) return H3D_E_ARG;
  h3d_arena ar(workspace, workspace_bytes);
  PresortWS w;
  if (!carve(ar, n, w)) return H3D_E_ARG;
  const unsigned G = h3d_grid(n, 256) > 4096 ? 4096 : h3d_grid(n, 256);
  long long *ord = reinterpret_cast<long long *>(order);
  cudaMemsetAsync(w.flag, 0, sizeof(int) * 16, s);
  h3d_count_launches(1);
  k_scan_init<<<1, 1, 0, s>>>(w.scan);
  const unsigned long long mm_init[2] = {~0ull, 0ull};
  cudaMemcpyAsync(w.mm, mm_init, sizeof(mm_init), cudaMemcpyHostToDevice, s);
  h3d_count_launches(2);
  k_scan_input<<<G > 1184 ? 1184 : G, 256, 0, s>>>(pts, n, w.flag + 1, w.mm, &w.scan->scale_bits);
  unsigned *k32a = reinterpret_cast<unsigned *>(w.k0), *k32b = reinterpret_cast<unsigned *>(w.k1);
  k_keys32<<<G, 256, 0, s>>>(pts, n, w.mm, k32a, nullptr);
  bool alt = false;
  h3d_count_launches(5);
  if (h3d_check(prim::rs_sort_pairs<unsigned>(w.prim_tmp, w.prim_bytes, k32a, w.v0, k32b, w.v1, n, 0, 32, &alt,
                                              s, true)))
    return H3D_E_CUDA;
  int *vs = alt ? w.v1 : w.v0;
  h3d_count_launches(1);
  k_tiefix<<<G, 256, 0, s>>>(pts, alt ? k32b : k32a, vs, n, w.flag + 2);
  // lexsort (x, y, z): the runs of equal x re-ordered by (y, z, index)
  cudaMemcpyAsync(w.v2, vs, sizeof(int) * n, cudaMemcpyDeviceToDevice, s);
  h3d_count_launches(4);
  k_lexruns<<<G, 256, 0, s>>>(pts, w.v2, n, w.flag + 8);
  k_gather_rows<<<G, 256, 0, s>>>(pts, w.v2, n, w.work, nullptr, nullptr);
  // perturb_ties (api.py:99-101): run heads by max-scan, then base + rank * step
  k_run_heads<<<G, 256, 0, s>>>(w.work, n, w.head);
  if (h3d_check(prim::scan<false, long long>(w.prim_tmp, w.prim_bytes, w.head, w.head, n, prim::OpMax(), -1ll,
                                             -1ll, s)))
    return H3D_E_CUDA;
  h3d_count_launches(5);
  k_perturb<<<G, 256, 0, s>>>(w.work, w.head, n);
  k_perturbed_order<<<G, 256, 0, s>>>(w.work, n, w.flag + 12);
  cudaMemcpyAsync(sorted_pts, w.work, 3 * sizeof(double) * n, cudaMemcpyDeviceToDevice, s);
  k_perm_to_order<<<G, 256, 0, s>>>(w.v2, n, ord);
  // the scale on the (perturbed) sorted rows, then the degeneracy scan
  k_scan_init<<<1, 1, 0, s>>>(w.scan);
  k_absmax<<<G, 256, 0, s>>>(sorted_pts, 3 * n, &w.scan->scale_bits);
  h3d_count_launches(5);
  k_degenerate_head<<<1, 1024, 0, s>>>(sorted_pts, n, w.scan, 16384);
  for (int stage = 0; stage < 3; ++stage)
    k_degenerate<<<G < 4 * 148 ? G : 4 * 148, 256, 0, s>>>(sorted_pts, n, w.scan, stage, 1, n);
  k_ties_gate<<<1, 1, 0, s>>>(w.flag, w.scan, err, perturbed);
  return h3d_check(cudaGetLastError()) ? H3D_E_CUDA : 0;
}

// The epilogue with no host synchronisation: the facet count comes from the
// device counts (k_lo + k_up), the kernels stride over it; the vertex count
// lands in *vcount (device).
int64_t orient_async(const double *sorted_pts, int64_t n, const int64_t *order, const int32_t *faces_raw,
                     const long long *counts, int64_t cap, int64_t *faces, int32_t *vertex_mark,
                     int64_t *vertices, long long *vcount, void *workspace, size_t workspace_bytes,
                     cudaStream_t s, int sums_ready) {
  h3d_arena ar(workspace, workspace_bytes);
  EpiWS w;
  if (!carve_epi(ar, n, w)) return H3D_E_ARG;
  h3d_count_launches(sums_ready ? 2 : 3);
  // sums_ready: the optimistic presort's gather made the partial sums
  if (!sums_ready) k_colsum<<<kColsumBlocks, 256, 0, s>>>(sorted_pts, n, w.partial);
  k_centroid<<<1, 32, 0, s>>>(w.partial, kColsumBlocks, n, w.centroid);
  cudaMemsetAsync(vertex_mark, 0, sizeof(int) * n, s);
  const unsigned G = h3d_grid(cap, 256) > 1184 ? 1184 : h3d_grid(cap, 256);
  k_orient<<<G, 256, 0, s>>>(sorted_pts, w.centroid, reinterpret_cast<const long long *>(order), faces_raw,
                             -1, reinterpret_cast<long long *>(faces), vertex_mark, counts);
  h3d_count_launches(3);
  if (h3d_check(prim::select_flagged(w.tmp, w.tmp_bytes, vertex_mark, n,
                                     reinterpret_cast<long long *>(vertices), vcount, s)))
    return H3D_E_CUDA;
  return h3d_check(cudaGetLastError()) ? H3D_E_CUDA : 0;
}

}  // namespace h3d

extern "C" {

size_t h3d_presort_workspace_bytes(int64_t n) {
  if (n < 1) n = 1;
  h3d_arena ar(nullptr, 0);
  PresortWS w;
  carve(ar, n, w);
  return ar.used + 4096;
}

int64_t h3d_presort(const double *pts, int64_t n, double *sorted_pts, int64_t *order,
                    void *workspace, size_t workspace_bytes, int32_t *perturbed,
                    void *stream) {
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (n < 1 || n > (1ll << 30)) return H3D_E_ARG;
  h3d_arena ar(workspace, workspace_bytes);
  PresortWS w;
  if (!carve(ar, n, w)) return H3D_E_ARG;
  const unsigned G = h3d_grid(n, 256) > 4096 ? 4096 : h3d_grid(n, 256);
  long long *ord = reinterpret_cast<long long *>(order);
  unsigned long long *ks;
  int *vs;
  *perturbed = 0;

  // finiteness, x range and |coordinate| scale in one pass over the input
  cudaMemsetAsync(w.flag, 0, sizeof(int) * 4, s);
  h3d_count_launches(1);
  k_scan_init<<<1, 1, 0, s>>>(w.scan);
  unsigned long long mm_init[2] = {~0ull, 0ull};
  cudaMemcpyAsync(w.mm, mm_init, sizeof(mm_init), cudaMemcpyHostToDevice, s);
  h3d_count_launches(4);
  k_scan_input<<<G > 1184 ? 1184 : G, 256, 0, s>>>(pts, n, w.flag + 1, w.mm, &w.scan->scale_bits);
  // stable argsort of x (api.py:97): 32-bit fixed-point keys + tie-run fix
  unsigned *k32a = reinterpret_cast<unsigned *>(w.k0), *k32b = reinterpret_cast<unsigned *>(w.k1);
  k_keys32<<<G, 256, 0, s>>>(pts, n, w.mm, k32a, nullptr);
  {
    // values = the row positions, generated by the first digit pass
    bool alt = false;
    h3d_count_launches(5);
    if (h3d_check(prim::rs_sort_pairs<unsigned>(w.prim_tmp, w.prim_bytes, k32a, w.v0, k32b, w.v1, n, 0, 32,
                                                &alt, s, true)))
      return H3D_E_CUDA;
    vs = alt ? w.v1 : w.v0;
    k_tiefix<<<G, 256, 0, s>>>(pts, alt ? k32b : k32a, vs, n, w.flag + 2);
  }
  // rows in x order, with the adjacent-tie test folded in (rare ties:
  // the rows are rebuilt by the lexsort/perturbation path below)
  k_gather_rows<<<G, 256, 0, s>>>(pts, vs, n, sorted_pts, ord, nullptr, w.flag);
  int hflag[3] = {0, 0, 0};
  if (h3d_check(cudaMemcpyAsync(hflag, w.flag, 3 * sizeof(int), cudaMemcpyDeviceToHost, s)) ||
      h3d_check(h3d_sync(s)))
    return H3D_E_CUDA;
  if (hflag[1]) return H3D_E_NONFINITE;
  if (hflag[2]) {  // long runs of equal 32-bit keys: the exact 64-bit sort
    cudaMemsetAsync(w.flag, 0, sizeof(int), s);
    h3d_count_launches(2);
    k_keys<<<G, 256, 0, s>>>(pts, nullptr, 0, n, w.k0, w.v0);
    if (!radix(w, w.k0, w.v0, w.k1, w.v1, n, &ks, &vs, s)) return H3D_E_CUDA;
    k_adjacent_tie<<<G, 256, 0, s>>>(ks, n, w.flag);
    if (h3d_check(cudaMemcpyAsync(hflag, w.flag, sizeof(int), cudaMemcpyDeviceToHost, s)) ||
        h3d_check(h3d_sync(s)))
      return H3D_E_CUDA;
    if (!hflag[0]) {
      h3d_count_launches(1);
      k_gather_rows<<<G, 256, 0, s>>>(pts, vs, n, sorted_pts, ord, nullptr);
    }
  }
  const int tie = hflag[0];
  if (tie) {
    // lexsort (x, y, z) (api.py:86-87): the runs of equal x of the stable x
    // order re-ordered by (y, z, index); with a run longer than RUN_MAX the
    // three stable LSD passes on z, then y, then x
    int lexflag[4] = {0, 0, 0, 0};
    cudaMemcpyAsync(w.v2, vs, sizeof(int) * n, cudaMemcpyDeviceToDevice, s);
    cudaMemsetAsync(w.flag, 0, sizeof(int) * 4, s);
    h3d_count_launches(1);
    k_lexruns<<<G, 256, 0, s>>>(pts, w.v2, n, w.flag + 2);
    if (h3d_check(cudaMemcpyAsync(lexflag, w.flag, sizeof(lexflag), cudaMemcpyDeviceToHost, s)) ||
        h3d_check(h3d_sync(s)))
      return H3D_E_CUDA;
    if (lexflag[2]) {
      int *perm = nullptr;
      h3d_count_launches(1);
      k_keys<<<G, 256, 0, s>>>(pts, nullptr, 2, n, w.k0, w.v0);
      if (!radix(w, w.k0, w.v0, w.k1, w.v1, n, &ks, &vs, s)) return H3D_E_CUDA;
      perm = vs;
      int *other = (perm == w.v0) ? w.v1 : w.v0;
      h3d_count_launches(1);
      k_keys<<<G, 256, 0, s>>>(pts, perm, 1, n, w.k0, other);
      if (!radix(w, w.k0, other, w.k1, perm, n, &ks, &vs, s)) return H3D_E_CUDA;
      perm = vs;
      other = (perm == w.v0) ? w.v1 : w.v0;
      h3d_count_launches(1);
      k_keys<<<G, 256, 0, s>>>(pts, perm, 0, n, w.k0, other);
      if (!radix(w, w.k0, other, w.k1, perm, n, &ks, &vs, s)) return H3D_E_CUDA;
      // lexsort permutation kept in v2
      cudaMemcpyAsync(w.v2, vs, sizeof(int) * n, cudaMemcpyDeviceToDevice, s);
    }
    // lex-sorted rows -> w.work
    h3d_count_launches(1);
    k_gather_rows<<<G, 256, 0, s>>>(pts, w.v2, n, w.work, nullptr, nullptr);
    // perturb_ties: run heads by max-scan, then base + rank*step
    h3d_count_launches(1);
    k_run_heads<<<G, 256, 0, s>>>(w.work, n, w.head);
    h3d_count_launches(1);
    if (h3d_check(prim::scan<false, long long>(w.prim_tmp, w.prim_bytes, w.head, w.head, n, prim::OpMax(),
                                               -1ll, -1ll, s)))
      return H3D_E_CUDA;
    h3d_count_launches(1);
    k_perturb<<<G, 256, 0, s>>>(w.work, w.head, n);
    // stable re-sort of the perturbed x (api.py:102-104): the identity when
    // x did not descend anywhere (checked on the device)
    cudaMemsetAsync(w.flag, 0, sizeof(int) * 4, s);
    h3d_count_launches(1);
    k_perturbed_order<<<G, 256, 0, s>>>(w.work, n, w.flag);
    int pflag[4] = {0, 0, 0, 0};
    if (h3d_check(cudaMemcpyAsync(pflag, w.flag, sizeof(pflag), cudaMemcpyDeviceToHost, s)) ||
        h3d_check(h3d_sync(s)))
      return H3D_E_CUDA;
    if (!pflag[3]) {
      cudaMemcpyAsync(sorted_pts, w.work, 3 * sizeof(double) * n, cudaMemcpyDeviceToDevice, s);
      h3d_count_launches(1);
      k_perm_to_order<<<G, 256, 0, s>>>(w.v2, n, ord);  // flag[0]: the ties that survived
    } else {
      h3d_count_launches(1);
      k_keys<<<G, 256, 0, s>>>(w.work, nullptr, 0, n, w.k0, w.v0);
      if (!radix(w, w.k0, w.v0, w.k1, w.v1, n, &ks, &vs, s)) return H3D_E_CUDA;
      h3d_count_launches(1);
      k_gather_rows<<<G, 256, 0, s>>>(w.work, vs, n, sorted_pts, ord, w.v2);
      cudaMemsetAsync(w.flag, 0, sizeof(int) * 4, s);
      h3d_count_launches(1);
      k_adjacent_tie<<<G, 256, 0, s>>>(ks, n, w.flag);
    }
    *perturbed = 1;
    // the perturbation changed x: the scale is re-taken on the sorted rows
    h3d_count_launches(2);
    k_scan_init<<<1, 1, 0, s>>>(w.scan);
    k_absmax<<<G, 256, 0, s>>>(sorted_pts, 3 * n, &w.scan->scale_bits);
  }
  // _scan_degenerate on the sorted rows (api.py:113-147)
  ScanState hs;
  int tie2 = 0;
  if (!degenerate_scan(sorted_pts, n, w.scan, w.flag, G, &hs, &tie2, 1, s)) return H3D_E_CUDA;
  if (tie && tie2) return H3D_E_TIES;
  const long long none = 0x7fffffffffffffffll;
  if (hs.i == none) return H3D_E_COINCIDENT;
  if (hs.j == none) return H3D_E_COLLINEAR;
  if (hs.k == none) return H3D_E_COPLANAR;
  return 0;
}

size_t h3d_epilogue_workspace_bytes(int64_t n) {
  if (n < 1) n = 1;
  h3d_arena ar(nullptr, 0);
  EpiWS w;
  carve_epi(ar, n, w);
  return ar.used + 4096;
}

size_t h3d_presort_slab_workspace_bytes(int64_t n, int64_t m) {
  if (n < 1) n = 1;
  if (m < 1) m = 1;
  h3d_arena ar(nullptr, 0);
  SlabWS w;
  carve_slab(ar, n, m, w);
  return ar.used + 4096;
}

int64_t h3d_presort_slab(const double *pts, int64_t n, int64_t q0, int64_t p1, int32_t scan,
                         double *sorted_pts, int64_t *order, void *workspace,
                         size_t workspace_bytes, void *stream) {
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (n < 2048 || n > (1ll << 30) || q0 < 0 || p1 > n || q0 >= p1) return H3D_E_ARG;
  h3d_arena ar(workspace, workspace_bytes);
  const long long m = p1 - q0;
  SlabWS w;
  if (!carve_slab(ar, n, m, w)) return H3D_E_ARG;
  const unsigned G = h3d_grid(n, 256) > 4096 ? 4096 : h3d_grid(n, 256);
  unsigned *k32 = w.k32;
  unsigned *lk = w.lk, *lk_alt = w.lk_alt;
  int *idx = w.idx, *idx_alt = w.idx_alt, *runs = w.runs;
  unsigned *hist = w.hist;
  SelState *st = w.st;
  SelState init{};
  init.b[0] = q0 > 0 ? q0 : -1;
  init.b[1] = p1 < n ? p1 : -1;
  init.rem[0] = q0;
  init.rem[1] = p1;
  cudaMemsetAsync(w.flag, 0, sizeof(int) * 4, s);
  cudaMemsetAsync(hist, 0, sizeof(unsigned) * 4096, s);
  cudaMemcpyAsync(st, &init, sizeof(init), cudaMemcpyHostToDevice, s);
  unsigned long long mm_init[2] = {~0ull, 0ull};
  cudaMemcpyAsync(w.mm, mm_init, sizeof(mm_init), cudaMemcpyHostToDevice, s);
  h3d_count_launches(2);
  k_scan_init<<<1, 1, 0, s>>>(w.scan);
  k_scan_input<<<G > 1184 ? 1184 : G, 256, 0, s>>>(pts, n, w.flag + 1, w.mm, &w.scan->scale_bits);
  // keys + the first select pass's histogram (every key has the empty prefix)
  h3d_count_launches(1);
  k_keys32_hist<<<1184, 256, 0, s>>>(pts, n, w.mm, k32, hist);
  if (init.b[0] >= 0 || init.b[1] >= 0) {
    for (int pass = 0; pass < 3; ++pass) {
      h3d_count_launches(pass ? 2 : 1);
      if (pass) k_sel_hist<<<296, 512, 0, s>>>(k32, n, st, pass, hist);
      k_sel_pick<<<1, 256, 0, s>>>(hist, st, pass);
    }
  }
  h3d_count_launches(3);
  k_sel_compact<<<1184, 256, 0, s>>>(k32, n, st, idx, runs, m);
  k_sel_runs<<<1, 256, 0, s>>>(pts, k32, st, runs, idx, m);
  const unsigned Gm = h3d_grid(m, 256) > 4096 ? 4096 : h3d_grid(m, 256);
  k_sel_keys<<<Gm, 256, 0, s>>>(k32, st, idx, lk, m);
  bool alt = false;
  h3d_count_launches(5);
  if (h3d_check(prim::rs_sort_pairs<unsigned>(w.tmp, w.tmp_bytes, lk, idx, lk_alt, idx_alt, m, 0, 32,
                                              &alt, s)))
    return H3D_E_CUDA;
  unsigned *kcur = alt ? lk_alt : lk;
  int *vcur = alt ? idx_alt : idx;
  h3d_count_launches(2);
  k_tiefix<<<Gm, 256, 0, s>>>(pts, kcur, vcur, m, w.flag + 2);
  k_gather_rows<<<Gm, 256, 0, s>>>(pts, vcur, m, sorted_pts + 3 * q0,
                                   reinterpret_cast<long long *>(order) + q0, nullptr, w.flag);
  int hflag[3] = {0, 0, 0};
  SelState hst;
  ScanState hs;
  if (h3d_check(cudaMemcpyAsync(&hst, st, sizeof(hst), cudaMemcpyDeviceToHost, s)))
    return H3D_E_CUDA;
  if (scan) {  // _scan_degenerate over this window (rank 0: rows [0, p1))
    if (!degenerate_scan(sorted_pts, p1, w.scan, w.flag, G, &hs, hflag, 3, s)) return H3D_E_CUDA;
  } else if (h3d_check(cudaMemcpyAsync(hflag, w.flag, 3 * sizeof(int), cudaMemcpyDeviceToHost, s)) ||
             h3d_check(h3d_sync(s))) {
    return H3D_E_CUDA;
  }
  // ties, long key runs, a bad selection, non-finite input or a degeneracy
  // the window cannot decide: the caller runs the replicated h3d_presort
  if (hflag[0] || hflag[1] || hflag[2] || hst.bad) return H3D_E_FASTPATH;
  const long long none = 0x7fffffffffffffffll;
  if (scan && (hs.i == none || hs.j == none || hs.k == none)) return H3D_E_FASTPATH;
  return 0;
}

int64_t h3d_orient_remap_ex(const double *sorted_pts, int64_t n, const int64_t *order,
                            const int32_t *faces_raw, int64_t nfaces, int64_t *faces,
                            int32_t *vertex_mark, int64_t *vertices,
                            const double *centroid_pts, void *workspace,
                            size_t workspace_bytes, void *stream) {
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  h3d_arena ar(workspace, workspace_bytes);
  EpiWS w;
  if (!carve_epi(ar, n, w)) return H3D_E_ARG;
  if (nfaces == 0) return H3D_E_NOFACETS;
  h3d_count_launches(1);
  k_colsum<<<kColsumBlocks, 256, 0, s>>>(centroid_pts ? centroid_pts : sorted_pts, n, w.partial);
  h3d_count_launches(1);
  k_centroid<<<1, 32, 0, s>>>(w.partial, kColsumBlocks, n, w.centroid);
  cudaMemsetAsync(vertex_mark, 0, sizeof(int) * n, s);
  const unsigned G = h3d_grid(nfaces, 256) > 4096 ? 4096 : h3d_grid(nfaces, 256);
  h3d_count_launches(1);
  k_orient<<<G, 256, 0, s>>>(sorted_pts, w.centroid, reinterpret_cast<const long long *>(order),
                             faces_raw, nfaces, reinterpret_cast<long long *>(faces),
                             vertex_mark);
  h3d_count_launches(3);
  if (h3d_check(prim::select_flagged(w.tmp, w.tmp_bytes, vertex_mark, n,
                                     reinterpret_cast<long long *>(vertices), w.count, s)))
    return H3D_E_CUDA;
  long long cnt = 0;
  if (h3d_check(cudaMemcpyAsync(&cnt, w.count, sizeof(cnt), cudaMemcpyDeviceToHost, s)) ||
      h3d_check(h3d_sync(s)))
    return H3D_E_CUDA;
  return cnt;
}

int64_t h3d_orient_remap(const double *sorted_pts, int64_t n, const int64_t *order,
                         const int32_t *faces_raw, int64_t nfaces, int64_t *faces,
                         int32_t *vertex_mark, int64_t *vertices, void *workspace,
                         size_t workspace_bytes, void *stream) {
  return h3d_orient_remap_ex(sorted_pts, n, order, faces_raw, nfaces, faces, vertex_mark, vertices,
                             nullptr, workspace, workspace_bytes, stream);
}

}  // extern "C"
