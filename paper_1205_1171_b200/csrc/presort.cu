// presort.cu -- device x-presort, tie perturbation, degeneracy scan, epilogue.
//
// Restates on the GPU the host numpy steps around the engine:
//   _sort_and_perturb / perturb_ties / _lex_order  pkg/src/hull3d/api.py:61-110
//   _scan_degenerate                               pkg/src/hull3d/api.py:113-147
//   orientation, remap, np.unique                  pkg/src/hull3d/api.py:252-266
//
// Sorting: stable LSD radix sort (CUB onesweep) of order-preserving u64 keys
// of the fp64 coordinates with the row index as payload.  -0.0 is folded
// onto +0.0 first so that the two compare equal, as they do under numpy's
// comparisons.  Stability + index payload reproduces argsort(kind="stable")
// and np.lexsort((z, y, x)) exactly (three stable passes z, y, x).
#include <cub/cub.cuh>

#include "h3d_device.cuh"
#include "h3d_host.h"

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

__global__ void k_keys32(const double *__restrict__ pts, long long n,
                         const unsigned long long *__restrict__ mm, unsigned *keys, int *vals) {
  const double lo = key_to_double(mm[0]), hi = key_to_double(mm[1]);
  const double span = __dsub_rn(hi, lo);
  const double sc = span > 0.0 ? __ddiv_rn(4294967295.0, span) : 0.0;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    double x = pts[3 * i];
    if (x == 0.0) x = 0.0;
    double f = __dmul_rn(__dsub_rn(x, lo), sc);  // monotone in x
    if (!(f >= 0.0)) f = 0.0;
    if (f > 4294967295.0) f = 4294967295.0;
    keys[i] = static_cast<unsigned>(f);
    vals[i] = static_cast<int>(i);
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
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    const double x = pts[3 * i], y = pts[3 * i + 1], z = pts[3 * i + 2];
    bad |= !isfinite(x) || !isfinite(y) || !isfinite(z);
    const unsigned long long k = order_key(x);
    lo = k < lo ? k : lo;
    hi = k > hi ? k : hi;
    amax = fmax(amax, fmax(fabs(x), fmax(fabs(y), fabs(z))));
  }
  for (int o = 16; o; o >>= 1) {
    const unsigned long long a = __shfl_xor_sync(0xffffffffu, lo, o),
                             b = __shfl_xor_sync(0xffffffffu, hi, o);
    lo = a < lo ? a : lo;
    hi = b > hi ? b : hi;
    amax = fmax(amax, __shfl_xor_sync(0xffffffffu, amax, o));
  }
  bad = __any_sync(0xffffffffu, bad);
  if ((threadIdx.x & 31) == 0) {
    atomicMin(mm, lo);
    atomicMax(mm + 1, hi);
    atomicMax(absmax_bits, static_cast<unsigned long long>(__double_as_longlong(amax)));
    if (bad) *nonfinite = 1;
  }
}

__global__ void k_gather_rows(const double *__restrict__ pts, const int *__restrict__ perm,
                              long long n, double *out, long long *order,
                              const int *__restrict__ outer, int *tie = nullptr) {
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

// run start index per row of lex-sorted x (0 where the row continues a run)
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
  typedef cub::BlockReduce<double, 256> BR;
  __shared__ typename BR::TempStorage tmp;
  const double b = BR(tmp).Reduce(best, cub::Max());
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
  typedef cub::BlockReduce<double, 256> BR;
  __shared__ typename BR::TempStorage tmp;
  double r = BR(tmp).Sum(s0);
  __syncthreads();
  if (threadIdx.x == 0) partial[3 * blockIdx.x] = r;
  r = BR(tmp).Sum(s1);
  __syncthreads();
  if (threadIdx.x == 0) partial[3 * blockIdx.x + 1] = r;
  r = BR(tmp).Sum(s2);
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
                         long long F, long long *faces, int *mark) {
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
  void *cub_tmp;
  size_t cub_bytes;
  int *flag;
  ScanState *scan;
  double *partial;
  double *centroid;
  long long *count;
  unsigned long long *mm;
};

constexpr int kColsumBlocks = 296;

size_t cub_bytes_for(long long n) {
  size_t a = 0, b = 0, c = 0, d = 0;
  cub::DoubleBuffer<unsigned long long> kb(nullptr, nullptr);
  cub::DoubleBuffer<int> vb(nullptr, nullptr);
  cub::DeviceRadixSort::SortPairs(nullptr, a, kb, vb, static_cast<int>(n));
  cub::DeviceScan::InclusiveScan(nullptr, b, static_cast<long long *>(nullptr),
                                 static_cast<long long *>(nullptr), cub::Max(),
                                 static_cast<int>(n));
  cub::DeviceSelect::Flagged(nullptr, c, cub::CountingInputIterator<long long>(0),
                             static_cast<int *>(nullptr), static_cast<long long *>(nullptr),
                             static_cast<long long *>(nullptr), static_cast<int>(n));
  (void)d;
  size_t m = a > b ? a : b;
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
  w.cub_bytes = cub_bytes_for(n);
  w.cub_tmp = ar.take<char>(w.cub_bytes);
  w.flag = ar.take<int>(4);
  w.scan = ar.take<ScanState>(1);
  w.partial = ar.take<double>(3 * kColsumBlocks);
  w.centroid = ar.take<double>(4);
  w.count = ar.take<long long>(2);
  w.mm = ar.take<unsigned long long>(2);
  return ar.base == nullptr || w.mm != nullptr;
}

// stable sort of (keys, vals) pairs; result in (*ko, *vo)
bool radix(PresortWS &w, unsigned long long *kin, int *vin, unsigned long long *kalt, int *valt,
           long long n, unsigned long long **ko, int **vo, cudaStream_t s) {
  cub::DoubleBuffer<unsigned long long> kb(kin, kalt);
  cub::DoubleBuffer<int> vb(vin, valt);
  size_t bytes = w.cub_bytes;
  if (h3d_check(cub::DeviceRadixSort::SortPairs(w.cub_tmp, bytes, kb, vb, static_cast<int>(n),
                                                0, 64, s)))
    return false;
  *ko = kb.Current();
  *vo = vb.Current();
  return true;
}

}  // namespace

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
  k_scan_input<<<G, 256, 0, s>>>(pts, n, w.flag + 1, w.mm, &w.scan->scale_bits);
  // stable argsort of x (api.py:97): 32-bit fixed-point keys + tie-run fix
  unsigned *k32a = reinterpret_cast<unsigned *>(w.k0), *k32b = reinterpret_cast<unsigned *>(w.k1);
  k_keys32<<<G, 256, 0, s>>>(pts, n, w.mm, k32a, w.v0);
  {
    cub::DoubleBuffer<unsigned> kb(k32a, k32b);
    cub::DoubleBuffer<int> vb(w.v0, w.v1);
    size_t bytes = w.cub_bytes;
    if (h3d_check(cub::DeviceRadixSort::SortPairs(w.cub_tmp, bytes, kb, vb, static_cast<int>(n),
                                                  0, 32, s)))
      return H3D_E_CUDA;
    vs = vb.Current();
    k_tiefix<<<G, 256, 0, s>>>(pts, kb.Current(), vs, n, w.flag + 2);
  }
  // rows in x order, with the adjacent-tie test folded in (rare ties:
  // the rows are rebuilt by the lexsort/perturbation path below)
  k_gather_rows<<<G, 256, 0, s>>>(pts, vs, n, sorted_pts, ord, nullptr, w.flag);
  int hflag[3] = {0, 0, 0};
  if (h3d_check(cudaMemcpyAsync(hflag, w.flag, 3 * sizeof(int), cudaMemcpyDeviceToHost, s)) ||
      h3d_check(cudaStreamSynchronize(s)))
    return H3D_E_CUDA;
  if (hflag[1]) return H3D_E_NONFINITE;
  if (hflag[2]) {  // long runs of equal 32-bit keys: the exact 64-bit sort
    cudaMemsetAsync(w.flag, 0, sizeof(int), s);
    h3d_count_launches(2);
    k_keys<<<G, 256, 0, s>>>(pts, nullptr, 0, n, w.k0, w.v0);
    if (!radix(w, w.k0, w.v0, w.k1, w.v1, n, &ks, &vs, s)) return H3D_E_CUDA;
    k_adjacent_tie<<<G, 256, 0, s>>>(ks, n, w.flag);
    if (h3d_check(cudaMemcpyAsync(hflag, w.flag, sizeof(int), cudaMemcpyDeviceToHost, s)) ||
        h3d_check(cudaStreamSynchronize(s)))
      return H3D_E_CUDA;
    if (!hflag[0]) {
      h3d_count_launches(1);
      k_gather_rows<<<G, 256, 0, s>>>(pts, vs, n, sorted_pts, ord, nullptr);
    }
  }
  const int tie = hflag[0];
  if (tie) {
    // lexsort (x, y, z): stable LSD passes on z, then y, then x (api.py:86-87)
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
    // lex-sorted rows -> w.work; lexsort permutation kept in v2
    cudaMemcpyAsync(w.v2, vs, sizeof(int) * n, cudaMemcpyDeviceToDevice, s);
    h3d_count_launches(1);
    k_gather_rows<<<G, 256, 0, s>>>(pts, w.v2, n, w.work, nullptr, nullptr);
    // perturb_ties: run heads by max-scan, then base + rank*step
    h3d_count_launches(1);
    k_run_heads<<<G, 256, 0, s>>>(w.work, n, w.head);
    size_t bytes = w.cub_bytes;
    if (h3d_check(cub::DeviceScan::InclusiveScan(w.cub_tmp, bytes, w.head, w.head, cub::Max(),
                                                 static_cast<int>(n), s)))
      return H3D_E_CUDA;
    h3d_count_launches(1);
    k_perturb<<<G, 256, 0, s>>>(w.work, w.head, n);
    // stable re-sort of the perturbed x (api.py:102-104)
    h3d_count_launches(1);
    k_keys<<<G, 256, 0, s>>>(w.work, nullptr, 0, n, w.k0, w.v0);
    if (!radix(w, w.k0, w.v0, w.k1, w.v1, n, &ks, &vs, s)) return H3D_E_CUDA;
    h3d_count_launches(1);
    k_gather_rows<<<G, 256, 0, s>>>(w.work, vs, n, sorted_pts, ord, w.v2);
    cudaMemsetAsync(w.flag, 0, sizeof(int) * 4, s);
    h3d_count_launches(1);
    k_adjacent_tie<<<G, 256, 0, s>>>(ks, n, w.flag);
    *perturbed = 1;
    // the perturbation changed x: the scale is re-taken on the sorted rows
    h3d_count_launches(2);
    k_scan_init<<<1, 1, 0, s>>>(w.scan);
    k_absmax<<<G, 256, 0, s>>>(sorted_pts, 3 * n, &w.scan->scale_bits);
  }
  // _scan_degenerate on the sorted rows (api.py:113-147)
  // each stage scans the first 16K rows with a small grid and the rest only
  // when they hold no hit (random inputs stop in the first block, as the
  // reference's block-wise scan does)
  h3d_count_launches(6);
  for (int stage = 0; stage < 3; ++stage) {
    k_degenerate<<<64, 256, 0, s>>>(sorted_pts, n, w.scan, stage, 1, 16384);
    k_degenerate<<<G, 256, 0, s>>>(sorted_pts, n, w.scan, stage, 16384, n);
  }
  ScanState hs;
  int tie2 = 0;
  if (h3d_check(cudaMemcpyAsync(&hs, w.scan, sizeof(hs), cudaMemcpyDeviceToHost, s)) ||
      h3d_check(cudaMemcpyAsync(&tie2, w.flag, sizeof(int), cudaMemcpyDeviceToHost, s)) ||
      h3d_check(cudaStreamSynchronize(s)))
    return H3D_E_CUDA;
  if (tie && tie2) return H3D_E_TIES;
  const long long none = 0x7fffffffffffffffll;
  if (hs.i == none) return H3D_E_COINCIDENT;
  if (hs.j == none) return H3D_E_COLLINEAR;
  if (hs.k == none) return H3D_E_COPLANAR;
  return 0;
}

int64_t h3d_orient_remap(const double *sorted_pts, int64_t n, const int64_t *order,
                         const int32_t *faces_raw, int64_t nfaces, int64_t *faces,
                         int32_t *vertex_mark, int64_t *vertices, void *workspace,
                         size_t workspace_bytes, void *stream) {
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  h3d_arena ar(workspace, workspace_bytes);
  PresortWS w;
  if (!carve(ar, n, w)) return H3D_E_ARG;
  if (nfaces == 0) return H3D_E_NOFACETS;
  h3d_count_launches(1);
  k_colsum<<<kColsumBlocks, 256, 0, s>>>(sorted_pts, n, w.partial);
  h3d_count_launches(1);
  k_centroid<<<1, 32, 0, s>>>(w.partial, kColsumBlocks, n, w.centroid);
  cudaMemsetAsync(vertex_mark, 0, sizeof(int) * n, s);
  const unsigned G = h3d_grid(nfaces, 256) > 4096 ? 4096 : h3d_grid(nfaces, 256);
  h3d_count_launches(1);
  k_orient<<<G, 256, 0, s>>>(sorted_pts, w.centroid, reinterpret_cast<const long long *>(order),
                             faces_raw, nfaces, reinterpret_cast<long long *>(faces),
                             vertex_mark);
  size_t bytes = w.cub_bytes;
  if (h3d_check(cub::DeviceSelect::Flagged(w.cub_tmp, bytes, cub::CountingInputIterator<long long>(0),
                                           vertex_mark, reinterpret_cast<long long *>(vertices),
                                           w.count, static_cast<int>(n), s)))
    return H3D_E_CUDA;
  long long cnt = 0;
  if (h3d_check(cudaMemcpyAsync(&cnt, w.count, sizeof(cnt), cudaMemcpyDeviceToHost, s)) ||
      h3d_check(cudaStreamSynchronize(s)))
    return H3D_E_CUDA;
  return cnt;
}

}  // extern "C"
