// prims.cuh -- device-wide primitives of the fused path, hand-written for
// sm_100a (no CUB kernels on the hot path):
//
//  * rs_sort_pairs: stable LSD radix sort of (key, int value) pairs, 8-bit
//    digits, "onesweep" structure: ONE histogram pass over the keys for all
//    digit positions, then ONE scatter kernel per digit whose tiles find
//    their global offsets by decoupled look-back (tiles numbered in start
//    order by an atomic ticket, so a tile only ever waits on tiles that are
//    already running).  Inside a tile each warp ranks its keys stably (digit
//    peers from per-bit ballots), the tile is locally sorted in shared memory and
//    written out digit run by digit run (coalesced stores).
//    The presort's x keys (api.py:97, `np.argsort(kind="stable")`) and the
//    lexsort / perturbation passes (api.py:86-87, :97-105) run on it, as do
//    the incidence lists of the time-split pipeline (big.cu).
//  * scan: inclusive or exclusive scan with any associative operator, one
//    pass with decoupled look-back (k_scan_1p);
//  * select_flagged: indices of the nonzero flags, in order (np.unique of
//    the facet vertices, api.py:266, as a vertex-mark compaction).
//
// Every routine takes a caller-owned temporary buffer (the library never
// allocates); *_temp_bytes gives its size.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace h3d {
namespace prim {

constexpr int RS_THREADS = 256;
constexpr int RS_WARPS = RS_THREADS / 32;
constexpr int RS_BINS = 256;
constexpr unsigned long long RS_AGG = 1ull << 62;  // look-back word: tile aggregate
constexpr unsigned long long RS_INC = 2ull << 62;  // look-back word: inclusive prefix

template <typename K>
struct RsItems;
template <>
struct RsItems<unsigned> {
  static constexpr int v = 18;  // 4608 keys per tile, 47 KB of shared memory (larger tiles: fewer look-backs; 16 -> 18: -8 %, tools/rs_bench.cu)
};
template <>
struct RsItems<unsigned long long> {
  static constexpr int v = 11;  // 2816 keys per tile, 45 KB
};

template <typename K>
__host__ __device__ constexpr int rs_tile() {
  return RS_THREADS * RsItems<K>::v;
}

// look-back words carry their flag and value in one 64-bit word (single-copy
// atomic): relaxed GPU-scope accesses suffice, nothing else is published
__device__ __forceinline__ unsigned long long ld_relaxed_u64(const unsigned long long *p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed_u64(unsigned long long *p, unsigned long long v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// Decoupled look-back of one digit over the tiles before `tile`, a window
// of LB_W predecessors per round trip (independent loads in flight instead
// of one dependent hop per tile: the first wave's tiles all start together
// and the inclusive prefixes only spread from tile 0 outwards)
constexpr int LB_W = 8;
__device__ __forceinline__ unsigned long long lookback(const unsigned long long *look, long long tile, int d) {
  unsigned long long prefix = 0;
  long long j = tile - 1;  // next predecessor to account for
  while (j >= 0) {
    unsigned long long w[LB_W];
#pragma unroll
    for (int q = 0; q < LB_W; ++q) w[q] = j - q >= 0 ? ld_relaxed_u64(look + (j - q) * RS_BINS + d) : RS_INC;
    int q = 0;
    bool done = false;
#pragma unroll
    for (int r = 0; r < LB_W; ++r) {
      if (done || (w[r] >> 62) == 0) { done = true; continue; }  // not ready: re-poll from here
      if (j - r >= 0) prefix += w[r] & 0xffffffffull;
      q = r + 1;
      if ((w[r] >> 62) == 2) { j = -1; done = true; }  // an inclusive prefix ends the walk
    }
    if (j >= 0) j -= q;
  }
  return prefix;
}

// exclusive scan of one value per thread over a 256-thread block (s_warp:
// 8 words of shared memory); *total, when given, gets the block's sum
template <typename T>
__device__ __forceinline__ T block_excl_sum256(T v, T *s_warp, T *total = nullptr) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  T x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const T t = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += t;
  }
  if (lane == 31) s_warp[w] = x;
  __syncthreads();
  T wp = 0, all = 0;
#pragma unroll
  for (int q = 0; q < RS_WARPS; ++q) {
    wp += q < w ? s_warp[q] : T(0);
    all += s_warp[q];
  }
  __syncthreads();
  if (total) *total = all;
  return wp + x - v;
}

// reduction over a 256-thread block, the result in every thread (fixed
// order: a butterfly within each warp, then the 8 warp values in order)
template <typename T, typename Op>
__device__ __forceinline__ T block_reduce256(T v, T *s_warp, Op op) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = op(v, __shfl_xor_sync(0xffffffffu, v, o));
  if ((threadIdx.x & 31) == 0) s_warp[threadIdx.x >> 5] = v;
  __syncthreads();
  T r = s_warp[0];
#pragma unroll
  for (int q = 1; q < RS_WARPS; ++q) r = op(r, s_warp[q]);
  __syncthreads();
  return r;
}

// digit histograms of every pass in one read of the keys
template <typename K>
__global__ void __launch_bounds__(256) k_rs_hist(const K *__restrict__ keys, long long n, int begin_bit,
                                                 int end_bit, unsigned *__restrict__ hist) {
  __shared__ unsigned sh[8][RS_BINS];
  const int passes = (end_bit - begin_bit + 7) / 8;
  for (int i = threadIdx.x; i < 8 * RS_BINS; i += blockDim.x) (&sh[0][0])[i] = 0;
  __syncthreads();
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    const K k = keys[i];
    for (int p = 0; p < passes; ++p) {
      const int sh_ = begin_bit + 8 * p;
      const int bits = end_bit - sh_ < 8 ? end_bit - sh_ : 8;
      atomicAdd(&sh[p][static_cast<unsigned>(k >> sh_) & ((1u << bits) - 1)], 1u);
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < passes * RS_BINS; i += blockDim.x) {
    const unsigned c = (&sh[0][0])[i];
    if (c) atomicAdd(hist + i, c);
  }
}

// one 8-bit digit pass: kin/vin -> kout/vout (vin == nullptr: values are the
// input positions).  hist = this pass's 256 digit counts; look = one word
// per (tile, digit), zeroed; ticket = zeroed tile counter.
template <typename K, int IT = RsItems<K>::v>
__global__ void __launch_bounds__(RS_THREADS) k_rs_pass(const K *__restrict__ kin, const int *__restrict__ vin,
                                                        K *__restrict__ kout, int *__restrict__ vout,
                                                        long long n, int shift, int bits,
                                                        const unsigned *__restrict__ hist,
                                                        unsigned long long *look, unsigned *ticket) {
  constexpr int TILE = RS_THREADS * IT;
  __shared__ K sk[TILE];
  __shared__ int sv[TILE];
  __shared__ unsigned whist[RS_WARPS][RS_BINS];
  __shared__ unsigned s_excl[RS_BINS];
  __shared__ long long s_base[RS_BINS];
  __shared__ unsigned s_warp[RS_WARPS];
  __shared__ int s_tile;
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  if (t == 0) s_tile = static_cast<int>(atomicAdd(ticket, 1u));
  for (int i = t; i < RS_WARPS * RS_BINS; i += RS_THREADS) (&whist[0][0])[i] = 0;
  __syncthreads();
  const long long tile = s_tile;
  const long long base = tile * TILE;
  const unsigned dmask = (1u << bits) - 1;
  // ---- load (warp-striped: item i of lane l is key base + w*32*IT + i*32 + l)
  K key[IT];
  int val[IT];
  unsigned rank[IT];
  const long long wbase = base + (long long)warp * 32 * IT;
#pragma unroll
  for (int i = 0; i < IT; ++i) {
    const long long idx = wbase + i * 32 + lane;
    if (idx < n) {
      key[i] = kin[idx];
      val[i] = vin ? vin[idx] : static_cast<int>(idx);
    }
  }
  // ---- stable rank inside the warp: items in (i, lane) order = input order.
  // The lanes holding the same digit come from 8 ballots (one per digit bit;
  // independent, so they pipeline -- __match_any_sync's latency serialised
  // this loop); only the warp histogram update is a dependent chain.
  const unsigned lt = (1u << lane) - 1u;
#pragma unroll
  for (int i = 0; i < IT; ++i) {
    const long long idx = wbase + i * 32 + lane;
    const bool valid = idx < n;
    const unsigned d = valid ? (static_cast<unsigned>(key[i] >> shift) & dmask) : 0u;
    unsigned peers = __ballot_sync(0xffffffffu, valid);
#pragma unroll
    for (int b = 0; b < 8; ++b) {
      const bool bit = (d >> b) & 1u;
      const unsigned bb = __ballot_sync(0xffffffffu, bit);
      peers &= bit ? bb : ~bb;
    }
    const unsigned old = valid ? whist[warp][d] : 0u;
    rank[i] = old + __popc(peers & lt);
    __syncwarp();
    if (valid && (peers & lt) == 0) whist[warp][d] = old + __popc(peers);  // the digit's first lane
    __syncwarp();
  }
  __syncthreads();
  // ---- per digit (thread t = digit t): warp offsets, tile count
  unsigned cnt = 0;
#pragma unroll
  for (int w = 0; w < RS_WARPS; ++w) {
    const unsigned c = whist[w][t];
    whist[w][t] = cnt;
    cnt += c;
  }
  unsigned long long *my = look + tile * RS_BINS + t;
  st_relaxed_u64(my, (tile == 0 ? RS_INC : RS_AGG) | cnt);
  // this pass's global digit offsets (exclusive scan of the histogram)
  const unsigned goff = block_excl_sum256(hist[t], s_warp);
  const unsigned excl = block_excl_sum256(cnt, s_warp);
  s_excl[t] = excl;
  // ---- decoupled look-back over the earlier tiles (this digit)
  unsigned long long prefix = 0;
  if (tile > 0) {
    prefix = lookback(look, tile, t);
    st_relaxed_u64(my, RS_INC | (prefix + cnt));
  }
  s_base[t] = static_cast<long long>(goff) + static_cast<long long>(prefix) - excl;
  __syncthreads();
  // ---- local sort in shared memory
#pragma unroll
  for (int i = 0; i < IT; ++i) {
    const long long idx = wbase + i * 32 + lane;
    if (idx < n) {
      const unsigned d = static_cast<unsigned>(key[i] >> shift) & dmask;
      const unsigned pos = s_excl[d] + whist[warp][d] + rank[i];
      sk[pos] = key[i];
      sv[pos] = val[i];
    }
  }
  __syncthreads();
  // ---- write out digit run by digit run
  const int valid_n = n - base < TILE ? static_cast<int>(n - base) : TILE;
  for (int j = t; j < valid_n; j += RS_THREADS) {
    const K k = sk[j];
    const unsigned d = static_cast<unsigned>(k >> shift) & dmask;
    const long long o = s_base[d] + j;
    kout[o] = k;
    vout[o] = sv[j];
  }
}

template <typename K>
inline size_t rs_temp_bytes(long long n) {
  const long long tiles = (n + rs_tile<K>() - 1) / rs_tile<K>();
  return 8 * RS_BINS * sizeof(unsigned) + 256 + static_cast<size_t>(tiles > 0 ? tiles : 1) * RS_BINS * 8;
}

// Stable sort of (keys, vals) by key bits [begin_bit, end_bit).  The data
// ping-pong between (k0, v0) and (k1, v1); *in_alt tells where the result is
// (false: k0/v0).  iota_vals: the input values are the positions 0..n-1
// (v0 is not read, only used as the ping-pong buffer).  Returns a CUDA
// error code.
template <typename K>
// hist_ready: the caller zeroed the histogram / ticket words at the front of
// tmp (rs_hist_bytes) and accumulated the digit histograms of k0 into them
// (e.g. while writing the keys) -- no histogram pass here
inline cudaError_t rs_sort_pairs(void *tmp, size_t tmp_bytes, K *k0, int *v0, K *k1, int *v1, long long n,
                                 int begin_bit, int end_bit, bool *in_alt, cudaStream_t s,
                                 bool iota_vals = false, bool hist_ready = false) {
  *in_alt = false;
  if (n <= 0 || end_bit <= begin_bit) return cudaSuccess;
  if (tmp_bytes < rs_temp_bytes<K>(n)) return cudaErrorInvalidValue;
  unsigned *hist = static_cast<unsigned *>(tmp);
  unsigned *ticket = hist + 8 * RS_BINS;  // 8 counters (one per pass)
  unsigned long long *look =
      reinterpret_cast<unsigned long long *>(static_cast<char *>(tmp) + 8 * RS_BINS * sizeof(unsigned) + 256);
  const int passes = (end_bit - begin_bit + 7) / 8;
  const long long tiles = (n + rs_tile<K>() - 1) / rs_tile<K>();
  cudaError_t e = cudaSuccess;
  if (!hist_ready) {
    e = cudaMemsetAsync(tmp, 0, 8 * RS_BINS * sizeof(unsigned) + 256, s);
    if (e != cudaSuccess) return e;
    long long hg = (n + 255) / 256;
    if (hg > 148 * 8) hg = 148 * 8;
    k_rs_hist<K><<<static_cast<unsigned>(hg), 256, 0, s>>>(k0, n, begin_bit, end_bit, hist);
  }
  K *ka = k0, *kb = k1;
  int *va = v0, *vb = v1;
  bool alt = false;
  for (int p = 0; p < passes; ++p) {
    const int shift = begin_bit + 8 * p;
    const int bits = end_bit - shift < 8 ? end_bit - shift : 8;
    e = cudaMemsetAsync(look, 0, static_cast<size_t>(tiles) * RS_BINS * 8, s);
    if (e != cudaSuccess) return e;
    k_rs_pass<K><<<static_cast<unsigned>(tiles), RS_THREADS, 0, s>>>(
        ka, (p == 0 && iota_vals) ? nullptr : va, kb, vb, n, shift, bits, hist + p * RS_BINS, look, ticket + p);
    K *tk = ka;
    ka = kb;
    kb = tk;
    int *tv = va;
    va = vb;
    vb = tv;
    alt = !alt;
  }
  *in_alt = alt;
  return cudaGetLastError();
}

// ----------------------------------------------------------------- scans
// `pad` must be a RIGHT identity of the operator (op(a, pad) == a): it fills
// the slots past the end, which never precede a real item.
constexpr int SC_THREADS = 256;
constexpr int SC_ITEMS = 8;
constexpr int SC_TILE = SC_THREADS * SC_ITEMS;

// block-wide inclusive scan of SC_ITEMS consecutive items per thread; the
// block aggregate is returned to every thread
template <typename T, typename Op>
__device__ __forceinline__ T block_incl_scan(T (&x)[SC_ITEMS], Op op, T *s_warp) {
  const int t = threadIdx.x, lane = t & 31, w = t >> 5;
#pragma unroll
  for (int i = 1; i < SC_ITEMS; ++i) x[i] = op(x[i - 1], x[i]);
  T tot = x[SC_ITEMS - 1];
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const T u = __shfl_up_sync(0xffffffffu, tot, o);
    if (lane >= o) tot = op(u, tot);
  }
  if (lane == 31) s_warp[w] = tot;
  __syncthreads();
  // carry: warps 0..w-1, then the lanes before this one (in order)
  T carry{};
  bool hc = false;
  for (int q = 0; q < w; ++q) {
    carry = hc ? op(carry, s_warp[q]) : s_warp[q];
    hc = true;
  }
  T lex = __shfl_up_sync(0xffffffffu, tot, 1);
  if (lane > 0) {
    carry = hc ? op(carry, lex) : lex;
    hc = true;
  }
  if (hc) {
#pragma unroll
    for (int i = 0; i < SC_ITEMS; ++i) x[i] = op(carry, x[i]);
  }
  T agg = s_warp[0];
  for (int q = 1; q < SC_THREADS / 32; ++q) agg = op(agg, s_warp[q]);
  __syncthreads();
  return agg;
}

template <typename T>
__device__ __forceinline__ void load_blocked(const T *__restrict__ in, long long base, long long n, T pad,
                                             T (&x)[SC_ITEMS], T *s_tile) {
  for (int i = threadIdx.x; i < SC_TILE; i += SC_THREADS) {
    const long long g = base + i;
    s_tile[i] = g < n ? in[g] : pad;
  }
  __syncthreads();
#pragma unroll
  for (int i = 0; i < SC_ITEMS; ++i) x[i] = s_tile[threadIdx.x * SC_ITEMS + i];
  __syncthreads();
}

template <typename T, typename Op>
__global__ void __launch_bounds__(SC_THREADS) k_scan_reduce(const T *__restrict__ in, long long n, Op op, T pad,
                                                            T *__restrict__ part) {
  __shared__ T s_tile[SC_TILE];
  __shared__ T s_warp[SC_THREADS / 32];
  T x[SC_ITEMS];
  load_blocked(in, (long long)blockIdx.x * SC_TILE, n, pad, x, s_tile);
  const T agg = block_incl_scan(x, op, s_warp);
  if (threadIdx.x == 0) part[blockIdx.x] = agg;
}

// exclusive scan of the block aggregates in place (one block, chunked):
// entry b becomes the combination of aggregates 0..b-1 (entry 0 unused)
template <typename T, typename Op>
__global__ void __launch_bounds__(SC_THREADS) k_scan_parts(T *part, long long np, Op op, T pad) {
  __shared__ T s_tile[SC_TILE + 1];
  __shared__ T s_warp[SC_THREADS / 32];
  T carry = pad;
  bool hc = false;
  for (long long base = 0; base < np; base += SC_TILE) {
    T x[SC_ITEMS];
    load_blocked(part, base, np, pad, x, s_tile);  // the chunk is in registers ...
    const T agg = block_incl_scan(x, op, s_warp);
#pragma unroll
    for (int i = 0; i < SC_ITEMS; ++i) s_tile[threadIdx.x * SC_ITEMS + i + 1] = hc ? op(carry, x[i]) : x[i];
    if (threadIdx.x == 0) s_tile[0] = carry;
    __syncthreads();
    // ... before its entries are overwritten with their exclusive prefixes
    const int nvalid = np - base < SC_TILE ? static_cast<int>(np - base) : SC_TILE;
    for (int i = threadIdx.x; i < nvalid; i += SC_THREADS)
      if (base + i > 0) part[base + i] = s_tile[i];
    carry = hc ? op(carry, agg) : agg;
    hc = true;
    __syncthreads();
  }
}

template <typename T, typename Op, bool EXCL>
__global__ void __launch_bounds__(SC_THREADS) k_scan_down(const T *__restrict__ in, T *__restrict__ out, long long n,
                                                          Op op, T pad, const T *__restrict__ part, T init) {
  __shared__ T s_tile[SC_TILE + 1];
  __shared__ T s_warp[SC_THREADS / 32];
  const long long base = (long long)blockIdx.x * SC_TILE;
  T x[SC_ITEMS];
  load_blocked(in, base, n, pad, x, s_tile);
  block_incl_scan(x, op, s_warp);
  const bool hc = blockIdx.x > 0;
  const T carry = hc ? part[blockIdx.x] : init;
#pragma unroll
  for (int i = 0; i < SC_ITEMS; ++i) s_tile[threadIdx.x * SC_ITEMS + i + (EXCL ? 1 : 0)] = hc ? op(carry, x[i]) : x[i];
  if (EXCL && threadIdx.x == 0) s_tile[0] = carry;
  __syncthreads();
  const int nvalid = n - base < SC_TILE ? static_cast<int>(n - base) : SC_TILE;
  for (int i = threadIdx.x; i < nvalid; i += SC_THREADS) out[base + i] = s_tile[i];
}

__device__ __forceinline__ unsigned ld_acquire_u32(const unsigned *p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_u32(unsigned *p, unsigned v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// Single-pass scan with decoupled look-back: tiles take tickets in start
// order, publish their aggregate, and warp 0 combines the predecessors'
// values 32 tiles per round trip (in tile order: the operator need not
// commute) until it meets an inclusive prefix.  One launch, one read and one
// write of the data.  Status per tile: flag (0 none, 1 aggregate, 2
// inclusive) + the two values in separate slots (an aggregate is never
// overwritten by the inclusive value a reader might be fetching).
template <typename T, typename Op, bool EXCL>
__global__ void __launch_bounds__(SC_THREADS) k_scan_1p(const T *__restrict__ in, T *__restrict__ out, long long n,
                                                        Op op, T pad, T init, unsigned *flags, T *aggv, T *incv,
                                                        unsigned *ticket) {
  __shared__ T s_tile[SC_TILE + 1];
  __shared__ T s_warp[SC_THREADS / 32];
  __shared__ T s_prefix;
  __shared__ long long s_tile_id;
  if (threadIdx.x == 0) s_tile_id = atomicAdd(ticket, 1u);
  __syncthreads();
  const long long tile = s_tile_id;
  const long long base = tile * SC_TILE;
  T x[SC_ITEMS];
  load_blocked(in, base, n, pad, x, s_tile);
  const T agg = block_incl_scan(x, op, s_warp);
  if (threadIdx.x < 32) {
    const int lane = threadIdx.x;
    if (tile == 0) {
      if (lane == 0) {
        incv[0] = agg;
        st_release_u32(flags, 2u);
      }
    } else {
      if (lane == 0) {
        aggv[tile] = agg;
        st_release_u32(flags + tile, 1u);
      }
      T prefix = pad;
      bool have = false;
      for (long long j = tile - 1;; j -= 32) {
        const long long tj = j - lane;  // lane 0 = the nearest predecessor
        unsigned f = 2u;
        T v = pad;
        if (tj >= 0) {
          do {
            f = ld_acquire_u32(flags + tj);
          } while (f == 0u);
          v = f == 2u ? incv[tj] : aggv[tj];
        }
        const unsigned incm = __ballot_sync(0xffffffffu, f == 2u);
        const int stop = incm ? __ffs(incm) - 1 : 31;  // lanes 0..stop count
        T acc = __shfl_sync(0xffffffffu, v, stop);     // the oldest first
        for (int l = stop - 1; l >= 0; --l) acc = op(acc, __shfl_sync(0xffffffffu, v, l));
        prefix = have ? op(acc, prefix) : acc;
        have = true;
        if (incm) break;
      }
      if (lane == 0) {
        incv[tile] = op(prefix, agg);
        st_release_u32(flags + tile, 2u);
        s_prefix = prefix;
      }
    }
  }
  __syncthreads();
  const bool hc = tile > 0;
  const T carry = hc ? s_prefix : init;
#pragma unroll
  for (int i = 0; i < SC_ITEMS; ++i) s_tile[threadIdx.x * SC_ITEMS + i + (EXCL ? 1 : 0)] = hc ? op(carry, x[i]) : x[i];
  if (EXCL && threadIdx.x == 0) s_tile[0] = carry;
  __syncthreads();
  const int nvalid = n - base < SC_TILE ? static_cast<int>(n - base) : SC_TILE;
  for (int i = threadIdx.x; i < nvalid; i += SC_THREADS) out[base + i] = s_tile[i];
}

template <typename T>
inline size_t scan_temp_bytes(long long n) {
  const long long np = (n + SC_TILE - 1) / SC_TILE;
  const size_t t = static_cast<size_t>(np > 0 ? np : 1);
  return 256 + ((t * 4 + 255) & ~size_t(255)) + 2 * ((t * sizeof(T) + 255) & ~size_t(255));
}

// inclusive (EXCL = false) or exclusive (EXCL = true: item 0 gets init)
// scan, one launch (k_scan_1p); in == out allowed (a tile reads its own
// input before it writes its own output, and only its own)
template <bool EXCL, typename T, typename Op>
inline cudaError_t scan(void *tmp, size_t tmp_bytes, const T *in, T *out, long long n, Op op, T pad, T init,
                        cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  if (tmp_bytes < scan_temp_bytes<T>(n)) return cudaErrorInvalidValue;
  const long long np = (n + SC_TILE - 1) / SC_TILE;
  char *b = static_cast<char *>(tmp);
  unsigned *ticket = reinterpret_cast<unsigned *>(b);
  unsigned *flags = reinterpret_cast<unsigned *>(b + 256);
  const size_t fb = (static_cast<size_t>(np) * 4 + 255) & ~size_t(255);
  T *aggv = reinterpret_cast<T *>(b + 256 + fb);
  T *incv = reinterpret_cast<T *>(b + 256 + fb + ((static_cast<size_t>(np) * sizeof(T) + 255) & ~size_t(255)));
  cudaError_t e = cudaMemsetAsync(tmp, 0, 256 + fb, s);  // ticket + flags
  if (e != cudaSuccess) return e;
  k_scan_1p<T, Op, EXCL><<<static_cast<unsigned>(np), SC_THREADS, 0, s>>>(in, out, n, op, pad, init, flags, aggv,
                                                                          incv, ticket);
  return cudaGetLastError();
}

struct OpSum {
  template <typename T>
  __host__ __device__ __forceinline__ T operator()(const T &a, const T &b) const {
    return a + b;
  }
};
struct OpMax {
  template <typename T>
  __host__ __device__ __forceinline__ T operator()(const T &a, const T &b) const {
    return a < b ? b : a;
  }
};

// ------------------------------------------------------- flagged select
// out = indices i (ascending) with flag[i] != 0; *count = how many.
static __global__ void __launch_bounds__(SC_THREADS) k_sel_count(const int *__restrict__ flag, long long n,
                                                          long long *__restrict__ part) {
  __shared__ unsigned s_warp[SC_THREADS / 32];
  const long long base = (long long)blockIdx.x * SC_TILE;
  unsigned c = 0;
  for (int i = threadIdx.x; i < SC_TILE; i += SC_THREADS)
    if (base + i < n && flag[base + i]) ++c;
  for (int o = 16; o; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
  if ((threadIdx.x & 31) == 0) s_warp[threadIdx.x >> 5] = c;
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned t = 0;
    for (int q = 0; q < SC_THREADS / 32; ++q) t += s_warp[q];
    part[blockIdx.x] = t;
  }
}

static __global__ void __launch_bounds__(SC_THREADS) k_sel_write(const int *__restrict__ flag, long long n,
                                                          const long long *__restrict__ part, long long np,
                                                          long long *__restrict__ out, long long *count) {
  __shared__ unsigned s_warp[SC_THREADS / 32];
  const long long base = (long long)blockIdx.x * SC_TILE;
  const long long off = blockIdx.x > 0 ? part[blockIdx.x] : 0;
  // blocked: thread t owns items [t*ITEMS, (t+1)*ITEMS) of the tile
  int f[SC_ITEMS];
  unsigned c = 0;
#pragma unroll
  for (int i = 0; i < SC_ITEMS; ++i) {
    const long long g = base + threadIdx.x * SC_ITEMS + i;
    f[i] = g < n && flag[g] != 0;
    c += f[i];
  }
  const unsigned ex = block_excl_sum256(c, s_warp);
  unsigned k = 0;
#pragma unroll
  for (int i = 0; i < SC_ITEMS; ++i) {
    if (f[i]) out[off + ex + k] = base + threadIdx.x * SC_ITEMS + i;
    k += f[i];
  }
  if (blockIdx.x == np - 1 && threadIdx.x == SC_THREADS - 1) *count = off + ex + c;
}

inline size_t select_temp_bytes(long long n) { return scan_temp_bytes<long long>(n); }

inline cudaError_t select_flagged(void *tmp, size_t tmp_bytes, const int *flag, long long n, long long *out,
                                  long long *count, cudaStream_t s) {
  if (n <= 0) return cudaMemsetAsync(count, 0, sizeof(long long), s);
  if (tmp_bytes < select_temp_bytes(n)) return cudaErrorInvalidValue;
  long long *part = static_cast<long long *>(tmp);
  const long long np = (n + SC_TILE - 1) / SC_TILE;
  k_sel_count<<<static_cast<unsigned>(np), SC_THREADS, 0, s>>>(flag, n, part);
  if (np > 1) k_scan_parts<long long, OpSum><<<1, SC_THREADS, 0, s>>>(part, np, OpSum(), 0ll);
  k_sel_write<<<static_cast<unsigned>(np), SC_THREADS, 0, s>>>(flag, n, part, np, out, count);
  return cudaGetLastError();
}

}  // namespace prim
}  // namespace h3d
