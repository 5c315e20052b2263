// Radix-pass variants (items per thread) on 2^24 u32 pairs:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_1205_1171_b200/csrc tools/rs_bench.cu -o /tmp/rs_bench
#include <cstdio>
#include <vector>
#include "prims.cuh"
using namespace h3d::prim;

template <int IT>
float run(unsigned *k0, int *v0, unsigned *k1, int *v1, long long n, void *tmp, cudaStream_t s) {
  constexpr int TILE = RS_THREADS * IT;
  const long long tiles = (n + TILE - 1) / TILE;
  unsigned *hist = static_cast<unsigned *>(tmp);
  unsigned *ticket = hist + 8 * RS_BINS;
  unsigned long long *look = reinterpret_cast<unsigned long long *>(static_cast<char *>(tmp) + 8 * RS_BINS * 4 + 256);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  float best = 1e9;
  for (int rep = 0; rep < 5; ++rep) {
    cudaMemsetAsync(tmp, 0, 8 * RS_BINS * 4 + 256, s);
    cudaEventRecord(a, s);
    k_rs_hist<unsigned><<<148 * 8, 256, 0, s>>>(k0, n, 0, 32, hist);
    unsigned *ka = k0, *kb = k1;
    int *va = v0, *vb = v1;
    for (int p = 0; p < 4; ++p) {
      cudaMemsetAsync(look, 0, tiles * RS_BINS * 8, s);
      k_rs_pass<unsigned, IT><<<tiles, RS_THREADS, 0, s>>>(ka, p == 0 ? nullptr : va, kb, vb, n, 8 * p, 8,
                                                          hist + p * RS_BINS, look, ticket + p);
      std::swap(ka, kb);
      std::swap(va, vb);
    }
    cudaEventRecord(b, s);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    if (ms < best) best = ms;
    // restore keys for the next rep (sorted output is fine as input too)
  }
  return best;
}

int main() {
  const long long n = 1ll << 24;
  std::vector<unsigned> h(n);
  unsigned x = 12345;
  for (auto &v : h) { x = x * 1664525u + 1013904223u; v = x; }
  unsigned *k0, *k1;
  int *v0, *v1;
  void *tmp;
  cudaMalloc(&k0, n * 4); cudaMalloc(&k1, n * 4); cudaMalloc(&v0, n * 4); cudaMalloc(&v1, n * 4);
  cudaMalloc(&tmp, 64 << 20);
  cudaStream_t s;
  cudaStreamCreate(&s);
#define RUN(IT) { cudaMemcpy(k0, h.data(), n * 4, cudaMemcpyHostToDevice); \
    printf("IT=%2d  %.3f ms (%s)\n", IT, run<IT>(k0, v0, k1, v1, n, tmp, s), cudaGetErrorString(cudaGetLastError())); }
  RUN(6) RUN(8) RUN(10) RUN(12) RUN(14) RUN(16) RUN(18)
  return 0;
}
