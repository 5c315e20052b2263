// Probe: CUDA dynamic parallelism tail-launch chains on this driver/GPU.
// Does a host-stream successor wait for the whole chain?  Order?  Latency?
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_work(int *log, int *ctr, int i) {
  if (threadIdx.x == 0 && blockIdx.x == 0) log[atomicAdd(ctr, 1)] = 1000 + i;
}
__global__ void k_step(int *log, int *ctr, int i, int depth) {
  log[atomicAdd(ctr, 1)] = i;
  if (i + 1 < depth) {
    k_work<<<4, 64, 0, cudaStreamTailLaunch>>>(log, ctr, i);
    k_step<<<1, 1, 0, cudaStreamTailLaunch>>>(log, ctr, i + 1, depth);
  }
}
__global__ void k_after(int *log, int *ctr) { log[atomicAdd(ctr, 1)] = -1; }
__global__ void k_empty() {}

int main() {
  int *log, *ctr;
  cudaMalloc(&log, 4096 * 4);
  cudaMalloc(&ctr, 4);
  cudaStream_t s;
  cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  for (int depth : {5, 30, 100}) {
    cudaMemsetAsync(ctr, 0, 4, s);
    cudaMemsetAsync(log, 0xff, 4096 * 4, s);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a, s);
    k_step<<<1, 1, 0, s>>>(log, ctr, 0, depth);
    k_after<<<1, 1, 0, s>>>(log, ctr);
    cudaEventRecord(b, s);
    cudaError_t e = cudaStreamSynchronize(s);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    int h[4096], c;
    cudaMemcpy(&c, ctr, 4, cudaMemcpyDeviceToHost);
    cudaMemcpy(h, log, 4096 * 4, cudaMemcpyDeviceToHost);
    printf("depth %d: err=%s count=%d time=%.3f ms (%.2f us/step)\n  log:", depth, cudaGetErrorString(e), c, ms,
           1e3 * ms / depth);
    int bad = 0;
    for (int k = 0; k < c; ++k) {
      if (k < 12) printf(" %d", h[k]);
      int expv = (k == c - 1) ? -1 : ((k & 1) ? 1000 + k / 2 : k / 2);
      if (h[k] != expv) bad++;
    }
    printf(" ... last %d | mismatches vs expected order: %d\n", h[c - 1], bad);
  }
  // reference: host launch latency of 100 empty kernels back to back
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a, s);
  for (int i = 0; i < 100; ++i) k_empty<<<1, 1, 0, s>>>();
  cudaEventRecord(b, s);
  cudaStreamSynchronize(s);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  printf("100 host-launched empty kernels: %.3f ms\n", ms);
  return 0;
}
