// Same-address atomicAdd throughput with many warps (one lane each), and the
// round-trip latency seen by one warp: is a single task ticket a bottleneck?
#include <cstdio>
#include <cuda_runtime.h>
__global__ void hammer(unsigned* t, int iters, unsigned long long* cyc) {
  const int lane = threadIdx.x & 31;
  unsigned long long t0 = clock64();
  unsigned s = 0;
  for (int i = 0; i < iters; ++i) {
    unsigned v = 0;
    if (lane == 0) v = atomicAdd(t, 1u);
    s += __shfl_sync(0xffffffffu, v, 0);
  }
  if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = clock64() - t0;
  if (s == 0xffffffffu) t[1] = s;
}
int main() {
  unsigned* t; unsigned long long* c; cudaMalloc(&t, 8); cudaMalloc(&c, 8);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  for (int wpb : {1, 8, 32}) for (int bps : {1, 2}) {
    const int iters = 2000;
    cudaMemset(t, 0, 8);
    hammer<<<sms * bps, 32 * wpb>>>(t, 10, c);
    cudaEventRecord(a);
    hammer<<<sms * bps, 32 * wpb>>>(t, iters, c);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    unsigned long long cyc; cudaMemcpy(&cyc, c, 8, cudaMemcpyDeviceToHost);
    double n = double(sms) * bps * wpb * iters;
    printf("warps %6d: %.3f ms, %.2f ns per atomic (aggregate), %.0f cycles per atomic per warp\n",
           sms * bps * wpb, ms, ms * 1e6 / n, double(cyc) / iters);
  }
}
