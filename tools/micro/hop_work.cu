// Hop latency with realistic per-hop work and background pollers.
#include <cstdio>
#include <cuda_runtime.h>
constexpr long long kUnset = 0x7FF4DEADBEEF0001ll;
__device__ __forceinline__ unsigned long long gns() { unsigned long long t; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)); return t; }
__device__ double warp_sum(double v) { for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o); return v; }
__device__ double poll(const double* p) {
  double v = __ldcg(p);
  while (__double_as_longlong(v) == kUnset) { __nanosleep(16); v = __ldcg(p); }
  return v;
}
// chain warps are every `stride`-th warp; other warps (if bg) poll a never-set
// value until the chain finishes (they watch v[n-1]).
template <int WORK>
__global__ void chain(double* v, const double* data, int n, int stride, int bg, unsigned long long* t) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (warp % stride != 0) {
    if (bg) { if (bg == 2) poll(v + n - 1); else if (lane == 0) poll(v + n - 1); }
    return;
  }
  const int i = warp / stride;
  if (i >= n) return;
  double x = 0.0;
  if (i > 0) {
    if (lane == 0) poll(v + i - 1);
    __syncwarp();
    x = __ldcg(v + i - 1);
    if (WORK >= 1) x += __ldcg(data + ((i * 977 + lane * 131) & 65535));  // scattered gather
    if (WORK >= 2) x = warp_sum(x) / (1.0 + lane);
  }
  if (lane == 0) {
    __stcg(v + i, x + 1.0);
    if (i == n - 1) t[0] = gns();
    if (i == 1) t[1] = gns();
  }
}
__global__ void reset(double* v, int n) { int i = blockIdx.x * blockDim.x + threadIdx.x; if (i < n) v[i] = __longlong_as_double(kUnset); }
__global__ void timer_res(unsigned long long* t) {
  unsigned long long a = gns(), b = a; int k = 0;
  while (k < 8) { unsigned long long c = gns(); if (c != b) { t[k++] = c - b; b = c; } }
}
template <int WORK>
void run(const char* name, int bps, int bg, double* v, const double* data, unsigned long long* t, int sms) {
  const int blocks = sms * bps, warps = blocks * 8;
  const int stride = 9, n = warps / stride;
  float best = 1e9;
  for (int rep = 0; rep < 5; ++rep) {
    reset<<<(n + 255) / 256, 256>>>(v, n);
    chain<WORK><<<blocks, 256>>>(v, data, n, stride, bg, t);
    cudaDeviceSynchronize();
    unsigned long long h[2]; cudaMemcpy(h, t, 16, cudaMemcpyDeviceToHost);
    float us = (h[0] - h[1]) / 1e3f / (n - 2);
    if (us < best) best = us;
  }
  printf("%-40s bps=%d bg=%d hops=%d : %.3f us/hop\n", name, bps, bg, n, best);
}
int main() {
  double *v, *data; unsigned long long* t;
  cudaMalloc(&v, 1 << 22); cudaMalloc(&data, 65536 * 8); cudaMemset(data, 0, 65536 * 8); cudaMalloc(&t, 128);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  timer_res<<<1, 1>>>(t); unsigned long long r[8]; cudaMemcpy(r, t, 64, cudaMemcpyDeviceToHost);
  printf("globaltimer deltas ns:"); for (int k = 0; k < 8; ++k) printf(" %llu", r[k]); printf("\n");
  run<0>("bare hop", 1, 0, v, data, t, sms);
  run<1>("hop + gather", 1, 0, v, data, t, sms);
  run<2>("hop + gather + warpsum + div", 1, 0, v, data, t, sms);
  run<2>("... 4 blocks/SM, no bg", 4, 0, v, data, t, sms);
  run<2>("... 4 blocks/SM, bg lane0 pollers", 4, 1, v, data, t, sms);
  run<2>("... 4 blocks/SM, bg 32-lane pollers", 4, 2, v, data, t, sms);
  run<2>("... 8 blocks/SM, bg 32-lane pollers", 8, 2, v, data, t, sms);
  return 0;
}
