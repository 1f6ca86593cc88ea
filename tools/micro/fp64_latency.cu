// Dependent-chain latencies on B200: DFMA, DADD, double division, sqrt,
// double shuffle, warp_sum of doubles.
#include <cstdio>
#include <cuda_runtime.h>

__device__ double warp_sum(double v) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

template <int OP>
__global__ void lat(double* out, long long* cyc, double a, double b, int n) {
  double x = a + threadIdx.x * 1e-3;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) {
    if (OP == 0) x = fma(x, b, a);
    if (OP == 1) x = x + b;
    if (OP == 2) x = a / x;
    if (OP == 3) x = sqrt(x) + a;
    if (OP == 4) x = __shfl_sync(0xffffffffu, x, (threadIdx.x + 1) & 31) + 0.0;
    if (OP == 5) x = warp_sum(x) * 1e-3;
    if (OP == 6) x = __fdividef((float)x, (float)b);
    if (OP == 7) x = __drcp_rn(x) + a;
  }
  long long t1 = clock64();
  out[threadIdx.x] = x;
  if (threadIdx.x == 0) *cyc = t1 - t0;
}

int main() {
  double* o; long long* c; cudaMalloc(&o, 4096); cudaMalloc(&c, 8);
  const char* names[] = {"dfma", "dadd", "ddiv", "dsqrt+add", "shfl.f64", "warp_sum.f64(5 steps)", "fdividef", "drcp+add"};
  const int n = 1000;
  for (int rep = 0; rep < 2; ++rep) {
#define RUN(K) { lat<K><<<1, 32>>>(o, c, 1.0000001, 0.9999999, n); long long h; cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost); if (rep) printf("%-24s %.1f cycles/op\n", names[K], (double)h / n); }
    RUN(0) RUN(1) RUN(2) RUN(3) RUN(4) RUN(5) RUN(6) RUN(7)
  }
  return 0;
}
