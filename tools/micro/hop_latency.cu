// Microbenchmark: latency of a cross-SM dependency hop (poll a value written
// by another warp, then publish your own), the unit of every sync-free
// triangular solve.  Chain of N hops; warp i waits for v[i-1] and writes v[i].
#include <cstdio>
#include <cuda_runtime.h>
constexpr long long kUnset = 0x7FF4DEADBEEF0001ll;

template <int MODE>
__device__ __forceinline__ double load(const double* p) {
  if (MODE == 0) return __ldcg(p);
  if (MODE == 1) { double v; asm volatile("ld.relaxed.gpu.global.f64 %0, [%1];" : "=d"(v) : "l"(p) : "memory"); return v; }
  if (MODE == 2) { double v; asm volatile("ld.volatile.global.f64 %0, [%1];" : "=d"(v) : "l"(p) : "memory"); return v; }
  return __ldcv(p);
}

template <int MODE, int SLEEP>
__global__ void chain(double* v, int n, int stride, unsigned long long* t) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (warp % stride != 0) return;
  const int i = warp / stride;
  if (i >= n) return;
  double x = 0.0;
  if (i > 0) {
    for (;;) {
      x = load<MODE>(v + i - 1);
      if (__double_as_longlong(x) != kUnset) break;
      if (SLEEP) __nanosleep(SLEEP);
    }
  }
  if (lane == 0) {
    if (MODE == 3) asm volatile("st.relaxed.gpu.global.f64 [%0], %1;" ::"l"(v + i), "d"(x + 1.0) : "memory");
    else __stcg(v + i, x + 1.0);
    if (i == n - 1) { unsigned long long g; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g)); *t = g; }
    if (i == 0) { unsigned long long g; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g)); t[1] = g; }
  }
}

__global__ void reset(double* v, int n) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) v[i] = __longlong_as_double(kUnset);
}

template <int MODE, int SLEEP>
void run(const char* name, int n, int stride, int blocks, double* v, unsigned long long* t) {
  float best = 1e9;
  for (int rep = 0; rep < 5; ++rep) {
    reset<<<(n + 255) / 256, 256>>>(v, n);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    cudaEventRecord(a);
    chain<MODE, SLEEP><<<blocks, 256>>>(v, n, stride, t);
    cudaEventRecord(b); cudaEventSynchronize(b);
    unsigned long long h[2]; cudaMemcpy(h, t, 16, cudaMemcpyDeviceToHost);
    float us = (h[0] - h[1]) / 1e3f;
    if (us < best) best = us;
  }
  printf("%-34s hops=%d stride=%d : %.3f us/hop\n", name, n, stride, best / (n - 1));
}

int main() {
  double* v; unsigned long long* t;
  cudaMalloc(&v, 1 << 20); cudaMalloc(&t, 64);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  // blocks = sms * 2 of 8 warps; stride 9 spreads consecutive hops over blocks/SMs
  const int blocks = sms * 2, n = (blocks * 8) / 9;
  run<0, 0>("ld.cg spin, st.cg", n, 9, blocks, v, t);
  run<0, 16>("ld.cg nanosleep16, st.cg", n, 9, blocks, v, t);
  run<0, 100>("ld.cg nanosleep100, st.cg", n, 9, blocks, v, t);
  run<1, 0>("ld.relaxed.gpu spin, st.cg", n, 9, blocks, v, t);
  run<2, 0>("ld.volatile spin, st.cg", n, 9, blocks, v, t);
  run<3, 0>("ld.cv spin, st.relaxed.gpu", n, 9, blocks, v, t);
  run<0, 0>("ld.cg spin, same-block stride1", 8, 1, 1, v, t);
  printf("sms=%d\n", sms);
  return 0;
}
