// FP64 peak on this GPU: DFMA (CUDA cores) vs DMMA (mma.sync.m8n8k4 f64,
// the FP64 tensor path; tcgen05 has no f64 kind).  Each thread / warp runs
// independent accumulator chains long enough to hide latency; the grid
// covers every SM.  Prints TFLOP/s (2 flops per FMA).
#include <cstdio>
#include <cuda_runtime.h>

constexpr int kIters = 4096;

__global__ void dfma_kernel(double* out, double a, double b) {
  double c[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) c[i] = threadIdx.x + i;
  for (int it = 0; it < kIters; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) c[i] = fma(c[i], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) s += c[i];
  if (s == 1.2345) out[0] = s;
}

__global__ void dmma_kernel(double* out, double a0, double b0) {
  double acc[8][2];
#pragma unroll
  for (int i = 0; i < 8; ++i) acc[i][0] = acc[i][1] = threadIdx.x + i;
  const double a = a0 + threadIdx.x * 1e-9, b = b0;
  for (int it = 0; it < kIters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(acc[i][0]), "+d"(acc[i][1]) : "d"(a), "d"(b));
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += acc[i][0] + acc[i][1];
  if (s == 1.2345) out[0] = s;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* out;
  cudaMalloc(&out, 8);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int threads = 256, blocks = sms * 8;
  for (int rep = 0; rep < 2; ++rep) {
    cudaEventRecord(e0);
    dfma_kernel<<<blocks, threads>>>(out, 1.0000001, 1e-9);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    const double flops = 2.0 * 16 * kIters * double(blocks) * threads;
    if (rep) printf("DFMA: %.2f TFLOP/s (%d SMs)\n", flops / (ms * 1e-3) / 1e12, sms);
    cudaEventRecord(e0);
    dmma_kernel<<<blocks, threads>>>(out, 1.0000001, 1e-9);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    // per warp per mma: 8x8x4 FMAs = 256 FMAs = 512 flops
    const double mflops = 512.0 * 8 * kIters * double(blocks) * (threads / 32);
    if (rep) printf("DMMA m8n8k4: %.2f TFLOP/s\n", mflops / (ms * 1e-3) / 1e12);
  }
  cudaError_t err = cudaGetLastError();
  if (err != cudaSuccess) printf("error: %s\n", cudaGetErrorString(err));
  return 0;
}
