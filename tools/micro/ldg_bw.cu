// Per-SM bandwidth of plain loads: one CTA of NT threads per SM, each thread
// keeps U independent 16-byte loads in flight (unrolled), optional stores of
// the loaded data to shared memory; also a variant with cp.async 16 B
// (LDGSTS) issued U-deep per thread.
#include <cstdio>
#include <cuda_runtime.h>
#include <cuda_pipeline.h>
extern __shared__ __align__(128) double sm[];
template <int U, bool STS>
__global__ void ldg(const double2* src, long long per_cta, double* out) {
  const double2* my = src + blockIdx.x * per_cta;
  double a = 0, b = 0;
  for (long long i = threadIdx.x; i < per_cta; i += (long long)blockDim.x * U) {
    double2 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = __ldcs(my + i + (long long)u * blockDim.x);
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if (STS) reinterpret_cast<double2*>(sm)[(threadIdx.x + u * blockDim.x) & 8191] = v[u];
      a += v[u].x;
      b += v[u].y;
    }
  }
  if (a + b == 12345.0) out[0] = a;
}
template <int U>
__global__ void ldgsts(const double2* src, long long per_cta, double* out) {
  const double2* my = src + blockIdx.x * per_cta;
  double2* buf = reinterpret_cast<double2*>(sm);
  const int nt = blockDim.x;
  long long i = threadIdx.x;
  // U groups in flight per thread
  for (int u = 0; u < U; ++u, i += nt) {
    __pipeline_memcpy_async(buf + (threadIdx.x + u * nt) % (8192), my + i, 16);
    __pipeline_commit();
  }
  double a = 0;
  int slot = 0;
  for (; i < per_cta; i += nt) {
    __pipeline_wait_prior(U - 1);
    a += buf[(threadIdx.x + slot * nt) % 8192].x;
    __pipeline_memcpy_async(buf + (threadIdx.x + slot * nt) % 8192, my + i, 16);
    __pipeline_commit();
    slot = (slot + 1) % U;
  }
  __pipeline_wait_prior(0);
  if (a == 12345.0) out[0] = a;
}
template <typename K>
void bench(const char* name, K kern, const double2* src, long long per_cta, double* out, int sms, int nt, size_t smem) {
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int grid : {sms, 1}) {
    kern<<<grid, nt, smem>>>(src, per_cta, out);
    cudaEventRecord(a);
    kern<<<grid, nt, smem>>>(src, per_cta, out);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    printf("%-14s nt %4d grid %3d: %8.1f GB/s total %6.1f GB/s per SM %s\n", name, nt, grid, per_cta * 16.0 * grid / ms / 1e6,
           per_cta * 16.0 / ms / 1e6, cudaGetErrorString(cudaGetLastError()));
  }
}
int main() {
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const long long per_cta = 1ll << 20;  // 16 MB per CTA
  double2* src;
  double* out;
  cudaMalloc(&src, per_cta * 16 * sms);
  cudaMemset(src, 1, per_cta * 16 * sms);
  cudaMalloc(&out, 8);
  for (int nt : {512, 1024}) {
    bench("ldg U1", ldg<1, false>, src, per_cta, out, sms, nt, 0);
    bench("ldg U4", ldg<4, false>, src, per_cta, out, sms, nt, 0);
    bench("ldg U8", ldg<8, false>, src, per_cta, out, sms, nt, 0);
    bench("ldg U8+sts", ldg<8, true>, src, per_cta, out, sms, nt, 131072);
    bench("ldgsts U4", ldgsts<4>, src, per_cta, out, sms, nt, 131072);
    bench("ldgsts U8", ldgsts<8>, src, per_cta, out, sms, nt, 131072);
    bench("ldgsts U16", ldgsts<16>, src, per_cta, out, sms, nt, 131072);
  }
}
