// TMA bulk-copy throughput with K independent issuing threads (one per warp,
// each with its own ring of nch chunks and mbarriers) in one CTA per SM.
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ unsigned su32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
extern __shared__ __align__(128) unsigned char sm[];
__global__ void run(const char* src, long long per_issuer, int chunk, int nch, int K, long long* out) {
  const int w = threadIdx.x >> 5;
  if ((threadIdx.x & 31) || w >= K) return;
  unsigned char* ring = sm + (size_t)w * chunk * nch;
  unsigned long long* bar = (unsigned long long*)(sm + (size_t)K * chunk * nch) + w * nch;
  for (int i = 0; i < nch; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(bar + i)) : "memory");
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  const char* my = src + ((size_t)blockIdx.x * K + w) * per_issuer;
  const long long nck = per_issuer / chunk;
  long long issued = 0;
  for (long long c = 0; c < nck; ++c) {
    for (; issued < nck && issued < c + nch; ++issued) {
      const int s = issued % nch;
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(bar + s)), "r"(chunk) : "memory");
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                       su32(ring + (size_t)s * chunk)), "l"(my + issued * chunk), "r"(chunk), "r"(su32(bar + s)) : "memory");
    }
    unsigned ok = 0;
    while (!ok)
      asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0,1,0,p;\n}\n"
                   : "=r"(ok) : "r"(su32(bar + c % nch)), "r"((unsigned)((c / nch) & 1)) : "memory");
  }
  out[blockIdx.x] = issued;
}
int main() {
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const long long total_per_cta = 32ll << 20;
  char* src;
  long long* out;
  cudaMalloc(&src, total_per_cta * sms);
  cudaMemset(src, 1, total_per_cta * sms);
  cudaMalloc(&out, 8 * sms);
  for (int chunk : {8192, 16384}) {
    for (int K : {1, 2, 4, 8}) {
      const int nch = 4;
      const size_t smem = (size_t)K * chunk * nch + 8 * K * nch;
      if (smem > 200000) continue;
      cudaFuncSetAttribute(run, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      cudaEvent_t a, b;
      cudaEventCreate(&a);
      cudaEventCreate(&b);
      const long long per = total_per_cta / K;
      run<<<sms, 256, smem>>>(src, per, chunk, nch, K, out);
      cudaEventRecord(a);
      run<<<sms, 256, smem>>>(src, per, chunk, nch, K, out);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      printf("chunk %6d x %d per issuer, %d issuers: %8.1f GB/s total  %6.1f GB/s per SM  %.0f ns per copy per issuer %s\n",
             chunk, nch, K, total_per_cta * sms / ms / 1e6, total_per_cta / ms / 1e6, ms * 1e6 / (per / chunk),
             cudaGetErrorString(cudaGetLastError()));
    }
  }
}
