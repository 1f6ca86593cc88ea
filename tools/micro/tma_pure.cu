// Pure TMA streaming: thread 0 issues 1-D bulk copies into an nch-deep ring
// and waits for them in order; no consumers, no CTA barriers.  `wrap` bytes:
// the source offset wraps every `wrap` bytes (small wrap = L2-resident).
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ unsigned su32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
extern __shared__ __align__(128) unsigned char sm[];
__global__ void run(const char* src, long long per_cta, long long wrap, int chunk, int nch, long long* out) {
  unsigned long long* bar = (unsigned long long*)(sm + (size_t)chunk * nch);
  if (threadIdx.x != 0) return;
  for (int i = 0; i < nch; ++i)
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(bar + i)) : "memory");
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  const char* my = src + blockIdx.x * per_cta;
  const long long nck = per_cta / chunk;
  long long issued = 0;
  for (long long c = 0; c < nck; ++c) {
    for (; issued < nck && issued < c + nch; ++issued) {
      const int s = issued % nch;
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(bar + s)), "r"(chunk) : "memory");
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                       su32(sm + (size_t)s * chunk)),
                   "l"(my + (issued * chunk) % wrap), "r"(chunk), "r"(su32(bar + s))
                   : "memory");
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
  const long long per_cta = 16ll << 20;
  char* src;
  long long* out;
  cudaMalloc(&src, per_cta * sms);
  cudaMemset(src, 1, per_cta * sms);
  cudaMalloc(&out, 8 * sms);
  int cfg[][2] = {{8192, 8}, {8192, 16}, {16384, 8}, {32768, 4}, {4096, 16}, {2048, 32}, {65536, 2}};
  for (long long wrap : {per_cta, 1ll << 16}) {
    for (auto& c : cfg) {
      for (int grid : {sms, 1}) {
        const size_t smem = (size_t)c[0] * c[1] + 8 * c[1];
        cudaFuncSetAttribute(run, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        cudaEvent_t a, b;
        cudaEventCreate(&a);
        cudaEventCreate(&b);
        run<<<grid, 32, smem>>>(src, per_cta, wrap, c[0], c[1], out);
        cudaEventRecord(a);
        run<<<grid, 32, smem>>>(src, per_cta, wrap, c[0], c[1], out);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        printf("wrap %9lld chunk %6d x %2d grid %3d: %8.1f GB/s total  %6.1f GB/s per SM  %.0f ns per chunk  %s\n", wrap,
               c[0], c[1], grid, per_cta * grid / ms / 1e6, per_cta / ms / 1e6, ms * 1e6 / (per_cta / c[0]),
               cudaGetErrorString(cudaGetLastError()));
      }
    }
  }
}
