// Microbenchmark: per-CTA streaming through a shared-memory ring filled by
// TMA bulk copies (cp.async.bulk + mbarrier), one CTA per SM, each CTA
// streaming its own region.  Consumers sum every element, and the CTA
// synchronises every `step` chunks (the stream interpreter's step barrier).
// Reports aggregate GB/s and the mean issue->complete latency of a chunk.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tma_ring tma_ring.cu
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned su32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mb_init(unsigned long long* b) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(b)) : "memory");
}
__device__ __forceinline__ void mb_tx(unsigned long long* b, unsigned n) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(n) : "memory");
}
__device__ __forceinline__ void mb_wait(unsigned long long* b, unsigned par) {
  unsigned ok = 0;
  while (!ok) {
    asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0,1,0,p;\n}\n"
                 : "=r"(ok) : "r"(su32(b)), "r"(par) : "memory");
  }
}
__device__ __forceinline__ void tma(void* d, const void* s, unsigned n, unsigned long long* b) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(su32(d)),
               "l"(s), "r"(n), "r"(su32(b)) : "memory");
}
__device__ __forceinline__ unsigned long long gt() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

extern __shared__ __align__(128) unsigned char sm[];
__global__ void ring(const double* src, long long per_cta, int chunk, int nch, int step, double* out,
                     unsigned long long* lat, int touch) {
  double* buf = (double*)sm;
  unsigned long long* bar = (unsigned long long*)(sm + (size_t)chunk * nch * 8);
  unsigned long long* tis = bar + nch;
  const double* my = src + blockIdx.x * per_cta;
  const long long nck = per_cta / chunk;
  if (threadIdx.x == 0) {
    for (int i = 0; i < nch; ++i) mb_init(bar + i);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  double acc = 0;
  long long issued = 0;
  unsigned long long lsum = 0;
  for (long long c0 = 0; c0 < nck; c0 += step) {
    if (threadIdx.x == 0) {
      for (; issued < nck && issued < c0 + nch; ++issued) {
        const int s = issued % nch;
        if (lat) tis[s] = clock64();
        mb_tx(bar + s, chunk * 8);
        tma(buf + (size_t)s * chunk, my + issued * chunk, chunk * 8, bar + s);
      }
      for (long long c = c0; c < c0 + step && c < nck; ++c) {
        mb_wait(bar + c % nch, (c / nch) & 1);
        if (lat) lsum += clock64() - tis[c % nch];
      }
    }
    __syncthreads();
    if (touch) {
      for (long long c = c0; c < c0 + step && c < nck; ++c) {
        const double* b = buf + (size_t)(c % nch) * chunk;
        for (int i = threadIdx.x; i < chunk; i += blockDim.x) acc += b[i];
      }
    }
    __syncthreads();
  }
  if (acc == 12345.0) out[0] = acc;
  if (threadIdx.x == 0 && lat) lat[blockIdx.x] = lsum / nck;
}

int main(int argc, char** argv) {
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const long long per_cta = 1ll << 21;  // 16 MB per CTA
  double* src;
  cudaMalloc(&src, per_cta * sms * 8);
  cudaMemset(src, 0, per_cta * sms * 8);
  double* out;
  cudaMalloc(&out, 8);
  unsigned long long* lat;
  cudaMalloc(&lat, sms * 8);
  int cfgs[][3] = {{1024, 8, 1}, {1024, 8, 2}, {1024, 8, 4}, {1024, 8, 6}, {2048, 4, 1}, {512, 16, 1},
                   {512, 16, 4}, {1024, 12, 1}, {1024, 16, 1}, {2048, 8, 1}, {4096, 4, 1}, {256, 32, 1}};
  for (auto& c : cfgs) {
    const int chunk = c[0], nch = c[1], step = c[2];
    const size_t smem = (size_t)chunk * nch * 8 + 16 * nch;
    cudaFuncSetAttribute(ring, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    for (int grid : {sms, 1}) {
      cudaEvent_t a, b;
      cudaEventCreate(&a);
      cudaEventCreate(&b);
     for (int touch : {1, 0}) {
      ring<<<grid, 512, smem>>>(src, per_cta, chunk, nch, step, out, nullptr, touch);
      cudaEventRecord(a);
      ring<<<grid, 512, smem>>>(src, per_cta, chunk, nch, step, out, nullptr, touch);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      ring<<<grid, 512, smem>>>(src, per_cta, chunk, nch, step, out, lat, touch);
      unsigned long long h[256];
      cudaMemcpy(h, lat, grid * 8, cudaMemcpyDeviceToHost);
      double l = 0;
      for (int i = 0; i < grid; ++i) l += h[i];
      printf("chunk %5d B x %2d  step %d  touch %d grid %3d: %8.1f GB/s  (%.1f GB/s per SM)  chunk issue->done %.0f cycles  %s\n",
             chunk * 8, nch, step, touch, grid, per_cta * grid * 8 / ms / 1e6, per_cta * 8 / ms / 1e6, l / grid,
             cudaGetErrorString(cudaGetLastError()));
     }
    }
  }
  return 0;
}
