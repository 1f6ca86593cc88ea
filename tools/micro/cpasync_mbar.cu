// Validates the ring feed used by ks_run: every thread copies its 16-byte
// slice of each chunk with cp.async and arrives (noinc) on the chunk's
// mbarrier (count = copying threads); one thread waits; CTA barrier; every
// thread verifies the chunk contents.  Reports mismatches.
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ unsigned su32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
extern __shared__ __align__(128) unsigned char sm[];
__global__ void run(const double* src, int nck, int nch, int* bad, int mode) {
  const int CH = 1024;
  double* ring = (double*)sm;
  unsigned long long* bar = (unsigned long long*)(sm + CH * nch * 8);
  const int tid = threadIdx.x;
  if (tid == 0) {
    for (int i = 0; i < nch; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(bar + i)), "r"(512) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  int issued = 0, errs = 0;
  for (int c = 0; c < nck; ++c) {
    // issue window [issued, c + nch)
    for (; issued < nck && issued < c + nch; ++issued) {
      const int slot = issued % nch;
      const double* s = src + (size_t)issued * CH + 2 * tid;
      double* d = ring + slot * CH + 2 * tid;
      if (mode == 0) {
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(su32(d)), "l"(s) : "memory");
      } else {
        unsigned long long pol;
        asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
        asm volatile("cp.async.cg.shared.global.L2::cache_hint [%0], [%1], 16, %2;" ::"r"(su32(d)), "l"(s), "l"(pol) : "memory");
      }
      asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(su32(bar + slot)) : "memory");
    }
    if (tid == 0) {
      unsigned ok = 0;
      while (!ok)
        asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0,1,0,p;\n}\n"
                     : "=r"(ok) : "r"(su32(bar + c % nch)), "r"((unsigned)((c / nch) & 1)) : "memory");
    }
    __syncthreads();
    const double* chunk = ring + (c % nch) * CH;
    for (int i = tid; i < CH; i += blockDim.x) errs += chunk[i] != (double)((size_t)c * CH + i);
    __syncthreads();
  }
  if (errs) atomicAdd(bad, errs);
}
int main() {
  const int nck = 4096;
  double* h = new double[(size_t)nck * 1024];
  for (size_t i = 0; i < (size_t)nck * 1024; ++i) h[i] = (double)i;
  double* d;
  cudaMalloc(&d, (size_t)nck * 1024 * 8);
  cudaMemcpy(d, h, (size_t)nck * 1024 * 8, cudaMemcpyHostToDevice);
  int* bad;
  cudaMalloc(&bad, 4);
  for (int mode : {0, 1}) {
    for (int nch : {4, 8}) {
      cudaMemset(bad, 0, 4);
      const size_t smem = (size_t)1024 * nch * 8 + 8 * nch;
      cudaFuncSetAttribute(run, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      run<<<148, 512, smem>>>(d, nck, nch, bad, mode);
      int hb = -1;
      cudaMemcpy(&hb, bad, 4, cudaMemcpyDeviceToHost);
      printf("mode %d nch %d: mismatches %d  %s\n", mode, nch, hb, cudaGetErrorString(cudaGetLastError()));
    }
  }
}
