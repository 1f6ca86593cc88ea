// Microbenchmark: per-SM streaming bandwidth of one CTA (512 threads) with
// different transports into shared memory, 148 CTAs, each streaming its own
// 16 MB region in "chunks" with a CTA barrier per chunk (the stream
// interpreter's access pattern):
//   tma1    cp.async.bulk by thread 0, nch chunks in flight
//   tma4    cp.async.bulk, chunk c issued by warp c % 4
//   tmasplit one chunk = 8 bulk copies issued by 8 warps
//   ldgsts  cp.async 16 B per thread, commit group per chunk, depth nch
//   ldg     plain 16 B loads to registers (depth 1 chunk ahead), st.shared
#include <cstdio>
#include <cuda_runtime.h>
#include <cuda_pipeline.h>

__device__ __forceinline__ unsigned su32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mb_init(unsigned long long* b, int n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(n) : "memory");
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

extern __shared__ __align__(128) unsigned char sm[];

template <int MODE>
__global__ void __launch_bounds__(512, 1) run(const double* src, long long per_cta, int chunk, int nch, double* out) {
  double* buf = (double*)sm;
  unsigned long long* bar = (unsigned long long*)(sm + (size_t)chunk * nch * 8);
  const double* my = src + blockIdx.x * per_cta;
  const long long nck = per_cta / chunk;
  const int tid = threadIdx.x, wid = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    for (int i = 0; i < nch; ++i) mb_init(bar + i, MODE == 2 ? 8 : 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  double acc = 0;
  if (MODE <= 2) {
    long long issued = 0;
    for (long long c = 0; c < nck; ++c) {
      for (; issued < nck && issued < c + nch; ++issued) {
        const int s = issued % nch;
        if (MODE == 0 && tid == 0) {
          mb_tx(bar + s, chunk * 8);
          tma(buf + (size_t)s * chunk, my + issued * chunk, chunk * 8, bar + s);
        } else if (MODE == 1 && lane == 0 && wid == (int)(issued % 4)) {
          mb_tx(bar + s, chunk * 8);
          tma(buf + (size_t)s * chunk, my + issued * chunk, chunk * 8, bar + s);
        } else if (MODE == 2 && lane == 0 && wid < 8) {
          const int part = chunk / 8;
          mb_tx(bar + s, part * 8);
          tma(buf + (size_t)s * chunk + wid * part, my + issued * chunk + wid * part, part * 8, bar + s);
        }
      }
      mb_wait(bar + c % nch, (c / nch) & 1);
      const double* b = buf + (size_t)(c % nch) * chunk;
      for (int i = tid; i < chunk; i += 512) acc += b[i];
      __syncthreads();
    }
  } else if (MODE == 3) {
    // cp.async 16 B per thread
    long long issued = 0;
    for (long long c = 0; c < nck; ++c) {
      for (; issued < nck && issued < c + nch; ++issued) {
        const int s = issued % nch;
        for (int i = tid * 2; i < chunk; i += 1024) {
          __pipeline_memcpy_async(buf + (size_t)s * chunk + i, my + issued * chunk + i, 16);
        }
        __pipeline_commit();
      }
      // groups committed after chunk c: issued - 1 - c
      const long long ahead = issued - 1 - c;
      if (ahead >= 7) __pipeline_wait_prior(7);
      else if (ahead == 6) __pipeline_wait_prior(6);
      else if (ahead == 5) __pipeline_wait_prior(5);
      else if (ahead == 4) __pipeline_wait_prior(4);
      else if (ahead == 3) __pipeline_wait_prior(3);
      else if (ahead == 2) __pipeline_wait_prior(2);
      else if (ahead == 1) __pipeline_wait_prior(1);
      else __pipeline_wait_prior(0);
      __syncthreads();
      const double* b = buf + (size_t)(c % nch) * chunk;
      for (int i = tid; i < chunk; i += 512) acc += b[i];
      __syncthreads();
    }
  } else {
    // plain loads, nch chunks ahead held in registers is impossible; one chunk ahead
    double2 r[8];
    const int per = chunk / 1024;  // double2 per thread per chunk
    for (int k = 0; k < per && k < 8; ++k) r[k] = ((const double2*)my)[tid + k * 512];
    for (long long c = 0; c < nck; ++c) {
      const int s = c % nch;
      for (int k = 0; k < per && k < 8; ++k) ((double2*)(buf + (size_t)s * chunk))[tid + k * 512] = r[k];
      if (c + 1 < nck)
        for (int k = 0; k < per && k < 8; ++k) r[k] = ((const double2*)(my + (c + 1) * chunk))[tid + k * 512];
      __syncthreads();
      const double* b = buf + (size_t)s * chunk;
      for (int i = tid; i < chunk; i += 512) acc += b[i];
      __syncthreads();
    }
  }
  if (acc == 12345.0) out[0] = acc;
}

template <int MODE>
void bench(const char* name, const double* src, long long per_cta, int chunk, int nch, double* out, int sms) {
  const size_t smem = (size_t)chunk * nch * 8 + 8 * nch;
  cudaFuncSetAttribute(run<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  run<MODE><<<sms, 512, smem>>>(src, per_cta, chunk, nch, out);
  cudaEventRecord(a);
  run<MODE><<<sms, 512, smem>>>(src, per_cta, chunk, nch, out);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  printf("%-8s chunk %6d B x %2d: %8.1f GB/s total (%5.1f GB/s per SM) %s\n", name, chunk * 8, nch,
         per_cta * sms * 8 / ms / 1e6, per_cta * 8 / ms / 1e6, cudaGetErrorString(cudaGetLastError()));
}

int main() {
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const long long per_cta = 1ll << 21;
  double *src, *out;
  cudaMalloc(&src, per_cta * sms * 8);
  cudaMemset(src, 0, per_cta * sms * 8);
  cudaMalloc(&out, 8);
  int cfg[][2] = {{1024, 8}, {2048, 4}, {2048, 8}, {4096, 4}, {1024, 16}};
  for (auto& c : cfg) {
    bench<0>("tma1", src, per_cta, c[0], c[1], out, sms);
    bench<1>("tma4", src, per_cta, c[0], c[1], out, sms);
    bench<2>("tmasplit", src, per_cta, c[0], c[1], out, sms);
    bench<3>("ldgsts", src, per_cta, c[0], c[1], out, sms);
    bench<4>("ldg", src, per_cta, c[0], c[1], out, sms);
  }
  return 0;
}
