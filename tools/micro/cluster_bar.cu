// Cluster barrier cost and dependent-L2-load chains inside a 16-CTA cluster.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o cluster_bar.bin cluster_bar.cu
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ void csync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ void csync_relaxed() {
  asm volatile("barrier.cluster.arrive.relaxed.aligned;\n\tbarrier.cluster.wait.aligned;" ::: "memory");
}
__device__ __forceinline__ unsigned long long gns() { unsigned long long t; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)); return t; }
__global__ void k(int mode, int iters, int chain, int* buf, unsigned long long* out) {
  unsigned rank; asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
  unsigned long long t0 = gns();
  int v = threadIdx.x;
  for (int it = 0; it < iters; ++it) {
    if (mode >= 1 && threadIdx.x < 32 && rank == (unsigned)(it % 16)) {
      // dependent chain of L2 loads (ld.global.cg), then a store
      int idx = (it * 97 + threadIdx.x) & 4095;
      for (int c = 0; c < chain; ++c) idx = __ldcg(buf + idx);
      if (mode == 2) { idx = 0; for (int c = 0; c < chain; ++c) idx = __ldg(buf + 4096 + idx); }
      buf[8192 + threadIdx.x] = idx;
      v += idx;
    }
    if (mode == 3) csync_relaxed(); else csync();
  }
  unsigned long long t1 = gns();
  if (threadIdx.x == 0 && rank == 0) { out[0] = t1 - t0; out[1] = v; }
}
int main() {
  int* buf; unsigned long long* out;
  cudaMalloc(&buf, 16384 * 4); cudaMalloc(&out, 16);
  int h[16384]; for (int i = 0; i < 16384; ++i) h[i] = (i * 131 + 7) & 4095;
  cudaMemcpy(buf, h, sizeof(h), cudaMemcpyHostToDevice);
  cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  for (int cs : {16, 8, 2}) for (int mode : {0, 3, 1, 2}) for (int chain : {1, 6}) {
    if (mode == 0 || mode == 3) { if (chain != 1) continue; }
    cudaLaunchConfig_t cfg = {}; cudaLaunchAttribute at[1];
    cfg.gridDim = dim3(cs); cfg.blockDim = dim3(512);
    at[0].id = cudaLaunchAttributeClusterDimension; at[0].val.clusterDim.x = cs; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
    cfg.attrs = at; cfg.numAttrs = 1;
    int iters = 2000;
    for (int rep = 0; rep < 2; ++rep) cudaLaunchKernelEx(&cfg, k, mode, iters, chain, buf, out);
    unsigned long long r[2]; cudaMemcpy(r, out, 16, cudaMemcpyDeviceToHost);
    printf("cluster %2d mode %d chain %d: %.3f us per iteration (%s)\n", cs, mode, chain, r[0] / 1e3 / iters, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
