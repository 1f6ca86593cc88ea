// Device-side primitives shared by the HyKKT kernels: acquire/release
// flags, a sense-reversing grid barrier for cooperative persistent kernels,
// bounded spin-waits (a logic error must never hang the GPU), warp and
// block reductions with a fixed combination order (deterministic results).
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace hykkt::dev {

// Spin budget: ~2^31 cycles (> 1 s at 1.9 GHz) before a waiter gives up,
// raises the abort flag and lets every other waiter fall through.
constexpr long long kSpinBudget = 1ll << 31;

__device__ __forceinline__ int ld_acquire(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(int* p, int v) {
  asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void st_release(unsigned* p, unsigned v) {
  asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ int ld_relaxed(const int* p) {
  int v;
  asm volatile("ld.relaxed.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned ld_relaxed(const unsigned* p) {
  unsigned v;
  asm volatile("ld.relaxed.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed(int* p, int v) {
  asm volatile("st.relaxed.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
// acq_rel fence at gpu scope.  Cheaper than __threadfence() (fence.sc) and,
// used once per task rather than per poll, keeps L1 invalidations (the
// CCTL.IVALL an acquire at gpu scope implies) off the spin loops.
__device__ __forceinline__ void fence_gpu() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }

// Producer side of a task flag: every lane orders its own writes, the warp
// converges, one lane publishes.
__device__ __forceinline__ void warp_publish(int* flag, int value, int lane) {
  fence_gpu();
  __syncwarp();
  if (lane == 0) st_relaxed(flag, value);
}

// Values produced by other SMs inside the same launch are read through L2
// (ld.global.cg); L1 is not coherent across SMs.
__device__ __forceinline__ double ldcg(const double* p) { return __ldcg(p); }
__device__ __forceinline__ int ldcg_int(const int* p) { return __ldcg(p); }
__device__ __forceinline__ void stcg(double* p, double v) { __stcg(p, v); }
// Warp-cooperative L1 prefetch of [p, p + bytes): one 128-byte line per lane
// per round, issued before a wait so later __ldg loads of static data hit L1.
__device__ __forceinline__ void prefetch_l1(const void* p, long long bytes, int lane) {
  const char* b = reinterpret_cast<const char*>(reinterpret_cast<unsigned long long>(p) & ~127ull);
  const char* e = reinterpret_cast<const char*>(p) + bytes;
  for (const char* q = b + 128 * lane; q < e; q += 128 * 32) asm volatile("prefetch.global.L1 [%0];" ::"l"(q));
}

// Waits until *flag == want. Returns false (and raises *abort) on timeout
// or when another waiter already aborted.  The shared abort word and the
// clock are only consulted every 256 polls: thousands of waiters polling one
// word would serialise on a single L2 slice and slow every wake-up.
__device__ __forceinline__ bool wait_flag(const int* flag, int want, int* abort) {
  if (ld_relaxed(flag) != want) {
    const long long t0 = clock64();
    for (unsigned it = 1;; ++it) {
      __nanosleep(20);
      if (ld_relaxed(flag) == want) break;
      if ((it & 255u) == 0u) {
        if (ld_relaxed(abort)) return false;
        if (clock64() - t0 > kSpinBudget) {
          atomicExch(abort, 1);
          return false;
        }
      }
    }
  }
  fence_gpu();
  return true;
}

// Dynamic task ticket: warps take tasks in topological order; a warp holds
// at most one task, so the smallest unfinished task always has its
// dependencies taken by running warps (deadlock-free) and a ready task is
// never stuck behind a blocked one on the same warp.
__device__ __forceinline__ long long grab_task(unsigned* ticket, int lane) {
  unsigned t = 0;
  if (lane == 0) t = atomicAdd(ticket, 1u);
  return static_cast<long long>(__shfl_sync(0xffffffffu, t, 0));
}

struct GridBarrier {
  unsigned* count;
  unsigned* gen;
};

// Sense-reversing barrier over all blocks of a cooperative launch.
__device__ __forceinline__ void grid_sync(const GridBarrier& b, int* abort) {
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned g = ld_relaxed(b.gen);
    fence_gpu();
    const unsigned arrived = atomicAdd(b.count, 1u);
    if (arrived == gridDim.x - 1) {
      atomicExch(b.count, 0u);
      fence_gpu();
      atomicExch(b.gen, g + 1);
    } else {
      const long long t0 = clock64();
      for (unsigned it = 1; ld_relaxed(b.gen) == g; ++it) {
        if ((it & 255u) == 0u && (ld_relaxed(abort) || clock64() - t0 > kSpinBudget)) {
          atomicExch(abort, 1);
          break;
        }
        __nanosleep(20);
      }
    }
    fence_gpu();
  }
  __syncthreads();
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Block sum with a fixed order (warp tree, then warp 0 over warp partials).
// `scratch` holds >= 32 doubles of shared memory. Result valid in all threads.
__device__ __forceinline__ double block_sum(double v, double* scratch) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  v = warp_sum(v);
  __syncthreads();
  if (lane == 0) scratch[wid] = v;
  __syncthreads();
  const int nw = (blockDim.x + 31) >> 5;
  double t = (lane < nw) ? scratch[lane] : 0.0;
  if (wid == 0) {
    t = warp_sum(t);
    if (lane == 0) scratch[32] = t;
  }
  __syncthreads();
  const double r = scratch[32];
  __syncthreads();
  return r;
}

// Non-negative doubles order like their bit patterns: exact max via atomics.
__device__ __forceinline__ void atomic_max_nonneg(double* addr, double v) {
  atomicMax(reinterpret_cast<unsigned long long*>(addr),
            static_cast<unsigned long long>(__double_as_longlong(v)));
}

}  // namespace hykkt::dev
