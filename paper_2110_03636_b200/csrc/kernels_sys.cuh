// System-per-CTA batched solve (BASELINE configs[4]): one CTA owns one KKT
// system at a time and runs, without any grid-wide synchronisation, the
// whole post-factorization half of solve_reduced / solve_full
// (proj/core/src/solver.cpp:252-287, ruiz.cpp:118-133, kkt_system.cpp:89-105):
//
//   w  = H^-1 r_hat_x                     (factor_solve, cholesky.cpp:139-168)
//   rhs = J w - r_y                       (solver.cpp:254-255)
//   cg_schur with the delta2 restart      (solver.cpp:154-201, 257-264)
//   dx = H^-1 (r_hat_x - J^T dy)          (solver.cpp:280-286)
//   unscale_solution + recover            (ruiz.cpp:118-133, kkt_system.cpp:89-105)
//
// The permuted solve vector (n_x doubles) lives in shared memory for the
// whole system.  The Schur operator's data arrive as two streams laid out
// in consumption order (sysplan.cpp, format in sysplan_format.h): the
// per-system value stream (L with reciprocal diagonals, J) and the shared
// index stream (step headers, descriptors, gather indices).  All threads
// copy the next chunks of both into shared-memory rings ahead of the
// consumers (cp.async, completion counted on one mbarrier per chunk), and
// thread 0 waits for the next step's chunks before each step's closing
// barrier, so the supernode-tree dependency chain only ever waits on shared
// memory and CTA barriers.  The CG vectors are owned per thread
// (index k = tid + j * NT).
#pragma once

#include "device_util.cuh"
#include "sysplan_format.h"

namespace hykkt::dev {

// ---- TMA bulk copy + mbarrier primitives (sm_90+ PTX, used on sm_100a) ----
__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_fence_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(unsigned long long* bar, unsigned parity) {
  unsigned ok;
  asm volatile(
      "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned parity) {
  while (!mbar_try_wait(bar, parity)) {
  }
}
__device__ __forceinline__ unsigned long long policy_evict_first() {
  unsigned long long p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ unsigned long long policy_evict_last() {
  unsigned long long p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ void tma_load_1d(void* dst, const void* src, unsigned bytes, unsigned long long* bar,
                                            unsigned long long policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}


// cp.async (LDGSTS) 16-byte copies with mbarrier completion: one TMA
// bulk copy per SM completes at a time (~400 ns each, whatever its size;
// tools/micro/tma_pure.cu), so small ring chunks are fed by all threads
// instead (tools/micro/ldg_bw.cu: ~48 GB/s per SM, HBM-saturating).
__device__ __forceinline__ void cp_async16(void* dst, const void* src, unsigned long long policy) {
  asm volatile("cp.async.cg.shared.global.L2::cache_hint [%0], [%1], 16, %2;" ::"r"(smem_u32(dst)), "l"(src),
               "l"(policy)
               : "memory");
}
// arrives on `bar` when all of this thread's prior cp.async copies landed
__device__ __forceinline__ void cp_async_arrive(unsigned long long* bar) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(bar)) : "memory");
}

struct KsArgs {
  int n, mc, md;
  // stream program (index stream shared by all systems)
  const int* idx;
  const double* vals;   // [B][vlen] value streams
  long long vlen;       // per-system value stream length (chunk multiple)
  int vchunk_lg, nvchunk, ichunk_lg, nichunk, pmax;
  long long bv0[4], bv1[4], bi0[4], bi1[4];  // block extents (JT, FWD, BWD, J)
  int bs0[4], bs1[4];
  const int* perm;      // perm[new] = old
  const int* iperm;
  const double* rhat;   // [B][n]
  const double* rys;    // [B][mc]
  // unscale + recover
  const double* d;      // [B][n + mc] Ruiz factors
  const int* jd_rp;
  const int* jd_ci;
  const int* jd_src;
  const double* jd;     // [B][nnz_jd] original J_d values
  long long nnz_jd;
  const double* ds_in;  // [B][md] D_s
  const double* rs;     // [B][md]
  const double* ryd;    // [B][md]
  double* odx;          // [B][n]
  double* ody;          // [B][mc]
  double* ods;          // [B][md]
  double* odyd;         // [B][md]
  // CG
  double* scratch;      // gridDim.x x 5 x mc: x, r, p, q, rhs
  double tol, thr, delta2;
  long long max_iter;
  const int* ok;        // [B] 1 = factorization succeeded
  long long* iters;     // [B]
  double* relres;       // [B]
  int* flags;           // [B] 1 converged, 2 small quadratic
  double* d2used;       // [B]
  unsigned* ticket;     // system counter (zero on entry)
  const int* order;     // ticket -> system (longest previous CG first), or null = identity
  int B;
  unsigned long long* prof;   // diagnostics: kPrN per CTA, or null
  unsigned long long* trace;  // diagnostics: CTA 0's first CG operator: end time per step
  int debug;                  // 1: the producer drains every issued chunk before each barrier
  int issuers;                // warps issuing TMA copies (feed 1)
  int feed;                   // 0 cp.async by all threads, 1 TMA bulk copies
};

// Per-CTA phase timers (thread 0's view, %globaltimer ns) when KsArgs::prof
// is set.
enum KsProf { kPrRhs, kPrWait, kPrA, kPrB, kPrPre, kPrJrow, kPrUpd, kPrPupd, kPrRecover, kPrSteps, kPrSolves,
              kPrIters, kPrJ, kPrSync, kPrN = 16 };
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
struct KsTimer {
  unsigned long long* acc;  // shared, kPrN counters (null = off)
  unsigned long long last;
  __device__ __forceinline__ void start() {
    if (acc && threadIdx.x == 0) last = gtimer();
  }
  __device__ __forceinline__ void lap(int i) {
    if (acc && threadIdx.x == 0) {
      const unsigned long long t = gtimer();
      acc[i] += t - last;
      last = t;
    }
  }
  __device__ __forceinline__ void count(int i, unsigned long long v = 1) {
    if (acc && threadIdx.x == 0) acc[i] += v;
  }
};

// dynamic shared memory of ks_solve (namespace scope, so helpers that derive
// pointers from it keep the shared address space: loads stay LDS, not
// generic)
extern __shared__ __align__(128) unsigned char ks_smem[];

struct KsSmem {
  double* v;
  double* rv;  // value ring
  int* ri;     // index ring
  double* part;
  unsigned long long* barv;
  unsigned long long* bari;
  double* red;  // 66
  int* sys;  // [0] system ticket, [2..3] late flags, [4..11] issue ranges (both by step parity)
  unsigned long long* prof;
};


// Shared-memory map of ks_solve: rings first (TMA destinations, aligned),
// then mbarriers, reduction scratch, flags, timers, partials, solve vector.
__device__ __forceinline__ KsSmem ks_layout(int nvchunk, int vchunk_lg, int nichunk, int ichunk_lg, int pmax) {
  KsSmem S;
  unsigned char* p = ks_smem;
  S.rv = reinterpret_cast<double*>(p);
  p += (8ll * nvchunk) << vchunk_lg;
  S.ri = reinterpret_cast<int*>(p);
  p += (4ll * nichunk) << ichunk_lg;
  S.barv = reinterpret_cast<unsigned long long*>(p);
  p += 8 * nvchunk;
  S.bari = reinterpret_cast<unsigned long long*>(p);
  p += 8 * nichunk;
  S.red = reinterpret_cast<double*>(p);
  p += 8 * 66;
  S.sys = reinterpret_cast<int*>(p);
  p += 64;
  S.prof = reinterpret_cast<unsigned long long*>(p);
  p += 8 * kPrN;
  S.part = reinterpret_cast<double*>(p);
  p += 8 * pmax;
  S.v = reinterpret_cast<double*>(p);
  return S;
}

// One stream's ring state (uniform across the CTA: every thread evolves it
// identically; thread 0 alone issues copies).
struct KsStream {
  long long G;       // global chunk index of the current run's first chunk
  long long issued;  // next global chunk to issue
  long long ready;   // last global chunk known complete to every thread
};

template <int NT>
__device__ __forceinline__ double ks_sum(double v, double* red) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  v = warp_sum(v);
  if (lane == 0) red[wid] = v;
  __syncthreads();
  double t = lane < NT / 32 ? red[lane] : 0.0;
  t = warp_sum(t);
  __syncthreads();  // red reusable afterwards
  return t;
}

template <int NT>
__device__ __forceinline__ double2 ks_sum2(double a, double b, double* red) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  a = warp_sum(a);
  b = warp_sum(b);
  if (lane == 0) {
    red[wid] = a;
    red[32 + wid] = b;
  }
  __syncthreads();
  double ta = lane < NT / 32 ? red[lane] : 0.0;
  double tb = lane < NT / 32 ? red[32 + lane] : 0.0;
  ta = warp_sum(ta);
  tb = warp_sum(tb);
  __syncthreads();
  return make_double2(ta, tb);
}

// J-step row consumer (runtime mode keeps one copy of the interpreter):
//   kJSchur  Schur rhs J w - r_y (solver.cpp:254-255)
//   kJCg     q = J t + delta2 p and curvature / |p|^2 partials
//            (solver.cpp:144-152, 172-176)
enum { kJNone = 0, kJSchur = 1, kJCg = 2 };
struct KsJOut {
  int mode;
  double* out;       // rhs (schur) or q (cg)
  const double* in;  // r_y (schur) or p (cg)
  double d2;
  double s1, s2;     // schur: |rhs|^2 ; cg: p.q, p.p
  __device__ __forceinline__ void row(int k, double acc) {
    if (mode == kJSchur) {
      const double v0 = __dsub_rn(acc, in[k]);
      out[k] = v0;
      s1 = fma(v0, v0, s1);
    } else if (mode == kJCg) {
      const double pk = in[k];
      if (d2 != 0.0) acc = __dadd_rn(acc, __dmul_rn(d2, pk));
      out[k] = acc;
      s1 = fma(pk, acc, s1);
      s2 = fma(pk, pk, s2);
    }
  }
};

// Ring view of one step: entry e of the step's value / index range.
struct KsRing {
  const double* rv;
  const int* ri;
  int bv, bi, vmask, imask;
  __device__ __forceinline__ double V(int e) const { return rv[(bv + e) & vmask]; }
  __device__ __forceinline__ int I(int e) const { return ri[(bi + e) & imask]; }
};

// Thread task (narrow supernode): one thread solves the supernode's
// diagonal block after its gathers.  One compact code path for every width
// (solved values are re-read from the shared vector, not kept in register
// arrays): a per-width unrolled version multiplies the kernel's code size
// and the step interpreter then stalls on instruction-cache misses.
__device__ __forceinline__ void ks_fwd_thread(const KsRing& R, double* v, const double* part, int voff, int ioff,
                                              int f, int w, bool inl) {
  int e = voff + w * (w + 1) / 2, ig = ioff + w + 1;
#pragma unroll 1
  for (int r = 0; r < w; ++r) {
    const int rowo = voff + r * (r + 1) / 2;
    double acc = v[f + r];
    if (inl) {
      const int c = R.I(ioff + r);
      double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
      int k = 0;
      for (; k + 4 <= c; k += 4) {
        a0 = fma(R.V(e + k), v[R.I(ig + k)], a0);
        a1 = fma(R.V(e + k + 1), v[R.I(ig + k + 1)], a1);
        a2 = fma(R.V(e + k + 2), v[R.I(ig + k + 2)], a2);
        a3 = fma(R.V(e + k + 3), v[R.I(ig + k + 3)], a3);
      }
      for (; k < c; ++k) a0 = fma(R.V(e + k), v[R.I(ig + k)], a0);
      acc -= (a0 + a1) + (a2 + a3);
      e += c;
      ig += c;
    } else {
      for (int g = R.I(ioff + r), g1 = R.I(ioff + r + 1); g < g1; ++g) acc -= part[g];
    }
    for (int j = 0; j < r; ++j) acc = fma(-R.V(rowo + j), v[f + j], acc);
    v[f + r] = acc * R.V(rowo + r);
  }
}

__device__ __forceinline__ void ks_bwd_thread(const KsRing& R, double* v, const double* part, int voff, int ioff,
                                              int f, int w, bool inl) {
  const int nb = inl ? R.I(ioff) : 0, e = voff + w * (w + 1) / 2;
#pragma unroll 1
  for (int k = w - 1; k >= 0; --k) {
    const int cs = voff + k * w - k * (k - 1) / 2;
    double sk = 0.0;
    if (inl) {
      double a1 = 0.0, a2 = 0.0, a3 = 0.0;
      int r = 0;
      for (; r + 4 <= nb; r += 4) {
        sk = fma(R.V(e + r * w + k), v[R.I(ioff + 1 + r)], sk);
        a1 = fma(R.V(e + (r + 1) * w + k), v[R.I(ioff + 2 + r)], a1);
        a2 = fma(R.V(e + (r + 2) * w + k), v[R.I(ioff + 3 + r)], a2);
        a3 = fma(R.V(e + (r + 3) * w + k), v[R.I(ioff + 4 + r)], a3);
      }
      for (; r < nb; ++r) sk = fma(R.V(e + r * w + k), v[R.I(ioff + 1 + r)], sk);
      sk += (a1 + a2) + a3;
    } else {
      for (int g = R.I(ioff + k), g1 = R.I(ioff + k + 1); g < g1; ++g) sk += part[g];
    }
    double acc = v[f + k] - sk;
    for (int j = k + 1; j < w; ++j) acc = fma(-R.V(cs + j - k), v[f + j], acc);
    v[f + k] = acc * R.V(cs);
  }
}

// Warp task (width > thread_task_w(), sysplan.cpp): lanes = rows (forward) /
// columns (backward) of a 32-block, shuffle triangular solve.
__device__ __forceinline__ void ks_warp_task(const KsRing& R, double* v, const double* part, int voff, int ioff,
                                             int f, int w, bool bwd, int lane) {
  if (!bwd) {
    for (int rb = 0; rb < w; rb += 32) {
      const int bw = min(32, w - rb), r = rb + lane;
      const bool valid = lane < bw;
      const int rowo = voff + r * (r + 1) / 2;
      double acc = 0.0;
      if (valid) {
        acc = v[f + r];
        for (int g = R.I(ioff + r), g1 = R.I(ioff + r + 1); g < g1; ++g) acc -= part[g];
        double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
        for (int j = 0; j < rb; j += 4) {  // rb is a multiple of 32
          a0 = fma(R.V(rowo + j), v[f + j], a0);
          a1 = fma(R.V(rowo + j + 1), v[f + j + 1], a1);
          a2 = fma(R.V(rowo + j + 2), v[f + j + 2], a2);
          a3 = fma(R.V(rowo + j + 3), v[f + j + 3], a3);
        }
        acc -= (a0 + a1) + (a2 + a3);
      }
      for (int k2 = 0; k2 < bw; ++k2) {
        if (lane == k2) acc *= R.V(rowo + r);
        const double yk = __shfl_sync(0xffffffffu, acc, k2);
        if (lane > k2 && valid) acc = fma(-R.V(rowo + rb + k2), yk, acc);
      }
      if (valid) v[f + r] = acc;
      __syncwarp();
    }
  } else {
    const int nblk = (w + 31) >> 5;
    for (int bi = nblk - 1; bi >= 0; --bi) {
      const int cb = bi * 32, bw = min(32, w - cb), kk = cb + lane;
      const bool valid = lane < bw;
      const int cs = voff + kk * w - kk * (kk - 1) / 2;
      double acc = 0.0;
      if (valid) {
        double sg = 0.0;
        for (int g = R.I(ioff + kk), g1 = R.I(ioff + kk + 1); g < g1; ++g) sg += part[g];
        acc = v[f + kk] - sg;
        double a0 = 0.0, a1 = 0.0;
        int j = cb + bw;
        for (; j + 2 <= w; j += 2) {
          a0 = fma(R.V(cs + j - kk), v[f + j], a0);
          a1 = fma(R.V(cs + j + 1 - kk), v[f + j + 1], a1);
        }
        if (j < w) a0 = fma(R.V(cs + j - kk), v[f + j], a0);
        acc -= a0 + a1;
      }
      for (int jj = bw - 1; jj >= 0; --jj) {
        if (lane == jj) acc *= R.V(cs);
        const double xj = __shfl_sync(0xffffffffu, acc, jj);
        if (lane < jj) acc = fma(-R.V(cs + jj - lane), xj, acc);
      }
      if (valid) v[f + kk] = acc;
      __syncwarp();
    }
  }
}

__device__ __forceinline__ void ks_bar_compute(int nthreads) {
  asm volatile("bar.sync 1, %0;" ::"r"(nthreads) : "memory");
}

// Runs program blocks ba..bb on S.v: JT (t = P J^T u, optionally
// base[perm i] - t), FWD, BWD, J (rows handed to `jout`).  Warps
// 0 .. NT/32-2 compute; the last warp is the PRODUCER: it copies the rings
// ahead (cp.async, mbarrier completion) and waits for the next step's
// chunks before each step's closing barrier, so compute warps never wait on
// memory and carry no ring bookkeeping.
template <int NT>
__device__ __noinline__ void ks_run(const KsArgs& a, const KsSmem& S, const double* __restrict__ vals, KsStream& sv_ref,
                                    KsStream& si_ref, int ba, int bb, const double* u, const double* base,
                                    KsJOut& jout_ref, KsTimer& tm_ref, bool trace) {
  // everything the step loop touches lives in registers: this function is
  // not inlined (one copy of the interpreter), so kernel arguments and the
  // shared-memory map arrive through the caller's stack frame
  KsStream sv = sv_ref, si = si_ref;
  KsJOut jout = jout_ref;
  KsTimer tm = tm_ref;
  const int nvchunk = a.nvchunk, nichunk = a.nichunk, s_begin = a.bs0[ba], s_end = a.bs1[bb];
  const int* __restrict__ perm = a.perm;
  const int* __restrict__ gidx = a.idx;
  const int dbg = a.debug;
  const KsSmem L = ks_layout(nvchunk, a.vchunk_lg, nichunk, a.ichunk_lg, a.pmax);
  unsigned long long* const prof = a.prof ? L.prof : nullptr;
  unsigned long long* const trace_out = a.trace;
  double* const rv_s = L.rv;
  int* const ri_s = L.ri;
  unsigned long long* const barv = L.barv;
  unsigned long long* const bari = L.bari;
  int* const sys = L.sys;
  constexpr int NC = NT - 32;  // compute threads
  constexpr int NWC = NC / 32;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const bool producer = tid >= NC;
  const int vlg = a.vchunk_lg, ilg = a.ichunk_lg;
  const long long cv0 = a.bv0[ba] >> vlg, cv1 = a.bv1[bb] >> vlg;
  const long long ci0 = a.bi0[ba] >> ilg, ci1 = a.bi1[bb] >> ilg;
  const int vmask = (nvchunk << vlg) - 1, imask = (nichunk << ilg) - 1;
  const long long Dv = (sv.G - cv0) << vlg, Di = (si.G - ci0) << ilg;
  double* __restrict__ v = L.v;
  double* __restrict__ part = L.part;
  long long vb = a.bv0[ba], ib = a.bi0[ba];
  // ---- ring feed (KsArgs::feed):
  //  0  cp.async: every thread copies its 16-byte slice of each chunk
  //     (LSU work spread over all warps; completion = one noinc arrival
  //     per copying thread on the chunk's mbarrier)
  //  1  TMA: one bulk copy per chunk, issued by producer lane
  //     (chunk mod issuers); bulk requests are accepted ~every 400 ns per
  //     issuing thread (tools/micro/tma_pure.cu), completion counted in bytes.
  const int feed = a.feed;
  // TMA requests come from lanes of the producer warp only: compute warps
  // carry no feed instructions
  const int issuers = min(a.issuers, 32);
  const bool issuer = producer && lane < issuers;
  const int vthr = (8 << vlg) / 16, ithr = (4 << ilg) / 16;  // cp.async copying threads per chunk
  const unsigned long long pol_v = policy_evict_first(), pol_i = policy_evict_last();
  auto issue_range = [&](long long v_from, long long v_to, long long i_from, long long i_to) {
    if (feed == 0) {
      if (tid < vthr) {
        for (long long gc = v_from; gc < v_to; ++gc) {
          const long long c = cv0 + (gc - sv.G);
          const int slot = static_cast<int>(gc & (nvchunk - 1));
          cp_async16(rv_s + (slot << vlg) + 2 * tid, vals + (c << vlg) + 2 * tid, pol_v);
          cp_async_arrive(barv + slot);
        }
      }
      if (tid < ithr) {
        for (long long gc = i_from; gc < i_to; ++gc) {
          const long long c = ci0 + (gc - si.G);
          const int slot = static_cast<int>(gc & (nichunk - 1));
          cp_async16(ri_s + (slot << ilg) + 4 * tid, gidx + (c << ilg) + 4 * tid, pol_i);
          cp_async_arrive(bari + slot);
        }
      }
      return;
    }
    if (!issuer) return;
    for (long long gc = v_from + ((lane - v_from) % issuers + issuers) % issuers; gc < v_to; gc += issuers) {
      const long long c = cv0 + (gc - sv.G);
      const int slot = static_cast<int>(gc & (nvchunk - 1));
      unsigned long long* bar = barv + slot;
      mbar_expect_tx(bar, 8u << vlg);
      tma_load_1d(rv_s + (slot << vlg), vals + (c << vlg), 8u << vlg, bar, pol_v);
    }
    for (long long gc = i_from + ((issuers - 1 - lane - i_from) % issuers + issuers) % issuers; gc < i_to;
         gc += issuers) {
      const long long c = ci0 + (gc - si.G);
      const int slot = static_cast<int>(gc & (nichunk - 1));
      unsigned long long* bar = bari + slot;
      mbar_expect_tx(bar, 4u << ilg);
      tma_load_1d(ri_s + (slot << ilg), gidx + (c << ilg), 4u << ilg, bar, pol_i);
    }
  };
  // producer: the window allowed when a step starting at program chunks
  // (cvs, cis) begins -> sys[2..5] (relative to the run's G), and the
  // issued counters advance
  // (double-buffered by step parity: threads of step k read buffer k & 1
  // while the producer fills buffer (k+1) & 1)
  auto plan_issue = [&](long long cvs, long long cis, int par) {
    const long long limv = sv.G + (min(cvs + nvchunk, cv1) - cv0);
    const long long limi = si.G + (min(cis + nichunk, ci1) - ci0);
    if (lane == 0) {
      int* pub = sys + 4 + 4 * par;
      pub[0] = static_cast<int>(sv.issued - sv.G);
      pub[1] = static_cast<int>(max(limv, sv.issued) - sv.G);
      pub[2] = static_cast<int>(si.issued - si.G);
      pub[3] = static_cast<int>(max(limi, si.issued) - si.G);
    }
    sv.issued = max(sv.issued, limv);
    si.issued = max(si.issued, limi);
  };
  auto issue_published = [&](int par) {
    const int* pub = sys + 4 + 4 * par;
    issue_range(sv.G + pub[0], sv.G + pub[1], si.G + pub[2], si.G + pub[3]);
  };
  // waits (producer) for program chunks [c0, c1] of each stream, as far as issued
  // (the producer's 32 lanes wait on different chunks in parallel: a
  // try_wait costs ~100 cycles even on a completed phase)
  auto wait_v = [&](long long c0, long long c1) {
    const long long g1 = min(sv.G + (c1 - cv0), sv.issued - 1);
    for (long long gc = max(sv.ready + 1, sv.G + (c0 - cv0)) + lane; gc <= g1; gc += 32) {
      mbar_wait(barv + (gc & (nvchunk - 1)), static_cast<unsigned>((gc / nvchunk) & 1));
    }
    __syncwarp();
    sv.ready = max(sv.ready, g1);
  };
  auto wait_i = [&](long long c0, long long c1) {
    const long long g1 = min(si.G + (c1 - ci0), si.issued - 1);
    for (long long gc = max(si.ready + 1, si.G + (c0 - ci0)) + lane; gc <= g1; gc += 32) {
      mbar_wait(bari + (gc & (nichunk - 1)), static_cast<unsigned>((gc / nichunk) & 1));
    }
    __syncwarp();
    si.ready = max(si.ready, g1);
  };
  // producer: wait for a whole step starting at (vb2, ib2); returns true
  // when everything it needs had been issued
  auto wait_step = [&](long long vb2, long long ib2) -> bool {
    wait_i(ib2 >> ilg, (ib2 + HYKKT_SP_HDR - 1) >> ilg);
    const int il = ri_s[(Di + ib2 + 1) & imask], vl = ri_s[(Di + ib2 + 2) & imask];
    const long long lv = (vb2 + vl - 1) >> vlg, li = (ib2 + il - 1) >> ilg;
    if (vl > 0) wait_v(vb2 >> vlg, lv);
    wait_i(ib2 >> ilg, li);
    return (vl <= 0 || sv.G + (lv - cv0) < sv.issued) && si.G + (li - ci0) < si.issued;
  };
  // first window: planned here, issued by the first loop iteration, which
  // waits for it (marked late)
  if (producer) {
    sv.ready = sv.G - 1;
    si.ready = si.G - 1;
    plan_issue(cv0, ci0, 0);
    if (lane == 0) sys[2] = 1;  // late flag of parity 0
  }
  __syncthreads();
  for (int s = s_begin; s < s_end; ++s) {
    const KsRing R{rv_s, ri_s, static_cast<int>((Dv + vb) & vmask), static_cast<int>((Di + ib) & imask), vmask, imask};
    unsigned long long* wst = (trace && lane == 0) ? trace_out + (s_end + 1) + (static_cast<long long>(s) * 16 + wid) * 5 : nullptr;
    if (wst) wst[0] = gtimer();
    // this step's window (published by the producer before the barrier)
    const int par = (s - s_begin) & 1;
    issue_published(par);
    if (sys[2 + par]) {  // step data issued late (run start, block boundary): wait before anyone reads it
      if (producer) wait_step(vb, ib);
      __syncthreads();
    }
    if (wst) wst[1] = gtimer();
    const int kind = R.I(0), ilen = R.I(1), vlen = R.I(2), h3 = R.I(3), h4 = R.I(4), h5 = R.I(5);
    const long long ibn = ib + ilen, vbn = vb + vlen;
    const bool more = s + 1 < s_end;
    if (wst) wst[2] = gtimer() + (static_cast<unsigned long long>(kind) << 60);
    tm.lap(kPrWait);
    tm.count(kPrSteps);
    if (producer) {
      const unsigned long long t0 = (prof && lane == 0) ? gtimer() : 0;
      int late = 0;
      if (more) {
        late = wait_step(vbn, ibn) ? 0 : 1;
        // the window the next step will issue
        plan_issue(vbn >> vlg, ibn >> ilg, par ^ 1);
      }
      if (dbg) {  // protocol check: drain every chunk issued at this step's start
        const int* pub = sys + 4 + 4 * par;
        for (long long gc = sv.ready + 1; gc < sv.G + pub[1]; ++gc)
          mbar_wait(barv + (gc & (nvchunk - 1)), static_cast<unsigned>((gc / nvchunk) & 1));
        for (long long gc = si.ready + 1; gc < si.G + pub[3]; ++gc)
          mbar_wait(bari + (gc & (nichunk - 1)), static_cast<unsigned>((gc / nichunk) & 1));
        sv.ready = max(sv.ready, sv.G + pub[1] - 1);
        si.ready = max(si.ready, si.G + pub[3] - 1);
        late = 0;
      }
      if (prof && lane == 0) prof[kPrPre] += gtimer() - t0;
      __syncwarp();
      if (lane == 0) sys[2 + (par ^ 1)] = late;  // read at the next step's start
    } else if (kind == HYKKT_STEP_JT || kind == HYKKT_STEP_J) {
      const int nr = h3, r0 = h4, xo = HYKKT_SP_HDR + nr + 1;
      for (int j = tid; j < nr; j += NC) {
        const int e0 = R.I(HYKKT_SP_HDR + j), e1 = R.I(HYKKT_SP_HDR + j + 1);
        double acc = 0.0;
        if (kind == HYKKT_STEP_JT) {
          // all of the row's u gathers (L2) in flight before the ordered sum
          for (int e = e0; e < e1; e += 8) {
            double ue[8];
#pragma unroll
            for (int q = 0; q < 8; ++q) ue[q] = e + q < e1 ? u[R.I(xo + e + q)] : 0.0;
#pragma unroll
            for (int q = 0; q < 8; ++q) {
              if (e + q < e1) acc = __dadd_rn(acc, __dmul_rn(R.V(e + q), ue[q]));
            }
          }
          const int i = r0 + j;
          v[i] = base ? __dsub_rn(base[__ldg(perm + i)], acc) : acc;
        } else {
          for (int e = e0; e < e1; ++e) {
            const double t = v[R.I(xo + e)];
            if (t == 0.0) continue;
            acc = __dadd_rn(acc, __dmul_rn(R.V(e), t));
          }
          jout.row(r0 + j, acc);
        }
      }
      tm.lap(kind == HYKKT_STEP_J ? kPrJ : kPrRhs);
    } else {
      const bool bwd = kind == HYKKT_STEP_BWD;
      const int nseg = h3, nw = h4, nt = h5, dtask = HYKKT_SP_HDR + HYKKT_SP_SEG_INTS * nseg;
      // ---- phase A: segment partial dot products ----
      for (int g = tid; g < nseg; g += NC) {
        const int d = HYKKT_SP_HDR + HYKKT_SP_SEG_INTS * g;
        const int voff = R.I(d), ioff = R.I(d + 1), ls = R.I(d + 2);
        const int len = ls & 0xffff;
        double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
        int q = 0;
        for (; q + 4 <= len; q += 4) {
          a0 = fma(R.V(voff + q), v[R.I(ioff + q)], a0);
          a1 = fma(R.V(voff + q + 1), v[R.I(ioff + q + 1)], a1);
          a2 = fma(R.V(voff + q + 2), v[R.I(ioff + q + 2)], a2);
          a3 = fma(R.V(voff + q + 3), v[R.I(ioff + q + 3)], a3);
        }
        for (; q < len; ++q) a0 = fma(R.V(voff + q), v[R.I(ioff + q)], a0);
        part[ls >> 16] = (a0 + a1) + (a2 + a3);
      }
      if (wst) wst[3] = gtimer();
      if (nw + nt > 0 && nseg > 0) ks_bar_compute(NC);
      tm.lap(kPrA);
      // ---- phase B: warps [0, ww) take the warp tasks, the other warps'
      // threads the thread tasks (dealt for that thread count by the builder)
      const int ww = R.I(7), tt0 = 32 * ww, ntt = NC - tt0;
      if (wid < ww) {
        for (int t = wid; t < nw; t += ww) {
          const int d = dtask + HYKKT_SP_TASK_INTS * t;
          ks_warp_task(R, v, part, R.I(d), R.I(d + 1), R.I(d + 2), R.I(d + 3) & 0xffff, bwd, lane);
        }
      }
      for (int t = tid - tt0; t >= 0 && t < nt; t += ntt) {
        const int d = dtask + HYKKT_SP_TASK_INTS * (nw + t);
        const int wm = R.I(d + 3);
        const bool inl = (wm >> 16) == HYKKT_TASK_INLINE;
        if (bwd) ks_bwd_thread(R, v, part, R.I(d), R.I(d + 1), R.I(d + 2), wm & 0xffff, inl);
        else ks_fwd_thread(R, v, part, R.I(d), R.I(d + 1), R.I(d + 2), wm & 0xffff, inl);
      }
      tm.lap(kPrB);
    }
    if (dbg == 2) asm volatile("cp.async.wait_all;" ::: "memory");
    if (wst) wst[4] = gtimer();
    __syncthreads();
    tm.lap(kPrSync);
    if (trace && tid == 0) trace_out[s] = gtimer();
    ib = ibn;
    vb = vbn;
  }
  sv.G += cv1 - cv0;
  si.G += ci1 - ci0;
  sv.issued = max(sv.issued, sv.G);
  si.issued = max(si.issued, si.G);
  sv_ref = sv;
  si_ref = si;
  jout_ref = jout;
  tm_ref.last = tm.last;
}

template <int NT>
__global__ void __launch_bounds__(NT, 1) ks_solve(KsArgs a) {
  const int tid = threadIdx.x;
  const KsSmem S = ks_layout(a.nvchunk, a.vchunk_lg, a.nichunk, a.ichunk_lg, a.pmax);
  if (tid == 0) {
    // feed 0: one noinc arrival per copying thread; feed 1: one
    // arrive.expect_tx per chunk (ks_run issue_range)
    for (int i = 0; i < a.nvchunk; ++i) mbar_init(S.barv + i, a.feed ? 1u : (8u << a.vchunk_lg) / 16);
    for (int i = 0; i < a.nichunk; ++i) mbar_init(S.bari + i, a.feed ? 1u : (4u << a.ichunk_lg) / 16);
    mbar_fence_init();
    for (int i = 0; i < kPrN; ++i) S.prof[i] = 0;
  }
  __syncthreads();
  KsTimer tm{a.prof ? S.prof : nullptr, 0};
  tm.start();
  KsStream sv{0, 0, -1}, si{0, 0, -1};
  const int mc = a.mc, n = a.n;
  double* x = a.scratch + static_cast<long long>(blockIdx.x) * 5 * mc;
  double* r = x + mc;
  double* p = r + mc;
  double* q = p + mc;
  double* rhs = q + mc;
  bool traced = false;
  for (;;) {
    if (tid == 0) {
      const int t = static_cast<int>(atomicAdd(a.ticket, 1u));
      S.sys[0] = t < a.B && a.order ? a.order[t] : t;
    }
    __syncthreads();
    const int b = S.sys[0];
    __syncthreads();
    if (b >= a.B) break;
    if (!a.ok[b]) continue;
    const double* vals = a.vals + static_cast<long long>(b) * a.vlen;
    const double* rhat = a.rhat + static_cast<long long>(b) * n;
    const double* rys = a.rys + static_cast<long long>(b) * mc;
    // ---- w = H^-1 r_hat_x; Schur rhs = J w - r_y ----
    for (int i = tid; i < n; i += NT) S.v[i] = rhat[__ldg(a.perm + i)];
    __syncthreads();
    KsJOut js{kJSchur, rhs, rys, 0.0, 0.0, 0.0};
    ks_run<NT>(a, S, vals, sv, si, 1, 3, nullptr, nullptr, js, tm, false);
    tm.count(kPrSolves);
    const double rhs_norm = sqrt(ks_sum<NT>(js.s1, S.red));
    // ---- cg_schur, restarted once with delta2 on a small quadratic form ----
    long long its = 0;
    double relres = 0.0, d2 = 0.0;
    int flag = 1;
    for (int attempt = 0; attempt < 2; ++attempt) {
      d2 = attempt == 0 ? 0.0 : a.delta2;
      for (int k = tid; k < mc; k += NT) {
        x[k] = 0.0;
        r[k] = rhs[k];
        p[k] = rhs[k];
      }
      its = 0;
      relres = 0.0;
      flag = 1;
      if (rhs_norm == 0.0) break;
      double rho = rhs_norm * rhs_norm, r_norm = rhs_norm;
      flag = 0;
      for (long long it = 1; it <= a.max_iter; ++it) {
        __syncthreads();  // p complete
        tm.lap(kPrPupd);
        tm.count(kPrIters);
        KsJOut jc{kJCg, q, p, d2, 0.0, 0.0};
        const bool tr = a.trace && blockIdx.x == 0 && !traced;
        traced = true;
        ks_run<NT>(a, S, vals, sv, si, 0, 3, p, nullptr, jc, tm, tr);
        tm.count(kPrSolves);
        const double2 red = ks_sum2<NT>(jc.s1, jc.s2, S.red);
        tm.lap(kPrJrow);
        if (red.x <= a.thr * red.y) {
          its = it - 1;
          relres = r_norm / rhs_norm;
          flag = 2;
          break;
        }
        const double alpha = rho / red.x;
        double rr = 0.0;
        for (int k = tid; k < mc; k += NT) {
          x[k] = __dadd_rn(x[k], __dmul_rn(alpha, p[k]));
          const double rk = __dsub_rn(r[k], __dmul_rn(alpha, q[k]));
          r[k] = rk;
          rr = fma(rk, rk, rr);
        }
        r_norm = sqrt(ks_sum<NT>(rr, S.red));
        tm.lap(kPrUpd);
        relres = r_norm / rhs_norm;
        its = it;
        if (relres <= a.tol) {
          flag = 1;
          break;
        }
        if (it == a.max_iter) break;
        const double rho_next = r_norm * r_norm;
        const double beta = rho_next / rho;
        rho = rho_next;
        for (int k = tid; k < mc; k += NT) p[k] = __dadd_rn(r[k], __dmul_rn(beta, p[k]));
      }
      if (flag != 2) break;
    }
    if (tid == 0) {
      a.iters[b] = its;
      a.relres[b] = relres;
      a.flags[b] = flag;
      a.d2used[b] = d2;
    }
    __syncthreads();  // x complete
    // ---- dx = H^-1 (r_hat_x - J^T dy); unscale; recover ----
    KsJOut jn{kJNone, nullptr, nullptr, 0.0, 0.0, 0.0};
    ks_run<NT>(a, S, vals, sv, si, 0, 2, x, rhat, jn, tm, false);
    tm.count(kPrSolves);
    const double* d = a.d + static_cast<long long>(b) * (n + mc);
    double* odx = a.odx + static_cast<long long>(b) * n;
    for (int t = tid; t < n; t += NT) odx[t] = __dmul_rn(d[t], S.v[__ldg(a.iperm + t)]);
    double* ody = a.ody + static_cast<long long>(b) * mc;
    for (int k = tid; k < mc; k += NT) ody[k] = __dmul_rn(d[n + k], x[k]);
    const double* jd = a.jd + static_cast<long long>(b) * a.nnz_jd;
    const long long mo = static_cast<long long>(b) * a.md;
    for (int k = tid; k < a.md; k += NT) {
      double acc = 0.0;
      for (int e = __ldg(a.jd_rp + k), e1 = __ldg(a.jd_rp + k + 1); e < e1; ++e) {
        const int c = __ldg(a.jd_ci + e);
        const double xc = __dmul_rn(d[c], S.v[__ldg(a.iperm + c)]);
        if (xc == 0.0) continue;
        acc = __dadd_rn(acc, __dmul_rn(jd[__ldg(a.jd_src + e)], xc));
      }
      const double s = __dsub_rn(acc, a.ryd[mo + k]);
      a.ods[mo + k] = s;
      a.odyd[mo + k] = __dsub_rn(__dmul_rn(a.ds_in[mo + k], s), a.rs[mo + k]);
    }
    __syncthreads();  // S.v reused by the next system
    tm.lap(kPrRecover);
  }
  if (a.prof && tid == 0) {
    for (int i = 0; i < kPrN; ++i) a.prof[blockIdx.x * kPrN + i] = S.prof[i];
  }
}

// Value streams: vals[b][e] = source of stream entry e for system b (panel
// value, its reciprocal, a scaled J value, or 0).  32 entries x 32 systems
// per tile through shared memory: coalesced reads of the lane-mode
// ([slot][system]) panels and J values, coalesced stream writes.
__global__ void ks_remap(const int* __restrict__ src, long long len, SnPlan s, const int* __restrict__ mode,
                         const int* __restrict__ slot_sn, int Bp, int B, const double* __restrict__ panel,
                         const double* __restrict__ js, double* __restrict__ vals) {
  __shared__ double tile[32][33];
  const long long e0 = static_cast<long long>(blockIdx.x) * 32;
  const int b0 = blockIdx.y * 32;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  for (int j = ty; j < 32; j += 8) {
    const long long e = e0 + j;
    const int b = b0 + tx;
    double val = 0.0;
    if (e < len && b < B) {
      const int sc = __ldg(src + e);
      if (sc >= 0) {
        const int sl = sc >> 1, sn = __ldg(slot_sn + sl);
        val = panel[pan_addr(s, mode, sn, sl - s.off[sn], Bp, b)];
        if (sc & 1) val = 1.0 / val;
      } else if (sc <= -2) {
        val = js[static_cast<long long>(-2 - sc) * Bp + b];
      }
    }
    tile[j][tx] = val;
  }
  __syncthreads();
  for (int j = ty; j < 32; j += 8) {
    const int b = b0 + j;
    const long long e = e0 + tx;
    if (b < B && e < len) vals[static_cast<long long>(b) * len + e] = tile[tx][j];
  }
}

}  // namespace hykkt::dev

namespace hykkt::dev {

// ---- system-per-CTA numeric factorization ---------------------------------
// numeric_cholesky (proj/core/src/cholesky.cpp:65-137) for every system still
// on the delta1 ladder (solver.cpp:108-142): one CTA per system at a time,
// the system's panels contiguous in global memory (so the descendant blocks
// it re-reads stay in L1/L2 while the CTA owns the system), supernodes in
// level order with a CTA barrier per level: narrow supernodes are warp
// tasks (left-looking updates from the descendant blocks, lanes over target
// rows, then the dense factor of the panel), wide ones CTA tasks with the
// panel staged in shared memory.  The pivot test is the reference's
// !(pivot > floor) with floor = pivot_floor * max|diag H_gamma|
// (solver.cpp:111); the first failing column is recorded with atomicMin.
struct KfArgs {
  SnPlan s;
  long long panel_size;
  double* panel;            // [B][panel_size]
  const double* hg;         // [B][nsrc] H_gamma values (lower CSC order)
  int nsrc;
  const int* to_panel;      // nsrc -> panel slot
  const int* srow;
  const int* scol;
  const double* delta1;     // [Bp]
  const int* active;        // [Bp]
  const double* maxdiag;    // [Bp]
  double floor_rel;
  int* fail_col;            // [Bp], INT_MAX on entry
  const int* lev_ptr;       // nlevels + 1 (narrow list)
  const int* lev_sn;        // narrow supernodes by level
  const int* wlev_ptr;      // nlevels + 1 (wide list)
  const int* wlev_sn;
  int nlevels;
  int smem_doubles;
  unsigned* ticket;
  int B;
  // per update u (SupernodalPlan upd_* order): {panel offset of the block's
  // first row (off[d] + upd_off), column stride nrows[d], rows m | cnt << 16,
  // descendant width}, and the block's row list start (rows_ptr[d] + upd_off)
  const int4* upd;
  const int* upd_rows;
  // per target supernode: staging batches of its update list (ends, in
  // update index), for the warp capacity and the CTA capacity
  const int* wb_ptr;   // nsup + 1 into wb_end
  const int* wb_end;
  const int* cb_ptr;
  const int* cb_end;
};

extern __shared__ __align__(16) double kf_smem[];

__device__ __forceinline__ void kf_dense_warp(double* P, int nr, int w, int f, double floor_v, int* fail, int lane) {
  for (int k = 0; k < w; ++k) {
    double* Pk = P + k * nr;
    const double pivot = Pk[k];
    if (!(pivot > floor_v) && lane == 0) atomicMin(fail, f + k);
    const double dk = sqrt(pivot);
    __syncwarp();
    for (int r = k + 1 + lane; r < nr; r += 32) Pk[r] = Pk[r] * (1.0 / dk);
    if (lane == 0) Pk[k] = dk;
    __syncwarp();
    for (int c = k + 1; c < w; ++c) {
      const double lck = Pk[c];
      double* Pc = P + c * nr;
      for (int r = c + lane; r < nr; r += 32) Pc[r] = fma(-Pk[r], lck, Pc[r]);
    }
    __syncwarp();
  }
}

// Per-warp staging area of ks_factor (doubles): a narrow target panel and
// one descendant block at a time.
constexpr int kKfWarpStage = 512;
// CTA tasks: target positions of the staged block rows (ints), carved from
// the end of the per-warp staging areas
constexpr int kKfPosStage = 2048;

// One left-looking update (cholesky.cpp:102-114 in supernodal form): target
// entries of panel P (nr x w, columns f..) -= L_d[rows, :] L_d[jj rows, :]^T
// for the cnt rows of descendant d that fall in the target's columns.  D =
// the descendant block (m x wd, column stride ld) in shared or global memory.
__device__ __forceinline__ void kf_apply(double* P, const int* R, int f, int w, int nr, const double* D, int ld,
                                         int wd, int m, int cnt, const int* Rdo, int lane, int cmod, int cres) {
  // row ii of the block (per lane): its target position is found once,
  // then every column jj <= ii of the run is updated
  for (int ii = lane; ii < m; ii += 32) {
    const int r = __ldg(Rdo + ii);
    const int pos = ii < cnt ? r - f : find_row(R, w, nr, r);
    const int jmax = min(cnt, ii + 1);
    for (int jj = 0; jj < jmax; ++jj) {
      const int cc = __ldg(Rdo + jj) - f;
      if (cmod > 1 && cc % cmod != cres) continue;
      double d0 = 0.0, d1 = 0.0;
      int k = 0;
      for (; k + 2 <= wd; k += 2) {
        d0 = fma(D[k * ld + ii], D[k * ld + jj], d0);
        d1 = fma(D[(k + 1) * ld + ii], D[(k + 1) * ld + jj], d1);
      }
      if (k < wd) d0 = fma(D[k * ld + ii], D[k * ld + jj], d0);
      P[cc * nr + pos] -= d0 + d1;
    }
  }
}

// All left-looking updates of target supernode sn, in update order, in
// host-planned batches that fit the staging area (every load of a batch in
// flight at once); a batch of one oversized block is applied straight from
// global memory.  Warp version: lanes over the block rows.  CTA version:
// warps over the block's target columns (each target entry owned by one
// warp), the block rows' target positions staged once in shared memory.
__device__ __forceinline__ void kf_updates_warp(const KfArgs& a, const double* Pb, int sn, double* P, const int* R,
                                                int f, int w, int nr, double* stage, int cap, int lane) {
  int u = a.s.upd_ptr[sn];
  for (int bi = a.wb_ptr[sn], be = a.wb_ptr[sn + 1]; bi < be; ++bi) {
    const int ue = __ldg(a.wb_end + bi);
    int4 q = __ldg(a.upd + u);
    if ((q.z & 0xffff) * q.w > cap) {  // oversized: direct
      kf_apply(P, R, f, w, nr, Pb + q.x, q.y, q.w, q.z & 0xffff, q.z >> 16, a.s.rows + __ldg(a.upd_rows + u), lane, 1, 0);
      __syncwarp();
      u = ue;
      continue;
    }
    int off = 0;
    for (int v = u; v < ue; ++v) {
      const int4 d = __ldg(a.upd + v);
      const int m = d.z & 0xffff;
      for (int e = lane; e < m * d.w; e += 32) {
        const int k = e / m, ii = e - k * m;
        stage[off + e] = Pb[d.x + k * d.y + ii];
      }
      off += m * d.w;
    }
    __syncwarp();
    off = 0;
    for (int v = u; v < ue; ++v) {
      const int4 d = __ldg(a.upd + v);
      const int m = d.z & 0xffff;
      kf_apply(P, R, f, w, nr, stage + off, m, d.w, m, d.z >> 16, a.s.rows + __ldg(a.upd_rows + v), lane, 1, 0);
      off += m * d.w;
      __syncwarp();
    }
    u = ue;
  }
}

template <int NT>
__device__ __forceinline__ void kf_updates_cta(const KfArgs& a, const double* Pb, int sn, double* P, const int* R,
                                               int f, int w, int nr, double* stage, int cap, int* pos_st) {
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  constexpr int NW = NT / 32;
  int u = a.s.upd_ptr[sn];
  for (int bi = a.cb_ptr[sn], be = a.cb_ptr[sn + 1]; bi < be; ++bi) {
    const int ue = __ldg(a.cb_end + bi);
    const int4 q0 = __ldg(a.upd + u);
    const bool direct = (q0.z & 0xffff) * q0.w > cap;
    // stage the blocks and their rows' target positions
    int off = 0, poff = 0;
    for (int v = u; v < ue; ++v) {
      const int4 d = __ldg(a.upd + v);
      const int m = d.z & 0xffff, cnt = d.z >> 16;
      const int* Rdo = a.s.rows + __ldg(a.upd_rows + v);
      if (!direct) {
        for (int e = tid; e < m * d.w; e += NT) {
          const int k = e / m, ii = e - k * m;
          stage[off + e] = Pb[d.x + k * d.y + ii];
        }
      }
      for (int ii = tid; ii < m; ii += NT) {
        const int r = __ldg(Rdo + ii);
        pos_st[poff + ii] = ii < cnt ? r - f : find_row(R, w, nr, r);
      }
      off += m * d.w;
      poff += m;
    }
    __syncthreads();
    off = 0;
    poff = 0;
    for (int v = u; v < ue; ++v) {
      const int4 d = __ldg(a.upd + v);
      const int m = d.z & 0xffff, cnt = d.z >> 16, wd = d.w;
      const double* D = direct ? Pb + d.x : stage + off;
      const int ld = direct ? d.y : m;
      const int* Rdo = a.s.rows + __ldg(a.upd_rows + v);
      // warps own target columns (cc mod NW): the updates of a batch are not
      // separated by barriers, so a target column must stay with one warp
      for (int jj = 0; jj < cnt; ++jj) {
        const int cc = __ldg(Rdo + jj) - f;
        if (cc % NW != wid) continue;
        for (int ii = jj + lane; ii < m; ii += 32) {
          double d0 = 0.0, d1 = 0.0;
          int k = 0;
          for (; k + 2 <= wd; k += 2) {
            d0 = fma(D[k * ld + ii], D[k * ld + jj], d0);
            d1 = fma(D[(k + 1) * ld + ii], D[(k + 1) * ld + jj], d1);
          }
          if (k < wd) d0 = fma(D[k * ld + ii], D[k * ld + jj], d0);
          P[cc * nr + pos_st[poff + ii]] -= d0 + d1;
        }
      }
      off += m * wd;
      poff += m;
    }
    __syncthreads();
    u = ue;
  }
}

// warp task: narrow supernode sn (w nr <= kKfWarpStage / 2 is staged)
__device__ void kf_warp_task(const KfArgs& a, double* Pb, int sn, double floor_v, int* fail, int lane, double* st) {
  const SnPlan& s = a.s;
  const int f = s.first[sn], w = s.first[sn + 1] - f, nr = s.nrows[sn], size = nr * w;
  const int* R = s.rows + s.rows_ptr[sn];
  double* Pg = Pb + s.off[sn];
  const bool pst = size <= kKfWarpStage / 2;
  double* P = pst ? st : Pg;
  double* Dst = st + kKfWarpStage / 2;
  if (pst) {
    for (int e = lane; e < size; e += 32) P[e] = Pg[e];
    __syncwarp();
  }
  kf_updates_warp(a, Pb, sn, P, R, f, w, nr, Dst, kKfWarpStage / 2, lane);
  kf_dense_warp(P, nr, w, f, floor_v, fail, lane);
  if (pst) {
    for (int e = lane; e < size; e += 32) Pg[e] = P[e];
    __syncwarp();
  }
}

// CTA task: wide supernode; panel staged in shared memory when it fits,
// each descendant block staged by the whole CTA (all loads in flight), warps
// own target columns cc = wid (mod NW)
template <int NT>
__device__ void kf_cta_task(const KfArgs& a, double* Pb, int sn, double floor_v, int* fail, double* pan_st,
                            double* blk_st, int blk_cap, int* pos_st) {
  const SnPlan& s = a.s;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  constexpr int NW = NT / 32;
  const int f = s.first[sn], w = s.first[sn + 1] - f, nr = s.nrows[sn], size = nr * w;
  const int* R = s.rows + s.rows_ptr[sn];
  double* Pg = Pb + s.off[sn];
  const bool fits = size <= a.smem_doubles;
  double* P = fits ? pan_st : Pg;
  if (fits) {
    for (int e = tid; e < size; e += NT) P[e] = Pg[e];
  }
  __syncthreads();
  kf_updates_cta<NT>(a, Pb, sn, P, R, f, w, nr, blk_st, blk_cap, pos_st);
  // blocked right-looking factor: warp 0 factors 8 columns, all warps apply
  // the rank-8 trailing update
  constexpr int KB = 8;
  for (int k0 = 0; k0 < w; k0 += KB) {
    const int kb = min(KB, w - k0);
    if (wid == 0) {
      for (int k = k0; k < k0 + kb; ++k) {
        double* Pk = P + k * nr;
        const double pivot = Pk[k];
        if (!(pivot > floor_v) && lane == 0) atomicMin(fail, f + k);
        const double dk = sqrt(pivot);
        __syncwarp();
        for (int r = k + 1 + lane; r < nr; r += 32) Pk[r] = Pk[r] * (1.0 / dk);
        if (lane == 0) Pk[k] = dk;
        __syncwarp();
        for (int c = k + 1; c < k0 + kb; ++c) {
          const double lck = Pk[c];
          double* Pc = P + c * nr;
          for (int r = c + lane; r < nr; r += 32) Pc[r] = fma(-Pk[r], lck, Pc[r]);
        }
        __syncwarp();
      }
    }
    __syncthreads();
    for (int c = k0 + kb + wid; c < w; c += NW) {
      double lc[KB];
#pragma unroll
      for (int k = 0; k < KB; ++k) lc[k] = k < kb ? P[(k0 + k) * nr + c] : 0.0;
      double* Pc = P + c * nr;
      for (int r = c + lane; r < nr; r += 32) {
        double v = Pc[r];
#pragma unroll
        for (int k = 0; k < KB; ++k) {
          if (k < kb) v = fma(-P[(k0 + k) * nr + r], lc[k], v);
        }
        Pc[r] = v;
      }
    }
    __syncthreads();
  }
  if (fits) {
    for (int e = tid; e < size; e += NT) Pg[e] = P[e];
    __syncthreads();
  }
}

template <int NT>
__global__ void __launch_bounds__(NT) ks_factor(KfArgs a) {
  __shared__ int s_sys;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  constexpr int NW = NT / 32;
  for (;;) {
    if (tid == 0) s_sys = static_cast<int>(atomicAdd(a.ticket, 1u));
    __syncthreads();
    const int b = s_sys;
    __syncthreads();
    if (b >= a.B) break;
    if (!a.active[b]) continue;
    double* Pb = a.panel + static_cast<long long>(b) * a.panel_size;
    const double* hg = a.hg + static_cast<long long>(b) * a.nsrc;
    const double d1 = a.delta1[b];
    for (long long i = tid; i < a.panel_size; i += NT) Pb[i] = 0.0;
    __syncthreads();
    for (int t = tid; t < a.nsrc; t += NT) {
      double v = hg[t];
      if (d1 != 0.0 && __ldg(a.srow + t) == __ldg(a.scol + t)) v = __dadd_rn(v, d1);
      Pb[__ldg(a.to_panel + t)] = v;
    }
    __syncthreads();
    const double floor_v = fmax(a.floor_rel * a.maxdiag[b], 0.0);
    int* fail = a.fail_col + b;
    // shared memory: [wide panel staging: smem_doubles][NW per-warp stages]
    double* wst = kf_smem + a.smem_doubles;
    for (int L = 0; L < a.nlevels; ++L) {
      for (int i = a.lev_ptr[L] + wid; i < a.lev_ptr[L + 1]; i += NW)
        kf_warp_task(a, Pb, a.lev_sn[i], floor_v, fail, lane, wst + wid * kKfWarpStage);
      __syncthreads();
      for (int i = a.wlev_ptr[L]; i < a.wlev_ptr[L + 1]; ++i)
        kf_cta_task<NT>(a, Pb, a.wlev_sn[i], floor_v, fail, kf_smem, wst, NW * kKfWarpStage - kKfPosStage / 2,
                        reinterpret_cast<int*>(wst + NW * kKfWarpStage - kKfPosStage / 2));
      if (a.wlev_ptr[L + 1] > a.wlev_ptr[L]) __syncthreads();
    }
    __syncthreads();
  }
}

// Value streams from per-system panels (ks_factor layout) and per-system
// scaled J values: vals[b][e] (see sysplan_format.h source encoding).
__global__ void ks_remap_sys(const int* __restrict__ src, long long len, long long panel_size,
                             const double* __restrict__ panel, const double* __restrict__ js, long long nnz_j,
                             double* __restrict__ vals) {
  const long long e = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
  const int b = blockIdx.y;
  if (e >= len) return;
  const int sc = __ldg(src + e);
  double val = 0.0;
  if (sc >= 0) {
    val = panel[b * panel_size + (sc >> 1)];
    if (sc & 1) val = 1.0 / val;
  } else if (sc <= -2) {
    val = js[b * nnz_j + (-2 - sc)];
  }
  vals[b * len + e] = val;
}

}  // namespace hykkt::dev
