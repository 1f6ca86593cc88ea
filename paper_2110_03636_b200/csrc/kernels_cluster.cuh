// Single-system solve on ONE thread-block cluster (level-synchronous).
//
// The sync-free grid-wide pass of kernels_solve.cuh pays one cross-SM
// hand-off (an L2 round trip plus the poll of a spinning warp sharing the SM
// with 15 other pollers) per supernode-tree link: 42-79 links per pass, so
// ~300-1700 us per CG iteration at C1-C4 whatever the size.  Here the
// supernode tree is walked level by level (forward: leaves first, backward:
// root first) by the CTAs of one cluster, with `barrier.cluster`
// (release / acquire at cluster scope, ~0.2 us) between levels instead of
// per-value polling:
//   * the right-hand side b - J^T u of every row is formed first in one
//     sweep (bt), so no task pays the J-column gather on its critical path;
//   * per level: thread tasks (w <= 4, rows <= 16, when the level is wide
//     enough to fill the cluster), warp tasks, and whole-CTA tasks for wide
//     panels -- the same arithmetic as fwd_thread / fwd_task / fwd_cta and
//     their backward counterparts;
//   * nothing is polled: every value a task reads was written at an earlier
//     level, before the last cluster barrier.
// The CG loop (cg_schur, proj/core/src/solver.cpp:154-201) runs inside the
// same launch: vector updates split over the cluster's threads, dot products
// reduced per CTA (fixed order), combined across CTAs through distributed
// shared memory in rank order (every CTA computes the same sum), so no grid
// barrier and no host round trip.
#pragma once

#include "kernels_solve.cuh"

namespace hykkt::dev {
#include "kernels_walk.cuh"
}  // namespace hykkt::dev

namespace hykkt::dev {

constexpr int kClThreads = 512;
constexpr int kClWarps = kClThreads / 32;
constexpr int kClMaxCtas = 16;

__device__ __forceinline__ void cluster_sync_all() {
  asm volatile(
      "barrier.cluster.arrive.release.aligned;\n\t"
      "barrier.cluster.wait.acquire.aligned;" ::: "memory");
}

__device__ __forceinline__ unsigned cluster_rank() {
  unsigned r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}

__device__ __forceinline__ unsigned cluster_size() {
  unsigned r;
  asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(r));
  return r;
}

// Load a double from the shared memory of CTA `rank` of this cluster.
__device__ __forceinline__ double ld_dsmem(const double* local, unsigned rank) {
  const unsigned a = static_cast<unsigned>(__cvta_generic_to_shared(local));
  unsigned r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(rank));
  double v;
  asm volatile("ld.shared::cluster.f64 %0, [%1];" : "=d"(v) : "r"(r) : "memory");
  return v;
}

struct ClSmem {
  TrsvSmem cta;                         // whole-CTA tasks
  ClWarpBuf warp[kClWarps];
  double scratch[33];
  double red[2][4];                     // per-CTA partial sums, double-buffered by iteration parity
  int lv[4 * 256 + 4];                  // the level table (a copy of ClArgs::lv when it fits)
  double part[4];                       // thread 0's copy of this CTA's partials before publishing
};

// Packed per-task descriptor (host-built, level order): two int4.
//   a = {sn, first column f, w | nrows << 16, panel offset}
//   b = {update-vector offset u_off[sn], row-slot base rows_ptr[sn], 0, 0}
// Gathers of row slot t (forward, multifrontal extend-add) come from
// gat4[t]: up to four u indices (-1 = none); a row with more has
// gat4[t].w = -2 - (gat_idx position of its fourth entry) and the rest is
// read from gat_idx up to gat_ptr[t + 1].
struct ClArgs {
  TrsvArgs tr;        // plan, panel, y / x / u, rhs (b, u = J^T operand), x_out
  double* bt;         // n: right-hand side of every permuted row
  int nlev;
  // per level l: [lv[4l], lv[4l+1]) thread tasks, [.., lv[4l+2]) warp tasks
  // (indices into desc), [lv[4l-1] (0 for l = 0), lv[4l+3]) CTA tasks
  // (indices into cta_sn)
  const int* lv;
  const int4* desc;   // 2 per task
  const int* cta_sn;
  const int4* gat4;   // per row slot (thread tasks)
  // warp tasks: per-warp lists (level order) of entries
  //   wl[2e] = {record offset (ints), value offset (doubles), w | nr << 16, u_off}
  //   wl[2e+1] = {first column, level, row-slot base, 0}
  // record: 4 gather ints per row (gat4 format), then the nr - w rows below
  const int4* wl;
  const int* wl_ptr;
  const int* rec;
  const double* vals;  // panels of the warp tasks, reciprocal diagonals (k_cl_remap)
  // CG (mode 1)
  int mode;           // 0: one H^-1 pass; 1: cg_schur
  int mc;
  const int* jcsr_rp;
  const int* jcsr_ci_perm;
  const double* jcsr;
  const double* rhs;
  double* x;
  double* r;
  double* p;
  double* q;
  double delta2;
  double tol;
  double thr;
  long long max_iter;
  CgResultDev* res;
  unsigned long long* stamps;  // diagnostics: per-level end times of CTA 0 (null = off)
};

// b - J^T u of every permuted row, written to bt.
__device__ __forceinline__ void cl_rhs(const ClArgs& a, int gt, int gs) {
  for (int i = gt; i < a.tr.s.n; i += gs) a.bt[i] = rhs_raw(a.tr, i);
}

__device__ __forceinline__ void cl_level_cta(const ClArgs& a, ClSmem& S, const int* lv, int l, bool fwd) {
  const int rank = static_cast<int>(cluster_rank()), nc = static_cast<int>(cluster_size());
  const int c0 = l ? lv[4 * l - 1] : 0, c1 = lv[4 * l + 3];
  for (int i = c0 + (nc - 1 - rank); i < c1; i += nc) {
    if (fwd) fwd_cta(a.tr, S.cta, a.cta_sn[i]);
    else bwd_cta(a.tr, S.cta, a.cta_sn[i]);
    __syncthreads();
  }
}

__device__ __forceinline__ void cl_level_threads(const ClArgs& a, const int* lv, int l, bool fwd) {
  const int rank = static_cast<int>(cluster_rank()), nc = static_cast<int>(cluster_size());
  const int p0 = lv[4 * l], p1 = lv[4 * l + 1];
  const int gt = rank * kClThreads + threadIdx.x, gs = nc * kClThreads;
  for (int i = p0 + gt; i < p1; i += gs) {
    const int4 da = __ldg(a.desc + 2 * i), db = __ldg(a.desc + 2 * i + 1);
    if (fwd) cl_fwd_thread(a, da, db);
    else cl_bwd_thread(a, da, db);
  }
}

// One H^-1 application: bt, forward levels, backward levels; x (permuted)
// complete in global memory (and x_out when set) after the final barrier.
__device__ void cl_pass(const ClArgs& a, ClSmem& S) {
  const int rank = static_cast<int>(cluster_rank()), nc = static_cast<int>(cluster_size());
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, gw = rank * kClWarps + wid;
  ClWarpBuf& B = S.warp[wid];
  cl_rhs(a, rank * kClThreads + threadIdx.x, nc * kClThreads);
  cluster_sync_all();
  const int* lv = a.nlev <= 256 ? S.lv : a.lv;
  ClWalk W;
  cl_walk_begin(a, W, B, gw, true, lane);
  for (int l = 0; l < a.nlev; ++l) {
    cl_level_cta(a, S, lv, l, true);
    cl_walk_level(a, W, B, l, true, lane, wid == 0 && rank == 0);
    cl_level_threads(a, lv, l, true);
    cluster_sync_all();
    if (a.stamps && rank == 0 && threadIdx.x == 0) a.stamps[l] = global_ns();
  }
  cp_async_wait_all();
  cl_walk_begin(a, W, B, gw, false, lane);
  for (int l = a.nlev - 1; l >= 0; --l) {
    cl_level_cta(a, S, lv, l, false);
    cl_walk_level(a, W, B, l, false, lane, wid == 0 && rank == 0);
    cl_level_threads(a, lv, l, false);
    cluster_sync_all();
    if (a.stamps && rank == 0 && threadIdx.x == 0) a.stamps[2 * a.nlev - 1 - l] = global_ns();
  }
  cp_async_wait_all();
}

// Cluster-wide sum of one per-thread value: CTA sum (fixed order), published
// in this CTA's shared memory, every CTA then adds the CTAs' sums in rank
// order.  `slot` / `par` select the buffer; callers alternate `par` so a
// buffer is rewritten only after the next cluster barrier.
__device__ __forceinline__ double cl_sum(double v, ClSmem& S, int slot, int par) {
  v = block_sum(v, S.scratch);
  if (threadIdx.x == 0) S.red[par][slot] = v;
  cluster_sync_all();
  const unsigned nc = cluster_size();
  double t = 0.0;
  if (threadIdx.x < 32) {
    for (unsigned c = 0; c < nc; ++c) t += ld_dsmem(&S.red[par][slot], c);
    if (threadIdx.x == 0) S.scratch[32] = t;
  }
  __syncthreads();
  t = S.scratch[32];
  __syncthreads();
  return t;
}

__global__ void __launch_bounds__(kClThreads, 1) k_cluster_solve(ClArgs a) {
  extern __shared__ __align__(16) unsigned char cl_smem_raw[];
  ClSmem& S = *reinterpret_cast<ClSmem*>(cl_smem_raw);
  const int rank = static_cast<int>(cluster_rank()), nc = static_cast<int>(cluster_size());
  const int gt = rank * kClThreads + threadIdx.x, gs = nc * kClThreads;
  if (a.nlev <= 256) {
    for (int i = threadIdx.x; i < 4 * a.nlev; i += blockDim.x) S.lv[i] = a.lv[i];
    __syncthreads();
  }
  if (a.mode == 0) {
    cl_pass(a, S);
    return;
  }
  double ss = 0.0;
  for (int k = gt; k < a.mc; k += gs) {
    const double v = a.rhs[k];
    a.x[k] = 0.0;
    a.r[k] = v;
    a.p[k] = v;
    ss = fma(v, v, ss);
  }
  const double rhs_norm = sqrt(cl_sum(ss, S, 0, 0));
  const bool writer = gt == 0;
  if (rhs_norm == 0.0) {
    if (writer) *a.res = CgResultDev{0, 0.0, 1, 0};
    return;
  }
  double rho = rhs_norm * rhs_norm;
  double r_norm = rhs_norm;
  for (long long it = 1; it <= a.max_iter; ++it) {
    const int par = static_cast<int>(it & 1);
    cl_pass(a, S);  // p complete (previous iteration's barrier) -> x = H^-1 J^T p
    double pq = 0.0, pp = 0.0;
    for (int k = gt; k < a.mc; k += gs) {
      double qk = j_row_dot(k, a.jcsr_rp, a.jcsr_ci_perm, a.jcsr, a.tr.x);
      const double pk = a.p[k];
      if (a.delta2 != 0.0) qk = __dadd_rn(qk, __dmul_rn(a.delta2, pk));
      a.q[k] = qk;
      pq = fma(pk, qk, pq);
      pp = fma(pk, pk, pp);
    }
    const double curvature = cl_sum(pq, S, 1, par);
    const double p_norm2 = cl_sum(pp, S, 2, par);
    if (curvature <= a.thr * p_norm2) {
      if (writer) *a.res = CgResultDev{it - 1, r_norm / rhs_norm, 0, 1};
      return;
    }
    const double alpha = rho / curvature;
    double rr = 0.0;
    for (int k = gt; k < a.mc; k += gs) {
      a.x[k] = __dadd_rn(a.x[k], __dmul_rn(alpha, a.p[k]));
      const double rk = __dsub_rn(a.r[k], __dmul_rn(alpha, a.q[k]));
      a.r[k] = rk;
      rr = fma(rk, rk, rr);
    }
    r_norm = sqrt(cl_sum(rr, S, 3, par));
    const double relres = r_norm / rhs_norm;
    if (relres <= a.tol) {
      if (writer) *a.res = CgResultDev{it, relres, 1, 0};
      return;
    }
    if (it == a.max_iter) {
      if (writer) *a.res = CgResultDev{it, relres, 0, 0};
      return;
    }
    const double rho_next = r_norm * r_norm;
    const double beta = rho_next / rho;
    rho = rho_next;
    for (int k = gt; k < a.mc; k += gs) a.p[k] = __dadd_rn(a.r[k], __dmul_rn(beta, a.p[k]));
    cluster_sync_all();
  }
  if (writer) *a.res = CgResultDev{0, r_norm / rhs_norm, 0, 0};
}

}  // namespace hykkt::dev
