// Sync-free supernodal triangular solves and the device-resident CG loop.
//
// factor_solve (proj/core/src/cholesky.cpp:139-168) becomes one pass of
// 2 * nsup warp tasks: forward tasks in level order (pull: a row gathers its
// strictly-lower entries from descendant supernodes through row lists, then
// a dense forward solve of the diagonal block), followed by backward tasks
// in reverse level order (gather over the panel's below-diagonal rows, then
// a dense backward solve).  A forward task waits on its children's flags; a
// backward task on its parent's (the root on its own forward flag).  The
// permutation is folded into the gathers: rows read b[perm[i]] / the J
// column perm[i], and outputs scatter to x[perm[i]].
//
// cg_schur (solver.cpp:154-201) runs as ONE cooperative persistent kernel:
// each iteration = [J^T p fused into the forward solve -> H^-1 -> J t +
// delta2 p, p.q, p.p] -> grid barrier -> [alpha, x, r, r.r] -> grid barrier
// -> [convergence, beta, p] -> grid barrier.  No host round trips; dot
// products use per-block partials combined in a fixed order, so results are
// deterministic.  Termination rules mirror solver.cpp:161-199 exactly
// (zero rhs -> 0 iterations; small quadratic pq <= thr * pp -> abort with
// iterations = it - 1; relres = ||r|| / ||rhs|| <= tol; iteration cap).
#pragma once

#include "kernels_factor.cuh"

namespace hykkt::dev {

struct SolveRhs {
  const double* b;   // original-order vector (n) or null
  const double* u;   // J^T u term (m_c) or null; b - J^T u when both
  const int* j_cp;
  const int* j_ri;
  const double* jval;
};

struct TrsvArgs {
  SnPlan s;
  const double* panel;
  double* y;       // permuted work vector, holds the solution afterwards
  double* x_out;   // original-order output or null
  int* fdone;
  int* bdone;
  int epoch;
  int* abort;
  SolveRhs rhs;
};

__device__ void fwd_task(const TrsvArgs& a, int sn, int lane) {
  const SnPlan& s = a.s;
  const int f = s.first[sn], w = s.first[sn + 1] - f, nr = s.nrows[sn];
  const double* P = a.panel + s.off[sn];
  for (int c = s.child_ptr[sn] + lane; c < s.child_ptr[sn + 1]; c += 32) {
    if (!wait_flag(a.fdone + s.child[c], a.epoch, a.abort)) break;
  }
  __syncwarp();
  __threadfence();
  for (int cb = 0; cb < w; cb += 32) {
    const int cw = min(32, w - cb);
    double acc = 0.0;
    if (lane < cw) {
      const int o = s.perm[f + cb + lane];
      double bi = a.rhs.b ? a.rhs.b[o] : 0.0;
      if (a.rhs.u) {
        double t = 0.0;  // spmv(J, u, transpose) order, csc_matrix.cpp:255-261
        for (int q = a.rhs.j_cp[o]; q < a.rhs.j_cp[o + 1]; ++q) {
          t = __dadd_rn(t, __dmul_rn(a.rhs.jval[q], ldcg(a.rhs.u + a.rhs.j_ri[q])));
        }
        bi = a.rhs.b ? __dsub_rn(bi, t) : t;
      }
      acc = bi;
    }
    for (int rr = 0; rr < cw; ++rr) {
      const int i = f + cb + rr;
      double part = 0.0;
      for (int e = s.lrow_ptr[i] + lane; e < s.lrow_ptr[i + 1]; e += 32) {
        part = fma(__ldg(a.panel + s.lrow_pos[e]), ldcg(a.y + s.lrow_col[e]), part);
      }
      for (int k = lane; k < cb; k += 32) part = fma(__ldg(P + k * nr + cb + rr), ldcg(a.y + f + k), part);
      part = warp_sum(part);
      if (lane == rr) acc -= part;
    }
    for (int k = 0; k < cw; ++k) {
      const double yk = __shfl_sync(0xffffffffu, acc, k) / __ldg(P + (cb + k) * nr + cb + k);
      if (lane == k) acc = yk;
      if (lane > k && lane < cw) acc = fma(-__ldg(P + (cb + k) * nr + cb + lane), yk, acc);
    }
    if (lane < cw) stcg(a.y + f + cb + lane, acc);
    __syncwarp();
  }
  __threadfence();
  if (lane == 0) st_release(a.fdone + sn, a.epoch);
}

__device__ void bwd_task(const TrsvArgs& a, int sn, int lane) {
  const SnPlan& s = a.s;
  const int f = s.first[sn], w = s.first[sn + 1] - f, nr = s.nrows[sn];
  const double* P = a.panel + s.off[sn];
  const int* R = s.rows + s.rows_ptr[sn];
  if (lane == 0) {
    const int par = s.parent[sn];
    if (par < 0) wait_flag(a.fdone + sn, a.epoch, a.abort);
    else wait_flag(a.bdone + par, a.epoch, a.abort);
  }
  __syncwarp();
  __threadfence();
  const int nchunks = (w + 31) >> 5;
  for (int ci = nchunks - 1; ci >= 0; --ci) {
    const int cb = ci * 32, cw = min(32, w - cb);
    double acc = (lane < cw) ? ldcg(a.y + f + cb + lane) : 0.0;
    for (int kk = 0; kk < cw; ++kk) {
      const double* Pc = P + (cb + kk) * nr;
      double part = 0.0;
      for (int r = cb + cw + lane; r < nr; r += 32) part = fma(__ldg(Pc + r), ldcg(a.y + __ldg(R + r)), part);
      part = warp_sum(part);
      if (lane == kk) acc -= part;
    }
    for (int k = cw - 1; k >= 0; --k) {
      const double xk = __shfl_sync(0xffffffffu, acc, k) / __ldg(P + (cb + k) * nr + cb + k);
      if (lane == k) acc = xk;
      if (lane < k) acc = fma(-__ldg(P + (cb + lane) * nr + cb + k), xk, acc);
    }
    if (lane < cw) {
      stcg(a.y + f + cb + lane, acc);
      if (a.x_out) a.x_out[s.perm[f + cb + lane]] = acc;
    }
    __syncwarp();
  }
  __threadfence();
  if (lane == 0) st_release(a.bdone + sn, a.epoch);
}

__device__ __forceinline__ void trsv_pass(const TrsvArgs& a) {
  const int lane = threadIdx.x & 31;
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  const int ns = a.s.nsup;
  for (int t = gw; t < 2 * ns; t += nw) {
    if (t < ns) fwd_task(a, a.s.order[t], lane);
    else bwd_task(a, a.s.order[2 * ns - 1 - t], lane);
  }
}

__global__ void __launch_bounds__(256) k_trsv(TrsvArgs a) { trsv_pass(a); }

// q = J t - r_y style products: out[k] = sum_e J_csr[e] * y[ci_perm[e]]
// (+ sub[k] subtracted), reference spmv scatter order (csc_matrix.cpp:250-254,
// zero entries of t skipped exactly as there).
__device__ __forceinline__ double j_row_dot(int k, const int* rp, const int* ci_perm,
                                            const double* jcsr, const double* y) {
  double acc = 0.0;
  for (int e = rp[k]; e < rp[k + 1]; ++e) {
    const double t = ldcg(y + ci_perm[e]);
    if (t == 0.0) continue;
    acc = __dadd_rn(acc, __dmul_rn(jcsr[e], t));
  }
  return acc;
}

// Schur right-hand side J w - r_y (solver.cpp:254-255).
__global__ void k_schur_rhs(int mc, const int* rp, const int* ci_perm,
                            const double* jcsr, const double* y,
                            const double* r_y, double* rhs) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k < mc) rhs[k] = __dsub_rn(j_row_dot(k, rp, ci_perm, jcsr, y), r_y[k]);
}

struct CgResultDev {
  long long iterations;
  double relres;
  int converged;
  int small_quadratic;
};

struct CgArgs {
  TrsvArgs tr;  // rhs.u must point at p
  int mc;
  const int* jcsr_rp;
  const int* jcsr_ci_perm;
  const double* jcsr;
  const double* rhs;
  double* x;
  double* r;
  double* p;
  double* q;
  double* partials;  // 4 per block
  double delta2;
  double tol;
  double thr;
  long long max_iter;
  int epoch_base;
  CgResultDev* res;
  GridBarrier bar;
};

// Deterministic all-blocks reduction of partials[b * 4 + slot].
__device__ __forceinline__ double reduce_partials(const double* partials, int slot, double* scratch) {
  double v = 0.0;
  for (int b = threadIdx.x; b < gridDim.x; b += blockDim.x) v += ldcg(partials + b * 4 + slot);
  return block_sum(v, scratch);
}

__global__ void __launch_bounds__(256) k_cg(CgArgs a) {
  __shared__ double scratch[33];
  const int gt = blockIdx.x * blockDim.x + threadIdx.x;
  const int gs = gridDim.x * blockDim.x;
  int* abort = a.tr.abort;
  double ss = 0.0;
  for (int k = gt; k < a.mc; k += gs) {
    const double v = a.rhs[k];
    a.x[k] = 0.0;
    a.r[k] = v;
    a.p[k] = v;
    ss = fma(v, v, ss);
  }
  ss = block_sum(ss, scratch);
  if (threadIdx.x == 0) a.partials[blockIdx.x * 4] = ss;
  grid_sync(a.bar, abort);
  const double rhs_norm = sqrt(reduce_partials(a.partials, 0, scratch));
  const bool writer = gt == 0;
  if (rhs_norm == 0.0) {
    if (writer) *a.res = CgResultDev{0, 0.0, 1, 0};
    return;
  }
  double rho = rhs_norm * rhs_norm;
  double r_norm = rhs_norm;
  TrsvArgs tr = a.tr;
  for (long long it = 1; it <= a.max_iter; ++it) {
    tr.epoch = a.epoch_base + static_cast<int>(it);
    trsv_pass(tr);
    grid_sync(a.bar, abort);
    double pq = 0.0, pp = 0.0;
    for (int k = gt; k < a.mc; k += gs) {
      double qk = j_row_dot(k, a.jcsr_rp, a.jcsr_ci_perm, a.jcsr, tr.y);
      const double pk = ldcg(a.p + k);
      if (a.delta2 != 0.0) qk = __dadd_rn(qk, __dmul_rn(a.delta2, pk));
      a.q[k] = qk;
      pq = fma(pk, qk, pq);
      pp = fma(pk, pk, pp);
    }
    pq = block_sum(pq, scratch);
    pp = block_sum(pp, scratch);
    if (threadIdx.x == 0) {
      a.partials[blockIdx.x * 4 + 1] = pq;
      a.partials[blockIdx.x * 4 + 2] = pp;
    }
    grid_sync(a.bar, abort);
    const double curvature = reduce_partials(a.partials, 1, scratch);
    const double p_norm2 = reduce_partials(a.partials, 2, scratch);
    if (curvature <= a.thr * p_norm2 || ld_relaxed(abort)) {
      if (writer) *a.res = CgResultDev{it - 1, r_norm / rhs_norm, 0, 1};
      return;
    }
    const double alpha = rho / curvature;
    double rr = 0.0;
    for (int k = gt; k < a.mc; k += gs) {
      a.x[k] = __dadd_rn(a.x[k], __dmul_rn(alpha, ldcg(a.p + k)));
      const double rk = __dsub_rn(a.r[k], __dmul_rn(alpha, a.q[k]));
      a.r[k] = rk;
      rr = fma(rk, rk, rr);
    }
    rr = block_sum(rr, scratch);
    if (threadIdx.x == 0) a.partials[blockIdx.x * 4 + 3] = rr;
    grid_sync(a.bar, abort);
    r_norm = sqrt(reduce_partials(a.partials, 3, scratch));
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
    for (int k = gt; k < a.mc; k += gs) {
      a.p[k] = __dadd_rn(a.r[k], __dmul_rn(beta, a.p[k]));
    }
    grid_sync(a.bar, abort);
  }
  if (writer) *a.res = CgResultDev{0, r_norm / rhs_norm, 0, 0};
}

}  // namespace hykkt::dev
