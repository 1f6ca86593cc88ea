// Assembly kernels: reduce -> Ruiz -> H_gamma on fixed index plans.
//
// Bit-exact restatement of the reference's arithmetic order (explicit
// __dmul_rn / __dadd_rn, no FMA contraction — the reference is built without
// -march, so it has none either):
//   reduce            kkt_system.cpp:66-87  (add_symmetric_lower
//                     csc_matrix.cpp:318-347, ata_lower :368-383)
//   ruiz_scale        ruiz.cpp:26-49 (row norms), :76-116 (sweeps + scaling)
//   assemble_h_gamma  solver.cpp:66-84
//   max_abs_diagonal  solver.cpp:30-42
// One thread per output slot; slot product lists are k-ascending, the
// reference's accumulation order.
#pragma once

#include "device_util.cuh"

namespace hykkt::dev {

struct AsmPlan {
  int nx, mc, md;
  // H_tilde slots
  int n_ht;
  const int *ht_row, *ht_col, *ht_hsrc, *ht_pp, *ht_pa, *ht_pb, *ht_pk;
  // H_gamma slots
  int n_hg;
  const int *hg_row, *hg_col, *hg_src, *hg_pp, *hg_pa, *hg_pb;
  // J (CSC: cp over n_x columns, ri rows; col of each entry), J CSR copy map
  int nnz_j;
  const int *j_cp, *j_ri, *j_col, *jcsr_src;
  // J_d CSC
  int nnz_jd;
  const int *jd_cp, *jd_ri;
};

// H_tilde slot values and r_x.
__global__ void k_reduce(AsmPlan p, const double* __restrict__ hval,
                         const double* __restrict__ jdval,
                         const double* __restrict__ d_x,
                         const double* __restrict__ d_s,
                         const double* __restrict__ r_tilde_x,
                         const double* __restrict__ r_s,
                         const double* __restrict__ r_yd,
                         double* __restrict__ ht, double* __restrict__ r_x) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t < p.n_ht) {
    const int col = p.ht_col[t];
    double v = (p.ht_row[t] == col) ? d_x[col] : 0.0;
    const int hs = p.ht_hsrc[t];
    if (hs >= 0) v = __dadd_rn(v, hval[hs]);
    const int q0 = p.ht_pp[t], q1 = p.ht_pp[t + 1];
    if (q1 > q0) {
      double s = 0.0;
      for (int q = q0; q < q1; ++q) {
        s = __dadd_rn(s, __dmul_rn(__dmul_rn(d_s[p.ht_pk[q]], jdval[p.ht_pa[q]]),
                                   jdval[p.ht_pb[q]]));
      }
      v = __dadd_rn(v, s);
    }
    ht[t] = v;
  }
  if (t < p.nx) {
    double acc = 0.0;
    for (int q = p.jd_cp[t]; q < p.jd_cp[t + 1]; ++q) {
      const int k = p.jd_ri[q];
      const double tk = __dadd_rn(__dmul_rn(d_s[k], r_yd[k]), r_s[k]);
      acc = __dadd_rn(acc, __dmul_rn(jdval[q], tk));
    }
    r_x[t] = __dadd_rn(acc, r_tilde_x[t]);
  }
}

struct RuizArgs {
  AsmPlan p;
  const double* ht;    // unscaled H_tilde slots
  const double* jval;  // unscaled J
  double* d;           // n_x + m_c
  double* norms;       // n_x + m_c
  int* unconverged;    // [max_iters + 1], zeroed
  int* sweeps_out;
  int max_iters;
  double tol;
  GridBarrier bar;
  int* abort;
};

// Cooperative persistent kernel: the whole sweep loop of ruiz_scale.
__global__ void k_ruiz(RuizArgs a) {
  const int nrow = a.p.nx + a.p.mc;
  const int gt = blockIdx.x * blockDim.x + threadIdx.x;
  const int gs = gridDim.x * blockDim.x;
  for (int i = gt; i < nrow; i += gs) a.d[i] = 1.0;
  int sweeps = 0;
  for (int it = 1; it <= a.max_iters; ++it) {
    sweeps = it;
    for (int i = gt; i < nrow; i += gs) a.norms[i] = 0.0;
    grid_sync(a.bar, a.abort);
    for (int t = gt; t < a.p.n_ht; t += gs) {
      const int i = a.p.ht_row[t], j = a.p.ht_col[t];
      const double v = __dmul_rn(__dmul_rn(fabs(a.ht[t]), ldcg(a.d + i)), ldcg(a.d + j));
      atomic_max_nonneg(a.norms + i, v);
      if (i != j) atomic_max_nonneg(a.norms + j, v);
    }
    for (int q = gt; q < a.p.nnz_j; q += gs) {
      const int k = a.p.j_ri[q], j = a.p.j_col[q];
      const double v =
          __dmul_rn(__dmul_rn(fabs(a.jval[q]), ldcg(a.d + a.p.nx + k)), ldcg(a.d + j));
      atomic_max_nonneg(a.norms + a.p.nx + k, v);
      atomic_max_nonneg(a.norms + j, v);
    }
    grid_sync(a.bar, a.abort);
    for (int i = gt; i < nrow; i += gs) {
      const double v = ldcg(a.norms + i);
      if (v > 0.0 && fabs(v - 1.0) > a.tol) {
        atomicOr(a.unconverged + it, 1);
        break;
      }
    }
    grid_sync(a.bar, a.abort);
    if (ld_relaxed(a.unconverged + it) == 0) break;
    for (int i = gt; i < nrow; i += gs) {
      const double v = ldcg(a.norms + i);
      if (v > 0.0) a.d[i] = __ddiv_rn(ldcg(a.d + i), __dsqrt_rn(v));
    }
    grid_sync(a.bar, a.abort);
  }
  if (gt == 0) *a.sweeps_out = sweeps;
}

// Scaled H_tilde, J (CSC + CSR copies), r_x, r_y  (ruiz.cpp:107-114, :51-72).
__global__ void k_scale(AsmPlan p, const double* __restrict__ d,
                        const double* __restrict__ ht,
                        const double* __restrict__ jval,
                        const double* __restrict__ r_x,
                        const double* __restrict__ r_y, double* __restrict__ hts,
                        double* __restrict__ js, double* __restrict__ js_csr,
                        double* __restrict__ rxs, double* __restrict__ rys) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t < p.n_ht) hts[t] = __dmul_rn(ht[t], __dmul_rn(d[p.ht_row[t]], d[p.ht_col[t]]));
  if (t < p.nnz_j) {
    js[t] = __dmul_rn(jval[t], __dmul_rn(d[p.nx + p.j_ri[t]], d[p.j_col[t]]));
    const int s = p.jcsr_src[t];
    js_csr[t] = __dmul_rn(jval[s], __dmul_rn(d[p.nx + p.j_ri[s]], d[p.j_col[s]]));
  }
  if (t < p.nx) rxs[t] = __dmul_rn(d[t], r_x[t]);
  if (t < p.mc) rys[t] = __dmul_rn(d[p.nx + t], r_y[t]);
}

// H_gamma slots, r_hat_x and max |diag H_gamma| (solver.cpp:66-84, :30-42).
__global__ void k_hgamma(AsmPlan p, double gamma, const double* __restrict__ hts,
                         const double* __restrict__ js,
                         const double* __restrict__ rxs,
                         const double* __restrict__ rys, double* __restrict__ hg,
                         double* __restrict__ rhat, double* __restrict__ maxdiag) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t < p.n_hg) {
    const int src = p.hg_src[t];
    double v = (src >= 0) ? __dadd_rn(0.0, hts[src]) : 0.0;
    const int q0 = p.hg_pp[t], q1 = p.hg_pp[t + 1];
    if (q1 > q0) {
      double s = 0.0;
      for (int q = q0; q < q1; ++q) s = __dadd_rn(s, __dmul_rn(js[p.hg_pa[q]], js[p.hg_pb[q]]));
      v = __dadd_rn(v, __dmul_rn(gamma, s));
    }
    hg[t] = v;
    if (p.hg_row[t] == p.hg_col[t]) atomic_max_nonneg(maxdiag, fabs(v));
  }
  if (t < p.nx) {
    double acc = 0.0;
    for (int q = p.j_cp[t]; q < p.j_cp[t + 1]; ++q) acc = __dadd_rn(acc, __dmul_rn(js[q], rys[p.j_ri[q]]));
    rhat[t] = __dadd_rn(rxs[t], __dmul_rn(gamma, acc));
  }
}

// H_delta = H_gamma + delta1 I scattered into zeroed supernodal panels
// (add_diagonal_shift solver.cpp:86-106 + the scatter of numeric_cholesky
// cholesky.cpp:92-100).  Generic: values in `src` CSC order.
__global__ void k_scatter(int nsrc, const double* __restrict__ src,
                          const int* __restrict__ src_to_panel,
                          const int* __restrict__ src_row,
                          const int* __restrict__ src_col, double delta1,
                          double* __restrict__ panel) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= nsrc) return;
  double v = src[t];
  if (delta1 != 0.0 && src_row[t] == src_col[t]) v = __dadd_rn(v, delta1);
  panel[src_to_panel[t]] = v;
}

// v[i] = value (identity Ruiz scaling of the Reduced2x2 entry points).
__global__ void k_fill(double* __restrict__ v, int n, double value) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t < n) v[t] = value;
}

// max |diag| of a matrix given as values in `src` CSC order
// (max_abs_diagonal, solver.cpp:30-42) for the Cholesky-level ladder.
__global__ void k_maxdiag_src(int nsrc, const double* __restrict__ src, const int* __restrict__ src_row,
                              const int* __restrict__ src_col, double* __restrict__ maxdiag) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t < nsrc && src_row[t] == src_col[t]) atomic_max_nonneg(maxdiag, fabs(src[t]));
}

// Unscale + recover (ruiz.cpp:118-133, kkt_system.cpp:89-105).
__global__ void k_recover(AsmPlan p, const int* __restrict__ jd_rp,
                          const int* __restrict__ jd_ci,
                          const int* __restrict__ jd_src,
                          const double* __restrict__ d,
                          const double* __restrict__ dx_s,
                          const double* __restrict__ dy_s,
                          const double* __restrict__ jdval,
                          const double* __restrict__ d_s,
                          const double* __restrict__ r_s,
                          const double* __restrict__ r_yd,
                          double* __restrict__ dx, double* __restrict__ dy,
                          double* __restrict__ ds, double* __restrict__ dyd) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t < p.nx) dx[t] = __dmul_rn(d[t], dx_s[t]);
  if (t < p.mc) dy[t] = __dmul_rn(d[p.nx + t], dy_s[t]);
  if (t < p.md) {
    // J_d dx in ascending column order (spmv scatter, csc_matrix.cpp:250-254);
    // dx recomputed from dx_s to avoid a dependency on the lines above.
    double acc = 0.0;
    for (int q = jd_rp[t]; q < jd_rp[t + 1]; ++q) {
      const int c = jd_ci[q];
      const double xc = __dmul_rn(d[c], dx_s[c]);
      if (xc == 0.0) continue;
      acc = __dadd_rn(acc, __dmul_rn(jdval[jd_src[q]], xc));
    }
    const double s = __dsub_rn(acc, r_yd[t]);
    ds[t] = s;
    dyd[t] = __dsub_rn(__dmul_rn(d_s[t], s), r_s[t]);
  }
}

}  // namespace hykkt::dev
