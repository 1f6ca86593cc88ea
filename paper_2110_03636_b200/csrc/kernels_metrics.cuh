// Backward error / relative residual of a solve on the device
// (error_report_kkt4x4 / error_report_kkt2x2, proj/core/src/metrics.cpp
// 28-240): the reports every SolveReport carries (solver.cpp:289-291,
// :318-325) without downloading the solution.
//
// For a system K x = b:  be = ||K x - b||_2 / (||K||_inf ||x||_2 + ||b||_2),
// rr = ||K x - b||_2 / ||b||_2 (0 / inf conventions of metrics.cpp:28-49);
// ||K||_inf is the maximum absolute row sum with H treated symmetrically and
// the diagonal overlap |H_ii + d_i| (metrics.cpp sym_plus_diag_row_sums).
// One thread per row of the 4x4 system and of the 2x2 systems (unscaled and
// Ruiz-scaled), rows read through row lists of [[H_tilde, J^T], [J, 0]]
// (every H_tilde entry in its row and, off the diagonal, its column's list;
// every J entry in its row and its column's list), J_d through CSC / CSR.
// Per-block partial sums / maxima, then one block combines them in a fixed
// order: deterministic.
#pragma once

#include "kernels_assemble.cuh"

namespace hykkt::dev {

// partial slots per block: 3 reports x (res^2, x^2, b^2, max row sum)
constexpr int kMetSlots = 12;

struct MetricsArgs {
  AsmPlan p;
  const int* rows_ptr;   // row lists of [[H_tilde, J^T], [J, 0]] (nx + mc + 1)
  const int4* rows_ent;  // (value index, row, col, -): value index < n_ht -> H_tilde slot, else J entry
  const int *jd_rp, *jd_ci, *jd_src;  // J_d CSR
  // original system (4x4)
  const double *h, *j, *jd, *d_x, *d_s, *r_tx, *r_s, *r_y, *r_yd;
  const double *dx, *ds, *dy, *dyd;
  // reduced systems: unscaled (H_tilde, J, r_x, r_y) and scaled (H_tilde_s, J_s, r_x_s, r_y_s)
  const double *ht, *rx, *hts, *js, *rxs, *rys;
  const double *dx_s, *dy_s;
  int with_4x4;
  double* partials;      // gridDim.x * kMetSlots
};

__device__ __forceinline__ double block_max(double v, double* scratch) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  __syncthreads();
  if (lane == 0) scratch[wid] = v;
  __syncthreads();
  const int nw = (blockDim.x + 31) >> 5;
  double t = (lane < nw) ? scratch[lane] : 0.0;
  if (wid == 0) {
    for (int o = 16; o > 0; o >>= 1) t = fmax(t, __shfl_xor_sync(0xffffffffu, t, o));
    if (lane == 0) scratch[32] = t;
  }
  __syncthreads();
  const double r = scratch[32];
  __syncthreads();
  return r;
}

__global__ void __launch_bounds__(256) k_metrics_rows(MetricsArgs a) {
  __shared__ double scratch[33];
  const AsmPlan& p = a.p;
  const int nx = p.nx, mc = p.mc, md = p.md;
  const int gt = blockIdx.x * blockDim.x + threadIdx.x, gs = gridDim.x * blockDim.x;
  double acc[kMetSlots];
#pragma unroll
  for (int k = 0; k < kMetSlots; ++k) acc[k] = 0.0;
  auto add = [&](int rep, double res, double x, double b, double rowsum) {
    acc[4 * rep] += res * res;
    acc[4 * rep + 1] += x * x;
    acc[4 * rep + 2] += b * b;
    acc[4 * rep + 3] = fmax(acc[4 * rep + 3], rowsum);
  };
  // ---- reduced 2x2 systems (report 1: unscaled, report 2: scaled) ----
  for (int i = gt; i < nx + mc; i += gs) {
    double ru = 0.0, rs = 0.0, du = 0.0, ds_ = 0.0, ou = 0.0, os = 0.0;
    const bool top = i < nx;
    for (int e = a.rows_ptr[i]; e < a.rows_ptr[i + 1]; ++e) {
      const int4 en = a.rows_ent[e];
      const int other = en.y == i ? en.z : en.y;
      double vu, vs;
      if (en.x < p.n_ht) {
        vu = a.ht[en.x];
        vs = a.hts[en.x];
        if (en.y == en.z) {
          du += vu;
          ds_ += vs;
          continue;
        }
      } else {
        vu = a.j[en.x - p.n_ht];
        vs = a.js[en.x - p.n_ht];
      }
      const double xu = other < nx ? a.dx[other] : a.dy[other - nx];
      const double xs = other < nx ? a.dx_s[other] : a.dy_s[other - nx];
      ru = fma(vu, xu, ru);
      rs = fma(vs, xs, rs);
      ou += fabs(vu);
      os += fabs(vs);
    }
    if (top) {
      ru = fma(du, a.dx[i], ru) - a.rx[i];
      rs = fma(ds_, a.dx_s[i], rs) - a.rxs[i];
      add(1, ru, a.dx[i], a.rx[i], ou + fabs(du));
      add(2, rs, a.dx_s[i], a.rxs[i], os + fabs(ds_));
    } else {
      const int k = i - nx;
      ru -= a.r_y[k];
      rs -= a.rys[k];
      add(1, ru, a.dy[k], a.r_y[k], ou);
      add(2, rs, a.dy_s[k], a.rys[k], os);
    }
  }
  // ---- the 4x4 system (report 0) ----
  if (a.with_4x4) {
    const int n4 = nx + 2 * md + mc;
    for (int i = gt; i < n4; i += gs) {
      double res = 0.0, rowsum = 0.0, x, b;
      if (i < nx) {
        double diag = 0.0;
        for (int e = a.rows_ptr[i]; e < a.rows_ptr[i + 1]; ++e) {
          const int4 en = a.rows_ent[e];
          if (en.x < p.n_ht) {
            const int hs = p.ht_hsrc[en.x];
            const double v = hs >= 0 ? a.h[hs] : 0.0;
            if (en.y == en.z) {
              diag += v;
            } else {
              res = fma(v, a.dx[en.y == i ? en.z : en.y], res);
              rowsum += fabs(v);
            }
          } else {
            const double v = a.j[en.x - p.n_ht];
            res = fma(v, a.dy[en.y - nx], res);
            rowsum += fabs(v);
          }
        }
        const double dd = diag + a.d_x[i];
        res = fma(dd, a.dx[i], res);
        rowsum += fabs(dd);
        for (int q = p.jd_cp[i]; q < p.jd_cp[i + 1]; ++q) {
          res = fma(a.jd[q], a.dyd[p.jd_ri[q]], res);
          rowsum += fabs(a.jd[q]);
        }
        x = a.dx[i];
        b = a.r_tx[i];
      } else if (i < nx + md) {
        const int k = i - nx;
        res = a.d_s[k] * a.ds[k] - a.dyd[k];
        rowsum = fabs(a.d_s[k]) + 1.0;
        x = a.ds[k];
        b = a.r_s[k];
      } else if (i < nx + md + mc) {
        const int k = i - nx - md;
        for (int e = a.rows_ptr[nx + k]; e < a.rows_ptr[nx + k + 1]; ++e) {
          const int4 en = a.rows_ent[e];
          const double v = a.j[en.x - p.n_ht];
          res = fma(v, a.dx[en.z], res);
          rowsum += fabs(v);
        }
        x = a.dy[k];
        b = a.r_y[k];
      } else {
        const int k = i - nx - md - mc;
        for (int q = a.jd_rp[k]; q < a.jd_rp[k + 1]; ++q) {
          const double v = a.jd[a.jd_src[q]];
          res = fma(v, a.dx[a.jd_ci[q]], res);
          rowsum += fabs(v);
        }
        res -= a.ds[k];
        rowsum += 1.0;
        x = a.dyd[k];
        b = a.r_yd[k];
      }
      add(0, res - b, x, b, rowsum);
    }
  }
#pragma unroll
  for (int k = 0; k < kMetSlots; ++k) {
    const double v = (k & 3) == 3 ? block_max(acc[k], scratch) : block_sum(acc[k], scratch);
    if (threadIdx.x == 0) a.partials[blockIdx.x * kMetSlots + k] = v;
  }
}

// out[2 r] = be, out[2 r + 1] = rr of report r (0: 4x4, 1: 2x2, 2: 2x2 scaled)
__global__ void __launch_bounds__(256) k_metrics_final(const double* partials, int nblocks, double* out) {
  __shared__ double scratch[33];
  for (int r = 0; r < 3; ++r) {
    double s[4];
    for (int k = 0; k < 4; ++k) {
      double v = 0.0;
      for (int b = threadIdx.x; b < nblocks; b += blockDim.x) {
        const double x = partials[b * kMetSlots + 4 * r + k];
        v = k == 3 ? fmax(v, x) : v + x;
      }
      s[k] = k == 3 ? block_max(v, scratch) : block_sum(v, scratch);
    }
    if (threadIdx.x == 0) {
      const double res = sqrt(s[0]), xn = sqrt(s[1]), bn = sqrt(s[2]), an = s[3];
      const double inf = __longlong_as_double(0x7ff0000000000000ll);
      const double den = an * xn + bn;
      out[2 * r] = den > 0.0 ? res / den : (res == 0.0 ? 0.0 : inf);
      out[2 * r + 1] = bn > 0.0 ? res / bn : (res == 0.0 ? 0.0 : inf);
    }
  }
}

}  // namespace hykkt::dev
