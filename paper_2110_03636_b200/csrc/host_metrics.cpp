#include "host_metrics.hpp"

#include <algorithm>
#include <cmath>
#include <limits>

namespace hykkt {

namespace {

using i64 = std::int64_t;

double norm2(const std::vector<double>& v) {
  double acc = 0.0;
  for (double x : v) acc += x * x;
  return std::sqrt(acc);
}

ErrorReport finish(const std::vector<double>& residual, const std::vector<double>& x,
                   const std::vector<double>& b, double a_norm) {
  ErrorReport rep;
  rep.a_norm_inf = a_norm;
  rep.rhs_norm = norm2(b);
  rep.solution_norm = norm2(x);
  const double res = norm2(residual);
  const double den = a_norm * rep.solution_norm + rep.rhs_norm;
  const double inf = std::numeric_limits<double>::infinity();
  rep.be = den > 0.0 ? res / den : (res == 0.0 ? 0.0 : inf);
  rep.rr = rep.rhs_norm > 0.0 ? res / rep.rhs_norm : (res == 0.0 ? 0.0 : inf);
  return rep;
}

// y += (L + L^T - diag L) x
void sym_apply(const CscView& a, const double* x, double* y) {
  for (i64 j = 0; j < a.ncols; ++j) {
    double acc = 0.0;
    for (i64 p = a.cp[j]; p < a.cp[j + 1]; ++p) {
      const i64 i = a.ri[p];
      y[i] += a.v[p] * x[j];
      if (i != j) acc += a.v[p] * x[i];
    }
    y[j] += acc;
  }
}

void apply(const CscView& a, const double* x, double* y) {  // y += A x
  for (i64 j = 0; j < a.ncols; ++j) {
    for (i64 p = a.cp[j]; p < a.cp[j + 1]; ++p) y[a.ri[p]] += a.v[p] * x[j];
  }
}

void apply_t(const CscView& a, const double* x, double* y) {  // y += A^T x
  for (i64 j = 0; j < a.ncols; ++j) {
    double acc = 0.0;
    for (i64 p = a.cp[j]; p < a.cp[j + 1]; ++p) acc += a.v[p] * x[a.ri[p]];
    y[j] += acc;
  }
}

// |H + diag(d)| row sums with the symmetric mirror; overlap |H_ii + d_i|.
std::vector<double> top_rows(const CscView& h, const double* d) {
  const i64 n = h.ncols;
  std::vector<double> diag(n, 0.0), off(n, 0.0);
  for (i64 j = 0; j < n; ++j) {
    for (i64 p = h.cp[j]; p < h.cp[j + 1]; ++p) {
      const i64 i = h.ri[p];
      if (i == j) {
        diag[i] += h.v[p];
      } else {
        off[i] += std::fabs(h.v[p]);
        off[j] += std::fabs(h.v[p]);
      }
    }
  }
  std::vector<double> s(n);
  for (i64 i = 0; i < n; ++i) s[i] = off[i] + std::fabs(diag[i] + (d ? d[i] : 0.0));
  return s;
}

void col_abs_sums(const CscView& a, double* t) {
  for (i64 j = 0; j < a.ncols; ++j) {
    double s = 0.0;
    for (i64 p = a.cp[j]; p < a.cp[j + 1]; ++p) s += std::fabs(a.v[p]);
    t[j] += s;
  }
}

void row_abs_sums(const CscView& a, double* t) {
  for (i64 j = 0; j < a.ncols; ++j) {
    for (i64 p = a.cp[j]; p < a.cp[j + 1]; ++p) t[a.ri[p]] += std::fabs(a.v[p]);
  }
}

}  // namespace

ErrorReport error_report_2x2(const CscView& h, const CscView& j, const double* r_x,
                             const double* r_y, const double* dx, const double* dy) {
  const i64 nx = h.ncols, mc = j.nrows;
  std::vector<double> out(nx + mc, 0.0), x(nx + mc), b(nx + mc);
  sym_apply(h, dx, out.data());
  apply_t(j, dy, out.data());
  apply(j, dx, out.data() + nx);
  for (i64 i = 0; i < nx; ++i) {
    x[i] = dx[i];
    b[i] = r_x[i];
  }
  for (i64 k = 0; k < mc; ++k) {
    x[nx + k] = dy[k];
    b[nx + k] = r_y[k];
  }
  for (i64 i = 0; i < nx + mc; ++i) out[i] -= b[i];
  std::vector<double> sums(nx + mc, 0.0);
  const std::vector<double> top = top_rows(h, nullptr);
  std::copy(top.begin(), top.end(), sums.begin());
  col_abs_sums(j, sums.data());
  row_abs_sums(j, sums.data() + nx);
  double an = 0.0;
  for (double v : sums) an = std::max(an, v);
  return finish(out, x, b, an);
}

ErrorReport error_report_4x4(const CscView& h, const CscView& j, const CscView& jd,
                             const double* d_x, const double* d_s,
                             const double* r_tilde_x, const double* r_s,
                             const double* r_y, const double* r_yd, const double* dx,
                             const double* ds, const double* dy, const double* dyd) {
  const i64 nx = h.ncols, mc = j.nrows, md = jd.nrows;
  const i64 n = nx + 2 * md + mc;
  std::vector<double> out(n, 0.0), x(n), b(n);
  // row 1: (H + D_x) dx + J^T dy + J_d^T dyd
  sym_apply(h, dx, out.data());
  for (i64 i = 0; i < nx; ++i) out[i] += d_x[i] * dx[i];
  apply_t(j, dy, out.data());
  apply_t(jd, dyd, out.data());
  // row 2: D_s ds - dyd
  for (i64 i = 0; i < md; ++i) out[nx + i] = d_s[i] * ds[i] - dyd[i];
  // row 3: J dx ; row 4: J_d dx - ds
  apply(j, dx, out.data() + nx + md);
  apply(jd, dx, out.data() + nx + md + mc);
  for (i64 i = 0; i < md; ++i) out[nx + md + mc + i] -= ds[i];
  i64 o = 0;
  for (i64 i = 0; i < nx; ++i, ++o) { x[o] = dx[i]; b[o] = r_tilde_x[i]; }
  for (i64 i = 0; i < md; ++i, ++o) { x[o] = ds[i]; b[o] = r_s[i]; }
  for (i64 i = 0; i < mc; ++i, ++o) { x[o] = dy[i]; b[o] = r_y[i]; }
  for (i64 i = 0; i < md; ++i, ++o) { x[o] = dyd[i]; b[o] = r_yd[i]; }
  for (i64 i = 0; i < n; ++i) out[i] -= b[i];

  std::vector<double> sums(n, 0.0);
  const std::vector<double> top = top_rows(h, d_x);
  std::copy(top.begin(), top.end(), sums.begin());
  col_abs_sums(j, sums.data());
  col_abs_sums(jd, sums.data());
  for (i64 i = 0; i < md; ++i) sums[nx + i] = std::fabs(d_s[i]) + 1.0;
  row_abs_sums(j, sums.data() + nx + md);
  row_abs_sums(jd, sums.data() + nx + md + mc);
  for (i64 i = 0; i < md; ++i) sums[nx + md + mc + i] += 1.0;
  double an = 0.0;
  for (double v : sums) an = std::max(an, v);
  return finish(out, x, b, an);
}

}  // namespace hykkt
