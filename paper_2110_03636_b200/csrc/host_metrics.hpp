// Backward error / relative residual of a returned solution, evaluated on
// the host from downloaded vectors.  Restates the reference's reporting
// formulas (proj/core/src/metrics.cpp:28-49 error_report, :128-162 exact
// block inf-norms, :164-201 block operators, :203-240 kkt reports) so that
// SolveReport fields carry the same meaning.  Not on the timed device path
// (BE/RR are reported separately).
#pragma once

#include <cstdint>
#include <vector>

namespace hykkt {

struct CscView {
  std::int64_t nrows, ncols;
  const std::int64_t* cp;
  const std::int64_t* ri;
  const double* v;
};

struct ErrorReport {
  double be = 0.0, rr = 0.0, a_norm_inf = 0.0, rhs_norm = 0.0, solution_norm = 0.0;
};

// [[H_tilde, J^T], [J, 0]] with H_tilde lower-stored.
ErrorReport error_report_2x2(const CscView& h_tilde, const CscView& j,
                             const double* r_x, const double* r_y,
                             const double* dx, const double* dy);

// Block-4x4 system (kkt_system.hpp:22-28).
ErrorReport error_report_4x4(const CscView& h, const CscView& j,
                             const CscView& jd, const double* d_x,
                             const double* d_s, const double* r_tilde_x,
                             const double* r_s, const double* r_y,
                             const double* r_yd, const double* dx,
                             const double* ds, const double* dy,
                             const double* dyd);

}  // namespace hykkt
