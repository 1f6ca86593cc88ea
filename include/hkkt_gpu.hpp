// hkkt_gpu.hpp — drop-in C++ replacement of the reference solver's hot path
// (proj/core/include/hkkt/{cholesky,solver}.hpp) backed by the B200 C ABI
// (hykkt.h, libhykkt.so).
//
// A maintainer of the reference compiles this header inside the reference
// tree (it includes the reference's own types: CscMatrix, SymbolicFactor,
// NumericCholesky, Reduced2x2, HGammaSystem, SolverConfig, ...) and links
// libhykkt.so.  Every function below has the signature of the reference
// function it replaces, in namespace hkkt::gpu; switching a caller over is
// `using namespace hkkt::gpu;` or a qualified call:
//
//   numeric_cholesky        cholesky.hpp:76-78
//   factor_solve            cholesky.hpp:82-83
//   assemble_h_gamma        solver.hpp:75
//   factorize_with_ladder   solver.hpp:92-94
//   cg_schur                solver.hpp:121-122   (CgTrace unsupported: throws)
//   solve_reduced           solver.hpp:167-170
//   solve_full              solver.hpp:182-184
//   solve_sequence          solver.hpp:204-205   (parallel_sequence -> batched path)
//
// Error conventions follow the reference: argument / structure errors throw
// hkkt::InvalidMatrixError (csc_matrix.hpp:29-33); not-SPD, ladder
// exhaustion, small quadratic and the CG cap are returned as values.  Device
// state lives in per-thread handle caches keyed by the SymbolicFactor (or
// pattern) a call uses, so repeated calls with one symbolic factor reuse one
// analysed device plan.
#ifndef HKKT_GPU_HPP_
#define HKKT_GPU_HPP_

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <limits>
#include <memory>
#include <span>
#include <string>
#include <utility>
#include <vector>

#include "hkkt/cholesky.hpp"
#include "hkkt/kkt_system.hpp"
#include "hkkt/metrics.hpp"
#include "hkkt/solver.hpp"
#include "hykkt.h"

namespace hkkt::gpu {

namespace detail {

inline void check(int code) {
  if (code != HYKKT_OK) {
    throw InvalidMatrixError(std::string("hykkt: ") + hykkt_last_error() + " (status " +
                             std::to_string(code) + ")");
  }
}

inline hykkt_config_t to_c(const SolverConfig& cfg) {
  hykkt_config_t c;
  c.gamma = cfg.gamma;
  c.delta_min = cfg.delta_min;
  c.delta_max = cfg.delta_max;
  c.delta2 = cfg.delta2;
  c.cg_tol = cfg.cg_tol;
  c.cg_max_iter = cfg.cg_max_iter;
  c.small_quadratic_threshold = cfg.small_quadratic_threshold;
  c.pivot_floor = cfg.pivot_floor;
  c.ruiz_tol = cfg.ruiz_tol;
  c.ruiz_max_iters = cfg.ruiz_max_iters;
  return c;
}

inline int& device_ordinal() {
  static int d = 0;
  return d;
}

class Handle {
 public:
  Handle() { check(hykkt_create(device_ordinal(), &h_)); }
  ~Handle() { hykkt_destroy(h_); }
  Handle(const Handle&) = delete;
  Handle& operator=(const Handle&) = delete;
  hykkt_t get() const { return h_; }

 private:
  hykkt_t h_ = nullptr;
};

inline bool same_pattern(const CscMatrix& a, const std::vector<index_t>& cp, const std::vector<index_t>& ri,
                         index_t rows) {
  return a.rows() == rows && a.col_ptr() == cp && a.row_idx() == ri;
}

// SymbolicFactor of an analysed handle, in the reference layout.
inline std::shared_ptr<const SymbolicFactor> symbolic_of(hykkt_t h) {
  hykkt_analysis_t info;
  check(hykkt_analysis_info(h, &info));
  auto s = std::make_shared<SymbolicFactor>();
  std::vector<index_t> perm(info.n);
  check(hykkt_get_perm(h, perm.data()));
  s->ordering = Permutation::from_vector(std::move(perm));
  s->parent.resize(info.n);
  s->l_col_ptr.resize(info.n + 1);
  s->l_row_idx.resize(info.nnz_l);
  check(hykkt_chol_get_factor(h, s->l_col_ptr.data(), s->l_row_idx.data(), nullptr, s->parent.data()));
  s->col_counts.resize(info.n);
  for (index_t j = 0; j < info.n; ++j) s->col_counts[j] = s->l_col_ptr[j + 1] - s->l_col_ptr[j];
  return s;
}

// ---- Cholesky-level handles, one per SymbolicFactor ----------------------
// The device plan is built from the symbolic factor's own L pattern (mapped
// back to original indices), so any matrix whose pattern is a subset of the
// symbolic basis factors on it (cholesky.hpp:66-70) and the device L has
// exactly SymbolicFactor::l_row_idx's layout.
struct CholEntry {
  std::weak_ptr<const SymbolicFactor> sym;
  const SymbolicFactor* key = nullptr;
  std::unique_ptr<Handle> h;
  std::vector<index_t> bcp, bri;         // basis pattern (original indices, lower CSC)
  std::vector<index_t> acp, ari;         // last input pattern and its positions in the basis
  std::vector<std::int64_t> apos;
  std::vector<double> resident;          // L values currently on the device
  const CscMatrix* j = nullptr;          // J currently set (identity of the last cg_schur)
  std::vector<index_t> jcp, jri;
  std::vector<double> jv;
};

inline std::vector<std::unique_ptr<CholEntry>>& chol_cache() {
  thread_local std::vector<std::unique_ptr<CholEntry>> cache;
  return cache;
}

inline CholEntry& chol_entry(const std::shared_ptr<const SymbolicFactor>& sym) {
  if (!sym) throw InvalidMatrixError("null symbolic factor");
  auto& cache = chol_cache();
  cache.erase(std::remove_if(cache.begin(), cache.end(), [](const auto& e) { return e->sym.expired(); }),
              cache.end());
  for (auto& e : cache) {
    if (e->key == sym.get()) return *e;
  }
  auto e = std::make_unique<CholEntry>();
  e->sym = sym;
  e->key = sym.get();
  const SymbolicFactor& s = *sym;
  const index_t n = s.size();
  const auto& perm = s.ordering.perm;
  // lower-triangle basis pattern in original indices: L(i, j) -> (perm i, perm j)
  std::vector<std::vector<index_t>> cols(n);
  for (index_t j = 0; j < n; ++j) {
    for (index_t p = s.l_col_ptr[j]; p < s.l_col_ptr[j + 1]; ++p) {
      const index_t a = perm[s.l_row_idx[p]], b = perm[j];
      cols[std::min(a, b)].push_back(std::max(a, b));
    }
  }
  e->bcp.assign(n + 1, 0);
  for (index_t j = 0; j < n; ++j) {
    std::sort(cols[j].begin(), cols[j].end());
    e->bcp[j + 1] = e->bcp[j] + static_cast<index_t>(cols[j].size());
    e->bri.insert(e->bri.end(), cols[j].begin(), cols[j].end());
  }
  e->h = std::make_unique<Handle>();
  check(hykkt_chol_analyze(e->h->get(), n, e->bcp.data(), e->bri.data(), perm.data()));
  cache.push_back(std::move(e));
  return *cache.back();
}

// values of `a` (pattern within the basis) scattered onto the basis pattern
inline std::vector<double> on_basis(CholEntry& e, const CscMatrix& a) {
  const index_t n = static_cast<index_t>(e.bcp.size()) - 1;
  if (!a.is_square() || a.cols() != n) throw InvalidMatrixError("matrix size differs from the symbolic factor");
  if (!same_pattern(a, e.acp, e.ari, n)) {
    e.acp = a.col_ptr();
    e.ari = a.row_idx();
    e.apos.assign(a.nnz(), -1);
    for (index_t j = 0; j < n; ++j) {
      const auto b0 = e.bri.begin() + e.bcp[j], b1 = e.bri.begin() + e.bcp[j + 1];
      for (index_t p = a.col_ptr()[j]; p < a.col_ptr()[j + 1]; ++p) {
        const auto it = std::lower_bound(b0, b1, a.row_idx()[p]);
        if (it == b1 || *it != a.row_idx()[p]) {
          e.acp.clear();
          throw InvalidMatrixError("matrix entry outside the symbolic pattern basis");
        }
        e.apos[p] = it - e.bri.begin();
      }
    }
  }
  std::vector<double> v(e.bri.size(), 0.0);
  for (index_t p = 0; p < a.nnz(); ++p) v[e.apos[p]] += a.values()[p];
  return v;
}

inline std::vector<double> download_l(CholEntry& e) {
  std::vector<double> l(e.key->l_nnz());
  check(hykkt_chol_get_factor(e.h->get(), nullptr, nullptr, l.data(), nullptr));
  e.resident = l;
  return l;
}

inline void make_resident(CholEntry& e, const NumericCholesky& f) {
  if (e.resident != f.l_values()) {
    check(hykkt_chol_set_factor(e.h->get(), f.l_values().data()));
    e.resident = f.l_values();
  }
}

// ---- KKT handles: one per (pattern, ordering) -----------------------------
struct KktEntry {
  bool reduced = false;
  std::unique_ptr<Handle> h;
  std::weak_ptr<const SymbolicFactor> sym;  // the ordering source (null: own ordering)
  const SymbolicFactor* key = nullptr;
  std::shared_ptr<const SymbolicFactor> own;  // symbolic of an own-ordering analysis
  std::vector<index_t> p[6];                   // H/H_tilde, J, J_d patterns
};

inline std::vector<std::unique_ptr<KktEntry>>& kkt_cache() {
  thread_local std::vector<std::unique_ptr<KktEntry>> cache;
  return cache;
}

template <typename Analyze>
KktEntry& kkt_entry(bool reduced, const std::shared_ptr<const SymbolicFactor>& sym,
                    std::initializer_list<const CscMatrix*> mats, bool& created, Analyze analyze) {
  auto& cache = kkt_cache();
  auto matches = [&](const KktEntry& e) {
    // the same ordering source, or the symbolic factor this entry created
    const bool same_sym = (e.key == sym.get() && (!sym || !e.sym.expired())) || (sym && e.own == sym);
    if (e.reduced != reduced || !same_sym) return false;
    int k = 0;
    for (const CscMatrix* m : mats) {
      if (m->col_ptr() != e.p[k] || m->row_idx() != e.p[k + 1]) return false;
      k += 2;
    }
    return true;
  };
  created = false;
  for (auto& e : cache) {
    if (matches(*e)) return *e;
  }
  if (cache.size() >= 8) cache.erase(cache.begin());
  auto e = std::make_unique<KktEntry>();
  e->reduced = reduced;
  e->sym = sym;
  e->key = sym.get();
  int k = 0;
  for (const CscMatrix* m : mats) {
    e->p[k] = m->col_ptr();
    e->p[k + 1] = m->row_idx();
    k += 2;
  }
  e->h = std::make_unique<Handle>();
  analyze(e->h->get(), sym ? sym->ordering.perm.data() : nullptr);
  if (!sym) {
    e->own = symbolic_of(e->h->get());
    created = true;
  }
  cache.push_back(std::move(e));
  return *cache.back();
}

inline void fill_report(const hykkt_report_t& r, SolveReport& out) {
  out.status = static_cast<SolveStatus>(r.status);
  out.delta1_final = r.delta1_final;
  out.delta2_used = r.delta2_used;
  out.cg_iterations = r.cg_iterations;
  out.factorization_attempts = r.factorization_attempts;
  out.ruiz_iterations = r.ruiz_iterations;
  out.density.nnz_op = r.nnz_op;
  out.density.nnz_fac = r.nnz_fac;
  out.density.ratio = r.density_ratio;
  out.density.rho_c = r.rho_c;
  if (out.status == SolveStatus::kFailedDeltaMaxExceeded) {
    out.failure_detail = "factorization failed up to delta1 = " + std::to_string(r.delta1_final) +
                         " at column " + std::to_string(r.failed_column);
  } else if (out.status == SolveStatus::kFailedCgNoConvergence) {
    out.failure_detail = "CG stalled at relative residual " + std::to_string(r.cg_relative_residual);
  }
}

inline void check_validate(const SolverConfig& cfg) { cfg.validate(); }

}  // namespace detail

// Device ordinal used for new handles (default 0).
inline void set_device(int device) { detail::device_ordinal() = device; }

// ---- cholesky.hpp ------------------------------------------------------------
inline FactorizeResult numeric_cholesky(const CscMatrix& a_lower, std::shared_ptr<const SymbolicFactor> symbolic,
                                        double pivot_floor) {
  auto& e = detail::chol_entry(symbolic);
  const std::vector<double> v = detail::on_basis(e, a_lower);
  std::int64_t col = -1;
  double piv = 0.0;
  detail::check(hykkt_chol_factor(e.h->get(), v.data(), std::max(pivot_floor, 0.0), &col, &piv));
  if (col >= 0) {
    e.resident.clear();
    return NotSpdFailure{col, piv};
  }
  return NumericCholesky(symbolic, detail::download_l(e));
}

inline std::vector<double> factor_solve(const NumericCholesky& factor, std::span<const double> b) {
  auto& e = detail::chol_entry(factor.symbolic_ptr());
  if (static_cast<index_t>(b.size()) != factor.symbolic().size()) {
    throw InvalidMatrixError("factor_solve: rhs has length " + std::to_string(b.size()) + ", expected " +
                             std::to_string(factor.symbolic().size()));
  }
  detail::make_resident(e, factor);
  std::vector<double> x(b.size());
  if (!b.empty()) detail::check(hykkt_chol_solve(e.h->get(), b.data(), x.data()));
  return x;
}

// ---- solver.hpp ----------------------------------------------------------------
inline LadderResult factorize_with_ladder(const HGammaSystem& hg, std::shared_ptr<const SymbolicFactor> symbolic,
                                          const SolverConfig& cfg, RegularizationState& state) {
  auto& e = detail::chol_entry(symbolic);
  const std::vector<double> v = detail::on_basis(e, hg.h_gamma);
  const hykkt_config_t c = detail::to_c(cfg);
  double dmin = state.delta_min_current, d1 = 0.0;
  std::int64_t attempts = 0, failed = -1;
  detail::check(hykkt_factor_ladder(e.h->get(), &c, v.data(), &dmin, &attempts, &d1, &failed));
  state.delta_min_current = dmin;
  state.delta1 = d1;
  state.attempts = attempts;
  if (failed >= 0) {
    e.resident.clear();
    return LadderFailure{attempts, d1, failed};
  }
  return NumericCholesky(symbolic, detail::download_l(e));
}

inline CgResult cg_schur(const SchurOperator& op, std::span<const double> rhs, const SolverConfig& cfg,
                         CgTrace* trace = nullptr) {
  if (trace) throw InvalidMatrixError("cg_schur: CgTrace needs every iterate on the host; not on the device path");
  if (!op.factor || !op.j) throw InvalidMatrixError("cg_schur: null operator");
  auto& e = detail::chol_entry(op.factor->symbolic_ptr());
  detail::make_resident(e, *op.factor);
  const CscMatrix& j = *op.j;
  if (static_cast<index_t>(rhs.size()) != j.rows()) throw InvalidMatrixError("cg_schur: rhs length != rows of J");
  if (e.j != op.j || e.jcp != j.col_ptr() || e.jri != j.row_idx() || e.jv != j.values()) {
    detail::check(hykkt_chol_set_j(e.h->get(), j.rows(), j.col_ptr().data(), j.row_idx().data(), j.values().data()));
    e.j = op.j;
    e.jcp = j.col_ptr();
    e.jri = j.row_idx();
    e.jv = j.values();
  }
  const hykkt_config_t c = detail::to_c(cfg);
  CgResult r;
  r.x.assign(rhs.size(), 0.0);
  std::int64_t it = 0;
  std::int32_t conv = 0, sq = 0;
  detail::check(hykkt_cg_schur(e.h->get(), &c, rhs.data(), op.delta2_active, r.x.data(), &it,
                               &r.relative_residual, &conv, &sq));
  r.iterations = it;
  r.converged = conv != 0;
  r.small_quadratic_detected = sq != 0;
  return r;
}

inline HGammaSystem assemble_h_gamma(const Reduced2x2& red, double gamma) {
  if (gamma < 0.0) throw InvalidMatrixError("gamma must be >= 0");
  bool created = false;
  auto& e = detail::kkt_entry(true, nullptr, {&red.h_tilde, &red.j}, created, [&](hykkt_t h, const index_t* perm) {
    detail::check(hykkt_analyze_reduced(h, red.n_x(), red.m_c(), red.h_tilde.col_ptr().data(),
                                        red.h_tilde.row_idx().data(), red.j.col_ptr().data(),
                                        red.j.row_idx().data(), perm));
  });
  hykkt_t h = e.h->get();
  detail::check(hykkt_upload_reduced(h, red.h_tilde.values().data(), red.j.values().data(), red.r_x.data(),
                                     red.r_y.data()));
  hykkt_analysis_t info;
  detail::check(hykkt_analysis_info(h, &info));
  std::vector<index_t> cp(red.n_x() + 1), ri(info.nnz_h_gamma);
  std::vector<double> v(info.nnz_h_gamma);
  HGammaSystem out;
  out.r_hat_x.assign(red.n_x(), 0.0);
  hykkt_config_t c;
  hykkt_config_default(&c);
  c.gamma = gamma;
  detail::check(hykkt_assemble(h, &c, v.data(), out.r_hat_x.data()));
  detail::check(hykkt_hgamma_pattern(h, cp.data(), ri.data()));
  out.h_gamma = CscMatrix(red.n_x(), red.n_x(), std::move(cp), std::move(ri), std::move(v));
  out.gamma_used = gamma;
  return out;
}

inline ReducedSolveResult solve_reduced(const Reduced2x2& red, const SolverConfig& cfg,
                                        std::shared_ptr<const SymbolicFactor> symbolic,
                                        RegularizationState& state) {
  detail::check_validate(cfg);
  bool created = false;
  auto& e = detail::kkt_entry(true, symbolic, {&red.h_tilde, &red.j}, created, [&](hykkt_t h, const index_t* perm) {
    detail::check(hykkt_analyze_reduced(h, red.n_x(), red.m_c(), red.h_tilde.col_ptr().data(),
                                        red.h_tilde.row_idx().data(), red.j.col_ptr().data(),
                                        red.j.row_idx().data(), perm));
  });
  ReducedSolveResult out;
  out.symbolic = symbolic ? symbolic : e.own;
  out.symbolic_created = !symbolic;
  const hykkt_config_t c = detail::to_c(cfg);
  hykkt_report_t r{};
  double dmin = state.delta_min_current;
  out.dx.assign(red.n_x(), 0.0);
  out.dy.assign(red.m_c(), 0.0);
  detail::check(hykkt_solve_reduced(e.h->get(), &c, red.h_tilde.values().data(), red.j.values().data(),
                                    red.r_x.data(), red.r_y.data(), &dmin, HYKKT_FLAG_METRICS, &r,
                                    out.dx.data(), out.dy.data()));
  state.delta_min_current = dmin;
  state.delta1 = r.delta1_final;
  state.attempts = r.factorization_attempts;
  detail::fill_report(r, out.report);
  out.report.ruiz_iterations = 0;
  if (out.ok()) {
    out.report.be_2x2 = r.be_2x2;
    out.report.rr_2x2 = r.rr_2x2;
  } else {
    const double nan = std::numeric_limits<double>::quiet_NaN();
    out.report.be_2x2 = out.report.rr_2x2 = nan;
    out.dx.clear();
    out.dy.clear();
  }
  return out;
}

inline FullSolveResult solve_full(const BlockKkt4x4& sys, const SolverConfig& cfg,
                                  std::shared_ptr<const SymbolicFactor> shared, RegularizationState& state) {
  sys.validate();
  detail::check_validate(cfg);
  bool created = false;
  auto& e = detail::kkt_entry(false, shared, {&sys.h, &sys.j, &sys.j_d}, created, [&](hykkt_t h, const index_t* perm) {
    detail::check(hykkt_analyze(h, sys.n_x(), sys.m_c(), sys.m_d(), sys.h.col_ptr().data(), sys.h.row_idx().data(),
                                sys.j.col_ptr().data(), sys.j.row_idx().data(), sys.j_d.col_ptr().data(),
                                sys.j_d.row_idx().data(), perm));
  });
  FullSolveResult out;
  out.symbolic = shared ? shared : e.own;
  out.symbolic_created = !shared;
  const hykkt_config_t c = detail::to_c(cfg);
  const hykkt_values_t v{sys.h.values().data(), sys.j.values().data(), sys.j_d.values().data(), sys.d_x.data(),
                         sys.d_s.data(), sys.r_tilde_x.data(), sys.r_s.data(), sys.r_y.data(), sys.r_yd.data()};
  FullSolution sol;
  sol.dx.assign(sys.n_x(), 0.0);
  sol.ds.assign(sys.m_d(), 0.0);
  sol.dy.assign(sys.m_c(), 0.0);
  sol.dyd.assign(sys.m_d(), 0.0);
  hykkt_report_t r{};
  double dmin = state.delta_min_current;
  detail::check(hykkt_solve_full(e.h->get(), &c, &v, &dmin, HYKKT_FLAG_METRICS, &r, sol.dx.data(), sol.ds.data(),
                                 sol.dy.data(), sol.dyd.data()));
  state.delta_min_current = dmin;
  state.delta1 = r.delta1_final;
  state.attempts = r.factorization_attempts;
  detail::fill_report(r, out.report);
  out.report.be_4x4 = r.be_4x4;
  out.report.rr_4x4 = r.rr_4x4;
  out.report.be_2x2 = r.be_2x2;
  out.report.rr_2x2 = r.rr_2x2;
  out.report.be_2x2_scaled = r.be_2x2_scaled;
  out.report.rr_2x2_scaled = r.rr_2x2_scaled;
  if (is_success(out.report.status)) out.solution = std::move(sol);
  return out;
}

inline SequenceResult solve_sequence(std::span<const BlockKkt4x4> systems, const SolverConfig& cfg) {
  if (systems.empty()) throw InvalidMatrixError("solve_sequence: empty sequence");
  detail::check_validate(cfg);
  SequenceResult result;
  result.pattern_uniform = true;
  for (std::size_t k = 1; k < systems.size(); ++k) {
    result.pattern_uniform = result.pattern_uniform && systems[k].h.same_pattern_as(systems[0].h) &&
                             systems[k].j.same_pattern_as(systems[0].j) &&
                             systems[k].j_d.same_pattern_as(systems[0].j_d);
  }
  result.reports.resize(systems.size());
  result.solutions.resize(systems.size());
  auto account = [&result](const FullSolveResult& r) {
    if (r.symbolic_created) result.stats.symbolic_analyses++;
    result.stats.factorization_attempts += r.report.factorization_attempts;
    if (r.report.status != SolveStatus::kFailedDeltaMaxExceeded) result.stats.numeric_factorizations++;
  };
  if (cfg.parallel_sequence && result.pattern_uniform) {
    // independent matrices, fresh state each: the batched device path
    // replaces the reference's thread pool (solver.cpp:374-398)
    const BlockKkt4x4& s0 = systems[0];
    detail::Handle h;
    detail::check(hykkt_analyze(h.get(), s0.n_x(), s0.m_c(), s0.m_d(), s0.h.col_ptr().data(), s0.h.row_idx().data(),
                                s0.j.col_ptr().data(), s0.j.row_idx().data(), s0.j_d.col_ptr().data(),
                                s0.j_d.row_idx().data(), nullptr));
    const std::size_t B = systems.size();
    std::vector<double> f[9];
    for (const BlockKkt4x4& s : systems) {
      const std::vector<double>* src[9] = {&s.h.values(), &s.j.values(), &s.j_d.values(), &s.d_x, &s.d_s,
                                           &s.r_tilde_x, &s.r_s, &s.r_y, &s.r_yd};
      for (int i = 0; i < 9; ++i) f[i].insert(f[i].end(), src[i]->begin(), src[i]->end());
    }
    const hykkt_values_t v{f[0].data(), f[1].data(), f[2].data(), f[3].data(), f[4].data(),
                           f[5].data(), f[6].data(), f[7].data(), f[8].data()};
    std::vector<hykkt_report_t> reps(B);
    const index_t nx = s0.n_x(), mc = s0.m_c(), md = s0.m_d();
    std::vector<double> dx(B * nx), ds(B * md), dy(B * mc), dyd(B * md);
    const hykkt_config_t c = detail::to_c(cfg);
    detail::check(hykkt_batch_solve(h.get(), &c, static_cast<std::int64_t>(B), &v, 0, reps.data(), dx.data(),
                                    ds.data(), dy.data(), dyd.data()));
    result.stats.symbolic_analyses = 1;
    for (std::size_t k = 0; k < B; ++k) {
      FullSolveResult r;
      detail::fill_report(reps[k], r.report);
      const double nan = std::numeric_limits<double>::quiet_NaN();
      r.report.be_4x4 = r.report.rr_4x4 = r.report.be_2x2 = r.report.rr_2x2 = nan;
      if (is_success(r.report.status)) {
        FullSolution sol;
        sol.dx.assign(dx.begin() + k * nx, dx.begin() + (k + 1) * nx);
        sol.ds.assign(ds.begin() + k * md, ds.begin() + (k + 1) * md);
        sol.dy.assign(dy.begin() + k * mc, dy.begin() + (k + 1) * mc);
        sol.dyd.assign(dyd.begin() + k * md, dyd.begin() + (k + 1) * md);
        r.solution = std::move(sol);
      }
      result.stats.factorization_attempts += r.report.factorization_attempts;
      if (r.report.status != SolveStatus::kFailedDeltaMaxExceeded) result.stats.numeric_factorizations++;
      result.reports[k] = std::move(r.report);
      result.solutions[k] = std::move(r.solution);
    }
    return result;
  }
  RegularizationState state = RegularizationState::initial(cfg);
  std::shared_ptr<const SymbolicFactor> shared;
  for (std::size_t k = 0; k < systems.size(); ++k) {
    FullSolveResult r = gpu::solve_full(systems[k], cfg, result.pattern_uniform ? shared : nullptr, state);
    if (result.pattern_uniform && !shared) shared = r.symbolic;
    r.report.symbolic_reused = result.pattern_uniform && k > 0;
    account(r);
    result.reports[k] = std::move(r.report);
    result.solutions[k] = std::move(r.solution);
  }
  return result;
}

}  // namespace hkkt::gpu

#endif  // HKKT_GPU_HPP_
