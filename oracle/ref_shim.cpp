// ORACLE / TEST INFRASTRUCTURE ONLY — never linked into the product.
//
// extern "C" shim over the UNMODIFIED reference library (hkkt, compiled
// from /root/reference/proj/core/src by oracle/Makefile into
// oracle/_ref/libhkkt_ref.so).  It exists so that tests/, smoke() and the
// cpu_baseline / --impl reference legs of bench.py can drive the
// reference's own public API through ctypes:
//
//   solve_full          proj/core/include/hkkt/solver.hpp:182-184
//   solve_reduced       proj/core/include/hkkt/solver.hpp:167-170
//   solve_sequence      proj/core/include/hkkt/solver.hpp:204-205
//   reduce / ruiz_scale proj/core/include/hkkt/kkt_system.hpp:76,
//                       proj/core/include/hkkt/ruiz.hpp:48
//   assemble_h_gamma    proj/core/include/hkkt/solver.hpp:75
//   factorize_with_ladder  solver.hpp:92-94
//   amd_order / symbolic_cholesky / numeric_cholesky / factor_solve
//                       ordering.hpp:25, cholesky.hpp:41-83
//   generate_systems    generator.hpp:67
//
// Nothing in here re-implements reference arithmetic; it only converts
// plain arrays to the reference's types and back.

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdint>
#include <cstring>
#include <limits>
#include <memory>
#include <string>
#include <thread>
#include <vector>

#include "hkkt/cholesky.hpp"
#include "hkkt/generator.hpp"
#include "hkkt/kkt_system.hpp"
#include "hkkt/metrics.hpp"
#include "hkkt/ordering.hpp"
#include "hkkt/ruiz.hpp"
#include "hkkt/solver.hpp"

using namespace hkkt;

namespace {

thread_local std::string g_err;

struct RefConfig {
  double gamma, delta_min, delta_max, delta2, cg_tol;
  int64_t cg_max_iter;
  double small_quadratic_threshold, pivot_floor, ruiz_tol;
  int64_t ruiz_max_iters;
};

struct RefSystem {
  int64_t n_x, m_c, m_d;
  const int64_t *h_colptr, *h_rowidx;
  const double* h_val;
  const int64_t *j_colptr, *j_rowidx;
  const double* j_val;
  const int64_t *jd_colptr, *jd_rowidx;
  const double* jd_val;
  const double *d_x, *d_s, *r_tilde_x, *r_s, *r_y, *r_yd;
};

struct RefReport {
  int32_t status;
  int32_t symbolic_reused;
  double delta1_final, delta2_used;
  int64_t cg_iterations, factorization_attempts;
  double be_4x4, rr_4x4, be_2x2, rr_2x2, be_2x2_scaled, rr_2x2_scaled;
  int64_t ruiz_iterations, nnz_op, nnz_fac;
  double density_ratio, rho_c;
};

SolverConfig to_cfg(const RefConfig* c) {
  SolverConfig cfg;
  if (!c) return cfg;
  cfg.gamma = c->gamma;
  cfg.delta_min = c->delta_min;
  cfg.delta_max = c->delta_max;
  cfg.delta2 = c->delta2;
  cfg.cg_tol = c->cg_tol;
  cfg.cg_max_iter = c->cg_max_iter;
  cfg.small_quadratic_threshold = c->small_quadratic_threshold;
  cfg.pivot_floor = c->pivot_floor;
  cfg.ruiz_tol = c->ruiz_tol;
  cfg.ruiz_max_iters = c->ruiz_max_iters;
  return cfg;
}

CscMatrix make_csc(int64_t rows, int64_t cols, const int64_t* cp,
                   const int64_t* ri, const double* v) {
  const int64_t nnz = cp[cols];
  std::vector<index_t> colptr(cp, cp + cols + 1);
  std::vector<index_t> rowidx(ri, ri + nnz);
  std::vector<double> vals(nnz, 0.0);
  if (v) std::copy(v, v + nnz, vals.begin());
  return CscMatrix(rows, cols, std::move(colptr), std::move(rowidx),
                   std::move(vals));
}

std::vector<double> vec(const double* p, int64_t n) {
  return p ? std::vector<double>(p, p + n) : std::vector<double>(n, 0.0);
}

BlockKkt4x4 make_sys(const RefSystem* s) {
  BlockKkt4x4 sys;
  sys.h = make_csc(s->n_x, s->n_x, s->h_colptr, s->h_rowidx, s->h_val);
  sys.j = make_csc(s->m_c, s->n_x, s->j_colptr, s->j_rowidx, s->j_val);
  sys.j_d = make_csc(s->m_d, s->n_x, s->jd_colptr, s->jd_rowidx, s->jd_val);
  sys.d_x = vec(s->d_x, s->n_x);
  sys.d_s = vec(s->d_s, s->m_d);
  sys.r_tilde_x = vec(s->r_tilde_x, s->n_x);
  sys.r_s = vec(s->r_s, s->m_d);
  sys.r_y = vec(s->r_y, s->m_c);
  sys.r_yd = vec(s->r_yd, s->m_d);
  return sys;
}

Permutation make_perm(const int64_t* perm, int64_t n) {
  return Permutation::from_vector(std::vector<index_t>(perm, perm + n));
}

// Symbolic factor of the H_gamma pattern of `sys` under `perm` (or the
// reference AMD when perm is null), exactly as solve_reduced builds it
// (solver.cpp:228-232).
std::shared_ptr<const SymbolicFactor> analyze_sys(const BlockKkt4x4& sys,
                                                  const SolverConfig& cfg,
                                                  const int64_t* perm) {
  const Reduced2x2 red = reduce(sys);
  const ScaledReduced sc = ruiz_scale(red, cfg.ruiz_max_iters, cfg.ruiz_tol);
  const HGammaSystem hg = assemble_h_gamma(sc.system, cfg.gamma);
  Permutation p = perm ? make_perm(perm, sys.n_x()) : amd_order(hg.h_gamma);
  return std::make_shared<SymbolicFactor>(
      symbolic_cholesky(hg.h_gamma, std::move(p)));
}

void fill_report(const SolveReport& r, RefReport* out) {
  out->status = static_cast<int32_t>(r.status);
  out->symbolic_reused = r.symbolic_reused ? 1 : 0;
  out->delta1_final = r.delta1_final;
  out->delta2_used = r.delta2_used;
  out->cg_iterations = r.cg_iterations;
  out->factorization_attempts = r.factorization_attempts;
  out->be_4x4 = r.be_4x4;
  out->rr_4x4 = r.rr_4x4;
  out->be_2x2 = r.be_2x2;
  out->rr_2x2 = r.rr_2x2;
  out->be_2x2_scaled = r.be_2x2_scaled;
  out->rr_2x2_scaled = r.rr_2x2_scaled;
  out->ruiz_iterations = r.ruiz_iterations;
  out->nnz_op = r.density.nnz_op;
  out->nnz_fac = r.density.nnz_fac;
  out->density_ratio = r.density.ratio;
  out->rho_c = r.density.rho_c;
}

template <typename F>
int guarded(F&& f) {
  try {
    return f();
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  } catch (...) {
    g_err = "unknown exception";
    return -1;
  }
}

void copy_out(const std::vector<double>& v, double* dst) {
  if (dst && !v.empty()) std::memcpy(dst, v.data(), v.size() * sizeof(double));
}

struct CholHandle {
  std::shared_ptr<const SymbolicFactor> sym;
  std::unique_ptr<NumericCholesky> fac;
};

struct BatchHandle {
  std::vector<BlockKkt4x4> systems;
};

struct GenHandle {
  std::vector<BlockKkt4x4> systems;
};

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

// solve_full (solver.cpp:295-328) on one system.  perm == null lets the
// reference run its own AMD (solve_reduced with a null symbolic);
// otherwise the symbolic factor is built from perm first and passed as
// the shared one.  *dmin_inout carries RegularizationState::delta_min_current
// (<= 0 on input means RegularizationState::initial).
int ref_solve_full(const RefSystem* s, const RefConfig* c, const int64_t* perm,
                   double* dmin_inout, RefReport* rep, double* dx, double* ds,
                   double* dy, double* dyd) {
  return guarded([&] {
    const SolverConfig cfg = to_cfg(c);
    const BlockKkt4x4 sys = make_sys(s);
    std::shared_ptr<const SymbolicFactor> shared;
    if (perm) shared = analyze_sys(sys, cfg, perm);
    RegularizationState st = RegularizationState::initial(cfg);
    if (dmin_inout && *dmin_inout > 0.0) st.delta_min_current = *dmin_inout;
    const FullSolveResult r = solve_full(sys, cfg, shared, st);
    if (dmin_inout) *dmin_inout = st.delta_min_current;
    fill_report(r.report, rep);
    if (r.solution) {
      copy_out(r.solution->dx, dx);
      copy_out(r.solution->ds, ds);
      copy_out(r.solution->dy, dy);
      copy_out(r.solution->dyd, dyd);
    }
    return 0;
  });
}

// amd_order (amd.cpp:68) of the H_gamma pattern solve_reduced would factor.
int ref_hgamma_amd(const RefSystem* s, const RefConfig* c, int64_t* perm_out) {
  return guarded([&] {
    const SolverConfig cfg = to_cfg(c);
    const BlockKkt4x4 sys = make_sys(s);
    const Reduced2x2 red = reduce(sys);
    const ScaledReduced sc = ruiz_scale(red, cfg.ruiz_max_iters, cfg.ruiz_tol);
    const HGammaSystem hg = assemble_h_gamma(sc.system, cfg.gamma);
    const Permutation p = amd_order(hg.h_gamma);
    std::copy(p.perm.begin(), p.perm.end(), perm_out);
    return 0;
  });
}

// reduce -> ruiz_scale -> assemble_h_gamma; returns H_gamma (lower CSC),
// r_hat_x, the Ruiz diagonal and the sweep count.  Call with colptr == null
// first to learn nnz (written to *nnz_out).
int ref_assemble(const RefSystem* s, const RefConfig* c, int64_t* nnz_out,
                 int64_t* colptr, int64_t* rowidx, double* vals, double* rhat,
                 double* dscale, int64_t* ruiz_iters, double* h_tilde_vals,
                 double* j_scaled_vals) {
  return guarded([&] {
    const SolverConfig cfg = to_cfg(c);
    const BlockKkt4x4 sys = make_sys(s);
    const Reduced2x2 red = reduce(sys);
    const ScaledReduced sc = ruiz_scale(red, cfg.ruiz_max_iters, cfg.ruiz_tol);
    const HGammaSystem hg = assemble_h_gamma(sc.system, cfg.gamma);
    *nnz_out = hg.h_gamma.nnz();
    if (!colptr) return 0;
    std::copy(hg.h_gamma.col_ptr().begin(), hg.h_gamma.col_ptr().end(), colptr);
    std::copy(hg.h_gamma.row_idx().begin(), hg.h_gamma.row_idx().end(), rowidx);
    copy_out(hg.h_gamma.values(), vals);
    copy_out(hg.r_hat_x, rhat);
    copy_out(sc.scaling.d_left, dscale);
    *ruiz_iters = sc.scaling.iterations_used;
    if (h_tilde_vals) copy_out(sc.system.h_tilde.values(), h_tilde_vals);
    if (j_scaled_vals) copy_out(sc.system.j.values(), j_scaled_vals);
    return 0;
  });
}

// nnz of the unscaled H_tilde pattern (reduce) and of H_gamma / L.
int ref_pattern_stats(const RefSystem* s, const RefConfig* c,
                      const int64_t* perm, int64_t* out4) {
  return guarded([&] {
    const SolverConfig cfg = to_cfg(c);
    const BlockKkt4x4 sys = make_sys(s);
    const Reduced2x2 red = reduce(sys);
    const ScaledReduced sc = ruiz_scale(red, cfg.ruiz_max_iters, cfg.ruiz_tol);
    const HGammaSystem hg = assemble_h_gamma(sc.system, cfg.gamma);
    Permutation p = perm ? make_perm(perm, sys.n_x()) : amd_order(hg.h_gamma);
    const SymbolicFactor sf = symbolic_cholesky(hg.h_gamma, std::move(p));
    out4[0] = red.h_tilde.nnz();
    out4[1] = hg.h_gamma.nnz();
    out4[2] = sf.l_nnz();
    index_t height = 0;
    std::vector<index_t> depth(sf.size(), 0);
    for (index_t j = sf.size() - 1; j >= 0; --j) {
      depth[j] = sf.parent[j] < 0 ? 1 : depth[sf.parent[j]] + 1;
      height = std::max(height, depth[j]);
    }
    out4[3] = height;
    return 0;
  });
}

// Per-phase CPU time of one system, in solve_full order, with a prebuilt
// shared symbolic factor: assembly = reduce +
// ruiz_scale + assemble_h_gamma; factor = factorize_with_ladder; cg =
// factor_solve(w) + spmv + cg_schur (+ delta2 restart) + factor_solve(dx).
// Median over `reps` runs, seconds.
int ref_time_phases(const RefSystem* s, const RefConfig* c,
                    const int64_t* perm, int reps, double* out3,
                    int64_t* cg_iters) {
  return guarded([&] {
    using clk = std::chrono::steady_clock;
    const SolverConfig cfg = to_cfg(c);
    const BlockKkt4x4 sys = make_sys(s);
    auto shared = analyze_sys(sys, cfg, perm);
    std::vector<double> ta, tf, tc;
    for (int r = 0; r < std::max(1, reps); ++r) {
      const auto t0 = clk::now();
      const Reduced2x2 red = reduce(sys);
      const ScaledReduced sc =
          ruiz_scale(red, cfg.ruiz_max_iters, cfg.ruiz_tol);
      const HGammaSystem hg = assemble_h_gamma(sc.system, cfg.gamma);
      const auto t1 = clk::now();
      RegularizationState st = RegularizationState::initial(cfg);
      LadderResult lad = factorize_with_ladder(hg, shared, cfg, st);
      const auto t2 = clk::now();
      if (!std::holds_alternative<NumericCholesky>(lad)) {
        throw std::runtime_error("ref_time_phases: ladder failed");
      }
      const NumericCholesky& f = std::get<NumericCholesky>(lad);
      const Reduced2x2& rs = sc.system;
      std::vector<double> w = factor_solve(f, hg.r_hat_x);
      std::vector<double> rhs = spmv(rs.j, w);
      for (index_t k = 0; k < rs.m_c(); ++k) rhs[k] -= rs.r_y[k];
      SchurOperator op{&f, &rs.j, 0.0};
      CgResult cg = cg_schur(op, rhs, cfg);
      if (cg.small_quadratic_detected) {
        op.delta2_active = cfg.delta2;
        cg = cg_schur(op, rhs, cfg);
      }
      std::vector<double> rx = spmv(rs.j, cg.x, true);
      for (index_t i = 0; i < rs.n_x(); ++i) rx[i] = hg.r_hat_x[i] - rx[i];
      std::vector<double> dxv = factor_solve(f, rx);
      const auto t3 = clk::now();
      if (cg_iters) *cg_iters = cg.iterations;
      ta.push_back(std::chrono::duration<double>(t1 - t0).count());
      tf.push_back(std::chrono::duration<double>(t2 - t1).count());
      tc.push_back(std::chrono::duration<double>(t3 - t2).count());
    }
    auto med = [](std::vector<double> v) {
      std::sort(v.begin(), v.end());
      return v[v.size() / 2];
    };
    out3[0] = med(ta);
    out3[1] = med(tf);
    out3[2] = med(tc);
    return 0;
  });
}

// ---- batched throughput (the reference's only multi-core mode) ----------
void* ref_batch_new(int64_t count, const RefSystem* systems) {
  try {
    auto* h = new BatchHandle;
    h->systems.reserve(count);
    for (int64_t b = 0; b < count; ++b) h->systems.push_back(make_sys(&systems[b]));
    return h;
  } catch (const std::exception& e) {
    g_err = e.what();
    return nullptr;
  }
}

void ref_batch_free(void* h) { delete static_cast<BatchHandle*>(h); }

// Solves systems [first, first + count) of the batch with `nthreads`
// std::threads, each running solve_full with one shared symbolic factor
// (built outside the timed region) and a fresh RegularizationState —
// BASELINE.md section 3 "Batched throughput".  *seconds = wall time.
int ref_batch_run(void* hv, const RefConfig* c, const int64_t* perm,
                  int64_t first, int64_t count, int nthreads, double* seconds,
                  int64_t* cg_iters_out, int32_t* status_out) {
  return guarded([&] {
    auto* h = static_cast<BatchHandle*>(hv);
    const SolverConfig cfg = to_cfg(c);
    auto shared = analyze_sys(h->systems[0], cfg, perm);
    std::atomic<int64_t> next{first};
    const int64_t end = first + count;
    const auto t0 = std::chrono::steady_clock::now();
    std::vector<std::thread> pool;
    for (int t = 0; t < std::max(1, nthreads); ++t) {
      pool.emplace_back([&] {
        for (;;) {
          const int64_t k = next.fetch_add(1);
          if (k >= end) break;
          RegularizationState st = RegularizationState::initial(cfg);
          const FullSolveResult r = solve_full(h->systems[k], cfg, shared, st);
          if (cg_iters_out) cg_iters_out[k - first] = r.report.cg_iterations;
          if (status_out) status_out[k - first] = static_cast<int32_t>(r.report.status);
        }
      });
    }
    for (auto& th : pool) th.join();
    *seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    return 0;
  });
}

// ---- Cholesky-level known-answer hooks -----------------------------------
// symbolic_cholesky + numeric_cholesky(a_lower, symbolic, floor).  perm ==
// null uses amd_order.  On NotSpdFailure the handle is still returned with
// *fail_col >= 0 and no factor.
void* ref_chol_new(int64_t n, const int64_t* cp, const int64_t* ri,
                   const double* v, const int64_t* perm, double floor,
                   int64_t* fail_col, double* fail_pivot, int64_t* l_nnz) {
  try {
    const CscMatrix a = make_csc(n, n, cp, ri, v);
    Permutation p = perm ? make_perm(perm, n) : amd_order(a);
    auto* h = new CholHandle;
    h->sym = std::make_shared<SymbolicFactor>(symbolic_cholesky(a, std::move(p)));
    *l_nnz = h->sym->l_nnz();
    FactorizeResult r = numeric_cholesky(a, h->sym, floor);
    if (std::holds_alternative<NotSpdFailure>(r)) {
      *fail_col = std::get<NotSpdFailure>(r).column;
      *fail_pivot = std::get<NotSpdFailure>(r).pivot;
    } else {
      *fail_col = -1;
      *fail_pivot = 0.0;
      h->fac = std::make_unique<NumericCholesky>(std::get<NumericCholesky>(std::move(r)));
    }
    return h;
  } catch (const std::exception& e) {
    g_err = e.what();
    return nullptr;
  }
}

int ref_chol_get(void* hv, int64_t* perm, int64_t* parent, int64_t* l_colptr,
                 int64_t* l_rowidx, double* l_val) {
  return guarded([&] {
    auto* h = static_cast<CholHandle*>(hv);
    const SymbolicFactor& s = *h->sym;
    if (perm) std::copy(s.ordering.perm.begin(), s.ordering.perm.end(), perm);
    if (parent) std::copy(s.parent.begin(), s.parent.end(), parent);
    if (l_colptr) std::copy(s.l_col_ptr.begin(), s.l_col_ptr.end(), l_colptr);
    if (l_rowidx) std::copy(s.l_row_idx.begin(), s.l_row_idx.end(), l_rowidx);
    if (l_val && h->fac) copy_out(h->fac->l_values(), l_val);
    return 0;
  });
}

int ref_chol_solve(void* hv, const double* b, double* x) {
  return guarded([&] {
    auto* h = static_cast<CholHandle*>(hv);
    if (!h->fac) throw std::runtime_error("no factor");
    const std::vector<double> out =
        factor_solve(*h->fac, std::span<const double>(b, h->sym->size()));
    copy_out(out, x);
    return 0;
  });
}

void ref_chol_free(void* h) { delete static_cast<CholHandle*>(h); }

// factorize_with_ladder (solver.cpp:108-142) on an explicit lower H_gamma.
int ref_ladder(int64_t n, const int64_t* cp, const int64_t* ri, const double* v,
               const int64_t* perm, const RefConfig* c, double* dmin_inout,
               int32_t* ok, int64_t* attempts, double* delta1,
               int64_t* failed_col) {
  return guarded([&] {
    const SolverConfig cfg = to_cfg(c);
    HGammaSystem hg;
    hg.h_gamma = make_csc(n, n, cp, ri, v);
    hg.r_hat_x.assign(n, 0.0);
    Permutation p = perm ? make_perm(perm, n) : amd_order(hg.h_gamma);
    auto sym = std::make_shared<SymbolicFactor>(symbolic_cholesky(hg.h_gamma, std::move(p)));
    RegularizationState st = RegularizationState::initial(cfg);
    if (dmin_inout && *dmin_inout > 0.0) st.delta_min_current = *dmin_inout;
    const LadderResult r = factorize_with_ladder(hg, sym, cfg, st);
    if (dmin_inout) *dmin_inout = st.delta_min_current;
    *attempts = st.attempts;
    *delta1 = st.delta1;
    if (std::holds_alternative<LadderFailure>(r)) {
      *ok = 0;
      *failed_col = std::get<LadderFailure>(r).failed_column;
    } else {
      *ok = 1;
      *failed_col = -1;
    }
    return 0;
  });
}

// ---- reference generator (generator.cpp:289-406) for KAT instances -------
void* ref_gen_new(int64_t n_x, int64_t m_c, int64_t m_d, int64_t degree,
                  int32_t klass, int64_t length, double drift, uint64_t seed) {
  try {
    GeneratorSpec spec;
    spec.n_x = n_x;
    spec.m_c = m_c;
    spec.m_d = m_d;
    spec.graph_degree = degree;
    spec.indefiniteness = static_cast<IndefinitenessClass>(klass);
    spec.sequence_length = length;
    spec.drift = drift;
    spec.seed = seed;
    auto* h = new GenHandle;
    h->systems = generate_systems(spec);
    return h;
  } catch (const std::exception& e) {
    g_err = e.what();
    return nullptr;
  }
}

void ref_gen_free(void* h) { delete static_cast<GenHandle*>(h); }

int ref_gen_dims(void* hv, int64_t k, int64_t* dims6) {
  return guarded([&] {
    const BlockKkt4x4& s = static_cast<GenHandle*>(hv)->systems.at(k);
    dims6[0] = s.n_x();
    dims6[1] = s.m_c();
    dims6[2] = s.m_d();
    dims6[3] = s.h.nnz();
    dims6[4] = s.j.nnz();
    dims6[5] = s.j_d.nnz();
    return 0;
  });
}

// Writes system k into caller arrays laid out like RefSystem (non-const).
int ref_gen_get(void* hv, int64_t k, int64_t* h_cp, int64_t* h_ri, double* h_v,
                int64_t* j_cp, int64_t* j_ri, double* j_v, int64_t* jd_cp,
                int64_t* jd_ri, double* jd_v, double* d_x, double* d_s,
                double* r_tilde_x, double* r_s, double* r_y, double* r_yd) {
  return guarded([&] {
    const BlockKkt4x4& s = static_cast<GenHandle*>(hv)->systems.at(k);
    auto put = [](const CscMatrix& m, int64_t* cp, int64_t* ri, double* v) {
      std::copy(m.col_ptr().begin(), m.col_ptr().end(), cp);
      std::copy(m.row_idx().begin(), m.row_idx().end(), ri);
      std::copy(m.values().begin(), m.values().end(), v);
    };
    put(s.h, h_cp, h_ri, h_v);
    put(s.j, j_cp, j_ri, j_v);
    put(s.j_d, jd_cp, jd_ri, jd_v);
    copy_out(s.d_x, d_x);
    copy_out(s.d_s, d_s);
    copy_out(s.r_tilde_x, r_tilde_x);
    copy_out(s.r_s, r_s);
    copy_out(s.r_y, r_y);
    copy_out(s.r_yd, r_yd);
    return 0;
  });
}

// cg_schur (solver.cpp:154-201) on S = J H^-1 J^T (+ delta2) for an explicit
// H (lower CSC, factored with perm or AMD) and J; returns x, iterations,
// relative residual and the flag bits (1 converged, 2 small quadratic).
int ref_cg_schur(int64_t n, const int64_t* h_cp, const int64_t* h_ri,
                 const double* h_v, int64_t m, const int64_t* j_cp,
                 const int64_t* j_ri, const double* j_v, const int64_t* perm,
                 const RefConfig* c, double delta2, const double* rhs,
                 double* x, int64_t* iters, double* relres, int32_t* flags) {
  return guarded([&] {
    const SolverConfig cfg = to_cfg(c);
    const CscMatrix h = make_csc(n, n, h_cp, h_ri, h_v);
    const CscMatrix j = make_csc(m, n, j_cp, j_ri, j_v);
    Permutation p = perm ? make_perm(perm, n) : amd_order(h);
    auto sym = std::make_shared<SymbolicFactor>(symbolic_cholesky(h, std::move(p)));
    FactorizeResult fr = numeric_cholesky(h, sym, 0.0);
    if (!std::holds_alternative<NumericCholesky>(fr)) throw std::runtime_error("H not SPD");
    const NumericCholesky& f = std::get<NumericCholesky>(fr);
    const SchurOperator op{&f, &j, delta2};
    const CgResult r = cg_schur(op, std::span<const double>(rhs, m), cfg);
    copy_out(r.x, x);
    *iters = r.iterations;
    *relres = r.relative_residual;
    *flags = (r.converged ? 1 : 0) | (r.small_quadratic_detected ? 2 : 0);
    return 0;
  });
}

// reduce (kkt_system.cpp:66-87): H_tilde (lower CSC) and r_x of one
// system.  Call with null outputs first to get *nnz_out.
int ref_reduce(const RefSystem* s, int64_t* nnz_out, int64_t* ht_cp, int64_t* ht_ri,
               double* ht_v, double* r_x) {
  return guarded([&] {
    const Reduced2x2 red = reduce(make_sys(s));
    *nnz_out = red.h_tilde.nnz();
    if (ht_cp) std::copy(red.h_tilde.col_ptr().begin(), red.h_tilde.col_ptr().end(), ht_cp);
    if (ht_ri) std::copy(red.h_tilde.row_idx().begin(), red.h_tilde.row_idx().end(), ht_ri);
    copy_out(red.h_tilde.values(), ht_v);
    copy_out(red.r_x, r_x);
    return 0;
  });
}

// solve_reduced (solver.cpp:222-293) on an explicit Reduced2x2; perm == null:
// the reference's own amd_order of H_gamma (a null symbolic).
int ref_solve_reduced(int64_t n_x, int64_t m_c, const int64_t* ht_cp, const int64_t* ht_ri,
                      const double* ht_v, const int64_t* j_cp, const int64_t* j_ri,
                      const double* j_v, const double* r_x, const double* r_y,
                      const RefConfig* c, const int64_t* perm, double* dmin_inout,
                      RefReport* rep, double* dx, double* dy) {
  return guarded([&] {
    const SolverConfig cfg = to_cfg(c);
    Reduced2x2 red;
    red.h_tilde = make_csc(n_x, n_x, ht_cp, ht_ri, ht_v);
    red.j = make_csc(m_c, n_x, j_cp, j_ri, j_v);
    red.r_x = vec(r_x, n_x);
    red.r_y = vec(r_y, m_c);
    std::shared_ptr<const SymbolicFactor> sym;
    if (perm) {
      const HGammaSystem hg = assemble_h_gamma(red, cfg.gamma);
      sym = std::make_shared<SymbolicFactor>(symbolic_cholesky(hg.h_gamma, make_perm(perm, n_x)));
    }
    RegularizationState st = RegularizationState::initial(cfg);
    if (dmin_inout && *dmin_inout > 0.0) st.delta_min_current = *dmin_inout;
    const ReducedSolveResult r = solve_reduced(red, cfg, sym, st);
    if (dmin_inout) *dmin_inout = st.delta_min_current;
    fill_report(r.report, rep);
    if (r.ok()) {
      copy_out(r.dx, dx);
      copy_out(r.dy, dy);
    }
    return 0;
  });
}

// solve_sequence (solver.cpp:352-412) on `count` systems: per-matrix
// reports, solutions stacked (dx, ds, dy, dyd) per system at stride N
// (NaN for failed ones) and stats = (symbolic_analyses,
// numeric_factorizations, factorization_attempts, pattern_uniform).
int ref_solve_sequence(int64_t count, const RefSystem* systems, const RefConfig* c,
                       RefReport* reps, double* solutions, int64_t* stats) {
  return guarded([&] {
    const SolverConfig cfg = to_cfg(c);
    std::vector<BlockKkt4x4> sys;
    sys.reserve(count);
    for (int64_t k = 0; k < count; ++k) sys.push_back(make_sys(systems + k));
    const SequenceResult r = solve_sequence(sys, cfg);
    for (int64_t k = 0; k < count; ++k) {
      fill_report(r.reports[k], reps + k);
      const int64_t N = sys[k].total_size();
      double* out = solutions + k * N;
      if (r.solutions[k]) {
        const FullSolution& f = *r.solutions[k];
        copy_out(f.dx, out);
        copy_out(f.ds, out + f.dx.size());
        copy_out(f.dy, out + f.dx.size() + f.ds.size());
        copy_out(f.dyd, out + f.dx.size() + f.ds.size() + f.dy.size());
      } else {
        std::fill(out, out + N, std::numeric_limits<double>::quiet_NaN());
      }
    }
    stats[0] = r.stats.symbolic_analyses;
    stats[1] = r.stats.numeric_factorizations;
    stats[2] = r.stats.factorization_attempts;
    stats[3] = r.pattern_uniform ? 1 : 0;
    return 0;
  });
}

}  // extern "C"
