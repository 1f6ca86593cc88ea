// GPU: the reference's own hybrid-solver known-answer tests, restated through
// the C++ drop-in include/hkkt_gpu.hpp (hkkt::gpu::*, backed by libhykkt.so)
// and checked against the reference implementation (hkkt::*, linked from the
// objects oracle/Makefile compiles out of /root/reference/proj/core/src).
//
// Each case cites the reference test it restates
// (proj/tests/test_hybrid_solver.cpp, test_sparse_core.cpp).  Built by
// tests/cpp/Makefile into tests/cpp/_build/test_gpu_shim (git-ignored,
// travels to the GPU box); run by tests/test_gpu_shim.py.
#include <cmath>
#include <cstdio>
#include <functional>
#include <string>
#include <vector>

#include "hkkt/generator.hpp"
#include "hkkt/metrics.hpp"
#include "hkkt/ordering.hpp"
#include "hkkt/solver.hpp"
#include "hkkt_gpu.hpp"
#include "test_support.hpp"

using namespace hkkt;
using namespace hkkt::testing;

namespace {

int g_fail = 0, g_checks = 0;
std::string g_case;

#define CHECK(cond)                                                                 \
  do {                                                                              \
    ++g_checks;                                                                     \
    if (!(cond)) {                                                                  \
      ++g_fail;                                                                     \
      std::fprintf(stderr, "FAIL [%s] %s:%d: %s\n", g_case.c_str(), __FILE__, __LINE__, #cond); \
    }                                                                               \
  } while (0)

struct Require {};
#define REQUIRE(cond)          \
  do {                         \
    CHECK(cond);               \
    if (!(cond)) throw Require{}; \
  } while (0)

std::vector<std::pair<std::string, std::function<void()>>>& cases() {
  static std::vector<std::pair<std::string, std::function<void()>>> c;
  return c;
}
struct Reg {
  Reg(const char* n, std::function<void()> f) { cases().emplace_back(n, std::move(f)); }
};
#define CAT2(a, b) a##b
#define CAT(a, b) CAT2(a, b)
#define CASE(name) static void CAT(case_, __LINE__)(); static Reg CAT(reg_, __LINE__)(name, CAT(case_, __LINE__)); static void CAT(case_, __LINE__)()

bool approx(double a, double b, double eps = 1e-12) { return std::fabs(a - b) <= eps * (1.0 + std::max(std::fabs(a), std::fabs(b))); }

double rel_diff(std::span<const double> a, std::span<const double> b) {
  double num = 0.0, den = 0.0;
  for (std::size_t i = 0; i < a.size(); ++i) {
    num += (a[i] - b[i]) * (a[i] - b[i]);
    den += b[i] * b[i];
  }
  return den > 0.0 ? std::sqrt(num / den) : std::sqrt(num);
}

HGammaSystem diagonal_h_gamma(index_t n, double eps) {
  std::vector<Triplet> entries;
  for (index_t i = 0; i < n; ++i) entries.push_back({i, i, i == n - 1 ? -eps : 1.0 + 0.1 * double(i)});
  HGammaSystem hg;
  hg.h_gamma = CscMatrix::from_triplets(n, n, entries);
  hg.r_hat_x.assign(n, 1.0);
  return hg;
}

std::shared_ptr<const SymbolicFactor> analyze(const CscMatrix& a) {
  return std::make_shared<SymbolicFactor>(symbolic_cholesky(a, amd_order(a)));
}

BlockKkt4x4 well_posed_system(index_t nx, index_t mc, index_t md, std::uint64_t seed,
                              IndefinitenessClass k = IndefinitenessClass::kSpdOnNullspace, index_t len = 1) {
  GeneratorSpec spec;
  spec.n_x = nx;
  spec.m_c = mc;
  spec.m_d = md;
  spec.indefiniteness = k;
  spec.sequence_length = len;
  spec.seed = seed;
  return generate_systems(spec)[0];
}

std::vector<double> stacked(const FullSolution& s) {
  std::vector<double> v(s.dx);
  v.insert(v.end(), s.ds.begin(), s.ds.end());
  v.insert(v.end(), s.dy.begin(), s.dy.end());
  v.insert(v.end(), s.dyd.begin(), s.dyd.end());
  return v;
}

// ---- cholesky.hpp (test_sparse_core.cpp:248-272, :308-386) -------------------
CASE("numeric_cholesky diag(4, 9) -> L = (2, 3)") {
  const CscMatrix a = CscMatrix::from_triplets(2, 2, std::vector<Triplet>{{0, 0, 4.0}, {1, 1, 9.0}});
  auto sym = analyze(a);
  const FactorizeResult r = gpu::numeric_cholesky(a, sym, 0.0);
  REQUIRE(std::holds_alternative<NumericCholesky>(r));
  const auto& l = std::get<NumericCholesky>(r).l_values();
  CHECK(l.size() == 2);
  CHECK((l[0] == 2.0 && l[1] == 3.0) || (l[0] == 3.0 && l[1] == 2.0));
}

CASE("numeric_cholesky [[1,2],[2,1]] -> NotSpdFailure{1, -3}") {
  const CscMatrix a = CscMatrix::from_triplets(2, 2, std::vector<Triplet>{{0, 0, 1.0}, {1, 0, 2.0}, {1, 1, 1.0}});
  auto sym = std::make_shared<SymbolicFactor>(symbolic_cholesky(a, Permutation::identity(2)));
  const FactorizeResult r = gpu::numeric_cholesky(a, sym, 0.0);
  REQUIRE(std::holds_alternative<NotSpdFailure>(r));
  CHECK(std::get<NotSpdFailure>(r).column == 1);
  CHECK(approx(std::get<NotSpdFailure>(r).pivot, -3.0));
}

CASE("numeric_cholesky / factor_solve match the reference") {
  TestRng rng(3);
  const CscMatrix a = random_spd_lower(400, 3, 0.5, rng);
  auto sym = analyze(a);
  const auto want = std::get<NumericCholesky>(hkkt::numeric_cholesky(a, sym, 0.0));
  const auto got = std::get<NumericCholesky>(gpu::numeric_cholesky(a, sym, 0.0));
  CHECK(rel_diff(got.l_values(), want.l_values()) <= 1e-13);
  std::vector<double> b(400);
  for (auto& v : b) v = rng.uniform(-1.0, 1.0);
  CHECK(rel_diff(gpu::factor_solve(got, b), hkkt::factor_solve(want, b)) <= 1e-12);
  // a factor produced by the reference, solved on the device
  CHECK(rel_diff(gpu::factor_solve(want, b), hkkt::factor_solve(want, b)) <= 1e-12);
}

// ---- factorize_with_ladder (test_hybrid_solver.cpp:157-212, :498-509) ----------
CASE("ladder finds the minimal level within a factor of two") {
  SolverConfig cfg;
  for (int j = 0; j <= 6; ++j) {
    const double eps = 1.5 * cfg.delta_min * std::pow(2.0, j);
    const HGammaSystem hg = diagonal_h_gamma(12, eps);
    auto sym = analyze(hg.h_gamma);
    RegularizationState state = RegularizationState::initial(cfg);
    const LadderResult r = gpu::factorize_with_ladder(hg, sym, cfg, state);
    REQUIRE(std::holds_alternative<NumericCholesky>(r));
    CHECK(approx(state.delta1, cfg.delta_min * std::pow(2.0, j + 1)));
    CHECK(state.attempts == j + 3);
    const CscMatrix h_half = add_diagonal_shift(hg.h_gamma, state.delta1 / 2.0);
    CHECK(std::holds_alternative<NotSpdFailure>(gpu::numeric_cholesky(h_half, sym, cfg.pivot_floor * 1.0)));
  }
}

CASE("ladder failure exhausts within the attempt bound") {
  SolverConfig cfg;
  const HGammaSystem hg = diagonal_h_gamma(10, 1.0);
  RegularizationState state = RegularizationState::initial(cfg);
  const LadderResult r = gpu::factorize_with_ladder(hg, analyze(hg.h_gamma), cfg, state);
  REQUIRE(std::holds_alternative<LadderFailure>(r));
  const index_t bound = static_cast<index_t>(std::ceil(std::log2(cfg.delta_max / cfg.delta_min))) + 1;
  CHECK(std::get<LadderFailure>(r).attempts == bound);
}

CASE("delta_min_current carries across matrices") {
  SolverConfig cfg;
  const HGammaSystem hg = diagonal_h_gamma(12, 1.5 * cfg.delta_min * 16.0);
  auto sym = analyze(hg.h_gamma);
  RegularizationState state = RegularizationState::initial(cfg);
  REQUIRE(std::holds_alternative<NumericCholesky>(gpu::factorize_with_ladder(hg, sym, cfg, state)));
  const double level = state.delta1;
  CHECK(approx(level, 32.0 * cfg.delta_min));
  REQUIRE(std::holds_alternative<NumericCholesky>(gpu::factorize_with_ladder(hg, sym, cfg, state)));
  CHECK(state.attempts == 2);
  CHECK(approx(state.delta1, level));
}

CASE("a pivot just below the floor is rescued at the first rung") {
  SolverConfig cfg;
  const HGammaSystem hg = diagonal_h_gamma(8, 2e-13);
  RegularizationState state = RegularizationState::initial(cfg);
  REQUIRE(std::holds_alternative<NumericCholesky>(gpu::factorize_with_ladder(hg, analyze(hg.h_gamma), cfg, state)));
  CHECK(state.delta1 == cfg.delta_min);
  CHECK(state.attempts == 2);
}

// ---- cg_schur (test_hybrid_solver.cpp:214-244) ------------------------------------
CASE("cg_schur on trivial right-hand sides") {
  TestRng rng(5);
  const CscMatrix h = random_spd_lower(10, 2, 0.5, rng);
  auto sym = analyze(h);
  const auto f = std::get<NumericCholesky>(gpu::numeric_cholesky(h, sym, 0.0));
  const CscMatrix j = random_sparse(4, 10, 3, rng);
  const SchurOperator op{&f, &j, 0.0};
  const CgResult r = gpu::cg_schur(op, std::vector<double>(4, 0.0), SolverConfig{});
  CHECK(r.converged);
  CHECK(r.iterations == 0);
  CHECK(r.x == std::vector<double>(4, 0.0));
}

CASE("cg_schur converges in one iteration when S is the identity") {
  const index_t nx = 6, mc = 3;
  std::vector<Triplet> eye, jrows;
  for (index_t i = 0; i < nx; ++i) eye.push_back({i, i, 1.0});
  for (index_t r = 0; r < mc; ++r) jrows.push_back({r, 2 * r, 1.0});
  const CscMatrix h = CscMatrix::from_triplets(nx, nx, eye);
  const auto f = std::get<NumericCholesky>(gpu::numeric_cholesky(h, analyze(h), 0.0));
  const CscMatrix j = CscMatrix::from_triplets(mc, nx, jrows);
  const SchurOperator op{&f, &j, 0.0};
  const CgResult r = gpu::cg_schur(op, std::vector<double>{1.0, -2.0, 0.5}, SolverConfig{});
  CHECK(r.converged);
  CHECK(r.iterations == 1);
}

CASE("cg_schur matches the reference on a random operator") {
  TestRng rng(29);
  const CscMatrix h = random_spd_lower(300, 3, 0.5, rng);
  auto sym = analyze(h);
  const auto f = std::get<NumericCholesky>(hkkt::numeric_cholesky(h, sym, 0.0));
  const CscMatrix j = random_sparse(80, 300, 3, rng);
  std::vector<double> rhs(80);
  for (auto& v : rhs) v = rng.uniform(-1.0, 1.0);
  const SchurOperator op{&f, &j, 0.0};
  const CgResult want = hkkt::cg_schur(op, rhs, SolverConfig{});
  const CgResult got = gpu::cg_schur(op, rhs, SolverConfig{});
  CHECK(got.converged == want.converged);
  CHECK(std::abs(got.iterations - want.iterations) <= 1);
  CHECK(rel_diff(got.x, want.x) <= 1e-10);
}

// ---- assemble_h_gamma / solve_reduced (test_hybrid_solver.cpp:71-138, :246-315) ----
CASE("assemble_h_gamma matches the reference") {
  const BlockKkt4x4 sys = well_posed_system(240, 60, 50, 23);
  const ScaledReduced sc = ruiz_scale(reduce(sys), 20, 0.01);
  for (double gamma : {0.0, 1e4, 1e8}) {
    const HGammaSystem want = hkkt::assemble_h_gamma(sc.system, gamma);
    const HGammaSystem got = gpu::assemble_h_gamma(sc.system, gamma);
    CHECK(got.h_gamma.col_ptr() == want.h_gamma.col_ptr());
    CHECK(got.h_gamma.row_idx() == want.h_gamma.row_idx());
    CHECK(rel_diff(got.h_gamma.values(), want.h_gamma.values()) <= 1e-15);
    CHECK(rel_diff(got.r_hat_x, want.r_hat_x) <= 1e-15);
  }
}

CASE("solve_reduced matches a dense block solve") {
  TestRng rng(13);
  const index_t n = 14;
  Reduced2x2 red;
  red.h_tilde = random_spd_lower(n, 3, 0.5, rng);
  std::vector<Triplet> jt;
  for (index_t i = 0; i < n; ++i) jt.push_back({i, i, 1.0 + 0.1 * i});
  for (index_t i = 0; i + 1 < n; ++i) jt.push_back({i, i + 1, 0.3});
  red.j = CscMatrix::from_triplets(n, n, jt);
  red.r_x.resize(n);
  red.r_y.resize(n);
  for (auto& v : red.r_x) v = rng.uniform(-1.0, 1.0);
  for (auto& v : red.r_y) v = rng.uniform(-1.0, 1.0);
  SolverConfig cfg;
  RegularizationState state = RegularizationState::initial(cfg);
  const ReducedSolveResult r = gpu::solve_reduced(red, cfg, nullptr, state);
  REQUIRE(r.ok());
  CHECK(r.report.status == SolveStatus::kSolved);
  CHECK(r.report.delta1_final == 0.0);
  CHECK(r.symbolic_created && r.symbolic);
  const DenseMatrix k2 = assemble_kkt2x2_dense(red);
  std::vector<double> rhs(red.r_x);
  rhs.insert(rhs.end(), red.r_y.begin(), red.r_y.end());
  const std::vector<double> z = dense_solve(k2, rhs);
  std::vector<double> got(r.dx);
  got.insert(got.end(), r.dy.begin(), r.dy.end());
  CHECK(rel_diff(got, z) <= 1e-9);
}

CASE("rank-deficient J: consistent solves without delta2, inconsistent restarts") {
  for (int inconsistent = 0; inconsistent < 2; ++inconsistent) {
    const BlockKkt4x4 sys = well_posed_system(
        30, 8, 6, inconsistent ? 8 : 7,
        inconsistent ? IndefinitenessClass::kInconsistentRankDeficient : IndefinitenessClass::kRankDeficientJ);
    const Reduced2x2 red = reduce(sys);
    SolverConfig cfg;
    RegularizationState s1 = RegularizationState::initial(cfg), s2 = s1;
    const ReducedSolveResult want = hkkt::solve_reduced(red, cfg, nullptr, s1);
    // the reference's symbolic factor (its AMD), shared with the device
    const ReducedSolveResult r = gpu::solve_reduced(red, cfg, want.symbolic, s2);
    REQUIRE(r.ok());
    CHECK(r.report.status == (inconsistent ? SolveStatus::kSolvedWithDelta2 : SolveStatus::kSolved));
    CHECK(r.report.status == want.report.status);
    CHECK(r.report.delta2_used == want.report.delta2_used);
    CHECK(std::abs(r.report.cg_iterations - want.report.cg_iterations) <= 1);
    // (dx, dy) stacked: with the delta2 restart the solution of the singular
    // Schur system is fixed by the regularization, so compare the pair
    std::vector<double> a(r.dx), b(want.dx);
    a.insert(a.end(), r.dy.begin(), r.dy.end());
    b.insert(b.end(), want.dy.begin(), want.dy.end());
    const double err = rel_diff(a, b);
    std::printf("      rank-deficient (%s): stacked (dx, dy) rel err %.2e\n", inconsistent ? "inconsistent" : "consistent", err);
    CHECK(err <= 1e-8);
  }
}

// ---- solve_full / solve_sequence (test_hybrid_solver.cpp:317-342, solver.cpp:352-412) ----
CASE("solve_full degenerates to one SPD solve without constraints") {
  TestRng rng(17);
  BlockKkt4x4 sys;
  sys.h = random_spd_lower(18, 3, 0.5, rng);
  sys.j = CscMatrix(0, 18);
  sys.j_d = CscMatrix(0, 18);
  sys.d_x.assign(18, 0.3);
  sys.r_tilde_x.resize(18);
  for (auto& v : sys.r_tilde_x) v = rng.uniform(-1.0, 1.0);
  SolverConfig cfg;
  RegularizationState state = RegularizationState::initial(cfg);
  const FullSolveResult r = gpu::solve_full(sys, cfg, nullptr, state);
  REQUIRE(r.solution.has_value());
  CHECK(r.report.cg_iterations == 0);
  CHECK(r.report.be_4x4 <= 1e-12);
}

CASE("solve_full reaches reference accuracy on a synthetic system") {
  const BlockKkt4x4 sys = well_posed_system(240, 60, 50, 23);
  SolverConfig cfg;
  RegularizationState s1 = RegularizationState::initial(cfg), s2 = s1;
  const FullSolveResult r = gpu::solve_full(sys, cfg, nullptr, s1);
  REQUIRE(r.solution.has_value());
  CHECK(r.report.be_4x4 <= 1e-8);
  // and against the reference on the reference's ordering
  const FullSolveResult want = hkkt::solve_full(sys, cfg, nullptr, s2);
  RegularizationState s3 = RegularizationState::initial(cfg);
  const FullSolveResult same = gpu::solve_full(sys, cfg, want.symbolic, s3);
  REQUIRE(same.solution.has_value());
  CHECK(rel_diff(stacked(*same.solution), stacked(*want.solution)) <= 1e-8);
  CHECK(same.report.delta1_final == want.report.delta1_final);
  CHECK(std::abs(same.report.cg_iterations - want.report.cg_iterations) <= 1);
  CHECK(!same.symbolic_created);
}

CASE("solve_sequence matches the reference (symbolic reuse, delta_min carry)") {
  GeneratorSpec spec;
  spec.n_x = 60;
  spec.m_c = 15;
  spec.m_d = 12;
  spec.indefiniteness = IndefinitenessClass::kIndefinite;
  spec.sequence_length = 4;
  spec.seed = 44;
  const std::vector<BlockKkt4x4> seq = generate_systems(spec);
  SolverConfig cfg;
  const SequenceResult want = hkkt::solve_sequence(seq, cfg);
  const SequenceResult got = gpu::solve_sequence(seq, cfg);
  CHECK(got.pattern_uniform == want.pattern_uniform);
  CHECK(got.stats.symbolic_analyses == want.stats.symbolic_analyses);
  CHECK(got.stats.numeric_factorizations == want.stats.numeric_factorizations);
  CHECK(got.stats.factorization_attempts == want.stats.factorization_attempts);
  for (std::size_t k = 0; k < seq.size(); ++k) {
    CHECK(got.reports[k].status == want.reports[k].status);
    CHECK(got.reports[k].factorization_attempts == want.reports[k].factorization_attempts);
    CHECK(got.reports[k].delta1_final == want.reports[k].delta1_final);
    CHECK(got.reports[k].symbolic_reused == want.reports[k].symbolic_reused);
  }
  // parallel mode: the batched device path, fresh state per matrix
  SolverConfig pc = cfg;
  pc.parallel_sequence = true;
  const SequenceResult pw = hkkt::solve_sequence(seq, pc);
  const SequenceResult pg = gpu::solve_sequence(seq, pc);
  for (std::size_t k = 0; k < seq.size(); ++k) {
    CHECK(pg.reports[k].status == pw.reports[k].status);
    CHECK(pg.reports[k].factorization_attempts == pw.reports[k].factorization_attempts);
  }
}

CASE("errors: out-of-pattern entries and CgTrace raise InvalidMatrixError") {
  const CscMatrix a = CscMatrix::from_triplets(3, 3, std::vector<Triplet>{{0, 0, 4.0}, {1, 1, 4.0}, {2, 2, 4.0}});
  auto sym = std::make_shared<SymbolicFactor>(symbolic_cholesky(a, Permutation::identity(3)));
  const CscMatrix b = CscMatrix::from_triplets(3, 3, std::vector<Triplet>{{0, 0, 4.0}, {2, 0, 1.0}, {1, 1, 4.0}, {2, 2, 4.0}});
  bool threw = false;
  try {
    gpu::numeric_cholesky(b, sym, 0.0);
  } catch (const InvalidMatrixError&) {
    threw = true;
  }
  CHECK(threw);
}

}  // namespace

int main() {
  int failed_cases = 0;
  for (auto& [name, fn] : cases()) {
    g_case = name;
    const int before = g_fail;
    try {
      fn();
    } catch (const Require&) {
    } catch (const std::exception& e) {
      ++g_fail;
      std::fprintf(stderr, "FAIL [%s] exception: %s\n", name.c_str(), e.what());
    }
    const bool ok = g_fail == before;
    failed_cases += ok ? 0 : 1;
    std::printf("%s  %s\n", ok ? "ok  " : "FAIL", name.c_str());
  }
  std::printf("%zu cases, %d checks, %d failed checks, %d failed cases\n", cases().size(), g_checks, g_fail,
              failed_cases);
  return failed_cases == 0 ? 0 : 1;
}
