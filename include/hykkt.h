/*
 * hykkt.h — C ABI of the B200-native HyKKT solve path.
 *
 * This is the drop-in boundary for the reference C++ solver API
 * (/root/reference/proj/core/include/hkkt/ *.hpp).  Plain pointers and
 * sizes only; no torch or CUDA types.  Host arrays use the reference's
 * conventions: int64 compressed-column indices (csc_matrix.hpp:25), strictly
 * increasing rows per column, symmetric matrices as their lower triangle,
 * FP64 values.  Every entry point returns an int status and never throws:
 *
 *     0  HYKKT_OK
 *    <0  invalid argument / CUDA / out-of-memory error; text in
 *        hykkt_last_error() (the C++ shim maps these to InvalidMatrixError,
 *        the reference's error type, csc_matrix.hpp:29-33)
 *
 * Normal numerical outcomes (not-SPD pivot, ladder exhaustion, small
 * quadratic form, CG cap) are reported through out-parameters and
 * hykkt_report_t.status, exactly as the reference returns them as values
 * (cholesky.hpp:47-50, solver.hpp:80-86, solver.hpp:124-129).
 *
 * One handle = one device + one stream + one symbolic structure.  A handle
 * is single-threaded; use one handle per host thread.
 */
#ifndef HYKKT_H_
#define HYKKT_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define HYKKT_OK 0
#define HYKKT_ERR_INVALID (-1)
#define HYKKT_ERR_CUDA (-2)
#define HYKKT_ERR_STATE (-3)
#define HYKKT_ERR_DEVICE_TIMEOUT (-4)

typedef struct hykkt_context* hykkt_t;

/* Mirrors hkkt::SolverConfig (solver.hpp:29-50), same names and defaults
 * (hykkt_config_default). parallel_sequence has no meaning on the device
 * path and is absent; batching replaces it (hykkt_batch_*). */
typedef struct {
  double gamma;                     /* 1e4   */
  double delta_min;                 /* 1e-9  */
  double delta_max;                 /* 1e-6  */
  double delta2;                    /* 1e-9  */
  double cg_tol;                    /* 1e-12 */
  int64_t cg_max_iter;              /* 500   */
  double small_quadratic_threshold; /* 1e-12 */
  double pivot_floor;               /* 1e-13, relative to max |diag H_gamma| */
  double ruiz_tol;                  /* 0.01  */
  int64_t ruiz_max_iters;           /* 20    */
} hykkt_config_t;

/* Values of one block-4x4 system (hkkt::BlockKkt4x4, kkt_system.hpp:31-50)
 * on the pattern given to hykkt_analyze.  The plain entry points accept host
 * or device pointers (CUDA unified addressing); the *_device variants
 * require device pointers and reject anything else. */
typedef struct {
  const double* h_val;   /* nnz(H), lower CSC order */
  const double* j_val;   /* nnz(J) */
  const double* jd_val;  /* nnz(J_d) */
  const double* d_x;     /* n_x */
  const double* d_s;     /* m_d */
  const double* r_tilde_x; /* n_x */
  const double* r_s;     /* m_d */
  const double* r_y;     /* m_c */
  const double* r_yd;    /* m_d */
} hykkt_values_t;

/* Mirrors hkkt::SolveReport (solver.hpp:134-150); status uses the
 * SolveStatus numbering (0 solved, 1 solved_delta2, 2 failed_delta_max,
 * 3 failed_cg). BE/RR are NaN for failed solves and when metrics were not
 * requested (HYKKT_FLAG_METRICS). */
typedef struct {
  int32_t status;
  int32_t symbolic_reused;
  double delta1_final;
  double delta2_used;
  int64_t cg_iterations;
  int64_t factorization_attempts;
  double be_4x4, rr_4x4, be_2x2, rr_2x2, be_2x2_scaled, rr_2x2_scaled;
  int64_t ruiz_iterations;
  int64_t nnz_op, nnz_fac;
  double density_ratio, rho_c;
  double cg_relative_residual;
  int64_t failed_column;          /* ladder failure column, else -1 */
} hykkt_report_t;

/* Symbolic statistics of the analysed pattern. */
typedef struct {
  int64_t n;              /* n_x */
  int64_t nnz_h_tilde;    /* stored lower entries of H_tilde */
  int64_t nnz_h_gamma;    /* stored lower entries of H_gamma */
  int64_t nnz_l;          /* SymbolicFactor::l_nnz() */
  int64_t n_supernodes;
  int64_t n_levels;       /* supernode-tree height */
  int64_t etree_height;   /* column elimination-tree height */
  int64_t max_sn_width;
  int64_t max_sn_rows;
  int64_t panel_slots;    /* dense supernodal storage, doubles */
  double factor_flops;    /* sum_j c_j^2 */
  int64_t nnz_j, nnz_jd, m_c, m_d;
  int64_t explicit_zeros; /* panel entries outside L's pattern (relaxed amalgamation) */
} hykkt_analysis_t;

/* Device-side phase timings of the last solve, milliseconds (CUDA events on
 * the handle's stream), filled when HYKKT_FLAG_TIMING was set. */
typedef struct {
  double assemble_ms;   /* reduce + Ruiz + H_gamma assembly */
  double factor_ms;     /* delta1 ladder incl. scatter into panels */
  double solve_w_ms;    /* w = H^-1 r_hat_x and the Schur rhs */
  double cg_ms;         /* CG (incl. a delta2 restart) */
  double solve_dx_ms;   /* dx solve, unscale, recover */
  double total_ms;
  int64_t kernel_launches;
  int64_t cg_kernel_launches;
} hykkt_timing_t;

#define HYKKT_FLAG_METRICS 1  /* compute BE/RR (host, outside the device path) */
#define HYKKT_FLAG_TIMING 2   /* record per-phase CUDA events */

void hykkt_config_default(hykkt_config_t* cfg);
const char* hykkt_last_error(void);

/* --- handle ------------------------------------------------------------ */
int hykkt_create(int device, hykkt_t* out);
void hykkt_destroy(hykkt_t h);

/* --- KKT path: replaces solve_reduced/solve_full (solver.hpp:167-184) ---
 * hykkt_analyze = the per-pattern half of solve_reduced (solver.cpp:230-235:
 * amd_order + symbolic_cholesky of H_gamma's pattern) done once.  perm may
 * be NULL (own minimum-degree ordering) or an ordering of the n_x primal
 * variables in hkkt::Permutation::perm convention (new i holds original
 * perm[i]); passing the reference's amd_order result reproduces its
 * elimination order exactly. */
int hykkt_analyze(hykkt_t h, int64_t n_x, int64_t m_c, int64_t m_d,
                  const int64_t* h_colptr, const int64_t* h_rowidx,
                  const int64_t* j_colptr, const int64_t* j_rowidx,
                  const int64_t* jd_colptr, const int64_t* jd_rowidx,
                  const int64_t* perm);
int hykkt_analysis_info(hykkt_t h, hykkt_analysis_t* out);
/* Host-only analysis (no device needed): the same ordering + symbolic +
 * supernode plan hykkt_analyze builds, returning its statistics and the
 * ordering used (perm_out may be NULL). */
int hykkt_host_analyze(int64_t n_x, int64_t m_c, int64_t m_d,
                       const int64_t* h_colptr, const int64_t* h_rowidx,
                       const int64_t* j_colptr, const int64_t* j_rowidx,
                       const int64_t* jd_colptr, const int64_t* jd_rowidx,
                       const int64_t* perm, int64_t* perm_out,
                       hykkt_analysis_t* out);
int hykkt_get_perm(hykkt_t h, int64_t* perm /* n */);

/* solve_full (solver.cpp:295-328) on one system: values and outputs are
 * host arrays (H2D / D2H inside). *delta_min_inout carries
 * RegularizationState::delta_min_current across a sequence (<= 0 means
 * RegularizationState::initial). Outputs may be NULL. */
int hykkt_solve_full(hykkt_t h, const hykkt_config_t* cfg,
                     const hykkt_values_t* values, double* delta_min_inout,
                     int flags, hykkt_report_t* report, double* dx,
                     double* ds, double* dy, double* dyd);

/* Same, split for device-resident timing: upload once, solve with values
 * already in HBM, download on request. */
int hykkt_upload_values(hykkt_t h, const hykkt_values_t* values);
int hykkt_solve_resident(hykkt_t h, const hykkt_config_t* cfg,
                         double* delta_min_inout, int flags,
                         hykkt_report_t* report);
int hykkt_download_solution(hykkt_t h, double* dx, double* ds, double* dy,
                            double* dyd);
int hykkt_last_timing(hykkt_t h, hykkt_timing_t* out);

/* --- Cholesky-level hooks: replace symbolic_cholesky / numeric_cholesky /
 * factor_solve (cholesky.hpp:41-83) for a general SPD matrix in lower CSC.
 * pivot_floor is absolute here, as in numeric_cholesky.  *failed_column is
 * -1 on success, else the first elimination-order column whose pivot
 * candidate was !(> floor), with that candidate in *failed_pivot
 * (NotSpdFailure, cholesky.hpp:47-50). */
int hykkt_chol_analyze(hykkt_t h, int64_t n, const int64_t* colptr,
                       const int64_t* rowidx, const int64_t* perm);
int hykkt_chol_factor(hykkt_t h, const double* values, double pivot_floor,
                      int64_t* failed_column, double* failed_pivot);
/* Also valid on a factored KKT handle: x = H_delta^-1 b (original order). */
int hykkt_chol_solve(hykkt_t h, const double* b, double* x);
/* Reference-layout factor (SymbolicFactor + NumericCholesky::l_values). */
int hykkt_chol_get_factor(hykkt_t h, int64_t* l_colptr /* n+1 */,
                          int64_t* l_rowidx /* nnz */, double* l_values,
                          int64_t* parent /* n */);

/* --- batched path: B independent systems on one shared pattern ---------
 * (the device replacement for solve_sequence's thread pool,
 * solver.cpp:374-398). Values are [system][entry] host arrays (system b at
 * offset b * nnz). Solutions are written [system][entry]. */
int hykkt_batch_solve(hykkt_t h, const hykkt_config_t* cfg, int64_t batch,
                      const hykkt_values_t* values, int flags,
                      hykkt_report_t* reports /* batch */, double* dx,
                      double* ds, double* dy, double* dyd);
int hykkt_batch_upload(hykkt_t h, int64_t batch, const hykkt_values_t* values);
int hykkt_batch_solve_resident(hykkt_t h, const hykkt_config_t* cfg,
                               int flags, hykkt_report_t* reports);
int hykkt_batch_download(hykkt_t h, double* dx, double* ds, double* dy,
                         double* dyd);

/* --- pipelined batch copies (no reference counterpart: the reference's
 * solve_sequence runs on host memory).  hykkt_batch_upload_async starts the
 * host-to-device copy of a batch (same layout as hykkt_batch_upload; pinned
 * host memory for true overlap) on the handle's copy stream and returns;
 * the next hykkt_batch_solve_resident consumes the oldest pending upload (at
 * most two pending), so the copy of batch k+1 overlaps the solve of batch k.
 * hykkt_batch_download_async starts the device-to-host copy of the last
 * solve's outputs (same layout as hykkt_batch_download) and returns; the
 * buffers are complete after hykkt_batch_sync (or the next synchronous
 * download).  A synchronous hykkt_batch_upload drops pending async uploads. */
int hykkt_batch_upload_async(hykkt_t h, int64_t batch, const hykkt_values_t* values);
int hykkt_batch_download_async(hykkt_t h, double* dx, double* ds, double* dy,
                               double* dyd);
int hykkt_batch_sync(hykkt_t h);

/* --- device-resident values (a GPU-side interior-point
 * method never round-trips values over PCIe).  Same layouts as the host
 * entry points; the copies are device-to-device on the handle's stream.
 * hykkt_solution_device / hykkt_batch_solution_device return the handle's
 * own solution buffers (valid until the next solve or analysis; batch
 * layout [system][entry] per field). */
int hykkt_upload_values_device(hykkt_t h, const hykkt_values_t* values);
int hykkt_batch_upload_device(hykkt_t h, int64_t batch, const hykkt_values_t* values);
int hykkt_solution_device(hykkt_t h, const double** dx, const double** ds,
                          const double** dy, const double** dyd);
int hykkt_batch_solution_device(hykkt_t h, const double** dx, const double** ds,
                                const double** dy, const double** dyd);

/* --- Reduced2x2 path: replaces solve_reduced (solver.hpp:167-170,
 * solver.cpp:222-293) for a caller that holds an (already scaled)
 * hkkt::Reduced2x2 (kkt_system.hpp:56-69): H_tilde lower CSC with its full
 * diagonal, J (m_c x n_x).  No Ruiz scaling, no recovery: dx, dy are the
 * reduced solution; report.be_2x2 / rr_2x2 are error_report_kkt2x2 on the
 * given system (HYKKT_FLAG_METRICS), the 4x4 fields stay NaN. */
int hykkt_analyze_reduced(hykkt_t h, int64_t n_x, int64_t m_c,
                          const int64_t* ht_colptr, const int64_t* ht_rowidx,
                          const int64_t* j_colptr, const int64_t* j_rowidx,
                          const int64_t* perm);
int hykkt_upload_reduced(hykkt_t h, const double* ht_val, const double* j_val,
                         const double* r_x, const double* r_y);
int hykkt_upload_reduced_device(hykkt_t h, const double* ht_val,
                                const double* j_val, const double* r_x,
                                const double* r_y);
int hykkt_solve_reduced(hykkt_t h, const hykkt_config_t* cfg,
                        const double* ht_val, const double* j_val,
                        const double* r_x, const double* r_y,
                        double* delta_min_inout, int flags,
                        hykkt_report_t* report, double* dx, double* dy);

/* --- the split API of solve_reduced, phase by phase ----------------------
 * hykkt_assemble replaces assemble_h_gamma (solver.hpp:75, solver.cpp:66-84)
 * on the uploaded values (reduced handle: of the given Reduced2x2; block-4x4
 * handle: of reduce() + ruiz_scale() of the system).  hg_val receives
 * H_gamma's values on the pattern of hykkt_hgamma_pattern (nnz_h_gamma
 * entries, the reference's add_symmetric_lower union pattern), r_hat_x the
 * n_x right-hand side; either may be NULL (stays on the device). */
int hykkt_assemble(hykkt_t h, const hykkt_config_t* cfg, double* hg_val,
                   double* r_hat_x);
int hykkt_hgamma_pattern(hykkt_t h, int64_t* colptr /* n_x+1 */,
                         int64_t* rowidx /* nnz_h_gamma */);

/* factorize_with_ladder (solver.hpp:92-94, solver.cpp:108-142): delta1 = 0,
 * then RegularizationState::delta_min_current doubling while the pivot-free
 * factorization fails and delta1 <= delta_max / 2; pivot floor =
 * cfg.pivot_floor * max |diag|.  On a KKT handle `values` must be NULL (the
 * H_gamma of the last hykkt_assemble); on a Cholesky-level handle it is the
 * matrix in the pattern given to hykkt_chol_analyze.  *failed_column = -1 on
 * success (the factor stays on the device for hykkt_chol_solve /
 * hykkt_cg_schur), else the LadderFailure column; *attempts and *delta1 are
 * RegularizationState::attempts / delta1. */
int hykkt_factor_ladder(hykkt_t h, const hykkt_config_t* cfg,
                        const double* values, double* delta_min_inout,
                        int64_t* attempts, double* delta1,
                        int64_t* failed_column);

/* Loads a factor given in the reference layout (NumericCholesky::l_values on
 * the SymbolicFactor pattern of hykkt_chol_get_factor) onto a
 * Cholesky-level handle, so factor_solve / cg_schur can run on an L that
 * was produced elsewhere. */
int hykkt_chol_set_factor(hykkt_t h, const double* l_values);
/* The constraint Jacobian J (m_c x n CSC) of SchurOperator (solver.hpp:97-103)
 * for hykkt_cg_schur on a Cholesky-level handle. */
int hykkt_chol_set_j(hykkt_t h, int64_t m_c, const int64_t* j_colptr,
                     const int64_t* j_rowidx, const double* j_val);
/* cg_schur (solver.hpp:121-122, solver.cpp:154-201) on
 * S = J H^-1 J^T + delta2 I with the handle's factor: KKT handles use the
 * scaled J of the last hykkt_assemble, Cholesky-level handles the J of
 * hykkt_chol_set_j.  One persistent kernel, no host round trips; the
 * outcome mirrors CgResult (iterations, relative_residual, converged,
 * small_quadratic_detected). */
int hykkt_cg_schur(hykkt_t h, const hykkt_config_t* cfg, const double* rhs,
                   double delta2, double* x, int64_t* iterations,
                   double* relative_residual, int32_t* converged,
                   int32_t* small_quadratic);

/* Knobs of a handle: "ks_lpt" = 1 (default) / 0 — the batched solve takes
 * systems longest-first by the previous call's CG iteration counts / in
 * natural order (never changes results); "amalg_width" (columns) and
 * "amalg_zeros_pct" — relaxed amalgamation of elimination-tree chains into
 * supernodes of at most that width and share of explicit zeros, applied by
 * the next hykkt_analyze / hykkt_chol_analyze (amalg_width <= 1: fundamental
 * supernodes only; changes only rounding). */
int hykkt_set_option(hykkt_t h, const char* name, int64_t value);

#ifdef __cplusplus
}
#endif

#endif /* HYKKT_H_ */
