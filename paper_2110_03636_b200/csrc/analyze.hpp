// Host-side, once-per-pattern analysis for the B200 HyKKT path.
//
// Replaces the reference's per-pattern work — amd_order (proj/core/src/
// amd.cpp:68), symbolic_cholesky (symbolic.cpp:80-119) and the pattern half
// of reduce / assemble_h_gamma (kkt_system.cpp:66-87, solver.cpp:66-84,
// csc_matrix.cpp:293-393) — with flat index plans that the device kernels
// consume every interior-method iteration without touching the pattern
// again:
//
//   * SupernodalPlan: ordering, etree, L pattern in the reference layout
//     (SymbolicFactor, cholesky.hpp:28-37), fundamental supernodes stored as
//     dense column-major panels, the supernode tree with its level schedule,
//     per-supernode update lists (left-looking factor), forward-solve row
//     lists and the scatter map input-entry -> panel slot.
//   * KktPlan: the union patterns of H_tilde and H_gamma with per-slot
//     product lists in the reference's accumulation order, J in CSC + CSR
//     form and J_d in CSC form.
#pragma once

#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

namespace hykkt {

using idx = std::int64_t;

struct InvalidArgument : std::invalid_argument {
  explicit InvalidArgument(const std::string& w) : std::invalid_argument(w) {}
};

// Compressed-column pattern (values live elsewhere).  Rows strictly
// increasing per column, as the reference requires (csc_matrix.cpp:59-78).
struct CscPattern {
  idx nrows = 0, ncols = 0;
  std::vector<idx> cp{0};
  std::vector<idx> ri;
  idx nnz() const { return static_cast<idx>(ri.size()); }
  void validate(const char* name) const;
};

// Pattern-only symbolic Cholesky of P A P^T, supernodal.
struct SupernodalPlan {
  idx n = 0;
  std::vector<idx> perm, iperm;  // perm[new] = old (Permutation::perm)
  std::vector<idx> parent;       // column etree (permuted indices)
  std::vector<idx> col_counts;   // nnz per L column incl. diagonal
  std::vector<idx> l_cp, l_ri;   // L pattern, reference layout

  // supernodes: columns [sn_first[s], sn_first[s+1])
  idx nsup = 0;
  std::vector<int> sn_first;      // nsup + 1
  std::vector<int> sn_of;         // column -> supernode
  std::vector<int> sn_nrows;      // rows of the panel (incl. diagonal block)
  std::vector<idx> sn_off;        // panel offset (column-major nrows x width)
  std::vector<int> sn_rows_ptr;   // nsup + 1
  std::vector<int> sn_rows;       // row structure, first `width` = own cols
  std::vector<int> sn_parent;     // supernode tree
  std::vector<int> sn_level;      // 0 = leaf
  std::vector<int> child_ptr, child;
  std::vector<int> order;         // topological (level-sorted) order
  int nlevels = 0;
  idx panel_size = 0;

  // left-looking updates: for target s, entries [upd_ptr[s], upd_ptr[s+1])
  // name a descendant d, the offset in d's row list of the first row that
  // falls in s's columns, and how many of d's rows fall in s's columns.
  std::vector<int> upd_ptr, upd_d, upd_off, upd_cnt;

  // forward-solve row lists: strictly-lower entries of L row i that lie in
  // earlier supernodes, as (column, panel slot), ascending column.
  std::vector<int> lrow_ptr, lrow_col, lrow_row;
  std::vector<int> lrow_pos;

  // multifrontal forward solve: supernode s passes an update vector u_s of
  // length nrows - width (rows below its diagonal block) to its parent.
  // u_off[s] = offset of u_s; for child c, ext_map[ext_ptr[c] + q] is the
  // index in u_c of the parent's row-structure position q, or -1.
  std::vector<int> u_off;      // nsup + 1
  std::vector<int> ext_ptr;    // nsup + 1
  std::vector<int> ext_map;
  // flattened gather lists: for position q of supernode s (slot
  // sn_rows_ptr[s] + q) the absolute u indices to sum, in child order.
  std::vector<int> gat_ptr;    // sn_rows_ptr[nsup] + 1
  std::vector<int> gat_idx;
  // child-side form of the same map: relind[u_off[c] + t] = position in the
  // parent's row structure of the child's update-vector entry t.
  std::vector<int> relind;

  // L CSC position (reference layout) -> panel slot
  std::vector<int> l_to_panel;

  // input lower pattern entry (CSC order, original indices) -> panel slot
  std::vector<int> src_to_panel;
  std::vector<int> diag_panel;  // column j (permuted) -> slot of L(j,j)

  // statistics
  idx l_nnz() const { return l_cp.empty() ? 0 : l_cp.back(); }
  double factor_flops = 0.0;  // sum_j c_j^2 (CSparse convention)
  int max_width = 0, max_nrows = 0;
  idx explicit_zeros = 0;     // panel entries outside L's pattern (amalgamation)
};

// Relaxed amalgamation of elimination-tree chains (build_supernodal_plan):
// merged supernodes at most `width` columns wide with at most `zeros` of
// their panel entries explicit zeros.  width <= 1 keeps fundamental
// supernodes only.  Defaults: HYKKT_AMALG_W / HYKKT_AMALG_Z or the B200 sweep.
struct AmalgParams {
  int width;
  double zeros;
  static AmalgParams defaults();
};

// Builds the plan for the lower-triangle pattern `a` (n x n, original
// indices) under `perm` (empty => own minimum-degree ordering).
SupernodalPlan build_supernodal_plan(const CscPattern& a,
                                     std::vector<idx> perm,
                                     AmalgParams amalg = AmalgParams::defaults());

// Own fill-reducing ordering: minimum degree on the explicit elimination
// graph, lowest index first on ties, followed by an etree postorder.
std::vector<idx> minimum_degree_order(const CscPattern& lower);

// ---------------------------------------------------------------------------
// KKT assembly plan.
struct KktPlan {
  idx nx = 0, mc = 0, md = 0;
  CscPattern h, j, jd;  // input patterns as given

  // H_tilde = H + diag(D_x) + J_d^T D_s J_d on the union pattern with a
  // full diagonal (kkt_system.cpp:71-75).  One slot per stored entry,
  // lower CSC order.
  CscPattern ht;
  std::vector<int> ht_hsrc;        // H value index or -1
  std::vector<int> ht_diag;        // 1 if diagonal slot
  std::vector<int> ht_col;         // column of each slot
  std::vector<int> ht_prod_ptr;    // products (k ascending)
  std::vector<int> ht_prod_a;      // J_d value index of (k, col)
  std::vector<int> ht_prod_b;      // J_d value index of (k, row)
  std::vector<int> ht_prod_k;      // k (row of J_d) for D_s[k]

  // H_gamma = H_tilde_scaled + gamma * lower(J^T J) (solver.cpp:73-77)
  CscPattern hg;
  std::vector<int> hg_htsrc;       // H_tilde slot or -1
  std::vector<int> hg_prod_ptr;
  std::vector<int> hg_prod_a;      // J value index of (k, col)
  std::vector<int> hg_prod_b;      // J value index of (k, row)

  // J in CSR form (row-wise), used by J*t.  jcsr_src maps to CSC index.
  std::vector<int> j_rp, j_ci, jcsr_src;
  // J_d in CSR form for J_d * dx (recover)
  std::vector<int> jd_rp, jd_ci, jdcsr_src;
};

KktPlan build_kkt_plan(idx nx, idx mc, idx md, const CscPattern& h,
                       const CscPattern& j, const CscPattern& jd);

}  // namespace hykkt
