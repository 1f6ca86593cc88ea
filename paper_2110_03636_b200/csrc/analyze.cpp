// Once-per-pattern host analysis; see analyze.hpp for the contract.
#include "analyze.hpp"

#include <algorithm>
#include <cstdlib>
#include <numeric>
#include <queue>
#include <utility>

namespace hykkt {

namespace {

[[noreturn]] void fail(const std::string& w) { throw InvalidArgument(w); }

// Upper-triangle adjacency of P A P^T: for every permuted column c the rows
// r < c with (r, c) in the symmetric pattern.  Feeds the etree and the row
// subtree walk (the reference builds the same set in symbolic.cpp:26-40).
void permuted_upper(const CscPattern& a, const std::vector<idx>& iperm,
                    std::vector<idx>& up_cp, std::vector<idx>& up_ri) {
  const idx n = a.ncols;
  up_cp.assign(n + 1, 0);
  for (idx j = 0; j < n; ++j) {
    for (idx p = a.cp[j]; p < a.cp[j + 1]; ++p) {
      const idx r = iperm[a.ri[p]], c = iperm[j];
      if (r != c) up_cp[std::max(r, c) + 1]++;
    }
  }
  std::partial_sum(up_cp.begin(), up_cp.end(), up_cp.begin());
  up_ri.assign(up_cp[n], 0);
  std::vector<idx> fill(up_cp.begin(), up_cp.end() - 1);
  for (idx j = 0; j < n; ++j) {
    for (idx p = a.cp[j]; p < a.cp[j + 1]; ++p) {
      const idx r = iperm[a.ri[p]], c = iperm[j];
      if (r != c) up_ri[fill[std::max(r, c)]++] = std::min(r, c);
    }
  }
}

// Liu's elimination tree with path compression over the upper pattern.
std::vector<idx> etree_of(idx n, const std::vector<idx>& up_cp,
                          const std::vector<idx>& up_ri) {
  std::vector<idx> parent(n, -1), anc(n, -1);
  for (idx k = 0; k < n; ++k) {
    for (idx p = up_cp[k]; p < up_cp[k + 1]; ++p) {
      idx i = up_ri[p];
      while (i != -1 && i < k) {
        const idx nxt = anc[i];
        anc[i] = k;
        if (nxt == -1) parent[i] = k;
        i = nxt;
      }
    }
  }
  return parent;
}

// Depth-first postorder of a forest given by parent[], children visited in
// ascending index order.
std::vector<idx> postorder_of(const std::vector<idx>& parent) {
  const idx n = static_cast<idx>(parent.size());
  std::vector<idx> head(n, -1), next(n, -1), post;
  post.reserve(n);
  for (idx j = n - 1; j >= 0; --j) {
    if (parent[j] >= 0) {
      next[j] = head[parent[j]];
      head[parent[j]] = j;
    }
  }
  std::vector<idx> stack;
  for (idx root = 0; root < n; ++root) {
    if (parent[root] >= 0) continue;
    stack.push_back(root);
    while (!stack.empty()) {
      const idx v = stack.back();
      const idx c = head[v];
      if (c == -1) {
        stack.pop_back();
        post.push_back(v);
      } else {
        head[v] = next[c];
        stack.push_back(c);
      }
    }
  }
  return post;
}

}  // namespace

void CscPattern::validate(const char* name) const {
  const std::string nm(name);
  if (nrows < 0 || ncols < 0) fail(nm + ": negative dimension");
  if (static_cast<idx>(cp.size()) != ncols + 1) fail(nm + ": col_ptr length must be ncols+1");
  if (cp.front() != 0 || cp.back() != nnz()) fail(nm + ": col_ptr must start at 0 and end at nnz");
  for (idx j = 0; j < ncols; ++j) {
    if (cp[j] > cp[j + 1]) fail(nm + ": col_ptr not nondecreasing at column " + std::to_string(j));
    idx prev = -1;
    for (idx p = cp[j]; p < cp[j + 1]; ++p) {
      const idx i = ri[p];
      if (i < 0 || i >= nrows) fail(nm + ": row index out of range in column " + std::to_string(j));
      if (i <= prev) fail(nm + ": row indices not strictly increasing in column " + std::to_string(j));
      prev = i;
    }
  }
}

std::vector<idx> minimum_degree_order(const CscPattern& lower) {
  const idx n = lower.ncols;
  std::vector<std::vector<int>> adj(n);
  for (idx j = 0; j < n; ++j) {
    for (idx p = lower.cp[j]; p < lower.cp[j + 1]; ++p) {
      const idx i = lower.ri[p];
      if (i == j) continue;
      adj[i].push_back(static_cast<int>(j));
      adj[j].push_back(static_cast<int>(i));
    }
  }
  for (auto& a : adj) {
    std::sort(a.begin(), a.end());
    a.erase(std::unique(a.begin(), a.end()), a.end());
  }
  using Key = std::pair<idx, idx>;  // (degree, index): lowest index on ties
  std::priority_queue<Key, std::vector<Key>, std::greater<Key>> heap;
  std::vector<idx> degree(n);
  for (idx v = 0; v < n; ++v) {
    degree[v] = static_cast<idx>(adj[v].size());
    heap.push({degree[v], v});
  }
  std::vector<char> gone(n, 0);
  std::vector<idx> order;
  order.reserve(n);
  std::vector<int> merged;
  while (!heap.empty()) {
    const auto [d, v] = heap.top();
    heap.pop();
    if (gone[v] || d != degree[v]) continue;
    gone[v] = 1;
    order.push_back(v);
    const std::vector<int> nb = std::move(adj[v]);
    adj[v].clear();
    adj[v].shrink_to_fit();
    // The eliminated node's neighbours become a clique.
    for (int u : nb) {
      std::vector<int>& au = adj[u];
      merged.clear();
      merged.reserve(au.size() + nb.size());
      std::size_t x = 0, y = 0;
      while (x < au.size() || y < nb.size()) {
        int pick;
        if (y >= nb.size() || (x < au.size() && au[x] < nb[y])) {
          pick = au[x++];
        } else if (x >= au.size() || nb[y] < au[x]) {
          pick = nb[y++];
        } else {
          pick = au[x++];
          ++y;
        }
        if (pick != u && pick != v) merged.push_back(pick);
      }
      au.swap(merged);
      degree[u] = static_cast<idx>(au.size());
      heap.push({degree[u], u});
    }
  }
  // Postorder the elimination tree so fundamental supernodes are contiguous.
  std::vector<idx> iperm(n);
  for (idx k = 0; k < n; ++k) iperm[order[k]] = k;
  std::vector<idx> up_cp, up_ri;
  permuted_upper(lower, iperm, up_cp, up_ri);
  const std::vector<idx> parent = etree_of(n, up_cp, up_ri);
  const std::vector<idx> post = postorder_of(parent);
  std::vector<idx> perm(n);
  for (idx k = 0; k < n; ++k) perm[k] = order[post[k]];
  return perm;
}

AmalgParams AmalgParams::defaults() {
  AmalgParams p{1, 0.6};
  if (const char* e = std::getenv("HYKKT_AMALG_W")) p.width = std::atoi(e);
  if (const char* e = std::getenv("HYKKT_AMALG_Z")) p.zeros = std::atof(e);
  return p;
}

SupernodalPlan build_supernodal_plan(const CscPattern& a,
                                     std::vector<idx> perm, AmalgParams amalg) {
  const idx amalg_width = amalg.width;
  const double amalg_zeros = amalg.zeros;
  a.validate("pattern");
  if (a.nrows != a.ncols) fail("symbolic analysis requires a square pattern");
  const idx n = a.ncols;
  for (idx j = 0; j < n; ++j) {
    for (idx p = a.cp[j]; p < a.cp[j + 1]; ++p) {
      if (a.ri[p] < j) fail("pattern must be in lower-triangle storage");
    }
  }
  if (perm.empty()) perm = minimum_degree_order(a);
  if (static_cast<idx>(perm.size()) != n) fail("symbolic analysis: ordering size mismatch");
  SupernodalPlan s;
  s.n = n;
  s.iperm.assign(n, -1);
  for (idx i = 0; i < n; ++i) {
    const idx v = perm[i];
    if (v < 0 || v >= n || s.iperm[v] != -1) fail("permutation is not a bijection on [0, n)");
    s.iperm[v] = i;
  }
  s.perm = std::move(perm);

  std::vector<idx> up_cp, up_ri;
  permuted_upper(a, s.iperm, up_cp, up_ri);
  s.parent = etree_of(n, up_cp, up_ri);

  // Column counts and L pattern through row-subtree walks; rows appended
  // in ascending order keep the diagonal first in every column.
  s.col_counts.assign(n, 1);
  std::vector<idx> stamp(n, -1);
  auto walk = [&](idx k, auto&& visit) {
    stamp[k] = k;
    for (idx p = up_cp[k]; p < up_cp[k + 1]; ++p) {
      idx i = up_ri[p];
      while (i < k && stamp[i] != k) {
        visit(i);
        stamp[i] = k;
        i = s.parent[i];
      }
    }
  };
  for (idx k = 0; k < n; ++k) walk(k, [&](idx j) { s.col_counts[j]++; });
  s.l_cp.assign(n + 1, 0);
  std::partial_sum(s.col_counts.begin(), s.col_counts.end(), s.l_cp.begin() + 1);
  if (s.l_cp[n] >= (idx{1} << 31)) fail("L has more than 2^31 entries");
  s.l_ri.assign(s.l_cp[n], 0);
  {
    std::vector<idx> cur(s.l_cp.begin(), s.l_cp.end() - 1);
    std::fill(stamp.begin(), stamp.end(), -1);
    for (idx k = 0; k < n; ++k) {
      s.l_ri[cur[k]++] = k;
      walk(k, [&](idx j) { s.l_ri[cur[j]++] = k; });
    }
  }

  // Supernodes.  Column j joins the supernode of j-1 when j is j-1's parent
  // and its only child (a chain in the elimination tree) and either
  //   * the column structures nest exactly (fundamental supernodes), or
  //   * relaxed amalgamation: the merged supernode stays at most
  //     `amalg_width` columns wide and at most `amalg_zeros` of its panel
  //     entries are explicit zeros.
  // Along such a chain every column's structure below the supernode lies in
  // the last column's, so the merged row structure is the own columns plus
  // the last column's rows below it.  Explicit zeros stay exactly zero
  // through the factorization (their updates are products with structural
  // zeros), so results are unchanged; what changes is that a chain of
  // narrow supernodes — one cross-SM hand-off per link in the sync-free
  // solves — becomes one dense diagonal block solved inside one warp/CTA.
  std::vector<idx> nchild(n, 0);
  for (idx j = 0; j < n; ++j) {
    if (s.parent[j] >= 0) nchild[s.parent[j]]++;
  }
  s.sn_of.assign(n, 0);
  s.sn_first.clear();
  {
    idx f = 0, truth = 0;  // current supernode's first column and true L entries
    for (idx j = 0; j < n; ++j) {
      bool merge = j > 0 && s.parent[j - 1] == j && nchild[j] == 1;
      if (merge && s.col_counts[j - 1] != s.col_counts[j] + 1) {
        const idx w = j - f + 1, nr = w + s.col_counts[j] - 1;
        const idx entries = w * nr - w * (w - 1) / 2;
        const idx zeros = entries - (truth + s.col_counts[j]);
        merge = w <= amalg_width && static_cast<double>(zeros) <= amalg_zeros * static_cast<double>(entries);
      }
      if (!merge) {
        s.sn_first.push_back(static_cast<int>(j));
        f = j;
        truth = 0;
      }
      truth += s.col_counts[j];
      s.sn_of[j] = static_cast<int>(s.sn_first.size()) - 1;
    }
  }
  s.nsup = static_cast<idx>(s.sn_first.size());
  s.sn_first.push_back(static_cast<int>(n));
  const idx ns = s.nsup;

  s.sn_nrows.resize(ns);
  s.sn_off.assign(ns + 1, 0);
  s.sn_rows_ptr.assign(ns + 1, 0);
  for (idx k = 0; k < ns; ++k) {
    const idx f = s.sn_first[k], w = s.sn_first[k + 1] - f, last = f + w - 1;
    s.sn_nrows[k] = static_cast<int>(w + s.col_counts[last] - 1);
    s.sn_off[k + 1] = s.sn_off[k] + idx{s.sn_nrows[k]} * w;
    s.sn_rows_ptr[k + 1] = s.sn_rows_ptr[k] + s.sn_nrows[k];
    s.max_width = std::max<int>(s.max_width, static_cast<int>(w));
    s.max_nrows = std::max(s.max_nrows, s.sn_nrows[k]);
    s.explicit_zeros += idx{s.sn_nrows[k]} * w - w * (w - 1) / 2;
  }
  s.explicit_zeros -= s.l_cp[n];
  s.panel_size = s.sn_off[ns];
  if (s.panel_size >= (idx{1} << 31)) fail("supernodal panels exceed 2^31 slots");
  s.sn_rows.resize(s.sn_rows_ptr[ns]);
  for (idx k = 0; k < ns; ++k) {
    const idx f = s.sn_first[k], w = s.sn_first[k + 1] - f, last = f + w - 1;
    int* out = s.sn_rows.data() + s.sn_rows_ptr[k];
    for (idx c = 0; c < w; ++c) out[c] = static_cast<int>(f + c);
    std::copy(s.l_ri.begin() + s.l_cp[last] + 1, s.l_ri.begin() + s.l_cp[last + 1], out + w);
  }

  // Supernode tree, levels, children, level-sorted order.
  s.sn_parent.assign(ns, -1);
  s.sn_level.assign(ns, 0);
  for (idx k = 0; k < ns; ++k) {
    const idx last = s.sn_first[k + 1] - 1;
    const idx p = s.parent[last];
    s.sn_parent[k] = p < 0 ? -1 : s.sn_of[p];
  }
  for (idx k = 0; k < ns; ++k) {
    const int p = s.sn_parent[k];
    if (p >= 0) s.sn_level[p] = std::max(s.sn_level[p], s.sn_level[k] + 1);
    s.nlevels = std::max(s.nlevels, s.sn_level[k] + 1);
  }
  s.child_ptr.assign(ns + 1, 0);
  for (idx k = 0; k < ns; ++k) {
    if (s.sn_parent[k] >= 0) s.child_ptr[s.sn_parent[k] + 1]++;
  }
  std::partial_sum(s.child_ptr.begin(), s.child_ptr.end(), s.child_ptr.begin());
  s.child.resize(s.child_ptr[ns]);
  {
    std::vector<int> cur(s.child_ptr.begin(), s.child_ptr.end() - 1);
    for (idx k = 0; k < ns; ++k) {
      if (s.sn_parent[k] >= 0) s.child[cur[s.sn_parent[k]]++] = static_cast<int>(k);
    }
  }
  s.order.resize(ns);
  std::iota(s.order.begin(), s.order.end(), 0);
  std::stable_sort(s.order.begin(), s.order.end(),
                   [&](int x, int y) { return s.sn_level[x] < s.sn_level[y]; });

  // Update lists (target supernode <- descendant block runs).
  s.upd_ptr.assign(ns + 1, 0);
  auto for_runs = [&](auto&& emit) {
    for (idx d = 0; d < ns; ++d) {
      const int w = s.sn_first[d + 1] - s.sn_first[d];
      const int nr = s.sn_nrows[d];
      const int* rows = s.sn_rows.data() + s.sn_rows_ptr[d];
      int t = w;
      while (t < nr) {
        const int tgt = s.sn_of[rows[t]];
        int e = t;
        while (e < nr && s.sn_of[rows[e]] == tgt) ++e;
        emit(tgt, static_cast<int>(d), t, e - t);
        t = e;
      }
    }
  };
  for_runs([&](int tgt, int, int, int) { s.upd_ptr[tgt + 1]++; });
  std::partial_sum(s.upd_ptr.begin(), s.upd_ptr.end(), s.upd_ptr.begin());
  s.upd_d.resize(s.upd_ptr[ns]);
  s.upd_off.resize(s.upd_ptr[ns]);
  s.upd_cnt.resize(s.upd_ptr[ns]);
  {
    std::vector<int> cur(s.upd_ptr.begin(), s.upd_ptr.end() - 1);
    for_runs([&](int tgt, int d, int off, int cnt) {
      const int q = cur[tgt]++;
      s.upd_d[q] = d;
      s.upd_off[q] = off;
      s.upd_cnt[q] = cnt;
    });
  }

  // Forward-solve row lists (entries of L below the diagonal blocks).
  s.lrow_ptr.assign(n + 1, 0);
  for (idx d = 0; d < ns; ++d) {
    const int w = s.sn_first[d + 1] - s.sn_first[d];
    const int nr = s.sn_nrows[d];
    const int* rows = s.sn_rows.data() + s.sn_rows_ptr[d];
    for (int t = w; t < nr; ++t) s.lrow_ptr[rows[t] + 1] += w;
  }
  std::partial_sum(s.lrow_ptr.begin(), s.lrow_ptr.end(), s.lrow_ptr.begin());
  s.lrow_col.resize(s.lrow_ptr[n]);
  s.lrow_row.resize(s.lrow_ptr[n]);
  s.lrow_pos.resize(s.lrow_ptr[n]);
  {
    std::vector<int> cur(s.lrow_ptr.begin(), s.lrow_ptr.end() - 1);
    for (idx d = 0; d < ns; ++d) {
      const int f = s.sn_first[d], w = s.sn_first[d + 1] - f;
      const int nr = s.sn_nrows[d];
      const int* rows = s.sn_rows.data() + s.sn_rows_ptr[d];
      for (int k = 0; k < w; ++k) {
        for (int t = w; t < nr; ++t) {
          const int q = cur[rows[t]]++;
          s.lrow_col[q] = f + k;
          s.lrow_row[q] = rows[t];
          s.lrow_pos[q] = static_cast<int>(s.sn_off[d] + idx{k} * nr + t);
        }
      }
    }
  }

  // Update-vector storage and child -> parent extend-add gather maps.
  s.u_off.assign(ns + 1, 0);
  s.ext_ptr.assign(ns + 1, 0);
  for (idx k = 0; k < ns; ++k) {
    const int w = s.sn_first[k + 1] - s.sn_first[k];
    s.u_off[k + 1] = s.u_off[k] + (s.sn_nrows[k] - w);
    const int p = s.sn_parent[k];
    s.ext_ptr[k + 1] = s.ext_ptr[k] + (p >= 0 ? s.sn_nrows[p] : 0);
  }
  s.ext_map.assign(s.ext_ptr[ns], -1);
  s.relind.assign(s.u_off[ns], -1);
  for (idx k = 0; k < ns; ++k) {
    const int p = s.sn_parent[k];
    if (p < 0) continue;
    const int w = s.sn_first[k + 1] - s.sn_first[k];
    const int* rc = s.sn_rows.data() + s.sn_rows_ptr[k];
    const int* rp = s.sn_rows.data() + s.sn_rows_ptr[p];
    const int nrp = s.sn_nrows[p];
    int q = 0;
    for (int t = w; t < s.sn_nrows[k]; ++t) {  // both lists ascending
      while (q < nrp && rp[q] < rc[t]) ++q;
      if (q == nrp || rp[q] != rc[t]) fail("internal: child row not in parent structure");
      s.ext_map[s.ext_ptr[k] + q] = t - w;
      s.relind[s.u_off[k] + t - w] = q;
    }
  }

  {
    const int nslot = s.sn_rows_ptr[ns];
    s.gat_ptr.assign(nslot + 1, 0);
    for (idx k = 0; k < ns; ++k) {
      const int p = s.sn_parent[k];
      if (p < 0) continue;
      for (int q = 0; q < s.sn_nrows[p]; ++q) {
        if (s.ext_map[s.ext_ptr[k] + q] >= 0) s.gat_ptr[s.sn_rows_ptr[p] + q + 1]++;
      }
    }
    std::partial_sum(s.gat_ptr.begin(), s.gat_ptr.end(), s.gat_ptr.begin());
    s.gat_idx.resize(s.gat_ptr[nslot]);
    std::vector<int> cur(s.gat_ptr.begin(), s.gat_ptr.end() - 1);
    for (idx p = 0; p < ns; ++p) {  // children in ascending order per parent
      for (int c = s.child_ptr[p]; c < s.child_ptr[p + 1]; ++c) {
        const int k = s.child[c];
        for (int q = 0; q < s.sn_nrows[p]; ++q) {
          const int t = s.ext_map[s.ext_ptr[k] + q];
          if (t >= 0) s.gat_idx[cur[s.sn_rows_ptr[p] + q]++] = s.u_off[k] + t;
        }
      }
    }
  }

  // Reference-layout L positions and diagonal slots.
  s.l_to_panel.resize(s.l_nnz());
  s.diag_panel.resize(n);
  for (idx j = 0; j < n; ++j) {
    const int k = s.sn_of[j];
    const int f = s.sn_first[k], w = s.sn_first[k + 1] - f, nr = s.sn_nrows[k];
    const idx c = j - f;
    const idx col0 = s.sn_off[k] + c * nr;
    s.diag_panel[j] = static_cast<int>(col0 + c);
    // rows of column j inside the supernode's (possibly amalgamated) structure
    const int* rows = s.sn_rows.data() + s.sn_rows_ptr[k];
    const int* lo = rows + w;
    for (idx t = 0; t < s.col_counts[j]; ++t) {
      const idx r = s.l_ri[s.l_cp[j] + t];
      idx pos;
      if (r < f + w) {
        pos = r - f;
      } else {
        lo = std::lower_bound(lo, rows + nr, static_cast<int>(r));
        if (lo == rows + nr || *lo != r) fail("internal: L entry outside its supernode structure");
        pos = lo - rows;
      }
      s.l_to_panel[s.l_cp[j] + t] = static_cast<int>(col0 + pos);
    }
  }

  // Input entry -> panel slot.
  s.src_to_panel.resize(a.nnz());
  for (idx j = 0; j < n; ++j) {
    for (idx p = a.cp[j]; p < a.cp[j + 1]; ++p) {
      const idx r0 = s.iperm[a.ri[p]], c0 = s.iperm[j];
      const idx row = std::max(r0, c0), col = std::min(r0, c0);
      const int k = s.sn_of[col];
      const int f = s.sn_first[k], w = s.sn_first[k + 1] - f, nr = s.sn_nrows[k];
      idx pos;
      if (row < f + w) {
        pos = row - f;
      } else {
        const int* rows = s.sn_rows.data() + s.sn_rows_ptr[k];
        const int* it = std::lower_bound(rows + w, rows + nr, static_cast<int>(row));
        if (it == rows + nr || *it != row) fail("internal: entry outside the symbolic pattern");
        pos = it - rows;
      }
      s.src_to_panel[p] = static_cast<int>(s.sn_off[k] + (col - f) * nr + pos);
    }
  }

  for (idx j = 0; j < n; ++j) {
    s.factor_flops += static_cast<double>(s.col_counts[j]) * s.col_counts[j];
  }
  return s;
}

// ---------------------------------------------------------------------------
namespace {

// Row-wise view (CSR) of a CSC pattern: for row k the (column, CSC index)
// pairs in ascending column order.
void csr_of(const CscPattern& m, std::vector<int>& rp, std::vector<int>& ci,
            std::vector<int>& src) {
  rp.assign(m.nrows + 1, 0);
  for (idx p = 0; p < m.nnz(); ++p) rp[m.ri[p] + 1]++;
  std::partial_sum(rp.begin(), rp.end(), rp.begin());
  ci.resize(m.nnz());
  src.resize(m.nnz());
  std::vector<int> cur(rp.begin(), rp.end() - 1);
  for (idx j = 0; j < m.ncols; ++j) {
    for (idx p = m.cp[j]; p < m.cp[j + 1]; ++p) {
      const int q = cur[m.ri[p]]++;
      ci[q] = static_cast<int>(j);
      src[q] = static_cast<int>(p);
    }
  }
}

// Products of lower(A^T D A) grouped by output slot (column j, row i >= j)
// and, within a slot, by ascending k — the accumulation order of
// ata_lower (csc_matrix.cpp:368-383).
struct ProductSet {
  std::vector<int> col_ptr;      // per output column: range into the arrays
  std::vector<int> row, k, a, b; // sorted by (col, row, k)
};

ProductSet products_of(const CscPattern& m) {
  std::vector<int> rp, ci, src;
  csr_of(m, rp, ci, src);
  const idx ncols = m.ncols;
  ProductSet ps;
  ps.col_ptr.assign(ncols + 1, 0);
  for (idx k = 0; k < m.nrows; ++k) {
    for (int x = rp[k]; x < rp[k + 1]; ++x) ps.col_ptr[ci[x] + 1] += rp[k + 1] - x;
  }
  std::partial_sum(ps.col_ptr.begin(), ps.col_ptr.end(), ps.col_ptr.begin());
  const idx total = ps.col_ptr[ncols];
  ps.row.resize(total);
  ps.k.resize(total);
  ps.a.resize(total);
  ps.b.resize(total);
  std::vector<int> cur(ps.col_ptr.begin(), ps.col_ptr.end() - 1);
  for (idx k = 0; k < m.nrows; ++k) {  // ascending k
    for (int x = rp[k]; x < rp[k + 1]; ++x) {
      for (int y = x; y < rp[k + 1]; ++y) {
        const int q = cur[ci[x]]++;
        ps.row[q] = ci[y];
        ps.k[q] = static_cast<int>(k);
        ps.a[q] = src[x];  // (k, col)
        ps.b[q] = src[y];  // (k, row)
      }
    }
  }
  // Stable sort by row inside each column keeps k ascending per slot.
  std::vector<int> perm;
  std::vector<int> tmp;
  for (idx j = 0; j < ncols; ++j) {
    const int lo = ps.col_ptr[j], hi = ps.col_ptr[j + 1];
    perm.resize(hi - lo);
    std::iota(perm.begin(), perm.end(), lo);
    std::stable_sort(perm.begin(), perm.end(),
                     [&](int x, int y) { return ps.row[x] < ps.row[y]; });
    for (std::vector<int>* arr : {&ps.row, &ps.k, &ps.a, &ps.b}) {
      tmp.resize(hi - lo);
      for (int t = 0; t < hi - lo; ++t) tmp[t] = (*arr)[perm[t]];
      std::copy(tmp.begin(), tmp.end(), arr->begin() + lo);
    }
  }
  return ps;
}

}  // namespace

KktPlan build_kkt_plan(idx nx, idx mc, idx md, const CscPattern& h,
                       const CscPattern& j, const CscPattern& jd) {
  h.validate("H");
  j.validate("J");
  jd.validate("J_d");
  if (h.nrows != nx || h.ncols != nx) fail("H must be n_x x n_x");
  if (j.nrows != mc || j.ncols != nx) fail("J must be m_c x n_x");
  if (jd.nrows != md || jd.ncols != nx) fail("J_d must be m_d x n_x");
  for (idx c = 0; c < nx; ++c) {
    for (idx p = h.cp[c]; p < h.cp[c + 1]; ++p) {
      if (h.ri[p] < c) fail("add_symmetric_lower: term not in lower-triangle storage");
    }
  }
  if (h.nnz() + j.nnz() + jd.nnz() >= (idx{1} << 31)) fail("input too large for 32-bit slots");
  KktPlan kp;
  kp.nx = nx;
  kp.mc = mc;
  kp.md = md;
  kp.h = h;
  kp.j = j;
  kp.jd = jd;

  // H_tilde slots.
  const ProductSet pd = products_of(jd);
  kp.ht.nrows = kp.ht.ncols = nx;
  kp.ht.cp.assign(nx + 1, 0);
  kp.ht_prod_ptr.assign(1, 0);
  for (idx c = 0; c < nx; ++c) {
    idx hp = h.cp[c];
    int qp = pd.col_ptr[c];
    const int qe = pd.col_ptr[c + 1];
    bool diag_done = false;  // the diagonal is always stored (and smallest)
    for (;;) {
      idx row = nx;
      if (!diag_done) row = c;
      if (hp < h.cp[c + 1]) row = std::min(row, h.ri[hp]);
      if (qp < qe) row = std::min<idx>(row, pd.row[qp]);
      if (row == nx) break;
      diag_done = true;
      kp.ht.ri.push_back(row);
      kp.ht_col.push_back(static_cast<int>(c));
      kp.ht_diag.push_back(row == c ? 1 : 0);
      int hsrc = -1;
      if (hp < h.cp[c + 1] && h.ri[hp] == row) hsrc = static_cast<int>(hp++);
      kp.ht_hsrc.push_back(hsrc);
      while (qp < qe && pd.row[qp] == row) {
        kp.ht_prod_a.push_back(pd.a[qp]);
        kp.ht_prod_b.push_back(pd.b[qp]);
        kp.ht_prod_k.push_back(pd.k[qp]);
        ++qp;
      }
      kp.ht_prod_ptr.push_back(static_cast<int>(kp.ht_prod_a.size()));
    }
    kp.ht.cp[c + 1] = kp.ht.nnz();
  }

  // H_gamma slots: H_tilde slots union lower(J^T J).
  const ProductSet pj = products_of(j);
  kp.hg.nrows = kp.hg.ncols = nx;
  kp.hg.cp.assign(nx + 1, 0);
  kp.hg_prod_ptr.assign(1, 0);
  for (idx c = 0; c < nx; ++c) {
    idx tp = kp.ht.cp[c];
    const idx te = kp.ht.cp[c + 1];
    int qp = pj.col_ptr[c];
    const int qe = pj.col_ptr[c + 1];
    for (;;) {
      idx best = nx;
      if (tp < te) best = std::min(best, kp.ht.ri[tp]);
      if (qp < qe) best = std::min<idx>(best, pj.row[qp]);
      if (best == nx) break;
      kp.hg.ri.push_back(best);
      int src = -1;
      if (tp < te && kp.ht.ri[tp] == best) src = static_cast<int>(tp++);
      kp.hg_htsrc.push_back(src);
      while (qp < qe && pj.row[qp] == best) {
        kp.hg_prod_a.push_back(pj.a[qp]);
        kp.hg_prod_b.push_back(pj.b[qp]);
        ++qp;
      }
      kp.hg_prod_ptr.push_back(static_cast<int>(kp.hg_prod_a.size()));
    }
    kp.hg.cp[c + 1] = kp.hg.nnz();
  }

  csr_of(j, kp.j_rp, kp.j_ci, kp.jcsr_src);
  csr_of(jd, kp.jd_rp, kp.jd_ci, kp.jdcsr_src);
  return kp;
}

}  // namespace hykkt
