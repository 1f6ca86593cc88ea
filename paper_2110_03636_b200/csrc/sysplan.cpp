// Builder of the streamed per-system Schur-operator program (sysplan.hpp,
// stream layouts in sysplan_format.h).
//
// The L steps restate factor_solve (proj/core/src/cholesky.cpp:139-168) in
// gather form on the supernodal factor:
//   forward  y_i = (b_i - sum_{j<i} L_ij y_j) / L_ii      (row gathers)
//   backward x_k = (y_k - sum_{i>k} L_ik x_i) / L_kk      (column gathers)
// the J / JT steps restate spmv (csc_matrix.cpp:236-263) row by row.
#include "sysplan.hpp"

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <numeric>
#include <string>

namespace hykkt {

namespace {

// longest gather a thread task does inline; longer ones are split into
// phase-A segments (measured: 8 beats 32 by ~9 % on the ACTIVSg2000 batch).
// HYKKT_KS_INLINE overrides.
int inline_max() {
  static const int v = std::getenv("HYKKT_KS_INLINE") ? std::atoi(std::getenv("HYKKT_KS_INLINE")) : 8;
  return v;
}
// widest supernode a single thread solves (wider ones are warp tasks)
int thread_task_w() {
  static const int v = std::getenv("HYKKT_KS_THREAD_W") ? std::atoi(std::getenv("HYKKT_KS_THREAD_W")) : 3;
  return v;
}
// shortest segment (partial dot product) of a long gather
int min_seg() {
  static const int v = std::getenv("HYKKT_KS_MINSEG") ? std::max(1, std::atoi(std::getenv("HYKKT_KS_MINSEG"))) : 8;
  return v;
}

struct Seg {
  std::vector<int> vsrc;  // value sources
  std::vector<int> ind;   // one index per value
  int slot = 0;
};

struct Task {
  bool warp = false, inline_ = false;
  int f = 0, w = 0;
  long long cost = 0;
  std::vector<int> vsrc;  // value payload
  std::vector<int> ipay;  // index payload
  int seg_rows = 0;
};

inline int panel_src(long long slot, bool recip) { return static_cast<int>(slot * 2 + (recip ? 1 : 0)); }

struct Builder {
  const SupernodalPlan& sp;
  const KktPlan& kp;
  SysPlan& P;
  long long capv, capi, capv_rows, capi_rows;
  long long last_hdr = -1;  // index position of the last emitted header

  Builder(const SupernodalPlan& s, const KktPlan& k, SysPlan& p) : sp(s), kp(k), P(p) {
    // L steps: at most n/2 - 1 chunks, so a step spans <= n/2 chunks at any
    // alignment and two consecutive steps always fit the ring: the data of
    // step k+1 is requested when step k starts (sysplan.hpp).  J / JT steps
    // (no dependencies between them) may use n - 2 chunks.
    capv = static_cast<long long>(P.step_chunks) << P.vchunk_lg;
    capi = static_cast<long long>(P.step_chunks) << P.ichunk_lg;
    capv_rows = static_cast<long long>(P.nvchunk - 2) << P.vchunk_lg;
    capi_rows = static_cast<long long>(P.nichunk - 2) << P.ichunk_lg;
  }

  int width(int s) const { return sp.sn_first[s + 1] - sp.sn_first[s]; }
  int below(int s) const { return sp.sn_nrows[s] - width(s); }
  int row_gather(int i) const { return sp.lrow_ptr[i + 1] - sp.lrow_ptr[i]; }
  long long vpos() const { return static_cast<long long>(P.src.size()); }
  long long ipos() const { return static_cast<long long>(P.idx.size()); }

  // ---- one L step ----------------------------------------------------------
  void emit_l_step(int kind, const std::vector<const Seg*>& segs, const std::vector<const Task*>& warp,
                   const std::vector<const Task*>& thr, bool reads_earlier, int ww) {
    const long long ib = ipos(), vb = vpos();
    const int nseg = static_cast<int>(segs.size()), nt = static_cast<int>(warp.size() + thr.size());
    last_hdr = ib;
    P.idx.insert(P.idx.end(), {kind, 0, 0, nseg, static_cast<int>(warp.size()), static_cast<int>(thr.size()),
                               reads_earlier ? 1 : 0, ww});
    const long long desc0 = ipos();
    P.idx.resize(desc0 + HYKKT_SP_SEG_INTS * nseg + HYKKT_SP_TASK_INTS * nt, 0);
    for (int g = 0; g < nseg; ++g) {
      const Seg& s = *segs[g];
      const long long d = desc0 + HYKKT_SP_SEG_INTS * g;
      P.idx[d] = static_cast<int>(vpos() - vb);
      P.idx[d + 1] = static_cast<int>(ipos() - ib);
      P.idx[d + 2] = static_cast<int>(s.vsrc.size()) | (s.slot << 16);
      P.src.insert(P.src.end(), s.vsrc.begin(), s.vsrc.end());
      P.idx.insert(P.idx.end(), s.ind.begin(), s.ind.end());
    }
    int t = 0;
    for (const auto* list : {&warp, &thr}) {
      for (const Task* tk : *list) {
        const long long d = desc0 + HYKKT_SP_SEG_INTS * nseg + HYKKT_SP_TASK_INTS * t;
        P.idx[d] = static_cast<int>(vpos() - vb);
        P.idx[d + 1] = static_cast<int>(ipos() - ib);
        P.idx[d + 2] = tk->f;
        P.idx[d + 3] = tk->w | ((tk->inline_ ? HYKKT_TASK_INLINE : HYKKT_TASK_SEGMENTED) << 16);
        P.src.insert(P.src.end(), tk->vsrc.begin(), tk->vsrc.end());
        P.idx.insert(P.idx.end(), tk->ipay.begin(), tk->ipay.end());
        ++t;
      }
    }
    P.idx[ib + 1] = static_cast<int>(ipos() - ib);
    P.idx[ib + 2] = static_cast<int>(vpos() - vb);
    if (ipos() - ib > capi || vpos() - vb > capv) throw InvalidArgument("sys plan: step does not fit the rings");
    P.nsteps++;
    P.nsegs += nseg;
    P.ntasks += nt;
  }

  // ---- L tasks -------------------------------------------------------------
  Task make_task(int s, bool bwd) const {
    Task t;
    const int f = sp.sn_first[s], w = width(s), nr = sp.sn_nrows[s];
    const int* R = sp.sn_rows.data() + sp.sn_rows_ptr[s];
    const long long off = sp.sn_off[s];
    t.f = f;
    t.w = w;
    t.warp = w > thread_task_w();
    long long g = 0;
    if (!bwd) {
      for (int r = 0; r < w; ++r) g += row_gather(f + r);
    } else {
      g = static_cast<long long>(below(s)) * w;
    }
    t.inline_ = !t.warp && g <= inline_max();
    t.seg_rows = t.inline_ ? 0 : w;
    t.cost = g + w * (w + 1) / 2;
    if (!bwd) {
      for (int r = 0; r < w; ++r) {
        for (int j = 0; j <= r; ++j) t.vsrc.push_back(panel_src(off + static_cast<long long>(j) * nr + r, j == r));
      }
      if (t.inline_) {
        for (int r = 0; r < w; ++r) t.ipay.push_back(row_gather(f + r));
        t.ipay.push_back(0);
        for (int r = 0; r < w; ++r) {
          for (int q = sp.lrow_ptr[f + r]; q < sp.lrow_ptr[f + r + 1]; ++q) {
            t.vsrc.push_back(panel_src(sp.lrow_pos[q], false));
            t.ipay.push_back(sp.lrow_col[q]);
          }
        }
      }
    } else {
      for (int k = 0; k < w; ++k) {
        for (int j = k; j < w; ++j) t.vsrc.push_back(panel_src(off + static_cast<long long>(k) * nr + j, j == k));
      }
      if (t.inline_) {
        t.ipay.push_back(nr - w);
        for (int q = w; q < nr; ++q) {
          t.ipay.push_back(R[q]);
          for (int k = 0; k < w; ++k) t.vsrc.push_back(panel_src(off + static_cast<long long>(k) * nr + q, false));
        }
      }
    }
    return t;
  }

  // Segments of the group's segmented tasks (each row / column split into
  // runs of at most sl entries); sets each segmented task's index payload
  // to its first-slot-per-row list plus the end slot.
  std::vector<Seg> make_segments(std::vector<Task>& g, const std::vector<int>& sns, bool bwd, int sl) const {
    std::vector<Seg> out;
    int slot = 0;
    for (std::size_t ti = 0; ti < g.size(); ++ti) {
      Task& t = g[ti];
      if (t.inline_) continue;
      const int s = sns[ti], f = t.f, w = t.w, nr = sp.sn_nrows[s];
      const int* R = sp.sn_rows.data() + sp.sn_rows_ptr[s];
      std::vector<int> slots;
      for (int r = 0; r < w; ++r) {
        slots.push_back(slot);
        if (!bwd) {
          const int q0 = sp.lrow_ptr[f + r], q1 = sp.lrow_ptr[f + r + 1];
          for (int q = q0; q < q1; q += sl) {
            Seg sg;
            sg.slot = slot++;
            for (int e = q; e < std::min(q + sl, q1); ++e) {
              sg.vsrc.push_back(panel_src(sp.lrow_pos[e], false));
              sg.ind.push_back(sp.lrow_col[e]);
            }
            out.push_back(std::move(sg));
          }
        } else {
          const long long base = sp.sn_off[s] + static_cast<long long>(r) * nr;
          for (int q = w; q < nr; q += sl) {
            Seg sg;
            sg.slot = slot++;
            for (int e = q; e < std::min(q + sl, nr); ++e) {
              sg.vsrc.push_back(panel_src(base + e, false));
              sg.ind.push_back(R[e]);
            }
            out.push_back(std::move(sg));
          }
        }
      }
      slots.push_back(slot);
      t.ipay = slots;
    }
    return out;
  }

  int seg_count(const std::vector<int>& sns, const std::vector<Task>& g, bool bwd, int sl) const {
    long long n = 0;
    for (std::size_t ti = 0; ti < g.size(); ++ti) {
      if (g[ti].inline_) continue;
      const int s = sns[ti], w = width(s);
      if (!bwd) {
        for (int r = 0; r < w; ++r) n += (row_gather(sp.sn_first[s] + r) + sl - 1) / sl;
      } else {
        n += static_cast<long long>(w) * ((below(s) + sl - 1) / sl);
      }
    }
    return static_cast<int>(std::min<long long>(n, 1 << 30));
  }

  void emit_group(const std::vector<int>& sns, bool bwd) {
    std::vector<Task> g;
    g.reserve(sns.size());
    for (int s : sns) g.push_back(make_task(s, bwd));
    int sl = min_seg();
    while (seg_count(sns, g, bwd, sl) > P.pmax) {
      sl *= 2;
      if (sl > capv / 4) throw InvalidArgument("sys plan: too many segments for the partials array");
    }
    std::vector<Seg> segs = make_segments(g, sns, bwd, sl);
    std::vector<const Task*> warp, thr;
    long long tv = 0, ti = 0;
    for (const Task& t : g) {
      (t.warp ? warp : thr).push_back(&t);
      tv += static_cast<long long>(t.vsrc.size());
      ti += static_cast<long long>(t.ipay.size()) + HYKKT_SP_TASK_INTS;
    }
    auto by_cost = [](const Task* a, const Task* b) { return a->cost > b->cost; };
    std::stable_sort(warp.begin(), warp.end(), by_cost);
    std::stable_sort(thr.begin(), thr.end(), by_cost);
    // warps [0, ww) take the warp tasks; thread tasks are dealt over the
    // remaining NT - 32 ww threads (sysplan_format.h header word 7)
    const int nwarps = P.nthreads / 32;
    static const int wwk = std::getenv("HYKKT_KS_WW8") ? std::atoi(std::getenv("HYKKT_KS_WW8")) : 5;  // eighths of the warps (B200 sweep)
    const int ww = warp.empty() ? 0 : thr.empty() ? std::min<int>(static_cast<int>(warp.size()), nwarps)
                                                  : std::min<int>(static_cast<int>(warp.size()),
                                                                  std::max(1, std::min(nwarps - 1, nwarps * wwk / 8)));
    // deal thread tasks: thread t takes positions t, t + NT, ...; snake order
    // over the full rounds balances every thread's total cost
    {
      const std::size_t NT = static_cast<std::size_t>(P.nthreads - 32 * ww);
      std::vector<const Task*> dealt(thr.size());
      const std::size_t full = thr.size() / NT;
      for (std::size_t i = 0; i < thr.size(); ++i) {
        const std::size_t r = i / NT, t = i % NT;
        dealt[i] = thr[(r < full && (r & 1)) ? r * NT + (NT - 1 - t) : i];
      }
      thr.swap(dealt);
    }
    // leading A-steps take segments; the final step carries the rest + tasks
    const int ns = static_cast<int>(segs.size());
    std::vector<long long> sv(ns + 1, 0), si(ns + 1, 0);
    for (int q = 0; q < ns; ++q) {
      sv[q + 1] = sv[q] + static_cast<long long>(segs[q].vsrc.size());
      si[q + 1] = si[q] + static_cast<long long>(segs[q].ind.size()) + HYKKT_SP_SEG_INTS;
    }
    auto fits = [&](int a, int b, long long extra_v, long long extra_i) {
      return sv[b] - sv[a] + extra_v <= capv && HYKKT_SP_HDR + si[b] - si[a] + extra_i <= capi;
    };
    int fa = ns;
    while (fa > 0 && fits(fa - 1, ns, tv, ti)) --fa;
    if (!fits(fa, ns, tv, ti)) throw InvalidArgument("sys plan: supernode group does not fit the rings");
    int a = 0;
    const std::vector<const Task*> none;
    while (a < fa) {
      int b = a;
      while (b < fa && fits(a, b + 1, 0, 0)) ++b;
      if (b == a) throw InvalidArgument("sys plan: segment does not fit the rings");
      std::vector<const Seg*> part;
      for (int q = a; q < b; ++q) part.push_back(&segs[q]);
      emit_l_step(bwd ? HYKKT_STEP_BWD : HYKKT_STEP_FWD, part, none, none, false, 0);
      a = b;
    }
    std::vector<const Seg*> part;
    for (int q = fa; q < ns; ++q) part.push_back(&segs[q]);
    emit_l_step(bwd ? HYKKT_STEP_BWD : HYKKT_STEP_FWD, part, warp, thr, fa > 0, ww);
    P.max_segs_per_step = std::max(P.max_segs_per_step, ns);
  }

  void l_pass(bool bwd) {
    const int ns = static_cast<int>(sp.nsup);
    std::vector<std::vector<int>> by_level(std::max(1, sp.nlevels));
    for (int s = 0; s < ns; ++s) by_level[sp.sn_level[s]].push_back(s);
    for (int li = 0; li < sp.nlevels; ++li) {
      const int L = bwd ? sp.nlevels - 1 - li : li;
      std::vector<int> group;
      long long gv = 0, gi = 0;
      int rows = 0;
      for (int s : by_level[L]) {
        const Task t = make_task(s, bwd);
        const long long v = static_cast<long long>(t.vsrc.size());
        const long long i = static_cast<long long>(t.ipay.size()) + HYKKT_SP_TASK_INTS + (t.inline_ ? 0 : t.w + 1);
        const long long ci = capi - HYKKT_SP_HDR;
        if (v > capv || i > ci) throw InvalidArgument("sys plan: supernode block larger than the rings");
        if (!group.empty() && (gv + v > capv || gi + i > ci || 2 * (rows + t.seg_rows) > P.pmax)) {
          emit_group(group, bwd);
          group.clear();
          gv = gi = 0;
          rows = 0;
        }
        group.push_back(s);
        gv += v;
        gi += i;
        rows += t.seg_rows;
      }
      if (!group.empty()) emit_group(group, bwd);
    }
  }

  // ---- J^T and J row blocks --------------------------------------------------
  // row(r, ent) appends (value source, index) pairs of row r
  template <typename RowFn>
  void row_pass(int kind, int nrows, RowFn&& row) {
    int r = 0;
    std::vector<std::pair<int, int>> ent;
    while (r < nrows) {
      std::vector<int> offs{0};
      std::vector<int> vs, is;
      int r1 = r;
      while (r1 < nrows) {
        ent.clear();
        row(r1, ent);
        const long long v = static_cast<long long>(vs.size() + ent.size());
        const long long i = HYKKT_SP_HDR + static_cast<long long>(offs.size() + 1 + is.size() + ent.size());
        if (v > capv_rows || i > capi_rows) {
          if (r1 == r) throw InvalidArgument("sys plan: matrix row does not fit the rings");
          break;
        }
        for (auto& e : ent) {
          vs.push_back(e.first);
          is.push_back(e.second);
        }
        offs.push_back(static_cast<int>(vs.size()));
        ++r1;
      }
      const long long ib = ipos();
      last_hdr = ib;
      P.idx.insert(P.idx.end(), {kind, 0, static_cast<int>(vs.size()), r1 - r, r, 0, 0, 0});
      P.idx.insert(P.idx.end(), offs.begin(), offs.end());
      P.idx.insert(P.idx.end(), is.begin(), is.end());
      P.src.insert(P.src.end(), vs.begin(), vs.end());
      P.idx[ib + 1] = static_cast<int>(ipos() - ib);
      P.nsteps++;
      r = r1;
    }
  }

  // Pads both streams to chunk boundaries, charging the padding to the
  // block's last step.
  void close_block(int b, long long v0, long long i0, int s0) {
    const long long cv = 1ll << P.vchunk_lg, ci = 1ll << P.ichunk_lg;
    const long long pv = (cv - vpos() % cv) % cv, pi = (ci - ipos() % ci) % ci;
    P.src.insert(P.src.end(), pv, HYKKT_SRC_ZERO);
    P.idx.insert(P.idx.end(), pi, 0);
    if (P.nsteps > s0) {
      P.idx[last_hdr + 1] += static_cast<int>(pi);
      P.idx[last_hdr + 2] += static_cast<int>(pv);
    }
    P.blk[b] = SysPlan::Block{v0, vpos(), i0, ipos(), s0, P.nsteps};
  }
};

}  // namespace

SysPlan build_sys_plan(const SupernodalPlan& sp, const KktPlan& kp, int vchunk_lg, int nvchunk, int ichunk_lg,
                       int nichunk, int pmax, int nthreads, int step_chunks) {
  if (nvchunk < 4 || nichunk < 4 || (nvchunk & (nvchunk - 1)) || (nichunk & (nichunk - 1)))
    throw InvalidArgument("sys plan: rings need a power-of-two count >= 4 of chunks");
  if (pmax < 64 || pmax >= (1 << 15)) throw InvalidArgument("sys plan: bad partials size");
  if (nthreads < 32 || nthreads % 32) throw InvalidArgument("sys plan: bad CTA size");
  SysPlan P;
  P.vchunk_lg = vchunk_lg;
  P.nvchunk = nvchunk;
  P.ichunk_lg = ichunk_lg;
  P.nichunk = nichunk;
  P.pmax = pmax;
  P.nthreads = nthreads;
  P.step_chunks = step_chunks > 0 ? std::min(step_chunks, std::min(nvchunk, nichunk) - 2)
                                  : std::min(nvchunk, nichunk) / 2 - 1;
  Builder b(sp, kp, P);
  const int n = static_cast<int>(sp.n), mc = static_cast<int>(kp.mc);
  // JT: row i of P J^T = column perm[i] of J (spmv transpose order)
  long long v0 = b.vpos(), i0 = b.ipos();
  int s0 = P.nsteps;
  b.row_pass(HYKKT_STEP_JT, n, [&](int i, std::vector<std::pair<int, int>>& e) {
    const idx o = sp.perm[i];
    for (idx q = kp.j.cp[o]; q < kp.j.cp[o + 1]; ++q) e.emplace_back(static_cast<int>(-2 - q), static_cast<int>(kp.j.ri[q]));
  });
  b.close_block(0, v0, i0, s0);
  v0 = b.vpos(), i0 = b.ipos(), s0 = P.nsteps;
  b.l_pass(false);
  b.close_block(1, v0, i0, s0);
  v0 = b.vpos(), i0 = b.ipos(), s0 = P.nsteps;
  b.l_pass(true);
  b.close_block(2, v0, i0, s0);
  // J: rows in CSR order, columns ascending (the reference's scatter order)
  v0 = b.vpos(), i0 = b.ipos(), s0 = P.nsteps;
  b.row_pass(HYKKT_STEP_J, mc, [&](int k, std::vector<std::pair<int, int>>& e) {
    for (int q = kp.j_rp[k]; q < kp.j_rp[k + 1]; ++q) {
      e.emplace_back(-2 - kp.jcsr_src[q], static_cast<int>(sp.iperm[kp.j_ci[q]]));
    }
  });
  b.close_block(3, v0, i0, s0);
  for (int x : P.src) P.value_entries += x != HYKKT_SRC_ZERO;
  if (static_cast<long long>(P.src.size()) >= (1ll << 31) || static_cast<long long>(P.idx.size()) >= (1ll << 31))
    throw InvalidArgument("sys plan: stream exceeds 2^31 entries");
  return P;
}

// ---------------------------------------------------------------------------
// Host emulation of the device interpreter (kernels_sys.cuh).
double sys_plan_selfcheck(const SupernodalPlan& sp, const KktPlan& kp, const SysPlan& P, unsigned seed) {
  const idx n = sp.n, mc = kp.mc;
  unsigned long long st = seed * 6364136223846793005ull + 1442695040888963407ull;
  auto rnd = [&] {
    st = st * 6364136223846793005ull + 1442695040888963407ull;
    return static_cast<double>(st >> 11) * (1.0 / 9007199254740992.0) - 0.5;
  };
  std::vector<double> panel(std::max<idx>(sp.panel_size, 1), 0.0);
  for (idx s = 0; s < sp.nsup; ++s) {
    const int f = sp.sn_first[s], w = sp.sn_first[s + 1] - f, nr = sp.sn_nrows[s];
    for (int k = 0; k < w; ++k) {
      for (int q = k; q < nr; ++q) panel[sp.sn_off[s] + static_cast<idx>(k) * nr + q] = q == k ? 2.0 + rnd() : 0.3 * rnd();
    }
  }
  std::vector<double> jv(std::max<idx>(kp.j.nnz(), 1)), u(std::max<idx>(mc, 1));
  for (auto& x : jv) x = rnd();
  for (auto& x : u) x = rnd();
  // reference: t = P J^T u, supernodal forward / backward solves, q = J x
  std::vector<double> y(n, 0.0);
  for (idx i = 0; i < n; ++i) {
    const idx o = sp.perm[i];
    for (idx q = kp.j.cp[o]; q < kp.j.cp[o + 1]; ++q) y[i] += jv[q] * u[kp.j.ri[q]];
  }
  for (idx s = 0; s < sp.nsup; ++s) {
    const int f = sp.sn_first[s], w = sp.sn_first[s + 1] - f, nr = sp.sn_nrows[s];
    const int* R = sp.sn_rows.data() + sp.sn_rows_ptr[s];
    for (int k = 0; k < w; ++k) {
      const double* col = panel.data() + sp.sn_off[s] + static_cast<idx>(k) * nr;
      y[f + k] /= col[k];
      for (int q = k + 1; q < nr; ++q) y[R[q]] -= col[q] * y[f + k];
    }
  }
  for (idx s = sp.nsup - 1; s >= 0; --s) {
    const int f = sp.sn_first[s], w = sp.sn_first[s + 1] - f, nr = sp.sn_nrows[s];
    const int* R = sp.sn_rows.data() + sp.sn_rows_ptr[s];
    for (int k = w - 1; k >= 0; --k) {
      const double* col = panel.data() + sp.sn_off[s] + static_cast<idx>(k) * nr;
      double acc = y[f + k];
      for (int q = k + 1; q < nr; ++q) acc -= col[q] * y[R[q]];
      y[f + k] = acc / col[k];
    }
  }
  std::vector<double> qref(mc, 0.0);
  for (idx j = 0; j < kp.nx; ++j) {
    for (idx q = kp.j.cp[j]; q < kp.j.cp[j + 1]; ++q) qref[kp.j.ri[q]] += jv[q] * y[sp.iperm[j]];
  }
  // emulation
  std::vector<double> vals(P.src.size());
  for (std::size_t e = 0; e < P.src.size(); ++e) {
    const int s = P.src[e];
    vals[e] = s == HYKKT_SRC_ZERO ? 0.0 : s < 0 ? jv[-2 - s] : ((s & 1) ? 1.0 / panel[s >> 1] : panel[s >> 1]);
  }
  std::vector<double> v(n, 0.0), part(P.pmax, 0.0), q(mc, 0.0);
  const long long capv = static_cast<long long>(P.nvchunk - 1) << P.vchunk_lg;
  const long long capi = static_cast<long long>(P.nichunk - 1) << P.ichunk_lg;
  long long vb = 0, ib = 0, vlen = 0, ilen = 0;
  auto V = [&](long long e) {
    if (e < 0 || e >= vlen) throw InvalidArgument("sys plan selfcheck: value entry outside the step");
    return vals[vb + e];
  };
  auto I = [&](long long e) {
    if (e < 0 || e >= ilen) throw InvalidArgument("sys plan selfcheck: index entry outside the step");
    return P.idx[ib + e];
  };
  auto slot = [&](int g) -> double& {
    if (g < 0 || g >= P.pmax) throw InvalidArgument("sys plan selfcheck: partial slot out of range");
    return part[g];
  };
  for (int b = 0; b < 4; ++b) {
    vb = P.blk[b].v0;
    ib = P.blk[b].i0;
    for (int sidx = P.blk[b].s0; sidx < P.blk[b].s1; ++sidx) {
      ilen = P.idx[ib + 1];
      vlen = P.idx[ib + 2];
      if (ilen > capi || vlen > capv) throw InvalidArgument("sys plan selfcheck: step wider than a ring");
      const int kind = I(0);
      if (kind == HYKKT_STEP_JT || kind == HYKKT_STEP_J) {
        const int nr = I(3), r0 = I(4);
        for (int j = 0; j < nr; ++j) {
          double acc = 0.0;
          for (int e = I(HYKKT_SP_HDR + j); e < I(HYKKT_SP_HDR + j + 1); ++e) {
            const int ix = I(HYKKT_SP_HDR + nr + 1 + e);
            acc += V(e) * (kind == HYKKT_STEP_JT ? u[ix] : v[ix]);
          }
          if (kind == HYKKT_STEP_JT) v[r0 + j] = acc;
          else q[r0 + j] = acc;
        }
      } else {
        const bool bwd = kind == HYKKT_STEP_BWD;
        const int nseg = I(3), nw = I(4), nt = I(5);
        for (int g = 0; g < nseg; ++g) {
          const int d = HYKKT_SP_HDR + HYKKT_SP_SEG_INTS * g;
          const int voff = I(d), ioff = I(d + 1), len = I(d + 2) & 0xffff, sl = I(d + 2) >> 16;
          double acc = 0.0;
          for (int e = 0; e < len; ++e) acc += V(voff + e) * v[I(ioff + e)];
          slot(sl) = acc;
        }
        for (int t = 0; t < nw + nt; ++t) {
          const int d = HYKKT_SP_HDR + HYKKT_SP_SEG_INTS * nseg + HYKKT_SP_TASK_INTS * t;
          const int voff = I(d), ioff = I(d + 1), f = I(d + 2), w = I(d + 3) & 0xffff, mode = I(d + 3) >> 16;
          if ((t < nw) != (w > thread_task_w())) throw InvalidArgument("sys plan selfcheck: task kind mismatch");
          const bool inl = mode == HYKKT_TASK_INLINE;
          if (!bwd) {
            long long e = voff + w * (w + 1) / 2;
            long long ig = ioff + w + 1;
            for (int r = 0; r < w; ++r) {
              const long long rowo = voff + static_cast<long long>(r) * (r + 1) / 2;
              double acc = v[f + r];
              if (inl) {
                const int c = I(ioff + r);
                for (int k = 0; k < c; ++k) acc -= V(e + k) * v[I(ig + k)];
                e += c;
                ig += c;
              } else {
                for (int g = I(ioff + r); g < I(ioff + r + 1); ++g) acc -= slot(g);
              }
              for (int j = 0; j < r; ++j) acc -= V(rowo + j) * v[f + j];
              v[f + r] = acc * V(rowo + r);
            }
          } else {
            std::vector<double> s(w, 0.0);
            if (inl) {
              const int nb = I(ioff);
              const long long e = voff + w * (w + 1) / 2;
              for (int r = 0; r < nb; ++r) {
                const double x = v[I(ioff + 1 + r)];
                for (int k = 0; k < w; ++k) s[k] += V(e + static_cast<long long>(r) * w + k) * x;
              }
            } else {
              for (int k = 0; k < w; ++k) {
                for (int g = I(ioff + k); g < I(ioff + k + 1); ++g) s[k] += slot(g);
              }
            }
            for (int k = w - 1; k >= 0; --k) {
              const long long cs = voff + static_cast<long long>(k) * w - static_cast<long long>(k) * (k - 1) / 2;
              double acc = v[f + k] - s[k];
              for (int j = k + 1; j < w; ++j) acc -= V(cs + j - k) * v[f + j];
              v[f + k] = acc * V(cs);
            }
          }
        }
      }
      vb += vlen;
      ib += ilen;
    }
    if (vb != P.blk[b].v1 || ib != P.blk[b].i1) throw InvalidArgument("sys plan selfcheck: block extents mismatch");
  }
  double num = 0.0, den = 0.0;
  for (idx i = 0; i < n; ++i) {
    num = std::max(num, std::abs(v[i] - y[i]));
    den = std::max(den, std::abs(y[i]));
  }
  double numq = 0.0, denq = 0.0;
  for (idx k = 0; k < mc; ++k) {
    numq = std::max(numq, std::abs(q[k] - qref[k]));
    denq = std::max(denq, std::abs(qref[k]));
  }
  return std::max(den > 0 ? num / den : num, denq > 0 ? numq / denq : numq);
}

}  // namespace hykkt
