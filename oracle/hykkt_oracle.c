/*
 * ORACLE / TEST INFRASTRUCTURE ONLY — never linked into the product.
 *
 * Plain-C restatement of the reference HyKKT path (/root/reference/proj),
 * written to reproduce the reference's floating-point operation ORDER so that
 * its outputs are bit-identical to the compiled reference (oracle/_ref) on
 * the same inputs and ordering; tests/test_oracle.py pins that.  Each function
 * names the reference code it restates.  Index type int64 like the reference
 * (csc_matrix.hpp:25).  Compiled with -ffp-contract=off (the reference is
 * built without -march, so it has no FMA contraction either).
 *
 * Parity status: PINNED — checked against the compiled reference itself
 * (bit-exact) and against the reference's known-answer tests restated in
 * tests/test_oracle.py.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef int64_t ix;

typedef struct {
  ix nrows, ncols;
  ix* cp;
  ix* ri;
  double* v;
} Csc;

static void* xcalloc(size_t n, size_t sz) {
  void* p = calloc(n ? n : 1, sz);
  if (!p) abort();
  return p;
}

static void csc_free(Csc* m) {
  free(m->cp);
  free(m->ri);
  free(m->v);
  memset(m, 0, sizeof(*m));
}

static int cmp_ix(const void* a, const void* b) {
  const ix x = *(const ix*)a, y = *(const ix*)b;
  return (x > y) - (x < y);
}

/* lower(A^T diag(d) A) on the full structural product pattern, k ascending
 * within each output slot: ata_lower (csc_matrix.cpp:352-393). */
static Csc ata_lower_c(const Csc* a, const double* d) {
  const ix n = a->ncols, m = a->nrows;
  /* transpose of a (rows as columns), values kept */
  ix* tcp = xcalloc(m + 1, sizeof(ix));
  ix* tri = xcalloc(a->cp[n], sizeof(ix));
  double* tv = xcalloc(a->cp[n], sizeof(double));
  for (ix p = 0; p < a->cp[n]; ++p) tcp[a->ri[p] + 1]++;
  for (ix i = 0; i < m; ++i) tcp[i + 1] += tcp[i];
  ix* next = xcalloc(m + 1, sizeof(ix));
  memcpy(next, tcp, m * sizeof(ix));
  for (ix j = 0; j < n; ++j)
    for (ix p = a->cp[j]; p < a->cp[j + 1]; ++p) {
      const ix q = next[a->ri[p]]++;
      tri[q] = j;
      tv[q] = a->v[p];
    }
  free(next);
  ix* mark = xcalloc(n, sizeof(ix));
  for (ix i = 0; i < n; ++i) mark[i] = -1;
  double* work = xcalloc(n, sizeof(double));
  ix* rows = xcalloc(n, sizeof(ix));
  ix cap = 16, nnz = 0;
  Csc out = {n, n, xcalloc(n + 1, sizeof(ix)), xcalloc(cap, sizeof(ix)), xcalloc(cap, sizeof(double))};
  for (ix j = 0; j < n; ++j) {
    ix nr = 0;
    for (ix p = a->cp[j]; p < a->cp[j + 1]; ++p) {
      const ix k = a->ri[p];
      const double w = (d ? d[k] : 1.0) * a->v[p];
      for (ix q = tcp[k]; q < tcp[k + 1]; ++q) {
        const ix i = tri[q];
        if (i < j) continue;
        if (mark[i] != j) {
          mark[i] = j;
          work[i] = 0.0;
          rows[nr++] = i;
        }
        work[i] += w * tv[q];
      }
    }
    qsort(rows, nr, sizeof(ix), cmp_ix);
    if (nnz + nr > cap) {
      while (nnz + nr > cap) cap *= 2;
      out.ri = realloc(out.ri, cap * sizeof(ix));
      out.v = realloc(out.v, cap * sizeof(double));
    }
    for (ix t = 0; t < nr; ++t) {
      out.ri[nnz] = rows[t];
      out.v[nnz++] = work[rows[t]];
    }
    out.cp[j + 1] = nnz;
  }
  free(tcp);
  free(tri);
  free(tv);
  free(mark);
  free(work);
  free(rows);
  return out;
}

/* sum_t coeff[t] * term[t] + diag(dg), union pattern with a full diagonal:
 * add_symmetric_lower (csc_matrix.cpp:293-350). */
static Csc add_sym_lower_c(const Csc* const* terms, const double* coeffs, int nt, const double* dg, ix n) {
  ix* mark = xcalloc(n, sizeof(ix));
  for (ix i = 0; i < n; ++i) mark[i] = -1;
  double* work = xcalloc(n, sizeof(double));
  ix* rows = xcalloc(n, sizeof(ix));
  ix cap = 16, nnz = 0;
  Csc out = {n, n, xcalloc(n + 1, sizeof(ix)), xcalloc(cap, sizeof(ix)), xcalloc(cap, sizeof(double))};
  for (ix j = 0; j < n; ++j) {
    ix nr = 0;
    mark[j] = j;
    work[j] = dg ? dg[j] : 0.0;
    rows[nr++] = j;
    for (int t = 0; t < nt; ++t) {
      const Csc* m = terms[t];
      for (ix p = m->cp[j]; p < m->cp[j + 1]; ++p) {
        const ix i = m->ri[p];
        if (mark[i] != j) {
          mark[i] = j;
          work[i] = 0.0;
          rows[nr++] = i;
        }
        work[i] += coeffs[t] * m->v[p];
      }
    }
    qsort(rows, nr, sizeof(ix), cmp_ix);
    if (nnz + nr > cap) {
      while (nnz + nr > cap) cap *= 2;
      out.ri = realloc(out.ri, cap * sizeof(ix));
      out.v = realloc(out.v, cap * sizeof(double));
    }
    for (ix t = 0; t < nr; ++t) {
      out.ri[nnz] = rows[t];
      out.v[nnz++] = work[rows[t]];
    }
    out.cp[j + 1] = nnz;
  }
  free(mark);
  free(work);
  free(rows);
  return out;
}

/* y = A x (scatter) or A^T x (gather): spmv (csc_matrix.cpp:236-263). */
static void spmv_c(const Csc* a, const double* x, int transpose, double* y) {
  if (!transpose) {
    for (ix i = 0; i < a->nrows; ++i) y[i] = 0.0;
    for (ix j = 0; j < a->ncols; ++j) {
      const double xj = x[j];
      if (xj == 0.0) continue;
      for (ix p = a->cp[j]; p < a->cp[j + 1]; ++p) y[a->ri[p]] += a->v[p] * xj;
    }
  } else {
    for (ix j = 0; j < a->ncols; ++j) {
      double acc = 0.0;
      for (ix p = a->cp[j]; p < a->cp[j + 1]; ++p) acc += a->v[p] * x[a->ri[p]];
      y[j] = acc;
    }
  }
}

typedef struct {
  ix n;
  ix* perm;
  ix* iperm;
  ix* parent;
  ix* lcp;
  ix* lri;
} Symbolic;

/* etree + column counts + L pattern of P A P^T under a given ordering:
 * symbolic_cholesky (symbolic.cpp:26-119). */
static Symbolic symbolic_c(const Csc* a, const ix* perm) {
  const ix n = a->ncols;
  Symbolic s = {n, xcalloc(n, sizeof(ix)), xcalloc(n, sizeof(ix)), xcalloc(n, sizeof(ix)), xcalloc(n + 1, sizeof(ix)), 0};
  for (ix i = 0; i < n; ++i) {
    s.perm[i] = perm[i];
    s.iperm[perm[i]] = i;
  }
  /* upper pattern by column: rows r < c (both triangles of the input) */
  ix* ucp = xcalloc(n + 1, sizeof(ix));
  for (ix j = 0; j < n; ++j)
    for (ix p = a->cp[j]; p < a->cp[j + 1]; ++p) {
      const ix r = s.iperm[a->ri[p]], c = s.iperm[j];
      if (r != c) ucp[(r > c ? r : c) + 1]++;
    }
  for (ix i = 0; i < n; ++i) ucp[i + 1] += ucp[i];
  ix* uri = xcalloc(ucp[n], sizeof(ix));
  ix* fill = xcalloc(n + 1, sizeof(ix));
  memcpy(fill, ucp, n * sizeof(ix));
  for (ix j = 0; j < n; ++j)
    for (ix p = a->cp[j]; p < a->cp[j + 1]; ++p) {
      const ix r = s.iperm[a->ri[p]], c = s.iperm[j];
      if (r != c) uri[fill[r > c ? r : c]++] = r < c ? r : c;
    }
  ix* anc = xcalloc(n, sizeof(ix));
  for (ix k = 0; k < n; ++k) {
    s.parent[k] = -1;
    anc[k] = -1;
  }
  for (ix k = 0; k < n; ++k)
    for (ix p = ucp[k]; p < ucp[k + 1]; ++p) {
      ix i = uri[p];
      while (i != -1 && i < k) {
        const ix nx = anc[i];
        anc[i] = k;
        if (nx == -1) s.parent[i] = k;
        i = nx;
      }
    }
  ix* cnt = xcalloc(n, sizeof(ix));
  ix* stamp = xcalloc(n, sizeof(ix));
  for (ix k = 0; k < n; ++k) {
    cnt[k] = 1;
    stamp[k] = -1;
  }
  for (ix k = 0; k < n; ++k) {
    stamp[k] = k;
    for (ix p = ucp[k]; p < ucp[k + 1]; ++p)
      for (ix i = uri[p]; i < k && stamp[i] != k; i = s.parent[i]) {
        cnt[i]++;
        stamp[i] = k;
      }
  }
  for (ix k = 0; k < n; ++k) s.lcp[k + 1] = s.lcp[k] + cnt[k];
  s.lri = xcalloc(s.lcp[n], sizeof(ix));
  ix* cur = xcalloc(n + 1, sizeof(ix));
  memcpy(cur, s.lcp, n * sizeof(ix));
  for (ix k = 0; k < n; ++k) stamp[k] = -1;
  for (ix k = 0; k < n; ++k) {
    s.lri[cur[k]++] = k;
    stamp[k] = k;
    for (ix p = ucp[k]; p < ucp[k + 1]; ++p)
      for (ix i = uri[p]; i < k && stamp[i] != k; i = s.parent[i]) {
        s.lri[cur[i]++] = k;
        stamp[i] = k;
      }
  }
  free(ucp);
  free(uri);
  free(fill);
  free(anc);
  free(cnt);
  free(stamp);
  free(cur);
  return s;
}

static void symbolic_free(Symbolic* s) {
  free(s->perm);
  free(s->iperm);
  free(s->parent);
  free(s->lcp);
  free(s->lri);
}

/* Left-looking simplicial Cholesky with column link lists:
 * numeric_cholesky (cholesky.cpp:32-137).  Returns the failing column or -1. */
static ix numeric_c(const Csc* a, const Symbolic* s, double floor_in, double* lv, double* fail_pivot) {
  const ix n = s->n;
  /* permuted lower, unsorted (permute_lower, cholesky.cpp:32-61) */
  ix* bcp = xcalloc(n + 1, sizeof(ix));
  for (ix j = 0; j < n; ++j)
    for (ix p = a->cp[j]; p < a->cp[j + 1]; ++p) {
      const ix r = s->iperm[a->ri[p]], c = s->iperm[j];
      bcp[(r < c ? r : c) + 1]++;
    }
  for (ix i = 0; i < n; ++i) bcp[i + 1] += bcp[i];
  ix* bri = xcalloc(bcp[n], sizeof(ix));
  double* bv = xcalloc(bcp[n], sizeof(double));
  ix* nxt = xcalloc(n + 1, sizeof(ix));
  memcpy(nxt, bcp, n * sizeof(ix));
  for (ix j = 0; j < n; ++j)
    for (ix p = a->cp[j]; p < a->cp[j + 1]; ++p) {
      const ix r = s->iperm[a->ri[p]], c = s->iperm[j];
      const ix q = nxt[r < c ? r : c]++;
      bri[q] = r > c ? r : c;
      bv[q] = a->v[p];
    }
  const ix* lp = s->lcp;
  const ix* li = s->lri;
  ix* head = xcalloc(n, sizeof(ix));
  ix* lnext = xcalloc(n, sizeof(ix));
  ix* pos = xcalloc(n, sizeof(ix));
  double* x = xcalloc(n, sizeof(double));
  for (ix i = 0; i < n; ++i) head[i] = lnext[i] = -1;
  for (ix p = 0; p < lp[n]; ++p) lv[p] = 0.0;
  const double fl = floor_in > 0.0 ? floor_in : 0.0;
  ix failed = -1;
  for (ix k = 0; k < n && failed < 0; ++k) {
    for (ix p = bcp[k]; p < bcp[k + 1]; ++p) x[bri[p]] += bv[p];
    for (ix j = head[k]; j != -1;) {
      const ix jn = lnext[j];
      const double lkj = lv[pos[j]];
      for (ix p = pos[j]; p < lp[j + 1]; ++p) x[li[p]] -= lv[p] * lkj;
      if (++pos[j] < lp[j + 1]) {
        const ix r = li[pos[j]];
        lnext[j] = head[r];
        head[r] = j;
      }
      j = jn;
    }
    const double pivot = x[k];
    if (!(pivot > fl)) {
      failed = k;
      if (fail_pivot) *fail_pivot = pivot;
      break;
    }
    const double dk = sqrt(pivot);
    lv[lp[k]] = dk;
    x[k] = 0.0;
    for (ix p = lp[k] + 1; p < lp[k + 1]; ++p) {
      lv[p] = x[li[p]] / dk;
      x[li[p]] = 0.0;
    }
    pos[k] = lp[k] + 1;
    if (pos[k] < lp[k + 1]) {
      const ix r = li[pos[k]];
      lnext[k] = head[r];
      head[r] = k;
    }
  }
  free(bcp);
  free(bri);
  free(bv);
  free(nxt);
  free(head);
  free(lnext);
  free(pos);
  free(x);
  return failed;
}

/* factor_solve (cholesky.cpp:139-168). */
static void factor_solve_c(const Symbolic* s, const double* lv, const double* b, double* out) {
  const ix n = s->n;
  double* w = xcalloc(n, sizeof(double));
  for (ix r = 0; r < n; ++r) w[r] = b[s->perm[r]];
  for (ix j = 0; j < n; ++j) {
    w[j] /= lv[s->lcp[j]];
    const double wj = w[j];
    for (ix p = s->lcp[j] + 1; p < s->lcp[j + 1]; ++p) w[s->lri[p]] -= lv[p] * wj;
  }
  for (ix j = n - 1; j >= 0; --j) {
    double acc = w[j];
    for (ix p = s->lcp[j] + 1; p < s->lcp[j + 1]; ++p) acc -= lv[p] * w[s->lri[p]];
    w[j] = acc / lv[s->lcp[j]];
  }
  for (ix r = 0; r < n; ++r) out[s->perm[r]] = w[r];
  free(w);
}

static double norm2_c(const double* v, ix n) {
  double acc = 0.0;
  for (ix i = 0; i < n; ++i) acc += v[i] * v[i];
  return sqrt(acc);
}

typedef struct {
  double gamma, delta_min, delta_max, delta2, cg_tol;
  int64_t cg_max_iter;
  double small_quadratic_threshold, pivot_floor, ruiz_tol;
  int64_t ruiz_max_iters;
} OConfig;

typedef struct {
  int32_t status;
  int32_t pad;
  double delta1_final, delta2_used;
  int64_t cg_iterations, factorization_attempts, ruiz_iterations;
} OReport;

/* S p = J H^-1 J^T p + delta2 p: SchurOperator::apply (solver.cpp:144-152). */
static void schur_apply(const Symbolic* s, const double* lv, const Csc* j, double d2, const double* v, double* out,
                        double* t1, double* t2) {
  spmv_c(j, v, 1, t1);
  factor_solve_c(s, lv, t1, t2);
  spmv_c(j, t2, 0, out);
  if (d2 != 0.0)
    for (ix i = 0; i < j->nrows; ++i) out[i] += d2 * v[i];
}

/* cg_schur (solver.cpp:154-201): flags bit0 converged, bit1 small quadratic. */
static int cg_c(const Symbolic* s, const double* lv, const Csc* j, double d2, const double* rhs, const OConfig* cfg,
                double* x, int64_t* iters, double* relres) {
  const ix m = j->nrows, n = j->ncols;
  for (ix i = 0; i < m; ++i) x[i] = 0.0;
  *iters = 0;
  *relres = 0.0;
  const double rn = norm2_c(rhs, m);
  if (rn == 0.0) return 1;
  double* r = xcalloc(m, sizeof(double));
  double* p = xcalloc(m, sizeof(double));
  double* q = xcalloc(m, sizeof(double));
  double* t1 = xcalloc(n, sizeof(double));
  double* t2 = xcalloc(n, sizeof(double));
  memcpy(r, rhs, m * sizeof(double));
  memcpy(p, rhs, m * sizeof(double));
  double rho = rn * rn;
  int flags = 0;
  for (int64_t it = 1; it <= cfg->cg_max_iter; ++it) {
    schur_apply(s, lv, j, d2, p, q, t1, t2);
    double curv = 0.0, pn2 = 0.0;
    for (ix i = 0; i < m; ++i) {
      curv += p[i] * q[i];
      pn2 += p[i] * p[i];
    }
    if (curv <= cfg->small_quadratic_threshold * pn2) {
      *relres = norm2_c(r, m) / rn;
      flags = 2;
      goto done;
    }
    const double alpha = rho / curv;
    for (ix i = 0; i < m; ++i) {
      x[i] += alpha * p[i];
      r[i] -= alpha * q[i];
    }
    *iters = it;
    const double rnorm = norm2_c(r, m);
    *relres = rnorm / rn;
    if (*relres <= cfg->cg_tol) {
      flags = 1;
      goto done;
    }
    const double rho_next = rnorm * rnorm;
    const double beta = rho_next / rho;
    rho = rho_next;
    for (ix i = 0; i < m; ++i) p[i] = r[i] + beta * p[i];
  }
done:
  free(r);
  free(p);
  free(q);
  free(t1);
  free(t2);
  return flags;
}

static Csc csc_view(ix nr, ix nc, const ix* cp, const ix* ri, const double* v) {
  Csc m = {nr, nc, (ix*)cp, (ix*)ri, (double*)v};
  return m;
}

static Csc csc_with_values(const Csc* pat, const double* v) {
  Csc m = {pat->nrows, pat->ncols, xcalloc(pat->ncols + 1, sizeof(ix)), xcalloc(pat->cp[pat->ncols], sizeof(ix)),
           xcalloc(pat->cp[pat->ncols], sizeof(double))};
  memcpy(m.cp, pat->cp, (pat->ncols + 1) * sizeof(ix));
  memcpy(m.ri, pat->ri, pat->cp[pat->ncols] * sizeof(ix));
  memcpy(m.v, v, pat->cp[pat->ncols] * sizeof(double));
  return m;
}

/*
 * solve_full (solver.cpp:295-328) = reduce (kkt_system.cpp:66-87) ->
 * ruiz_scale (ruiz.cpp:76-116) -> solve_reduced (solver.cpp:222-293: assemble
 * (66-84), ladder (108-142), w, CG (+delta2), dx) -> unscale (ruiz.cpp:118-133)
 * -> recover (kkt_system.cpp:89-105), with the symbolic factor built from the
 * given ordering.  *dmin_inout carries RegularizationState::delta_min_current.
 */
int oracle_solve_full(ix nx, ix mc, ix md, const ix* hcp, const ix* hri, const double* hv, const ix* jcp, const ix* jri,
                      const double* jv, const ix* jdcp, const ix* jdri, const double* jdv, const double* d_x,
                      const double* d_s, const double* rtx, const double* r_s, const double* r_y, const double* r_yd,
                      const ix* perm, const OConfig* cfg, double* dmin_inout, OReport* rep, double* dx, double* ds,
                      double* dy, double* dyd) {
  memset(rep, 0, sizeof(*rep));
  const Csc H = csc_view(nx, nx, hcp, hri, hv), J = csc_view(mc, nx, jcp, jri, jv), JD = csc_view(md, nx, jdcp, jdri, jdv);
  /* reduce */
  Csc jdtj = ata_lower_c(&JD, d_s);
  const Csc* t1[2] = {&H, &jdtj};
  const double c1[2] = {1.0, 1.0};
  Csc ht = add_sym_lower_c(t1, c1, 2, d_x, nx);
  double* rx = xcalloc(nx, sizeof(double));
  double* tt = xcalloc(md, sizeof(double));
  for (ix i = 0; i < md; ++i) tt[i] = d_s[i] * r_yd[i] + r_s[i];
  spmv_c(&JD, tt, 1, rx);
  for (ix i = 0; i < nx; ++i) rx[i] += rtx[i];
  /* ruiz */
  const ix nt = nx + mc;
  double* d = xcalloc(nt, sizeof(double));
  double* nrm = xcalloc(nt, sizeof(double));
  for (ix i = 0; i < nt; ++i) d[i] = 1.0;
  int64_t sweeps = 0;
  for (int64_t it = 1; it <= cfg->ruiz_max_iters; ++it) {
    sweeps = it;
    for (ix i = 0; i < nt; ++i) nrm[i] = 0.0;
    for (ix c = 0; c < nx; ++c)
      for (ix p = ht.cp[c]; p < ht.cp[c + 1]; ++p) {
        const ix i = ht.ri[p];
        const double v = fabs(ht.v[p]) * d[i] * d[c];
        if (v > nrm[i]) nrm[i] = v;
        if (i != c && v > nrm[c]) nrm[c] = v;
      }
    for (ix c = 0; c < nx; ++c)
      for (ix p = J.cp[c]; p < J.cp[c + 1]; ++p) {
        const ix k = J.ri[p];
        const double v = fabs(J.v[p]) * d[nx + k] * d[c];
        if (v > nrm[nx + k]) nrm[nx + k] = v;
        if (v > nrm[c]) nrm[c] = v;
      }
    int conv = 1;
    for (ix i = 0; i < nt; ++i)
      if (nrm[i] > 0.0 && fabs(nrm[i] - 1.0) > cfg->ruiz_tol) {
        conv = 0;
        break;
      }
    if (conv) break;
    for (ix i = 0; i < nt; ++i)
      if (nrm[i] > 0.0) d[i] /= sqrt(nrm[i]);
  }
  rep->ruiz_iterations = sweeps;
  Csc hts = csc_with_values(&ht, ht.v);
  for (ix c = 0; c < nx; ++c)
    for (ix p = hts.cp[c]; p < hts.cp[c + 1]; ++p) hts.v[p] *= d[hts.ri[p]] * d[c];
  Csc js = csc_with_values(&J, J.v);
  for (ix c = 0; c < nx; ++c)
    for (ix p = js.cp[c]; p < js.cp[c + 1]; ++p) js.v[p] *= d[nx + js.ri[p]] * d[c];
  double* rxs = xcalloc(nx, sizeof(double));
  double* rys = xcalloc(mc, sizeof(double));
  for (ix i = 0; i < nx; ++i) rxs[i] = d[i] * rx[i];
  for (ix k = 0; k < mc; ++k) rys[k] = d[nx + k] * r_y[k];
  /* assemble H_gamma */
  Csc jtj = ata_lower_c(&js, NULL);
  const Csc* t2[2] = {&hts, &jtj};
  const double c2[2] = {1.0, cfg->gamma};
  double* zero = xcalloc(nx, sizeof(double));
  Csc hg = add_sym_lower_c(t2, c2, 2, zero, nx);
  double* rhat = xcalloc(nx, sizeof(double));
  spmv_c(&js, rys, 1, rhat);
  for (ix i = 0; i < nx; ++i) rhat[i] = rxs[i] + cfg->gamma * rhat[i];
  /* ladder */
  Symbolic sym = symbolic_c(&hg, perm);
  double maxd = 0.0;
  for (ix c = 0; c < nx; ++c)
    for (ix p = hg.cp[c]; p < hg.cp[c + 1]; ++p)
      if (hg.ri[p] == c) {
        if (fabs(hg.v[p]) > maxd) maxd = fabs(hg.v[p]);
        break;
      }
  const double floorv = cfg->pivot_floor * maxd;
  double* lv = xcalloc(sym.lcp[nx], sizeof(double));
  double dmin = (dmin_inout && *dmin_inout > 0.0) ? *dmin_inout : cfg->delta_min;
  double delta1 = 0.0;
  int64_t attempts = 0;
  Csc hd = csc_with_values(&hg, hg.v);
  ix failed;
  for (;;) {
    ++attempts;
    for (ix c = 0; c < nx; ++c)
      for (ix p = hg.cp[c]; p < hg.cp[c + 1]; ++p) hd.v[p] = (delta1 != 0.0 && hg.ri[p] == c) ? hg.v[p] + delta1 : hg.v[p];
    failed = numeric_c(&hd, &sym, floorv, lv, NULL);
    if (failed < 0 || !(delta1 <= cfg->delta_max / 2.0)) break;
    if (delta1 == 0.0) {
      delta1 = dmin;
    } else {
      dmin *= 2.0;
      delta1 = dmin;
    }
  }
  if (dmin_inout) *dmin_inout = dmin;
  rep->factorization_attempts = attempts;
  rep->delta1_final = delta1;
  int rc = 0;
  if (failed >= 0) {
    rep->status = 2;
  } else {
    double* w = xcalloc(nx, sizeof(double));
    factor_solve_c(&sym, lv, rhat, w);
    double* srhs = xcalloc(mc, sizeof(double));
    spmv_c(&js, w, 0, srhs);
    for (ix k = 0; k < mc; ++k) srhs[k] -= rys[k];
    double* y = xcalloc(mc, sizeof(double));
    int64_t its;
    double rr;
    int fl = cg_c(&sym, lv, &js, 0.0, srhs, cfg, y, &its, &rr);
    if (fl & 2) {
      fl = cg_c(&sym, lv, &js, cfg->delta2, srhs, cfg, y, &its, &rr);
      rep->delta2_used = cfg->delta2;
    }
    rep->cg_iterations = its;
    if (!(fl & 1)) {
      rep->status = 3;
    } else {
      rep->status = rep->delta2_used > 0.0 ? 1 : 0;
      double* rxx = xcalloc(nx, sizeof(double));
      spmv_c(&js, y, 1, rxx);
      for (ix i = 0; i < nx; ++i) rxx[i] = rhat[i] - rxx[i];
      double* xs = xcalloc(nx, sizeof(double));
      factor_solve_c(&sym, lv, rxx, xs);
      for (ix i = 0; i < nx; ++i) dx[i] = d[i] * xs[i];
      for (ix k = 0; k < mc; ++k) dy[k] = d[nx + k] * y[k];
      spmv_c(&JD, dx, 0, ds);
      for (ix i = 0; i < md; ++i) ds[i] -= r_yd[i];
      for (ix i = 0; i < md; ++i) dyd[i] = d_s[i] * ds[i] - r_s[i];
      free(rxx);
      free(xs);
    }
    free(w);
    free(srhs);
    free(y);
  }
  csc_free(&jdtj);
  csc_free(&ht);
  csc_free(&hts);
  csc_free(&js);
  csc_free(&jtj);
  csc_free(&hg);
  csc_free(&hd);
  symbolic_free(&sym);
  free(rx);
  free(tt);
  free(d);
  free(nrm);
  free(rxs);
  free(rys);
  free(zero);
  free(rhat);
  free(lv);
  return rc;
}

/* numeric_cholesky + factor_solve on an explicit lower matrix under `perm`;
 * returns the failing column (or -1) and writes L values (reference layout). */
ix oracle_cholesky(ix n, const ix* cp, const ix* ri, const double* v, const ix* perm, double floor_abs, ix* l_nnz,
                   double* lv_out, ix lv_cap, double* fail_pivot, const double* b, double* x) {
  const Csc A = csc_view(n, n, cp, ri, v);
  Symbolic s = symbolic_c(&A, perm);
  *l_nnz = s.lcp[n];
  double* lv = xcalloc(s.lcp[n], sizeof(double));
  const ix failed = numeric_c(&A, &s, floor_abs, lv, fail_pivot);
  if (lv_out && lv_cap >= s.lcp[n]) memcpy(lv_out, lv, s.lcp[n] * sizeof(double));
  if (failed < 0 && b && x) factor_solve_c(&s, lv, b, x);
  free(lv);
  symbolic_free(&s);
  return failed;
}
