// Batched HyKKT: B independent systems on one shared pattern (BASELINE
// configs[4]).  Lane = system: every value array is interleaved
// [entry][system] with a system stride Bp (B rounded up to 32; pad lanes
// replicate the last system), so a warp touching one entry for 32 systems
// issues one fully coalesced 256-byte access.  Tasks are (supernode, tile of
// 32 systems) warp tasks on the same level-sorted sync-free schedule as the
// single-system path; each lane runs the scalar algorithm for its system, so
// the per-hop latency of the elimination tree is amortised over 32 systems
// and the batch becomes bandwidth-bound.
//
// Arithmetic follows the single-system kernels (which restate the
// reference: kkt_system.cpp:66-105, ruiz.cpp:26-133, solver.cpp:66-201,
// cholesky.cpp:65-168) lane by lane; per-system outcomes (Ruiz sweeps, delta1
// ladder, CG iterations, small quadratic) are tracked per lane.
#pragma once

#include "kernels_assemble.cuh"
#include "kernels_solve.cuh"

namespace hykkt::dev {

struct BDims {
  int B;    // real systems
  int Bp;   // padded stride (a power of two >= 32: index splits are shifts / masks)
  int T;    // tiles = Bp / 32
};

__device__ __forceinline__ long long bidx(long long e, int Bp, int b) { return e * Bp + b; }

// Dynamic shared memory of the batched persistent kernels (8 warps x
// smem_rows x 32 doubles): per-warp accumulators of the lane-mode tasks, or
// one staging area for a wide (per-system) task.
extern __shared__ double bsmem[];

// Panel layout of the batch.  Lane-mode supernodes (the narrow bulk of the
// tree) interleave their panel [entry][system] (stride Bp, lane = system);
// wide-mode supernodes (every supernode whose subtree holds a wide panel:
// the top of the tree) store each system's panel contiguously inside the
// same region, [system][entry], so one CTA can stage one system's panel with
// coalesced loads.
__device__ __forceinline__ long long pan_addr(const SnPlan& s, const int* mode, int sn, int local, int Bp,
                                              int b) {
  const long long off = s.off[sn];
  if (mode[sn]) return off * Bp + (long long)b * (s.nrows[sn] * (s.first[sn + 1] - s.first[sn])) + local;
  return (off + local) * Bp + b;
}

// [system][entry] (field-major, B systems) -> [entry][system] (Bp stride).
__global__ void kb_interleave(const double* __restrict__ in, double* __restrict__ out, int n, int B,
                              int Bp) {
  __shared__ double tile[32][33];
  const int e0 = blockIdx.x * 32, b0 = blockIdx.y * 32;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // 32 x 8 threads
  for (int j = ty; j < 32; j += 8) {
    const int b = min(b0 + j, B - 1), e = e0 + tx;
    tile[j][tx] = e < n ? in[(long long)b * n + e] : 0.0;
  }
  __syncthreads();
  for (int j = ty; j < 32; j += 8) {
    const int e = e0 + j, b = b0 + tx;
    if (e < n) out[(long long)e * Bp + b] = tile[tx][j];
  }
}

// [entry][system] -> [system][entry] for the first B systems.
__global__ void kb_deinterleave(const double* __restrict__ in, double* __restrict__ out, int n, int B,
                                int Bp) {
  __shared__ double tile[32][33];
  const int e0 = blockIdx.x * 32, b0 = blockIdx.y * 32;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  for (int j = ty; j < 32; j += 8) {
    const int e = e0 + j;
    tile[j][tx] = e < n ? in[(long long)e * Bp + b0 + tx] : 0.0;
  }
  __syncthreads();
  for (int j = ty; j < 32; j += 8) {
    const int b = b0 + j, e = e0 + tx;
    if (b < B && e < n) out[(long long)b * n + e] = tile[tx][j];
  }
}

struct BVals {  // interleaved inputs
  const double *h, *j, *jd, *dx, *ds, *rtx, *rs, *ry, *ryd;
};

// ---- assembly ---------------------------------------------------------------
__global__ void kb_reduce(AsmPlan p, BDims bd, BVals v, double* __restrict__ ht, double* __restrict__ r_x) {
  const long long g = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  const int b = static_cast<int>(g & (bd.Bp - 1));
  const long long t = (g >> (__ffs(bd.Bp) - 1));
  const int Bp = bd.Bp;
  if (t < p.n_ht) {
    const int col = p.ht_col[t];
    double x = (p.ht_row[t] == col) ? v.dx[bidx(col, Bp, b)] : 0.0;
    const int hs = p.ht_hsrc[t];
    if (hs >= 0) x = __dadd_rn(x, v.h[bidx(hs, Bp, b)]);
    const int q0 = p.ht_pp[t], q1 = p.ht_pp[t + 1];
    if (q1 > q0) {
      double s = 0.0;
      for (int q = q0; q < q1; ++q) {
        s = __dadd_rn(s, __dmul_rn(__dmul_rn(v.ds[bidx(p.ht_pk[q], Bp, b)], v.jd[bidx(p.ht_pa[q], Bp, b)]),
                                   v.jd[bidx(p.ht_pb[q], Bp, b)]));
      }
      x = __dadd_rn(x, s);
    }
    ht[bidx(t, Bp, b)] = x;
  }
  if (t < p.nx) {
    double acc = 0.0;
    for (int q = p.jd_cp[t]; q < p.jd_cp[t + 1]; ++q) {
      const int k = p.jd_ri[q];
      const double tk = __dadd_rn(__dmul_rn(v.ds[bidx(k, Bp, b)], v.ryd[bidx(k, Bp, b)]), v.rs[bidx(k, Bp, b)]);
      acc = __dadd_rn(acc, __dmul_rn(v.jd[bidx(q, Bp, b)], tk));
    }
    r_x[bidx(t, Bp, b)] = __dadd_rn(acc, v.rtx[bidx(t, Bp, b)]);
  }
}

struct BRuizArgs {
  AsmPlan p;
  BDims bd;
  const double* ht;
  const double* jval;
  double* d;            // (n_x + m_c) x Bp
  double* norms;        // (n_x + m_c) x Bp
  int* unconverged;     // (max_iters + 1) x Bp, zeroed
  int* active_count;    // max_iters + 1, zeroed
  int* sweeps;          // Bp
  int max_iters;
  double tol;
  GridBarrier bar;
  int* abort;
};

// ruiz_scale (ruiz.cpp:76-116) for every system in lockstep; a system stops
// updating after the sweep at which its norms converge.
__global__ void kb_ruiz(BRuizArgs a) {
  const int Bp = a.bd.Bp;
  const long long nrow = (long long)(a.p.nx + a.p.mc) * Bp;
  const long long gt = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  const long long gs = (long long)gridDim.x * blockDim.x;
  for (long long i = gt; i < nrow; i += gs) a.d[i] = 1.0;
  for (long long b = gt; b < Bp; b += gs) a.sweeps[b] = a.max_iters;
  grid_sync(a.bar, a.abort);
  for (int it = 1; it <= a.max_iters; ++it) {
    const int* prev = a.unconverged + (it - 1) * Bp;  // row 0 is all-unconverged by convention
    for (long long i = gt; i < nrow; i += gs) a.norms[i] = 0.0;
    grid_sync(a.bar, a.abort);
    const long long nh = (long long)a.p.n_ht * Bp;
    for (long long g = gt; g < nh; g += gs) {
      const int b = static_cast<int>(g & (Bp - 1));
      if (it > 1 && !ldcg_int(prev + b)) continue;
      const long long t = (g >> (__ffs(Bp) - 1));
      const int i = a.p.ht_row[t], j = a.p.ht_col[t];
      const double v = __dmul_rn(__dmul_rn(fabs(a.ht[g]), ldcg(a.d + bidx(i, Bp, b))), ldcg(a.d + bidx(j, Bp, b)));
      atomic_max_nonneg(a.norms + bidx(i, Bp, b), v);
      if (i != j) atomic_max_nonneg(a.norms + bidx(j, Bp, b), v);
    }
    const long long nj = (long long)a.p.nnz_j * Bp;
    for (long long g = gt; g < nj; g += gs) {
      const int b = static_cast<int>(g & (Bp - 1));
      if (it > 1 && !ldcg_int(prev + b)) continue;
      const long long q = (g >> (__ffs(Bp) - 1));
      const int k = a.p.j_ri[q], j = a.p.j_col[q];
      const double v = __dmul_rn(__dmul_rn(fabs(a.jval[g]), ldcg(a.d + bidx(a.p.nx + k, Bp, b))),
                                 ldcg(a.d + bidx(j, Bp, b)));
      atomic_max_nonneg(a.norms + bidx(a.p.nx + k, Bp, b), v);
      atomic_max_nonneg(a.norms + bidx(j, Bp, b), v);
    }
    grid_sync(a.bar, a.abort);
    int* cur = a.unconverged + it * Bp;
    for (long long g = gt; g < nrow; g += gs) {
      const int b = static_cast<int>(g & (Bp - 1));
      if (it > 1 && !ldcg_int(prev + b)) continue;
      const double v = ldcg(a.norms + g);
      if (v > 0.0 && fabs(v - 1.0) > a.tol) atomicOr(cur + b, 1);
    }
    grid_sync(a.bar, a.abort);
    for (long long b = gt; b < Bp; b += gs) {
      const bool was_active = it == 1 || ldcg_int(prev + b);
      if (was_active && !ldcg_int(cur + b)) a.sweeps[b] = it;  // converged at this sweep
      if (ldcg_int(cur + b)) atomicAdd(a.active_count + it, 1);
    }
    for (long long g = gt; g < nrow; g += gs) {
      const int b = static_cast<int>(g & (Bp - 1));
      if (!ldcg_int(cur + b)) continue;
      const double v = ldcg(a.norms + g);
      if (v > 0.0) a.d[g] = __ddiv_rn(ldcg(a.d + g), __dsqrt_rn(v));
    }
    grid_sync(a.bar, a.abort);
    if (ldcg_int(a.active_count + it) == 0) break;
  }
}

// ruiz_scale (ruiz.cpp:76-116) for every system in lockstep, by ROW
// GATHERS instead of atomics: thread (row i, system b) — lanes are systems,
// so every load is coalesced over the interleaved layout — takes the max of
// the scaled magnitudes of row i of [[H_tilde, J^T], [J, 0]] from a host-built
// row list (rp / ent: value index, ht slot or n_ht + J entry, and the entry's
// stored row and column).  Each magnitude is formed exactly as kb_ruiz and
// the reference do ((|a| d_row) d_col), and max is order-free, so d and the
// sweep counts are bit-identical to kb_ruiz; two grid barriers per sweep.
struct BRuizRowsArgs {
  BRuizArgs r;
  const int* rp;    // n_x + m_c + 1
  const int4* ent;  // {value index, d row, d col, 0}
};

__global__ void kb_ruiz_rows(BRuizRowsArgs ar) {
  const BRuizArgs& a = ar.r;
  const int Bp = a.bd.Bp, nht = a.p.n_ht;
  const long long nrow = (long long)(a.p.nx + a.p.mc) * Bp;
  const long long gt = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  const long long gs = (long long)gridDim.x * blockDim.x;
  for (long long i = gt; i < nrow; i += gs) a.d[i] = 1.0;
  for (long long b = gt; b < Bp; b += gs) a.sweeps[b] = a.max_iters;
  grid_sync(a.bar, a.abort);
  for (int it = 1; it <= a.max_iters; ++it) {
    const int* prev = a.unconverged + (it - 1) * Bp;
    int* cur = a.unconverged + it * Bp;
    for (long long g = gt; g < nrow; g += gs) {
      const int b = static_cast<int>(g & (Bp - 1));
      if (it > 1 && !ldcg_int(prev + b)) continue;
      const int i = static_cast<int>((g >> (__ffs(Bp) - 1)));
      double nm = 0.0;
      for (int e = __ldg(ar.rp + i), e1 = __ldg(ar.rp + i + 1); e < e1; ++e) {
        const int4 q = __ldg(ar.ent + e);
        const double av = q.x < nht ? a.ht[bidx(q.x, Bp, b)] : a.jval[bidx(q.x - nht, Bp, b)];
        nm = fmax(nm, __dmul_rn(__dmul_rn(fabs(av), ldcg(a.d + bidx(q.y, Bp, b))), ldcg(a.d + bidx(q.z, Bp, b))));
      }
      a.norms[g] = nm;
      if (nm > 0.0 && fabs(nm - 1.0) > a.tol) cur[b] = 1;
    }
    grid_sync(a.bar, a.abort);
    for (long long b = gt; b < Bp; b += gs) {
      const bool was_active = it == 1 || ldcg_int(prev + b);
      if (was_active && !ldcg_int(cur + b)) a.sweeps[b] = it;
      if (ldcg_int(cur + b)) atomicAdd(a.active_count + it, 1);
    }
    for (long long g = gt; g < nrow; g += gs) {
      const int b = static_cast<int>(g & (Bp - 1));
      if (!ldcg_int(cur + b)) continue;
      const double v = ldcg(a.norms + g);
      if (v > 0.0) a.d[g] = __ddiv_rn(ldcg(a.d + g), __dsqrt_rn(v));
    }
    grid_sync(a.bar, a.abort);
    if (ldcg_int(a.active_count + it) == 0) break;
  }
}

__global__ void kb_scale(AsmPlan p, BDims bd, const double* __restrict__ d, const double* __restrict__ ht,
                         const double* __restrict__ jval, const double* __restrict__ r_x,
                         const double* __restrict__ r_y, double* __restrict__ hts, double* __restrict__ js,
                         double* __restrict__ js_csr, double* __restrict__ rxs, double* __restrict__ rys) {
  const long long g = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  const int Bp = bd.Bp, b = static_cast<int>(g & (Bp - 1));
  const long long t = (g >> (__ffs(Bp) - 1));
  if (t < p.n_ht) hts[g] = __dmul_rn(ht[g], __dmul_rn(d[bidx(p.ht_row[t], Bp, b)], d[bidx(p.ht_col[t], Bp, b)]));
  if (t < p.nnz_j) {
    js[g] = __dmul_rn(jval[g], __dmul_rn(d[bidx(p.nx + p.j_ri[t], Bp, b)], d[bidx(p.j_col[t], Bp, b)]));
    const int s = p.jcsr_src[t];
    js_csr[g] = __dmul_rn(jval[bidx(s, Bp, b)], __dmul_rn(d[bidx(p.nx + p.j_ri[s], Bp, b)], d[bidx(p.j_col[s], Bp, b)]));
  }
  if (t < p.nx) rxs[g] = __dmul_rn(d[g], r_x[g]);
  if (t < p.mc) rys[g] = __dmul_rn(d[bidx(p.nx + t, Bp, b)], r_y[g]);
}

__global__ void kb_hgamma(AsmPlan p, BDims bd, double gamma, const double* __restrict__ hts,
                          const double* __restrict__ js, const double* __restrict__ rxs,
                          const double* __restrict__ rys, double* __restrict__ hg, double* __restrict__ rhat,
                          double* __restrict__ maxdiag) {
  const long long g = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  const int Bp = bd.Bp, b = static_cast<int>(g & (Bp - 1));
  const long long t = (g >> (__ffs(Bp) - 1));
  if (t < p.n_hg) {
    const int src = p.hg_src[t];
    double v = (src >= 0) ? __dadd_rn(0.0, hts[bidx(src, Bp, b)]) : 0.0;
    const int q0 = p.hg_pp[t], q1 = p.hg_pp[t + 1];
    if (q1 > q0) {
      double s = 0.0;
      for (int q = q0; q < q1; ++q) s = __dadd_rn(s, __dmul_rn(js[bidx(p.hg_pa[q], Bp, b)], js[bidx(p.hg_pb[q], Bp, b)]));
      v = __dadd_rn(v, __dmul_rn(gamma, s));
    }
    hg[g] = v;
    if (p.hg_row[t] == p.hg_col[t]) atomic_max_nonneg(maxdiag + b, fabs(v));
  }
  if (t < p.nx) {
    double acc = 0.0;
    for (int q = p.j_cp[t]; q < p.j_cp[t + 1]; ++q) acc = __dadd_rn(acc, __dmul_rn(js[bidx(q, Bp, b)], rys[bidx(p.j_ri[q], Bp, b)]));
    rhat[g] = __dadd_rn(rxs[g], __dmul_rn(gamma, acc));
  }
}

// H_delta slots of the systems still on the ladder -> their panels.
__global__ void kb_scatter(int nsrc, BDims bd, SnPlan sp, const int* __restrict__ mode, const int* __restrict__ slot_sn,
                           const double* __restrict__ src, const int* __restrict__ to_panel,
                           const int* __restrict__ srow, const int* __restrict__ scol,
                           const double* __restrict__ delta1, const int* __restrict__ active,
                           double* __restrict__ panel) {
  const long long g = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  const int Bp = bd.Bp, b = static_cast<int>(g & (Bp - 1));
  const long long t = (g >> (__ffs(Bp) - 1));
  if (t >= nsrc || !active[b]) return;
  double v = src[g];
  const double d1 = delta1[b];
  if (d1 != 0.0 && srow[t] == scol[t]) v = __dadd_rn(v, d1);
  const int p = to_panel[t], sn = slot_sn[p];
  panel[pan_addr(sp, mode, sn, p - sp.off[sn], Bp, b)] = v;
}

__global__ void kb_zero_panels(long long nslots, BDims bd, SnPlan sp, const int* __restrict__ mode,
                               const int* __restrict__ slot_sn, const int* __restrict__ active,
                               double* __restrict__ panel) {
  const long long g = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (g >= nslots * bd.Bp) return;
  const int b = static_cast<int>(g & (bd.Bp - 1));
  if (!active[b]) return;
  const int p = static_cast<int>((g >> (__ffs(bd.Bp) - 1))), sn = slot_sn[p];
  panel[pan_addr(sp, mode, sn, p - sp.off[sn], bd.Bp, b)] = 0.0;
}

// ---- factorization ----------------------------------------------------------
struct BFactorArgs {
  SnPlan s;
  BDims bd;
  double* panel;        // panel_size x Bp
  int* done;            // nsup x T
  int epoch;
  const double* maxdiag;
  double floor_rel;
  double floor_abs;
  const int* active;    // Bp
  int* fail_col;        // Bp
  int* abort;
  unsigned* ticket;     // job counter (zero on entry)
  const int* mode;      // nsup: 1 = wide (per-system task), 0 = lane mode
  int* wdone;           // nsup x Bp done flags of wide tasks
  const int* job_ptr;   // CTA jobs in topological order (see btrsv_pass)
  const int* job_items;
  const unsigned char* job_kind;  // 0: up to 8 lane tasks; 1: one wide task (sn * Bp + b)
  int njobs;
  int smem_doubles;     // dynamic shared memory available to a wide task
};

// Per-lane dense work is written as blocks of independent loads followed by
// the dependent arithmetic and stores: the compiler cannot move loads across
// stores to possibly-aliasing global addresses, so without the explicit
// blocking every step of a lane's sequential loop would pay an L2 round trip.
constexpr int kIlp = 8;
constexpr int kUb = 4;  // descendant rows held in registers per left-looking update block

__device__ void bfactor_task(const BFactorArgs& a, int sn, int tile, int lane) {
  const SnPlan& s = a.s;
  const int Bp = a.bd.Bp, T = a.bd.T, b = tile * 32 + lane;
  const int f = s.first[sn], w = s.first[sn + 1] - f, nr = s.nrows[sn];
  const int* R = s.rows + s.rows_ptr[sn];
  for (int c = s.child_ptr[sn] + lane; c < s.child_ptr[sn + 1]; c += 32) {
    wait_flag(a.done + s.child[c] * T + tile, a.epoch, a.abort);
  }
  __syncwarp();
  fence_gpu();
  // Only systems still on the ladder recompute (the others keep their L).
  const bool act = a.active[b] != 0;
  if (act) {
    double* P = a.panel + (long long)s.off[sn] * Bp + b;
    const double floor_v = fmax(a.maxdiag ? a.floor_rel * a.maxdiag[b] : a.floor_abs, 0.0);
    for (int u = s.upd_ptr[sn]; u < s.upd_ptr[sn + 1]; ++u) {
      const int d = s.upd_d[u], o = s.upd_off[u], cnt = s.upd_cnt[u];
      const int nrd = s.nrows[d], wd = s.first[d + 1] - s.first[d];
      const double* Pd = a.panel + (long long)s.off[d] * Bp + b;
      const int* Rd = s.rows + s.rows_ptr[d];
      const int m = nrd - o;
      const int* upos = s.upd_pos + s.upd_pbase[u];
      // k-blocks of 4 descendant columns; for each block of kUb descendant
      // rows the row values stay in registers while every target column jj
      // (<= the block's last row) is updated: each target entry receives its
      // k-block dots in ascending k0, as a plain left-looking sweep would.
      for (int k0 = 0; k0 < wd; k0 += 4) {
        const int kn = min(4, wd - k0);
        for (int i0 = 0; i0 < m; i0 += kUb) {
          double li[kUb][4];
          int pos[kUb];
#pragma unroll
          for (int t = 0; t < kUb; ++t) {
            const int ii = i0 + t;
            pos[t] = ii < m ? __ldg(upos + ii) : -1;
#pragma unroll
            for (int k = 0; k < 4; ++k)
              li[t][k] = (ii < m && k < kn) ? ldcg(Pd + (long long)((k0 + k) * nrd + o + ii) * Bp) : 0.0;
          }
          const int jend = min(cnt, i0 + kUb);
          for (int jj = 0; jj < jend; ++jj) {
            const int cc = __ldg(Rd + o + jj) - f;
            double lj[4];
#pragma unroll
            for (int k = 0; k < 4; ++k) lj[k] = k < kn ? ldcg(Pd + (long long)((k0 + k) * nrd + o + jj) * Bp) : 0.0;
            double cur[kUb];
#pragma unroll
            for (int t = 0; t < kUb; ++t) {
              const bool ok = pos[t] >= 0 && i0 + t >= jj;
              cur[t] = ok ? P[(long long)(cc * nr + pos[t]) * Bp] : 0.0;
            }
#pragma unroll
            for (int t = 0; t < kUb; ++t) {
              if (pos[t] >= 0 && i0 + t >= jj) {
                double dot = 0.0;
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                  if (k < kn) dot = fma(li[t][k], lj[k], dot);
                }
                P[(long long)(cc * nr + pos[t]) * Bp] = cur[t] - dot;
              }
            }
          }
        }
      }
    }
    bool failed = false;
    for (int k = 0; k < w; ++k) {
      double* Pk = P + (long long)k * nr * Bp;
      const double pivot = Pk[(long long)k * Bp];
      if (!(pivot > floor_v) && !failed) {
        failed = true;
        atomicMin(a.fail_col + b, f + k);
      }
      const double dk = sqrt(pivot);
      const double rdk = 1.0 / dk;  // one division per column, the scaling multiplies
      Pk[(long long)k * Bp] = dk;
      for (int r0 = k + 1; r0 < nr; r0 += kIlp) {
        double v[kIlp];
#pragma unroll
        for (int t = 0; t < kIlp; ++t) v[t] = r0 + t < nr ? Pk[(long long)(r0 + t) * Bp] : 0.0;
#pragma unroll
        for (int t = 0; t < kIlp; ++t) {
          if (r0 + t < nr) Pk[(long long)(r0 + t) * Bp] = v[t] * rdk;
        }
      }
      for (int c = k + 1; c < w; ++c) {
        const double lck = Pk[(long long)c * Bp];
        double* Pc = P + (long long)c * nr * Bp;
        for (int r0 = c; r0 < nr; r0 += kIlp) {
          double lk[kIlp], pc[kIlp];
#pragma unroll
          for (int t = 0; t < kIlp; ++t) {
            lk[t] = r0 + t < nr ? Pk[(long long)(r0 + t) * Bp] : 0.0;
            pc[t] = r0 + t < nr ? Pc[(long long)(r0 + t) * Bp] : 0.0;
          }
#pragma unroll
          for (int t = 0; t < kIlp; ++t) {
            if (r0 + t < nr) Pc[(long long)(r0 + t) * Bp] = fma(-lk[t], lck, pc[t]);
          }
        }
      }
    }
  }
  warp_publish(a.done + sn * T + tile, a.epoch, lane);
}

// Wide factor task: one CTA, one system b.  The panel is staged in shared
// memory; descendant blocks are staged in batches (all loads of a batch in
// flight at once) and applied with warp-owned target columns (no races, a
// fixed order per target entry); then a blocked right-looking Cholesky:
// warp 0 factors kFB columns, all warps apply the rank-kFB trailing update.
constexpr int kFB = 8;

__device__ void wfactor_task(const BFactorArgs& a, int sn, int b, double* sm) {
  const SnPlan& s = a.s;
  const int Bp = a.bd.Bp, T = a.bd.T, tile = b >> 5;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int f = s.first[sn], w = s.first[sn + 1] - f, nr = s.nrows[sn];
  const int size = nr * w;
  const int* R = s.rows + s.rows_ptr[sn];
  for (int c = s.child_ptr[sn] + tid; c < s.child_ptr[sn + 1]; c += blockDim.x) {
    const int ch = s.child[c];
    if (a.mode[ch]) wait_flag(a.wdone + (long long)ch * Bp + b, a.epoch, a.abort);
    else wait_flag(a.done + ch * T + tile, a.epoch, a.abort);
  }
  __syncthreads();
  fence_gpu();
  const bool act = a.active[b] != 0;
  double* Pg = a.panel + (long long)s.off[sn] * Bp + (long long)b * size;
  if (act) {
    // shared layout: panel | rows (int) | staging values | staging positions (int)
    const bool fits = size + (nr + 1) / 2 + 1 + 512 <= a.smem_doubles;
    double* PS = fits ? sm : Pg;
    int* RS = reinterpret_cast<int*>(sm + (fits ? size : 0));
    const int stage0 = (fits ? size : 0) + (nr + 1) / 2 + 1;
    const int budget = a.smem_doubles - stage0;
    double* DS = sm + stage0;
    if (fits) {
      for (int e = tid; e < size; e += blockDim.x) PS[e] = Pg[e];
    }
    for (int q = tid; q < nr; q += blockDim.x) RS[q] = R[q];
    __syncthreads();
    // ---- descendant updates, in batches that fit the staging area ----
    const int u0 = s.upd_ptr[sn], u1 = s.upd_ptr[sn + 1];
    int ub = u0;
    while (ub < u1) {
      // batch [ub, ue): staged values m * wd doubles + m positions each
      int ue = ub, used = 0;
      while (ue < u1) {
        const int d = s.upd_d[ue];
        const int m = s.nrows[d] - s.upd_off[ue], wd = s.first[d + 1] - s.first[d];
        const int need = m * wd + (m + 1) / 2 + 1;
        if (ue > ub && used + need > budget) break;
        used += need;
        ++ue;
        if (used > budget) break;  // a single oversized block: staged area overflows -> handled below
      }
      const bool staged = used <= budget;
      // stage
      if (staged) {
        int o2 = 0;
        for (int u = ub; u < ue; ++u) {
          const int d = s.upd_d[u], o = s.upd_off[u], cnt = s.upd_cnt[u];
          const int nrd = s.nrows[d], wd = s.first[d + 1] - s.first[d], m = nrd - o;
          const int* Rd = s.rows + s.rows_ptr[d];
          double* V = DS + o2;
          int* POS = reinterpret_cast<int*>(DS + o2 + m * wd);
          for (int e = tid; e < m * wd; e += blockDim.x) {
            const int k = e / m, ii = e - k * m;
            V[e] = a.panel[pan_addr(s, a.mode, d, k * nrd + o + ii, Bp, b)];
          }
          const int* upos = s.upd_pos + s.upd_pbase[u];
          for (int ii = tid; ii < m; ii += blockDim.x) POS[ii] = __ldg(upos + ii);
          o2 += m * wd + (m + 1) / 2 + 1;
        }
      }
      __syncthreads();
      // apply: warp owns target columns cc = wid (mod 8)
      int o2 = 0;
      for (int u = ub; u < ue; ++u) {
        const int d = s.upd_d[u], o = s.upd_off[u], cnt = s.upd_cnt[u];
        const int nrd = s.nrows[d], wd = s.first[d + 1] - s.first[d], m = nrd - o;
        const int* Rd = s.rows + s.rows_ptr[d];
        const double* V = DS + o2;
        const int* POS = reinterpret_cast<const int*>(DS + o2 + m * wd);
        for (int jj = 0; jj < cnt; ++jj) {
          const int cc = __ldg(Rd + o + jj) - f;
          if ((cc & 7) != wid) continue;
          for (int ii = jj + lane; ii < m; ii += 32) {
            double dot = 0.0;
            int pos;
            if (staged) {
              for (int k = 0; k < wd; ++k) dot = fma(V[k * m + ii], V[k * m + jj], dot);
              pos = POS[ii];
            } else {
              for (int k = 0; k < wd; ++k) {
                dot = fma(a.panel[pan_addr(s, a.mode, d, k * nrd + o + ii, Bp, b)],
                          a.panel[pan_addr(s, a.mode, d, k * nrd + o + jj, Bp, b)], dot);
              }
              pos = __ldg(s.upd_pos + s.upd_pbase[u] + ii);
            }
            PS[cc * nr + pos] -= dot;
          }
        }
        // the next update may hit the same entries from other lanes
        __syncwarp();
        if (staged) o2 += m * wd + (m + 1) / 2 + 1;
      }
      __syncthreads();
      ub = ue;
    }
    // ---- dense blocked Cholesky of the panel ----
    const double floor_v = fmax(a.maxdiag ? a.floor_rel * a.maxdiag[b] : a.floor_abs, 0.0);
    for (int k0 = 0; k0 < w; k0 += kFB) {
      const int kb = min(kFB, w - k0);
      if (wid == 0) {
        bool failed = false;
        for (int k = k0; k < k0 + kb; ++k) {
          double* Pk = PS + k * nr;
          const double pivot = Pk[k];
          if (!(pivot > floor_v) && !failed) {
            failed = true;
            if (lane == 0) atomicMin(a.fail_col + b, f + k);
          }
          const double dk = sqrt(pivot), rdk = 1.0 / dk;
          __syncwarp();
          if (lane == 0) Pk[k] = dk;
          for (int r = k + 1 + lane; r < nr; r += 32) Pk[r] = Pk[r] * rdk;
          __syncwarp();
          for (int c = k + 1; c < k0 + kb; ++c) {
            const double lck = Pk[c];
            double* Pc = PS + c * nr;
            for (int r = c + lane; r < nr; r += 32) Pc[r] = fma(-Pk[r], lck, Pc[r]);
          }
          __syncwarp();
        }
      }
      __syncthreads();
      for (int c = k0 + kb + wid; c < w; c += 8) {
        double lc[kFB];
#pragma unroll
        for (int k = 0; k < kFB; ++k) lc[k] = k < kb ? PS[(k0 + k) * nr + c] : 0.0;
        double* Pc = PS + c * nr;
        for (int r = c + lane; r < nr; r += 32) {
          double v = Pc[r];
#pragma unroll
          for (int k = 0; k < kFB; ++k) {
            if (k < kb) v = fma(-PS[(k0 + k) * nr + r], lc[k], v);
          }
          Pc[r] = v;
        }
      }
      __syncthreads();
    }
    if (fits) {
      for (int e = tid; e < size; e += blockDim.x) Pg[e] = PS[e];
    }
  }
  __syncthreads();
  if (tid == 0) {
    fence_gpu();
    st_relaxed(a.wdone + (long long)sn * Bp + b, a.epoch);
  }
}

__global__ void __launch_bounds__(256) kb_factor(BFactorArgs a) {
  __shared__ int s_job;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int T = a.bd.T, Bp = a.bd.Bp;
  for (;;) {
    if (threadIdx.x == 0) s_job = static_cast<int>(atomicAdd(a.ticket, 1u));
    __syncthreads();
    const int j = s_job;
    if (j >= a.njobs) break;
    const int i0 = __ldg(a.job_ptr + j), i1 = __ldg(a.job_ptr + j + 1);
    if (a.job_kind[j]) {
      const int it = __ldg(a.job_items + i0);
      wfactor_task(a, (it >> (__ffs(Bp) - 1)), (it & (Bp - 1)), bsmem);
    } else if (i0 + wid < i1) {
      const int t = __ldg(a.job_items + i0 + wid);
      bfactor_task(a, a.s.order[t / T], t % T, lane);
    }
    __syncthreads();
  }
}

// ---- triangular solves ------------------------------------------------------
struct BTrsvArgs {
  SnPlan s;
  BDims bd;
  const double* panel;
  double* y;         // n x Bp forward result (permuted)
  double* x;         // n x Bp backward result (permuted)
  double* u;         // u_size x Bp
  double* acc;       // rows_ptr[nsup] x Bp scratch
  double* x_out;     // original order n x Bp, or null
  int* fdone;        // nsup x T
  int* bdone;        // nsup x T
  int epoch;
  int* abort;
  // rhs: b[perm i] (- or +) J^T u
  const double* rb;  // n x Bp original order, or null
  const double* ru;  // m_c x Bp, or null
  const int* j_cp;
  const int* j_ri;
  const double* jval;  // nnz(J) x Bp
  const int* lane_on;  // Bp: 0 = system finished, skip its arithmetic (or null)
  GridBarrier bar;
  int smem_rows;       // per-warp shared accumulator rows (dynamic smem = 8 * rows * 256 B)
  unsigned* ticket;    // job counter of this pass (zero on entry)
  unsigned long long* trace = nullptr;  // diagnostics
  // CTA jobs in topological order: job j = items [job_ptr[j], job_ptr[j+1]).
  // job_kind 0: up to 8 lane-mode tasks (task ids as in btrsv_pass), one per
  // warp; 1 / 2: one wide forward / backward task (item = sn * Bp + b) done
  // by the whole CTA for one system.
  const int* job_ptr;
  const int* job_items;
  const unsigned char* job_kind;
  int njobs;
  const int* mode;     // nsup: 1 = wide
  int smem_doubles;
};

__device__ __forceinline__ double brhs(const BTrsvArgs& a, int i, int b) {
  const int Bp = a.bd.Bp;
  const int o = a.s.perm[i];
  double bi = a.rb ? a.rb[bidx(o, Bp, b)] : 0.0;
  if (a.ru) {
    double t = 0.0;
    for (int q = a.j_cp[o]; q < a.j_cp[o + 1]; ++q) {
      t = __dadd_rn(t, __dmul_rn(a.jval[bidx(q, Bp, b)], ldcg(a.ru + bidx(a.j_ri[q], Bp, b))));
    }
    bi = a.rb ? __dsub_rn(bi, t) : t;
  }
  return bi;
}

// Per-warp shared-memory accumulator for supernodes with <= 32 structure
// rows: A[q][lane].  Larger ones use the global scratch (stride Bp).
constexpr int kSmemRows = 32;
// Dense parts are processed in chunks of kC columns held in registers, so a
// lane's global read-modify-writes happen once per chunk, not per column.
constexpr int kC = 8;

// Forward task (multifrontal, lane = system): extend-add the children's
// update vectors, chunked triangular solve of the diagonal block, rank-kC
// updates of the rows below, publish y and u.  Values are the
// synchronisation: every value read from another task is checked against
// kUnset (and polled if not there yet), so no flags or fences are needed.
__device__ __forceinline__ void bfwd_core(const BTrsvArgs& a, int sn, int b, double* A, long long as) {
  const SnPlan& s = a.s;
  const int Bp = a.bd.Bp;
  const int f = s.first[sn], w = s.first[sn + 1] - f, nr = s.nrows[sn];
  // Wait: one coalesced poll per child on its last update entry for this
  // lane's system; the loads below re-check every value anyway.
  for (int c = s.child_ptr[sn]; c < s.child_ptr[sn + 1]; ++c) {
    const int ch = s.child[c];
    poll_value(a.u + (long long)(s.u_off[ch + 1] - 1) * Bp + b, a.abort);
  }
  for (int c = s.child_ptr[sn]; c < s.child_ptr[sn + 1]; ++c) {
    const int ch = s.child[c];
    const int m = s.nrows[ch] - (s.first[ch + 1] - s.first[ch]);
    const double* uc = a.u + (long long)s.u_off[ch] * Bp + b;
    const int* rel = s.relind + s.u_off[ch];
    for (int t0 = 0; t0 < m; t0 += kIlp) {
      int q[kIlp];
      double v[kIlp], cur[kIlp];
#pragma unroll
      for (int t = 0; t < kIlp; ++t) q[t] = t0 + t < m ? __ldg(rel + t0 + t) : -1;
#pragma unroll
      for (int t = 0; t < kIlp; ++t) v[t] = q[t] >= 0 ? ldcg(uc + (long long)(t0 + t) * Bp) : 0.0;
#pragma unroll
      for (int t = 0; t < kIlp; ++t) cur[t] = q[t] >= 0 ? A[q[t] * as] : 0.0;
      bool bad = false;
#pragma unroll
      for (int t = 0; t < kIlp; ++t) bad |= (q[t] >= 0) && __double_as_longlong(v[t]) == kUnset;
      if (bad) {
#pragma unroll
        for (int t = 0; t < kIlp; ++t) {
          if (q[t] >= 0) v[t] = load_ready(uc + (long long)(t0 + t) * Bp, a.abort);
        }
      }
#pragma unroll
      for (int t = 0; t < kIlp; ++t) {
        if (q[t] >= 0) A[q[t] * as] = cur[t] + ((q[t] < w) ? -v[t] : v[t]);
      }
    }
  }
  const double* P = a.panel + (long long)s.off[sn] * Bp + b;
  for (int cb = 0; cb < w; cb += kC) {
    const int cw = min(kC, w - cb);
    double yv[kC], ad[kC];
#pragma unroll
    for (int k = 0; k < kC; ++k) ad[k] = k < cw ? A[(cb + k) * as] : 0.0;
#pragma unroll
    for (int k = 0; k < kC; ++k) {
      yv[k] = 0.0;
      if (k < cw) {
        double acc = ad[k];
#pragma unroll
        for (int j = 0; j < kC; ++j) {
          if (j < k) acc = fma(-__ldg(P + (long long)((cb + j) * nr + cb + k) * Bp), yv[j], acc);
        }
        yv[k] = acc * (1.0 / __ldg(P + (long long)((cb + k) * nr + cb + k) * Bp));
        stcg(a.y + bidx(f + cb + k, Bp, b), yv[k]);
      }
    }
    for (int q0 = cb + cw; q0 < nr; q0 += kIlp) {
      double av[kIlp];
#pragma unroll
      for (int t = 0; t < kIlp; ++t) av[t] = q0 + t < nr ? A[(q0 + t) * as] : 0.0;
#pragma unroll
      for (int k = 0; k < kC; ++k) {
        if (k < cw) {
#pragma unroll
          for (int t = 0; t < kIlp; ++t) {
            const int q = q0 + t;
            if (q < nr) {
              const double l = __ldg(P + (long long)((cb + k) * nr + q) * Bp);
              av[t] = (q < w) ? fma(-l, yv[k], av[t]) : fma(l, yv[k], av[t]);
            }
          }
        }
      }
#pragma unroll
      for (int t = 0; t < kIlp; ++t) {
        if (q0 + t < nr) A[(q0 + t) * as] = av[t];
      }
    }
  }
  double* U = a.u + (long long)s.u_off[sn] * Bp + b;
  for (int q0 = w; q0 < nr; q0 += kIlp) {
    double v[kIlp];
#pragma unroll
    for (int t = 0; t < kIlp; ++t) v[t] = q0 + t < nr ? A[(q0 + t) * as] : 0.0;
#pragma unroll
    for (int t = 0; t < kIlp; ++t) {
      if (q0 + t < nr) stcg(U + (long long)(q0 + t - w) * Bp, v[t]);
    }
  }
}

__device__ void bfwd_task(const BTrsvArgs& a, int sn, int tile, int lane, double* smem_warp) {
  const SnPlan& s = a.s;
  const int Bp = a.bd.Bp, b = tile * 32 + lane;
  const int f = s.first[sn], w = s.first[sn + 1] - f, nr = s.nrows[sn];
  if (a.lane_on && !a.lane_on[b]) return;
  const bool small = nr <= a.smem_rows;
  if (small) {
    double* A = smem_warp + lane;  // shared: the compiler keeps it in the .shared window
    for (int q = 0; q < nr; ++q) A[q * 32] = q < w ? brhs(a, f + q, b) : 0.0;
    bfwd_core(a, sn, b, A, 32);
  } else {
    double* A = a.acc + (long long)s.rows_ptr[sn] * Bp + b;
    for (int q = 0; q < nr; ++q) A[(long long)q * Bp] = q < w ? brhs(a, f + q, b) : 0.0;
    bfwd_core(a, sn, b, A, Bp);
  }
}

// Backward task: wait for the parent's first column (it is published last),
// then chunked from the last chunk: partial sums over the rows below the
// chunk (x values checked), backward triangular solve in registers.
__device__ void bbwd_task(const BTrsvArgs& a, int sn, int tile, int lane) {
  const SnPlan& s = a.s;
  const int Bp = a.bd.Bp, b = tile * 32 + lane;
  const int f = s.first[sn], w = s.first[sn + 1] - f, nr = s.nrows[sn];
  const int* R = s.rows + s.rows_ptr[sn];
  if (a.lane_on && !a.lane_on[b]) return;
  const int par = s.parent[sn];
  if (par >= 0) poll_value(a.x + bidx(s.first[par], Bp, b), a.abort);
  const double* P = a.panel + (long long)s.off[sn] * Bp + b;
  const int nchunks = (w + kC - 1) / kC;
  for (int ci = nchunks - 1; ci >= 0; --ci) {
    const int cb = ci * kC, cw = min(kC, w - cb);
    double S[kC];
#pragma unroll
    for (int k = 0; k < kC; ++k) S[k] = 0.0;
    for (int r0 = cb + cw; r0 < nr; r0 += kIlp) {
      double xv[kIlp];
#pragma unroll
      for (int t = 0; t < kIlp; ++t) xv[t] = r0 + t < nr ? load_ready(a.x + bidx(__ldg(R + r0 + t), Bp, b), a.abort) : 0.0;
#pragma unroll
      for (int k = 0; k < kC; ++k) {
        if (k < cw) {
#pragma unroll
          for (int t = 0; t < kIlp; ++t) {
            if (r0 + t < nr) S[k] = fma(__ldg(P + (long long)((cb + k) * nr + r0 + t) * Bp), xv[t], S[k]);
          }
        }
      }
    }
    double xc[kC];
#pragma unroll
    for (int k = kC - 1; k >= 0; --k) {
      xc[k] = 0.0;
      if (k < cw) {
        double acc = load_ready(a.y + bidx(f + cb + k, Bp, b), a.abort) - S[k];
#pragma unroll
        for (int j = 0; j < kC; ++j) {
          if (j > k && j < cw) acc = fma(-__ldg(P + (long long)((cb + k) * nr + cb + j) * Bp), xc[j], acc);
        }
        xc[k] = acc * (1.0 / __ldg(P + (long long)((cb + k) * nr + cb + k) * Bp));
        stcg(a.x + bidx(f + cb + k, Bp, b), xc[k]);
        if (a.x_out) a.x_out[bidx(s.perm[f + cb + k], Bp, b)] = xc[k];
      }
    }
  }
}


__device__ __forceinline__ void brearm(const BTrsvArgs& a) {
  const double u = __longlong_as_double(kUnset);
  const long long gt = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  const long long gs = (long long)gridDim.x * blockDim.x;
  const long long ny = (long long)a.s.n * a.bd.Bp, nu = (long long)a.s.u_size * a.bd.Bp;
  for (long long i = gt; i < ny; i += gs) {
    a.y[i] = u;
    a.x[i] = u;
  }
  for (long long i = gt; i < nu; i += gs) a.u[i] = u;
}

// ---- wide (per-system) solve tasks ---------------------------------------
// One CTA solves one system's supernode: the panel (contiguous per system in
// wide mode) is staged in shared memory with coalesced loads issued before
// the task waits on its inputs; warp 0 runs the dense triangular solve of
// the diagonal block 32 columns at a time in registers (shuffles), all warps
// apply each chunk to the remaining rows.  Vectors stay interleaved
// [entry][system], shared with the lane-mode tasks.

__device__ void wfwd_task(const BTrsvArgs& a, int sn, int b, double* sm) {
  const SnPlan& s = a.s;
  const int Bp = a.bd.Bp;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  if (a.lane_on && !a.lane_on[b]) return;  // CTA-uniform
  const int f = s.first[sn], w = s.first[sn + 1] - f, nr = s.nrows[sn], rp = s.rows_ptr[sn];
  const int size = nr * w;
  const double* Pg = a.panel + (long long)s.off[sn] * Bp + (long long)b * size;
  const bool fits = size + nr + 32 <= a.smem_doubles;
  double* PS = sm;
  double* V = fits ? sm + size : sm;
  double* Ys = V + nr;
  const double* P = fits ? PS : Pg;
  if (fits) {
    for (int e = tid; e < size; e += blockDim.x) PS[e] = __ldg(Pg + e);
  }
  for (int q = tid; q < nr; q += blockDim.x) {
    double v = q < w ? brhs(a, f + q, b) : 0.0;
    const int g0 = __ldg(s.gat_ptr + rp + q), g1 = __ldg(s.gat_ptr + rp + q + 1);
    for (int g = g0; g < g1; ++g) {
      const double u = load_ready(a.u + (long long)__ldg(s.gat_idx + g) * Bp + b, a.abort);
      v = q < w ? v - u : v + u;
    }
    V[q] = v;
  }
  __syncthreads();
  for (int cb = 0; cb < w; cb += 32) {
    const int cw = min(32, w - cb);
    if (wid == 0) {
      double d[32];  // row cb+lane of the chunk's diagonal block
#pragma unroll
      for (int k = 0; k < 32; ++k) d[k] = (k < cw && lane < cw) ? P[(cb + k) * nr + cb + lane] : 0.0;
      double acc = lane < cw ? V[cb + lane] : 0.0;
      const double rdl = lane < cw ? 1.0 / P[(cb + lane) * nr + cb + lane] : 1.0;
#pragma unroll
      for (int k = 0; k < 32; ++k) {
        if (k < cw) {
          const double yk = __shfl_sync(0xffffffffu, acc * rdl, k);
          if (lane == k) acc = yk;
          if (lane > k && lane < cw) acc = fma(-d[k], yk, acc);
        }
      }
      if (lane < cw) {
        Ys[lane] = acc;
        stcg(a.y + bidx(f + cb + lane, Bp, b), acc);
      }
    }
    __syncthreads();
    for (int q = cb + cw + tid; q < nr; q += blockDim.x) {
      double v = V[q];
      for (int k = 0; k < cw; ++k) {
        const double l = P[(cb + k) * nr + q];
        v = q < w ? fma(-l, Ys[k], v) : fma(l, Ys[k], v);
      }
      V[q] = v;
    }
    __syncthreads();
  }
  double* U = a.u + (long long)s.u_off[sn] * Bp + b;
  for (int q = w + tid; q < nr; q += blockDim.x) stcg(U + (long long)(q - w) * Bp, V[q]);
}

__device__ void wbwd_task(const BTrsvArgs& a, int sn, int b, double* sm) {
  const SnPlan& s = a.s;
  const int Bp = a.bd.Bp;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  if (a.lane_on && !a.lane_on[b]) return;
  const int f = s.first[sn], w = s.first[sn + 1] - f, nr = s.nrows[sn];
  const int size = nr * w, nbl = nr - w;
  const int* R = s.rows + s.rows_ptr[sn];
  const double* Pg = a.panel + (long long)s.off[sn] * Bp + (long long)b * size;
  const bool fits = size + nr + 32 <= a.smem_doubles;
  double* X = fits ? sm + size : sm;  // x of the rows below (nbl)
  double* S = X + nbl;                // w partial sums
  double* Xc = S + w;                 // chunk x (32)
  const double* P = fits ? sm : Pg;
  if (fits) {
    for (int e = tid; e < size; e += blockDim.x) sm[e] = __ldg(Pg + e);
  }
  const int par = s.parent[sn];
  if (par >= 0 && tid == 0) poll_value(a.x + bidx(s.first[par], Bp, b), a.abort);
  __syncthreads();
  for (int r = tid; r < nbl; r += blockDim.x) X[r] = load_ready(a.x + bidx(__ldg(R + w + r), Bp, b), a.abort);
  __syncthreads();
  for (int k = wid; k < w; k += 8) {
    double t = 0.0;
    for (int r = lane; r < nbl; r += 32) t = fma(P[k * nr + w + r], X[r], t);
    t = warp_sum(t);
    if (lane == 0) S[k] = t;
  }
  __syncthreads();
  const int nchunks = (w + 31) >> 5;
  for (int ci = nchunks - 1; ci >= 0; --ci) {
    const int cb = ci * 32, cw = min(32, w - cb);
    if (wid == 0) {
      double d[32];  // column cb+lane: L(cb+j, cb+lane)
#pragma unroll
      for (int j = 0; j < 32; ++j) d[j] = (j < cw && lane < cw) ? P[(cb + lane) * nr + cb + j] : 0.0;
      double acc = lane < cw ? load_ready(a.y + bidx(f + cb + lane, Bp, b), a.abort) - S[cb + lane] : 0.0;
      const double rdl = lane < cw ? 1.0 / P[(cb + lane) * nr + cb + lane] : 1.0;
#pragma unroll
      for (int j = 31; j >= 0; --j) {
        if (j < cw) {
          const double xj = __shfl_sync(0xffffffffu, acc * rdl, j);
          if (lane == j) acc = xj;
          if (lane < j) acc = fma(-d[j], xj, acc);
        }
      }
      if (lane < cw) {
        Xc[lane] = acc;
        stcg(a.x + bidx(f + cb + lane, Bp, b), acc);
        if (a.x_out) a.x_out[bidx(s.perm[f + cb + lane], Bp, b)] = acc;
      }
    }
    __syncthreads();
    if (ci > 0) {
      for (int k = tid; k < cb; k += blockDim.x) {
        double t = S[k];
        for (int j = 0; j < cw; ++j) t = fma(P[k * nr + cb + j], Xc[j], t);
        S[k] = t;
      }
      __syncthreads();
    }
  }
}

// One forward + backward pass over the CTA job list; y, x, u must hold
// kUnset on entry.  Jobs are taken in topological order by whole CTAs
// (deadlock-free for the same reason as warp tasks: every job's
// dependencies lie in earlier jobs, all held by resident CTAs).
__device__ __forceinline__ void btrsv_pass(const BTrsvArgs& a) {
  __shared__ int s_job;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  double* smem_warp = bsmem + wid * a.smem_rows * 32;
  const int T = a.bd.T;
  const long long ns = (long long)a.s.nsup * T;
  for (;;) {
    if (threadIdx.x == 0) s_job = static_cast<int>(atomicAdd(a.ticket, 1u));
    __syncthreads();
    const int j = s_job;
    if (j >= a.njobs) break;
    const int i0 = __ldg(a.job_ptr + j), i1 = __ldg(a.job_ptr + j + 1);
    const int kind = a.job_kind[j];
    if (kind) {
      const int it = __ldg(a.job_items + i0);
      if (a.trace && threadIdx.x == 0) a.trace[a.njobs + j] = global_ns();
      if (kind == 1) wfwd_task(a, (it >> (__ffs(a.bd.Bp) - 1)), (it & (a.bd.Bp - 1)), bsmem);
      else wbwd_task(a, (it >> (__ffs(a.bd.Bp) - 1)), (it & (a.bd.Bp - 1)), bsmem);
      if (a.trace && threadIdx.x == 0) a.trace[j] = global_ns();
    } else if (i0 + wid < i1) {
      const long long t = __ldg(a.job_items + i0 + wid);
      if (a.trace && threadIdx.x == 0) a.trace[a.njobs + j] = global_ns();
      if (t < ns) {
        bfwd_task(a, a.s.order[t / T], static_cast<int>(t % T), lane, smem_warp);
      } else {
        const long long tb = 2 * ns - 1 - t;
        bbwd_task(a, a.s.order[tb / T], static_cast<int>(tb % T), lane);
      }
      __syncwarp();
      if (a.trace && lane == 0) atomicMax(a.trace + j, global_ns());
    }
    __syncthreads();
  }
}

__global__ void __launch_bounds__(256) kb_trsv(BTrsvArgs a) {
  brearm(a);
  grid_sync(a.bar, a.abort);
  btrsv_pass(a);
}

// Schur rhs J w - r_y per system (w = y after the pass, permuted).
__global__ void kb_schur_rhs(int mc, BDims bd, const int* rp, const int* ci_perm, const double* jcsr,
                             const double* y, const double* r_y, double* rhs) {
  const long long g = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  const int Bp = bd.Bp, b = static_cast<int>(g & (Bp - 1));
  const long long k = (g >> (__ffs(Bp) - 1));
  if (k >= mc) return;
  double acc = 0.0;
  for (int e = rp[k]; e < rp[k + 1]; ++e) {
    const double t = y[bidx(ci_perm[e], Bp, b)];
    if (t == 0.0) continue;
    acc = __dadd_rn(acc, __dmul_rn(jcsr[bidx(e, Bp, b)], t));
  }
  rhs[g] = __dsub_rn(acc, r_y[g]);
}

// ---- batched CG ---------------------------------------------------------------
struct BCgArgs {
  BTrsvArgs tr;       // ru = p, lane_on = running
  int mc;
  const int* jcsr_rp;
  const int* jcsr_ci_perm;
  const double* jcsr;  // nnz x Bp
  const double* rhs;   // mc x Bp
  double* x;
  double* r;
  double* p;
  double* q;
  double* part;        // gridsize doubles (per-thread partials)
  int* running;        // Bp: 1 while the system iterates (also tr.lane_on)
  const int* start;    // Bp: systems to run in this launch
  double delta2;
  double tol;
  double thr;
  long long max_iter;
  int epoch_base;
  long long* iters;    // Bp
  double* relres;      // Bp
  int* flags;          // Bp: 1 converged, 2 small quadratic
  int* live;           // max_iter + 2 counters, zeroed
  unsigned* tickets;   // max_iter + 2 task counters, zeroed
  GridBarrier bar;
};

// Per-system reduction: thread g holds a partial for system g % Bp; the
// grid size is a multiple of Bp, so every thread's systems are fixed.
__device__ __forceinline__ double bsum(const BCgArgs& a, double v) {
  const long long gt = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  const long long gs = (long long)gridDim.x * blockDim.x;
  a.part[gt] = v;
  grid_sync(a.bar, a.tr.abort);
  const int Bp = a.tr.bd.Bp;
  double s = 0.0;
  for (long long j = gt % Bp; j < gs; j += Bp) s += ldcg(a.part + j);
  grid_sync(a.bar, a.tr.abort);  // partials may be overwritten after this
  return s;
}

__global__ void __launch_bounds__(256) kb_cg(BCgArgs a) {
  const int Bp = a.tr.bd.Bp;
  const long long gt = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  const long long gs = (long long)gridDim.x * blockDim.x;
  const int b = static_cast<int>(gt % Bp);
  const long long mcB = (long long)a.mc * Bp;
  const bool mine = a.start[b] != 0;
  brearm(a.tr);
  double ss = 0.0;
  for (long long g = gt; g < mcB; g += gs) {
    if (!mine) continue;
    const double v = a.rhs[g];
    a.x[g] = 0.0;
    a.r[g] = v;
    stcg(a.p + g, v);
    ss = fma(v, v, ss);
  }
  const double rhs_norm = sqrt(bsum(a, ss));
  bool run = mine && rhs_norm != 0.0;
  if (gt < Bp) {
    a.running[b] = run ? 1 : 0;
    if (mine && !run) {
      a.iters[b] = 0;
      a.relres[b] = 0.0;
      a.flags[b] = 1;
    }
  }
  double rho = rhs_norm * rhs_norm, r_norm = rhs_norm;
  grid_sync(a.bar, a.tr.abort);
  BTrsvArgs tr = a.tr;
  for (long long it = 1; it <= a.max_iter; ++it) {
    // any system still running?
    if (gt == 0) a.live[it] = 0;
    grid_sync(a.bar, a.tr.abort);
    if (gt < Bp && run) atomicAdd(a.live + it, 1);
    grid_sync(a.bar, a.tr.abort);
    if (ld_relaxed(a.live + it) == 0 || ld_relaxed(a.tr.abort)) break;
    tr.epoch = a.epoch_base + static_cast<int>(it);
    tr.ticket = a.tickets + it;
    btrsv_pass(tr);
    grid_sync(a.bar, a.tr.abort);
    double pq = 0.0, pp = 0.0;
    for (long long g = gt; g < mcB; g += gs) {
      if (!run) continue;
      const long long k = (g >> (__ffs(Bp) - 1));
      double qk = 0.0;
      for (int e = a.jcsr_rp[k]; e < a.jcsr_rp[k + 1]; ++e) {
        const double t = ldcg(tr.x + bidx(a.jcsr_ci_perm[e], Bp, b));
        if (t == 0.0) continue;
        qk = __dadd_rn(qk, __dmul_rn(a.jcsr[bidx(e, Bp, b)], t));
      }
      const double pk = ldcg(a.p + g);
      if (a.delta2 != 0.0) qk = __dadd_rn(qk, __dmul_rn(a.delta2, pk));
      a.q[g] = qk;
      pq = fma(pk, qk, pq);
      pp = fma(pk, pk, pp);
    }
    const double curvature = bsum(a, pq);
    const double p_norm2 = bsum(a, pp);
    brearm(tr);  // x no longer needed this iteration: re-arm for the next pass
    bool stop_small = run && curvature <= a.thr * p_norm2;
    const double alpha = rho / curvature;
    double rr = 0.0;
    for (long long g = gt; g < mcB; g += gs) {
      if (!run || stop_small) continue;
      a.x[g] = __dadd_rn(a.x[g], __dmul_rn(alpha, ldcg(a.p + g)));
      const double rk = __dsub_rn(a.r[g], __dmul_rn(alpha, a.q[g]));
      a.r[g] = rk;
      rr = fma(rk, rk, rr);
    }
    const double rn = sqrt(bsum(a, rr));
    if (stop_small) {
      if (gt < Bp) {
        a.iters[b] = it - 1;
        a.relres[b] = r_norm / rhs_norm;
        a.flags[b] = 2;
      }
      run = false;
    } else if (run) {
      r_norm = rn;
      const double relres = r_norm / rhs_norm;
      if (relres <= a.tol || it == a.max_iter) {
        if (gt < Bp) {
          a.iters[b] = it;
          a.relres[b] = relres;
          a.flags[b] = relres <= a.tol ? 1 : 0;
        }
        run = false;
      } else {
        const double rho_next = r_norm * r_norm;
        const double beta = rho_next / rho;
        rho = rho_next;
        for (long long g = gt; g < mcB; g += gs) stcg(a.p + g, __dadd_rn(a.r[g], __dmul_rn(beta, ldcg(a.p + g))));
      }
    }
    if (gt < Bp) a.running[b] = run ? 1 : 0;
    grid_sync(a.bar, a.tr.abort);
  }
}

// unscale + recover per system (ruiz.cpp:118-133, kkt_system.cpp:89-105)
__global__ void kb_recover(AsmPlan p, BDims bd, const int* __restrict__ jd_rp, const int* __restrict__ jd_ci,
                           const int* __restrict__ jd_src, const double* __restrict__ d,
                           const double* __restrict__ dx_s, const double* __restrict__ dy_s, BVals v,
                           double* __restrict__ dx, double* __restrict__ dy, double* __restrict__ ds,
                           double* __restrict__ dyd) {
  const long long g = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  const int Bp = bd.Bp, b = static_cast<int>(g & (Bp - 1));
  const long long t = (g >> (__ffs(Bp) - 1));
  if (t < p.nx) dx[g] = __dmul_rn(d[g], dx_s[g]);
  if (t < p.mc) dy[g] = __dmul_rn(d[bidx(p.nx + t, Bp, b)], dy_s[g]);
  if (t < p.md) {
    double acc = 0.0;
    for (int q = jd_rp[t]; q < jd_rp[t + 1]; ++q) {
      const int c = jd_ci[q];
      const double xc = __dmul_rn(d[bidx(c, Bp, b)], dx_s[bidx(c, Bp, b)]);
      if (xc == 0.0) continue;
      acc = __dadd_rn(acc, __dmul_rn(v.jd[bidx(jd_src[q], Bp, b)], xc));
    }
    const double s = __dsub_rn(acc, v.ryd[g]);
    ds[g] = s;
    dyd[g] = __dsub_rn(__dmul_rn(v.ds[g], s), v.rs[g]);
  }
}

}  // namespace hykkt::dev
