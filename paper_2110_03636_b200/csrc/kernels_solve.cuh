// Sync-free supernodal triangular solves and the device-resident CG loop.
//
// factor_solve (proj/core/src/cholesky.cpp:139-168) becomes one pass over the
// supernode tree, forward (children before parents, multifrontal: a supernode
// sums its children's update vectors, solves its diagonal block and hands
// L_below y to its parent) then backward (parents before children).  Three
// kinds of work per pass (trsv_pass):
//   * bottom levels (each >= HYKKT_TRSV_BOTTOM_MIN narrow supernodes):
//     level-synchronous, one thread per supernode, a grid barrier per level;
//   * wide supernodes (panel >= HYKKT_TRSV_WIDE entries): whole-CTA tasks on
//     reserved CTAs, rows staged in shared memory;
//   * the rest: warp tasks on warp tickets over the other CTAs.
// Both task streams are in topological order.  y / x / update vectors are
// their own completion flags (reset to kUnset before each pass; consumers
// poll the value they need).  The permutation is folded into the gathers:
// rows read b[perm[i]] / the J column perm[i], outputs scatter to x[perm[i]].
//
// cg_schur (solver.cpp:154-201) runs as ONE cooperative persistent kernel:
// each iteration = [J^T p fused into the forward solve -> H^-1 -> J t +
// delta2 p, p.q, p.p] -> grid barrier -> [alpha, x, r, r.r] -> grid barrier
// -> [convergence, beta, p] -> grid barrier.  No host round trips; dot
// products use per-block partials combined in a fixed order, so results are
// deterministic.  Termination rules mirror solver.cpp:161-199 exactly
// (zero rhs -> 0 iterations; small quadratic pq <= thr * pp -> abort with
// iterations = it - 1; relres = ||r|| / ||rhs|| <= tol; iteration cap).
#pragma once

#include "kernels_factor.cuh"

namespace hykkt::dev {

struct SolveRhs {
  const double* b;   // original-order vector (n) or null
  const double* u;   // J^T u term (m_c) or null; b - J^T u when both
  const int* j_cp;
  const int* j_ri;
  const double* jval;
};

// Unset-value marker: a signalling-NaN bit pattern that arithmetic never
// produces.  y (forward result) and x (backward result) are reset to it
// before each pass; a consumer spins on the VALUE it needs, so the data is
// its own completion flag — no per-task flags, no fences on the hot path.
constexpr long long kUnset = 0x7FF4DEADBEEF0001ll;

__device__ unsigned long long g_poll_fail_addr = 0;  // diagnostics: first value whose wait timed out
__device__ unsigned g_poll_fail_who = 0;              // and its waiter (block << 10 | thread)

// Raises the abort flag for a wait that exceeded the spin budget and
// records the first such wait (read by the host when HYKKT_DEBUG is set).
__device__ __noinline__ void poll_timed_out(const double* p, int* abort) {
  if (atomicCAS(&g_poll_fail_addr, 0ull, reinterpret_cast<unsigned long long>(p)) == 0ull)
    g_poll_fail_who = (blockIdx.x << 10) | threadIdx.x;
  atomicExch(abort, 1);
}

// Poll back-off (ns): first sleep, doubling up to the cap (HYKKT_POLL_NS /
// HYKKT_POLL_MAX_NS, set once per context; 16 / 16 by default: longer
// sleeps or a back-off measured no gain at C1-C4, r02 ab3).
__device__ unsigned g_poll_ns = 16, g_poll_max_ns = 16;

__device__ __forceinline__ double poll_value(const double* p, int* abort) {
  double v = ldcg(p);
  if (__double_as_longlong(v) != kUnset) return v;
  const long long t0 = clock64();
  unsigned ns = g_poll_ns;
  const unsigned cap = g_poll_max_ns;
  for (unsigned it = 1;; ++it) {
    __nanosleep(ns);
    ns = min(2 * ns, cap);
    v = ldcg(p);
    if (__double_as_longlong(v) != kUnset) return v;
    if ((it & 255u) == 0u) {
      if (ld_relaxed(abort)) return 0.0;
      if (clock64() - t0 > kSpinBudget) {
        poll_timed_out(p, abort);
        return 0.0;
      }
    }
  }
}

// Load a value that is expected to be set; poll only if it is not yet.
__device__ __forceinline__ double load_ready(const double* p, int* abort) {
  const double v = ldcg(p);
  return __double_as_longlong(v) != kUnset ? v : poll_value(p, abort);
}

struct TrsvArgs {
  SnPlan s;
  const double* panel;
  double* y;       // forward result (permuted), reset to kUnset per pass
  double* x;       // backward result (permuted), reset to kUnset per pass
  double* u;       // update vectors (SnPlan::u_off), reset to kUnset per pass
  double* acc_buf; // per-supernode accumulators for wide supernodes
  double* x_out;   // original-order output or null
  int* abort;
  SolveRhs rhs;
  GridBarrier bar;
  unsigned* ticket;           // task counter of this pass (zero on entry)
  unsigned long long* trace;  // diagnostics: per-task end / start times (ns)
  unsigned long long* pstamp; // diagnostics: per-CTA phase times of k_trsv (8 per CTA), or null
  // task streams (trsv_pass): wide supernodes for the first nwc CTAs,
  // narrow ones for the warps of the others; ticket[0] / ticket[1]
  const int* wid_sn;   // forward order
  const int* wid_bwd;  // backward order
  int nwid;
  const int* nar_sn;
  int nnar;
  int nwc;
  // narrow tasks: poll one flag value before loading (bit 0 fwd narrow,
  // 1 fwd general, 2 bwd narrow, 3 bwd general); otherwise every value is
  // polled where it is loaded
  int pre_wait;
  const int* pos;             // supernode -> position in s.order (trace slots)
  // bottom levels (w <= 8, nrows <= 32) solved level-synchronously, one
  // thread per supernode, before / after the task passes
  int nbot;
  const int* bot_ptr;         // nbot + 1
  const int* bot_sn;
  const unsigned char* bot_wide;  // per bottom level: 1 -> (w <= 8, nrows <= 32) variant
  // precomputed right-hand side of every permuted row (kernels_cluster.cuh),
  // null: rhs_at forms b - J^T u on the fly
  const double* bt;
  // Q-form wide supernodes (qslice_fwd / qslice_bwd): Q = [L_ss^-1;
  // L_below L_ss^-1] (nrows x w, column-major at qoff[sn]); the wide stream
  // then runs independent row slices (forward, int4 {sn, r0, r1, 0}) and
  // column slices (backward, {sn, c0, c1, 0}) instead of whole supernodes
  const double* q;
  const long long* qoff;
  const int4* qs_f;
  int nqf;
  const int4* qs_b;
  int nqb;
  // chains of the narrow stream (nar_sn entries < 0): chain k's supernodes
  // bottom-up in chain_sn[chain_ptr[k] .. chain_ptr[k+1])
  const int* chain_ptr;
  const int* chain_sn;
  const int* nar_bwd;  // backward order of the narrow stream (chains at their top member)
  // register hand-off tables of the chains (per row slot): forward, member
  // i > 0, row q: the lane of member i-1 holding the row's update value
  // (-1: none); backward, member i < top, rows below: lane | kind << 8 of
  // member i+1's registers holding that row's x (kind 0: its own columns,
  // 1: its rows below)
  const int* chain_fsrc;
  const int* chain_bsrc;
  // wide CTAs [0, nwd) serve only the wide stream; [nwd, nwc) are flex
  // (narrow forward stream first, see trsv_pass); tstride = counters per
  // pass (k_cg: pass it uses ticket + tstride * it)
  int nwd;
  int tstride;
  int prefetch;  // general tasks: L1 prefetch of their static data before the wait
  // forward right-hand side precomputed in the pass (k_cg): when bt_fill is
  // set, the pass first writes bt_fill[r] = b - J^T u for the rows of every
  // supernode above the bottom levels (bt_rows), alongside bottom level 0,
  // and the tasks then read it through bt (= bt_fill); the bottom levels
  // form their own rows' right-hand sides (rhs_raw)
  double* bt_fill;
  const int* bt_rows;
  int nbt_rows;
  int bt_all;
  int cta_gather;  // fwd_cta: row-side gathers instead of the per-child extend-add  // 1: bt_fill covers every row, filled before the bottom levels (one extra grid barrier)
};

#ifndef HYKKT_INLINE_MID
#define HYKKT_INLINE_MID 0  // 8 measured 1450 vs 1428 us per CG iteration at C4 (r02)
#endif
constexpr int kInlineMid = HYKKT_INLINE_MID;  // medium branch width cap of the inlined task loop (0 = off)
constexpr int kWideMaxRows = 2048;  // wide (CTA) solve tasks stage nrows doubles in shared memory
constexpr int kWarpRows = kWideMaxRows / 8;  // narrow-task CTAs: each warp's slice of the same buffer
struct TrsvSmem {
  double a[kWideMaxRows];
  double t[64];  // bwd_cta: one partial per (column < 32) x slice; sized for 512-thread CTAs
  int task;  // wide-stream ticket value broadcast to the CTA
};

__device__ __forceinline__ unsigned long long global_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__device__ __forceinline__ void reset_unset(double* v, int n) {
  const double u = __longlong_as_double(kUnset);
  const int gt = blockIdx.x * blockDim.x + threadIdx.x, gs = gridDim.x * blockDim.x;
  for (int i = gt; i < n; i += gs) v[i] = u;
}

// Right-hand side entry of permuted row i: b[perm i] and/or J^T u in the
// reference's spmv(J, u, transpose) order (csc_matrix.cpp:255-261).
__device__ __forceinline__ double rhs_raw(const TrsvArgs& a, int i) {
  const int o = a.s.perm[i];
  double bi = a.rhs.b ? a.rhs.b[o] : 0.0;
  if (a.rhs.u) {
    // entries four at a time with all their loads in flight, summed in
    // entry order (the reference's order, bit-identical to one at a time)
    double t = 0.0;
    const int q0 = a.rhs.j_cp[o], q1 = a.rhs.j_cp[o + 1];
    for (int q = q0; q < q1; q += 4) {
      int ri[4];
      double jv[4], uv[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        ri[k] = q + k < q1 ? __ldg(a.rhs.j_ri + q + k) : 0;
        jv[k] = q + k < q1 ? __ldg(a.rhs.jval + q + k) : 0.0;
      }
#pragma unroll
      for (int k = 0; k < 4; ++k) uv[k] = q + k < q1 ? ldcg(a.rhs.u + ri[k]) : 0.0;
#pragma unroll
      for (int k = 0; k < 4; ++k)
        if (q + k < q1) t = __dadd_rn(t, __dmul_rn(jv[k], uv[k]));
    }
    bi = a.rhs.b ? __dsub_rn(bi, t) : t;
  }
  return bi;
}

__device__ __forceinline__ double rhs_at(const TrsvArgs& a, int i) {
  return a.bt ? ldcg(a.bt + i) : rhs_raw(a, i);
}

// Sum of u[gat_idx[g]] for g in [gb, ge) in list order, four loads in
// flight; only values still unset are polled.
__device__ __forceinline__ double gather_u(const TrsvArgs& a, int gb, int ge) {
  double v = 0.0;
  for (int g = gb; g < ge; g += 4) {
    int i[4];
    double x[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) i[k] = (g + k < ge) ? __ldg(a.s.gat_idx + g + k) : -1;
#pragma unroll
    for (int k = 0; k < 4; ++k) x[k] = i[k] >= 0 ? ldcg(a.u + i[k]) : 0.0;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      if (i[k] >= 0 && __double_as_longlong(x[k]) == kUnset) x[k] = poll_value(a.u + i[k], a.abort);
      v += x[k];
    }
  }
  return v;
}

// One lane per child polls the child's last update-vector entry; the rest
// of the warp sleeps at the barrier instead of flooding the SM's L1TEX queue
// with one poll per lane.  Values are re-checked when actually loaded.
__device__ __forceinline__ void wait_children(const TrsvArgs& a, int sn, int lane) {
  const SnPlan& s = a.s;
  for (int c = s.child_ptr[sn] + lane; c < s.child_ptr[sn + 1]; c += 32) {
    const int ch = s.child[c];
    poll_value(a.u + s.u_off[ch + 1] - 1, a.abort);
  }
  __syncwarp();
}

// Forward task, multifrontal form: acc = sum of children's update vectors
// (extend-add through flattened gather lists), own rows:
// y = L_ss^-1 (b - acc), rows below: u_s = acc + L_below y, handed to the
// parent.  Every static load (gather indices, L, right-hand side) is issued
// before the first wait, so a tree level costs about one L2 round trip.
template <int MID>
__device__ __forceinline__ void fwd_task(const TrsvArgs& a, int sn, int lane, int tslot, double* sA = nullptr) {
  const SnPlan& s = a.s;
  const int f = s.first[sn], w = s.first[sn + 1] - f, nr = s.nrows[sn];
  const int rp = s.rows_ptr[sn];
  const double* P = a.panel + s.off[sn];
  double* U = a.u + s.u_off[sn];
  if (nr <= 32 && w <= 4) {
    // Narrow supernode: lane q owns row-structure position q.
    const bool own = lane < w, row = lane < nr;
    int gb = 0, ge = 0;
    if (row) {
      gb = __ldg(s.gat_ptr + rp + lane);
      ge = __ldg(s.gat_ptr + rp + lane + 1);
    }
    int gi[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) gi[k] = (gb + k < ge) ? __ldg(s.gat_idx + gb + k) : -1;
    double lrow[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) lrow[k] = (row && k < w) ? __ldg(P + k * nr + lane) : 0.0;
    const double bi = own ? rhs_at(a, f + lane) : 0.0;
    // reciprocal of this lane's diagonal entry, off the dependency chain
    const double rdl = own ? 1.0 / __ldg(P + lane * nr + lane) : 1.0;
    if (a.pre_wait & 1) wait_children(a, sn, lane);
    double xv[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) xv[k] = gi[k] >= 0 ? ldcg(a.u + gi[k]) : 0.0;
    double acc = 0.0;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      if (gi[k] >= 0 && __double_as_longlong(xv[k]) == kUnset) xv[k] = poll_value(a.u + gi[k], a.abort);
      acc += xv[k];
    }
    if (ge - gb > 4) acc += gather_u(a, gb + 4, ge);
    acc = own ? bi - acc : acc;
    if (a.trace) { __syncwarp(); if (lane == 0) a.trace[4 * a.s.nsup + tslot] = global_ns(); }
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      if (k < w) {
        const double yk = __shfl_sync(0xffffffffu, acc * rdl, k);
        if (lane == k) acc = yk;
        if (lane > k && lane < w) acc = fma(-lrow[k], yk, acc);
        if (lane >= w && row) acc = fma(lrow[k], yk, acc);
      }
    }
    if (own) stcg(a.y + f + lane, acc);
    if (lane >= w && row) stcg(U + lane - w, acc);
    return;
  }
  if (MID > 0 && nr <= 64 && w <= MID) {
    // Medium supernode: lane owns rows lane and lane + 32.  The same flow as
    // the narrow branch -- every static load (gather lists, panel rows,
    // right-hand side, reciprocal diagonal) before the first wait, the
    // children's values gathered row-side in child order, then a shuffle
    // chain -- instead of the general branch's per-child extend-add and
    // per-chunk panel loads.
    const int q0 = lane, q1 = lane + 32;
    const bool own = lane < w, row0 = q0 < nr, row1 = q1 < nr;
    const int gb0 = row0 ? __ldg(s.gat_ptr + rp + q0) : 0, ge0 = row0 ? __ldg(s.gat_ptr + rp + q0 + 1) : 0;
    const int gb1 = row1 ? __ldg(s.gat_ptr + rp + q1) : 0, ge1 = row1 ? __ldg(s.gat_ptr + rp + q1 + 1) : 0;
    int g0[3], g1[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      g0[k] = (gb0 + k < ge0) ? __ldg(s.gat_idx + gb0 + k) : -1;
      g1[k] = (gb1 + k < ge1) ? __ldg(s.gat_idx + gb1 + k) : -1;
    }
    constexpr int MW = MID > 0 ? MID : 1;
    double p0[MW], p1[MW];
#pragma unroll
    for (int k = 0; k < MW; ++k) {
      p0[k] = (row0 && k < w) ? __ldg(P + k * nr + q0) : 0.0;
      p1[k] = (row1 && k < w) ? __ldg(P + k * nr + q1) : 0.0;
    }
    const double bi = own ? rhs_at(a, f + lane) : 0.0;
    const double rdl = own ? 1.0 / __ldg(P + lane * nr + lane) : 1.0;
    if (a.pre_wait & 2) wait_children(a, sn, lane);
    double A0 = 0.0, A1 = 0.0;
    {
      double v0[3], v1[3];
#pragma unroll
      for (int k = 0; k < 3; ++k) {
        v0[k] = g0[k] >= 0 ? ldcg(a.u + g0[k]) : 0.0;
        v1[k] = g1[k] >= 0 ? ldcg(a.u + g1[k]) : 0.0;
      }
#pragma unroll
      for (int k = 0; k < 3; ++k) {
        if (g0[k] >= 0 && __double_as_longlong(v0[k]) == kUnset) v0[k] = poll_value(a.u + g0[k], a.abort);
        if (g1[k] >= 0 && __double_as_longlong(v1[k]) == kUnset) v1[k] = poll_value(a.u + g1[k], a.abort);
        A0 += v0[k];
        A1 += v1[k];
      }
      if (ge0 - gb0 > 3) A0 += gather_u(a, gb0 + 3, ge0);
      if (ge1 - gb1 > 3) A1 += gather_u(a, gb1 + 3, ge1);
    }
    if (own) A0 = bi - A0;
    if (a.trace) { __syncwarp(); if (lane == 0) a.trace[4 * a.s.nsup + tslot] = global_ns(); }
#pragma unroll
    for (int k = 0; k < MW; ++k) {
      if (k < w) {
        const double yk = __shfl_sync(0xffffffffu, A0 * rdl, k);
        if (lane == k) A0 = yk;
        if (lane > k && lane < w) A0 = fma(-p0[k], yk, A0);
        if (lane >= w && row0) A0 = fma(p0[k], yk, A0);
        if (row1) A1 = fma(p1[k], yk, A1);
      }
    }
    if (own) stcg(a.y + f + lane, A0);
    else if (row0) stcg(U + q0 - w, A0);
    if (row1) stcg(U + q1 - w, A1);
    return;
  }
  // General supernode: A[q] (per-supernode scratch) holds, for own rows,
  // b - (children's contributions) and for rows below, the running update.
  // (the warp's slice of shared memory when the caller has one and the rows fit)
  double* A = (sA && nr <= kWarpRows) ? sA : a.acc_buf + rp;
  if (a.prefetch) {  // static data of the extend-add and the panel, into L1 before the wait
    prefetch_l1(P, 8ll * w * nr, lane);
    for (int c = s.child_ptr[sn]; c < s.child_ptr[sn + 1]; ++c) {
      const int ch = s.child[c];
      prefetch_l1(s.relind + s.u_off[ch], 4ll * (s.nrows[ch] - (s.first[ch + 1] - s.first[ch])), lane);
    }
  }
  for (int q = lane; q < nr; q += 32) A[q] = q < w ? rhs_at(a, f + q) : 0.0;
  __syncwarp();
  if (a.pre_wait & 2) wait_children(a, sn, lane);
  // Extend-add the children's update vectors (child-side relative indices:
  // coalesced, four loads in flight per lane).
  for (int c = s.child_ptr[sn]; c < s.child_ptr[sn + 1]; ++c) {
    const int ch = s.child[c];
    const int m = s.nrows[ch] - (s.first[ch + 1] - s.first[ch]);
    const double* uc = a.u + s.u_off[ch];
    const int* rel = s.relind + s.u_off[ch];
    for (int tb = 0; tb < m; tb += 128) {
      int q[4];
      double v[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int t = tb + lane + 32 * j;
        q[j] = t < m ? __ldg(rel + t) : -1;
        v[j] = t < m ? ldcg(uc + t) : 0.0;
      }
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        if (q[j] >= 0) {
          if (__double_as_longlong(v[j]) == kUnset) v[j] = poll_value(uc + tb + lane + 32 * j, a.abort);
          A[q[j]] += (q[j] < w) ? -v[j] : v[j];
        }
      }
    }
    __syncwarp();
  }
  for (int cb = 0; cb < w; cb += 32) {
    const int cw = min(32, w - cb);
    double d[32];  // row cb+lane of the chunk's diagonal block, all loads in flight
#pragma unroll
    for (int k = 0; k < 32; ++k) d[k] = (k < cw && lane < cw) ? __ldg(P + (cb + k) * nr + cb + lane) : 0.0;
    const double rdl = lane < cw ? 1.0 / __ldg(P + (cb + lane) * nr + cb + lane) : 1.0;
    double acc = lane < cw ? A[cb + lane] : 0.0;
#pragma unroll
    for (int k = 0; k < 32; ++k) {
      if (k < cw) {
        const double yk = __shfl_sync(0xffffffffu, acc * rdl, k);
        if (lane == k) acc = yk;
        if (lane > k && lane < cw) acc = fma(-d[k], yk, acc);
      }
    }
    if (lane < cw) stcg(a.y + f + cb + lane, acc);
    for (int qb = cb + cw; qb < nr; qb += 32) {  // warp-uniform trip count
      const int q = qb + lane;
      double t = 0.0;
#pragma unroll
      for (int k = 0; k < 32; ++k) {
        if (k < cw) {
          const double yk = __shfl_sync(0xffffffffu, acc, k);
          if (q < nr) t = fma(__ldg(P + (cb + k) * nr + q), yk, t);
        }
      }
      if (q < nr) A[q] += (q < w) ? -t : t;
    }
    __syncwarp();
  }
  for (int q = w + lane; q < nr; q += 32) stcg(U + q - w, A[q]);
}

// The parent publishes its first column last; once it is visible every
// ancestor value this task reads has been written.  One lane polls.
__device__ __forceinline__ void wait_parent(const TrsvArgs& a, int sn, int lane) {
  const int par = a.s.parent[sn];
  if (lane == 0) poll_value(par >= 0 ? a.x + a.s.first[par] : a.y + a.s.first[sn], a.abort);
  __syncwarp();
}

template <int MID>
__device__ __forceinline__ void bwd_task(const TrsvArgs& a, int sn, int lane, int tslot) {
  const SnPlan& s = a.s;
  const int f = s.first[sn], w = s.first[sn + 1] - f, nr = s.nrows[sn];
  const double* P = a.panel + s.off[sn];
  const int* R = s.rows + s.rows_ptr[sn];
  if (w <= 4 && nr - w <= 32) {
    // Narrow: lane r owns below row w + r; lane l < w owns column l.
    const int below = nr - w;
    int gr = 0;
    double lv[4], ld[4];
    if (lane < below) gr = __ldg(R + w + lane);
#pragma unroll
    for (int k = 0; k < 4; ++k) lv[k] = (lane < below && k < w) ? __ldg(P + k * nr + w + lane) : 0.0;
#pragma unroll
    for (int k = 0; k < 4; ++k) ld[k] = (lane < w && k < w) ? __ldg(P + lane * nr + k) : 0.0;  // L(k, lane)
    const double rdl = lane < w ? 1.0 / __ldg(P + lane * nr + lane) : 1.0;
    if (a.pre_wait & 4) wait_parent(a, sn, lane);
    double acc = lane < w ? load_ready(a.y + f + lane, a.abort) : 0.0;
    const double xr = lane < below ? load_ready(a.x + gr, a.abort) : 0.0;
    if (a.trace) { __syncwarp(); if (lane == 0) a.trace[4 * a.s.nsup + tslot] = global_ns(); }
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      if (k < w) {
        const double t = warp_sum(lv[k] * xr);
        if (lane == k) acc -= t;
      }
    }
#pragma unroll
    for (int k = 3; k >= 0; --k) {
      if (k < w) {
        const double xk = __shfl_sync(0xffffffffu, acc * rdl, k);
        if (lane == k) acc = xk;
        if (lane < k) acc = fma(-ld[k], xk, acc);
      }
    }
    if (lane < w) {
      stcg(a.x + f + lane, acc);
      if (a.x_out) a.x_out[s.perm[f + lane]] = acc;
    }
    return;
  }
  if (MID > 0 && w <= MID && nr - w <= 64) {
    // Medium supernode: lanes hold the rows below (two each, x gathered
    // once), column sums by warp reductions, then the diagonal block's chain
    // with lane = column; all static loads before the wait.
    const int below = nr - w, r0 = lane, r1 = lane + 32;
    const int gr0 = r0 < below ? __ldg(R + w + r0) : 0, gr1 = r1 < below ? __ldg(R + w + r1) : 0;
    constexpr int MW = MID > 0 ? MID : 1;
    double l0[MW], l1[MW], ld[MW];
#pragma unroll
    for (int k = 0; k < MW; ++k) {
      l0[k] = (r0 < below && k < w) ? __ldg(P + k * nr + w + r0) : 0.0;
      l1[k] = (r1 < below && k < w) ? __ldg(P + k * nr + w + r1) : 0.0;
      ld[k] = (lane < w && k < w) ? __ldg(P + lane * nr + k) : 0.0;  // L(k, lane)
    }
    const double rdl = lane < w ? 1.0 / __ldg(P + lane * nr + lane) : 1.0;
    if (a.pre_wait & 8) wait_parent(a, sn, lane);
    double acc = lane < w ? load_ready(a.y + f + lane, a.abort) : 0.0;
    const double x0 = r0 < below ? load_ready(a.x + gr0, a.abort) : 0.0;
    const double x1 = r1 < below ? load_ready(a.x + gr1, a.abort) : 0.0;
    if (a.trace) { __syncwarp(); if (lane == 0) a.trace[4 * a.s.nsup + tslot] = global_ns(); }
#pragma unroll
    for (int k = 0; k < MW; ++k) {
      if (k < w) {
        const double t = warp_sum(fma(l1[k], x1, l0[k] * x0));
        if (lane == k) acc -= t;
      }
    }
#pragma unroll
    for (int k = MW - 1; k >= 0; --k) {
      if (k < w) {
        const double xk = __shfl_sync(0xffffffffu, acc * rdl, k);
        if (lane == k) acc = xk;
        if (lane < k) acc = fma(-ld[k], xk, acc);
      }
    }
    if (lane < w) {
      stcg(a.x + f + lane, acc);
      if (a.x_out) a.x_out[s.perm[f + lane]] = acc;
    }
    return;
  }
  const int nchunks = (w + 31) >> 5;
  if (a.prefetch) {  // panel and row indices into L1 before the wait
    prefetch_l1(P, 8ll * w * nr, lane);
    prefetch_l1(R, 4ll * nr, lane);
  }
  for (int ci = nchunks - 1; ci >= 0; --ci) {
    const int cb = ci * 32, cw = min(32, w - cb);
    double d[32];  // column cb+lane of the chunk's diagonal block: L(cb+k, cb+lane)
#pragma unroll
    for (int k = 0; k < 32; ++k) d[k] = (k < cw && lane < cw) ? __ldg(P + (cb + lane) * nr + cb + k) : 0.0;
    const double rdl = lane < cw ? 1.0 / __ldg(P + (cb + lane) * nr + cb + lane) : 1.0;
    if (ci == nchunks - 1 && (a.pre_wait & 8)) wait_parent(a, sn, lane);
    double acc = lane < cw ? load_ready(a.y + f + cb + lane, a.abort) : 0.0;
    const int rb0 = cb + cw;  // rows below this chunk (own later chunks + ancestors)
    double t = 0.0;           // lane = column: sum_r L(r, cb+lane) x_r
    for (int rb = rb0; rb < nr; rb += 32) {
      const int r = rb + lane;
      const double xr = r < nr ? load_ready(a.x + __ldg(R + r), a.abort) : 0.0;
#pragma unroll
      for (int qq = 0; qq < 32; ++qq) {
        const double xq = __shfl_sync(0xffffffffu, xr, qq);
        if (lane < cw && rb + qq < nr) t = fma(__ldg(P + (cb + lane) * nr + rb + qq), xq, t);
      }
    }
    acc -= t;
#pragma unroll
    for (int k = 31; k >= 0; --k) {
      if (k < cw) {
        const double xk = __shfl_sync(0xffffffffu, acc * rdl, k);
        if (lane == k) acc = xk;
        if (lane < k) acc = fma(-d[k], xk, acc);
      }
    }
    if (lane < cw) {
      stcg(a.x + f + cb + lane, acc);
      if (a.x_out) a.x_out[s.perm[f + cb + lane]] = acc;
    }
    __syncwarp();
  }
}

// Wide supernode, forward, whole CTA (multifrontal form as fwd_task):
// A (shared) = b - children's contributions for own rows, running update for
// rows below; per 32-column chunk warp 0 solves the diagonal block (shuffle
// chain, reciprocal of the diagonal off the chain), then one thread per row
// applies the chunk to the rows below with all 32 panel loads in flight.
__device__ void fwd_cta(const TrsvArgs& a, TrsvSmem& S, int sn) {
  const SnPlan& s = a.s;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int f = s.first[sn], w = s.first[sn + 1] - f, nr = s.nrows[sn];
  const double* P = a.panel + s.off[sn];
  double* U = a.u + s.u_off[sn];
  double* A = S.a;
  if (a.cta_gather) {
    // row-side gathers of the children's update values (every row at once,
    // four loads in flight): no barrier per child
    const int rp = s.rows_ptr[sn];
    for (int q = tid; q < nr; q += blockDim.x) {
      const double g = gather_u(a, __ldg(s.gat_ptr + rp + q), __ldg(s.gat_ptr + rp + q + 1));
      A[q] = q < w ? rhs_at(a, f + q) - g : g;
    }
    __syncthreads();
  } else {
  for (int q = tid; q < nr; q += blockDim.x) A[q] = q < w ? rhs_at(a, f + q) : 0.0;
  for (int c = s.child_ptr[sn] + tid; c < s.child_ptr[sn + 1]; c += blockDim.x) {
    const int ch = s.child[c];
    poll_value(a.u + s.u_off[ch + 1] - 1, a.abort);
  }
  __syncthreads();
  for (int c = s.child_ptr[sn]; c < s.child_ptr[sn + 1]; ++c) {
    const int ch = s.child[c];
    const int m = s.nrows[ch] - (s.first[ch + 1] - s.first[ch]);
    const double* uc = a.u + s.u_off[ch];
    const int* rel = s.relind + s.u_off[ch];
    for (int t = tid; t < m; t += blockDim.x) {
      const int q = __ldg(rel + t);
      const double v = load_ready(uc + t, a.abort);
      A[q] += (q < w) ? -v : v;
    }
    __syncthreads();
  }
  }
  for (int cb = 0; cb < w; cb += 32) {
    const int cw = min(32, w - cb);
    if (wid == 0) {
      const int rl = cb + min(lane, cw - 1);
      double d[32];
#pragma unroll
      for (int k = 0; k < 32; ++k) d[k] = __ldg(P + (cb + min(k, cw - 1)) * nr + rl);
      const double rd = 1.0 / __ldg(P + rl * nr + rl);
      double acc = lane < cw ? A[cb + lane] : 0.0;
#pragma unroll
      for (int k = 0; k < 32; ++k) {
        if (k < cw) {
          const double yk = __shfl_sync(0xffffffffu, acc, k) * __shfl_sync(0xffffffffu, rd, k);
          if (lane == k) acc = yk;
          if (lane > k && lane < cw) acc = fma(-d[k], yk, acc);
        }
      }
      if (lane < cw) {
        A[cb + lane] = acc;
        stcg(a.y + f + cb + lane, acc);
      }
    }
    __syncthreads();
    for (int q = cb + cw + tid; q < nr; q += blockDim.x) {
      double l[32];
#pragma unroll
      for (int k = 0; k < 32; ++k) l[k] = __ldg(P + (cb + min(k, cw - 1)) * nr + q);
      double t = 0.0;
#pragma unroll
      for (int k = 0; k < 32; ++k) {
        if (k < cw) t = fma(l[k], A[cb + k], t);
      }
      A[q] += (q < w) ? -t : t;
    }
    __syncthreads();
  }
  for (int q = w + tid; q < nr; q += blockDim.x) stcg(U + q - w, A[q]);
}

// Wide supernode, backward, whole CTA: X (shared) holds the solution at the
// panel's rows; per chunk (last first) the below-chunk dot products are split
// over 8 row slices per column and combined in a fixed order, then warp 0
// runs the backward chain of the diagonal block.  The first chunk (holding
// the supernode's first column, which children poll) is written last.
__device__ void bwd_cta(const TrsvArgs& a, TrsvSmem& S, int sn) {
  const SnPlan& s = a.s;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int f = s.first[sn], w = s.first[sn + 1] - f, nr = s.nrows[sn];
  const double* P = a.panel + s.off[sn];
  const int* R = s.rows + s.rows_ptr[sn];
  double* X = S.a;
  const int par = s.parent[sn];
  if (tid == 0) poll_value(par >= 0 ? a.x + s.first[par] : a.y + f, a.abort);
  __syncthreads();
  for (int r = w + tid; r < nr; r += blockDim.x) X[r] = load_ready(a.x + __ldg(R + r), a.abort);
  __syncthreads();
  const int nchunks = (w + 31) >> 5;
  const int col = tid >> 3, slice = tid & 7;  // 32 columns x 8 row slices
  for (int ci = nchunks - 1; ci >= 0; --ci) {
    const int cb = ci * 32, cw = min(32, w - cb), rb0 = cb + cw;
    double t = 0.0;
    if (col < cw) {
      const double* Pc = P + (cb + col) * nr;
      int r = rb0 + slice;
      for (; r + 24 < nr; r += 32) {
        t = fma(__ldg(Pc + r), X[r], t);
        t = fma(__ldg(Pc + r + 8), X[r + 8], t);
        t = fma(__ldg(Pc + r + 16), X[r + 16], t);
        t = fma(__ldg(Pc + r + 24), X[r + 24], t);
      }
      for (; r < nr; r += 8) t = fma(__ldg(Pc + r), X[r], t);
    }
    t += __shfl_xor_sync(0xffffffffu, t, 1);
    t += __shfl_xor_sync(0xffffffffu, t, 2);
    t += __shfl_xor_sync(0xffffffffu, t, 4);
    if (slice == 0) S.t[col] = t;
    __syncthreads();
    if (wid == 0) {
      const int cl = cb + min(lane, cw - 1);
      double d[32];  // L(cb+k, cb+lane)
#pragma unroll
      for (int k = 0; k < 32; ++k) d[k] = __ldg(P + cl * nr + cb + min(k, cw - 1));
      const double rd = 1.0 / __ldg(P + cl * nr + cl);
      double acc = lane < cw ? load_ready(a.y + f + cb + lane, a.abort) - S.t[lane] : 0.0;
#pragma unroll
      for (int k = 31; k >= 0; --k) {
        if (k < cw) {
          const double xk = __shfl_sync(0xffffffffu, acc, k) * __shfl_sync(0xffffffffu, rd, k);
          if (lane == k) acc = xk;
          if (lane < k) acc = fma(-d[k], xk, acc);
        }
      }
      if (lane < cw) {
        X[cb + lane] = acc;
        if (lane > 0 || ci > 0) stcg(a.x + f + cb + lane, acc);
        if (a.x_out) a.x_out[s.perm[f + cb + lane]] = acc;
      }
      if (ci == 0) {
        __syncwarp();
        if (lane == 0) {
          fence_gpu();
          stcg(a.x + f, acc);
        }
      }
    }
    __syncthreads();
  }
}

// Q-form forward row slice [r0, r1) (<= 32 rows) of wide supernode sn:
// a = b - (children's contributions) on the w own rows (every slice forms
// it), then out_q = sum_k Q[q,k] a_k for its rows, split over the CTA's
// warps by k ranges and combined in a fixed order: own rows -> y, rows
// below -> u_sn (children's contributions to the row added).  Slices of one
// supernode are independent (no intra-supernode synchronisation).
__device__ void qslice_fwd(const TrsvArgs& a, TrsvSmem& S, int sn, int r0, int r1) {
  const SnPlan& s = a.s;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5, nwarp = blockDim.x >> 5;
  const int f = s.first[sn], w = s.first[sn + 1] - f, nr = s.nrows[sn], rp = s.rows_ptr[sn];
  const double* Q = a.q + a.qoff[sn];
  double* A = S.a;  // w own-row values, then the partial sums
  for (int qq = tid; qq < w; qq += blockDim.x)
    A[qq] = rhs_at(a, f + qq) - gather_u(a, __ldg(s.gat_ptr + rp + qq), __ldg(s.gat_ptr + rp + qq + 1));
  __syncthreads();
  const int q = r0 + lane;
  const bool row = q < r1;
  const int kb = (w * wid) / nwarp, ke = (w * (wid + 1)) / nwarp;
  double t0 = 0.0, t1 = 0.0;
  int k = kb;
#pragma unroll 4
  for (; k + 2 <= ke; k += 2) {
    if (row) {
      t0 = fma(__ldg(Q + static_cast<long long>(k) * nr + q), A[k], t0);
      t1 = fma(__ldg(Q + static_cast<long long>(k + 1) * nr + q), A[k + 1], t1);
    }
  }
  if (k < ke && row) t0 = fma(__ldg(Q + static_cast<long long>(k) * nr + q), A[k], t0);
  double* part = A + ((w + 1) & ~1);  // [nwarp][32]
  part[wid * 32 + lane] = t0 + t1;
  __syncthreads();
  if (wid == 0 && row) {
    double out = 0.0;
    for (int j = 0; j < nwarp; ++j) out += part[j * 32 + lane];
    if (q < w) {
      stcg(a.y + f + q, out);
    } else {
      const double g = gather_u(a, __ldg(s.gat_ptr + rp + q), __ldg(s.gat_ptr + rp + q + 1));
      stcg(a.u + s.u_off[sn] + q - w, g + out);
    }
  }
}

// Q-form backward column slice [c0, c1) (<= one column per warp):
// v = [y_own; -x_below] (staged once per slice), x_c = sum_q Q[q,c] v_q.
__device__ void qslice_bwd(const TrsvArgs& a, TrsvSmem& S, int sn, int c0, int c1) {
  const SnPlan& s = a.s;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5, nwarp = blockDim.x >> 5;
  const int f = s.first[sn], w = s.first[sn + 1] - f, nr = s.nrows[sn];
  const int* R = s.rows + s.rows_ptr[sn];
  const double* Q = a.q + a.qoff[sn];
  double* V = S.a;
  for (int qq = tid; qq < nr; qq += blockDim.x)
    V[qq] = qq < w ? load_ready(a.y + f + qq, a.abort) : -load_ready(a.x + __ldg(R + qq), a.abort);
  __syncthreads();
  for (int c = c0 + wid; c < c1; c += nwarp) {
    const double* Qc = Q + static_cast<long long>(c) * nr;
    double t0 = 0.0, t1 = 0.0;
    int qq = lane;
#pragma unroll 4
    for (; qq + 32 < nr; qq += 64) {
      t0 = fma(__ldg(Qc + qq), V[qq], t0);
      t1 = fma(__ldg(Qc + qq + 32), V[qq + 32], t1);
    }
    if (qq < nr) t0 = fma(__ldg(Qc + qq), V[qq], t0);
    const double xc = warp_sum(t0 + t1);
    if (lane == 0) {
      stcg(a.x + f + c, xc);
      if (a.x_out) a.x_out[s.perm[f + c]] = xc;
    }
  }
  __syncthreads();
}

// Q = [L_ss^-1; L_below L_ss^-1] of the Q-form supernodes, one warp per
// row q: Q[q,k] = (E[q,k] - sum_{j>k} Q[q,j] L[j,k]) / L[k,k] for
// k = w-1 .. 0, E = [I; L_below] (the row of Q times L_ss equals E's row).
// The row lives in registers (lane holds columns lane + 32 i).
constexpr int kQMaxW = 512;
__global__ void __launch_bounds__(256) k_qform(int nrows_total, const int2* __restrict__ items, SnPlan s,
                                               const double* __restrict__ panel, const long long* __restrict__ qoff,
                                               double* __restrict__ q) {
  const int item = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (item >= nrows_total) return;
  const int2 it = items[item];
  const int sn = it.x, qr = it.y;
  const int f = s.first[sn], w = s.first[sn + 1] - f, nr = s.nrows[sn];
  const double* P = panel + s.off[sn];
  double* Qo = q + qoff[sn];
  constexpr int NC = kQMaxW / 32;
  double v[NC];
#pragma unroll
  for (int i = 0; i < NC; ++i) v[i] = 0.0;
  // own rows: M = L_ss^-1 is lower triangular, Q[qr, k] = 0 for k > qr
  for (int k = qr < w ? qr : w - 1; k >= 0; --k) {
    // the reciprocal diagonal does not depend on the chain (no FP64 division on it)
    const double rd = 1.0 / __ldg(P + static_cast<long long>(k) * nr + k);
    const double e = qr < w ? (qr == k ? 1.0 : 0.0) : __ldg(P + static_cast<long long>(k) * nr + qr);
    double t = 0.0;
#pragma unroll
    for (int i = 0; i < NC; ++i) {
      const int j = lane + 32 * i;
      if (j > k && j < w) t = fma(v[i], __ldg(P + static_cast<long long>(k) * nr + j), t);
    }
    t = warp_sum(t);
    const double qk = (e - t) * rd;
#pragma unroll
    for (int i = 0; i < NC; ++i) {
      if (lane + 32 * i == k) v[i] = qk;
    }
  }
#pragma unroll
  for (int i = 0; i < NC; ++i) {
    const int j = lane + 32 * i;
    if (j < w) Qo[static_cast<long long>(j) * nr + qr] = v[i];
  }
}

// Bottom-level supernode, forward, one thread (w <= W, nrows <= NR): the
// same arithmetic in the same order as fwd_task's narrow branch.
template <int NR, int W>
__device__ __forceinline__ void fwd_thread(const TrsvArgs& a, int sn) {
  // Bottom levels are grid-synchronous: every value read here is complete,
  // so nothing is polled and the loads of all rows are issued together
  // (row bounds, then the first two gather indices of every row, then their
  // values); rows with more gathers finish in a second pass.  Same sums in
  // the same order as the polling form.
  const SnPlan& s = a.s;
  const int f = s.first[sn], w = s.first[sn + 1] - f, nr = s.nrows[sn];
  const int rp = s.rows_ptr[sn];
  const double* P = a.panel + s.off[sn];
  int gp[NR + 1];
#pragma unroll
  for (int q = 0; q <= NR; ++q) gp[q] = q <= nr ? __ldg(s.gat_ptr + rp + q) : 0;
  double rb[W];
#pragma unroll
  for (int q = 0; q < W; ++q) rb[q] = q < w ? (a.bt_all ? ldcg(a.bt + f + q) : rhs_raw(a, f + q)) : 0.0;
  int i0[NR], i1[NR];
#pragma unroll
  for (int q = 0; q < NR; ++q) {
    const bool row = q < nr;
    i0[q] = (row && gp[q] < gp[q + 1]) ? __ldg(s.gat_idx + gp[q]) : -1;
    i1[q] = (row && gp[q] + 1 < gp[q + 1]) ? __ldg(s.gat_idx + gp[q] + 1) : -1;
  }
  double acc[NR];
#pragma unroll
  for (int q = 0; q < NR; ++q) {
    const double v0 = i0[q] >= 0 ? ldcg(a.u + i0[q]) : 0.0;
    const double v1 = i1[q] >= 0 ? ldcg(a.u + i1[q]) : 0.0;
    double g = 0.0;
    g += v0;
    g += v1;
    acc[q] = g;
  }
#pragma unroll
  for (int q = 0; q < NR; ++q) {
    if (q < nr) {
      for (int e = gp[q] + 2; e < gp[q + 1]; ++e) acc[q] += ldcg(a.u + __ldg(s.gat_idx + e));
      if (q < W && q < w) acc[q] = rb[q < W ? q : 0] - acc[q];
    } else {
      acc[q] = 0.0;
    }
  }
  double rd[W];
#pragma unroll
  for (int k = 0; k < W; ++k) rd[k] = k < w ? 1.0 / __ldg(P + k * nr + k) : 1.0;
#pragma unroll
  for (int k = 0; k < W; ++k) {
    if (k < w) {
      const double yk = acc[k] * rd[k];
      acc[k] = yk;
#pragma unroll
      for (int q = k + 1; q < NR; ++q) {
        if (q < nr) {
          const double l = __ldg(P + k * nr + q);
          acc[q] = q < w ? fma(-l, yk, acc[q]) : fma(l, yk, acc[q]);
        }
      }
    }
  }
  double* U = a.u + s.u_off[sn];
#pragma unroll
  for (int q = 0; q < NR; ++q) {
    if (q < w) stcg(a.y + f + q, acc[q]);
    else if (q < nr) stcg(U + q - w, acc[q]);
  }
}

template <int NR, int W>
__device__ __forceinline__ void bwd_thread(const TrsvArgs& a, int sn) {
  const SnPlan& s = a.s;
  const int f = s.first[sn], w = s.first[sn + 1] - f, nr = s.nrows[sn];
  const double* P = a.panel + s.off[sn];
  const int* R = s.rows + s.rows_ptr[sn];
  // grid-synchronous bottom level (see fwd_thread): plain loads, all in flight
  double xb[NR], acc[W];
  int gr[NR];
#pragma unroll
  for (int r = 0; r < NR; ++r) gr[r] = (r >= w && r < nr) ? __ldg(R + r) : -1;
#pragma unroll
  for (int r = 0; r < NR; ++r) xb[r] = gr[r] >= 0 ? ldcg(a.x + gr[r]) : 0.0;
#pragma unroll
  for (int k = 0; k < W; ++k) {
    acc[k] = 0.0;
    if (k < w) {
      double t = 0.0;
#pragma unroll
      for (int r = 0; r < NR; ++r) {
        if (r >= w && r < nr) t = fma(__ldg(P + k * nr + r), xb[r], t);
      }
      acc[k] = ldcg(a.y + f + k) - t;
    }
  }
  double rd[W];
#pragma unroll
  for (int k = 0; k < W; ++k) rd[k] = k < w ? 1.0 / __ldg(P + k * nr + k) : 1.0;
#pragma unroll
  for (int k = W - 1; k >= 0; --k) {
    if (k < w) {
      const double xk = acc[k] * rd[k];
      acc[k] = xk;
#pragma unroll
      for (int j = 0; j < k; ++j) acc[j] = fma(-__ldg(P + j * nr + k), xk, acc[j]);
    }
  }
#pragma unroll
  for (int k = 0; k < W; ++k) {
    if (k < w) {
      stcg(a.x + f + k, acc[k]);
      if (a.x_out) a.x_out[s.perm[f + k]] = acc[k];
    }
  }
}

// Bottom levels, forward (levels ascending) or backward (descending), one
// grid barrier after each level.
__device__ __forceinline__ void trsv_bottom(const TrsvArgs& a, bool fwd) {
  const int gt = blockIdx.x * blockDim.x + threadIdx.x, gs = gridDim.x * blockDim.x;
  for (int li = 0; li < a.nbot; ++li) {
    const int l = fwd ? li : a.nbot - 1 - li;
    if (fwd && li == 0 && a.bt_fill && !a.bt_all) {
      for (int k = gt; k < a.nbt_rows; k += gs) {
        const int r = __ldg(a.bt_rows + k);
        a.bt_fill[r] = rhs_raw(a, r);
      }
    }
    const bool wide = a.bot_wide[l];
    for (int i = a.bot_ptr[l] + gt; i < a.bot_ptr[l + 1]; i += gs) {
      if (wide) {
        if (fwd) fwd_thread<32, 8>(a, a.bot_sn[i]);
        else bwd_thread<32, 8>(a, a.bot_sn[i]);
      } else {
        if (fwd) fwd_thread<16, 4>(a, a.bot_sn[i]);
        else bwd_thread<16, 4>(a, a.bot_sn[i]);
      }
    }
    grid_sync(a.bar, a.abort);
  }
}

// A chain of single-child narrow supernodes (w <= 4, rows <= 32, at most
// 32 members), forward, one warp: member i+1's static data (panel rows,
// right-hand side, reciprocal diagonal, hand-off lanes) is loaded while
// member i is solved, and member i's update values reach member i+1 by
// shuffles (chain_fsrc), so a chain link costs no memory round trip.  Only
// the lowest member gathers (and polls) its children's update vectors, and
// only the top member stores its update vector.  Same arithmetic as
// fwd_task's narrow branch.
struct ChainStatic {
  double l[4], b, rd;
  int src;
};

__device__ __forceinline__ void chain_fwd_static(const TrsvArgs& a, int f, int w, int nr, int rp, int off,
                                                 int lane, bool first, ChainStatic& c) {
  const double* P = a.panel + off;
  const bool own = lane < w, row = lane < nr;
#pragma unroll
  for (int k = 0; k < 4; ++k) c.l[k] = (row && k < w) ? __ldg(P + k * nr + lane) : 0.0;
  c.b = own ? rhs_at(a, f + lane) : 0.0;
  c.rd = own ? 1.0 / __ldg(P + lane * nr + lane) : 1.0;
  c.src = (!first && row) ? __ldg(a.chain_fsrc + rp + lane) : -1;
}

__device__ __noinline__ void chain_fwd(const TrsvArgs& a, const int* cs, int cn, int lane) {
  const SnPlan& s = a.s;
  // lane k holds member k's supernode and metadata
  const int msn = cs[min(lane, cn - 1)];
  const int mf = s.first[msn], mw = s.first[msn + 1] - mf, mnr = s.nrows[msn];
  const int mrp = s.rows_ptr[msn], moff = s.off[msn], mu = s.u_off[msn];
  ChainStatic cur, nxt;
  chain_fwd_static(a, __shfl_sync(0xffffffffu, mf, 0), __shfl_sync(0xffffffffu, mw, 0),
                   __shfl_sync(0xffffffffu, mnr, 0), __shfl_sync(0xffffffffu, mrp, 0),
                   __shfl_sync(0xffffffffu, moff, 0), lane, true, cur);
  double prev = 0.0;
  for (int i = 0; i < cn; ++i) {
    const int f = __shfl_sync(0xffffffffu, mf, i), w = __shfl_sync(0xffffffffu, mw, i);
    const int nr = __shfl_sync(0xffffffffu, mnr, i), rp = __shfl_sync(0xffffffffu, mrp, i);
    if (i + 1 < cn)
      chain_fwd_static(a, __shfl_sync(0xffffffffu, mf, i + 1), __shfl_sync(0xffffffffu, mw, i + 1),
                       __shfl_sync(0xffffffffu, mnr, i + 1), __shfl_sync(0xffffffffu, mrp, i + 1),
                       __shfl_sync(0xffffffffu, moff, i + 1), lane, false, nxt);
    const bool own = lane < w, row = lane < nr;
    double acc = 0.0;
    if (i == 0) {
      const int sn = cs[0];
      if (a.pre_wait & 1) wait_children(a, sn, lane);
      if (row) acc = gather_u(a, __ldg(s.gat_ptr + rp + lane), __ldg(s.gat_ptr + rp + lane + 1));
    } else {
      const double v = __shfl_sync(0xffffffffu, prev, cur.src >= 0 ? cur.src : 0);
      acc = cur.src >= 0 ? 0.0 + v : 0.0;
    }
    acc = own ? cur.b - acc : acc;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      if (k < w) {
        const double yk = __shfl_sync(0xffffffffu, acc * cur.rd, k);
        if (lane == k) acc = yk;
        if (lane > k && lane < w) acc = fma(-cur.l[k], yk, acc);
        if (lane >= w && row) acc = fma(cur.l[k], yk, acc);
      }
    }
    const int uo = __shfl_sync(0xffffffffu, mu, i);  // (every lane: full-mask shuffle)
    if (own) stcg(a.y + f + lane, acc);
    if (i == cn - 1 && lane >= w && row) stcg(a.u + uo + lane - w, acc);
    prev = acc;
    cur = nxt;
  }
}

// Backward counterpart: top member first (x of its rows from memory,
// polled), then down the chain with each member's x of the rows below
// taken from the previous member's registers (chain_bsrc): the member's
// own columns (kind 0) or the rows it had loaded (kind 1).
struct ChainStaticB {
  double lv[4], ld[4], rd, y;
  int src;
};

__device__ __forceinline__ void chain_bwd_static(const TrsvArgs& a, int f, int w, int nr, int rp, int off,
                                                 int lane, bool top, ChainStaticB& c) {
  const double* P = a.panel + off;
  const int below = nr - w;
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    c.lv[k] = (lane < below && k < w) ? __ldg(P + k * nr + w + lane) : 0.0;
    c.ld[k] = (lane < w && k < w) ? __ldg(P + lane * nr + k) : 0.0;
  }
  c.rd = lane < w ? 1.0 / __ldg(P + lane * nr + lane) : 1.0;
  // y is complete once the top member's parent values are (the backward of
  // the chain starts after every forward task); the top member loads it
  // after that wait, the others are prefetched after it
  c.y = (!top && lane < w) ? ldcg(a.y + f + lane) : 0.0;
  c.src = lane < below ? (top ? __ldg(a.s.rows + rp + w + lane) : __ldg(a.chain_bsrc + rp + w + lane)) : -1;
}

__device__ __noinline__ void chain_bwd(const TrsvArgs& a, const int* cs, int cn, int lane) {
  const SnPlan& s = a.s;
  const int msn = cs[min(lane, cn - 1)];
  const int mf = s.first[msn], mw = s.first[msn + 1] - mf, mnr = s.nrows[msn];
  const int mrp = s.rows_ptr[msn], moff = s.off[msn];
  const int t0 = cn - 1;
  ChainStaticB cur, nxt;
  chain_bwd_static(a, __shfl_sync(0xffffffffu, mf, t0), __shfl_sync(0xffffffffu, mw, t0),
                   __shfl_sync(0xffffffffu, mnr, t0), __shfl_sync(0xffffffffu, mrp, t0),
                   __shfl_sync(0xffffffffu, moff, t0), lane, true, cur);
  double pacc = 0.0, pxr = 0.0;
  for (int i = cn - 1; i >= 0; --i) {
    const int f = __shfl_sync(0xffffffffu, mf, i), w = __shfl_sync(0xffffffffu, mw, i);
    const int nr = __shfl_sync(0xffffffffu, mnr, i), below = nr - w;
    double xr = 0.0;
    if (i == cn - 1) {
      if (a.pre_wait & 4) wait_parent(a, cs[i], lane);
      xr = lane < below ? load_ready(a.x + cur.src, a.abort) : 0.0;
      if (lane < w) cur.y = load_ready(a.y + f + lane, a.abort);
    }
    // the next member's static data (its y is complete from here on)
    if (i > 0)
      chain_bwd_static(a, __shfl_sync(0xffffffffu, mf, i - 1), __shfl_sync(0xffffffffu, mw, i - 1),
                       __shfl_sync(0xffffffffu, mnr, i - 1), __shfl_sync(0xffffffffu, mrp, i - 1),
                       __shfl_sync(0xffffffffu, moff, i - 1), lane, false, nxt);
    if (i != cn - 1) {
      const int sl = cur.src & 0xff;
      const double vo = __shfl_sync(0xffffffffu, pacc, cur.src >= 0 ? sl : 0);
      const double vb = __shfl_sync(0xffffffffu, pxr, cur.src >= 0 ? sl : 0);
      xr = cur.src < 0 ? 0.0 : ((cur.src >> 8) ? vb : vo);
    }
    double acc = lane < w ? cur.y : 0.0;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      if (k < w) {
        const double t = warp_sum(cur.lv[k] * xr);
        if (lane == k) acc -= t;
      }
    }
#pragma unroll
    for (int k = 3; k >= 0; --k) {
      if (k < w) {
        const double xk = __shfl_sync(0xffffffffu, acc * cur.rd, k);
        if (lane == k) acc = xk;
        if (lane < k) acc = fma(-cur.ld[k], xk, acc);
      }
    }
    if (lane < w) {
      stcg(a.x + f + lane, acc);
      if (a.x_out) a.x_out[s.perm[f + lane]] = acc;
    }
    pacc = acc;
    pxr = xr;
    cur = nxt;
  }
}

// The narrow-stream tasks as real calls (trsv_pass<true>): a smaller task
// loop, separately allocated registers and the medium (w <= 16) branches;
// measured faster on the smaller trees (C1-C3) together with pre-wait on
// every task kind, slower at C4 (hykkt_cuda.cu picks per analysis;
// DESIGN.md §10).
__device__ __noinline__ void fwd_task_call(const TrsvArgs& a, int sn, int lane, int tslot, double* sA) {
  fwd_task<16>(a, sn, lane, tslot, sA);
}
__device__ __noinline__ void bwd_task_call(const TrsvArgs& a, int sn, int lane, int tslot) {
  bwd_task<16>(a, sn, lane, tslot);
}

// One forward + backward pass; y and x must hold kUnset on entry.
// Task streams, each taken in one topological order per pass:
//   wide supernodes -> CTA tasks (ticket[0]: forward list, then the backward
//                      list) on the first `nwc` CTAs;
//   narrow ones     -> warp tasks, forward (ticket[1]) then backward
//                      (ticket[2]).
// CTAs: narrow CTAs (index >= nwc) run the narrow forward stream, then the
// narrow backward stream.  Wide CTAs below `nwd` are dedicated to the wide
// stream; the other wide CTAs ("flex") first help with the narrow forward
// stream (their warps would otherwise wait for the top of the tree), then
// join the wide stream.  Every wide CTA joins the narrow backward stream once
// the wide stream is exhausted.  Deadlock freedom: a CTA enters the wide
// stream only after its narrow forward work is done, and the narrow backward
// stream only after the wide stream has been fully claimed; with at least one
// dedicated wide CTA, the smallest unfinished task of every stream is held
// by a CTA / warp that is working on it.
template <bool CALL>
__device__ __forceinline__ void trsv_pass(const TrsvArgs& a, TrsvSmem& S) {
  const int tid = threadIdx.x, lane = tid & 31;
  const int ns = a.s.nsup;
  unsigned long long* ps = (a.pstamp && threadIdx.x == 0) ? a.pstamp + 8 * blockIdx.x : nullptr;
  if (a.bt_fill && a.bt_all) {
    // every row's right-hand side, two rows per thread in flight
    const int gt = blockIdx.x * blockDim.x + threadIdx.x, gs = gridDim.x * blockDim.x;
    const int n = a.s.n;
    for (int k = gt; k < n; k += 2 * gs) {
      const int k2 = k + gs;
      const double v1 = rhs_raw(a, k);
      const double v2 = k2 < n ? rhs_raw(a, k2) : 0.0;
      a.bt_fill[k] = v1;
      if (k2 < n) a.bt_fill[k2] = v2;
    }
    grid_sync(a.bar, a.abort);
    if (a.nbot > 0) trsv_bottom(a, true);
  } else if (a.nbot > 0) {
    trsv_bottom(a, true);  // fills bt_fill with level 0 (a grid barrier follows)
  } else if (a.bt_fill) {
    const int gt = blockIdx.x * blockDim.x + threadIdx.x, gs = gridDim.x * blockDim.x;
    for (int k = gt; k < a.nbt_rows; k += gs) {
      const int r = __ldg(a.bt_rows + k);
      a.bt_fill[r] = rhs_raw(a, r);
    }
    grid_sync(a.bar, a.abort);
  }
  if (ps) ps[2] = global_ns();
  const int nt = a.nnar;
  // one narrow-stream entry: e >= 0 one supernode; e < 0 chain -e - 1 of
  // single-child narrow supernodes, solved in order by this warp (forward
  // bottom-up, backward top-down) with no hand-off to another warp
  auto run_entry = [&](long long t, int e) {
    const bool fwd = t < nt;
    const int c0 = e >= 0 ? 0 : a.chain_ptr[-e - 1], cn = e >= 0 ? 1 : a.chain_ptr[-e] - c0;
    if (CALL && e < 0 && a.chain_fsrc) {  // register hand-off along the chain
      if (fwd) chain_fwd(a, a.chain_sn + c0, cn, lane);
      else chain_bwd(a, a.chain_sn + c0, cn, lane);
      __syncwarp();
      return;
    }
    for (int ci = 0; ci < cn; ++ci) {
      const int sn = e >= 0 ? e : a.chain_sn[c0 + (fwd ? ci : cn - 1 - ci)];
      const int slot = fwd ? a.pos[sn] : 2 * ns - 1 - a.pos[sn];
      if (a.trace && lane == 0) a.trace[2 * ns + slot] = global_ns();
      if (CALL) {
        if (fwd) fwd_task_call(a, sn, lane, slot, S.a + (threadIdx.x >> 5) * kWarpRows);
        else bwd_task_call(a, sn, lane, slot);
      } else {
        if (fwd) fwd_task<kInlineMid>(a, sn, lane, slot, S.a + (threadIdx.x >> 5) * kWarpRows);
        else bwd_task<kInlineMid>(a, sn, lane, slot);
      }
      if (a.trace && lane == 0) a.trace[slot] = global_ns();
      __syncwarp();
    }
  };
  auto narrow_fwd = [&]() {
    for (long long t = grab_task(a.ticket + 1, lane); t < nt; t = grab_task(a.ticket + 1, lane))
      run_entry(t, a.nar_sn[t]);
  };
  auto narrow_bwd = [&]() {
    for (long long k = grab_task(a.ticket + 2, lane); k < nt; k = grab_task(a.ticket + 2, lane))
      run_entry(nt + k, a.nar_bwd[k]);
  };
  const bool wide_cta = static_cast<int>(blockIdx.x) < a.nwc;
  if (!wide_cta) {
    narrow_fwd();
    narrow_bwd();
  } else {
    if (static_cast<int>(blockIdx.x) >= a.nwd) {
      narrow_fwd();
      __syncthreads();
    }
    if (a.nqf > 0) {
      // Q-form slices: forward row slices, then backward column slices
      for (;;) {
        if (tid == 0) S.task = static_cast<int>(atomicAdd(a.ticket, 1u));
        __syncthreads();
        const int t = S.task;
        __syncthreads();
        if (t >= a.nqf + a.nqb) break;
        if (t < a.nqf) {
          const int4 e = a.qs_f[t];
          qslice_fwd(a, S, e.x, e.y, e.z);
        } else {
          const int4 e = a.qs_b[t - a.nqf];
          qslice_bwd(a, S, e.x, e.y, e.z);
        }
        __syncthreads();
      }
    } else {
      const int nw = a.nwid;
      for (;;) {
        if (tid == 0) S.task = static_cast<int>(atomicAdd(a.ticket, 1u));
        __syncthreads();
        const int t = S.task;
        __syncthreads();
        if (t >= 2 * nw) break;
        const bool fwd = t < nw;
        const int sn = fwd ? a.wid_sn[t] : a.wid_bwd[t - nw];
        const int slot = fwd ? a.pos[sn] : 2 * ns - 1 - a.pos[sn];
        if (a.trace && tid == 0) a.trace[2 * ns + slot] = global_ns();
        if (fwd) fwd_cta(a, S, sn);
        else bwd_cta(a, S, sn);
        if (a.trace && tid == 0) a.trace[slot] = global_ns();
        __syncthreads();
      }
    }
    narrow_bwd();
  }
  if (ps) ps[3] = global_ns();
  if (a.nbot > 0) {
    grid_sync(a.bar, a.abort);
    if (ps) ps[4] = global_ns();
    trsv_bottom(a, false);
  }
  if (ps) ps[5] = global_ns();
}

__device__ __forceinline__ void rearm(const TrsvArgs& a) {
  reset_unset(a.y, a.s.n);
  reset_unset(a.x, a.s.n);
  reset_unset(a.u, a.s.u_size);
}

template <bool CALL>
__global__ void __launch_bounds__(256, 2) k_trsv(TrsvArgs a) {
  __shared__ TrsvSmem S;
  unsigned long long* ps = (a.pstamp && threadIdx.x == 0) ? a.pstamp + 8 * blockIdx.x : nullptr;
  if (ps) ps[0] = global_ns();
  rearm(a);
  grid_sync(a.bar, a.abort);
  if (ps) ps[1] = global_ns();
  trsv_pass<CALL>(a, S);
  if (ps) ps[7] = global_ns();
}

// L values in forward row-list order (after a successful factorization).
__global__ void k_gather_lrow(int nnz, const int* __restrict__ pos, const double* __restrict__ panel,
                              double* __restrict__ out) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e < nnz) out[e] = panel[pos[e]];
}

// q = J t - r_y style products: out[k] = sum_e J_csr[e] * y[ci_perm[e]]
// (+ sub[k] subtracted), reference spmv scatter order (csc_matrix.cpp:250-254,
// zero entries of t skipped exactly as there).
__device__ __forceinline__ double j_row_dot(int k, const int* rp, const int* ci_perm,
                                            const double* jcsr, const double* y) {
  double acc = 0.0;
  const int e0 = rp[k], e1 = rp[k + 1];
  for (int e = e0; e < e1; e += 4) {  // four entries' loads in flight, summed in order
    int ci[4];
    double jv[4], tv[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      ci[u] = e + u < e1 ? __ldg(ci_perm + e + u) : 0;
      jv[u] = e + u < e1 ? __ldg(jcsr + e + u) : 0.0;
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) tv[u] = e + u < e1 ? ldcg(y + ci[u]) : 0.0;
#pragma unroll
    for (int u = 0; u < 4; ++u)
      if (e + u < e1 && tv[u] != 0.0) acc = __dadd_rn(acc, __dmul_rn(jv[u], tv[u]));
  }
  return acc;
}

// Schur right-hand side J w - r_y (solver.cpp:254-255).
__global__ void k_schur_rhs(int mc, const int* rp, const int* ci_perm,
                            const double* jcsr, const double* y,
                            const double* r_y, double* rhs) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k < mc) rhs[k] = __dsub_rn(j_row_dot(k, rp, ci_perm, jcsr, y), r_y[k]);
}

struct CgResultDev {
  long long iterations;
  double relres;
  int converged;
  int small_quadratic;
};

struct CgArgs {
  TrsvArgs tr;  // rhs.u must point at p; tr.bar is the grid barrier
  int mc;
  const int* jcsr_rp;
  const int* jcsr_ci_perm;
  const double* jcsr;
  const double* rhs;
  double* x;
  double* r;
  double* p;
  double* q;
  double* partials;  // 4 per block
  double delta2;
  double tol;
  double thr;
  long long max_iter;
  CgResultDev* res;
  unsigned* tickets;  // max_iter + 2 task counters, zeroed
  unsigned long long* cstamp;  // diagnostics: per-CTA CG phase times (8 per CTA), or null
};

// Deterministic all-blocks reduction of partials[b * 4 + slot].
__device__ __forceinline__ double reduce_partials(const double* partials, int slot, double* scratch) {
  double v = 0.0;
  for (int b = threadIdx.x; b < gridDim.x; b += blockDim.x) v += ldcg(partials + b * 4 + slot);
  return block_sum(v, scratch);
}

template <int MINB, bool CALL>
__global__ void __launch_bounds__(256, MINB) k_cg(CgArgs a) {
  __shared__ double scratch[33];
  __shared__ TrsvSmem S;
  const int gt = blockIdx.x * blockDim.x + threadIdx.x;
  const int gs = gridDim.x * blockDim.x;
  int* abort = a.tr.abort;
  const GridBarrier bar = a.tr.bar;
  rearm(a.tr);
  double ss = 0.0;
  for (int k = gt; k < a.mc; k += gs) {
    const double v = a.rhs[k];
    a.x[k] = 0.0;
    a.r[k] = v;
    a.p[k] = v;
    ss = fma(v, v, ss);
  }
  ss = block_sum(ss, scratch);
  if (threadIdx.x == 0) a.partials[blockIdx.x * 4] = ss;
  grid_sync(bar, abort);
  const double rhs_norm = sqrt(reduce_partials(a.partials, 0, scratch));
  const bool writer = gt == 0;
  if (rhs_norm == 0.0) {
    if (writer) *a.res = CgResultDev{0, 0.0, 1, 0};
    return;
  }
  double rho = rhs_norm * rhs_norm;
  double r_norm = rhs_norm;
  TrsvArgs tr = a.tr;
  unsigned long long* cs = (a.cstamp && threadIdx.x == 0) ? a.cstamp + 8 * blockIdx.x : nullptr;
  for (long long it = 1; it <= a.max_iter; ++it) {
    tr.ticket = a.tickets + static_cast<long long>(tr.tstride) * it;
    if (cs) cs[0] = global_ns();
    trsv_pass<CALL>(tr, S);
    if (cs) cs[1] = global_ns();
    grid_sync(bar, abort);
    if (cs) cs[2] = global_ns();
    double pq = 0.0, pp = 0.0;
    for (int k = gt; k < a.mc; k += gs) {
      double qk = j_row_dot(k, a.jcsr_rp, a.jcsr_ci_perm, a.jcsr, tr.x);
      const double pk = ldcg(a.p + k);
      if (a.delta2 != 0.0) qk = __dadd_rn(qk, __dmul_rn(a.delta2, pk));
      a.q[k] = qk;
      pq = fma(pk, qk, pq);
      pp = fma(pk, pk, pp);
    }
    pq = block_sum(pq, scratch);
    pp = block_sum(pp, scratch);
    if (threadIdx.x == 0) {
      a.partials[blockIdx.x * 4 + 1] = pq;
      a.partials[blockIdx.x * 4 + 2] = pp;
    }
    if (cs) cs[3] = global_ns();
    grid_sync(bar, abort);
    if (cs) cs[4] = global_ns();
    const double curvature = reduce_partials(a.partials, 1, scratch);
    const double p_norm2 = reduce_partials(a.partials, 2, scratch);
    if (curvature <= a.thr * p_norm2 || ld_relaxed(abort)) {
      if (writer) *a.res = CgResultDev{it - 1, r_norm / rhs_norm, 0, 1};
      return;
    }
    const double alpha = rho / curvature;
    rearm(tr);  // q no longer needs x: re-arm for the next pass
    double rr = 0.0;
    for (int k = gt; k < a.mc; k += gs) {
      a.x[k] = __dadd_rn(a.x[k], __dmul_rn(alpha, ldcg(a.p + k)));
      const double rk = __dsub_rn(a.r[k], __dmul_rn(alpha, a.q[k]));
      a.r[k] = rk;
      rr = fma(rk, rk, rr);
    }
    rr = block_sum(rr, scratch);
    if (threadIdx.x == 0) a.partials[blockIdx.x * 4 + 3] = rr;
    if (cs) cs[5] = global_ns();
    grid_sync(bar, abort);
    if (cs) cs[6] = global_ns();
    r_norm = sqrt(reduce_partials(a.partials, 3, scratch));
    const double relres = r_norm / rhs_norm;
    if (relres <= a.tol) {
      if (writer) *a.res = CgResultDev{it, relres, 1, 0};
      return;
    }
    if (it == a.max_iter) {
      if (writer) *a.res = CgResultDev{it, relres, 0, 0};
      return;
    }
    const double rho_next = r_norm * r_norm;
    const double beta = rho_next / rho;
    rho = rho_next;
    for (int k = gt; k < a.mc; k += gs) {
      a.p[k] = __dadd_rn(a.r[k], __dmul_rn(beta, a.p[k]));
    }
    grid_sync(bar, abort);
  }
  if (writer) *a.res = CgResultDev{0, r_norm / rhs_norm, 0, 0};
}

}  // namespace hykkt::dev
