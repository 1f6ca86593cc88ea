// Pivot-free supernodal numeric Cholesky, one persistent cooperative launch
// per factorization attempt.
//
// Replaces numeric_cholesky (proj/core/src/cholesky.cpp:65-137; left-looking
// simplicial with column link lists) by a left-looking SUPERNODAL variant:
// every supernode is a dense column-major panel (rows x width) and is one
// warp task.  Tasks are dealt round-robin to all resident warps in
// level-sorted (topological) order; a task waits only on its children's
// done flags (sync-free, no per-level launches).  Because tasks are taken in
// topological order and every warp is resident (cooperative launch), the
// smallest unfinished task can always run — no deadlock.  Completion of a
// child implies completion of its whole subtree, so a supernode can pull
// updates from every descendant once its children are done.
//
// Pivot semantics follow cholesky.cpp:116-120: the factorization fails at
// the first (smallest elimination-order) column whose candidate is
// !(pivot > floor) (NaN included); *fail_col receives that column through an
// atomicMin.  Supernodes whose first column lies beyond an already-recorded
// failure skip their work (they cannot change the reported column).
#pragma once

#include "device_util.cuh"

namespace hykkt::dev {

struct SnPlan {
  int n, nsup;
  const int* order;      // level-sorted supernodes
  const int* first;      // nsup + 1
  const int* nrows;
  const int* off;        // panel offsets
  const int* rows_ptr;
  const int* rows;
  const int* parent;
  const int* child_ptr;
  const int* child;
  const int* upd_ptr;
  const int* upd_d;
  const int* upd_off;
  const int* upd_cnt;
  const int* lrow_ptr;
  const int* lrow_col;
  const int* lrow_pos;
  const int* perm;
  const int* iperm;
  const int* u_off;
  const int* ext_ptr;
  const int* ext_map;
  const int* gat_ptr;
  const int* gat_idx;
  const int* relind;
  int u_size;
  // left-looking update u, descendant row ii (from upd_off): position of that
  // row in the target's row structure, at upd_pos[upd_pbase[u] + ii]
  const int* upd_pbase;
  const int* upd_pos;
};

struct FactorArgs {
  SnPlan s;
  double* panel;
  int* done;
  int epoch;
  double floor_abs;          // used when floor_scale_ptr == nullptr
  const double* maxdiag;     // floor = floor_rel * *maxdiag
  double floor_rel;
  int* fail_col;
  int* abort;
  unsigned* ticket;
};

__device__ __forceinline__ int find_row(const int* rows, int lo, int hi, int r) {
  // rows[lo..hi) ascending; r is guaranteed present.
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if (__ldg(rows + mid) <= r) lo = mid; else hi = mid;
  }
  return lo;
}

__device__ void factor_task(const FactorArgs& a, int sn, int lane, double floor_v) {
  const SnPlan& s = a.s;
  const int f = s.first[sn], w = s.first[sn + 1] - f, nr = s.nrows[sn];
  double* P = a.panel + s.off[sn];
  const int* R = s.rows + s.rows_ptr[sn];
  for (int c = s.child_ptr[sn] + lane; c < s.child_ptr[sn + 1]; c += 32) {
    if (!wait_flag(a.done + s.child[c], a.epoch, a.abort)) break;
  }
  __syncwarp();
  // Past a recorded failure the result cannot change the reported column;
  // such supernodes still publish (nobody waits forever) but skip the work.
  const bool ok = __shfl_sync(0xffffffffu, ld_relaxed(a.fail_col), 0) >= f;
  if (ok) {
    // Pull updates from descendants, ascending d.
    for (int u = s.upd_ptr[sn]; u < s.upd_ptr[sn + 1]; ++u) {
      const int d = s.upd_d[u], o = s.upd_off[u], cnt = s.upd_cnt[u];
      const int nrd = s.nrows[d], wd = s.first[d + 1] - s.first[d];
      const double* Pd = a.panel + s.off[d];
      const int* Rd = s.rows + s.rows_ptr[d];
      const int m = nrd - o;
      const int total = m * cnt;
      for (int e = lane; e < total; e += 32) {
        const int jj = e / m, ii = e - jj * m;
        if (ii < jj) continue;
        double dot = 0.0;
        for (int k = 0; k < wd; ++k) {
          dot = fma(ldcg(Pd + k * nrd + o + ii), ldcg(Pd + k * nrd + o + jj), dot);
        }
        const int r = __ldg(Rd + o + ii);
        const int cc = __ldg(Rd + o + jj) - f;
        const int pos = (ii < cnt) ? (r - f) : find_row(R, w, nr, r);
        double* tgt = P + cc * nr + pos;
        stcg(tgt, ldcg(tgt) - dot);
      }
      __syncwarp();
    }
    // Dense right-looking Cholesky of the panel.
    for (int k = 0; k < w; ++k) {
      double* Pk = P + k * nr;
      const double pivot = ldcg(Pk + k);
      if (!(pivot > floor_v)) {
        if (lane == 0) atomicMin(a.fail_col, f + k);
        break;
      }
      const double dk = sqrt(pivot), rdk = 1.0 / dk;
      for (int r = k + 1 + lane; r < nr; r += 32) stcg(Pk + r, ldcg(Pk + r) * rdk);
      __syncwarp();
      if (lane == 0) stcg(Pk + k, dk);
      for (int c = k + 1; c < w; ++c) {
        const double lck = ldcg(Pk + c);
        double* Pc = P + c * nr;
        for (int r = c + lane; r < nr; r += 32) stcg(Pc + r, fma(-ldcg(Pk + r), lck, ldcg(Pc + r)));
      }
      __syncwarp();
    }
  }
  warp_publish(a.done + sn, a.epoch, lane);
}

__global__ void __launch_bounds__(256) k_factor(FactorArgs a) {
  const int lane = threadIdx.x & 31;
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  const double floor_v = fmax(a.maxdiag ? a.floor_rel * *a.maxdiag : a.floor_abs, 0.0);
  (void)gw;
  (void)nw;
  for (long long t = grab_task(a.ticket, lane); t < a.s.nsup; t = grab_task(a.ticket, lane)) {
    factor_task(a, a.s.order[t], lane, floor_v);
  }
}

}  // namespace hykkt::dev
