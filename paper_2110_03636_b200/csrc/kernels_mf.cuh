// Multifrontal supernodal numeric Cholesky for ONE large system (configs
// [1]-[3]), one persistent cooperative launch per factorization attempt.
//
// Same result layout as k_factor (kernels_factor.cuh): every supernode s is a
// dense column-major panel P_s (nrows x width) in the supernodal plan, and the
// factorization semantics follow numeric_cholesky (proj/core/src/
// cholesky.cpp:65-137): pivot-free, failure at the first column whose
// candidate pivot is !(pivot > floor).  The schedule differs: instead of a
// left-looking pull of every descendant's columns (one warp per supernode,
// which leaves the few wide supernodes at the top of the tree — hundreds of
// columns at ACTIVSg70k — to a single warp each), every supernode s passes
// its Schur-complement update matrix
//     U_s = sum_children extend(U_c)[w:, w:] - L21 L21^T      (m x m, m = nrows - width)
// to its parent, which adds it (extend-add through the plan's relind map) into
// its own panel / update matrix.  The work is then dense: a blocked Cholesky
// of the panel (32-column blocks: GEMM update from the previous blocks, a
// warp-level factor of the diagonal block, a per-row triangular solve of the
// rows below) and one SYRK for U_s, tiled through shared memory with register
// blocking.  On B200 the FP64 FMA pipe and the FP64 tensor path have the same
// nominal peak (~40 TF/s), so the tiles use DFMA.
//
// Scheduling: host-built task list in level order; a task is either ONE wide
// supernode (nrows >= big threshold) processed by the whole CTA, or up to 8
// narrow supernodes of one level, one per warp.  CTAs take tasks from a
// ticket in order and wait on their children's done flags; as every CTA is
// resident (cooperative launch) and holds one task, the smallest unfinished
// task always has its dependencies running -> no deadlock.  Sums are formed in
// a fixed order (children in plan order, k ascending inside each tile), so the
// factor is bit-reproducible run to run.
#pragma once

#include "kernels_factor.cuh"

namespace hykkt::dev {

struct MfArgs {
  SnPlan s;
  double* panel;
  double* ubuf;               // update matrices, U_s at uoff[s] (m x m column-major, lower used)
  const long long* uoff;      // nsup + 1
  const int* task_ptr;        // ntasks + 1 (into task_sn)
  const int* task_sn;
  const unsigned char* task_big;
  int ntasks;
  int* done;
  int epoch;
  double floor_abs;
  const double* maxdiag;
  double floor_rel;
  int* fail_col;
  int* abort;
  unsigned* ticket;
};

constexpr int kMfThreads = 256;
constexpr int kMfNb = 32;   // column block of the wide-panel factor
constexpr int kMfBM = 64;   // GEMM tile rows
constexpr int kMfBK = 32;   // GEMM k-tile

struct MfSmem {
  double a[kMfBK][kMfBM + 1];
  double b[kMfBK][kMfBM + 1];
  double d[kMfNb][kMfNb + 1];  // diagonal block, d[col][row]
  double rdiag[kMfNb];          // reciprocals of its diagonal
  int task, first, count, big, stop;
};

// C[i + j ldc] -= sum_k A[i + k lda] B[j + k ldb] for i < M, j < N, stored
// only where i + diag >= j (lower part relative to the diagonal offset).
// Whole CTA; operands read through L2.
template <int BN>
__device__ void mf_gemm_nt_sub(MfSmem& S, double* C, int ldc, const double* A, int lda, const double* B, int ldb,
                               int M, int N, int K, int diag) {
  constexpr int TM = kMfBM / 16, TN = BN / 16;
  constexpr int LA = kMfBK * kMfBM / kMfThreads, LB = kMfBK * BN / kMfThreads;  // loads per thread
  const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
  const int tiles_m = (M + kMfBM - 1) / kMfBM, tiles_n = (N + BN - 1) / BN;
  for (int tile = 0; tile < tiles_m * tiles_n; ++tile) {
    const int tm = tile % tiles_m, tn = tile / tiles_m;
    const int i0 = tm * kMfBM, j0 = tn * BN;
    if (i0 + kMfBM - 1 + diag < j0) continue;  // tile entirely above the diagonal
    double acc[TM][TN];
#pragma unroll
    for (int p = 0; p < TM; ++p)
#pragma unroll
      for (int q = 0; q < TN; ++q) acc[p][q] = 0.0;
    // k-tiles are prefetched into registers one tile ahead, so their L2
    // latency overlaps the previous tile's FMAs
    double ra[LA], rb[LB];
    auto load = [&](int k0) {
#pragma unroll
      for (int l = 0; l < LA; ++l) {
        const int e = tid + l * kMfThreads, i = e % kMfBM, k = e / kMfBM;
        ra[l] = (i0 + i < M && k0 + k < K) ? ldcg(A + (i0 + i) + static_cast<long long>(k0 + k) * lda) : 0.0;
      }
#pragma unroll
      for (int l = 0; l < LB; ++l) {
        const int e = tid + l * kMfThreads, j = e % BN, k = e / BN;
        rb[l] = (j0 + j < N && k0 + k < K) ? ldcg(B + (j0 + j) + static_cast<long long>(k0 + k) * ldb) : 0.0;
      }
    };
    load(0);
    for (int k0 = 0; k0 < K; k0 += kMfBK) {
      __syncthreads();
#pragma unroll
      for (int l = 0; l < LA; ++l) {
        const int e = tid + l * kMfThreads;
        S.a[e / kMfBM][e % kMfBM] = ra[l];
      }
#pragma unroll
      for (int l = 0; l < LB; ++l) {
        const int e = tid + l * kMfThreads;
        S.b[e / BN][e % BN] = rb[l];
      }
      __syncthreads();
      if (k0 + kMfBK < K) load(k0 + kMfBK);
#pragma unroll 8
      for (int k = 0; k < kMfBK; ++k) {
        double av[TM], bv[TN];
#pragma unroll
        for (int p = 0; p < TM; ++p) av[p] = S.a[k][ty + 16 * p];
#pragma unroll
        for (int q = 0; q < TN; ++q) bv[q] = S.b[k][tx + 16 * q];
#pragma unroll
        for (int p = 0; p < TM; ++p)
#pragma unroll
          for (int q = 0; q < TN; ++q) acc[p][q] = fma(av[p], bv[q], acc[p][q]);
      }
    }
#pragma unroll
    for (int p = 0; p < TM; ++p) {
#pragma unroll
      for (int q = 0; q < TN; ++q) {
        const int i = i0 + ty + 16 * p, j = j0 + tx + 16 * q;
        if (i < M && j < N && i + diag >= j) {
          double* c = C + i + static_cast<long long>(j) * ldc;
          *c = ldcg(c) - acc[p][q];
        }
      }
    }
  }
  __syncthreads();
}

// extend-add of child c's update matrix into supernode s (panel columns or U_s)
// by `nt` threads starting at thread t of the group.
__device__ __forceinline__ void mf_extend_add(const MfArgs& a, int s, int c, double* P, int nr, int w, double* U,
                                              int m, int t, int nt) {
  const SnPlan& p = a.s;
  const int mcc = p.nrows[c] - (p.first[c + 1] - p.first[c]);
  const double* Uc = a.ubuf + a.uoff[c];
  const int* ri = p.relind + p.u_off[c];
  // lower triangle of Uc over the flattened square (e = t1 + t2 mcc), four
  // entries per thread in flight: the map is injective within one child, so
  // the four read-modify-writes never alias
  const long long tot = static_cast<long long>(mcc) * mcc;
  for (long long e0 = t; e0 < tot; e0 += 4ll * nt) {
    double v[4];
    double* q[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const long long e = e0 + static_cast<long long>(j) * nt;
      q[j] = nullptr;
      v[j] = 0.0;
      if (e < tot) {  // tot = mcc^2 < 2^31: 32-bit index split (a 64-bit division costs ~5x more)
        const int ei = static_cast<int>(e), t2 = ei / mcc, t1 = ei - t2 * mcc;
        if (t1 >= t2) {
          const int r1 = __ldg(ri + t1), r2 = __ldg(ri + t2);
          v[j] = ldcg(Uc + e);
          q[j] = r2 < w ? P + r1 + static_cast<long long>(r2) * nr : U + (r1 - w) + static_cast<long long>(r2 - w) * m;
        }
      }
    }
    double cur[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) cur[j] = q[j] ? ldcg(q[j]) : 0.0;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      if (q[j]) *q[j] = cur[j] + v[j];
    }
  }
  (void)s;
}

// Narrow supernode, one warp, everything through L2.
__device__ void mf_warp_task(const MfArgs& a, int sn, int lane, double floor_v) {
  const SnPlan& s = a.s;
  const int f = s.first[sn], w = s.first[sn + 1] - f, nr = s.nrows[sn], m = nr - w;
  double* P = a.panel + s.off[sn];
  double* U = a.ubuf + a.uoff[sn];
  for (int c = s.child_ptr[sn] + lane; c < s.child_ptr[sn + 1]; c += 32) {
    if (!wait_flag(a.done + s.child[c], a.epoch, a.abort)) break;
  }
  __syncwarp();
  const bool ok = __shfl_sync(0xffffffffu, ld_relaxed(a.fail_col), 0) >= f;
  if (ok) {
    for (int e = lane; e < m * m; e += 32) U[e] = 0.0;
    __syncwarp();
    for (int ci = s.child_ptr[sn]; ci < s.child_ptr[sn + 1]; ++ci) {
      mf_extend_add(a, sn, s.child[ci], P, nr, w, U, m, lane, 32);
      __syncwarp();
    }
    bool failed = false;
    for (int k = 0; k < w; ++k) {
      double* Pk = P + k * nr;
      const double pivot = ldcg(Pk + k);
      if (!(pivot > floor_v)) {
        if (lane == 0) atomicMin(a.fail_col, f + k);
        failed = true;
        break;
      }
      const double dk = sqrt(pivot), rdk = 1.0 / dk;  // one division per column
      for (int r = k + 1 + lane; r < nr; r += 32) Pk[r] = ldcg(Pk + r) * rdk;
      __syncwarp();
      if (lane == 0) Pk[k] = dk;
      for (int c = k + 1; c < w; ++c) {
        const double lck = ldcg(Pk + c);
        double* Pc = P + c * nr;
        for (int r = c + lane; r < nr; r += 32) Pc[r] = fma(-ldcg(Pk + r), lck, ldcg(Pc + r));
      }
      __syncwarp();
    }
    if (!failed && m > 0) {
      // U -= L21 L21^T (lower), L21 = rows w.. of the panel
      for (int e = lane; e < m * m; e += 32) {
        const int i = e % m, j = e / m;
        if (i < j) continue;
        double dot = 0.0;
        for (int k = 0; k < w; ++k) dot = fma(ldcg(P + w + i + k * nr), ldcg(P + w + j + k * nr), dot);
        U[e] = ldcg(U + e) - dot;
      }
    }
  }
  warp_publish(a.done + sn, a.epoch, lane);
}

// Wide supernode, whole CTA.
__device__ void mf_cta_task(const MfArgs& a, MfSmem& S, int sn, double floor_v) {
  const SnPlan& s = a.s;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int f = s.first[sn], w = s.first[sn + 1] - f, nr = s.nrows[sn], m = nr - w;
  double* P = a.panel + s.off[sn];
  double* U = a.ubuf + a.uoff[sn];
  const int c0 = s.child_ptr[sn], c1 = s.child_ptr[sn + 1];
  for (int c = c0 + tid; c < c1; c += kMfThreads) {
    if (!wait_flag(a.done + s.child[c], a.epoch, a.abort)) break;
  }
  if (tid == 0) S.stop = ld_relaxed(a.fail_col) < f ? 1 : 0;
  __syncthreads();
  if (!S.stop) {
    const long long mm = static_cast<long long>(m) * m;
    for (long long e = tid; e < mm; e += kMfThreads) U[e] = 0.0;
    __syncthreads();
    for (int ci = c0; ci < c1; ++ci) {
      mf_extend_add(a, sn, s.child[ci], P, nr, w, U, m, tid, kMfThreads);
      __syncthreads();
    }
    for (int j0 = 0; j0 < w && !S.stop; j0 += kMfNb) {
      const int jb = min(kMfNb, w - j0);
      // (a) left-looking update of the block columns from columns [0, j0)
      if (j0 > 0) mf_gemm_nt_sub<32>(S, P + j0 + static_cast<long long>(j0) * nr, nr, P + j0, nr, P + j0, nr,
                                     nr - j0, jb, j0, 0);
      // (b1) diagonal block: warp 0 factors it in shared memory
      if (wid == 0) {
        for (int c = 0; c < kMfNb; ++c) {
          const int r = lane;
          double v = 0.0;
          if (c < jb && r < jb && r >= c) v = ldcg(P + (j0 + r) + static_cast<long long>(j0 + c) * nr);
          else if (r == c) v = 1.0;  // identity padding
          S.d[c][r] = v;
        }
        __syncwarp();
        int fail = -1;
        for (int k = 0; k < jb; ++k) {
          const double piv = S.d[k][k];
          if (!(piv > floor_v)) {
            fail = k;
            break;
          }
          const double dk = sqrt(piv), rdk = 1.0 / dk;
          __syncwarp();
          if (lane > k) S.d[k][lane] *= rdk;
          __syncwarp();
          if (lane == k) S.d[k][k] = dk;  // the row's owner: no cross-lane hazard
          const double lrk = S.d[k][lane];
          for (int c = k + 1; c < jb; ++c) {
            if (lane >= c) S.d[c][lane] = fma(-lrk, S.d[k][c], S.d[c][lane]);
          }
          __syncwarp();
        }
        if (fail >= 0) {
          if (lane == 0) {
            atomicMin(a.fail_col, f + j0 + fail);
            S.stop = 1;
          }
        } else {
          for (int c = 0; c < jb; ++c) {
            if (lane >= c && lane < jb) P[(j0 + lane) + static_cast<long long>(j0 + c) * nr] = S.d[c][lane];
          }
        }
      }
      if (tid < kMfNb) S.rdiag[tid] = tid < jb ? 1.0 / S.d[tid][tid] : 1.0;
      __syncthreads();
      if (S.stop) break;
      // (b2) rows below the diagonal block: x L11^T = a, one thread per row
      // (reciprocal diagonals: no FP64 division per element)
      for (int r = j0 + jb + tid; r < nr; r += kMfThreads) {
        double x[kMfNb];
#pragma unroll
        for (int k = 0; k < kMfNb; ++k) x[k] = k < jb ? ldcg(P + r + static_cast<long long>(j0 + k) * nr) : 0.0;
#pragma unroll
        for (int k = 0; k < kMfNb; ++k) {
          x[k] = x[k] * S.rdiag[k];
#pragma unroll
          for (int j = k + 1; j < kMfNb; ++j) x[j] = fma(-x[k], S.d[k][j], x[j]);
        }
#pragma unroll
        for (int k = 0; k < kMfNb; ++k) {
          if (k < jb) P[r + static_cast<long long>(j0 + k) * nr] = x[k];
        }
      }
      __syncthreads();
    }
    // U_s -= L21 L21^T
    if (!S.stop && m > 0) mf_gemm_nt_sub<64>(S, U, m, P + w, nr, P + w, nr, m, m, w, 0);
  }
  __syncthreads();
  if (tid == 0) {
    fence_gpu();
    st_relaxed(a.done + sn, a.epoch);
  }
}

__global__ void __launch_bounds__(kMfThreads, 2) k_mf_factor(MfArgs a) {
  __shared__ MfSmem S;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const double floor_v = fmax(a.maxdiag ? a.floor_rel * *a.maxdiag : a.floor_abs, 0.0);
  for (;;) {
    if (tid == 0) {
      const int t = static_cast<int>(atomicAdd(a.ticket, 1u));
      S.task = t;
      if (t < a.ntasks) {
        S.first = a.task_ptr[t];
        S.count = a.task_ptr[t + 1] - a.task_ptr[t];
        S.big = a.task_big[t];
      }
    }
    __syncthreads();
    const int t = S.task;
    if (t >= a.ntasks) break;
    const int first = S.first, count = S.count, big = S.big;
    if (big) {
      mf_cta_task(a, S, a.task_sn[first], floor_v);
    } else if (wid < count) {
      mf_warp_task(a, a.task_sn[first + wid], lane, floor_v);
    }
    __syncthreads();
  }
}

}  // namespace hykkt::dev
