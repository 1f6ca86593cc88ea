// Warp / thread tasks of the level-walking H^-1 pass of the cluster solve
// (kernels_cluster.cuh).  Templated on the argument struct A, which
// provides: tr (TrsvArgs), bt (b - J^T u per permuted row), rec / vals (the
// warp tasks' int and value records), wl / wl_ptr (per-warp task lists),
// gat4 (4-slot gather table of thread tasks), nlev, stamps.
#pragma once
// (included inside namespace hykkt::dev by kernels_cluster.cuh)

// Warp tasks (w <= 32, rows <= kClRows, panel <= kClVals entries) read
// their static data -- gather table rows / rows below, the panel with
// reciprocal diagonals, and b or y of their own columns -- from a per-warp
// shared-memory slot filled by cp.async one task ahead (two slots).
constexpr int kClRows = 64;
constexpr int kClVals = 512;
constexpr int kClInts = 4 * kClRows + kClRows;
struct alignas(16) ClSlot {
  double v[kClVals];
  double aux[32];
  int i[kClInts];
};
struct alignas(16) ClWarpBuf {
  ClSlot slot[2];
  double xs[kClRows];
};

__device__ __forceinline__ void cp_async8(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(static_cast<unsigned>(__cvta_generic_to_shared(dst))),
               "l"(src)
               : "memory");
}
__device__ __forceinline__ void cp_async16g(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(static_cast<unsigned>(__cvta_generic_to_shared(dst))),
               "l"(src)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait1() { asm volatile("cp.async.wait_group 1;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

// Issues the copies of one warp task's static data into a slot (the caller
// commits the group).  aux = b - J^T u (forward) or y (backward) of the
// task's own columns.
template <class A>
__device__ __forceinline__ void cl_issue(const A& a, int4 ta, int4 tb, ClSlot& sl, bool fwd, int lane) {
  const int w = ta.z & 0xffff, nr = ta.z >> 16;
  const int ni = (4 * nr + (nr - w) + 3) >> 2, nv = (w * nr + 1) >> 1;
  const int* ri = a.rec + ta.x;
  const double* rv = a.vals + ta.y;
  for (int c = lane; c < ni; c += 32) cp_async16g(sl.i + 4 * c, ri + 4 * c);
  for (int c = lane; c < nv; c += 32) cp_async16g(sl.v + 2 * c, rv + 2 * c);
  if (lane < w) cp_async8(sl.aux + lane, (fwd ? a.bt : a.tr.y) + tb.x + lane);
}

// Sum of a row's gathered update-vector entries (gat4 format), list order.
template <class A>
__device__ __forceinline__ double cl_gather(const A& a, int4 g, int slot) {
  const double* u = a.tr.u;
  const double v0 = g.x >= 0 ? ldcg(u + g.x) : 0.0;
  const double v1 = g.y >= 0 ? ldcg(u + g.y) : 0.0;
  const double v2 = g.z >= 0 ? ldcg(u + g.z) : 0.0;
  const double v3 = g.w >= 0 ? ldcg(u + g.w) : 0.0;
  double s = 0.0;
  s += v0;
  s += v1;
  s += v2;
  if (g.w >= -1) return s + v3;
  const int e1 = __ldg(a.tr.s.gat_ptr + slot + 1);
  for (int e = -2 - g.w; e < e1; ++e) s += ldcg(u + __ldg(a.tr.s.gat_idx + e));
  return s;
}

// Forward, one warp (w <= 32, rows <= 64), static data in `sl`: lane owns
// rows lane and lane + 32; after the update-vector gathers (the only
// dependent loads) the diagonal block is solved by a shuffle chain
// (reciprocal diagonals from the slot).
template <class A>
__device__ __forceinline__ void cl_fwd_warp(const A& a, int4 ta, int4 tb, const ClSlot& sl, int lane,
                                            unsigned long long* ts) {
  const int f = tb.x, w = ta.z & 0xffff, nr = ta.z >> 16;
  const int q0 = lane, q1 = lane + 32;
  const int4 g0 = q0 < nr ? *reinterpret_cast<const int4*>(sl.i + 4 * q0) : make_int4(-1, -1, -1, -1);
  const int4 g1 = q1 < nr ? *reinterpret_cast<const int4*>(sl.i + 4 * q1) : make_int4(-1, -1, -1, -1);
  double A0 = cl_gather(a, g0, tb.z + q0);
  double A1 = cl_gather(a, g1, tb.z + q1);
  const bool own = lane < w;
  if (own) A0 = sl.aux[lane] - A0;
  const double rd = own ? sl.v[lane * nr + lane] : 1.0;
  if (ts) {
    const double z = __shfl_sync(0xffffffffu, A0 + A1, 0);
    if (z != 1.2345e300 && lane == 0) ts[2] = global_ns();
  }
#pragma unroll 4
  for (int k = 0; k < w; ++k) {
    const double yk = __shfl_sync(0xffffffffu, A0 * rd, k);
    if (lane == k) A0 = yk;
    const double* Pk = sl.v + k * nr;
    if (q0 > k && q0 < nr) A0 = q0 < w ? fma(-Pk[q0], yk, A0) : fma(Pk[q0], yk, A0);
    if (q1 < nr) A1 = fma(Pk[q1], yk, A1);
  }
  if (ts) {
    const double z = __shfl_sync(0xffffffffu, A0 + A1, 0);
    if (z != 1.2345e300 && lane == 0) ts[3] = global_ns();
  }
  double* U = a.tr.u + ta.w;
  if (q0 < w) stcg(a.tr.y + f + q0, A0);
  else if (q0 < nr) stcg(U + q0 - w, A0);
  if (q1 < nr) stcg(U + q1 - w, A1);
}

// Backward, one warp (w <= 32, rows below <= 64): the rows' x values are
// gathered once into shared memory, lane k forms column k's dot product,
// then the diagonal block's backward chain.
template <class A>
__device__ __forceinline__ void cl_bwd_warp(const A& a, int4 ta, int4 tb, const ClSlot& sl, double* xs,
                                            int lane, unsigned long long* ts) {
  const int f = tb.x, w = ta.z & 0xffff, nr = ta.z >> 16, nb = nr - w;
  const int* rows = sl.i + 4 * nr;
  const int r0 = lane, r1 = lane + 32;
  double x0 = r0 < nb ? ldcg(a.tr.x + rows[r0]) : 0.0;
  double x1 = r1 < nb ? ldcg(a.tr.x + rows[r1]) : 0.0;
  if (tb.w) {  // rows below computed by other CTAs without a barrier in between: poll
    if (r0 < nb && __double_as_longlong(x0) == kUnset) x0 = poll_value(a.tr.x + rows[r0], a.tr.abort);
    if (r1 < nb && __double_as_longlong(x1) == kUnset) x1 = poll_value(a.tr.x + rows[r1], a.tr.abort);
  }
  if (r0 < nb) xs[r0] = x0;
  if (r1 < nb) xs[r1] = x1;
  __syncwarp();
  if (ts && lane == 0) ts[2] = global_ns();
  const bool own = lane < w;
  double acc = 0.0, rd = 1.0;
  if (own) {
    const double* Pc = sl.v + lane * nr + w;
    double t0 = 0.0, t1 = 0.0, t2 = 0.0, t3 = 0.0;
    int r = 0;
    for (; r + 4 <= nb; r += 4) {
      t0 = fma(Pc[r], xs[r], t0);
      t1 = fma(Pc[r + 1], xs[r + 1], t1);
      t2 = fma(Pc[r + 2], xs[r + 2], t2);
      t3 = fma(Pc[r + 3], xs[r + 3], t3);
    }
    for (; r < nb; ++r) t0 = fma(Pc[r], xs[r], t0);
    acc = sl.aux[lane] - ((t0 + t1) + (t2 + t3));
    rd = sl.v[lane * nr + lane];
  }
  for (int k = w - 1; k >= 0; --k) {
    const double xk = __shfl_sync(0xffffffffu, acc * rd, k);
    if (lane == k) acc = xk;
    if (lane < k) acc = fma(-sl.v[lane * nr + k], xk, acc);
  }
  if (ts) {
    const double z = __shfl_sync(0xffffffffu, acc, 0);
    if (z != 1.2345e300 && lane == 0) ts[3] = global_ns();
  }
  if (own) {
    stcg(a.tr.x + f + lane, acc);
    if (a.tr.x_out) a.tr.x_out[a.tr.s.perm[f + lane]] = acc;
  }
}

// Walks this warp's task list through one pass (forward: levels ascending,
// backward: descending), with static data for task k + 1 copied while task
// k runs.  Thread and CTA tasks of each level run before (CTA) / after
// (thread) the warp's tasks of that level; one cluster barrier per level.
struct ClWalk {
  int k, kend, dir, slot;
  int4 t0a, t0b, t1a, t1b;
};

template <class A>
__device__ __forceinline__ void cl_entry(const A& a, int e, bool ok, int4& ta, int4& tb) {
  if (ok) {
    ta = __ldg(a.wl + 2 * e);
    tb = __ldg(a.wl + 2 * e + 1);
  } else {
    ta = make_int4(0, 0, 0, 0);
    tb = make_int4(0, -1, 0, 0);
  }
}

template <class A>
__device__ __forceinline__ void cl_walk_begin(const A& a, ClWalk& W, ClWarpBuf& B, int gw, bool fwd, int lane) {
  const int e0 = a.wl_ptr[gw], e1 = a.wl_ptr[gw + 1];
  W.dir = fwd ? 1 : -1;
  W.k = fwd ? e0 : e1 - 1;
  W.kend = fwd ? e1 : e0 - 1;
  W.slot = 0;
  cl_entry(a, W.k, W.k != W.kend, W.t0a, W.t0b);
  cl_entry(a, W.k + W.dir, W.k != W.kend && W.k + W.dir != W.kend, W.t1a, W.t1b);
  if (W.k != W.kend) cl_issue(a, W.t0a, W.t0b, B.slot[0], fwd, lane);
  cp_async_commit();
}

template <class A>
__device__ __forceinline__ void cl_walk_level(const A& a, ClWalk& W, ClWarpBuf& B, int l, bool fwd, int lane,
                                              bool stamp_owner = false) {
  // diagnostics: warp 0 of CTA 0 stamps its first 64 tasks of each pass
  unsigned long long* ts = nullptr;
  if (a.stamps && stamp_owner) ts = a.stamps + 2 * a.nlev + (fwd ? 0 : 6 * 64);
  while (W.k != W.kend && W.t0b.y == l) {
    const int k1 = W.k + W.dir, k2 = k1 + W.dir;
    const int ti = ts ? (fwd ? W.k - a.wl_ptr[0] : a.wl_ptr[1] - 1 - W.k) : 64;
    if (ts && ti < 64 && lane == 0) ts[6 * ti] = global_ns();
    int4 t2a, t2b;
    cl_entry(a, k2, k1 != W.kend && k2 != W.kend, t2a, t2b);
    if (k1 != W.kend) cl_issue(a, W.t1a, W.t1b, B.slot[W.slot ^ 1], fwd, lane);
    cp_async_commit();
    if (ts && ti < 64 && lane == 0) ts[6 * ti + 1] = global_ns();
    cp_async_wait1();
    __syncwarp();
    if (ts && ti < 64 && lane == 0) ts[6 * ti + 2] = global_ns();
    if (fwd) cl_fwd_warp(a, W.t0a, W.t0b, B.slot[W.slot], lane, (ts && ti < 64) ? ts + 6 * ti + 1 : nullptr);
    else cl_bwd_warp(a, W.t0a, W.t0b, B.slot[W.slot], B.xs, lane, (ts && ti < 64) ? ts + 6 * ti + 1 : nullptr);
    __syncwarp();
    if (ts && ti < 64 && lane == 0) ts[6 * ti + 5] = global_ns();
    W.k = k1;
    W.slot ^= 1;
    W.t0a = W.t1a;
    W.t0b = W.t1b;
    W.t1a = t2a;
    W.t1b = t2b;
  }
}

// Forward, one thread (w <= 4, rows <= 16).
template <class A>
__device__ __forceinline__ void cl_fwd_thread(const A& a, int4 da, int4 db) {
  constexpr int NR = 16, W = 4;
  const int f = da.y, w = da.z & 0xffff, nr = da.z >> 16;
  const double* __restrict__ P = a.tr.panel + da.w;
  double acc[NR];
#pragma unroll
  for (int q0 = 0; q0 < NR; q0 += 4) {
    int4 g[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) g[j] = q0 + j < nr ? __ldg(a.gat4 + db.y + q0 + j) : make_int4(-1, -1, -1, -1);
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[q0 + j] = cl_gather(a, g[j], db.y + q0 + j);
  }
#pragma unroll
  for (int q = 0; q < W; ++q) {
    if (q < w) acc[q] = ldcg(a.bt + f + q) - acc[q];
  }
#pragma unroll
  for (int k = 0; k < W; ++k) {
    if (k < w) {
      const double yk = acc[k] * (1.0 / __ldg(P + k * nr + k));
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
  double* U = a.tr.u + db.x;
#pragma unroll
  for (int q = 0; q < NR; ++q) {
    if (q < w) stcg(a.tr.y + f + q, acc[q]);
    else if (q < nr) stcg(U + q - w, acc[q]);
  }
}

template <class A>
__device__ __forceinline__ void cl_bwd_thread(const A& a, int4 da, int4 db) {
  constexpr int NR = 16, W = 4;
  const int f = da.y, w = da.z & 0xffff, nr = da.z >> 16;
  const double* __restrict__ P = a.tr.panel + da.w;
  const int* R0 = a.tr.s.rows + db.y;
  double xb[NR], acc[W];
#pragma unroll
  for (int r = 0; r < NR; ++r) {
    const int gr = (r >= w && r < nr) ? __ldg(R0 + r) : -1;
    xb[r] = gr >= 0 ? ldcg(a.tr.x + gr) : 0.0;
  }
#pragma unroll
  for (int k = 0; k < W; ++k) {
    acc[k] = 0.0;
    if (k < w) {
      double t = 0.0;
#pragma unroll
      for (int r = 1; r < NR; ++r) {
        if (r >= w && r < nr) t = fma(__ldg(P + k * nr + r), xb[r], t);
      }
      acc[k] = ldcg(a.tr.y + f + k) - t;
    }
  }
#pragma unroll
  for (int k = W - 1; k >= 0; --k) {
    if (k < w) {
      const double xk = acc[k] * (1.0 / __ldg(P + k * nr + k));
      acc[k] = xk;
#pragma unroll
      for (int j = 0; j < k; ++j) acc[j] = fma(-__ldg(P + j * nr + k), xk, acc[j]);
    }
  }
#pragma unroll
  for (int k = 0; k < W; ++k) {
    if (k < w) {
      stcg(a.tr.x + f + k, acc[k]);
      if (a.tr.x_out) a.tr.x_out[a.tr.s.perm[f + k]] = acc[k];
    }
  }
}

// Warp-task value records from the factor's panels (reciprocal diagonals).
__global__ void k_cl_remap(int n, const int* __restrict__ vmap, const double* __restrict__ panel,
                           double* __restrict__ vals) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= n) return;
  const int m = vmap[j];
  vals[j] = m < 0 ? 0.0 : ((m & 1) ? 1.0 / panel[m >> 1] : panel[m >> 1]);
}

