// B200 (sm_100a) HyKKT device context and the C ABI declared in
// include/hykkt.h.
//
// Per interior-method iteration the whole of solve_full's numeric work
// (proj/core/src/solver.cpp:295-328: reduce, ruiz_scale, assemble_h_gamma,
// factorize_with_ladder, w solve, cg_schur with the delta2 restart, dx
// solve, unscale, recover) runs on the handle's stream from values resident
// in HBM.  The host only makes the ladder decision per factorization
// attempt and reads the CG outcome; the CG loop itself is one cooperative
// persistent kernel.
#include <cuda_runtime.h>

#include <algorithm>
#include <climits>
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <cstring>
#include <limits>
#include <memory>
#include <numeric>
#include <string>
#include <vector>

#include "../../include/hykkt.h"
#include "analyze.hpp"
#include "host_metrics.hpp"
#include "kernels_assemble.cuh"
#include "kernels_solve.cuh"
#include "kernels_batch.cuh"
#include "kernels_sys.cuh"
#include "kernels_mf.cuh"
#include "kernels_metrics.cuh"
#include "kernels_cluster.cuh"
#include "sysplan.hpp"

namespace hykkt {

namespace {

thread_local std::string g_last_error;

struct CudaError : std::runtime_error {
  explicit CudaError(const std::string& w) : std::runtime_error(w) {}
};
struct StateError : std::runtime_error {
  explicit StateError(const std::string& w) : std::runtime_error(w) {}
};
struct TimeoutError : std::runtime_error {
  explicit TimeoutError(const std::string& w) : std::runtime_error(w) {}
};

#define CK(x)                                                                  \
  do {                                                                         \
    cudaError_t e_ = (x);                                                      \
    if (e_ != cudaSuccess)                                                     \
      throw CudaError(std::string(#x) + ": " + cudaGetErrorString(e_));        \
  } while (0)

template <typename T>
struct DBuf {
  T* p = nullptr;
  std::size_t n = 0;
  DBuf() = default;
  DBuf(const DBuf&) = delete;
  DBuf& operator=(const DBuf&) = delete;
  ~DBuf() { reset(); }
  void reset() {
    if (p) cudaFree(p);
    p = nullptr;
    n = 0;
  }
  void alloc(std::size_t count) {
    if (count == n && p) return;
    reset();
    n = count;
    CK(cudaMalloc(&p, std::max<std::size_t>(count, 1) * sizeof(T)));
  }
  void upload(const T* src, std::size_t count, cudaStream_t s) {
    alloc(count);
    if (count) CK(cudaMemcpyAsync(p, src, count * sizeof(T), cudaMemcpyHostToDevice, s));
  }
  void upload(const std::vector<T>& v, cudaStream_t s) { upload(v.data(), v.size(), s); }
};

template <typename A>
std::vector<int> to_i32(const std::vector<A>& v) {
  return std::vector<int>(v.begin(), v.end());
}

constexpr int kThreads = 256;
int blocks_for(long long n) { return static_cast<int>(std::max<long long>(1, (n + kThreads - 1) / kThreads)); }

// Per-launch status block read back after each decision point.
struct StatusBlock {
  int fail_col;
  int abort;
  int ruiz_sweeps;
  int pad;
  dev::CgResultDev cg;
};

}  // namespace

}  // namespace hykkt

struct hykkt_context {
  int device = 0;
  cudaStream_t stream = nullptr;
  int num_sms = 0;
  int coop_factor_blocks = 0, coop_trsv_blocks = 0, coop_cg_blocks = 0, coop_ruiz_blocks = 0;
  int coop_bfactor_blocks = 0, coop_btrsv_blocks = 0, coop_bcg_blocks = 0, coop_bruiz_blocks = 0;
  int coop_bruiz_rows_blocks = 0, coop_mf_blocks = 0;
  int cg_grid = 0, trsv_grid = 0;  // per analysed plan: CTAs of k_cg / k_trsv (<= coop_*_blocks)
  const void* cg_fn = nullptr;
  // multifrontal single-system factor (kernels_mf.cuh)
  hykkt::DBuf<long long> mf_uoff;
  hykkt::DBuf<int> mf_task_ptr, mf_task_sn;
  hykkt::DBuf<unsigned char> mf_task_big;
  hykkt::DBuf<double> mf_ubuf;
  int mf_ntasks = 0, mf_on = 1;
  // single-system triangular-solve task streams (kernels_solve.cuh trsv_pass)
  hykkt::DBuf<int> tr_bt_rows, tr_wid, tr_wid_bwd, tr_nar, tr_nar_bwd, tr_pos, tr_chain_ptr, tr_chain_sn, tr_chain_fsrc, tr_chain_bsrc;
  int tr_chain_regs = 0;
  int tr_nwid = 0, tr_nnar = 0, tr_nbot = 0;
  int tr_call = 0;  // narrow tasks as real calls (trsv_pass<true>), chosen per analysis
  hykkt::DBuf<int> tr_bot_ptr, tr_bot_sn;
  hykkt::DBuf<unsigned char> tr_bot_wide;
  // asynchronous batch copies (hykkt_batch_upload_async / _download_async):
  // two staging slots of field-major host values filled on copy_stream, the
  // next batched solve consumes the oldest; outputs staged for the D2H
  cudaStream_t copy_stream = nullptr;
  hykkt::DBuf<double> stage[2], out_stage;
  long long stage_batch[2] = {0, 0};
  cudaEvent_t stage_ready[2] = {nullptr, nullptr}, stage_free[2] = {nullptr, nullptr};
  cudaEvent_t out_ready = nullptr, out_free = nullptr;
  bool stage_free_rec[2] = {false, false}, out_free_rec = false;
  int stage_q[2] = {-1, -1}, stage_nq = 0, stage_next = 0;
  // Q-form wide supernodes (kernels_solve.cuh qslice_fwd / qslice_bwd / k_qform)
  hykkt::DBuf<double> q_buf;
  hykkt::DBuf<long long> q_off;
  hykkt::DBuf<int> q_items, q_sf, q_sb;
  int q_nrows = 0, q_nsf = 0, q_nsb = 0;
  long long panel_ver = 0, q_ver = -1;
  // single-system solve on one thread-block cluster (kernels_cluster.cuh)
  int cl_on = 0, cl_ctas = 0, cl_nlev = 0;
  hykkt::DBuf<int> cl_lv_ptr, cl_lv_sn, cl_desc, cl_gat4, cl_wl, cl_wptr, cl_rec, cl_vmap;
  hykkt::DBuf<double> cl_vals;
  int cl_nvals = 0;
  hykkt::DBuf<double> cl_bt;
  hykkt::DBuf<double> cg_bt;  // k_cg: precomputed forward right-hand side (TrsvArgs::bt_fill)
  int tr_nbt_rows = 0;
  int cg_bt_on = 0;
  unsigned long long* cg_stamps = nullptr;  // diagnostics: 16 per CG CTA (hykkt_debug_cg_phases)
  hykkt::DBuf<unsigned long long> cl_stamps;
  // kb_ruiz_rows: row lists of [[H_tilde, J^T], [J, 0]] (built on first batched solve)
  hykkt::DBuf<int> ruiz_rp, ruiz_ent;
  bool ruiz_rows_built = false;
  hykkt::DBuf<double> met_partials;  // device BE / RR (kernels_metrics.cuh)

  bool have_plan = false, have_kkt = false, have_values = false, have_factor = false;
  bool have_assembled = false;
  hykkt::AmalgParams amalg = hykkt::AmalgParams::defaults();  // hykkt_set_option, before analysis
  // Reduced2x2 handle (hykkt_analyze_reduced): m_d = 0, D_x = 0 and identity
  // Ruiz scaling, so the 4x4 kernels compute solve_reduced exactly
  bool reduced = false;
  // Cholesky-level handle with a constraint Jacobian (hykkt_chol_set_j)
  bool have_j = false;
  hykkt::SupernodalPlan sp;
  hykkt::KktPlan kp;

  // device supernodal plan
  hykkt::DBuf<int> order, first, nrows, off, rows_ptr, rows, parent, child_ptr, child;
  hykkt::DBuf<int> upd_ptr, upd_d, upd_off, upd_cnt, lrow_ptr, lrow_col, lrow_pos, lrow_row, upd_pbase, upd_pos;
  hykkt::DBuf<double> lrow_val, xsol, ubuf, accbuf;
  hykkt::DBuf<int> u_off, ext_ptr, ext_map, gat_ptr, gat_idx, relind;
  hykkt::DBuf<int> perm, iperm, src_to_panel, src_row, src_col;
  hykkt::DBuf<double> panel, y, src_vals, bvec, xvec;
  hykkt::DBuf<int> fac_done;
  hykkt::DBuf<unsigned> barrier;  // count, gen
  hykkt::DBuf<unsigned> tickets;  // dynamic task counters
  hykkt::DBuf<hykkt::StatusBlock> status;
  int epoch = 0;

  // KKT plan arrays
  hykkt::DBuf<int> ht_row, ht_col, ht_hsrc, ht_pp, ht_pa, ht_pb, ht_pk;
  hykkt::DBuf<int> hg_row, hg_col, hg_src, hg_pp, hg_pa, hg_pb;
  hykkt::DBuf<int> j_cp, j_ri, j_col, jcsr_src, jcsr_rp, jcsr_ci_perm;
  hykkt::DBuf<int> jd_cp, jd_ri, jdcsr_rp, jdcsr_ci, jdcsr_src;
  // values
  hykkt::DBuf<double> hval, jval, jdval, d_x, d_s, r_tx, r_s, r_y, r_yd;
  // work
  hykkt::DBuf<double> ht, hts, js, js_csr, r_x, rxs, rys, dscale, norms, hg, rhat, maxdiag;
  hykkt::DBuf<int> ruiz_flags;
  hykkt::DBuf<double> cg_rhs, cg_x, cg_r, cg_p, cg_q, partials;
  hykkt::DBuf<double> dx_s, dx, dy, ds, dyd;

  hykkt_timing_t timing{};
  long long launches = 0;

  // Active value / output pointers: the single-system buffers above, or one
  // slot of the resident batch below.
  struct VPtr { double *h, *j, *jd, *dx, *ds, *rtx, *rs, *ry, *ryd; } v{};
  struct OPtr { double *dx, *dy, *ds, *dyd; } o{};
  hykkt::DBuf<double> bvals, bouts;  // [batch][values], [batch][solution]
  long long batch = 0;
  struct BatchBufsT {
    int Bp = 32;
    bool flags_init = false;
    hykkt::DBuf<double> xs, vals, ht, hts, js, jscsr, rx, rxs, rys, d, norms, hg, rhat, maxdiag, panel, y, u, acc;
    hykkt::DBuf<double> cgrhs, cgx, cgr, cgp, cgq, part, dxs, odx, ody, ods, odyd, delta1, relres;
    hykkt::DBuf<int> ruiz_unconv, ruiz_active, sweeps, active, fail, running, start, flags, live;
    hykkt::DBuf<int> fac_done, fdone, bdone;
    hykkt::DBuf<long long> iters;
    // CTA job list of the batched solve (rebuilt when the tile count changes)
    hykkt::DBuf<int> job_ptr, job_items, fjob_ptr, fjob_items, mode, slot_sn, wdone;
    hykkt::DBuf<unsigned char> job_kind, fjob_kind;
    int jobs_T = -1, njobs = 0, nfjobs = 0;
    long long nwide = 0;
    double* f[9] = {};
  } bb;
  std::vector<hykkt_report_t> batch_reports;
  // system-per-CTA solve (kernels_sys.cuh): stream program + per-system data
  struct SysBufsT {
    int state = 0;  // 0 unbuilt, 1 ready, -1 infeasible (lane path)
    std::string why;
    hykkt::SysPlan plan;
    std::size_t smem = 0;
    hykkt::DBuf<int> idx, src, ok, flags;
    hykkt::DBuf<double> vals, rhat, rys, d, scratch, relres, d2;
    hykkt::DBuf<long long> iters;
    hykkt::DBuf<unsigned long long> prof, trace;
    // ks_factor: per-level narrow (warp) and wide (CTA) supernode lists
    hykkt::DBuf<int> lev_ptr, lev_sn, wlev_ptr, wlev_sn, upd, upd_rows, wb_ptr, wb_end, cb_ptr, cb_end;
    hykkt::DBuf<double> hg, js;
    std::size_t fsmem = 0;
    int factor_on = 0;  // ks_factor opt-in (HYKKT_KS_FACTOR=1): correct, slower than kb_factor so far
    int prof_on = -1, prof_ctas = 0;
    hykkt::DBuf<int> order;   // history-based longest-first system order (HYKKT_KS_LPT=0 disables)
    long long lpt_for = -1;
    int lpt_on = std::getenv("HYKKT_KS_LPT") ? std::atoi(std::getenv("HYKKT_KS_LPT")) : 1;
  } ks;

  hykkt::dev::SnPlan snplan() const {
    hykkt::dev::SnPlan s;
    s.n = static_cast<int>(sp.n);
    s.nsup = static_cast<int>(sp.nsup);
    s.order = order.p;
    s.first = first.p;
    s.nrows = nrows.p;
    s.off = off.p;
    s.rows_ptr = rows_ptr.p;
    s.rows = rows.p;
    s.parent = parent.p;
    s.child_ptr = child_ptr.p;
    s.child = child.p;
    s.upd_ptr = upd_ptr.p;
    s.upd_d = upd_d.p;
    s.upd_off = upd_off.p;
    s.upd_cnt = upd_cnt.p;
    s.lrow_ptr = lrow_ptr.p;
    s.lrow_col = lrow_col.p;
    s.lrow_pos = lrow_pos.p;
    s.perm = perm.p;
    s.iperm = iperm.p;
    s.u_off = u_off.p;
    s.ext_ptr = ext_ptr.p;
    s.ext_map = ext_map.p;
    s.gat_ptr = gat_ptr.p;
    s.gat_idx = gat_idx.p;
    s.relind = relind.p;
    s.u_size = sp.u_off.empty() ? 0 : sp.u_off.back();
    s.upd_pbase = upd_pbase.p;
    s.upd_pos = upd_pos.p;
    return s;
  }

  hykkt::dev::AsmPlan asmplan() const {
    hykkt::dev::AsmPlan a;
    a.nx = static_cast<int>(kp.nx);
    a.mc = static_cast<int>(kp.mc);
    a.md = static_cast<int>(kp.md);
    a.n_ht = static_cast<int>(kp.ht.nnz());
    a.ht_row = ht_row.p;
    a.ht_col = ht_col.p;
    a.ht_hsrc = ht_hsrc.p;
    a.ht_pp = ht_pp.p;
    a.ht_pa = ht_pa.p;
    a.ht_pb = ht_pb.p;
    a.ht_pk = ht_pk.p;
    a.n_hg = static_cast<int>(kp.hg.nnz());
    a.hg_row = hg_row.p;
    a.hg_col = hg_col.p;
    a.hg_src = hg_src.p;
    a.hg_pp = hg_pp.p;
    a.hg_pa = hg_pa.p;
    a.hg_pb = hg_pb.p;
    a.nnz_j = static_cast<int>(kp.j.nnz());
    a.j_cp = j_cp.p;
    a.j_ri = j_ri.p;
    a.j_col = j_col.p;
    a.jcsr_src = jcsr_src.p;
    a.nnz_jd = static_cast<int>(kp.jd.nnz());
    a.jd_cp = jd_cp.p;
    a.jd_ri = jd_ri.p;
    return a;
  }
};

namespace hykkt {
namespace {

using Ctx = hykkt_context;

// kb_trsv / kb_cg per-warp accumulators: 8 warps x rows x 32 systems.
int batch_smem_rows() {
  int r = 48;
  if (const char* e = std::getenv("HYKKT_BATCH_SMEM_ROWS")) r = std::max(8, std::atoi(e));
  return r;
}
const std::size_t kBatchSmem = 8 * static_cast<std::size_t>(batch_smem_rows()) * 32 * sizeof(double);

// Supernodes with width * rows >= this (or more rows than a warp's shared
// accumulator) are solved by a whole CTA in the batched solve.
long long big_task_wnr() {
  // B200 sweeps on the batch of 256 ACTIVSg2000: 320 in level order (12.8 ->
  // 11.5 ms of factor); with the depth-ordered job list (r02) 640: 10.8 ->
  // 8.9 ms (level order at 640: 13.3 ms)
  long long v = 640;
  if (const char* e = std::getenv("HYKKT_BIG_WNR")) v = std::max(1ll, std::atoll(e));
  return v;
}

void coop_launch(Ctx& c, const void* fn, int blocks, void* args, std::size_t smem = 0) {
  void* argv[] = {args};
  CK(cudaLaunchCooperativeKernel(fn, dim3(blocks), dim3(kThreads), argv, smem, c.stream));
  c.launches++;
}

void check_launch(Ctx& c) {
  CK(cudaGetLastError());
  c.launches++;
}

// Resident blocks for a cooperative persistent kernel: occupancy-limited and
// capped at HYKKT_BLOCKS_PER_SM (default 4 -> 32 warps per SM): more
// resident warps than that only add pollers.
int occupancy_blocks(Ctx& c, const void* fn, std::size_t smem = 0) {
  int per_sm = 0;
  if (smem) CK(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, kThreads, smem));
  int cap = 4;
  if (const char* e = std::getenv("HYKKT_BLOCKS_PER_SM")) cap = std::max(1, std::atoi(e));
  return std::max(1, std::min(per_sm, cap)) * c.num_sms;
}

int pick_cluster_ctas(Ctx& c);

void init_ctx(Ctx& c, int device) {
  c.device = device;
  CK(cudaSetDevice(device));
  CK(cudaStreamCreateWithFlags(&c.stream, cudaStreamNonBlocking));
  CK(cudaDeviceGetAttribute(&c.num_sms, cudaDevAttrMultiProcessorCount, device));
  int coop = 0;
  CK(cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, device));
  if (!coop) throw CudaError("device does not support cooperative launch");
  c.coop_factor_blocks = occupancy_blocks(c, (const void*)dev::k_factor);
  c.coop_mf_blocks = occupancy_blocks(c, (const void*)dev::k_mf_factor);
  c.coop_trsv_blocks = std::min(occupancy_blocks(c, (const void*)dev::k_trsv<false>),
                                occupancy_blocks(c, (const void*)dev::k_trsv<true>));
  {
    c.cg_fn = (const void*)dev::k_cg<2, false>;  // 2 CTAs per SM (B200 sweep of 2 / 3 / 4 in round 1)
  }
  c.coop_cg_blocks = std::min(occupancy_blocks(c, c.cg_fn), occupancy_blocks(c, (const void*)dev::k_cg<2, true>));
  c.coop_ruiz_blocks = std::min(occupancy_blocks(c, (const void*)dev::k_ruiz), 2 * c.num_sms);
  c.coop_bfactor_blocks = occupancy_blocks(c, (const void*)dev::kb_factor, kBatchSmem);
  c.coop_btrsv_blocks = occupancy_blocks(c, (const void*)dev::kb_trsv, kBatchSmem);
  // batched CG: grid * 256 must be a multiple of the system stride (a power
  // of two <= 2^16): use a power-of-two number of blocks.
  {
    int nb = occupancy_blocks(c, (const void*)dev::kb_cg, kBatchSmem), p2 = 1;
    while (p2 * 2 <= nb) p2 *= 2;
    c.coop_bcg_blocks = p2;
  }
  c.coop_bruiz_blocks = std::min(occupancy_blocks(c, (const void*)dev::kb_ruiz), 2 * c.num_sms);
  c.coop_bruiz_rows_blocks = occupancy_blocks(c, (const void*)dev::kb_ruiz_rows);
  {
    unsigned ns = 16, mx = 16;
    if (const char* e = std::getenv("HYKKT_POLL_NS")) ns = static_cast<unsigned>(std::max(0, std::atoi(e)));
    if (const char* e = std::getenv("HYKKT_POLL_MAX_NS")) mx = static_cast<unsigned>(std::max(0, std::atoi(e)));
    mx = std::max(mx, ns);
    CK(cudaMemcpyToSymbol(dev::g_poll_ns, &ns, sizeof(ns)));
    CK(cudaMemcpyToSymbol(dev::g_poll_max_ns, &mx, sizeof(mx)));
  }
  c.barrier.alloc(2);
  CK(cudaMemsetAsync(c.barrier.p, 0, 2 * sizeof(unsigned), c.stream));
  c.status.alloc(1);
  CK(cudaMemsetAsync(c.status.p, 0, sizeof(StatusBlock), c.stream));
}

// Level-ordered CTA task list: supernodes with big(sn) are single-supernode
// (whole CTA) tasks, the others are grouped per level, up to one per warp.
// Depth of every supernode below the root of its tree (s.order lists
// children before parents).
std::vector<int> sn_depth(const SupernodalPlan& s) {
  std::vector<int> depth(s.nsup, 0);
  for (idx q = s.nsup - 1; q >= 0; --q) {
    const int sn = s.order[q], p = s.sn_parent[sn];
    depth[sn] = p < 0 ? 0 : depth[p] + 1;
  }
  return depth;
}

template <class Pred>
void level_tasks(const SupernodalPlan& s, Pred big, std::vector<int>& tp, std::vector<int>& tsn,
                 std::vector<unsigned char>& tbig, bool by_depth = false) {
  tp.assign(1, 0);
  tsn.clear();
  tbig.clear();
  // by_depth: descending depth below the root instead of ascending level
  // (both topological; supernodes sharing a key never depend on each other)
  std::vector<int> seq(s.order.begin(), s.order.end()), key(s.nsup);
  if (by_depth) {
    const std::vector<int> depth = sn_depth(s);
    std::stable_sort(seq.begin(), seq.end(), [&](int x, int y) { return depth[x] > depth[y]; });
    for (idx k = 0; k < s.nsup; ++k) key[k] = -depth[k];
  } else {
    for (idx k = 0; k < s.nsup; ++k) key[k] = s.sn_level[k];
  }
  idx q = 0;
  while (q < s.nsup) {
    const int lev = key[seq[q]];
    std::vector<int> narrow;
    for (; q < s.nsup && key[seq[q]] == lev; ++q) {
      const int sn = seq[q];
      if (big(sn)) {
        tsn.push_back(sn);
        tp.push_back(static_cast<int>(tsn.size()));
        tbig.push_back(1);
      } else {
        narrow.push_back(sn);
      }
    }
    for (std::size_t g = 0; g < narrow.size(); g += kThreads / 32) {
      for (std::size_t h = g; h < std::min(narrow.size(), g + kThreads / 32); ++h) tsn.push_back(narrow[h]);
      tp.push_back(static_cast<int>(tsn.size()));
      tbig.push_back(0);
    }
  }
}

// Level lists of the cluster solve (kernels_cluster.cuh): per level of the
// supernode tree, thread tasks (w <= 4, rows <= 16, on levels with at least
// HYKKT_CL_THREAD_MIN supernodes), warp tasks (w <= 32, rows <= kClRows,
// panel <= kClVals) and whole-CTA tasks (the rest).  Warp tasks go to
// per-warp lists in level order (round robin over the cluster's warps; a
// run of levels holding a single parent chain of warp tasks is merged into
// one level on one warp), each with an int record (4-slot gathers, rows
// below) and a value record (panel, reciprocal diagonal) rebuilt from the
// factor by k_cl_remap.
void build_cluster_plan(Ctx& c) {
  const SupernodalPlan& s = c.sp;
  c.cl_nlev = 0;
  if (const char* e = std::getenv("HYKKT_CLUSTER")) c.cl_on = std::atoi(e) != 0;
  if (!c.cl_on || s.nsup == 0) return;
  if (s.max_nrows > dev::kWideMaxRows) return;  // CTA tasks stage their rows in shared memory
  c.cl_ctas = pick_cluster_ctas(c);
  const int nwarps = c.cl_ctas * dev::kClWarps;
  int thread_min = 1024;
  if (const char* e = std::getenv("HYKKT_CL_THREAD_MIN")) thread_min = std::atoi(e);
  const bool chain_on = !std::getenv("HYKKT_CL_CHAIN") || std::atoi(std::getenv("HYKKT_CL_CHAIN")) != 0;
  // levels of s.order
  std::vector<std::vector<int>> levels;
  for (idx q = 0; q < s.nsup;) {
    const int lev = s.sn_level[s.order[q]];
    levels.emplace_back();
    for (; q < s.nsup && s.sn_level[s.order[q]] == lev; ++q) levels.back().push_back(s.order[q]);
  }
  auto kind = [&](int sn, bool many) {  // 0 thread, 1 warp, 2 CTA
    const int w = s.sn_first[sn + 1] - s.sn_first[sn], nr = s.sn_nrows[sn];
    if (w > 32 || nr > dev::kClRows || w * nr > dev::kClVals) return 2;
    if (many && w <= 4 && nr <= 16) return 0;
    return 1;
  };
  std::vector<int> lv, csn, desc, rec, vmap;
  std::vector<std::vector<int>> wlist(nwarps);  // 8 ints per entry
  auto push_desc = [&](int sn) {
    const int f = s.sn_first[sn], w = s.sn_first[sn + 1] - f, nr = s.sn_nrows[sn];
    desc.insert(desc.end(), {sn, f, w | (nr << 16), static_cast<int>(s.sn_off[sn]), s.u_off[sn],
                             s.sn_rows_ptr[sn], 0, 0});
  };
  auto push_warp = [&](int sn, int gw, int level) {
    const int f = s.sn_first[sn], w = s.sn_first[sn + 1] - f, nr = s.sn_nrows[sn], rp = s.sn_rows_ptr[sn];
    const int roff = static_cast<int>(rec.size()), voff = static_cast<int>(vmap.size());
    for (int q = 0; q < nr; ++q) {
      const int t = rp + q, e0 = s.gat_ptr[t], e1 = s.gat_ptr[t + 1];
      int g[4] = {-1, -1, -1, -1};
      if (e1 - e0 <= 4) {
        for (int e = e0; e < e1; ++e) g[e - e0] = s.gat_idx[e];
      } else {
        for (int k = 0; k < 3; ++k) g[k] = s.gat_idx[e0 + k];
        g[3] = -2 - (e0 + 3);
      }
      rec.insert(rec.end(), g, g + 4);
    }
    for (int q = w; q < nr; ++q) rec.push_back(s.sn_rows[rp + q]);
    while (rec.size() % 4) rec.push_back(0);
    for (int k = 0; k < w; ++k)
      for (int q = 0; q < nr; ++q) vmap.push_back(2 * static_cast<int>(s.sn_off[sn] + k * nr + q) + (q == k ? 1 : 0));
    if (vmap.size() % 2) vmap.push_back(-1);
    wlist[gw].insert(wlist[gw].end(), {roff, voff, w | (nr << 16), s.u_off[sn], f, level, rp, 0});
  };
  int nl = 0;
  for (std::size_t L = 0; L < levels.size();) {
    const auto& g = levels[L];
    const bool many = static_cast<int>(g.size()) >= thread_min;
    // a chain: consecutive single-warp-task levels, each task the parent's child
    std::size_t L2 = L + 1;
    if (chain_on && g.size() == 1 && kind(g[0], false) == 1) {
      while (L2 < levels.size() && levels[L2].size() == 1 && kind(levels[L2][0], false) == 1 &&
             s.sn_parent[levels[L2 - 1][0]] == levels[L2][0])
        ++L2;
    }
    lv.push_back(static_cast<int>(desc.size() / 8));
    if (L2 > L + 1) {
      for (std::size_t k = L; k < L2; ++k) push_warp(levels[k][0], 0, nl);
    } else {
      int rr = 0;
      for (int sn : g) {
        const int kd = kind(sn, many);
        if (kd == 0) push_desc(sn);
        else if (kd == 2) csn.push_back(sn);
        else push_warp(sn, (rr++) % nwarps, nl);
      }
    }
    lv.push_back(static_cast<int>(desc.size() / 8));  // thread tasks end
    lv.push_back(static_cast<int>(desc.size() / 8));  // (unused)
    lv.push_back(static_cast<int>(csn.size()));       // CTA tasks end (start: previous level's end)
    ++nl;
    L = L2;
  }
  c.cl_nlev = nl;
  std::vector<int> wl, wptr{0};
  for (auto& v : wlist) {
    wl.insert(wl.end(), v.begin(), v.end());
    wptr.push_back(static_cast<int>(wl.size() / 8));
  }
  std::vector<int> g4(4 * static_cast<std::size_t>(std::max(1, s.sn_rows_ptr.back())), -1);
  for (int t = 0; t < s.sn_rows_ptr.back(); ++t) {
    const int e0 = s.gat_ptr[t], e1 = s.gat_ptr[t + 1];
    if (e1 - e0 <= 4) {
      for (int e = e0; e < e1; ++e) g4[4 * t + (e - e0)] = s.gat_idx[e];
    } else {
      for (int k = 0; k < 3; ++k) g4[4 * t + k] = s.gat_idx[e0 + k];
      g4[4 * t + 3] = -2 - (e0 + 3);
    }
  }
  rec.resize(rec.size() + 8, 0);  // copy over-reach
  vmap.resize(vmap.size() + 2, -1);
  c.cl_lv_ptr.upload(lv, c.stream);
  c.cl_desc.upload(desc.empty() ? std::vector<int>(8, 0) : desc, c.stream);
  c.cl_lv_sn.upload(csn.empty() ? std::vector<int>{0} : csn, c.stream);
  c.cl_gat4.upload(g4, c.stream);
  c.cl_wl.upload(wl.empty() ? std::vector<int>(8, 0) : wl, c.stream);
  c.cl_wptr.upload(wptr, c.stream);
  c.cl_rec.upload(rec, c.stream);
  c.cl_vmap.upload(vmap, c.stream);
  c.cl_vals.alloc(vmap.size());
  c.cl_nvals = static_cast<int>(vmap.size());
  c.cl_bt.alloc(std::max<idx>(1, s.n));
  c.cl_stamps.alloc(2 * c.cl_nlev + 2 + 768);
}

std::size_t cluster_smem() { return sizeof(dev::ClSmem); }

// Cluster size for k_cluster_solve: HYKKT_CL_CTAS (default 16, the
// non-portable maximum), reduced until the device can host one cluster.
int pick_cluster_ctas(Ctx& c) {
  int want = 16;
  if (const char* e = std::getenv("HYKKT_CL_CTAS")) want = std::max(1, std::min(16, std::atoi(e)));
  const void* fn = (const void*)dev::k_cluster_solve;
  CK(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(cluster_smem())));
  CK(cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  for (int cs = want; cs >= 1; cs /= 2) {
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute at[1];
    cfg.gridDim = dim3(cs);
    cfg.blockDim = dim3(dev::kClThreads);
    cfg.dynamicSmemBytes = cluster_smem();
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = cs;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    int n = 0;
    if (cudaOccupancyMaxActiveClusters(&n, fn, &cfg) == cudaSuccess && n >= 1) return cs;
    cudaGetLastError();
  }
  throw CudaError("no cluster configuration fits k_cluster_solve");
}

void launch_cluster(Ctx& c, dev::ClArgs& a) {
  if (c.cl_nvals > 0) {  // warp-task value records from the current factor
    dev::k_cl_remap<<<(c.cl_nvals + kThreads - 1) / kThreads, kThreads, 0, c.stream>>>(c.cl_nvals, c.cl_vmap.p,
                                                                                     c.panel.p, c.cl_vals.p);
    check_launch(c);
  }
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute at[1];
  cfg.gridDim = dim3(c.cl_ctas);
  cfg.blockDim = dim3(dev::kClThreads);
  cfg.dynamicSmemBytes = cluster_smem();
  cfg.stream = c.stream;
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = c.cl_ctas;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  CK(cudaLaunchKernelEx(&cfg, dev::k_cluster_solve, a));
  c.launches++;
}

void upload_plan(Ctx& c, const CscPattern& src_pattern) {
  const SupernodalPlan& s = c.sp;
  cudaStream_t st = c.stream;
  c.order.upload(s.order, st);
  c.first.upload(s.sn_first, st);
  c.nrows.upload(s.sn_nrows, st);
  c.off.upload(to_i32(s.sn_off), st);
  c.rows_ptr.upload(s.sn_rows_ptr, st);
  c.rows.upload(s.sn_rows, st);
  c.parent.upload(s.sn_parent, st);
  c.child_ptr.upload(s.child_ptr, st);
  c.child.upload(s.child, st);
  c.upd_ptr.upload(s.upd_ptr, st);
  c.upd_d.upload(s.upd_d, st);
  c.upd_off.upload(s.upd_off, st);
  c.upd_cnt.upload(s.upd_cnt, st);
  {
    // positions of every descendant row of every left-looking update in the
    // target's row structure (replaces a per-entry binary search on device)
    std::vector<int> pbase(s.upd_d.size() + 1, 0), pos;
    for (idx t = 0; t < s.nsup; ++t) {
      const int f = s.sn_first[t], w = s.sn_first[t + 1] - f;
      const int* R = s.sn_rows.data() + s.sn_rows_ptr[t];
      const int* Re = s.sn_rows.data() + s.sn_rows_ptr[t + 1];
      for (int u = s.upd_ptr[t]; u < s.upd_ptr[t + 1]; ++u) {
        const int d = s.upd_d[u], o = s.upd_off[u], cnt = s.upd_cnt[u];
        const int* Rd = s.sn_rows.data() + s.sn_rows_ptr[d];
        const int m = s.sn_nrows[d] - o;
        for (int ii = 0; ii < m; ++ii) {
          const int r = Rd[o + ii];
          pos.push_back(ii < cnt ? r - f : static_cast<int>(std::lower_bound(R + w, Re, r) - R));
        }
        pbase[u + 1] = static_cast<int>(pos.size());
      }
    }
    c.upd_pbase.upload(pbase, st);
    c.upd_pos.upload(pos.empty() ? std::vector<int>{0} : pos, st);
  }
  c.lrow_ptr.upload(s.lrow_ptr, st);
  c.lrow_col.upload(s.lrow_col, st);
  c.lrow_pos.upload(s.lrow_pos, st);
  c.lrow_row.upload(s.lrow_row, st);
  c.lrow_val.alloc(s.lrow_pos.size());
  c.xsol.alloc(s.n);
  c.u_off.upload(s.u_off, st);
  c.ext_ptr.upload(s.ext_ptr, st);
  c.ext_map.upload(s.ext_map, st);
  c.gat_ptr.upload(s.gat_ptr, st);
  c.gat_idx.upload(s.gat_idx, st);
  c.relind.upload(s.relind, st);
  c.ubuf.alloc(s.u_off.back());
  c.accbuf.alloc(s.sn_rows_ptr.back());
  c.perm.upload(to_i32(s.perm), st);
  c.iperm.upload(to_i32(s.iperm), st);
  c.src_to_panel.upload(s.src_to_panel, st);
  std::vector<int> srow(src_pattern.nnz()), scol(src_pattern.nnz());
  for (idx j = 0; j < src_pattern.ncols; ++j) {
    for (idx p = src_pattern.cp[j]; p < src_pattern.cp[j + 1]; ++p) {
      srow[p] = static_cast<int>(src_pattern.ri[p]);
      scol[p] = static_cast<int>(j);
    }
  }
  c.src_row.upload(srow, st);
  c.src_col.upload(scol, st);
  c.panel.alloc(s.panel_size);
  c.y.alloc(s.n);
  c.bvec.alloc(s.n);
  c.xvec.alloc(s.n);
  c.fac_done.alloc(s.nsup);
  {
    // multifrontal factor: update-matrix offsets and the level-ordered task
    // list (one wide supernode per CTA task, up to 8 narrow ones of a level
    // per warp-group task)
    int big_rows = 24;  // B200 sweep at C2-C4 (was 64: C2 factor 1.24 -> 0.77 ms)
    if (const char* e = std::getenv("HYKKT_MF_BIG")) big_rows = std::max(1, std::atoi(e));
    if (const char* e = std::getenv("HYKKT_FACTOR")) c.mf_on = std::string(e) != "ll";
    std::vector<long long> uo(s.nsup + 1, 0);
    for (idx k = 0; k < s.nsup; ++k) {
      const long long m = s.sn_nrows[k] - (s.sn_first[k + 1] - s.sn_first[k]);
      uo[k + 1] = uo[k] + m * m;
    }
    std::vector<int> tp, tsn;
    std::vector<unsigned char> tbig;
    // descending depth below the root (r02 A/B, bit-identical: factor C3
    // 1.75 -> 1.54 ms, C4 10.56 -> 9.94 ms, C2 within 1 %)
    bool by_depth = true;
    if (const char* e = std::getenv("HYKKT_MF_ORDER")) by_depth = std::atoi(e) == 1;
    level_tasks(s, [&](int sn) { return s.sn_nrows[sn] >= big_rows; }, tp, tsn, tbig, by_depth);
    c.mf_uoff.upload(uo, st);
    c.mf_task_ptr.upload(tp, st);
    c.mf_task_sn.upload(tsn.empty() ? std::vector<int>{0} : tsn, st);
    c.mf_task_big.upload(tbig.empty() ? std::vector<unsigned char>{0} : tbig, st);
    c.mf_ntasks = static_cast<int>(tbig.size());
    c.mf_ubuf.alloc(static_cast<std::size_t>(std::max<long long>(1, uo.back())));
  }
  {
    // triangular-solve task list: wide supernodes (panel >= HYKKT_TRSV_WIDE
    // entries, rows within the shared staging buffer) as CTA tasks
    // B200 sweep: smaller trees (C1-C3) gain from more CTA tasks (256 entries),
    // the 324k-supernode C4 tree from keeping the 48 wide CTAs to its top (1024)
    // trees up to 16384 supernodes (one CTA per SM): 512 with 16 wide CTAs
    // (r02 A/B: ACTIVSg500 179 -> 175, ACTIVSg2000 245 -> 239.5 us per CG iteration)
    long long wide = s.nsup <= 16384 ? 512 : (s.nsup <= 65536 ? 256 : 1024);
    // trees up to 65536 supernodes (C1-C3): narrow tasks as calls with every
    // task kind pre-waiting (r02: C1 322 -> 260, C2 392 -> 323, C3 567 -> 544
    // us / CG iteration); larger trees keep them inlined (C4 1553 vs 1897)
    c.tr_call = s.nsup <= 65536 ? 1 : 0;
    {
      // solve grids: one CTA per SM for trees up to 16384 supernodes (r02
      // A/B: C1 197 -> 181, C2 257 -> 249 us per CG iteration: fewer pollers
      // and cheaper grid barriers), two above
      int per_sm = s.nsup <= 16384 ? 1 : 2;
      if (const char* e = std::getenv("HYKKT_SOLVE_CTAS_PER_SM")) per_sm = std::max(1, std::atoi(e));
      c.cg_grid = std::min(c.coop_cg_blocks, per_sm * c.num_sms);
      c.trsv_grid = std::min(c.coop_trsv_blocks, per_sm * c.num_sms);
    }
    if (const char* e = std::getenv("HYKKT_TRSV_CALL")) c.tr_call = std::atoi(e) != 0;
    if (const char* e = std::getenv("HYKKT_TRSV_WIDE")) wide = std::max(1ll, std::atoll(e));
    std::vector<int> pos(std::max<idx>(1, s.nsup));

    for (idx k = 0; k < s.nsup; ++k) pos[s.order[k]] = static_cast<int>(k);
    // bottom levels: every supernode narrow enough for a thread (w <= 4,
    // nrows <= 16) and the level wide enough to fill the GPU
    // (the w <= 8 / 32-row variant serialises each row's gathers in one
    // thread and loses to the warp tasks at ACTIVSg10k / 70k: opt-in only)
    int nbot = 0, minlev = 16384;
    if (const char* e = std::getenv("HYKKT_TRSV_BOTTOM_MIN")) minlev = std::atoi(e);
    const bool allow_wide = std::getenv("HYKKT_TRSV_BOTTOM_WIDE") != nullptr;
    std::vector<int> bptr{0}, bsn;
    std::vector<unsigned char> bwide;
    {
      idx q = 0;
      while (q < s.nsup) {
        const int lev = s.sn_level[s.order[q]];
        idx q1 = q;
        bool ok = true, small = true;
        while (q1 < s.nsup && s.sn_level[s.order[q1]] == lev) {
          const int sn = s.order[q1];
          const int w = s.sn_first[sn + 1] - s.sn_first[sn], nr = s.sn_nrows[sn];
          ok = ok && (allow_wide ? w <= 8 && nr <= 32 : w <= 4 && nr <= 16);
          small = small && w <= 4 && nr <= 16;
          ++q1;
        }
        if (!ok || q1 - q < minlev || lev != nbot) break;
        for (idx k = q; k < q1; ++k) bsn.push_back(s.order[k]);
        bptr.push_back(static_cast<int>(bsn.size()));
        bwide.push_back(small ? 0 : 1);
        ++nbot;
        q = q1;
      }
    }
    c.tr_bot_wide.upload(bwide.empty() ? std::vector<unsigned char>{0} : bwide, st);
    c.tr_nbot = nbot;
    c.tr_bot_ptr.upload(bptr, st);
    c.tr_bot_sn.upload(bsn.empty() ? std::vector<int>{0} : bsn, st);
    // Task-stream orders.  Backward: parents before children by descending
    // level (height above the leaves: the longest remaining path first).
    // Forward: either ascending level, or (HYKKT_TRSV_FWD_ORDER=1) by
    // descending depth below the root, so the supernodes with the longest
    // path still ahead of them (the deep chains under the top separators)
    // are claimed first.  Both are topological; the wide and narrow streams
    // of one pass always share the pass's order (deadlock freedom).
    std::vector<int> fwd_seq(s.order.begin() + static_cast<std::ptrdiff_t>(bsn.size()), s.order.end());
    {
      // depth order above 32768 supernodes (r02 A/B, bit-identical results:
      // C3 497 -> 451, C4 1383 -> 1157 us per CG iteration; C1 / C2 within 1 %)
      int fo = s.nsup > 32768 ? 1 : 0;
      if (const char* e = std::getenv("HYKKT_TRSV_FWD_ORDER")) fo = std::atoi(e);
      if (fo == 1) {
        const std::vector<int> depth = sn_depth(s);
        std::stable_sort(fwd_seq.begin(), fwd_seq.end(), [&](int x, int y) { return depth[x] > depth[y]; });
      }
    }
    {
      // rows above the bottom levels (TrsvArgs::bt_rows)
      std::vector<int> rows;
      for (int sn : fwd_seq)
        for (int r = s.sn_first[sn]; r < s.sn_first[sn + 1]; ++r) rows.push_back(r);
      c.tr_nbt_rows = static_cast<int>(rows.size());
      c.tr_bt_rows.upload(rows.empty() ? std::vector<int>{0} : rows, st);
      c.cg_bt.alloc(std::max<idx>(1, s.n));
      // on by default (r02 A/B, bit-identical: C1 226 -> 200, C2 281 -> 255,
      // C3 466 -> 434, C4 1160 -> 1035 us per CG iteration)
      c.cg_bt_on = 1;
      if (const char* e = std::getenv("HYKKT_CG_BT")) c.cg_bt_on = std::atoi(e) != 0;
    }
    auto is_wide = [&](int sn) {
      const long long w = s.sn_first[sn + 1] - s.sn_first[sn];
      return s.sn_nrows[sn] <= dev::kWideMaxRows && w * s.sn_nrows[sn] >= wide;
    };
    std::vector<int> wid, nar, wid_lev, nar_lev;  // forward order / level order
    for (int sn : fwd_seq) (is_wide(sn) ? wid : nar).push_back(sn);
    {
      // backward lists: reverse level order (descending height), or the
      // reverse of the forward order (r02 A/B: ACTIVSg10k-sized trees 435 ->
      // 423 us per CG iteration, the 324k-supernode C4 tree 892 -> 934)
      const char* e = std::getenv("HYKKT_TRSV_BWD_ORDER");
      const bool rev_fwd = e ? std::atoi(e) == 1 : (s.nsup > 32768 && s.nsup <= 65536);
      if (rev_fwd) {
        for (int sn : fwd_seq) (is_wide(sn) ? wid_lev : nar_lev).push_back(sn);
      } else {
        for (idx q = static_cast<idx>(bsn.size()); q < s.nsup; ++q) {
          const int sn = s.order[q];
          (is_wide(sn) ? wid_lev : nar_lev).push_back(sn);
        }
      }
    }
    // Q-form: every wide supernode (w <= kQMaxW) gets Q = [L_ss^-1; L_below
    // L_ss^-1] after each factorization and runs as independent row /
    // column slices over the wide CTAs (HYKKT_QFORM=0 keeps whole-supernode
    // substitution tasks)
    c.q_nrows = c.q_nsf = c.q_nsb = 0;
    {
      // default on for trees above 65536 supernodes (C4: 1491 -> 1430 us per
      // CG iteration with 96 wide CTAs, r02); the smaller trees are neutral
      const char* e = std::getenv("HYKKT_QFORM");
      bool on = e ? std::atoi(e) != 0 : s.nsup > 65536;
      for (int sn : wid)
        if (s.sn_first[sn + 1] - s.sn_first[sn] > dev::kQMaxW) on = false;
      if (on && !wid.empty()) {
        std::vector<long long> qo(s.nsup, -1);
        std::vector<int> items, sf, sb;
        long long tot = 0;
        for (int sn : wid) {
          const int w = s.sn_first[sn + 1] - s.sn_first[sn], nr = s.sn_nrows[sn];
          qo[sn] = tot;
          tot += static_cast<long long>(w) * nr;
          for (int qr = 0; qr < nr; ++qr) items.insert(items.end(), {sn, qr});
          for (int r0 = 0; r0 < nr; r0 += 32) sf.insert(sf.end(), {sn, r0, std::min(r0 + 32, nr), 0});
        }
        for (auto it = wid_lev.rbegin(); it != wid_lev.rend(); ++it) {
          const int sn = *it, w = s.sn_first[sn + 1] - s.sn_first[sn];
          for (int c0 = 0; c0 < w; c0 += kThreads / 32) sb.insert(sb.end(), {sn, c0, std::min(c0 + kThreads / 32, w), 0});
        }
        c.q_buf.alloc(static_cast<std::size_t>(tot));
        c.q_off.upload(qo, st);
        c.q_items.upload(items, st);
        c.q_sf.upload(sf, st);
        c.q_sb.upload(sb, st);
        c.q_nrows = static_cast<int>(items.size() / 2);
        c.q_nsf = static_cast<int>(sf.size() / 4);
        c.q_nsb = static_cast<int>(sb.size() / 4);
        c.q_ver = -1;
      }
    }
    // chains: a narrow supernode (w <= 4, rows <= 32) whose parent is a
    // narrow supernode with no other child continues into it; each maximal
    // chain becomes one narrow-stream entry, at its lowest member's position
    // forward and its top member's position backward, solved by one warp.
    // With the inlined tasks (C4) the members run one after the other
    // through the ordinary task code (1445 -> 1392 us per CG iteration);
    // with task calls (C1-C3) the chain kernels hand values over in
    // registers and prefetch each member's static data (chain_fwd /
    // chain_bwd: C3 530 -> 501; without the hand-off chains were slower,
    // C2 285 -> 351).  HYKKT_TRSV_CHAINS=0/1, HYKKT_TRSV_CHAIN_REGS=0/1.
    std::vector<int> chain_ptr{0}, chain_sn, nar_bwd;
    {
      const char* e = std::getenv("HYKKT_TRSV_CHAINS");
      const bool on = e ? std::atoi(e) != 0 : true;
      std::vector<char> is_nar(s.nsup, 0), link_up(s.nsup, 0), linked_from_below(s.nsup, 0);
      auto small = [&](int sn) {
        return s.sn_first[sn + 1] - s.sn_first[sn] <= 4 && s.sn_nrows[sn] <= 32;
      };
      for (int sn : nar) is_nar[sn] = 1;
      if (on) {
        for (int sn : nar) {
          const int p = s.sn_parent[sn];
          if (p >= 0 && is_nar[p] && small(sn) && small(p) && s.child_ptr[p + 1] - s.child_ptr[p] == 1) {
            link_up[sn] = 1;
            linked_from_below[p] = 1;
          }
        }
      }
      std::vector<int> out, top_of(s.nsup, -1);
      out.reserve(nar.size());
      for (int sn : nar) {
        if (linked_from_below[sn]) continue;  // emitted with the chain below it
        if (!link_up[sn]) {
          out.push_back(sn);
          continue;
        }
        // split into chains of at most 32 members (one lane per member)
        int x = sn;
        for (;;) {
          const int k = static_cast<int>(chain_ptr.size()) - 1;
          int len = 0, top = x;
          for (;; x = s.sn_parent[x]) {
            chain_sn.push_back(x);
            top = x;
            ++len;
            if (!link_up[x] || len == 32) break;
          }
          top_of[top] = k;
          chain_ptr.push_back(static_cast<int>(chain_sn.size()));
          out.push_back(-k - 1);
          if (!link_up[top]) break;
          x = s.sn_parent[top];  // the next piece starts above this one
        }
      }
      // backward order: reverse topological, each chain at its top member
      for (auto it = nar_lev.rbegin(); it != nar_lev.rend(); ++it) {
        const int sn = *it;
        if (top_of[sn] >= 0) nar_bwd.push_back(-top_of[sn] - 1);
        else if (!link_up[sn] && !linked_from_below[sn]) nar_bwd.push_back(sn);
      }
      nar.swap(out);
    }
    c.tr_nar_bwd.upload(nar_bwd.empty() ? std::vector<int>{0} : nar_bwd, st);
    // register hand-off tables (kernels_solve.cuh chain_fwd / chain_bwd)
    {
      const int nslot = s.sn_rows_ptr.back();
      std::vector<int> fsrc(std::max(1, nslot), -1), bsrc(std::max(1, nslot), -1);
      for (std::size_t k = 0; k + 1 < chain_ptr.size(); ++k) {
        for (int i = chain_ptr[k]; i < chain_ptr[k + 1]; ++i) {
          const int sn = chain_sn[i], rp = s.sn_rows_ptr[sn], w = s.sn_first[sn + 1] - s.sn_first[sn];
          const int nr = s.sn_nrows[sn];
          if (i > chain_ptr[k]) {  // forward: from the member below
            const int c2 = chain_sn[i - 1], wc = s.sn_first[c2 + 1] - s.sn_first[c2];
            for (int q = 0; q < nr; ++q) {
              const int e0 = s.gat_ptr[rp + q], e1 = s.gat_ptr[rp + q + 1];
              if (e1 - e0 > 1) throw std::logic_error("chain member row with more than one gather");
              if (e1 > e0) fsrc[rp + q] = wc + (s.gat_idx[e0] - s.u_off[c2]);
            }
          }
          if (i + 1 < chain_ptr[k + 1]) {  // backward: from the member above
            const int p = chain_sn[i + 1], fp = s.sn_first[p], wp = s.sn_first[p + 1] - fp;
            const int* Rp = s.sn_rows.data() + s.sn_rows_ptr[p];
            const int nrp = s.sn_nrows[p];
            for (int q = w; q < nr; ++q) {
              const int col = s.sn_rows[rp + q];
              if (col >= fp && col < fp + wp) {
                bsrc[rp + q] = col - fp;
              } else {
                const int pos = static_cast<int>(std::lower_bound(Rp + wp, Rp + nrp, col) - Rp);
                if (pos >= nrp || Rp[pos] != col) throw std::logic_error("chain member row outside its parent");
                bsrc[rp + q] = (pos - wp) | (1 << 8);
              }
            }
          }
        }
      }
      const char* e = std::getenv("HYKKT_TRSV_CHAIN_REGS");
      c.tr_chain_regs = chain_sn.empty() ? 0 : (e ? std::atoi(e) != 0 : 1);
      c.tr_chain_fsrc.upload(fsrc, st);
      c.tr_chain_bsrc.upload(bsrc, st);
    }
    c.tr_chain_ptr.upload(chain_ptr, st);
    c.tr_chain_sn.upload(chain_sn.empty() ? std::vector<int>{0} : chain_sn, st);
    c.tr_wid.upload(wid.empty() ? std::vector<int>{0} : wid, st);
    std::vector<int> wid_bwd(wid_lev.rbegin(), wid_lev.rend());
    c.tr_wid_bwd.upload(wid_bwd.empty() ? std::vector<int>{0} : wid_bwd, st);
    c.tr_nar.upload(nar.empty() ? std::vector<int>{0} : nar, st);
    c.tr_nwid = static_cast<int>(wid.size());
    c.tr_nnar = static_cast<int>(nar.size());
    c.tr_pos.upload(pos, st);
  }
  build_cluster_plan(c);
  CK(cudaMemsetAsync(c.fac_done.p, 0, sizeof(int) * std::max<idx>(1, s.nsup), st));
  c.epoch = 0;
  c.have_plan = true;
  // the batch buffers and completion flags belong to the previous pattern:
  // a new hykkt_batch_upload is required, and the flags are zeroed again
  // before the next batched factor (epochs restart at 0)
  c.batch = 0;
  c.bb.flags_init = false;
  c.bb.jobs_T = -1;
  c.ks.state = 0;
  c.ruiz_rows_built = false;
  c.have_factor = false;
}

// Zeroed task counters for the next launch (one per pass).
unsigned* fresh_tickets(Ctx& c, long long n) {
  if (static_cast<long long>(c.tickets.n) < n) c.tickets.alloc(static_cast<std::size_t>(n));
  CK(cudaMemsetAsync(c.tickets.p, 0, n * sizeof(unsigned), c.stream));
  return c.tickets.p;
}

StatusBlock read_status(Ctx& c) {
  StatusBlock sb;
  CK(cudaMemcpyAsync(&sb, c.status.p, sizeof(sb), cudaMemcpyDeviceToHost, c.stream));
  CK(cudaStreamSynchronize(c.stream));
  if (sb.abort) {
    unsigned long long fa = 0;
    cudaMemcpyFromSymbol(&fa, dev::g_poll_fail_addr, sizeof(fa));
    if (std::getenv("HYKKT_DEBUG") && fa) {
      const auto* p = reinterpret_cast<const double*>(fa);
      auto in = [&](const hykkt::DBuf<double>& b) { return p >= b.p && p < b.p + b.n; };
      const char* which = in(c.y) ? "y" : in(c.xsol) ? "x" : in(c.ubuf) ? "u" : "?";
      long long off = in(c.y) ? p - c.y.p : in(c.xsol) ? p - c.xsol.p : in(c.ubuf) ? p - c.ubuf.p : -1;
      int owner = -1;
      if (which[0] == 'u') {
        for (idx k = 0; k < c.sp.nsup; ++k)
          if (c.sp.u_off[k] <= off && off < c.sp.u_off[k + 1]) owner = static_cast<int>(k);
      } else if (off >= 0) {
        owner = c.sp.sn_of[off];
      }
      unsigned who = 0;
      cudaMemcpyFromSymbol(&who, dev::g_poll_fail_who, sizeof(who));
      std::fprintf(stderr, "[hykkt] first timed-out wait: %s[%lld] (supernode %d, parent %d) by block %u thread %u\n",
                   which, off, owner, owner >= 0 ? c.sp.sn_parent[owner] : -1, who >> 10, who & 1023);
    }
    throw TimeoutError("device wait timed out (dependency deadlock or lost wake-up); results discarded");
  }
  return sb;
}

void reset_fail(Ctx& c) {
  // fail_col = INT_MAX-ish (0x7f7f7f7f), abort = 0
  CK(cudaMemsetAsync(&c.status.p->fail_col, 0x7f, sizeof(int), c.stream));
  CK(cudaMemsetAsync(&c.status.p->abort, 0, sizeof(int), c.stream));
}

// One factorization attempt on the values in c.src_vals (KKT: H_gamma
// slots), shifted by delta1.  Returns failed column or -1.
int factor_attempt(Ctx& c, const double* src, double delta1, double floor_abs,
                   const double* maxdiag, double floor_rel) {
  const SupernodalPlan& s = c.sp;
  CK(cudaMemsetAsync(c.panel.p, 0, sizeof(double) * std::max<idx>(1, s.panel_size), c.stream));
  c.panel_ver++;
  const int nsrc = static_cast<int>(s.src_to_panel.size());
  if (nsrc > 0) {
    dev::k_scatter<<<blocks_for(nsrc), kThreads, 0, c.stream>>>(
        nsrc, src, c.src_to_panel.p, c.src_row.p, c.src_col.p, delta1, c.panel.p);
    check_launch(c);
  }
  reset_fail(c);
  dev::FactorArgs fa;
  fa.s = c.snplan();
  fa.panel = c.panel.p;
  fa.done = c.fac_done.p;
  fa.epoch = ++c.epoch;
  fa.floor_abs = floor_abs;
  fa.maxdiag = maxdiag;
  fa.floor_rel = floor_rel;
  fa.fail_col = &c.status.p->fail_col;
  fa.abort = &c.status.p->abort;
  fa.ticket = fresh_tickets(c, 1);
  if (s.nsup > 0 && c.mf_on) {
    dev::MfArgs ma;
    ma.s = fa.s;
    ma.panel = c.panel.p;
    ma.ubuf = c.mf_ubuf.p;
    ma.uoff = c.mf_uoff.p;
    ma.task_ptr = c.mf_task_ptr.p;
    ma.task_sn = c.mf_task_sn.p;
    ma.task_big = c.mf_task_big.p;
    ma.ntasks = c.mf_ntasks;
    ma.done = fa.done;
    ma.epoch = fa.epoch;
    ma.floor_abs = floor_abs;
    ma.maxdiag = maxdiag;
    ma.floor_rel = floor_rel;
    ma.fail_col = fa.fail_col;
    ma.abort = fa.abort;
    ma.ticket = fa.ticket;
    coop_launch(c, (const void*)dev::k_mf_factor, c.coop_mf_blocks, &ma);
  } else if (s.nsup > 0) {
    coop_launch(c, (const void*)dev::k_factor, c.coop_factor_blocks, &fa);
  }
  const StatusBlock sb = read_status(c);
  const int failed = sb.fail_col >= static_cast<int>(s.n) ? -1 : sb.fail_col;
  if (std::getenv("HYKKT_DEBUG")) std::fprintf(stderr, "[hykkt] factor attempt delta1=%g failed=%d\n", delta1, failed);
  return failed;
}

dev::TrsvArgs trsv_args(Ctx& c) {
  dev::TrsvArgs ta;
  ta.s = c.snplan();
  ta.panel = c.panel.p;
  ta.y = c.y.p;
  ta.x = c.xsol.p;
  ta.u = c.ubuf.p;
  ta.acc_buf = c.accbuf.p;
  ta.x_out = nullptr;
  ta.abort = &c.status.p->abort;
  ta.rhs.b = nullptr;
  ta.rhs.u = nullptr;
  ta.rhs.j_cp = c.j_cp.p;
  ta.rhs.j_ri = c.j_ri.p;
  ta.rhs.jval = nullptr;
  ta.bar = dev::GridBarrier{c.barrier.p, c.barrier.p + 1};
  ta.trace = nullptr;
  ta.pstamp = nullptr;
  ta.wid_sn = c.tr_wid.p;
  ta.wid_bwd = c.tr_wid_bwd.p;
  ta.nwid = c.tr_nwid;
  ta.nar_sn = c.tr_nar.p;
  ta.nnar = c.tr_nnar;
  ta.nar_bwd = c.tr_nar_bwd.p;
  ta.chain_ptr = c.tr_chain_ptr.p;
  ta.chain_fsrc = c.tr_chain_regs ? c.tr_chain_fsrc.p : nullptr;
  ta.chain_bsrc = c.tr_chain_bsrc.p;
  ta.chain_sn = c.tr_chain_sn.p;
  {
    // CTAs reserved for the wide stream (B200 sweep at C2-C4: 48 of 296)
    int nwc = c.q_nsf > 0 ? 96 : (c.sp.nsup <= 16384 ? 16 : 48);  // Q-form slices are independent: more CTAs pay (r02)
    if (const char* e = std::getenv("HYKKT_TRSV_WIDE_CTAS")) nwc = std::max(1, std::atoi(e));
    nwc = std::min({nwc, c.tr_nwid, std::max(1, std::min(c.cg_grid, c.trsv_grid) / 2)});
    ta.nwc = c.tr_nwid > 0 ? nwc : 0;
    // dedicated wide CTAs (the rest of the nwc help with the narrow forward
    // stream first); at least one
    int nwd = ta.nwc;
    if (const char* e = std::getenv("HYKKT_TRSV_WIDE_DEDICATED")) nwd = std::atoi(e);
    ta.nwd = std::max(1, std::min(nwd, ta.nwc));
    // pre-wait bits: 1 fwd narrow, 2 fwd general, 4 bwd narrow, 8 bwd general
    // (poll one value per dependency before loading); with inlined tasks
    // only the general kinds pre-wait, with task calls all of them (r02 A/B)
    ta.pre_wait = c.tr_call ? 15 : 10;
    if (const char* e = std::getenv("HYKKT_TRSV_PREWAIT")) ta.pre_wait = std::atoi(e);
  }
  ta.tstride = 4;  // wide, narrow forward, narrow backward
  // L1 prefetch in the general tasks (r02 A/B: C4 1036 -> 1022 us per CG
  // iteration, C1-C3 neutral)
  ta.prefetch = 1;
  if (const char* e = std::getenv("HYKKT_TRSV_PREFETCH")) ta.prefetch = std::atoi(e) != 0;
  ta.bt_fill = nullptr;
  ta.bt_rows = c.tr_bt_rows.p;
  ta.nbt_rows = c.tr_nbt_rows;
  // every row's right-hand side before the bottom levels (r02 A/B: C4 903 ->
  // 890 us per CG iteration, C1-C3 -1 %)
  // (r02 A/B: C1-C3 -1.3 / -1.9 / -2.5 % per CG iteration; sums regrouped,
  // <= 1e-13 relative change of the solution)
  ta.cta_gather = 1;
  if (const char* e = std::getenv("HYKKT_CTA_GATHER")) ta.cta_gather = std::atoi(e) != 0;
  ta.bt_all = 1;
  if (const char* e = std::getenv("HYKKT_BT_ALL")) ta.bt_all = std::atoi(e) != 0;
  ta.pos = c.tr_pos.p;
  ta.nbot = c.tr_nbot;
  ta.bot_ptr = c.tr_bot_ptr.p;
  ta.bot_sn = c.tr_bot_sn.p;
  ta.bot_wide = c.tr_bot_wide.p;
  ta.bt = nullptr;
  ta.q = c.q_buf.p;
  ta.qoff = c.q_off.p;
  ta.qs_f = reinterpret_cast<const int4*>(c.q_sf.p);
  ta.nqf = c.q_nsf;
  ta.qs_b = reinterpret_cast<const int4*>(c.q_sb.p);
  ta.nqb = c.q_nsb;
  return ta;
}

// One H^-1 application; the result stays in c.xsol (permuted order) and,
// when x_out is given, is scattered to original order there.
dev::ClArgs cluster_args(Ctx& c) {
  dev::ClArgs a{};
  a.tr = trsv_args(c);
  a.tr.pre_wait = 0;
  a.tr.nbot = 0;
  a.tr.bt = c.cl_bt.p;
  a.bt = c.cl_bt.p;
  a.nlev = c.cl_nlev;
  a.lv = c.cl_lv_ptr.p;
  a.desc = reinterpret_cast<const int4*>(c.cl_desc.p);
  a.cta_sn = c.cl_lv_sn.p;
  a.gat4 = reinterpret_cast<const int4*>(c.cl_gat4.p);
  a.wl = reinterpret_cast<const int4*>(c.cl_wl.p);
  a.wl_ptr = c.cl_wptr.p;
  a.rec = c.cl_rec.p;
  a.vals = c.cl_vals.p;
  a.stamps = std::getenv("HYKKT_CL_STAMPS") ? c.cl_stamps.p : nullptr;
  return a;
}

// Q of the Q-form supernodes from the current factor (once per factor).
void ensure_qform(Ctx& c) {
  if (c.q_nrows == 0 || c.q_ver == c.panel_ver) return;
  const int wpb = kThreads / 32;
  dev::k_qform<<<(c.q_nrows + wpb - 1) / wpb, kThreads, 0, c.stream>>>(
      c.q_nrows, reinterpret_cast<const int2*>(c.q_items.p), c.snplan(), c.panel.p, c.q_off.p, c.q_buf.p);
  check_launch(c);
  c.q_ver = c.panel_ver;
}

void run_trsv(Ctx& c, const double* b, const double* u, const double* jval, double* x_out) {
  const SupernodalPlan& s = c.sp;
  if (s.nsup == 0) return;
  if (c.cl_nlev > 0) {
    dev::ClArgs a = cluster_args(c);
    a.tr.x_out = x_out;
    a.tr.rhs.b = b;
    a.tr.rhs.u = u;
    a.tr.rhs.jval = jval;
    a.mode = 0;
    launch_cluster(c, a);
    return;
  }
  ensure_qform(c);
  dev::TrsvArgs ta = trsv_args(c);
  ta.x_out = x_out;
  ta.rhs.b = b;
  ta.rhs.u = u;
  ta.rhs.jval = jval;
  if (c.cg_bt_on) {
    ta.bt_fill = c.cg_bt.p;
    ta.bt = c.cg_bt.p;
  }
  ta.ticket = fresh_tickets(c, ta.tstride);
  coop_launch(c, c.tr_call ? (const void*)dev::k_trsv<true> : (const void*)dev::k_trsv<false>, c.trsv_grid,
              &ta);
}

dev::CgResultDev run_cg(Ctx& c, const hykkt_config_t& cfg, double delta2) {
  dev::CgArgs a;
  a.tr = trsv_args(c);
  a.tr.rhs.u = c.cg_p.p;
  a.tr.rhs.jval = c.js.p;
  if (c.cg_bt_on) {
    a.tr.bt_fill = c.cg_bt.p;
    a.tr.bt = c.cg_bt.p;
  }
  a.mc = static_cast<int>(c.kp.mc);
  a.jcsr_rp = c.jcsr_rp.p;
  a.jcsr_ci_perm = c.jcsr_ci_perm.p;
  a.jcsr = c.js_csr.p;
  a.rhs = c.cg_rhs.p;
  a.x = c.cg_x.p;
  a.r = c.cg_r.p;
  a.p = c.cg_p.p;
  a.q = c.cg_q.p;
  a.partials = c.partials.p;
  a.delta2 = delta2;
  a.tol = cfg.cg_tol;
  a.thr = cfg.small_quadratic_threshold;
  a.max_iter = cfg.cg_max_iter;
  a.res = &c.status.p->cg;
  if (c.sp.nsup == 0 && c.kp.mc > 0) throw StateError("empty factor with constraints");
  if (c.cl_nlev > 0) {
    dev::ClArgs ca = cluster_args(c);
    ca.tr.rhs = a.tr.rhs;
    ca.mode = 1;
    ca.mc = a.mc;
    ca.jcsr_rp = a.jcsr_rp;
    ca.jcsr_ci_perm = a.jcsr_ci_perm;
    ca.jcsr = a.jcsr;
    ca.rhs = a.rhs;
    ca.x = a.x;
    ca.r = a.r;
    ca.p = a.p;
    ca.q = a.q;
    ca.delta2 = a.delta2;
    ca.tol = a.tol;
    ca.thr = a.thr;
    ca.max_iter = a.max_iter;
    ca.res = a.res;
    launch_cluster(c, ca);
    return read_status(c).cg;
  }
  ensure_qform(c);
  a.tickets = fresh_tickets(c, static_cast<long long>(a.tr.tstride) * (cfg.cg_max_iter + 2));
  a.cstamp = nullptr;
  if (c.cg_stamps) {  // diagnostics (hykkt_debug_cg_phases)
    a.tr.pstamp = c.cg_stamps;
    a.cstamp = c.cg_stamps + 8 * c.cg_grid;
  }
  coop_launch(c, c.tr_call ? (const void*)dev::k_cg<2, true> : c.cg_fn, c.cg_grid, &a);
  return read_status(c).cg;
}

void validate_cfg(const hykkt_config_t& cfg) {
  if (cfg.gamma < 0.0) throw InvalidArgument("gamma must be >= 0");
  if (!(cfg.delta_min > 0.0) || !(cfg.delta_max > 0.0) || cfg.delta_min > cfg.delta_max)
    throw InvalidArgument("need 0 < delta_min <= delta_max");
  if (!std::isfinite(cfg.delta_max)) throw InvalidArgument("delta_max must be finite (the ladder doubles up to it)");
  if (cfg.delta2 < 0.0) throw InvalidArgument("delta2 must be >= 0");
  if (!(cfg.cg_tol > 0.0)) throw InvalidArgument("cg_tol must be positive");
  if (cfg.cg_max_iter <= 0) throw InvalidArgument("cg_max_iter must be > 0");
  if (!(cfg.small_quadratic_threshold > 0.0)) throw InvalidArgument("small_quadratic_threshold must be positive");
  if (!(cfg.pivot_floor > 0.0)) throw InvalidArgument("pivot_floor must be positive");
  if (!(cfg.ruiz_tol > 0.0)) throw InvalidArgument("ruiz_tol must be positive");
  if (cfg.ruiz_max_iters <= 0) throw InvalidArgument("ruiz_max_iters must be > 0");
}

CscPattern pattern_from(idx nrows, idx ncols, const std::int64_t* cp, const std::int64_t* ri) {
  if (!cp) throw InvalidArgument("null column pointer");
  CscPattern p;
  p.nrows = nrows;
  p.ncols = ncols;
  p.cp.assign(cp, cp + ncols + 1);
  if (p.cp.back() < 0) throw InvalidArgument("col_ptr must start at 0 and end at nnz");
  if (p.cp.back() > 0 && !ri) throw InvalidArgument("null row index array");
  p.ri.assign(ri, ri + p.cp.back());
  return p;
}

void analyze_kkt(Ctx& c, idx nx, idx mc, idx md, const std::int64_t* hcp, const std::int64_t* hri,
                 const std::int64_t* jcp, const std::int64_t* jri, const std::int64_t* jdcp,
                 const std::int64_t* jdri, const std::int64_t* perm) {
  if (nx < 0 || mc < 0 || md < 0) throw InvalidArgument("negative dimension");
  if (nx >= (idx{1} << 30) || mc >= (idx{1} << 30) || md >= (idx{1} << 30)) throw InvalidArgument("dimension too large");
  CscPattern h = pattern_from(nx, nx, hcp, hri);
  CscPattern j = pattern_from(mc, nx, jcp, jri);
  CscPattern jd = pattern_from(md, nx, jdcp, jdri);
  c.kp = build_kkt_plan(nx, mc, md, h, j, jd);
  std::vector<idx> pv;
  if (perm) pv.assign(perm, perm + nx);
  c.sp = build_supernodal_plan(c.kp.hg, std::move(pv), c.amalg);
  upload_plan(c, c.kp.hg);
  const KktPlan& k = c.kp;
  cudaStream_t st = c.stream;
  std::vector<int> htc(k.ht.nnz()), hgc(k.hg.nnz());
  for (idx col = 0; col < nx; ++col) {
    for (idx p = k.ht.cp[col]; p < k.ht.cp[col + 1]; ++p) htc[p] = static_cast<int>(col);
    for (idx p = k.hg.cp[col]; p < k.hg.cp[col + 1]; ++p) hgc[p] = static_cast<int>(col);
  }
  c.ht_row.upload(to_i32(k.ht.ri), st);
  c.ht_col.upload(htc, st);
  c.ht_hsrc.upload(k.ht_hsrc, st);
  c.ht_pp.upload(k.ht_prod_ptr, st);
  c.ht_pa.upload(k.ht_prod_a, st);
  c.ht_pb.upload(k.ht_prod_b, st);
  c.ht_pk.upload(k.ht_prod_k, st);
  c.hg_row.upload(to_i32(k.hg.ri), st);
  c.hg_col.upload(hgc, st);
  c.hg_src.upload(k.hg_htsrc, st);
  c.hg_pp.upload(k.hg_prod_ptr, st);
  c.hg_pa.upload(k.hg_prod_a, st);
  c.hg_pb.upload(k.hg_prod_b, st);
  std::vector<int> jcol(k.j.nnz());
  for (idx col = 0; col < nx; ++col) {
    for (idx p = k.j.cp[col]; p < k.j.cp[col + 1]; ++p) jcol[p] = static_cast<int>(col);
  }
  c.j_cp.upload(to_i32(k.j.cp), st);
  c.j_ri.upload(to_i32(k.j.ri), st);
  c.j_col.upload(jcol, st);
  c.jcsr_src.upload(k.jcsr_src, st);
  c.jcsr_rp.upload(k.j_rp, st);
  std::vector<int> ci_perm(k.j_ci.size());
  for (std::size_t e = 0; e < ci_perm.size(); ++e) ci_perm[e] = static_cast<int>(c.sp.iperm[k.j_ci[e]]);
  c.jcsr_ci_perm.upload(ci_perm, st);
  c.jd_cp.upload(to_i32(k.jd.cp), st);
  c.jd_ri.upload(to_i32(k.jd.ri), st);
  c.jdcsr_rp.upload(k.jd_rp, st);
  c.jdcsr_ci.upload(k.jd_ci, st);
  c.jdcsr_src.upload(k.jdcsr_src, st);
  // work buffers
  c.hval.alloc(k.h.nnz());
  c.jval.alloc(k.j.nnz());
  c.jdval.alloc(k.jd.nnz());
  c.d_x.alloc(nx);
  c.d_s.alloc(md);
  c.r_tx.alloc(nx);
  c.r_s.alloc(md);
  c.r_y.alloc(mc);
  c.r_yd.alloc(md);
  c.ht.alloc(k.ht.nnz());
  c.hts.alloc(k.ht.nnz());
  c.js.alloc(k.j.nnz());
  c.js_csr.alloc(k.j.nnz());
  c.r_x.alloc(nx);
  c.rxs.alloc(nx);
  c.rys.alloc(mc);
  c.dscale.alloc(nx + mc);
  c.norms.alloc(nx + mc);
  c.hg.alloc(k.hg.nnz());
  c.rhat.alloc(nx);
  c.maxdiag.alloc(1);
  c.cg_rhs.alloc(mc);
  c.cg_x.alloc(mc);
  c.cg_r.alloc(mc);
  c.cg_p.alloc(mc);
  c.cg_q.alloc(mc);
  c.partials.alloc(4 * static_cast<std::size_t>(std::max(c.coop_cg_blocks, 1)));
  c.dx_s.alloc(nx);
  c.dx.alloc(nx);
  c.dy.alloc(mc);
  c.ds.alloc(md);
  c.dyd.alloc(md);
  CK(cudaStreamSynchronize(st));
  c.have_kkt = true;
  c.have_values = false;
  c.have_assembled = false;
  c.reduced = false;
  c.have_j = true;
}

// Host or device source (UVA: cudaMemcpyDefault); `device_only` rejects
// anything but device memory (the *_device entry points).
void copy_in(double* dst, const double* src, idx n, const char* name, cudaStream_t st, bool device_only) {
  if (n <= 0) return;
  if (!src) throw InvalidArgument(std::string("null ") + name);
  if (device_only) {
    cudaPointerAttributes at{};
    if (cudaPointerGetAttributes(&at, src) != cudaSuccess || at.type != cudaMemoryTypeDevice) {
      cudaGetLastError();
      throw InvalidArgument(std::string(name) + " is not a device pointer");
    }
  }
  CK(cudaMemcpyAsync(dst, src, n * sizeof(double), cudaMemcpyDefault, st));
}

void upload_values(Ctx& c, const hykkt_values_t* v, bool device_only = false) {
  if (!c.have_kkt) throw StateError("hykkt_analyze must be called first");
  if (c.reduced) throw StateError("reduced handle: use hykkt_upload_reduced");
  if (!v) throw InvalidArgument("null values");
  const KktPlan& k = c.kp;
  cudaStream_t st = c.stream;
  copy_in(c.hval.p, v->h_val, k.h.nnz(), "h_val", st, device_only);
  copy_in(c.jval.p, v->j_val, k.j.nnz(), "j_val", st, device_only);
  copy_in(c.jdval.p, v->jd_val, k.jd.nnz(), "jd_val", st, device_only);
  copy_in(c.d_x.p, v->d_x, k.nx, "d_x", st, device_only);
  copy_in(c.d_s.p, v->d_s, k.md, "d_s", st, device_only);
  copy_in(c.r_tx.p, v->r_tilde_x, k.nx, "r_tilde_x", st, device_only);
  copy_in(c.r_s.p, v->r_s, k.md, "r_s", st, device_only);
  copy_in(c.r_y.p, v->r_y, k.mc, "r_y", st, device_only);
  copy_in(c.r_yd.p, v->r_yd, k.md, "r_yd", st, device_only);
  c.v = {c.hval.p, c.jval.p, c.jdval.p, c.d_x.p, c.d_s.p, c.r_tx.p, c.r_s.p, c.r_y.p, c.r_yd.p};
  c.o = {c.dx.p, c.dy.p, c.ds.p, c.dyd.p};
  c.have_values = true;
  c.have_assembled = false;
}

// Reduced2x2 values (kkt_system.hpp:56-69): H_tilde on the analysed lower
// pattern, J, r_x, r_y.  D_x = 0 and no J_d, so reduce() returns H_tilde
// and r_x unchanged.
void upload_reduced(Ctx& c, const double* ht, const double* j, const double* rx, const double* ry,
                    bool device_only = false) {
  if (!c.have_kkt || !c.reduced) throw StateError("hykkt_analyze_reduced must be called first");
  const KktPlan& k = c.kp;
  cudaStream_t st = c.stream;
  copy_in(c.hval.p, ht, k.h.nnz(), "h_tilde values", st, device_only);
  copy_in(c.jval.p, j, k.j.nnz(), "j values", st, device_only);
  copy_in(c.r_tx.p, rx, k.nx, "r_x", st, device_only);
  copy_in(c.r_y.p, ry, k.mc, "r_y", st, device_only);
  if (k.nx > 0) CK(cudaMemsetAsync(c.d_x.p, 0, k.nx * sizeof(double), st));
  c.v = {c.hval.p, c.jval.p, c.jdval.p, c.d_x.p, c.d_s.p, c.r_tx.p, c.r_s.p, c.r_y.p, c.r_yd.p};
  c.o = {c.dx.p, c.dy.p, c.ds.p, c.dyd.p};
  c.have_values = true;
  c.have_assembled = false;
}

struct Events {
  cudaEvent_t e[6] = {};
  bool on = false;
  void create() {
    for (auto& x : e) CK(cudaEventCreate(&x));
    on = true;
  }
  void rec(int i, cudaStream_t s) {
    if (on) CK(cudaEventRecord(e[i], s));
  }
  ~Events() {
    for (auto& x : e) if (x) cudaEventDestroy(x);
  }
};

// ---- solve_full / solve_reduced in phases (solver.cpp:222-328) ------------
// Each phase is also reachable on its own through the C ABI
// (hykkt_assemble, hykkt_factor_ladder, hykkt_cg_schur), so a caller of the
// reference's split API (assemble_h_gamma -> factorize_with_ladder ->
// factor_solve / cg_schur) drives the same device code as solve_full.

// reduce -> ruiz_scale (identity for the Reduced2x2 entry points) -> scale
// -> assemble_h_gamma.  Returns the Ruiz sweep count (0 for reduced handles).
void assemble_phase(Ctx& c, const hykkt_config_t& cfg) {
  if (!c.have_values) throw StateError("no values uploaded");
  const dev::AsmPlan ap = c.asmplan();
  cudaStream_t st = c.stream;
  const long long nred = std::max<long long>(ap.n_ht, ap.nx);
  dev::k_reduce<<<blocks_for(nred), kThreads, 0, st>>>(ap, c.v.h, c.v.jd, c.v.dx, c.v.ds,
                                                       c.v.rtx, c.v.rs, c.v.ryd, c.ht.p, c.r_x.p);
  check_launch(c);
  CK(cudaMemsetAsync(&c.status.p->abort, 0, sizeof(int), st));
  if (c.reduced) {
    // solve_reduced takes an already scaled Reduced2x2: D = I (x * 1 = x exactly)
    const int nd = static_cast<int>(ap.nx + ap.mc);
    if (nd > 0) {
      dev::k_fill<<<blocks_for(nd), kThreads, 0, st>>>(c.dscale.p, nd, 1.0);
      check_launch(c);
    }
    CK(cudaMemsetAsync(&c.status.p->ruiz_sweeps, 0, sizeof(int), st));
  } else {
    c.ruiz_flags.alloc(cfg.ruiz_max_iters + 2);
    CK(cudaMemsetAsync(c.ruiz_flags.p, 0, sizeof(int) * (cfg.ruiz_max_iters + 2), st));
    dev::RuizArgs ra;
    ra.p = ap;
    ra.ht = c.ht.p;
    ra.jval = c.v.j;
    ra.d = c.dscale.p;
    ra.norms = c.norms.p;
    ra.unconverged = c.ruiz_flags.p;
    ra.sweeps_out = &c.status.p->ruiz_sweeps;
    ra.max_iters = static_cast<int>(cfg.ruiz_max_iters);
    ra.tol = cfg.ruiz_tol;
    ra.bar = dev::GridBarrier{c.barrier.p, c.barrier.p + 1};
    ra.abort = &c.status.p->abort;
    coop_launch(c, (const void*)dev::k_ruiz, c.coop_ruiz_blocks, &ra);
  }
  const long long nsc = std::max<long long>({(long long)ap.n_ht, (long long)ap.nnz_j, (long long)ap.nx, (long long)ap.mc});
  dev::k_scale<<<blocks_for(nsc), kThreads, 0, st>>>(ap, c.dscale.p, c.ht.p, c.v.j, c.r_x.p, c.v.ry,
                                                     c.hts.p, c.js.p, c.js_csr.p, c.rxs.p, c.rys.p);
  check_launch(c);
  CK(cudaMemsetAsync(c.maxdiag.p, 0, sizeof(double), st));
  const long long nhg = std::max<long long>(ap.n_hg, ap.nx);
  dev::k_hgamma<<<blocks_for(nhg), kThreads, 0, st>>>(ap, cfg.gamma, c.hts.p, c.js.p, c.rxs.p, c.rys.p,
                                                      c.hg.p, c.rhat.p, c.maxdiag.p);
  check_launch(c);
  c.have_assembled = true;
  c.have_factor = false;
}

struct LadderOut {
  int attempts = 0;
  double delta1 = 0.0;
  long long failed = -1;  // failed elimination column of the last attempt, -1 on success
};

// factorize_with_ladder (solver.cpp:108-142) on the H_gamma values `src`
// (slots of the analysed pattern) with the pivot floor relative to
// max |diag| in `maxdiag`: delta1 = 0, then delta_min_current doubling while
// the attempt fails and delta1 <= delta_max / 2.  *dmin_inout carries
// RegularizationState::delta_min_current (<= 0: cfg.delta_min).
LadderOut ladder_phase(Ctx& c, const hykkt_config_t& cfg, const double* src, const double* maxdiag,
                       double* dmin_inout) {
  LadderOut o;
  double dmin = (dmin_inout && *dmin_inout > 0.0) ? *dmin_inout : cfg.delta_min;
  auto attempt = [&](double d1) {
    ++o.attempts;
    return factor_attempt(c, src, d1, 0.0, maxdiag, cfg.pivot_floor);
  };
  int failed = attempt(0.0);
  while (failed >= 0 && o.delta1 <= cfg.delta_max / 2.0) {
    if (o.delta1 == 0.0) {
      o.delta1 = dmin;
    } else {
      dmin *= 2.0;
      o.delta1 = dmin;
    }
    failed = attempt(o.delta1);
  }
  if (dmin_inout) *dmin_inout = dmin;
  o.failed = failed;
  c.have_factor = failed < 0;
  return o;
}

struct CgOut {
  dev::CgResultDev cg{};
  double delta2_used = 0.0;
  long long launches = 0;
};

// cg_schur with the delta2 restart of solve_reduced (solver.cpp:257-264) on
// the rhs already in c.cg_rhs; the solution stays in c.cg_x.
CgOut cg_phase(Ctx& c, const hykkt_config_t& cfg) {
  CgOut o;
  const long long cg0 = c.launches;
  o.cg = run_cg(c, cfg, 0.0);
  if (o.cg.small_quadratic) {
    o.cg = run_cg(c, cfg, cfg.delta2);
    o.delta2_used = cfg.delta2;
  }
  o.launches = c.launches - cg0;
  return o;
}

// w = H^-1 r_hat_x; Schur rhs = J w - r_y (solver.cpp:252-255).
void w_phase(Ctx& c) {
  run_trsv(c, c.rhat.p, nullptr, c.js.p, nullptr);
  if (c.kp.mc > 0) {
    dev::k_schur_rhs<<<blocks_for(c.kp.mc), kThreads, 0, c.stream>>>(
        static_cast<int>(c.kp.mc), c.jcsr_rp.p, c.jcsr_ci_perm.p, c.js_csr.p, c.xsol.p, c.rys.p, c.cg_rhs.p);
    check_launch(c);
  }
}

// dx = H^-1 (r_hat_x - J^T dy) (solver.cpp:276-281); unscale; recover.
void dx_phase(Ctx& c) {
  const KktPlan& k = c.kp;
  const dev::AsmPlan ap = c.asmplan();
  run_trsv(c, c.rhat.p, c.cg_x.p, c.js.p, c.dx_s.p);
  const long long nrec = std::max<long long>({(long long)k.nx, (long long)k.mc, (long long)k.md});
  dev::k_recover<<<blocks_for(nrec), kThreads, 0, c.stream>>>(ap, c.jdcsr_rp.p, c.jdcsr_ci.p, c.jdcsr_src.p,
                                                             c.dscale.p, c.dx_s.p, c.cg_x.p, c.v.jd, c.v.ds,
                                                             c.v.rs, c.v.ryd, c.o.dx, c.o.dy, c.o.ds, c.o.dyd);
  check_launch(c);
}

// density_report (metrics.cpp:242-255) on the reduced pattern.
void density_fields(const Ctx& c, hykkt_report_t& r) {
  const KktPlan& k = c.kp;
  const idx hdiag = k.nx;  // H_tilde always stores the full diagonal
  const idx hfull = 2 * (k.ht.nnz() - hdiag) + hdiag;
  r.nnz_op = hfull + 2 * k.j.nnz() + k.nx;
  r.nnz_fac = 2 * c.sp.l_nnz();
  r.density_ratio = r.nnz_op > 0 ? static_cast<double>(r.nnz_fac) / r.nnz_op : 0.0;
  r.rho_c = k.nx > 0 ? static_cast<double>(r.nnz_fac) / k.nx : 0.0;
}

void metrics_phase(Ctx& c, hykkt_report_t& r);

void solve_resident(Ctx& c, const hykkt_config_t& cfg, double* dmin_inout, int flags,
                    hykkt_report_t* rep) {
  if (!c.have_values) throw StateError("no values uploaded");
  validate_cfg(cfg);
  cudaStream_t st = c.stream;
  const long long launches0 = c.launches;
  Events ev;
  if (flags & HYKKT_FLAG_TIMING) ev.create();
  hykkt_report_t r{};
  const double nan = std::numeric_limits<double>::quiet_NaN();
  r.be_4x4 = r.rr_4x4 = r.be_2x2 = r.rr_2x2 = r.be_2x2_scaled = r.rr_2x2_scaled = nan;
  r.failed_column = -1;
  r.symbolic_reused = 0;
  density_fields(c, r);
  c.timing = hykkt_timing_t{};

  ev.rec(0, st);
  assemble_phase(c, cfg);
  ev.rec(1, st);
  const LadderOut lo = ladder_phase(c, cfg, c.hg.p, c.maxdiag.p, dmin_inout);
  r.factorization_attempts = lo.attempts;
  r.delta1_final = lo.delta1;
  {
    StatusBlock sb;
    CK(cudaMemcpy(&sb, c.status.p, sizeof(sb), cudaMemcpyDeviceToHost));
    r.ruiz_iterations = sb.ruiz_sweeps;
  }
  ev.rec(2, st);
  if (lo.failed >= 0) {
    r.status = 2;  // kFailedDeltaMaxExceeded
    r.failed_column = lo.failed;
    if (rep) *rep = r;
    c.timing.kernel_launches = c.launches - launches0;
    return;
  }
  w_phase(c);
  ev.rec(3, st);
  const CgOut co = cg_phase(c, cfg);
  r.delta2_used = co.delta2_used;
  r.cg_iterations = co.cg.iterations;
  r.cg_relative_residual = co.cg.relres;
  ev.rec(4, st);
  if (!co.cg.converged) {
    r.status = 3;  // kFailedCgNoConvergence
    if (rep) *rep = r;
    c.timing.kernel_launches = c.launches - launches0;
    c.timing.cg_kernel_launches = co.launches;
    return;
  }
  r.status = co.delta2_used > 0.0 ? 1 : 0;
  dx_phase(c);
  ev.rec(5, st);
  CK(cudaStreamSynchronize(st));
  {
    StatusBlock sb;
    CK(cudaMemcpy(&sb, c.status.p, sizeof(sb), cudaMemcpyDeviceToHost));
    if (sb.abort) throw TimeoutError("device wait timed out in the dx solve");
  }
  if (ev.on) {
    float ms[5];
    for (int i = 0; i < 5; ++i) CK(cudaEventElapsedTime(&ms[i], ev.e[i], ev.e[i + 1]));
    c.timing.assemble_ms = ms[0];
    c.timing.factor_ms = ms[1];
    c.timing.solve_w_ms = ms[2];
    c.timing.cg_ms = ms[3];
    c.timing.solve_dx_ms = ms[4];
    float tot;
    CK(cudaEventElapsedTime(&tot, ev.e[0], ev.e[5]));
    c.timing.total_ms = tot;
  }
  c.timing.kernel_launches = c.launches - launches0;
  c.timing.cg_kernel_launches = co.launches;
  if (flags & HYKKT_FLAG_METRICS) metrics_phase(c, r);
  if (rep) *rep = r;
}

void ruiz_rows_prepare(Ctx& c);

// BE / RR of the 4x4, 2x2 and scaled 2x2 systems (metrics.cpp:28-240) on
// the device (kernels_metrics.cuh): only the six numbers come back.
// HYKKT_METRICS_HOST=1 computes them on the host from downloaded vectors
// instead (the cross-check of tests/test_gpu_api.py).
void metrics_host(Ctx& c, hykkt_report_t& r);
void metrics_phase(Ctx& c, hykkt_report_t& r) {
  const bool host = std::getenv("HYKKT_METRICS_HOST") && std::atoi(std::getenv("HYKKT_METRICS_HOST")) != 0;
  if (host) {
    metrics_host(c, r);
    return;
  }
  const KktPlan& k = c.kp;
  ruiz_rows_prepare(c);
  dev::MetricsArgs ma;
  ma.p = c.asmplan();
  ma.rows_ptr = c.ruiz_rp.p;
  ma.rows_ent = reinterpret_cast<const int4*>(c.ruiz_ent.p);
  ma.jd_rp = c.jdcsr_rp.p;
  ma.jd_ci = c.jdcsr_ci.p;
  ma.jd_src = c.jdcsr_src.p;
  ma.h = c.v.h;
  ma.j = c.v.j;
  ma.jd = c.v.jd;
  ma.d_x = c.v.dx;
  ma.d_s = c.v.ds;
  ma.r_tx = c.v.rtx;
  ma.r_s = c.v.rs;
  ma.r_y = c.v.ry;
  ma.r_yd = c.v.ryd;
  ma.dx = c.o.dx;
  ma.ds = c.o.ds;
  ma.dy = c.o.dy;
  ma.dyd = c.o.dyd;
  ma.ht = c.ht.p;
  ma.rx = c.r_x.p;
  ma.hts = c.hts.p;
  ma.js = c.js.p;
  ma.rxs = c.rxs.p;
  ma.rys = c.rys.p;
  ma.dx_s = c.dx_s.p;
  ma.dy_s = c.cg_x.p;
  ma.with_4x4 = c.reduced ? 0 : 1;
  const long long rows = std::max<long long>(k.nx + k.mc, k.nx + 2 * k.md + k.mc);
  const int grid = std::max(1, std::min(blocks_for(rows), 2 * c.num_sms));
  c.met_partials.alloc(static_cast<std::size_t>(grid) * dev::kMetSlots + 6);
  ma.partials = c.met_partials.p;
  double* out = c.met_partials.p + static_cast<std::size_t>(grid) * dev::kMetSlots;
  dev::k_metrics_rows<<<grid, kThreads, 0, c.stream>>>(ma);
  check_launch(c);
  dev::k_metrics_final<<<1, kThreads, 0, c.stream>>>(c.met_partials.p, grid, out);
  check_launch(c);
  double v[6];
  CK(cudaMemcpyAsync(v, out, sizeof(v), cudaMemcpyDeviceToHost, c.stream));
  CK(cudaStreamSynchronize(c.stream));
  if (!c.reduced) {
    r.be_4x4 = v[0];
    r.rr_4x4 = v[1];
  }
  r.be_2x2 = v[2];
  r.rr_2x2 = v[3];
  r.be_2x2_scaled = v[4];
  r.rr_2x2_scaled = v[5];
}

// Host form of the same reports (downloads every vector; diagnostics).
void metrics_host(Ctx& c, hykkt_report_t& r) {
  const KktPlan& k = c.kp;
  const idx nx = k.nx, mc = k.mc, md = k.md;
  auto dl = [&](const double* src, idx n) {
    std::vector<double> h(n);
    if (n) CK(cudaMemcpy(h.data(), src, n * sizeof(double), cudaMemcpyDeviceToHost));
    return h;
  };
  const auto hv = dl(c.v.h, k.h.nnz()), jv = dl(c.v.j, k.j.nnz()), jdv = dl(c.v.jd, k.jd.nnz());
  const auto dxv = dl(c.v.dx, nx), dsv = dl(c.v.ds, md), rtx = dl(c.v.rtx, nx), rs = dl(c.v.rs, md),
             ry = dl(c.v.ry, mc), ryd = dl(c.v.ryd, md);
  const auto htv = dl(c.ht.p, k.ht.nnz()), htsv = dl(c.hts.p, k.ht.nnz()), jsv = dl(c.js.p, k.j.nnz());
  const auto rx = dl(c.r_x.p, nx), rxs = dl(c.rxs.p, nx), rys = dl(c.rys.p, mc);
  const auto sdx = dl(c.dx_s.p, nx), sdy = dl(c.cg_x.p, mc);
  const auto odx = dl(c.o.dx, nx), ody = dl(c.o.dy, mc), ods = dl(c.o.ds, md), odyd = dl(c.o.dyd, md);
  const CscView H{nx, nx, k.h.cp.data(), k.h.ri.data(), hv.data()};
  const CscView J{mc, nx, k.j.cp.data(), k.j.ri.data(), jv.data()};
  const CscView JD{md, nx, k.jd.cp.data(), k.jd.ri.data(), jdv.data()};
  const CscView HT{nx, nx, k.ht.cp.data(), k.ht.ri.data(), htv.data()};
  const CscView HTS{nx, nx, k.ht.cp.data(), k.ht.ri.data(), htsv.data()};
  const CscView JS{mc, nx, k.j.cp.data(), k.j.ri.data(), jsv.data()};
  const ErrorReport e2s = error_report_2x2(HTS, JS, rxs.data(), rys.data(), sdx.data(), sdy.data());
  const ErrorReport e2 = error_report_2x2(HT, J, rx.data(), ry.data(), odx.data(), ody.data());
  r.be_2x2_scaled = e2s.be;
  r.rr_2x2_scaled = e2s.rr;
  r.be_2x2 = e2.be;
  r.rr_2x2 = e2.rr;
  if (!c.reduced) {
    const ErrorReport e4 = error_report_4x4(H, J, JD, dxv.data(), dsv.data(), rtx.data(), rs.data(), ry.data(),
                                            ryd.data(), odx.data(), ods.data(), ody.data(), odyd.data());
    r.be_4x4 = e4.be;
    r.rr_4x4 = e4.rr;
  }
}

void download_solution(Ctx& c, double* dx, double* ds, double* dy, double* dyd) {
  const KktPlan& k = c.kp;
  auto dl = [&](const double* src, double* out, idx n) {
    if (out && n) CK(cudaMemcpyAsync(out, src, n * sizeof(double), cudaMemcpyDefault, c.stream));
  };
  dl(c.o.dx, dx, k.nx);
  dl(c.o.ds, ds, k.md);
  dl(c.o.dy, dy, k.mc);
  dl(c.o.dyd, dyd, k.md);
  CK(cudaStreamSynchronize(c.stream));
}

// ---- resident batch: B systems on the analysed pattern ----------------------
// Values are kept field-major on the device ([field][system][entry]); the
// systems are solved back to back through the single-system path, each with
// a fresh RegularizationState (the reference's independent-matrix mode,
// solver.cpp:374-398).
struct BatchLayout {
  idx sizes[9];
  idx total_per_sys;
};

BatchLayout batch_layout(const KktPlan& k) {
  BatchLayout L;
  const idx s[9] = {k.h.nnz(), k.j.nnz(), k.jd.nnz(), k.nx, k.md, k.nx, k.md, k.mc, k.md};
  L.total_per_sys = 0;
  for (int i = 0; i < 9; ++i) {
    L.sizes[i] = s[i];
    L.total_per_sys += s[i];
  }
  return L;
}

int pow2_at_least(long long v);
void batch_interleave_inputs(Ctx& c, const double* src);

void batch_upload(Ctx& c, idx batch, const hykkt_values_t* v, bool device_only = false) {
  if (!c.have_kkt) throw StateError("hykkt_analyze must be called first");
  if (c.reduced) throw StateError("the batched path takes block-4x4 systems (hykkt_analyze)");
  if (batch <= 0) throw InvalidArgument("batch must be positive");
  if (!v) throw InvalidArgument("null values");
  const BatchLayout L = batch_layout(c.kp);
  c.bvals.alloc(static_cast<std::size_t>(batch * L.total_per_sys));
  const double* src[9] = {v->h_val, v->j_val, v->jd_val, v->d_x, v->d_s, v->r_tilde_x, v->r_s, v->r_y, v->r_yd};
  idx off = 0;
  for (int i = 0; i < 9; ++i) {
    const idx n = batch * L.sizes[i];
    copy_in(c.bvals.p + off, src[i], n, "batch value array", c.stream, device_only);
    off += n;
  }
  const idx nout = c.kp.nx + c.kp.mc + 2 * c.kp.md;
  c.bouts.alloc(static_cast<std::size_t>(batch * nout));
  c.batch = batch;
  c.batch_reports.assign(batch, hykkt_report_t{});
  const int newBp = pow2_at_least(batch);
  if (newBp != c.bb.Bp) c.bb.flags_init = false;
  c.bb.Bp = newBp;
  c.stage_nq = 0;  // a synchronous upload supersedes pending asynchronous ones
  batch_interleave_inputs(c, c.bvals.p);
}

// Asynchronous host upload of the NEXT batch (pinned host memory for true
// overlap): the field-major values go to a staging slot on the handle's copy
// stream while the current batched solve runs; the next
// hykkt_batch_solve_resident consumes the oldest pending upload (at most two
// pending).  Slot reuse waits for its previous consumer.
void ensure_copy_stream(Ctx& c) {
  if (c.copy_stream) return;
  CK(cudaStreamCreateWithFlags(&c.copy_stream, cudaStreamNonBlocking));
  for (int i = 0; i < 2; ++i) {
    CK(cudaEventCreateWithFlags(&c.stage_ready[i], cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&c.stage_free[i], cudaEventDisableTiming));
  }
  CK(cudaEventCreateWithFlags(&c.out_ready, cudaEventDisableTiming));
  CK(cudaEventCreateWithFlags(&c.out_free, cudaEventDisableTiming));
}

void batch_upload_async(Ctx& c, idx batch, const hykkt_values_t* v) {
  if (!c.have_kkt) throw StateError("hykkt_analyze must be called first");
  if (c.reduced) throw StateError("the batched path takes block-4x4 systems (hykkt_analyze)");
  if (batch <= 0) throw InvalidArgument("batch must be positive");
  if (!v) throw InvalidArgument("null values");
  if (c.stage_nq >= 2) throw StateError("two asynchronous uploads already pending");
  ensure_copy_stream(c);
  const BatchLayout L = batch_layout(c.kp);
  const int sl = c.stage_next;
  c.stage_next ^= 1;
  c.stage[sl].alloc(static_cast<std::size_t>(batch * L.total_per_sys));
  if (c.stage_free_rec[sl]) CK(cudaStreamWaitEvent(c.copy_stream, c.stage_free[sl], 0));
  const double* src[9] = {v->h_val, v->j_val, v->jd_val, v->d_x, v->d_s, v->r_tilde_x, v->r_s, v->r_y, v->r_yd};
  idx off = 0;
  for (int i = 0; i < 9; ++i) {
    const idx n = batch * L.sizes[i];
    copy_in(c.stage[sl].p + off, src[i], n, "batch value array", c.copy_stream, false);
    off += n;
  }
  CK(cudaEventRecord(c.stage_ready[sl], c.copy_stream));
  c.stage_batch[sl] = batch;
  c.stage_q[c.stage_nq++] = sl;
}

// Consumes the oldest pending asynchronous upload (called at the start of a
// batched solve): the solve stream waits for its copies, adopts the staged
// buffer as the batch's values and interleaves it.
void batch_take_async(Ctx& c) {
  if (c.stage_nq == 0) return;
  const int sl = c.stage_q[0];
  c.stage_q[0] = c.stage_q[1];
  --c.stage_nq;
  const idx batch = c.stage_batch[sl];
  CK(cudaStreamWaitEvent(c.stream, c.stage_ready[sl], 0));
  const idx nout = c.kp.nx + c.kp.mc + 2 * c.kp.md;
  c.bouts.alloc(static_cast<std::size_t>(batch * nout));
  c.batch = batch;
  c.batch_reports.assign(batch, hykkt_report_t{});
  const int newBp = pow2_at_least(batch);
  if (newBp != c.bb.Bp) c.bb.flags_init = false;
  c.bb.Bp = newBp;
  // the staged values become the batch's field-major values (the in-kernel
  // recover of ks_solve reads J_d, D_s, r_s, r_yd from there); the slot
  // takes the previous buffer, free since the previous solve returned
  std::swap(c.bvals.p, c.stage[sl].p);
  std::swap(c.bvals.n, c.stage[sl].n);
  batch_interleave_inputs(c, c.bvals.p);
  CK(cudaEventRecord(c.stage_free[sl], c.stream));
  c.stage_free_rec[sl] = true;
}

// Asynchronous download of the last batched solve's outputs (pinned host
// memory): a device copy on the solve stream, then the D2H on the copy
// stream, so the next solve overlaps it.  hykkt_batch_sync waits for it.
void batch_download_async(Ctx& c, double* dx, double* ds, double* dy, double* dyd) {
  if (c.batch <= 0) throw StateError("no batch uploaded");
  ensure_copy_stream(c);
  const KktPlan& k = c.kp;
  const idx B = c.batch, nout = k.nx + k.mc + 2 * k.md;
  c.out_stage.alloc(static_cast<std::size_t>(B * nout));
  if (c.out_free_rec) CK(cudaStreamWaitEvent(c.stream, c.out_free, 0));
  CK(cudaMemcpyAsync(c.out_stage.p, c.bouts.p, B * nout * sizeof(double), cudaMemcpyDeviceToDevice, c.stream));
  CK(cudaEventRecord(c.out_ready, c.stream));
  CK(cudaStreamWaitEvent(c.copy_stream, c.out_ready, 0));
  auto dl = [&](const double* srcp, double* out, idx n) {
    if (out && n) CK(cudaMemcpyAsync(out, srcp, n * sizeof(double), cudaMemcpyDefault, c.copy_stream));
  };
  const double* o = c.out_stage.p;
  dl(o, dx, B * k.nx);
  dl(o + B * k.nx, dy, B * k.mc);
  dl(o + B * (k.nx + k.mc), ds, B * k.md);
  dl(o + B * (k.nx + k.mc + k.md), dyd, B * k.md);
  CK(cudaEventRecord(c.out_free, c.copy_stream));
  c.out_free_rec = true;
}

void batch_sync(Ctx& c) {
  if (c.copy_stream) CK(cudaStreamSynchronize(c.copy_stream));
  CK(cudaStreamSynchronize(c.stream));
}

int pow2_at_least(long long v) {
  int p = 32;
  while (p < v) p <<= 1;
  return p;
}

// Interleaved [entry][system] copies of the uploaded field-major values.
void batch_interleave_inputs(Ctx& c, const double* src) {
  auto& bb = c.bb;
  const BatchLayout L = batch_layout(c.kp);
  const int B = static_cast<int>(c.batch), Bp = bb.Bp;
  idx total = 0;
  for (int i = 0; i < 9; ++i) total += L.sizes[i];
  bb.vals.alloc(static_cast<std::size_t>(total) * Bp);
  idx off_in = 0, off_out = 0;
  for (int i = 0; i < 9; ++i) {
    const idx n = L.sizes[i];
    bb.f[i] = bb.vals.p + off_out * Bp;
    if (n > 0) {
      dim3 grid(static_cast<unsigned>((n + 31) / 32), static_cast<unsigned>(Bp / 32));
      dev::kb_interleave<<<grid, 256, 0, c.stream>>>(src + off_in, bb.f[i], static_cast<int>(n), B, Bp);
      check_launch(c);
    }
    off_in += n * B;
    off_out += n;
  }
}

template <typename T>
void balloc(hykkt::DBuf<T>& buf, idx n, int Bp) { buf.alloc(static_cast<std::size_t>(std::max<idx>(n, 1)) * Bp); }

// Batch schedule (rebuilt when the tile count changes).  A supernode is
// WIDE when its panel is large (width * rows >= HYKKT_BIG_WNR, or more rows
// than a warp's shared accumulator) or any child is wide: the top of the
// tree.  Wide supernodes get one CTA job per (supernode, system) and a
// per-system panel layout; the narrow bulk stays lane-mode (lane = system),
// 8 (supernode, tile) warp tasks to a CTA job.  Jobs are in topological
// order: the factor list, then the solve list (forward tasks in level
// order, backward tasks in reverse).
void build_batch_jobs(Ctx& c, int T) {
  const SupernodalPlan& sp = c.sp;
  const long long ns = sp.nsup;
  const int Bp = T * 32;
  const long long wnr = big_task_wnr();
  const int srows = batch_smem_rows();
  std::vector<int> mode(ns, 0);
  for (long long pos = 0; pos < ns; ++pos) {  // children before parents
    const int sn = sp.order[pos];
    const long long w = sp.sn_first[sn + 1] - sp.sn_first[sn], nr = sp.sn_nrows[sn];
    if (w * nr >= wnr || nr > srows) mode[sn] = 1;
    if (mode[sn] && sp.sn_parent[sn] >= 0) mode[sp.sn_parent[sn]] = 1;
  }
  // propagate upward again (a parent marked late still sits after its
  // children in level order, so one more forward sweep closes the set)
  for (long long pos = 0; pos < ns; ++pos) {
    const int sn = sp.order[pos];
    if (mode[sn] && sp.sn_parent[sn] >= 0) mode[sp.sn_parent[sn]] = 1;
  }
  std::vector<int> slot_sn(std::max<idx>(1, sp.panel_size), 0);
  for (long long k = 0; k < ns; ++k) {
    for (idx p = sp.sn_off[k]; p < sp.sn_off[k + 1]; ++p) slot_sn[p] = static_cast<int>(k);
  }
  // factor / forward-solve job order: descending depth below the root, or
  // (HYKKT_BATCH_ORDER=0) level order; both topological
  std::vector<long long> fpos(ns);
  for (long long k = 0; k < ns; ++k) fpos[k] = k;
  // (r02 A/B on the bench batch: factor 11.23 -> 10.79 ms per step)
  const char* bo = std::getenv("HYKKT_BATCH_ORDER");
  if (!bo || std::atoi(bo) == 1) {
    const std::vector<int> depth = sn_depth(sp);
    std::stable_sort(fpos.begin(), fpos.end(),
                     [&](long long x, long long y) { return depth[sp.order[x]] > depth[sp.order[y]]; });
  }
  auto build = [&](bool solve, std::vector<int>& ptr, std::vector<int>& items, std::vector<unsigned char>& kind) {
    ptr.assign(1, 0);
    items.clear();
    kind.clear();
    std::vector<int> group;
    auto flush = [&] {
      if (group.empty()) return;
      items.insert(items.end(), group.begin(), group.end());
      ptr.push_back(static_cast<int>(items.size()));
      kind.push_back(0);
      group.clear();
    };
    for (int pass = 0; pass < (solve ? 2 : 1); ++pass) {
      for (long long k = 0; k < ns; ++k) {
        // items encode the forward position / the backward loop index
        // (kb_trsv decodes backward items as order[ns - 1 - index])
        const long long pos = pass == 0 ? fpos[k] : k;
        const int sn = pass == 0 ? sp.order[pos] : sp.order[ns - 1 - k];
        if (mode[sn]) {
          flush();
          for (int b = 0; b < Bp; ++b) {
            items.push_back(sn * Bp + b);
            ptr.push_back(static_cast<int>(items.size()));
            kind.push_back(static_cast<unsigned char>(pass == 0 ? 1 : 2));
          }
        } else {
          for (int tile = 0; tile < T; ++tile) {
            group.push_back(static_cast<int>(pass * ns * T + pos * T + tile));
            if (group.size() == 8) flush();
          }
        }
      }
      flush();
    }
  };
  std::vector<int> ptr, items;
  std::vector<unsigned char> kind;
  auto& bb = c.bb;
  build(true, ptr, items, kind);
  bb.job_ptr.upload(ptr, c.stream);
  bb.job_items.upload(items, c.stream);
  bb.job_kind.upload(kind, c.stream);
  bb.njobs = static_cast<int>(kind.size());
  build(false, ptr, items, kind);
  bb.fjob_ptr.upload(ptr, c.stream);
  bb.fjob_items.upload(items, c.stream);
  bb.fjob_kind.upload(kind, c.stream);
  bb.nfjobs = static_cast<int>(kind.size());
  bb.mode.upload(mode, c.stream);
  bb.slot_sn.upload(slot_sn, c.stream);
  bb.nwide = std::count(mode.begin(), mode.end(), 1);
  bb.wdone.alloc(static_cast<std::size_t>(std::max<long long>(1, ns)) * Bp);
  CK(cudaMemsetAsync(bb.wdone.p, 0, bb.wdone.n * sizeof(int), c.stream));
  bb.jobs_T = T;
}

// ---- system-per-CTA solve (kernels_sys.cuh) ---------------------------------
constexpr int kKsThreads = 512;
// ring chunk: 2^lg entries (lg = 10: 8 KB of values, 4 KB of indices)
int ks_chunk_lg() {
  static const int v = std::getenv("HYKKT_KS_CHUNK_LG") ? std::max(8, std::min(12, std::atoi(std::getenv("HYKKT_KS_CHUNK_LG")))) : 10;
  return v;
}
constexpr int kKsPmax = 1024;

std::size_t ks_smem_bytes(idx n, int nv, int ni) {
  const std::size_t vbytes = (static_cast<std::size_t>(n) * 8 + 127) & ~static_cast<std::size_t>(127);
  return (static_cast<std::size_t>(nv) * 8 + static_cast<std::size_t>(ni) * 4) * (std::size_t{1} << ks_chunk_lg()) +
         8 * static_cast<std::size_t>(nv + ni) + 8 * 66 + 64 + 8 * dev::kPrN + 8 * kKsPmax + vbytes;
}

// Builds (once per pattern) the stream program of the system-per-CTA solve
// with the largest rings that fit one CTA's shared memory next to the
// solve vector.  Infeasible (the lane-per-system kernels are used) when not
// even 4-chunk rings fit or a supernode block does not fit the rings;
// HYKKT_BATCH_PATH=lane forces the lane path.
// Row lists for kb_ruiz_rows: every stored entry of H_tilde (CSC, lower)
// appears in the list of its row and, off the diagonal, of its column; every
// J entry (CSC) in the list of constraint row n_x + k and of column j.
void ruiz_rows_prepare(Ctx& c) {
  if (c.ruiz_rows_built) return;
  const KktPlan& k = c.kp;
  const idx nrow = k.nx + k.mc, nht = k.ht.nnz();
  std::vector<int> cnt(nrow + 1, 0);
  for (idx col = 0; col < k.nx; ++col) {
    for (idx t = k.ht.cp[col]; t < k.ht.cp[col + 1]; ++t) {
      cnt[k.ht.ri[t] + 1]++;
      if (k.ht.ri[t] != col) cnt[col + 1]++;
    }
    for (idx q = k.j.cp[col]; q < k.j.cp[col + 1]; ++q) {
      cnt[k.nx + k.j.ri[q] + 1]++;
      cnt[col + 1]++;
    }
  }
  std::partial_sum(cnt.begin(), cnt.end(), cnt.begin());
  std::vector<int> ent(4 * std::max<idx>(cnt[nrow], 1), 0), cur(cnt.begin(), cnt.end() - 1);
  auto put = [&](idx r, idx vi, idx da, idx db) {
    const int e = cur[r]++;
    ent[4 * e] = static_cast<int>(vi);
    ent[4 * e + 1] = static_cast<int>(da);
    ent[4 * e + 2] = static_cast<int>(db);
  };
  for (idx col = 0; col < k.nx; ++col) {
    for (idx t = k.ht.cp[col]; t < k.ht.cp[col + 1]; ++t) {
      const idx row = k.ht.ri[t];
      put(row, t, row, col);
      if (row != col) put(col, t, row, col);
    }
    for (idx q = k.j.cp[col]; q < k.j.cp[col + 1]; ++q) {
      const idx r = k.nx + k.j.ri[q];
      put(r, nht + q, r, col);
      put(col, nht + q, r, col);
    }
  }
  c.ruiz_rp.upload(cnt, c.stream);
  c.ruiz_ent.upload(ent, c.stream);
  c.ruiz_rows_built = true;
}

bool ks_prepare(Ctx& c) {
  auto& ks = c.ks;
  if (ks.state != 0) return ks.state == 1;
  ks.state = -1;
  if (const char* e = std::getenv("HYKKT_BATCH_PATH")) {
    if (std::string(e) == "lane") {
      ks.why = "HYKKT_BATCH_PATH=lane";
      return false;
    }
  }
  const SupernodalPlan& sp = c.sp;
  if (sp.nsup == 0) {
    ks.why = "empty factor";
    return false;
  }
  int optin = 0;
  CK(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, c.device));
  int nch = 16 << std::max(0, 10 - ks_chunk_lg());
  while (nch >= 4 && ks_smem_bytes(sp.n, nch, nch) > static_cast<std::size_t>(optin)) nch /= 2;
  if (nch < 4) {
    ks.why = "solve vector does not fit shared memory";
    return false;
  }
  try {
    // L steps of up to n-2 chunks: fewer, larger steps beat a guaranteed
    // one-step lookahead (measured: 62 -> 54 ms per 256-system CG launch)
    int step_chunks = nch - 2;
    if (const char* e = std::getenv("HYKKT_KS_STEP_CHUNKS")) step_chunks = std::atoi(e);
    ks.plan = build_sys_plan(sp, c.kp, ks_chunk_lg(), nch, ks_chunk_lg(), nch, kKsPmax, kKsThreads - 32, step_chunks);
  } catch (const InvalidArgument& e) {
    ks.why = e.what();
    return false;
  }
  cudaStream_t st = c.stream;
  ks.idx.upload(ks.plan.idx, st);
  ks.src.upload(ks.plan.src, st);

  {
    // ks_factor level lists: wide supernodes (CTA tasks) vs narrow (warp tasks)
    std::vector<int> lp(sp.nlevels + 1, 0), wp(sp.nlevels + 1, 0), ls, ws;
    long long wide_max = 0;
    for (int L = 0; L < sp.nlevels; ++L) {
      for (idx k = 0; k < sp.nsup; ++k) {
        if (sp.sn_level[k] != L) continue;
        const long long w = sp.sn_first[k + 1] - sp.sn_first[k], nr = sp.sn_nrows[k];
        if (w * nr > dev::kKfWarpStage / 2) {
          ws.push_back(static_cast<int>(k));
          wide_max = std::max(wide_max, w * nr);
        } else {
          ls.push_back(static_cast<int>(k));
        }
      }
      lp[L + 1] = static_cast<int>(ls.size());
      wp[L + 1] = static_cast<int>(ws.size());
    }
    // per-update descriptors and staging batches (no dependent loads on the
    // device to find block sizes)
    {
      const int nu = sp.upd_ptr[sp.nsup];
      std::vector<int> ud(4 * std::max(nu, 1), 0), ur(std::max(nu, 1), 0);
      std::vector<int> wbp(sp.nsup + 1, 0), wbe, cbp(sp.nsup + 1, 0), cbe;
      const int wcap = dev::kKfWarpStage / 2, ccap = (kKsThreads / 32) * dev::kKfWarpStage - dev::kKfPosStage / 2;
      for (idx t = 0; t < sp.nsup; ++t) {
        auto batches = [&](int cap, std::vector<int>& ends, bool cta) {
          int u = sp.upd_ptr[t];
          while (u < sp.upd_ptr[t + 1]) {
            int ue = u, used = 0, pused = 0;
            while (ue < sp.upd_ptr[t + 1]) {
              const int d = sp.upd_d[ue];
              const int m = sp.sn_nrows[d] - sp.upd_off[ue], wd = sp.sn_first[d + 1] - sp.sn_first[d];
              if (used + m * wd > cap || (cta && pused + m > dev::kKfPosStage)) break;
              used += m * wd;
              pused += m;
              ++ue;
            }
            if (ue == u) ++ue;  // oversized block alone (applied from global memory)
            ends.push_back(ue);
            u = ue;
          }
        };
        batches(wcap, wbe, false);
        wbp[t + 1] = static_cast<int>(wbe.size());
        batches(ccap, cbe, true);
        cbp[t + 1] = static_cast<int>(cbe.size());
      }
      for (int u = 0; u < nu; ++u) {
        const int d = sp.upd_d[u], o = sp.upd_off[u];
        const int m = sp.sn_nrows[d] - o;
        if (m >= (1 << 16) || sp.upd_cnt[u] >= (1 << 15)) throw InvalidArgument("supernode too tall for ks_factor");
        ud[4 * u] = static_cast<int>(sp.sn_off[d] + o);
        ud[4 * u + 1] = sp.sn_nrows[d];
        ud[4 * u + 2] = m | (sp.upd_cnt[u] << 16);
        ud[4 * u + 3] = sp.sn_first[d + 1] - sp.sn_first[d];
        ur[u] = sp.sn_rows_ptr[d] + o;
      }
      ks.upd.upload(ud, st);
      ks.upd_rows.upload(ur, st);
      ks.wb_ptr.upload(wbp, st);
      ks.wb_end.upload(wbe.empty() ? std::vector<int>{0} : wbe, st);
      ks.cb_ptr.upload(cbp, st);
      ks.cb_end.upload(cbe.empty() ? std::vector<int>{0} : cbe, st);
    }
    ks.lev_ptr.upload(lp, st);
    ks.lev_sn.upload(ls.empty() ? std::vector<int>{0} : ls, st);
    ks.wlev_ptr.upload(wp, st);
    ks.wlev_sn.upload(ws.empty() ? std::vector<int>{0} : ws, st);
    // [wide panel staging][per-warp staging areas]
    ks.fsmem = (static_cast<std::size_t>(std::min<long long>(std::max<long long>(wide_max, 1), 12288)) +
                static_cast<std::size_t>(kKsThreads / 32) * dev::kKfWarpStage) * 8;
    CK(cudaFuncSetAttribute((const void*)dev::ks_factor<kKsThreads>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                            static_cast<int>(ks.fsmem)));
    if (const char* e = std::getenv("HYKKT_KS_FACTOR")) ks.factor_on = std::atoi(e) ? 1 : 0;
  }
  ks.smem = ks_smem_bytes(sp.n, nch, nch);
  CK(cudaFuncSetAttribute((const void*)dev::ks_solve<kKsThreads>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                          static_cast<int>(ks.smem)));
  ks.state = 1;
  return true;
}

// The batched device path: every phase of solve_full for all systems at once
// (lane = system).  Per-system outcomes follow the reference exactly: Ruiz
// sweeps, the delta1 ladder (solver.cpp:108-142) with a fresh
// RegularizationState per system, CG stop rules, the delta2 restart.
void batch_solve_resident(Ctx& c, const hykkt_config_t& cfg, int flags, hykkt_report_t* reports) {
  batch_take_async(c);
  if (c.batch <= 0) throw StateError("no batch uploaded");
  validate_cfg(cfg);
  const KktPlan& k = c.kp;
  const SupernodalPlan& sp = c.sp;
  auto& bb = c.bb;
  const int B = static_cast<int>(c.batch), Bp = bb.Bp, T = Bp / 32;
  const dev::BDims bd{B, Bp, T};
  const dev::AsmPlan ap = c.asmplan();
  cudaStream_t st = c.stream;
  const long long launches0 = c.launches;
  Events ev;
  if (flags & HYKKT_FLAG_TIMING) ev.create();
  const idx nx = k.nx, mc = k.mc, md = k.md;
  // work buffers (x Bp)
  balloc(bb.ht, k.ht.nnz(), Bp); balloc(bb.hts, k.ht.nnz(), Bp); balloc(bb.js, k.j.nnz(), Bp);
  balloc(bb.jscsr, k.j.nnz(), Bp); balloc(bb.rx, nx, Bp); balloc(bb.rxs, nx, Bp); balloc(bb.rys, mc, Bp);
  balloc(bb.d, nx + mc, Bp); balloc(bb.norms, nx + mc, Bp); balloc(bb.hg, k.hg.nnz(), Bp);
  balloc(bb.rhat, nx, Bp); balloc(bb.maxdiag, 1, Bp); balloc(bb.panel, sp.panel_size, Bp);
  balloc(bb.y, sp.n, Bp); balloc(bb.xs, sp.n, Bp); balloc(bb.u, sp.u_off.back(), Bp); balloc(bb.acc, sp.sn_rows_ptr.back(), Bp);
  balloc(bb.cgrhs, mc, Bp); balloc(bb.cgx, mc, Bp); balloc(bb.cgr, mc, Bp); balloc(bb.cgp, mc, Bp);
  balloc(bb.cgq, mc, Bp); balloc(bb.dxs, nx, Bp); balloc(bb.odx, nx, Bp); balloc(bb.ody, mc, Bp);
  balloc(bb.ods, md, Bp); balloc(bb.odyd, md, Bp);
  balloc(bb.ruiz_unconv, cfg.ruiz_max_iters + 1, Bp); bb.ruiz_active.alloc(cfg.ruiz_max_iters + 2);
  bb.sweeps.alloc(Bp); bb.delta1.alloc(Bp); bb.active.alloc(Bp); bb.fail.alloc(Bp);
  bb.running.alloc(Bp); bb.start.alloc(Bp); bb.flags.alloc(Bp); bb.iters.alloc(Bp); bb.relres.alloc(Bp);
  bb.live.alloc(cfg.cg_max_iter + 2);
  {
    // a reallocated flag array holds garbage: zero it again
    const int* before[3] = {bb.fac_done.p, bb.fdone.p, bb.bdone.p};
    bb.fac_done.alloc(std::max<idx>(1, sp.nsup) * T); bb.fdone.alloc(std::max<idx>(1, sp.nsup) * T);
    bb.bdone.alloc(std::max<idx>(1, sp.nsup) * T);
    if (before[0] != bb.fac_done.p || before[1] != bb.fdone.p || before[2] != bb.bdone.p) bb.flags_init = false;
  }
  if (!bb.flags_init) {
    CK(cudaMemsetAsync(bb.fac_done.p, 0, bb.fac_done.n * sizeof(int), st));
    CK(cudaMemsetAsync(bb.fdone.p, 0, bb.fdone.n * sizeof(int), st));
    CK(cudaMemsetAsync(bb.bdone.p, 0, bb.bdone.n * sizeof(int), st));
    bb.flags_init = true;
  }
  if (bb.jobs_T != T) build_batch_jobs(c, T);
  dev::BVals v{bb.f[0], bb.f[1], bb.f[2], bb.f[3], bb.f[4], bb.f[5], bb.f[6], bb.f[7], bb.f[8]};
  int* abort = &c.status.p->abort;
  CK(cudaMemsetAsync(abort, 0, sizeof(int), st));
  auto grid_of = [&](long long n) { return blocks_for(n * Bp); };

  ev.rec(0, st);
  // ---- assembly ----
  dev::kb_reduce<<<grid_of(std::max<idx>(k.ht.nnz(), nx)), kThreads, 0, st>>>(ap, bd, v, bb.ht.p, bb.rx.p);
  check_launch(c);
  CK(cudaMemsetAsync(bb.ruiz_unconv.p, 0, bb.ruiz_unconv.n * sizeof(int), st));
  CK(cudaMemsetAsync(bb.ruiz_active.p, 0, bb.ruiz_active.n * sizeof(int), st));
  {
    dev::BRuizArgs ra;
    ra.p = ap;
    ra.bd = bd;
    ra.ht = bb.ht.p;
    ra.jval = v.j;
    ra.d = bb.d.p;
    ra.norms = bb.norms.p;
    ra.unconverged = bb.ruiz_unconv.p;
    ra.active_count = bb.ruiz_active.p;
    ra.sweeps = bb.sweeps.p;
    ra.max_iters = static_cast<int>(cfg.ruiz_max_iters);
    ra.tol = cfg.ruiz_tol;
    ra.bar = dev::GridBarrier{c.barrier.p, c.barrier.p + 1};
    ra.abort = abort;
    static const bool atomics = [] {
      const char* e = std::getenv("HYKKT_RUIZ_ATOMIC");
      return e && std::atoi(e) != 0;
    }();
    if (!atomics) {
      ruiz_rows_prepare(c);
      dev::BRuizRowsArgs rr{ra, c.ruiz_rp.p, reinterpret_cast<const int4*>(c.ruiz_ent.p)};
      coop_launch(c, (const void*)dev::kb_ruiz_rows, c.coop_bruiz_rows_blocks, &rr);
    } else {
      coop_launch(c, (const void*)dev::kb_ruiz, c.coop_bruiz_blocks, &ra);
    }
  }
  dev::kb_scale<<<grid_of(std::max<idx>({k.ht.nnz(), k.j.nnz(), nx, mc})), kThreads, 0, st>>>(
      ap, bd, bb.d.p, bb.ht.p, v.j, bb.rx.p, v.ry, bb.hts.p, bb.js.p, bb.jscsr.p, bb.rxs.p, bb.rys.p);
  check_launch(c);
  CK(cudaMemsetAsync(bb.maxdiag.p, 0, Bp * sizeof(double), st));
  dev::kb_hgamma<<<grid_of(std::max<idx>(k.hg.nnz(), nx)), kThreads, 0, st>>>(
      ap, bd, cfg.gamma, bb.hts.p, bb.js.p, bb.rxs.p, bb.rys.p, bb.hg.p, bb.rhat.p, bb.maxdiag.p);
  check_launch(c);
  ev.rec(1, st);

  // ---- delta1 ladder per system (solver.cpp:108-142) ----
  std::vector<double> d1(Bp, 0.0), dmin(Bp, cfg.delta_min);
  std::vector<int> act(Bp, 1), attempts(Bp, 0), fail(Bp, 0), failed_col(Bp, -1), ok(Bp, 0);
  const dev::SnPlan snp = c.snplan();
  const int nsrc = static_cast<int>(sp.src_to_panel.size());
  const bool sysf = ks_prepare(c) && c.ks.factor_on;
  if (sysf) {
    // per-system contiguous H_gamma values for ks_factor
    auto& ks = c.ks;
    ks.hg.alloc(static_cast<std::size_t>(std::max<idx>(k.hg.nnz(), 1)) * B);
    if (k.hg.nnz() > 0) {
      dim3 grid(static_cast<unsigned>((k.hg.nnz() + 31) / 32), static_cast<unsigned>(Bp / 32));
      dev::kb_deinterleave<<<grid, 256, 0, st>>>(bb.hg.p, ks.hg.p, static_cast<int>(k.hg.nnz()), B, Bp);
      check_launch(c);
    }
  }
  // every round doubles each active system's delta1 until it exceeds
  // delta_max / 2 (solver.cpp:108-142), so the loop ends without a cap
  for (;;) {
    bool any = false;
    for (int b = 0; b < Bp; ++b) any = any || act[b];
    if (!any) break;
    CK(cudaMemcpyAsync(bb.delta1.p, d1.data(), Bp * sizeof(double), cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(bb.active.p, act.data(), Bp * sizeof(int), cudaMemcpyHostToDevice, st));
    if (sysf) {
      auto& ks = c.ks;
      CK(cudaMemsetAsync(bb.fail.p, 0x7f, Bp * sizeof(int), st));
      dev::KfArgs fa{};
      fa.s = snp;
      fa.panel_size = sp.panel_size;
      fa.panel = bb.panel.p;
      fa.hg = ks.hg.p;
      fa.nsrc = nsrc;
      fa.to_panel = c.src_to_panel.p;
      fa.srow = c.src_row.p;
      fa.scol = c.src_col.p;
      fa.delta1 = bb.delta1.p;
      fa.active = bb.active.p;
      fa.maxdiag = bb.maxdiag.p;
      fa.floor_rel = cfg.pivot_floor;
      fa.fail_col = bb.fail.p;
      fa.lev_ptr = ks.lev_ptr.p;
      fa.lev_sn = ks.lev_sn.p;
      fa.wlev_ptr = ks.wlev_ptr.p;
      fa.wlev_sn = ks.wlev_sn.p;
      fa.nlevels = sp.nlevels;
      fa.smem_doubles = static_cast<int>(ks.fsmem / 8) - (kKsThreads / 32) * dev::kKfWarpStage;
      fa.ticket = fresh_tickets(c, 1);
      fa.B = B;
      fa.upd = reinterpret_cast<const int4*>(ks.upd.p);
      fa.upd_rows = ks.upd_rows.p;
      fa.wb_ptr = ks.wb_ptr.p;
      fa.wb_end = ks.wb_end.p;
      fa.cb_ptr = ks.cb_ptr.p;
      fa.cb_end = ks.cb_end.p;
      const int grid = static_cast<int>(std::min<long long>(B, c.num_sms));
      dev::ks_factor<kKsThreads><<<grid, kKsThreads, ks.fsmem, st>>>(fa);
      check_launch(c);
    } else {
    dev::kb_zero_panels<<<blocks_for(sp.panel_size * Bp), kThreads, 0, st>>>(sp.panel_size, bd, snp, bb.mode.p,
                                                                             bb.slot_sn.p, bb.active.p, bb.panel.p);
    check_launch(c);
    if (nsrc > 0) {
      dev::kb_scatter<<<grid_of(nsrc), kThreads, 0, st>>>(nsrc, bd, snp, bb.mode.p, bb.slot_sn.p, bb.hg.p,
                                                          c.src_to_panel.p, c.src_row.p, c.src_col.p, bb.delta1.p,
                                                          bb.active.p, bb.panel.p);
      check_launch(c);
    }
    CK(cudaMemsetAsync(bb.fail.p, 0x7f, Bp * sizeof(int), st));
    dev::BFactorArgs fa;
    fa.s = snp;
    fa.bd = bd;
    fa.panel = bb.panel.p;
    fa.done = bb.fac_done.p;
    fa.epoch = ++c.epoch;
    fa.maxdiag = bb.maxdiag.p;
    fa.floor_rel = cfg.pivot_floor;
    fa.floor_abs = 0.0;
    fa.active = bb.active.p;
    fa.fail_col = bb.fail.p;
    fa.abort = abort;
    fa.ticket = fresh_tickets(c, 1);
    fa.mode = bb.mode.p;
    fa.wdone = bb.wdone.p;
    fa.job_ptr = bb.fjob_ptr.p;
    fa.job_items = bb.fjob_items.p;
    fa.job_kind = bb.fjob_kind.p;
    fa.njobs = bb.nfjobs;
    fa.smem_doubles = static_cast<int>(kBatchSmem / sizeof(double));
    if (sp.nsup > 0) coop_launch(c, (const void*)dev::kb_factor, c.coop_bfactor_blocks, &fa, kBatchSmem);
    }
    CK(cudaMemcpyAsync(fail.data(), bb.fail.p, Bp * sizeof(int), cudaMemcpyDeviceToHost, st));
    read_status(c);
    for (int b = 0; b < Bp; ++b) {
      if (!act[b]) continue;
      ++attempts[b];
      const bool failed = fail[b] < static_cast<int>(sp.n);
      if (!failed) {
        act[b] = 0;
        ok[b] = 1;
      } else if (d1[b] <= cfg.delta_max / 2.0) {
        if (d1[b] == 0.0) {
          d1[b] = dmin[b];
        } else {
          dmin[b] *= 2.0;
          d1[b] = dmin[b];
        }
      } else {
        act[b] = 0;
        failed_col[b] = fail[b];
      }
    }
  }
  ev.rec(2, st);

  std::vector<long long> iters(Bp, 0);
  std::vector<double> relres(Bp, 0.0), d2used(Bp, 0.0);
  std::vector<int> cflags(Bp, 0);
  long long cg_launches = 0;
  if (ks_prepare(c)) {
    // ---- system-per-CTA: w solve, Schur rhs, CG (+ delta2), dx solve,
    // unscale, recover — one launch, one CTA per system at a time ----
    auto& ks = c.ks;
    const SysPlan& P = ks.plan;
    const long long vlen = static_cast<long long>(P.src.size());
    ks.vals.alloc(static_cast<std::size_t>(B) * vlen);
    if (sysf) {
      ks.js.alloc(static_cast<std::size_t>(std::max<idx>(k.j.nnz(), 1)) * B);
      if (k.j.nnz() > 0) {
        dim3 grid(static_cast<unsigned>((k.j.nnz() + 31) / 32), static_cast<unsigned>(Bp / 32));
        dev::kb_deinterleave<<<grid, 256, 0, st>>>(bb.js.p, ks.js.p, static_cast<int>(k.j.nnz()), B, Bp);
        check_launch(c);
      }
      dim3 rg(static_cast<unsigned>((vlen + 255) / 256), static_cast<unsigned>(B));
      dev::ks_remap_sys<<<rg, 256, 0, st>>>(ks.src.p, vlen, sp.panel_size, bb.panel.p, ks.js.p, k.j.nnz(),
                                            ks.vals.p);
      check_launch(c);
    } else {
      dim3 rg(static_cast<unsigned>((vlen + 31) / 32), static_cast<unsigned>((B + 31) / 32));
      dev::ks_remap<<<rg, 256, 0, st>>>(ks.src.p, vlen, snp, bb.mode.p, bb.slot_sn.p, Bp, B, bb.panel.p, bb.js.p,
                                         ks.vals.p);
      check_launch(c);
    }
    auto deint = [&](const double* in, hykkt::DBuf<double>& out, idx n) {
      out.alloc(static_cast<std::size_t>(std::max<idx>(n, 1)) * B);
      if (n <= 0) return;
      dim3 grid(static_cast<unsigned>((n + 31) / 32), static_cast<unsigned>(Bp / 32));
      dev::kb_deinterleave<<<grid, 256, 0, st>>>(in, out.p, static_cast<int>(n), B, Bp);
      check_launch(c);
    };
    deint(bb.rhat.p, ks.rhat, nx);
    deint(bb.rys.p, ks.rys, mc);
    deint(bb.d.p, ks.d, nx + mc);
    ks.ok.upload(ok.data(), B, st);
    ks.iters.alloc(B);
    ks.relres.alloc(B);
    ks.flags.alloc(B);
    ks.d2.alloc(B);
    const int grid = static_cast<int>(std::min<long long>(B, c.num_sms));
    ks.scratch.alloc(static_cast<std::size_t>(grid) * 5 * std::max<idx>(mc, 1));
    ev.rec(3, st);
    dev::KsArgs a{};
    a.n = static_cast<int>(nx);
    a.mc = static_cast<int>(mc);
    a.md = static_cast<int>(md);
    a.idx = ks.idx.p;
    a.vals = ks.vals.p;
    a.vlen = vlen;
    a.vchunk_lg = P.vchunk_lg;
    a.nvchunk = P.nvchunk;
    a.ichunk_lg = P.ichunk_lg;
    a.nichunk = P.nichunk;
    a.pmax = P.pmax;
    for (int i = 0; i < 4; ++i) {
      a.bv0[i] = P.blk[i].v0;
      a.bv1[i] = P.blk[i].v1;
      a.bi0[i] = P.blk[i].i0;
      a.bi1[i] = P.blk[i].i1;
      a.bs0[i] = P.blk[i].s0;
      a.bs1[i] = P.blk[i].s1;
    }
    a.perm = c.perm.p;
    a.iperm = c.iperm.p;
    a.rhat = ks.rhat.p;
    a.rys = ks.rys.p;
    a.d = ks.d.p;
    a.jd_rp = c.jdcsr_rp.p;
    a.jd_ci = c.jdcsr_ci.p;
    a.jd_src = c.jdcsr_src.p;
    {
      // original per-system values as uploaded: [field][system][entry]
      const BatchLayout L = batch_layout(k);
      const double* f[9];
      idx off = 0;
      for (int i = 0; i < 9; ++i) {
        f[i] = c.bvals.p + off;
        off += L.sizes[i] * B;
      }
      a.jd = f[2];
      a.ds_in = f[4];
      a.rs = f[6];
      a.ryd = f[8];
    }
    a.nnz_jd = k.jd.nnz();
    a.odx = c.bouts.p;
    a.ody = c.bouts.p + static_cast<idx>(B) * nx;
    a.ods = a.ody + static_cast<idx>(B) * mc;
    a.odyd = a.ods + static_cast<idx>(B) * md;
    a.scratch = ks.scratch.p;
    a.tol = cfg.cg_tol;
    a.thr = cfg.small_quadratic_threshold;
    a.delta2 = cfg.delta2;
    a.max_iter = cfg.cg_max_iter;
    a.ok = ks.ok.p;
    a.iters = ks.iters.p;
    a.relres = ks.relres.p;
    a.flags = ks.flags.p;
    a.d2used = ks.d2.p;
    a.ticket = fresh_tickets(c, 1);
    a.B = B;
    // history-based longest-first: systems in descending order of their CG
    // iterations in the previous call on this batch (interior-method steps
    // change the values little), so the last wave is not left with the
    // longest systems; first call / other batch size: natural order
    a.order = (static_cast<long long>(ks.lpt_for) == B && ks.lpt_on) ? ks.order.p : nullptr;
    if (ks.prof_on < 0) ks.prof_on = std::getenv("HYKKT_KS_PROF") ? 1 : 0;
    a.debug = std::getenv("HYKKT_KS_DEBUG") ? std::atoi(std::getenv("HYKKT_KS_DEBUG")) : 0;
    a.issuers = 4;
    if (const char* e = std::getenv("HYKKT_KS_ISSUERS")) a.issuers = std::max(1, std::min(32, std::atoi(e)));
    a.feed = 0;  // cp.async from all threads: 2 % faster than the TMA producer lanes since r01e (B200)
    if (const char* e = std::getenv("HYKKT_KS_FEED")) a.feed = std::atoi(e) ? 1 : 0;
    a.prof = nullptr;
    if (ks.prof_on) {
      ks.prof.alloc(static_cast<std::size_t>(grid) * dev::kPrN);
      ks.prof_ctas = grid;
      a.prof = ks.prof.p;
      ks.trace.alloc(static_cast<std::size_t>(P.nsteps + 1) * 81);
      CK(cudaMemsetAsync(ks.trace.p, 0, ks.trace.n * 8, st));
      a.trace = ks.trace.p;
    }
    const long long cg0 = c.launches;
    dev::ks_solve<kKsThreads><<<grid, kKsThreads, ks.smem, st>>>(a);
    check_launch(c);
    cg_launches = c.launches - cg0;
    ev.rec(4, st);
    // failed factorizations: no solution (NaN), as the reference returns none
    for (int b = 0; b < B; ++b) {
      if (ok[b]) continue;
      CK(cudaMemsetAsync(a.odx + static_cast<idx>(b) * nx, 0xff, nx * sizeof(double), st));
      CK(cudaMemsetAsync(a.ody + static_cast<idx>(b) * mc, 0xff, mc * sizeof(double), st));
      CK(cudaMemsetAsync(a.ods + static_cast<idx>(b) * md, 0xff, md * sizeof(double), st));
      CK(cudaMemsetAsync(a.odyd + static_cast<idx>(b) * md, 0xff, md * sizeof(double), st));
    }
    std::vector<int> fl(B);
    std::vector<double> d2(B);
    CK(cudaMemcpyAsync(iters.data(), ks.iters.p, B * sizeof(long long), cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(relres.data(), ks.relres.p, B * sizeof(double), cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(fl.data(), ks.flags.p, B * sizeof(int), cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(d2.data(), ks.d2.p, B * sizeof(double), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    for (int b = 0; b < B; ++b) {
      cflags[b] = fl[b];
      d2used[b] = d2[b];
    }
    if (ks.lpt_on) {
      std::vector<int> ord(B);
      std::iota(ord.begin(), ord.end(), 0);
      std::stable_sort(ord.begin(), ord.end(), [&](int x, int y) { return iters[x] > iters[y]; });
      ks.order.upload(ord, st);
      ks.lpt_for = B;
    }
  } else {

    // ---- w solve + Schur rhs ----
    auto trsv_args = [&](const double* rb, const double* ru, double* x_out, const int* lane_on) {
      dev::BTrsvArgs ta;
      ta.s = snp;
      ta.bd = bd;
      ta.panel = bb.panel.p;
      ta.y = bb.y.p;
      ta.x = bb.xs.p;
      ta.u = bb.u.p;
      ta.acc = bb.acc.p;
      ta.x_out = x_out;
      ta.bar = dev::GridBarrier{c.barrier.p, c.barrier.p + 1};
      ta.smem_rows = batch_smem_rows();
      ta.fdone = bb.fdone.p;
      ta.bdone = bb.bdone.p;
      ta.epoch = 0;
      ta.abort = abort;
      ta.rb = rb;
      ta.ru = ru;
      ta.j_cp = c.j_cp.p;
      ta.j_ri = c.j_ri.p;
      ta.jval = bb.js.p;
      ta.lane_on = lane_on;
      ta.job_ptr = bb.job_ptr.p;
      ta.job_items = bb.job_items.p;
      ta.job_kind = bb.job_kind.p;
      ta.njobs = bb.njobs;
      ta.mode = bb.mode.p;
      ta.smem_doubles = static_cast<int>(kBatchSmem / sizeof(double));
      return ta;
    };
    if (sp.nsup > 0) {
      dev::BTrsvArgs ta = trsv_args(bb.rhat.p, nullptr, nullptr, nullptr);
      ta.epoch = ++c.epoch;
      ta.ticket = fresh_tickets(c, 1);
      coop_launch(c, (const void*)dev::kb_trsv, c.coop_btrsv_blocks, &ta, kBatchSmem);
    }
    if (mc > 0) {
      dev::kb_schur_rhs<<<grid_of(mc), kThreads, 0, st>>>(static_cast<int>(mc), bd, c.jcsr_rp.p, c.jcsr_ci_perm.p,
                                                          bb.jscsr.p, bb.xs.p, bb.rys.p, bb.cgrhs.p);
      check_launch(c);
    }
    ev.rec(3, st);

    // ---- CG (+ delta2 restart) ----
    std::vector<int> start(Bp, 0);
    const long long cg0 = c.launches;
    auto run_bcg = [&](const std::vector<int>& which, double delta2) {
      CK(cudaMemcpyAsync(bb.start.p, which.data(), Bp * sizeof(int), cudaMemcpyHostToDevice, st));
      CK(cudaMemsetAsync(bb.live.p, 0, bb.live.n * sizeof(int), st));
      dev::BCgArgs a;
      a.tr = trsv_args(nullptr, bb.cgp.p, nullptr, bb.running.p);
      a.mc = static_cast<int>(mc);
      a.jcsr_rp = c.jcsr_rp.p;
      a.jcsr_ci_perm = c.jcsr_ci_perm.p;
      a.jcsr = bb.jscsr.p;
      a.rhs = bb.cgrhs.p;
      a.x = bb.cgx.p;
      a.r = bb.cgr.p;
      a.p = bb.cgp.p;
      a.q = bb.cgq.p;
      a.part = nullptr;
      a.running = bb.running.p;
      a.start = bb.start.p;
      a.delta2 = delta2;
      a.tol = cfg.cg_tol;
      a.thr = cfg.small_quadratic_threshold;
      a.max_iter = cfg.cg_max_iter;
      a.epoch_base = c.epoch;
      a.iters = bb.iters.p;
      a.relres = bb.relres.p;
      a.flags = bb.flags.p;
      a.live = bb.live.p;
      a.tickets = fresh_tickets(c, cfg.cg_max_iter + 2);
      a.bar = dev::GridBarrier{c.barrier.p, c.barrier.p + 1};
      const int blocks = c.coop_bcg_blocks;
      bb.part.alloc(static_cast<std::size_t>(blocks) * kThreads);
      a.part = bb.part.p;
      coop_launch(c, (const void*)dev::kb_cg, blocks, &a, kBatchSmem);
      c.epoch += static_cast<int>(std::min<long long>(cfg.cg_max_iter, 1 << 28)) + 1;
      CK(cudaMemcpyAsync(iters.data(), bb.iters.p, Bp * sizeof(long long), cudaMemcpyDeviceToHost, st));
      CK(cudaMemcpyAsync(relres.data(), bb.relres.p, Bp * sizeof(double), cudaMemcpyDeviceToHost, st));
      CK(cudaMemcpyAsync(cflags.data(), bb.flags.p, Bp * sizeof(int), cudaMemcpyDeviceToHost, st));
      read_status(c);
    };
    if (mc > 0) {
      run_bcg(ok, 0.0);
      std::vector<int> redo(Bp, 0);
      bool any = false;
      for (int b = 0; b < Bp; ++b) {
        if (ok[b] && cflags[b] == 2) {
          redo[b] = 1;
          d2used[b] = cfg.delta2;
          any = true;
        }
      }
      if (any) run_bcg(redo, cfg.delta2);
    } else {
      CK(cudaMemsetAsync(bb.cgx.p, 0, bb.cgx.n * sizeof(double), st));
      for (int b = 0; b < Bp; ++b) cflags[b] = 1;
    }
    cg_launches = c.launches - cg0;
    ev.rec(4, st);

    // ---- dx solve, unscale, recover ----
    if (sp.nsup > 0) {
      dev::BTrsvArgs ta = trsv_args(bb.rhat.p, bb.cgx.p, bb.dxs.p, nullptr);
      ta.epoch = ++c.epoch;
      ta.ticket = fresh_tickets(c, 1);
      coop_launch(c, (const void*)dev::kb_trsv, c.coop_btrsv_blocks, &ta, kBatchSmem);
    }
    dev::kb_recover<<<grid_of(std::max<idx>({nx, mc, md})), kThreads, 0, st>>>(
        ap, bd, c.jdcsr_rp.p, c.jdcsr_ci.p, c.jdcsr_src.p, bb.d.p, bb.dxs.p, bb.cgx.p, v, bb.odx.p, bb.ody.p,
        bb.ods.p, bb.odyd.p);
    check_launch(c);
    {
      const idx ns[4] = {nx, mc, md, md};
      const double* src[4] = {bb.odx.p, bb.ody.p, bb.ods.p, bb.odyd.p};
      idx off = 0;
      for (int i = 0; i < 4; ++i) {
        if (ns[i] > 0) {
          dim3 grid(static_cast<unsigned>((ns[i] + 31) / 32), static_cast<unsigned>(Bp / 32));
          dev::kb_deinterleave<<<grid, 256, 0, st>>>(src[i], c.bouts.p + off, static_cast<int>(ns[i]), B, Bp);
          check_launch(c);
        }
        off += ns[i] * B;
      }
    }
  }
  ev.rec(5, st);
  std::vector<int> sweeps(Bp, 0);
  CK(cudaMemcpyAsync(sweeps.data(), bb.sweeps.p, Bp * sizeof(int), cudaMemcpyDeviceToHost, st));
  read_status(c);

  c.timing = hykkt_timing_t{};
  if (ev.on) {
    float ms[5];
    for (int i = 0; i < 5; ++i) CK(cudaEventElapsedTime(&ms[i], ev.e[i], ev.e[i + 1]));
    c.timing.assemble_ms = ms[0];
    c.timing.factor_ms = ms[1];
    c.timing.solve_w_ms = ms[2];
    c.timing.cg_ms = ms[3];
    c.timing.solve_dx_ms = ms[4];
    float tot;
    CK(cudaEventElapsedTime(&tot, ev.e[0], ev.e[5]));
    c.timing.total_ms = tot;
  }
  c.timing.kernel_launches = c.launches - launches0;
  c.timing.cg_kernel_launches = cg_launches;

  const double nan = std::numeric_limits<double>::quiet_NaN();
  const idx hdiag = k.nx, hfull = 2 * (k.ht.nnz() - hdiag) + hdiag;
  for (int b = 0; b < B; ++b) {
    hykkt_report_t r{};
    r.be_4x4 = r.rr_4x4 = r.be_2x2 = r.rr_2x2 = r.be_2x2_scaled = r.rr_2x2_scaled = nan;
    r.nnz_op = hfull + 2 * k.j.nnz() + k.nx;
    r.nnz_fac = 2 * sp.l_nnz();
    r.density_ratio = r.nnz_op > 0 ? static_cast<double>(r.nnz_fac) / r.nnz_op : 0.0;
    r.rho_c = k.nx > 0 ? static_cast<double>(r.nnz_fac) / k.nx : 0.0;
    r.ruiz_iterations = sweeps[b];
    r.factorization_attempts = attempts[b];
    r.delta1_final = d1[b];
    r.failed_column = failed_col[b];
    if (!ok[b]) {
      r.status = 2;
    } else {
      r.delta2_used = d2used[b];
      r.cg_iterations = iters[b];
      r.cg_relative_residual = relres[b];
      r.status = cflags[b] == 1 ? (d2used[b] > 0.0 ? 1 : 0) : 3;
    }
    c.batch_reports[b] = r;
    if (reports) reports[b] = r;
  }
}

void batch_download(Ctx& c, double* dx, double* ds, double* dy, double* dyd) {
  if (c.batch <= 0) throw StateError("no batch uploaded");
  const KktPlan& k = c.kp;
  const idx B = c.batch;
  auto dl = [&](const double* src, double* out, idx n) {
    if (out && n) CK(cudaMemcpyAsync(out, src, n * sizeof(double), cudaMemcpyDefault, c.stream));
  };
  const double* o = c.bouts.p;
  dl(o, dx, B * k.nx);
  dl(o + B * k.nx, dy, B * k.mc);
  dl(o + B * (k.nx + k.mc), ds, B * k.md);
  dl(o + B * (k.nx + k.mc + k.md), dyd, B * k.md);
  CK(cudaStreamSynchronize(c.stream));
}

template <typename F>
int guarded(F&& f) {
  try {
    f();
    return HYKKT_OK;
  } catch (const InvalidArgument& e) {
    g_last_error = e.what();
    return HYKKT_ERR_INVALID;
  } catch (const CudaError& e) {
    g_last_error = e.what();
    return HYKKT_ERR_CUDA;
  } catch (const StateError& e) {
    g_last_error = e.what();
    return HYKKT_ERR_STATE;
  } catch (const TimeoutError& e) {
    g_last_error = e.what();
    return HYKKT_ERR_DEVICE_TIMEOUT;
  } catch (const std::bad_alloc&) {
    g_last_error = "out of host memory";
    return HYKKT_ERR_CUDA;
  } catch (const std::exception& e) {
    g_last_error = e.what();
    return HYKKT_ERR_INVALID;
  }
}

Ctx& ctx(hykkt_t h) {
  if (!h) throw InvalidArgument("null handle");
  CK(cudaSetDevice(h->device));
  return *h;
}

}  // namespace
}  // namespace hykkt

using namespace hykkt;

extern "C" {

void hykkt_config_default(hykkt_config_t* cfg) {
  if (!cfg) return;
  cfg->gamma = 1e4;
  cfg->delta_min = 1e-9;
  cfg->delta_max = 1e-6;
  cfg->delta2 = 1e-9;
  cfg->cg_tol = 1e-12;
  cfg->cg_max_iter = 500;
  cfg->small_quadratic_threshold = 1e-12;
  cfg->pivot_floor = 1e-13;
  cfg->ruiz_tol = 0.01;
  cfg->ruiz_max_iters = 20;
}

const char* hykkt_last_error(void) { return g_last_error.c_str(); }

int hykkt_create(int device, hykkt_t* out) {
  return guarded([&] {
    if (!out) throw InvalidArgument("null output handle");
    auto c = std::make_unique<hykkt_context>();
    init_ctx(*c, device);
    *out = c.release();
  });
}

void hykkt_destroy(hykkt_t h) {
  if (!h) return;
  cudaSetDevice(h->device);
  if (h->copy_stream) {
    cudaStreamSynchronize(h->copy_stream);
    cudaStreamDestroy(h->copy_stream);
    for (int i = 0; i < 2; ++i) {
      cudaEventDestroy(h->stage_ready[i]);
      cudaEventDestroy(h->stage_free[i]);
    }
    cudaEventDestroy(h->out_ready);
    cudaEventDestroy(h->out_free);
  }
  if (h->stream) {
    cudaStreamSynchronize(h->stream);
    cudaStreamDestroy(h->stream);
  }
  delete h;
}

int hykkt_analyze(hykkt_t h, int64_t n_x, int64_t m_c, int64_t m_d, const int64_t* h_colptr,
                  const int64_t* h_rowidx, const int64_t* j_colptr, const int64_t* j_rowidx,
                  const int64_t* jd_colptr, const int64_t* jd_rowidx, const int64_t* perm) {
  return guarded([&] {
    Ctx& c = ctx(h);
    analyze_kkt(c, n_x, m_c, m_d, h_colptr, h_rowidx, j_colptr, j_rowidx, jd_colptr, jd_rowidx, perm);
  });
}

static hykkt_analysis_t stats_of(const SupernodalPlan& s, const KktPlan* kp) {
    hykkt_analysis_t a{};
    a.n = s.n;
    a.nnz_h_tilde = kp ? kp->ht.nnz() : 0;
    a.nnz_h_gamma = kp ? kp->hg.nnz() : 0;
    a.nnz_l = s.l_nnz();
    a.n_supernodes = s.nsup;
    a.n_levels = s.nlevels;
    idx height = 0;
    std::vector<idx> depth(s.n, 0);
    for (idx j = s.n - 1; j >= 0; --j) {
      depth[j] = s.parent[j] < 0 ? 1 : depth[s.parent[j]] + 1;
      height = std::max(height, depth[j]);
    }
    a.etree_height = height;
    a.max_sn_width = s.max_width;
    a.max_sn_rows = s.max_nrows;
    a.panel_slots = s.panel_size;
    a.factor_flops = s.factor_flops;
    a.nnz_j = kp ? kp->j.nnz() : 0;
    a.nnz_jd = kp ? kp->jd.nnz() : 0;
    a.m_c = kp ? kp->mc : 0;
    a.m_d = kp ? kp->md : 0;
    a.explicit_zeros = s.explicit_zeros;
    return a;
}

int hykkt_analysis_info(hykkt_t h, hykkt_analysis_t* out) {
  return guarded([&] {
    Ctx& c = ctx(h);
    if (!c.have_plan) throw StateError("no analysis");
    if (!out) throw InvalidArgument("null output");
    *out = stats_of(c.sp, c.have_kkt ? &c.kp : nullptr);
  });
}

int hykkt_host_analyze(int64_t n_x, int64_t m_c, int64_t m_d, const int64_t* h_colptr,
                       const int64_t* h_rowidx, const int64_t* j_colptr, const int64_t* j_rowidx,
                       const int64_t* jd_colptr, const int64_t* jd_rowidx, const int64_t* perm,
                       int64_t* perm_out, hykkt_analysis_t* out) {
  return guarded([&] {
    if (n_x < 0 || m_c < 0 || m_d < 0) throw InvalidArgument("negative dimension");
    KktPlan kp = build_kkt_plan(n_x, m_c, m_d, pattern_from(n_x, n_x, h_colptr, h_rowidx),
                                pattern_from(m_c, n_x, j_colptr, j_rowidx),
                                pattern_from(m_d, n_x, jd_colptr, jd_rowidx));
    std::vector<idx> pv;
    if (perm) pv.assign(perm, perm + n_x);
    const SupernodalPlan sp = build_supernodal_plan(kp.hg, std::move(pv));
    if (perm_out) std::copy(sp.perm.begin(), sp.perm.end(), perm_out);
    if (out) *out = stats_of(sp, &kp);
  });
}

// Diagnostics (host only): per-supernode work of the analysed plan,
// 8 doubles per supernode: width, rows, level, descendant updates,
// left-looking update FMAs (sum over updates of m * cnt * wd, lower half),
// dense panel FMAs (w^2 nr / 2), forward row-gather entries (sum over
// updates of cnt * wd), supernode parent.  Returns the supernode count.
int hykkt_debug_host_sn_stats(int64_t n_x, int64_t m_c, int64_t m_d, const int64_t* h_colptr,
                              const int64_t* h_rowidx, const int64_t* j_colptr, const int64_t* j_rowidx,
                              const int64_t* jd_colptr, const int64_t* jd_rowidx, const int64_t* perm,
                              int64_t* nsup, double* out) {
  return guarded([&] {
    KktPlan kp = build_kkt_plan(n_x, m_c, m_d, pattern_from(n_x, n_x, h_colptr, h_rowidx),
                                pattern_from(m_c, n_x, j_colptr, j_rowidx),
                                pattern_from(m_d, n_x, jd_colptr, jd_rowidx));
    std::vector<idx> pv;
    if (perm) pv.assign(perm, perm + n_x);
    const SupernodalPlan sp = build_supernodal_plan(kp.hg, std::move(pv));
    *nsup = sp.nsup;
    for (idx k = 0; k < sp.nsup; ++k) {
      const double w = sp.sn_first[k + 1] - sp.sn_first[k], nr = sp.sn_nrows[k];
      double uf = 0.0, ge = 0.0;
      for (int u = sp.upd_ptr[k]; u < sp.upd_ptr[k + 1]; ++u) {
        const int d = sp.upd_d[u];
        const double m = sp.sn_nrows[d] - sp.upd_off[u], cnt = sp.upd_cnt[u];
        const double wd = sp.sn_first[d + 1] - sp.sn_first[d];
        uf += (m * cnt - cnt * (cnt - 1) / 2.0) * wd;
        ge += cnt * wd;
      }
      double* o = out + 8 * k;
      o[6] = ge;
      o[7] = sp.sn_parent[k];
      o[0] = w;
      o[1] = nr;
      o[2] = sp.sn_level[k];
      o[3] = sp.upd_ptr[k + 1] - sp.upd_ptr[k];
      o[4] = uf;
      o[5] = w * w * nr / 2.0;
    }
  });
}

// Diagnostics (host only): builds the system-per-CTA stream program for the
// KKT pattern with rings of nchunk x 1024 entries and runs its host
// emulation (sys_plan_selfcheck).  out[0] = max relative error vs a plain
// J^T / supernodal solve / J reference, out[1] = value stream entries,
// out[2] = index stream entries, out[3] = steps, out[4] = tasks,
// out[5] = segments, out[6] = max segments per step, out[7] = non-padding
// value entries.
int hykkt_debug_sysplan_check(int64_t n_x, int64_t m_c, int64_t m_d, const int64_t* h_colptr,
                              const int64_t* h_rowidx, const int64_t* j_colptr, const int64_t* j_rowidx,
                              const int64_t* jd_colptr, const int64_t* jd_rowidx, const int64_t* perm,
                              int nchunk, double* out) {
  return guarded([&] {
    KktPlan kp = build_kkt_plan(n_x, m_c, m_d, pattern_from(n_x, n_x, h_colptr, h_rowidx),
                                pattern_from(m_c, n_x, j_colptr, j_rowidx),
                                pattern_from(m_d, n_x, jd_colptr, jd_rowidx));
    std::vector<idx> pv;
    if (perm) pv.assign(perm, perm + n_x);
    const SupernodalPlan sp = build_supernodal_plan(kp.hg, std::move(pv));
    const SysPlan P = build_sys_plan(sp, kp, ks_chunk_lg(), nchunk, ks_chunk_lg(), nchunk, kKsPmax, kKsThreads - 32);
    out[0] = sys_plan_selfcheck(sp, kp, P, 12345u);
    out[1] = static_cast<double>(P.src.size());
    out[2] = static_cast<double>(P.idx.size());
    out[3] = P.nsteps;
    out[4] = static_cast<double>(P.ntasks);
    out[5] = static_cast<double>(P.nsegs);
    out[6] = P.max_segs_per_step;
    out[7] = static_cast<double>(P.value_entries);
  });
}

// Diagnostics: per-CTA phase timers of the last system-per-CTA batched solve
// (HYKKT_KS_PROF=1): 16 counters per CTA (kernels_sys.cuh KsProf), and
// (trace, nsteps + 1 entries) CTA 0's end time of each substep of its first
// solve, start time last.  Returns the CTA count in *nctas (0 = off).
int hykkt_debug_ks_prof(hykkt_t h, uint64_t* out, int64_t* nctas, uint64_t* trace) {
  return guarded([&] {
    Ctx& c = ctx(h);
    *nctas = c.ks.prof_on == 1 ? c.ks.prof_ctas : 0;
    if (*nctas && out) {
      CK(cudaMemcpy(out, c.ks.prof.p, static_cast<std::size_t>(*nctas) * dev::kPrN * 8, cudaMemcpyDeviceToHost));
    }
    if (*nctas && trace) {
      CK(cudaMemcpy(trace, c.ks.trace.p, c.ks.trace.n * 8, cudaMemcpyDeviceToHost));
    }
  });
}

// Diagnostics: the system-per-CTA program's steps, 8 ints each (kind, index
// length, value length, header words 3-6, widest task); returns the count.
int hykkt_debug_ks_program(hykkt_t h, int32_t* steps, int64_t* nsteps) {
  return guarded([&] {
    Ctx& c = ctx(h);
    if (!ks_prepare(c)) throw StateError("system-per-CTA path unavailable: " + c.ks.why);
    const SysPlan& P = c.ks.plan;
    *nsteps = P.nsteps;
    if (!steps) return;
    int k = 0;
    for (int b = 0; b < 4; ++b) {
      long long ib = P.blk[b].i0;
      for (int s = P.blk[b].s0; s < P.blk[b].s1; ++s, ++k) {
        const int* hd = P.idx.data() + ib;
        int maxw = 0;
        if (hd[0] <= HYKKT_STEP_BWD) {
          const int dt = HYKKT_SP_HDR + HYKKT_SP_SEG_INTS * hd[3];
          for (int t = 0; t < hd[4] + hd[5]; ++t) maxw = std::max(maxw, hd[dt + HYKKT_SP_TASK_INTS * t + 3] & 0xffff);
        }
        const int v8[8] = {hd[0], hd[1], hd[2], hd[3], hd[4], hd[5], hd[6], maxw};
        std::copy(v8, v8 + 8, steps + 8 * k);
        ib += hd[1];
      }
    }
  });
}

int hykkt_get_perm(hykkt_t h, int64_t* perm) {
  return guarded([&] {
    Ctx& c = ctx(h);
    if (!c.have_plan) throw StateError("no analysis");
    if (!perm) throw InvalidArgument("null output");
    std::copy(c.sp.perm.begin(), c.sp.perm.end(), perm);
  });
}

int hykkt_upload_values(hykkt_t h, const hykkt_values_t* values) {
  return guarded([&] { upload_values(ctx(h), values); });
}

int hykkt_solve_resident(hykkt_t h, const hykkt_config_t* cfg, double* delta_min_inout, int flags,
                         hykkt_report_t* report) {
  return guarded([&] {
    hykkt_config_t d;
    hykkt_config_default(&d);
    solve_resident(ctx(h), cfg ? *cfg : d, delta_min_inout, flags, report);
  });
}

int hykkt_download_solution(hykkt_t h, double* dx, double* ds, double* dy, double* dyd) {
  return guarded([&] {
    Ctx& c = ctx(h);
    if (!c.have_kkt) throw StateError("no analysis");
    download_solution(c, dx, ds, dy, dyd);
  });
}

int hykkt_solve_full(hykkt_t h, const hykkt_config_t* cfg, const hykkt_values_t* values,
                     double* delta_min_inout, int flags, hykkt_report_t* report, double* dx, double* ds,
                     double* dy, double* dyd) {
  return guarded([&] {
    Ctx& c = ctx(h);
    hykkt_config_t d;
    hykkt_config_default(&d);
    upload_values(c, values);
    hykkt_report_t r{};
    solve_resident(c, cfg ? *cfg : d, delta_min_inout, flags, &r);
    if (r.status <= 1) download_solution(c, dx, ds, dy, dyd);
    if (report) *report = r;
  });
}

int hykkt_last_timing(hykkt_t h, hykkt_timing_t* out) {
  return guarded([&] {
    Ctx& c = ctx(h);
    if (!out) throw InvalidArgument("null output");
    *out = c.timing;
  });
}

// ---- Cholesky-level hooks ---------------------------------------------------
int hykkt_chol_analyze(hykkt_t h, int64_t n, const int64_t* colptr, const int64_t* rowidx,
                       const int64_t* perm) {
  return guarded([&] {
    Ctx& c = ctx(h);
    if (n < 0) throw InvalidArgument("negative dimension");
    CscPattern a = pattern_from(n, n, colptr, rowidx);
    std::vector<idx> pv;
    if (perm) pv.assign(perm, perm + n);
    c.have_kkt = false;
    c.have_values = false;
    c.have_assembled = false;
    c.reduced = false;
    c.have_j = false;
    c.kp = KktPlan{};
    c.kp.hg = a;  // source pattern for scatter bookkeeping
    c.sp = build_supernodal_plan(a, std::move(pv), c.amalg);
    upload_plan(c, a);
    c.src_vals.alloc(a.nnz());
    CK(cudaStreamSynchronize(c.stream));
  });
}

int hykkt_chol_factor(hykkt_t h, const double* values, double pivot_floor, int64_t* failed_column,
                      double* failed_pivot) {
  return guarded([&] {
    Ctx& c = ctx(h);
    if (!c.have_plan) throw StateError("hykkt_chol_analyze must be called first");
    const idx nnz = static_cast<idx>(c.sp.src_to_panel.size());
    if (nnz > 0 && !values) throw InvalidArgument("null values");
    if (c.src_vals.n < static_cast<std::size_t>(nnz)) c.src_vals.alloc(nnz);
    if (nnz) CK(cudaMemcpyAsync(c.src_vals.p, values, nnz * sizeof(double), cudaMemcpyHostToDevice, c.stream));
    const int fc = factor_attempt(c, c.src_vals.p, 0.0, pivot_floor, nullptr, 0.0);
    if (failed_column) *failed_column = fc;
    if (fc >= 0) {
      double piv = 0.0;
      CK(cudaMemcpy(&piv, c.panel.p + c.sp.diag_panel[fc], sizeof(double), cudaMemcpyDeviceToHost));
      if (failed_pivot) *failed_pivot = piv;
      c.have_factor = false;
    } else {
      if (failed_pivot) *failed_pivot = 0.0;
      c.have_factor = true;
    }
  });
}

int hykkt_chol_solve(hykkt_t h, const double* b, double* x) {
  return guarded([&] {
    Ctx& c = ctx(h);
    if (!c.have_factor) throw StateError("no successful factorization");
    const idx n = c.sp.n;
    if (n == 0) return;
    if (!b || !x) throw InvalidArgument("null vector");
    CK(cudaMemcpyAsync(c.bvec.p, b, n * sizeof(double), cudaMemcpyDefault, c.stream));
    CK(cudaMemsetAsync(&c.status.p->abort, 0, sizeof(int), c.stream));
    run_trsv(c, c.bvec.p, nullptr, nullptr, c.xvec.p);
    CK(cudaMemcpyAsync(x, c.xvec.p, n * sizeof(double), cudaMemcpyDefault, c.stream));
    read_status(c);
  });
}

int hykkt_chol_get_factor(hykkt_t h, int64_t* l_colptr, int64_t* l_rowidx, double* l_values,
                          int64_t* parent) {
  return guarded([&] {
    Ctx& c = ctx(h);
    if (!c.have_plan) throw StateError("no analysis");
    const SupernodalPlan& s = c.sp;
    if (l_colptr) std::copy(s.l_cp.begin(), s.l_cp.end(), l_colptr);
    if (l_rowidx) std::copy(s.l_ri.begin(), s.l_ri.end(), l_rowidx);
    if (parent) std::copy(s.parent.begin(), s.parent.end(), parent);
    if (l_values) {
      if (!c.have_factor) throw StateError("no successful factorization");
      std::vector<double> pan(s.panel_size);
      if (s.panel_size) CK(cudaMemcpy(pan.data(), c.panel.p, s.panel_size * sizeof(double), cudaMemcpyDeviceToHost));
      for (std::size_t q = 0; q < s.l_to_panel.size(); ++q) l_values[q] = pan[s.l_to_panel[q]];
    }
  });
}

// Diagnostics: one traced batched H^-1 pass over the last batch (needs a
// solved batch); out[j] / out[njobs + j] = end / start ns of CTA job j.
// With out == NULL, *njobs_out receives the job count only.
int hykkt_debug_btrsv_trace(hykkt_t h, uint64_t* out, int64_t* njobs_out) {
  return guarded([&] {
    Ctx& c = ctx(h);
    auto& bb = c.bb;
    if (bb.jobs_T < 0) throw StateError("no batch schedule");
    if (njobs_out) *njobs_out = bb.njobs;
    if (!out) return;
    const int T = bb.Bp / 32;
    hykkt::DBuf<unsigned long long> tr;
    tr.alloc(2 * static_cast<std::size_t>(bb.njobs));
    CK(cudaMemsetAsync(tr.p, 0, tr.n * sizeof(unsigned long long), c.stream));
    dev::BTrsvArgs ta;
    ta.s = c.snplan();
    ta.bd = dev::BDims{static_cast<int>(c.batch), bb.Bp, T};
    ta.panel = bb.panel.p;
    ta.y = bb.y.p;
    ta.x = bb.xs.p;
    ta.u = bb.u.p;
    ta.acc = bb.acc.p;
    ta.x_out = nullptr;
    ta.bar = dev::GridBarrier{c.barrier.p, c.barrier.p + 1};
    ta.smem_rows = batch_smem_rows();
    ta.fdone = bb.fdone.p;
    ta.bdone = bb.bdone.p;
    ta.epoch = ++c.epoch;
    ta.abort = &c.status.p->abort;
    ta.rb = bb.rhat.p;
    ta.ru = nullptr;
    ta.j_cp = c.j_cp.p;
    ta.j_ri = c.j_ri.p;
    ta.jval = bb.js.p;
    ta.lane_on = nullptr;
    ta.job_ptr = bb.job_ptr.p;
    ta.job_items = bb.job_items.p;
    ta.job_kind = bb.job_kind.p;
    ta.njobs = bb.njobs;
    ta.mode = bb.mode.p;
    ta.smem_doubles = static_cast<int>(kBatchSmem / sizeof(double));
    ta.trace = tr.p;
    ta.ticket = fresh_tickets(c, 1);
    coop_launch(c, (const void*)dev::kb_trsv, c.coop_btrsv_blocks, &ta, kBatchSmem);
    read_status(c);
    CK(cudaMemcpy(out, tr.p, tr.n * sizeof(unsigned long long), cudaMemcpyDeviceToHost));
  });
}

// Diagnostics: the batched solve schedule: job_ptr (njobs + 1), items,
// kind (njobs) and the supernode mode (nsup).  Any pointer may be NULL.
int hykkt_debug_batch_jobs(hykkt_t h, int32_t* job_ptr, int32_t* items, uint8_t* kind, int32_t* mode) {
  return guarded([&] {
    Ctx& c = ctx(h);
    auto& bb = c.bb;
    if (bb.jobs_T < 0) throw StateError("no batch schedule");
    if (job_ptr) CK(cudaMemcpy(job_ptr, bb.job_ptr.p, (bb.njobs + 1) * sizeof(int), cudaMemcpyDeviceToHost));
    int nitems = 0;
    CK(cudaMemcpy(&nitems, bb.job_ptr.p + bb.njobs, sizeof(int), cudaMemcpyDeviceToHost));
    if (items) CK(cudaMemcpy(items, bb.job_items.p, nitems * sizeof(int), cudaMemcpyDeviceToHost));
    if (kind) CK(cudaMemcpy(kind, bb.job_kind.p, bb.njobs, cudaMemcpyDeviceToHost));
    if (mode) CK(cudaMemcpy(mode, bb.mode.p, c.sp.nsup * sizeof(int), cudaMemcpyDeviceToHost));
  });
}

// Diagnostics: supernode structure (order, first column, rows, parent).
int hykkt_debug_plan(hykkt_t h, int32_t* order, int32_t* first, int32_t* nrows, int32_t* parent) {
  return guarded([&] {
    Ctx& c = ctx(h);
    if (!c.have_plan) throw StateError("no analysis");
    const SupernodalPlan& s = c.sp;
    std::copy(s.order.begin(), s.order.end(), order);
    std::copy(s.sn_first.begin(), s.sn_first.end(), first);
    std::copy(s.sn_nrows.begin(), s.sn_nrows.end(), nrows);
    std::copy(s.sn_parent.begin(), s.sn_parent.end(), parent);
  });
}

// Diagnostics: one traced H^-1 pass (b = r_hat_x of the last KKT solve);
// out[t] / out[2 nsup + t] = end / start time (ns) of task t (t < nsup:
// forward task of order[t]; else backward task of order[2 nsup - 1 - t]).
// Diagnostics: one k_trsv pass on r_hat (w solve); copies the permuted
// forward (y) and backward (x) results to the host.
int hykkt_debug_trsv_vectors(hykkt_t h, double* y, double* x) {
  return guarded([&] {
    Ctx& c = ctx(h);
    if (!c.have_factor || !c.have_kkt) throw StateError("needs a factored KKT system");
    run_trsv(c, c.rhat.p, nullptr, c.js.p, nullptr);
    read_status(c);
    CK(cudaMemcpy(y, c.y.p, c.sp.n * sizeof(double), cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(x, c.xsol.p, c.sp.n * sizeof(double), cudaMemcpyDeviceToHost));
  });
}

// Diagnostics: one k_trsv pass (w solve) with per-CTA phase stamps
// (8 per CTA: start, after rearm barrier, after the forward bottom levels,
// task loop exit, after the backward bottom barrier, after backward bottom /
// levels, -, end).  Returns the grid size in *nblk.
int hykkt_debug_trsv_phases(hykkt_t h, uint64_t* out, int64_t cap, int64_t* nblk) {
  return guarded([&] {
    Ctx& c = ctx(h);
    if (!c.have_factor || !c.have_kkt) throw StateError("needs a factored KKT system");
    *nblk = c.trsv_grid;
    if (cap < 8 * c.trsv_grid) return;
    hykkt::DBuf<unsigned long long> st;
    st.alloc(8 * c.trsv_grid);
    CK(cudaMemset(st.p, 0, 8 * c.trsv_grid * sizeof(unsigned long long)));
    ensure_qform(c);
      dev::TrsvArgs ta = trsv_args(c);
    ta.rhs.b = c.rhat.p;
    ta.pstamp = st.p;
    ta.ticket = fresh_tickets(c, ta.tstride);
    coop_launch(c, c.tr_call ? (const void*)dev::k_trsv<true> : (const void*)dev::k_trsv<false>, c.trsv_grid,
                &ta);
    read_status(c);
    CK(cudaMemcpy(out, st.p, 8 * c.trsv_grid * sizeof(unsigned long long), cudaMemcpyDeviceToHost));
  });
}

// Diagnostics: per-CTA phase times of the last CG iteration of one k_cg run
// on the current factor and Schur right-hand side (after a solve): 8 per
// CTA for the pass (as hykkt_debug_trsv_phases), then 8 per CTA for the CG
// phases (iteration start, pass end, after barrier, J product end, after
// barrier, x / r end, after barrier).
int hykkt_debug_cg_phases(hykkt_t h, const hykkt_config_t* cfg, uint64_t* out, int64_t cap, int64_t* nblk) {
  return guarded([&] {
    Ctx& c = ctx(h);
    if (!c.have_factor || !c.have_kkt) throw StateError("needs a factored KKT system");
    *nblk = c.cg_grid;
    if (cap < 16 * c.cg_grid) return;
    hykkt::DBuf<unsigned long long> st;
    st.alloc(16 * c.cg_grid);
    CK(cudaMemset(st.p, 0, 16 * c.cg_grid * sizeof(unsigned long long)));
    c.cg_stamps = st.p;
    try {
      run_cg(c, *cfg, 0.0);
    } catch (...) {
      c.cg_stamps = nullptr;
      throw;
    }
    c.cg_stamps = nullptr;
    CK(cudaMemcpy(out, st.p, 16 * c.cg_grid * sizeof(unsigned long long), cudaMemcpyDeviceToHost));
  });
}

// Diagnostics: the cluster solve's per-level end times of the last pass
// (HYKKT_CL_STAMPS=1 at analysis), 2 * levels values (forward levels, then
// backward), and the level lists' sizes (4 per level: thread, warp, CTA, 0).
int hykkt_debug_cluster_stamps(hykkt_t h, uint64_t* out, int* sizes, int64_t cap, int64_t* nlev) {
  return guarded([&] {
    Ctx& c = ctx(h);
    *nlev = c.cl_nlev;
    if (c.cl_nlev == 0 || cap < 2 * c.cl_nlev) return;
    CK(cudaStreamSynchronize(c.stream));
    if (cap < 2 * c.cl_nlev + 768) return;
    CK(cudaMemcpy(out, c.cl_stamps.p, (2 * c.cl_nlev + 768) * sizeof(unsigned long long), cudaMemcpyDeviceToHost));
    std::vector<int> lp(4 * c.cl_nlev);
    CK(cudaMemcpy(lp.data(), c.cl_lv_ptr.p, lp.size() * sizeof(int), cudaMemcpyDeviceToHost));
    for (int l = 0; l < c.cl_nlev; ++l) {
      sizes[4 * l] = lp[4 * l + 1] - lp[4 * l];
      sizes[4 * l + 1] = lp[4 * l + 2] - lp[4 * l + 1];
      sizes[4 * l + 2] = lp[4 * l + 3] - (l ? lp[4 * l - 1] : 0);
      sizes[4 * l + 3] = 0;
    }
  });
}

int hykkt_debug_trsv_trace(hykkt_t h, uint64_t* out) {
  return guarded([&] {
    Ctx& c = ctx(h);
    if (!c.have_factor || !c.have_kkt) throw StateError("needs a factored KKT system");
    const idx ns = c.sp.nsup;
    hykkt::DBuf<unsigned long long> tr;
    tr.alloc(6 * ns);
    ensure_qform(c);
      dev::TrsvArgs ta = trsv_args(c);
    ta.rhs.b = c.rhat.p;
    ta.trace = tr.p;
    ta.ticket = fresh_tickets(c, ta.tstride);
    coop_launch(c, c.tr_call ? (const void*)dev::k_trsv<true> : (const void*)dev::k_trsv<false>, c.trsv_grid,
                &ta);
    read_status(c);
    CK(cudaMemcpy(out, tr.p, 6 * ns * sizeof(unsigned long long), cudaMemcpyDeviceToHost));
  });
}

}  // extern "C"

extern "C" {

int hykkt_batch_upload(hykkt_t h, int64_t batch, const hykkt_values_t* values) {
  return guarded([&] { batch_upload(ctx(h), batch, values); });
}

int hykkt_batch_solve_resident(hykkt_t h, const hykkt_config_t* cfg, int flags, hykkt_report_t* reports) {
  return guarded([&] {
    hykkt_config_t d;
    hykkt_config_default(&d);
    batch_solve_resident(ctx(h), cfg ? *cfg : d, flags, reports);
  });
}

int hykkt_batch_download(hykkt_t h, double* dx, double* ds, double* dy, double* dyd) {
  return guarded([&] { batch_download(ctx(h), dx, ds, dy, dyd); });
}

int hykkt_batch_upload_async(hykkt_t h, int64_t batch, const hykkt_values_t* values) {
  return guarded([&] { batch_upload_async(ctx(h), batch, values); });
}

int hykkt_batch_download_async(hykkt_t h, double* dx, double* ds, double* dy, double* dyd) {
  return guarded([&] { batch_download_async(ctx(h), dx, ds, dy, dyd); });
}

int hykkt_batch_sync(hykkt_t h) {
  return guarded([&] { batch_sync(ctx(h)); });
}

int hykkt_batch_solve(hykkt_t h, const hykkt_config_t* cfg, int64_t batch, const hykkt_values_t* values,
                      int flags, hykkt_report_t* reports, double* dx, double* ds, double* dy, double* dyd) {
  return guarded([&] {
    Ctx& c = ctx(h);
    hykkt_config_t d;
    hykkt_config_default(&d);
    batch_upload(c, batch, values);
    batch_solve_resident(c, cfg ? *cfg : d, flags, reports);
    batch_download(c, dx, ds, dy, dyd);
  });
}

}  // extern "C"

// ---- the split reference API (solver.hpp:75, :92-94, :121-122, :167-170) ----
namespace hykkt {
namespace {

void require_factor(const Ctx& c) {
  if (!c.have_factor) throw StateError("no successful factorization on this handle");
}

// Reference-layout L values (SymbolicFactor::l_col_ptr order) into the
// supernodal panels: the inverse of hykkt_chol_get_factor.
void set_factor(Ctx& c, const double* l_values) {
  if (!c.have_plan) throw StateError("no analysis");
  const SupernodalPlan& s = c.sp;
  if (!l_values && !s.l_to_panel.empty()) throw InvalidArgument("null l_values");
  std::vector<double> pan(std::max<idx>(1, s.panel_size), 0.0);
  for (std::size_t q = 0; q < s.l_to_panel.size(); ++q) pan[s.l_to_panel[q]] = l_values[q];
  CK(cudaMemcpyAsync(c.panel.p, pan.data(), s.panel_size * sizeof(double), cudaMemcpyHostToDevice, c.stream));
  c.panel_ver++;
  CK(cudaStreamSynchronize(c.stream));
  c.have_factor = true;
}

// J (m_c x n, CSC) for hykkt_cg_schur on a Cholesky-level handle: CSC for the
// J^T gathers of the forward solve, CSR (ascending columns, the reference's
// spmv scatter order, csc_matrix.cpp:250-254) for J t.
void chol_set_j(Ctx& c, idx mc, const std::int64_t* cp, const std::int64_t* ri, const double* val) {
  if (!c.have_plan || c.have_kkt) throw StateError("hykkt_chol_set_j needs a Cholesky-level handle");
  if (mc < 0) throw InvalidArgument("negative m_c");
  const idx n = c.sp.n;
  CscPattern j = pattern_from(mc, n, cp, ri);
  const idx nnz = j.nnz();
  if (nnz > 0 && !val) throw InvalidArgument("null J values");
  for (idx q = 0; q < nnz; ++q) {
    if (j.ri[q] < 0 || j.ri[q] >= mc) throw InvalidArgument("J row index out of range");
  }
  std::vector<int> rp(mc + 1, 0), ci(std::max<idx>(nnz, 1)), cip(std::max<idx>(nnz, 1));
  std::vector<double> vcsr(std::max<idx>(nnz, 1));
  for (idx q = 0; q < nnz; ++q) rp[j.ri[q] + 1]++;
  std::partial_sum(rp.begin(), rp.end(), rp.begin());
  std::vector<int> cur(rp.begin(), rp.end() - 1);
  for (idx col = 0; col < n; ++col) {
    for (idx q = j.cp[col]; q < j.cp[col + 1]; ++q) {
      const int e = cur[j.ri[q]]++;
      cip[e] = static_cast<int>(c.sp.iperm[col]);
      vcsr[e] = val[q];
    }
  }
  cudaStream_t st = c.stream;
  c.kp.mc = mc;
  c.j_cp.upload(to_i32(j.cp), st);
  c.j_ri.upload(to_i32(j.ri), st);
  c.js.alloc(std::max<idx>(nnz, 1));
  if (nnz) CK(cudaMemcpyAsync(c.js.p, val, nnz * sizeof(double), cudaMemcpyHostToDevice, st));
  c.jcsr_rp.upload(rp, st);
  c.jcsr_ci_perm.upload(cip, st);
  c.js_csr.upload(vcsr, st);
  c.cg_rhs.alloc(std::max<idx>(mc, 1));
  c.cg_x.alloc(std::max<idx>(mc, 1));
  c.cg_r.alloc(std::max<idx>(mc, 1));
  c.cg_p.alloc(std::max<idx>(mc, 1));
  c.cg_q.alloc(std::max<idx>(mc, 1));
  c.partials.alloc(4 * static_cast<std::size_t>(std::max(c.coop_cg_blocks, 1)));
  CK(cudaStreamSynchronize(st));
  c.have_j = true;
}

}  // namespace
}  // namespace hykkt

extern "C" {

int hykkt_analyze_reduced(hykkt_t h, int64_t n_x, int64_t m_c, const int64_t* ht_colptr,
                          const int64_t* ht_rowidx, const int64_t* j_colptr, const int64_t* j_rowidx,
                          const int64_t* perm) {
  return guarded([&] {
    Ctx& c = ctx(h);
    if (n_x < 0) throw InvalidArgument("negative dimension");
    const std::vector<int64_t> jd_cp(static_cast<std::size_t>(n_x) + 1, 0);
    analyze_kkt(c, n_x, m_c, 0, ht_colptr, ht_rowidx, j_colptr, j_rowidx, jd_cp.data(), nullptr, perm);
    c.reduced = true;
  });
}

int hykkt_upload_reduced(hykkt_t h, const double* ht_val, const double* j_val, const double* r_x,
                         const double* r_y) {
  return guarded([&] { upload_reduced(ctx(h), ht_val, j_val, r_x, r_y); });
}

int hykkt_upload_reduced_device(hykkt_t h, const double* ht_val, const double* j_val, const double* r_x,
                                const double* r_y) {
  return guarded([&] { upload_reduced(ctx(h), ht_val, j_val, r_x, r_y, true); });
}

int hykkt_solve_reduced(hykkt_t h, const hykkt_config_t* cfg, const double* ht_val, const double* j_val,
                        const double* r_x, const double* r_y, double* delta_min_inout, int flags,
                        hykkt_report_t* report, double* dx, double* dy) {
  return guarded([&] {
    Ctx& c = ctx(h);
    hykkt_config_t d;
    hykkt_config_default(&d);
    upload_reduced(c, ht_val, j_val, r_x, r_y);
    hykkt_report_t r{};
    solve_resident(c, cfg ? *cfg : d, delta_min_inout, flags, &r);
    if (r.status <= 1) download_solution(c, dx, nullptr, dy, nullptr);
    if (report) *report = r;
  });
}

int hykkt_upload_values_device(hykkt_t h, const hykkt_values_t* values) {
  return guarded([&] { upload_values(ctx(h), values, true); });
}

int hykkt_batch_upload_device(hykkt_t h, int64_t batch, const hykkt_values_t* values) {
  return guarded([&] { batch_upload(ctx(h), batch, values, true); });
}

int hykkt_solution_device(hykkt_t h, const double** dx, const double** ds, const double** dy,
                          const double** dyd) {
  return guarded([&] {
    Ctx& c = ctx(h);
    if (!c.have_kkt) throw StateError("no analysis");
    if (dx) *dx = c.o.dx;
    if (ds) *ds = c.o.ds;
    if (dy) *dy = c.o.dy;
    if (dyd) *dyd = c.o.dyd;
  });
}

int hykkt_batch_solution_device(hykkt_t h, const double** dx, const double** ds, const double** dy,
                                const double** dyd) {
  return guarded([&] {
    Ctx& c = ctx(h);
    if (c.batch <= 0) throw StateError("no batch uploaded");
    const KktPlan& k = c.kp;
    const idx B = c.batch;
    const double* o = c.bouts.p;
    if (dx) *dx = o;
    if (dy) *dy = o + B * k.nx;
    if (ds) *ds = o + B * (k.nx + k.mc);
    if (dyd) *dyd = o + B * (k.nx + k.mc + k.md);
  });
}

int hykkt_assemble(hykkt_t h, const hykkt_config_t* cfg, double* hg_val, double* r_hat_x) {
  return guarded([&] {
    Ctx& c = ctx(h);
    if (!c.have_kkt) throw StateError("hykkt_analyze / hykkt_analyze_reduced must be called first");
    hykkt_config_t d;
    hykkt_config_default(&d);
    const hykkt_config_t& cf = cfg ? *cfg : d;
    validate_cfg(cf);
    assemble_phase(c, cf);
    if (hg_val && c.kp.hg.nnz())
      CK(cudaMemcpyAsync(hg_val, c.hg.p, c.kp.hg.nnz() * sizeof(double), cudaMemcpyDefault, c.stream));
    if (r_hat_x && c.kp.nx)
      CK(cudaMemcpyAsync(r_hat_x, c.rhat.p, c.kp.nx * sizeof(double), cudaMemcpyDefault, c.stream));
    read_status(c);
  });
}

int hykkt_hgamma_pattern(hykkt_t h, int64_t* colptr, int64_t* rowidx) {
  return guarded([&] {
    Ctx& c = ctx(h);
    if (!c.have_kkt) throw StateError("no KKT analysis");
    if (colptr) std::copy(c.kp.hg.cp.begin(), c.kp.hg.cp.end(), colptr);
    if (rowidx) std::copy(c.kp.hg.ri.begin(), c.kp.hg.ri.end(), rowidx);
  });
}

int hykkt_factor_ladder(hykkt_t h, const hykkt_config_t* cfg, const double* values, double* delta_min_inout,
                        int64_t* attempts, double* delta1, int64_t* failed_column) {
  return guarded([&] {
    Ctx& c = ctx(h);
    if (!c.have_plan) throw StateError("no analysis");
    hykkt_config_t d;
    hykkt_config_default(&d);
    const hykkt_config_t& cf = cfg ? *cfg : d;
    validate_cfg(cf);
    LadderOut lo;
    if (c.have_kkt) {
      if (values) throw InvalidArgument("KKT handle: the ladder runs on the assembled H_gamma (values must be NULL)");
      if (!c.have_assembled) throw StateError("hykkt_assemble must be called first");
      lo = ladder_phase(c, cf, c.hg.p, c.maxdiag.p, delta_min_inout);
    } else {
      const idx nnz = static_cast<idx>(c.sp.src_to_panel.size());
      if (c.src_vals.n < static_cast<std::size_t>(std::max<idx>(nnz, 1))) c.src_vals.alloc(std::max<idx>(nnz, 1));
      copy_in(c.src_vals.p, values, nnz, "values", c.stream, false);
      c.maxdiag.alloc(1);
      CK(cudaMemsetAsync(c.maxdiag.p, 0, sizeof(double), c.stream));
      if (nnz > 0) {
        dev::k_maxdiag_src<<<blocks_for(nnz), kThreads, 0, c.stream>>>(static_cast<int>(nnz), c.src_vals.p,
                                                                       c.src_row.p, c.src_col.p, c.maxdiag.p);
        check_launch(c);
      }
      lo = ladder_phase(c, cf, c.src_vals.p, c.maxdiag.p, delta_min_inout);
    }
    if (attempts) *attempts = lo.attempts;
    if (delta1) *delta1 = lo.delta1;
    if (failed_column) *failed_column = lo.failed;
  });
}

int hykkt_chol_set_factor(hykkt_t h, const double* l_values) {
  return guarded([&] { set_factor(ctx(h), l_values); });
}

int hykkt_chol_set_j(hykkt_t h, int64_t m_c, const int64_t* j_colptr, const int64_t* j_rowidx,
                     const double* j_val) {
  return guarded([&] { chol_set_j(ctx(h), m_c, j_colptr, j_rowidx, j_val); });
}

int hykkt_cg_schur(hykkt_t h, const hykkt_config_t* cfg, const double* rhs, double delta2, double* x,
                   int64_t* iterations, double* relative_residual, int32_t* converged,
                   int32_t* small_quadratic) {
  return guarded([&] {
    Ctx& c = ctx(h);
    require_factor(c);
    if (!c.have_j) throw StateError("no constraint Jacobian on this handle (hykkt_chol_set_j)");
    hykkt_config_t d;
    hykkt_config_default(&d);
    const hykkt_config_t& cf = cfg ? *cfg : d;
    validate_cfg(cf);
    if (delta2 < 0.0) throw InvalidArgument("delta2 must be >= 0");
    const idx mc = c.kp.mc;
    dev::CgResultDev r{0, 0.0, 1, 0};
    if (mc > 0) {
      copy_in(c.cg_rhs.p, rhs, mc, "rhs", c.stream, false);
      CK(cudaMemsetAsync(&c.status.p->abort, 0, sizeof(int), c.stream));
      r = run_cg(c, cf, delta2);
      if (x) CK(cudaMemcpyAsync(x, c.cg_x.p, mc * sizeof(double), cudaMemcpyDefault, c.stream));
      CK(cudaStreamSynchronize(c.stream));
    }
    if (iterations) *iterations = r.iterations;
    if (relative_residual) *relative_residual = r.relres;
    if (converged) *converged = r.converged;
    if (small_quadratic) *small_quadratic = r.small_quadratic;
  });
}

}  // extern "C"

extern "C" {

// Per-handle scheduling knobs (no effect on results): "ks_lpt" = 1 / 0 turns
// the history longest-first system order of the batched solve on / off.
int hykkt_set_option(hykkt_t h, const char* name, int64_t value) {
  return guarded([&] {
    Ctx& c = ctx(h);
    if (!name) throw InvalidArgument("null option name");
    const std::string n(name);
    if (n == "ks_lpt") {
      c.ks.lpt_on = value ? 1 : 0;
    } else if (n == "amalg_width") {
      c.amalg.width = static_cast<int>(value);
    } else if (n == "amalg_zeros_pct") {
      if (value < 0 || value > 100) throw InvalidArgument("amalg_zeros_pct must be in [0, 100]");
      c.amalg.zeros = static_cast<double>(value) / 100.0;
    } else {
      throw InvalidArgument("unknown option: " + n);
    }
  });
}

}  // extern "C"
