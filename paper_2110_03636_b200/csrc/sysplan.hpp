// Host-side program for the system-per-CTA streamed Schur-complement
// operator (batched path, BASELINE configs[4]).
//
// Replaces the data movement of the reference's SchurOperator::apply
// (proj/core/src/solver.cpp:144-152): spmv(J^T) -> factor_solve
// (cholesky.cpp:139-168: permute, forward column sweep, backward row sweep)
// -> spmv(J).  One CTA owns one system and keeps the permuted solve vector
// resident in shared memory; everything else it needs arrives as two
// STREAMS laid out in exactly the order the CTA consumes them:
//
//   value stream  (per system, FP64, HBM): L values (diagonal stored as its
//                 reciprocal) and J values, each entry read once per pass;
//   index stream  (shared by all systems, int32, L2-resident): every step's
//                 header, segment / task descriptors, gather indices.
//
// Both are copied into shared-memory rings by TMA bulk copies
// (cp.async.bulk) that run ahead of the consumers, so no global load sits on
// the dependency chain of the supernode tree.
//
// Program = four blocks, each starting on a chunk boundary of both streams:
//   JT   t = P J^T u              (rows of J^T in permuted order)
//   FWD  L y = t                  supernode levels bottom-up
//   BWD  L^T x = y                supernode levels top-down
//   J    q = J x                  (rows of J, CSR order)
// A solve runs a contiguous block range: w solve FWD..J, CG operator JT..J,
// dx solve JT..BWD.
//
// L blocks are cut into STEPS (separated by CTA barriers):
//   phase A: SEGMENTS — partial dot products over long gathers (a forward
//            row of L left of its supernode / a backward column below the
//            diagonal block) into a shared partials array;
//   phase B: TASKS — one supernode each: warp tasks (width > kThreadTaskW;
//            lanes = rows / columns, shuffle triangular solve) and thread
//            tasks (narrow supernodes, gather inline from the stream or
//            from phase-A partials, dense solve of the diagonal block).
#pragma once

#include <cstdint>
#include <vector>

#include "analyze.hpp"
#include "sysplan_format.h"

namespace hykkt {

struct SysPlan {
  int vchunk_lg = 0, nvchunk = 0;  // value ring: nvchunk chunks of 2^vchunk_lg doubles
  int ichunk_lg = 0, nichunk = 0;  // index ring: nichunk chunks of 2^ichunk_lg ints
  int pmax = 0;                    // partial slots
  int nthreads = 0;                // CTA size the thread tasks were dealt for
  int step_chunks = 0;             // L-step cap in chunks (<= n/2 - 1: the next step is
                                   // always requested when a step starts)
  std::vector<int> idx;            // index stream
  std::vector<int> src;            // value stream source (sysplan_format.h kSrc*)
  struct Block {
    long long v0 = 0, v1 = 0, i0 = 0, i1 = 0;  // stream ranges (chunk aligned)
    int s0 = 0, s1 = 0;                        // steps
  } blk[4];
  int nsteps = 0;
  // statistics
  long long value_entries = 0;  // non-padding value entries
  int max_segs_per_step = 0;
  long long ntasks = 0, nsegs = 0;
};

// Builds the program.  Throws InvalidArgument when a supernode block does
// not fit the rings (the caller then uses the lane-per-system path).
SysPlan build_sys_plan(const SupernodalPlan& sp, const KktPlan& kp, int vchunk_lg, int nvchunk, int ichunk_lg,
                       int nichunk, int pmax, int nthreads, int step_chunks = 0);

// Host emulation of the device program on random panel / J values (tests):
// runs JT -> FWD -> BWD -> J and returns the max relative difference to a
// plain dense-free reference (J^T, supernodal solves, J); throws when a step
// touches an entry outside its resident ring windows or a partial slot out
// of range.
double sys_plan_selfcheck(const SupernodalPlan& sp, const KktPlan& kp, const SysPlan& P, unsigned seed);

}  // namespace hykkt
