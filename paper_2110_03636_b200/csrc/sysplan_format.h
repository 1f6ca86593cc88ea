// Stream-program format shared by the host builder (sysplan.cpp) and the
// device interpreter (kernels_sys.cuh).  Plain C constants only.
//
// Every step starts in the index stream with a header of kHdr ints:
//   [0] kind      kStepFwd / kStepBwd / kStepJT / kStepJ
//   [1] ilen      index entries of the step (header included)
//   [2] vlen      value entries of the step
//   [3] L: segments              J/JT: rows
//   [4] L: warp tasks            J/JT: first row
//   [5] L: thread tasks
//   [6] L: 1 if phase B reads partials written by an earlier step
//   [7] L: warps taking the warp tasks (thread tasks are dealt over the
//       remaining compute threads)
// L steps continue with segment descriptors (kSegInts each: value offset,
// index offset, len | slot << 16; offsets relative to the step's bases),
// task descriptors (kTaskInts each: value offset, index offset, first
// column, width | mode << 16; warp tasks first, thread tasks dealt so that
// thread task t goes to compute thread 32 ww + (t mod (NT - 32 ww))), then
// the payload.
// J / JT steps continue with rows + 1 relative value offsets, then one index
// per value entry.
//
// Task payloads (value side / index side):
//   forward  tri w(w+1)/2 row-major (r, j<=r) at r(r+1)/2 + j, diagonal as
//            reciprocal; inline: then row r's gathers (ascending column) /
//            counts c_0..c_{w-1}, pad, then the gathers' columns;
//            segmented: / first partial slot of rows 0..w-1, end slot
//   backward tri column-major (j>=k, k) at k*w - k(k-1)/2 + (j-k), diagonal
//            as reciprocal; inline: then the rows below, row-major nb x w /
//            nb, then the nb rows;  segmented: / first partial slot of
//            columns 0..w-1, end slot
#ifndef HYKKT_SYSPLAN_FORMAT_H_
#define HYKKT_SYSPLAN_FORMAT_H_

#define HYKKT_SP_HDR 8
#define HYKKT_SP_SEG_INTS 3
#define HYKKT_SP_TASK_INTS 4

#define HYKKT_STEP_FWD 0
#define HYKKT_STEP_BWD 1
#define HYKKT_STEP_JT 2
#define HYKKT_STEP_J 3

#define HYKKT_TASK_INLINE 1
#define HYKKT_TASK_SEGMENTED 2

// The widest supernode a single thread solves is a host-side choice
// (sysplan.cpp thread_task_w(), default 3 from the B200 sweep): the device
// reads the task kind from the step header, not from the width.

// Value stream source encoding (int32):
//   s >= 0   panel slot (s >> 1); (s & 1) = store the reciprocal
//   s == -1  zero (padding)
//   s <= -2  scaled J value, CSC entry (-2 - s)
#define HYKKT_SRC_ZERO (-1)

#endif  // HYKKT_SYSPLAN_FORMAT_H_
