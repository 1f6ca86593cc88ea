// Batched path (B systems, one shared pattern).  Placeholder entry points
// until the lane-per-system kernels land; they fail loudly.
#include "../../include/hykkt.h"

extern "C" {
int hykkt_batch_solve(hykkt_t, const hykkt_config_t*, int64_t, const hykkt_values_t*, int,
                      hykkt_report_t*, double*, double*, double*, double*) {
  return HYKKT_ERR_STATE;
}
int hykkt_batch_upload(hykkt_t, int64_t, const hykkt_values_t*) { return HYKKT_ERR_STATE; }
int hykkt_batch_solve_resident(hykkt_t, const hykkt_config_t*, int, hykkt_report_t*) {
  return HYKKT_ERR_STATE;
}
int hykkt_batch_download(hykkt_t, double*, double*, double*, double*) { return HYKKT_ERR_STATE; }
}
