// Per-interval stop logic of WaveformRelaxation.solve (allatonce.py:250-278), shared by the
// commit kernels of both all-at-once paths (wr_kernels.cu, wr_modal.cu).
#pragma once

#include "pe.h"
#include "pe_internal.h"

namespace pe {

// One sweep's residual for one interval: record it, then the tests in the reference's
// order: tol, diverged (non-finite or > 1e8 max(1, r0)), stall floor, and the max_iter cap.
// Returns true when the interval keeps iterating.
__device__ __forceinline__ bool wr_stop_update(WrColumnState& c, double resid, double tol,
                                               int max_iter, double* resid_hist_row) {
  const int it = c.iterations;
  if (resid_hist_row) resid_hist_row[it] = resid;
  if (it == 0) c.r0 = resid;
  c.iterations = it + 1;
  bool stop = false;
  if (resid <= tol) {
    c.reason = PE_STOP_TOL;
    stop = true;
  } else if (!isfinite(resid) || resid > 1e8 * fmax(1.0, c.r0)) {
    c.reason = PE_STOP_DIVERGED;
    stop = true;
  } else {
    c.stall = (resid >= c.prev) ? c.stall + 1 : 0;
    if (c.stall >= 2 && resid <= 1e3 * tol) {
      c.reason = PE_STOP_FLOOR;
      stop = true;
    }
    c.prev = resid;
  }
  if (!stop && c.iterations >= max_iter) {
    c.reason = PE_STOP_MAX_ITER;
    stop = true;
  }
  c.active = stop ? 0 : 1;
  return !stop;
}

}  // namespace pe
