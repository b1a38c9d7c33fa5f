// dm_mitm.cuh — launcher of the meet-in-the-middle split sweep (dm_mitm.cu).
#pragma once

#include <cuda_runtime.h>

#include "../../include/dagmesh_b200.h"

namespace dm {

// Grid of the cross-product microbenchmark for a device with `sms` SMs.
int mitm_grid(int sms);

// Device workspace (bytes) the sweep's side tables need, or -1 when the
// sweep does not apply to the instance.
int64_t mitm_workspace_bytes(const dm_tables& t);

// Whole-population identity-split sweep of one instance (memo_valid(t) must
// hold): builds the side tables in `ws` (stream-ordered allocation when ws is
// NULL or smaller than mitm_workspace_bytes) and writes mitm_grid(sms)
// dm_winner partials (*n_partials, at most 2 per SM) into `partial`.  Part `part` of `nparts` takes every
// nparts-th tile, so the parts of one population are disjoint and their merged
// records equal the single sweep.  Returns DM_E_TOO_LARGE when the instance
// does not fit the kernel (the caller falls back to the rank-range kernels).
// phase: 1 = T image + side tables, 2 = the sweep kernel, 3 = both (phases
// 1 and 2 apart need the caller's workspace, which carries the tables).
int launch_splits_mitm(const dm_tables& t, int part, int nparts, dm_winner* partial, int sms, void* ws,
                       int64_t ws_bytes, int* n_partials, cudaStream_t stream, int phase = 3);

}  // namespace dm
