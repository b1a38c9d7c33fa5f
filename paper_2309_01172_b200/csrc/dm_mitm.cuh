// dm_mitm.cuh — launcher of the meet-in-the-middle split sweep (dm_mitm.cu).
#pragma once

#include <cuda_runtime.h>

#include "../../include/dagmesh_b200.h"

namespace dm {

// Number of per-CTA partial records the sweep writes (grid size) for a
// device with `sms` SMs.
int mitm_grid(int sms);

// Whole-population identity-split sweep of one instance (memo_valid(t) must
// hold): writes mitm_grid(sms) dm_winner partials into `partial`.  Part
// `part` of `nparts` takes every nparts-th tile, so the parts of one
// population are disjoint and their merged records equal the single sweep.
// Returns DM_E_TOO_LARGE when the instance does not fit the kernel (the
// caller falls back to the rank-range kernels).
int launch_splits_mitm(const dm_tables& t, int part, int nparts, dm_winner* partial, int sms,
                       cudaStream_t stream);

}  // namespace dm
