// dm_sched.cu — the report half of one schedule() call on the device.
//
// schedule() (scheduling.py:391-423) ends with _evaluate over the chosen runs
// (:210-232): per run compute and read (_run_cost :156-169), the first
// capacity violation in run order (verify_assignment :199-203) and the
// makespan.  schedule_report_kernel derives the runs from the owner vector the
// DP / hill-climb kernels left in device memory and writes everything the
// host needs to assemble the ScheduleReport into one small record, so a
// schedule() call is: one H2D of the tables, the search kernel(s), this
// kernel, one D2H, one synchronisation.
#include "dm_common.cuh"
#include "dm_abi_util.cuh"

namespace dm {

// record layout (dm_sched_out_bytes): header {found, n_runs, code, bad_run,
// makespan}, bounds[n + 1] (int32), peers[n] (int32), compute[n], read[n]
__host__ __device__ inline size_t sched_off_bounds() { return 32; }
__host__ __device__ inline size_t sched_off_peers(int n) { return 32 + (((size_t)(n + 1) * 4 + 7) & ~(size_t)7); }
__host__ __device__ inline size_t sched_off_compute(int n) {
    return sched_off_peers(n) + (((size_t)n * 4 + 7) & ~(size_t)7);
}
__host__ __device__ inline size_t sched_off_read(int n) { return sched_off_compute(n) + (size_t)n * 8; }
__host__ __device__ inline size_t sched_bytes(int n) { return sched_off_read(n) + (size_t)n * 8; }

__global__ void __launch_bounds__(32) schedule_report_kernel(const dm_tables* __restrict__ tables,
                                                             const int16_t* __restrict__ owner,
                                                             const int32_t* __restrict__ found_in,
                                                             unsigned char* out) {
    const dm_tables t = tables[0];
    const int n = t.n, lane = threadIdx.x;
    const int found = found_in ? found_in[0] : 1;
    int32_t* bounds = reinterpret_cast<int32_t*>(out + sched_off_bounds());
    int32_t* peers = reinterpret_cast<int32_t*>(out + sched_off_peers(n));
    double* comp = reinterpret_cast<double*>(out + sched_off_compute(n));
    double* rdo = reinterpret_cast<double*>(out + sched_off_read(n));
    // runs of the owner vector (no feasible DP state: the reference scores
    // ((workers[0], all stages),), :408-410)
    int r = 0;
    for (int base = 0; base < n; base += 32) {
        const int i = base + lane;
        const int oi = i < n ? (found ? owner[i] : 0) : -1;
        const int op = (i < n && i > 0) ? (found ? owner[i - 1] : 0) : -1;
        const bool start = i < n && (i == 0 || oi != op);
        const unsigned bal = __ballot_sync(0xffffffffu, start);
        if (start) {
            const int k = r + __popc(bal & ((1u << lane) - 1u));
            bounds[k] = i;
            peers[k] = oi;
        }
        r += __popc(bal);
    }
    __syncwarp();
    if (lane == 0) bounds[r] = n;
    __syncwarp();
    int first_bad = 0x7fffffff, bad_code = 0;
    double mk = 0.0;
    for (int q = lane; q < r; q += 32) {
        const int a = bounds[q], b = bounds[q + 1], w = peers[q];
        const int v = cap_violation(t, w, a, b);
        if (v && q < first_bad) { first_bad = q; bad_code = v; }
        double c, rd;
        if (chain(t)) {
            const int prev = q > 0 ? peers[q - 1] : -1;
            run_cost_contig(t, a, b, w, [&](int) { return prev; }, c, rd);
        } else {
            BoundsOwner own{bounds, peers, r};
            run_cost_contig(t, a, b, w, own, c, rd);
        }
        comp[q] = c;
        rdo[q] = rd;
        const double load = c + rd;               // _evaluate :221
        mk = load > mk ? load : mk;               // :222
    }
    for (int off = 16; off > 0; off >>= 1) {
        const double o = __shfl_xor_sync(0xffffffffu, mk, off);
        mk = o > mk ? o : mk;
        const int of = __shfl_xor_sync(0xffffffffu, first_bad, off);
        const int oc = __shfl_xor_sync(0xffffffffu, bad_code, off);
        if (of < first_bad) { first_bad = of; bad_code = oc; }
    }
    if (lane == 0) {
        int32_t* h = reinterpret_cast<int32_t*>(out);
        h[0] = found; h[1] = r; h[2] = bad_code; h[3] = bad_code ? first_bad : -1;
        *reinterpret_cast<double*>(out + 16) = mk;
    }
}

}  // namespace dm

extern "C" {

int64_t dm_sched_out_bytes(int32_t n) { return n > 0 ? (int64_t)dm::sched_bytes(n) : -1; }

int dm_schedule_report(const dm_tables* tables, int32_t n, const int16_t* owner, const int32_t* found, void* out,
                       void* stream) {
    if (!tables || !owner || !out || n <= 0) return dmabi::fail(DM_E_ARG, "dm_schedule_report: bad arguments");
    dm::schedule_report_kernel<<<1, 32, 0, (cudaStream_t)stream>>>(tables, owner, found, (unsigned char*)out);
    DM_CHECK_LAUNCH();
    return DM_OK;
}

}  // extern "C"
