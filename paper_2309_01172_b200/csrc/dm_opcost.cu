// dm_opcost.cu — per-operator PALEO cost T = R + C + W (hardware.op_time,
// hardware.py:190-206) and the per-cell bounds of hardware.subgraph_time
// (:219-226), batched over placements: one thread per (placement, op).
#include "dm_common.cuh"
#include "dm_abi_util.cuh"

namespace dm {

__global__ void __launch_bounds__(256) op_costs_kernel(dm_ops ops, dm_tables t, const double* __restrict__ write_bw,
                                                       int32_t n_place, const int32_t* __restrict__ place,
                                                       double* __restrict__ out, uint8_t* __restrict__ out_np) {
    const int64_t gid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int n = ops.n_ops;
    if (gid >= (int64_t)n_place * n) return;
    const int64_t b = gid / n;
    const int i = (int)(gid % n);
    const int32_t* pl = place + b * n;
    const int me = pl[i];
    double* o = out + gid * 3;
    if (me < 0 || me >= t.P) {   // op placed on a peer unknown to the fleet: fleet.peer raises (host)
        o[0] = o[1] = o[2] = __longlong_as_double(0x7ff8000000000000LL);
        if (out_np) out_np[gid] = 0;
        return;
    }
    bool is_np = t.peer_np && t.peer_np[me];                           // compute_s type
    double read = 0.0;
    for (int e = ops.arg_ptr[i]; e < ops.arg_ptr[i + 1]; ++e) {        // :197-201
        const int a = ops.arg_idx[e];
        const int src = pl[a];
        if (src != me) {
            double al, be;
            link_of(t, src, me, al, be);
            read = __dadd_rn(read, comm_time(al, be, ops.mbytes[a]));
            is_np |= (ops.flags & DM_OPS_NP_LINKS) != 0;
        }
    }
    const double compute = ops.flops[i] / t.speed[me];                // :202, :209-210
    double write = 0.0;
    for (int e = ops.user_ptr[i]; e < ops.user_ptr[i + 1]; ++e)        // :204-205
        if (pl[ops.user_idx[e]] != me) {
            write = ops.mbytes[i] / write_bw[me];
            is_np |= ops.write_np && ops.write_np[me];
            break;
        }
    o[0] = read; o[1] = compute; o[2] = write;
    if (out_np) out_np[gid] = is_np;
}

// subgraph_time: totals = R + C + W per op (OpCost.total_s, :185-187); lower
// = max(totals), upper = sequential = CPython sum(totals) (Neumaier, naive
// from the first numpy total on).
__global__ void subgraph_kernel(int32_t n_ops, int32_t n_place, const double* __restrict__ op_out,
                                const uint8_t* __restrict__ op_np, int32_t n_sub,
                                const int32_t* __restrict__ sub_ptr, const int32_t* __restrict__ sub_idx,
                                double* __restrict__ out) {
    const int64_t gid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (gid >= (int64_t)n_place * n_sub) return;
    const int64_t b = gid / n_sub;
    const int s = (int)(gid % n_sub);
    PySum acc;
    double mx = 0.0;
    bool any = false;
    for (int e = sub_ptr[s]; e < sub_ptr[s + 1]; ++e) {
        const double* o = op_out + (b * n_ops + sub_idx[e]) * 3;
        const double tot = __dadd_rn(__dadd_rn(o[0], o[1]), o[2]);
        acc.add(tot, !(op_np && op_np[b * n_ops + sub_idx[e]]));
        if (!any || tot > mx) mx = tot;
        any = true;
    }
    double* r = out + gid * 3;
    const double seq = any ? acc.value() : 0.0;
    r[0] = any ? mx : 0.0; r[1] = seq; r[2] = seq;
}

}  // namespace dm

extern "C" {

int dm_op_costs(const dm_ops* ops, const dm_tables* t, const double* write_bw, int32_t n_place,
                const int32_t* place, double* out, uint8_t* out_np, void* stream) {
    if (!ops || !t || !write_bw || n_place < 0 || !place || !out) return dmabi::fail(DM_E_ARG, "dm_op_costs: bad arguments");
    int64_t work = (int64_t)n_place * ops->n_ops;
    if (work == 0) return DM_OK;
    int blocks = (int)((work + 255) / 256);
    dm::op_costs_kernel<<<blocks, 256, 0, (cudaStream_t)stream>>>(*ops, *t, write_bw, n_place, place, out, out_np);
    DM_CHECK_LAUNCH();
    return DM_OK;
}

int dm_subgraph_times(int32_t n_ops, int32_t n_place, const double* op_out, const uint8_t* op_np, int32_t n_sub,
                      const int32_t* sub_ptr,
                      const int32_t* sub_idx, double* out, void* stream) {
    if (n_ops < 0 || n_place < 0 || n_sub < 0 || !op_out || !sub_ptr || !out)
        return dmabi::fail(DM_E_ARG, "dm_subgraph_times: bad arguments");
    int64_t work = (int64_t)n_place * n_sub;
    if (work == 0) return DM_OK;
    int blocks = (int)((work + 255) / 256);
    dm::subgraph_kernel<<<blocks, 256, 0, (cudaStream_t)stream>>>(n_ops, n_place, op_out, op_np, n_sub, sub_ptr, sub_idx, out);
    DM_CHECK_LAUNCH();
    return DM_OK;
}

}  // extern "C"
