// dm_common.cuh — device-side building blocks of the placement-cost model.
//
// Every helper restates one piece of /root/reference/pkg/src/dagmesh
// (cited per function) with the reference's exact IEEE-754 binary64 rounding
// sequence.  The whole library is compiled with -fmad=false so `a + b * c`
// stays a DMUL followed by a DADD (two roundings, as CPython evaluates it);
// `/` on double is the correctly rounded div.rn.f64.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include "../../include/dagmesh_b200.h"

namespace dm {

constexpr int kMaxStages = 1024;   // device-side stage limit (bounds arrays)

__host__ __device__ inline bool flops_exact(const dm_tables& t) { return t.flags & DM_F_FLOPS_EXACT; }
__host__ __device__ inline bool bytes_exact(const dm_tables& t) { return t.flags & DM_F_BYTES_EXACT; }
__host__ __device__ inline bool include_comm(const dm_tables& t) { return t.flags & DM_F_INCLUDE_COMM; }
__host__ __device__ inline bool pair_links(const dm_tables& t) { return t.flags & DM_F_PAIR_LINKS; }
__host__ __device__ inline bool chain(const dm_tables& t) { return t.flags & DM_F_CHAIN; }
__host__ __device__ inline bool np_flops(const dm_tables& t) { return t.flags & DM_F_NP_FLOPS; }
__host__ __device__ inline bool np_bytes(const dm_tables& t) { return t.flags & DM_F_NP_BYTES; }
__host__ __device__ inline bool np_comm(const dm_tables& t) { return t.flags & DM_F_NP_COMM; }

// CPython 3.12 builtin sum() (bltinmodule.c builtin_sum_impl).  Over exact
// `float` items: 0 + x0, then Neumaier compensation, compensation added when
// non-zero and finite.  An item that is not an exact float (numpy.float64)
// ends the fast path: the compensation gathered so far is applied and every
// later item is added naively.  The reference calls sum() over floats at
// scheduling.py:160, 174-176, 200, 295, 332-333 and pipeline.py:43.
struct PySum {
    double f = 0.0, c = 0.0;
    bool any = false, naive = false;
    __device__ __forceinline__ void add(double v, bool exact = true) {
        if (!any) { f = 0.0 + v; any = true; naive = !exact; return; }
        if (!naive && !exact) {
            if (c != 0.0 && isfinite(c)) f += c;
            naive = true;
        }
        if (naive) { f = f + v; return; }
        double t = f + v;
        if (fabs(f) >= fabs(v)) c += (f - t) + v;
        else c += (v - t) + f;
        f = t;
    }
    __device__ __forceinline__ double value() const {
        double r = f;
        if (!naive && c != 0.0 && isfinite(c)) r += c;
        return r;
    }
};

// Python sum over col[a..b) (index order): exact int64 prefix difference when
// the column is integral with every prefix < 2^53, else the restated sum()
// (naive when the column holds numpy floats).
__device__ __forceinline__ double col_range(const double* col, const int64_t* pre,
                                            bool exact, int a, int b, bool np_items = false) {
    if (exact) return (double)(pre[b] - pre[a]);
    PySum s;
    for (int i = a; i < b; ++i) s.add(col[i], !np_items);
    return s.value();
}

// hardware.Fleet.link_between (hardware.py:136-140) resolved to peer indices.
__device__ __forceinline__ void link_of(const dm_tables& t, int a, int b,
                                        double& al, double& be) {
    if (a == b) { al = 0.0; be = 0.0; return; }
    if (pair_links(t) && a >= 0 && a < t.P && b >= 0 && b < t.P) {
        int64_t o = (int64_t)a * t.P + b;
        al = __ldg(t.link_alpha + o);
        be = __ldg(t.link_beta + o);
        return;
    }
    al = t.def_alpha; be = t.def_beta;
}

// hardware.comm_time (hardware.py:147-150): alpha + beta*M (DMUL then DADD).
__device__ __forceinline__ double comm_time(double al, double be, double m) {
    return __dadd_rn(al, __dmul_rn(be, m));
}

// scheduling._fits (scheduling.py:172-176) on the contiguous range [a, b).
__device__ __forceinline__ bool fits_range(const dm_tables& t, int w, int a, int b) {
    bool ex = bytes_exact(t), nb = np_bytes(t);
    return col_range(t.gpu, t.pre_gpu, ex, a, b, nb) <= t.cap_gpu[w]
        && col_range(t.cpu, t.pre_cpu, ex, a, b, nb) <= t.cap_cpu[w]
        && col_range(t.disk, t.pre_disk, ex, a, b, nb) <= t.cap_disk[w];
}

// First failing capacity dimension of a contiguous run (verify_assignment
// :199-203): 0 = fits, else DM_V_GPU / DM_V_CPU / DM_V_DISK.
__device__ __forceinline__ int cap_violation(const dm_tables& t, int w, int a, int b) {
    bool ex = bytes_exact(t), nb = np_bytes(t);
    if (col_range(t.gpu, t.pre_gpu, ex, a, b, nb) > t.cap_gpu[w]) return DM_V_GPU;
    if (col_range(t.cpu, t.pre_cpu, ex, a, b, nb) > t.cap_cpu[w]) return DM_V_CPU;
    if (col_range(t.disk, t.pre_disk, ex, a, b, nb) > t.cap_disk[w]) return DM_V_DISK;
    return 0;
}

// scheduling._run_cost (scheduling.py:156-169) for a contiguous run [a, b) on
// peer w, returning compute + read (one DADD, as _evaluate's load :221 and the
// 2-tuple sum() in brute_force_schedule :269 / _hill_climb :361 — for two float
// items CPython's compensated sum equals the plain rounded sum).
// own(src) gives the owner of a stage outside the run.
template <class OwnerFn>
__device__ __forceinline__ void run_cost_contig(const dm_tables& t, int a, int b, int w,
                                                OwnerFn own, double& compute, double& read) {
    double fl = col_range(t.flops, t.pre_flops, flops_exact(t), a, b, np_flops(t));
    compute = fl / t.speed[w];
    double rd = 0.0;
    if (include_comm(t)) {
        if (chain(t)) {
            if (a > 0) {
                int o = own(a - 1);
                double al, be;
                link_of(t, o, w, al, be);
                for (int e = t.edge_ptr[a]; e < t.edge_ptr[a + 1]; ++e)
                    rd = __dadd_rn(rd, comm_time(al, be, t.edge_m[e]));
            }
        } else {
            for (int i = a; i < b; ++i)
                for (int e = t.edge_ptr[i]; e < t.edge_ptr[i + 1]; ++e) {
                    int src = t.edge_src[e];
                    if (src < a || src >= b) {
                        double al, be;
                        link_of(t, own(src), w, al, be);
                        rd = __dadd_rn(rd, comm_time(al, be, t.edge_m[e]));
                    }
                }
        }
    }
    read = rd;
}

// Owner lookup over contiguous runs bounds[0..r] / peers[0..r): binary search.
struct BoundsOwner {
    const int32_t* bounds;
    const int32_t* peers;
    int r;
    __device__ __forceinline__ int operator()(int s) const {
        int lo = 0, hi = r - 1;
        while (lo < hi) {
            int mid = (lo + hi + 1) >> 1;
            if (bounds[mid] <= s) lo = mid; else hi = mid - 1;
        }
        return peers[lo];
    }
};

// ------------------------------------------------------------ arg-min record
struct Win {
    double mk;
    int64_t rank;
    int64_t n_eval;
    int64_t n_feas;
    uint64_t csum;
};

__device__ __forceinline__ void win_init(Win& w) {
    w.mk = __longlong_as_double(0x7ff0000000000000LL);
    w.rank = -1; w.n_eval = 0; w.n_feas = 0; w.csum = 0;
}

// first strict minimum in rank order (brute_force_schedule :271): a candidate
// replaces the incumbent iff mk < best.mk, or equal mk with a smaller rank
// (merging partial results computed out of order).
__device__ __forceinline__ bool win_better(double mk, int64_t rank, double bmk, int64_t brank) {
    if (brank < 0) return rank >= 0;
    if (rank < 0) return false;
    return mk < bmk || (mk == bmk && rank < brank);
}

__device__ __forceinline__ void win_merge(Win& a, const Win& b) {
    if (win_better(b.mk, b.rank, a.mk, a.rank)) { a.mk = b.mk; a.rank = b.rank; }
    a.n_eval += b.n_eval; a.n_feas += b.n_feas; a.csum += b.csum;
}

__device__ __forceinline__ Win warp_reduce_win(Win w) {
    for (int off = 16; off > 0; off >>= 1) {
        Win o;
        o.mk = __shfl_down_sync(0xffffffffu, w.mk, off);
        o.rank = __shfl_down_sync(0xffffffffu, w.rank, off);
        o.n_eval = __shfl_down_sync(0xffffffffu, w.n_eval, off);
        o.n_feas = __shfl_down_sync(0xffffffffu, w.n_feas, off);
        o.csum = __shfl_down_sync(0xffffffffu, w.csum, off);
        win_merge(w, o);
    }
    return w;
}

// Block reduce into partial[blockIdx.x] (blockDim.x multiple of 32, <= 1024).
__device__ __forceinline__ void block_reduce_win_store(Win w, dm_winner* partial) {
    __shared__ Win red[32];
    w = warp_reduce_win(w);
    int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    if (lane == 0) red[wid] = w;
    __syncthreads();
    if (wid == 0) {
        int nw = (blockDim.x + 31) >> 5;
        Win v;
        if (lane < nw) v = red[lane]; else win_init(v);
        v = warp_reduce_win(v);
        if (lane == 0) {
            dm_winner o;
            o.makespan = v.mk; o.rank = v.rank; o.n_evaluated = v.n_eval;
            o.n_feasible = v.n_feas; o.checksum = v.csum;
            partial[blockIdx.x] = o;
        }
    }
}

}  // namespace dm
