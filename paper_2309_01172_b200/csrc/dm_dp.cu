// dm_dp.cu — batched exact subset DP (scheduling._subset_dp, scheduling.py:288-325).
//
// The reference pushes states (stage prefix i, used-worker mask) forward in
// the order: layers i ascending, masks ascending, workers ascending, j
// ascending (with the _fits break), keeping the FIRST strict minimum per
// target.  For a fixed target (j, M') the sources arrive in the order
// (i ascending, source mask ascending) = (i ascending, worker wi descending),
// so the pull form below reduces every target with the associative key
//     (value, i, p-1-wi)   lexicographic minimum,
// which reproduces the reference's winner exactly (including ties) while
// letting a warp evaluate all (i, wi) sources of a target in parallel.
// Level j depends only on levels < j: one __syncthreads per level.
//
// One CTA per scenario (persistent loop over scenarios), per-CTA scratch in
// global memory (L1/L2 resident for the sizes the reference's gate admits:
// n*n*p*2^p <= 3e6).
#include "dm_common.cuh"
#include "dm_abi_util.cuh"
#include <cstdlib>

namespace dm {

struct DpScratch {
    double* cc;       // [(n+1) * (n+1) * p] chunk_cost(i, j, wi)
    int16_t* jlim;    // [(n+1) * p] first j failing _fits for (i, wi)
    double* mk;       // [(n+1) << p]
    int32_t* back;    // [(n+1) << p]  (i << 8) | wi, -1 = absent
};

__host__ __device__ inline size_t align_up(size_t x) { return (x + 255) & ~(size_t)255; }

__host__ __device__ inline size_t dp_scratch_bytes(int n, int p) {
    size_t n1 = (size_t)n + 1;
    return align_up(n1 * n1 * p * sizeof(double)) + align_up(n1 * p * sizeof(int16_t)) +
           align_up((n1 << p) * sizeof(double)) + align_up((n1 << p) * sizeof(int32_t));
}

__device__ inline DpScratch dp_carve(unsigned char* base, int n, int p) {
    size_t n1 = (size_t)n + 1;
    DpScratch s;
    s.cc = (double*)base; base += align_up(n1 * n1 * p * sizeof(double));
    s.jlim = (int16_t*)base; base += align_up(n1 * p * sizeof(int16_t));
    s.mk = (double*)base; base += align_up((n1 << p) * sizeof(double));
    s.back = (int32_t*)base;
    return s;
}

__device__ __forceinline__ bool key_less(double v, int sec, double bv, int bsec) {
    return v < bv || (v == bv && sec < bsec);
}

// smem_mode: 0 = all tables in per-CTA global scratch, 1 = DP states and
// break points in shared memory (chunk costs in scratch), 2 = everything in
// shared memory.
__global__ void __launch_bounds__(256) subset_dp_kernel(const dm_tables* __restrict__ tables, int32_t n_scen,
                                                        int32_t n_max, int32_t p_max, int16_t* out_owner,
                                                        double* out_mk, int32_t* out_found, unsigned char* scratch,
                                                        size_t scratch_per_cta, int smem_mode) {
    extern __shared__ __align__(16) unsigned char dsm[];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
    for (int sc = blockIdx.x; sc < n_scen; sc += gridDim.x) {
        __syncthreads();
        const dm_tables t = tables[sc];
        const int n = t.n, p = t.p;
        const int64_t S = (int64_t)1 << p;
        DpScratch d = dp_carve(scratch + (size_t)blockIdx.x * scratch_per_cta, n, p);
        const int n1 = n + 1;
        if (smem_mode >= 1) {   // states + break points (sized for this scenario) in shared memory
            unsigned char* b = dsm;
            d.mk = reinterpret_cast<double*>(b); b += align_up(((size_t)n1 << p) * sizeof(double));
            d.back = reinterpret_cast<int32_t*>(b); b += align_up(((size_t)n1 << p) * sizeof(int32_t));
            d.jlim = reinterpret_cast<int16_t*>(b); b += align_up((size_t)n1 * p * sizeof(int16_t));
            if (smem_mode == 2) d.cc = reinterpret_cast<double*>(b);
        }
        // ---- _fits break points (:313-315): first j with !_fits(w, range(i, j))
        for (int it = threadIdx.x; it < n * p; it += blockDim.x) {
            int i = it / p, wi = it % p;
            int j = i + 1;
            while (j <= n && fits_range(t, wi, i, j)) ++j;
            d.jlim[i * p + wi] = (int16_t)j;
        }
        // ---- chunk_cost (:294-302): default link, edges with src < i only;
        //      one thread per (i, wi), the read growing stage by stage in the
        //      reference's (stage, edge) order
        for (int it = threadIdx.x; it < n * p; it += blockDim.x) {
            const int i = it / p, wi = it % p;
            double rd = 0.0;
            for (int j = i + 1; j <= n; ++j) {
                if (include_comm(t))
                    for (int e = t.edge_ptr[j - 1]; e < t.edge_ptr[j]; ++e)
                        if (t.edge_src[e] < i) rd = __dadd_rn(rd, comm_time(t.def_alpha, t.def_beta, t.edge_m[e]));
                const double fl = col_range(t.flops, t.pre_flops, flops_exact(t), i, j, np_flops(t));
                d.cc[((size_t)i * n1 + j) * p + wi] = fl / t.speed[wi] + rd;
            }
        }
        for (int64_t it = threadIdx.x; it < (int64_t)n1 * S; it += blockDim.x) d.back[it] = -1;
        __syncthreads();
        if (threadIdx.x == 0) { d.mk[0] = 0.0; d.back[0] = 0; }  // state (0, 0)
        __syncthreads();
        // ---- levels j = 1..n, one warp per target mask
        for (int j = 1; j <= n; ++j) {
            for (int64_t M = wid; M < S; M += nwarps) {
                int pc = __popcll((unsigned long long)M);
                if (pc == 0 || pc > j) continue;
                double bv = 0.0; int bsec = 0x7fffffff; int bsrc = -1;
                // lanes over the source prefix i, every worker wi of M in turn
                for (int i = lane; i < j; i += 32) {
                    const double* ccrow = d.cc + ((size_t)i * n1 + j) * p;
                    for (uint32_t mm = (uint32_t)M; mm; mm &= mm - 1) {
                        const int wi = __ffs(mm) - 1;
                        const int64_t src = (int64_t)i * S + (M ^ ((int64_t)1 << wi));
                        if (d.back[src] < 0 || j >= d.jlim[i * p + wi]) continue;
                        const double m0 = d.mk[src];
                        const double cc = ccrow[wi];
                        const double v = cc > m0 ? cc : m0;        // max(mk, chunk_cost) :316
                        const int sec = i * 64 + (63 - wi);
                        if (bsrc < 0 || key_less(v, sec, bv, bsec)) { bv = v; bsec = sec; bsrc = (i << 8) | wi; }
                    }
                }
                for (int off = 16; off > 0; off >>= 1) {
                    double ov = __shfl_down_sync(0xffffffffu, bv, off);
                    int osec = __shfl_down_sync(0xffffffffu, bsec, off);
                    int osrc = __shfl_down_sync(0xffffffffu, bsrc, off);
                    if (osrc >= 0 && (bsrc < 0 || key_less(ov, osec, bv, bsec))) { bv = ov; bsec = osec; bsrc = osrc; }
                }
                if (lane == 0 && bsrc >= 0) {
                    int64_t key = (int64_t)j * S + M;
                    d.mk[key] = bv;
                    d.back[key] = bsrc;
                }
            }
            __syncthreads();
        }
        // ---- finals: smallest (makespan, mask) among states with j == n (:321-325)
        __shared__ double fv[32];
        __shared__ long long fm[32];
        double bv = 0.0; long long bm = -1;
        for (int64_t M = threadIdx.x; M < S; M += blockDim.x) {
            int64_t key = (int64_t)n * S + M;
            if (d.back[key] < 0) continue;
            double v = d.mk[key];
            if (bm < 0 || v < bv || (v == bv && M < bm)) { bv = v; bm = M; }
        }
        for (int off = 16; off > 0; off >>= 1) {
            double ov = __shfl_down_sync(0xffffffffu, bv, off);
            long long om = __shfl_down_sync(0xffffffffu, bm, off);
            if (om >= 0 && (bm < 0 || ov < bv || (ov == bv && om < bm))) { bv = ov; bm = om; }
        }
        if (lane == 0) { fv[wid] = bv; fm[wid] = bm; }
        __syncthreads();
        if (threadIdx.x == 0) {
            for (int w = 1; w < nwarps; ++w)
                if (fm[w] >= 0 && (bm < 0 || fv[w] < bv || (fv[w] == bv && fm[w] < bm))) { bv = fv[w]; bm = fm[w]; }
            int16_t* own = out_owner + (size_t)sc * n_max;
            for (int i = 0; i < n_max; ++i) own[i] = -1;
            if (bm >= 0) {
                int j = n; int64_t M = bm;
                while (j > 0) {
                    int32_t b = d.back[(int64_t)j * S + M];
                    int i = b >> 8, wi = b & 0xff;
                    for (int s = i; s < j; ++s) own[s] = (int16_t)wi;
                    M &= ~((int64_t)1 << wi);
                    j = i;
                }
                out_mk[sc] = bv;
                out_found[sc] = 1;
            } else {
                out_mk[sc] = __longlong_as_double(0x7ff0000000000000LL);
                out_found[sc] = 0;
            }
        }
    }
}

// ---- small fleets (2^p <= 32 masks): one WARP per scenario, lanes over the
//      target masks of a level, __syncwarp between levels, every table in the
//      warp's slice of shared memory.  Same pull-form key and finals as above.
constexpr int kDpWarps = 4;

// Per-warp shared memory: chunk costs, states, back pointers, break points,
// then the instance columns the DP reads (staged once, so the table builds
// run from shared memory instead of dependent global loads).
__host__ __device__ inline size_t dpw_cols_bytes(int n, int p, int e_max) {
    const size_t n1 = (size_t)n + 1;
    return align_up(4 * n1 * 8) + align_up(4 * (size_t)n * 8) + align_up(n1 * 4) + align_up((size_t)e_max * 4) +
           align_up((size_t)e_max * 8) + align_up(4 * (size_t)p * 8);
}

__host__ __device__ inline size_t dpw_bytes(int n, int p, int e_max) {
    const size_t n1 = (size_t)n + 1, S = (size_t)1 << p;
    return align_up((size_t)n * n1 / 2 * p * 8) + align_up(n1 * S * 8) + align_up(n1 * S * 4) + align_up(n1 * p * 2) +
           dpw_cols_bytes(n, p, e_max);
}

// Copy the DP's columns of t into smem at b (warp-cooperative) and return a
// dm_tables whose pointers refer to the copies.
__device__ inline dm_tables dpw_stage(const dm_tables& t, unsigned char* b, int lane, int e_max, int stride = 32) {
    const int n = t.n, p = t.p, n1 = n + 1, E = t.n_edges;
    dm_tables c = t;
    int64_t* pre = reinterpret_cast<int64_t*>(b); b += align_up(4 * (size_t)n1 * 8);
    double* col = reinterpret_cast<double*>(b); b += align_up(4 * (size_t)n * 8);
    int32_t* eptr = reinterpret_cast<int32_t*>(b); b += align_up((size_t)n1 * 4);
    int32_t* esrc = reinterpret_cast<int32_t*>(b); b += align_up((size_t)e_max * 4);
    double* em = reinterpret_cast<double*>(b); b += align_up((size_t)e_max * 8);
    double* peer = reinterpret_cast<double*>(b);
    for (int i = lane; i < n1; i += stride) {
        pre[i] = t.pre_flops[i]; pre[n1 + i] = t.pre_gpu[i]; pre[2 * n1 + i] = t.pre_cpu[i];
        pre[3 * n1 + i] = t.pre_disk[i]; eptr[i] = t.edge_ptr[i];
    }
    for (int i = lane; i < n; i += stride) {
        col[i] = t.flops[i]; col[n + i] = t.gpu[i]; col[2 * n + i] = t.cpu[i]; col[3 * n + i] = t.disk[i];
    }
    const bool stage_edges = E <= e_max;
    if (stage_edges)
        for (int e = lane; e < E; e += stride) { esrc[e] = t.edge_src[e]; em[e] = t.edge_m[e]; }
    for (int w = lane; w < p; w += stride) {
        peer[w] = t.speed[w]; peer[p + w] = t.cap_gpu[w]; peer[2 * p + w] = t.cap_cpu[w]; peer[3 * p + w] = t.cap_disk[w];
    }
    c.pre_flops = pre; c.pre_gpu = pre + n1; c.pre_cpu = pre + 2 * n1; c.pre_disk = pre + 3 * n1;
    c.flops = col; c.gpu = col + n; c.cpu = col + 2 * n; c.disk = col + 3 * n;
    c.edge_ptr = eptr;
    if (stage_edges) { c.edge_src = esrc; c.edge_m = em; }
    c.speed = peer; c.cap_gpu = peer + p; c.cap_cpu = peer + 2 * p; c.cap_disk = peer + 3 * p;
    return c;
}

__device__ __forceinline__ int dpw_pair(int i, int j, int n) { return i * n - i * (i - 1) / 2 + (j - i - 1); }

constexpr int kDpLaneMaxP = 8;   // fleets of up to 8 workers: 2^p <= 256 target masks

// ---- mid-size fleets (32 < 2^p <= 256): one CTA per scenario, one thread
//      per (target mask, worker) SOURCE FAMILY: thread (M, wi) folds sources
//      (i, M - wi) over i in key order (a value-only compare keeps the first
//      strict minimum), writes its best to shared memory, and one thread per
//      mask then reduces its workers with the full key — every thread of a
//      level carries ~j source evaluations (a thread per mask would carry
//      popcount(M) x j, and the masks with most workers would set each
//      level's length).  Pairs are ordered by popcount so a warp's pairs have
//      the same source count; states of every level in shared memory (int16
//      back pointers), each level's chunk-cost column staged in shared memory
//      while the previous level reduces, instance columns staged once.
constexpr int kDpPairThreads = 1024;
__host__ __device__ inline size_t dpp_smem(int n_max, int e_max) {
    const size_t n1 = (size_t)n_max + 1, S = (size_t)1 << kDpLaneMaxP, P = (size_t)kDpLaneMaxP;
    return align_up(n1 * S * sizeof(double)) + align_up(n1 * S * sizeof(int16_t)) +
           align_up(n1 * P * sizeof(int16_t)) + align_up(S * P * 2) +             // jlim, pair (mask, worker)
           align_up(S * P * sizeof(double)) + align_up(S * P) +                      // per-pair best value, stage
           2 * align_up((size_t)n_max * P * 8) + dpw_cols_bytes(n_max, kDpLaneMaxP, e_max);
}

__global__ void __launch_bounds__(kDpPairThreads, 1) subset_dp_pair_kernel(const dm_tables* __restrict__ tables,
                                                                           int32_t n_scen, int32_t n_max,
                                                                           int32_t e_max, int16_t* out_owner,
                                                                           double* out_mk, int32_t* out_found,
                                                                           unsigned char* scratch,
                                                                           size_t scratch_per_cta) {
    extern __shared__ __align__(16) unsigned char dsm[];
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5, nwarps = blockDim.x >> 5;
    for (int sc = blockIdx.x; sc < n_scen; sc += gridDim.x) {
        __syncthreads();
        const dm_tables tg = tables[sc];
        const int n = tg.n, p = tg.p, S = 1 << p, n1 = n + 1;
        const int npairs = p << (p - 1);                      // sum of popcounts over the 2^p masks
        DpScratch d = dp_carve(scratch + (size_t)blockIdx.x * scratch_per_cta, n, p);
        unsigned char* b = dsm;
        double* mk = reinterpret_cast<double*>(b); b += align_up((size_t)n1 * S * sizeof(double));
        int16_t* back = reinterpret_cast<int16_t*>(b); b += align_up((size_t)n1 * S * sizeof(int16_t));
        int16_t* jlim = reinterpret_cast<int16_t*>(b); b += align_up((size_t)n1 * p * sizeof(int16_t));
        uint8_t* pm = b;                                      // pair -> mask
        uint8_t* pw = b + (size_t)S * kDpLaneMaxP; b += align_up((size_t)S * kDpLaneMaxP * 2);   // pair -> worker
        double* cv = reinterpret_cast<double*>(b); b += align_up((size_t)S * kDpLaneMaxP * sizeof(double));
        int8_t* ci = reinterpret_cast<int8_t*>(b); b += align_up((size_t)S * kDpLaneMaxP);
        double* ccb[2];
        ccb[0] = reinterpret_cast<double*>(b); b += align_up((size_t)n_max * kDpLaneMaxP * 8);
        ccb[1] = reinterpret_cast<double*>(b); b += align_up((size_t)n_max * kDpLaneMaxP * 8);
        const dm_tables t = dpw_stage(tg, b, tid, e_max, blockDim.x);
        __syncthreads();
        // ---- _fits break points (:313-315) and chunk_cost (:294-302), as subset_dp_kernel
        for (int it = tid; it < n * p; it += blockDim.x) {
            const int i = it / p, wi = it % p;
            int j = i + 1;
            while (j <= n && fits_range(t, wi, i, j)) ++j;
            jlim[i * p + wi] = (int16_t)j;
        }
        for (int it = tid; it < n * p; it += blockDim.x) {
            const int i = it / p, wi = it % p;
            double rd = 0.0;
            for (int j = i + 1; j <= n; ++j) {
                if (include_comm(t))
                    for (int e = t.edge_ptr[j - 1]; e < t.edge_ptr[j]; ++e)
                        if (t.edge_src[e] < i) rd = __dadd_rn(rd, comm_time(t.def_alpha, t.def_beta, t.edge_m[e]));
                const double fl = col_range(t.flops, t.pre_flops, flops_exact(t), i, j, np_flops(t));
                d.cc[((size_t)i * n1 + j) * p + wi] = fl / t.speed[wi] + rd;
            }
        }
        // pairs in (popcount, mask, worker) order: mask M's first pair sits
        // after every pair of the masks with fewer workers and of the masks
        // with as many workers and a smaller value
        if (tid < S) {
            const int M = tid, pc = __popc(M);
            int base = 0;
            for (int q = 0; q < M; ++q) base += __popc(q) == pc ? pc : 0;
            for (int q = 0; q < S; ++q) base += __popc(q) < pc ? __popc(q) : 0;
            int r = 0;
            for (uint32_t mm = (uint32_t)M; mm; mm &= mm - 1, ++r) {
                pm[base + r] = (uint8_t)M;
                pw[base + r] = (uint8_t)(__ffs(mm) - 1);
            }
        }
        for (int it = tid; it < n1 * S; it += blockDim.x) back[it] = -1;
        for (int it = tid; it < p; it += blockDim.x) ccb[1][it] = d.cc[((size_t)0 * n1 + 1) * p + it];   // level 1
        __syncthreads();
        if (tid == 0) { mk[0] = 0.0; back[0] = 0; }  // state (0, 0)
        __syncthreads();
        for (int j = 1; j <= n; ++j) {
            const double* ccj = ccb[j & 1];
            // ---- every (mask, worker) source family of level j
            for (int q = tid; q < npairs; q += blockDim.x) {
                const int M = pm[q], wi = pw[q], pc = __popc(M);
                double bv = __longlong_as_double(0x7ff0000000000000LL);
                int bi = -1;
                if (pc <= j) {
                    const int srcm = M ^ (1 << wi);
#pragma unroll 4
                    for (int i = pc - 1; i < j; ++i) {
                        const int src = i * S + srcm;
                        const bool ok = back[src] >= 0 && j < jlim[i * p + wi];
                        const double m0 = mk[src];
                        const double cc = ccj[i * p + wi];
                        const double v = cc > m0 ? cc : m0;        // max(mk, chunk_cost) :316
                        if (ok && v < bv) { bv = v; bi = i; }
                    }
                }
                cv[M * p + wi] = bv;
                ci[M * p + wi] = (int8_t)bi;
            }
            __syncthreads();
            // ---- each target mask reduces its workers with the full key;
            //      the other threads stage level j+1's chunk costs
            if (tid < S) {
                const int M = tid, pc = __popc(M);
                if (pc > 0 && pc <= j) {
                    double bv = 0.0;
                    int bsec = 0x7fffffff, bsrc = -1;
                    for (uint32_t mm = (uint32_t)M; mm; mm &= mm - 1) {
                        const int wi = __ffs(mm) - 1;
                        const int i = ci[M * p + wi];
                        if (i < 0) continue;
                        const double v = cv[M * p + wi];
                        const int sec = i * 64 + (63 - wi);
                        if (bsrc < 0 || key_less(v, sec, bv, bsec)) { bv = v; bsec = sec; bsrc = (i << 8) | wi; }
                    }
                    if (bsrc >= 0) {
                        mk[j * S + M] = bv;
                        back[j * S + M] = (int16_t)bsrc;
                    }
                }
            } else if (j < n) {
                double* nxt = ccb[(j + 1) & 1];
                for (int it = tid - S; it < (j + 1) * p; it += blockDim.x - S)
                    nxt[it] = d.cc[((size_t)(it / p) * n1 + j + 1) * p + (it % p)];
            }
            __syncthreads();
        }
        // ---- finals: smallest (makespan, mask) among states with j == n (:321-325)
        __shared__ double fv[32];
        __shared__ int fm[32];
        double bv = 0.0;
        int bm = -1;
        for (int q = tid; q < S; q += blockDim.x) {
            if (back[n * S + q] < 0) continue;
            const double v = mk[n * S + q];
            if (bm < 0 || v < bv || (v == bv && q < bm)) { bv = v; bm = q; }
        }
        for (int off = 16; off > 0; off >>= 1) {
            const double ov = __shfl_down_sync(0xffffffffu, bv, off);
            const int om = __shfl_down_sync(0xffffffffu, bm, off);
            if (om >= 0 && (bm < 0 || ov < bv || (ov == bv && om < bm))) { bv = ov; bm = om; }
        }
        if (lane == 0) { fv[wid] = bv; fm[wid] = bm; }
        __syncthreads();
        if (tid == 0) {
            for (int w = 1; w < nwarps; ++w)
                if (fm[w] >= 0 && (bm < 0 || fv[w] < bv || (fv[w] == bv && fm[w] < bm))) { bv = fv[w]; bm = fm[w]; }
            int16_t* own = out_owner + (size_t)sc * n_max;
            for (int i = 0; i < n_max; ++i) own[i] = -1;
            if (bm >= 0) {
                int j = n, q = bm;
                while (j > 0) {
                    const int bb = back[j * S + q];
                    const int i = bb >> 8, wi = bb & 0xff;
                    for (int s2 = i; s2 < j; ++s2) own[s2] = (int16_t)wi;
                    q &= ~(1 << wi);
                    j = i;
                }
                out_mk[sc] = bv;
                out_found[sc] = 1;
            } else {
                out_mk[sc] = __longlong_as_double(0x7ff0000000000000LL);
                out_found[sc] = 0;
            }
        }
    }
}

__global__ void __launch_bounds__(32 * kDpWarps) subset_dp_warp_kernel(const dm_tables* __restrict__ tables,
                                                                       int32_t n_scen, int32_t n_max,
                                                                       int32_t p_max, int32_t e_max,
                                                                       int16_t* out_owner, double* out_mk,
                                                                       int32_t* out_found) {
    extern __shared__ __align__(16) unsigned char dsm[];
    const int lane = threadIdx.x & 31, wl = threadIdx.x >> 5;
    unsigned char* base = dsm + (size_t)wl * dpw_bytes(n_max, p_max, e_max);
    for (int sc = blockIdx.x * kDpWarps + wl; sc < n_scen; sc += gridDim.x * kDpWarps) {
        const dm_tables tg = tables[sc];
        const int n = tg.n, p = tg.p, S = 1 << p, n1 = n + 1;
        unsigned char* b = base;
        double* cc = reinterpret_cast<double*>(b); b += align_up((size_t)n * n1 / 2 * p * 8);
        double* mk = reinterpret_cast<double*>(b); b += align_up((size_t)n1 * S * 8);
        int32_t* back = reinterpret_cast<int32_t*>(b); b += align_up((size_t)n1 * S * 4);
        int16_t* jlim = reinterpret_cast<int16_t*>(b); b += align_up((size_t)n1 * p * 2);
        __syncwarp();
        const dm_tables t = dpw_stage(tg, b, lane, e_max);
        __syncwarp();
        for (int it = lane; it < n * p; it += 32) {             // _fits break points (:313-315)
            const int i = it / p, wi = it % p;
            int j = i + 1;
            while (j <= n && fits_range(t, wi, i, j)) ++j;
            jlim[i * p + wi] = (int16_t)j;
        }
        for (int i = lane; i < n; i += 32) {                   // chunk_cost (:294-302), lanes over i:
            double rd = 0.0;                                    // the read grows stage by stage, in the
            for (int j = i + 1; j <= n; ++j) {                  // reference's (stage, edge) order
                if (include_comm(t))
                    for (int e = t.edge_ptr[j - 1]; e < t.edge_ptr[j]; ++e)
                        if (t.edge_src[e] < i) rd = __dadd_rn(rd, comm_time(t.def_alpha, t.def_beta, t.edge_m[e]));
                const double fl = col_range(t.flops, t.pre_flops, flops_exact(t), i, j, np_flops(t));
                double* row = cc + (size_t)dpw_pair(i, j, n) * p;
                for (int wi = 0; wi < p; ++wi) row[wi] = fl / t.speed[wi] + rd;
            }
        }
        for (int it = lane; it < n1 * S; it += 32) back[it] = -1;
        __syncwarp();
        if (lane == 0) { mk[0] = 0.0; back[0] = 0; }
        __syncwarp();
        // levels: lane = (target mask M, source-prefix class g); lanes of one M
        // split the prefixes i (i = g mod G) and combine by shuffles
        const int G = 32 / S;                                   // lanes per target mask (S <= 32)
        const int M = lane & (S - 1), g = lane / S;
        const int pc = __popc(M);
        for (int j = 1; j <= n; ++j) {
            double bv = 0.0;
            int bsec = 0x7fffffff, bsrc = -1;
            if (pc >= 1 && pc <= j) {
                for (int i = g; i < j; i += G) {
                    const double* crow = cc + (size_t)dpw_pair(i, j, n) * p;
                    for (uint32_t mm = (uint32_t)M; mm; mm &= mm - 1) {
                        const int wi = __ffs(mm) - 1;
                        const int src = i * S + (M ^ (1 << wi));
                        const int32_t bk = back[src];          // all loads first: one round trip
                        const int jl = jlim[i * p + wi];
                        const double m0 = mk[src], c = crow[wi];
                        const double v = c > m0 ? c : m0;      // max(mk, chunk_cost) :316
                        const int sec = i * 64 + (63 - wi);
                        if (bk >= 0 && j < jl && (bsrc < 0 || key_less(v, sec, bv, bsec))) {
                            bv = v; bsec = sec; bsrc = (i << 8) | wi;
                        }
                    }
                }
            }
            for (int off = S; off < 32; off <<= 1) {           // combine the G lanes of this M
                const double ov = __shfl_xor_sync(0xffffffffu, bv, off);
                const int osec = __shfl_xor_sync(0xffffffffu, bsec, off);
                const int osrc = __shfl_xor_sync(0xffffffffu, bsrc, off);
                if (osrc >= 0 && (bsrc < 0 || key_less(ov, osec, bv, bsec))) { bv = ov; bsec = osec; bsrc = osrc; }
            }
            if (g == 0 && bsrc >= 0) { mk[j * S + M] = bv; back[j * S + M] = bsrc; }
            __syncwarp();
        }
        // finals: smallest (makespan, mask) among states with j == n (:321-325)
        double bv = 0.0;
        long long bm = -1;
        if (lane < S && back[n * S + lane] >= 0) { bv = mk[n * S + lane]; bm = lane; }
        for (int off = 16; off > 0; off >>= 1) {
            const double ov = __shfl_down_sync(0xffffffffu, bv, off);
            const long long om = __shfl_down_sync(0xffffffffu, bm, off);
            if (om >= 0 && (bm < 0 || ov < bv || (ov == bv && om < bm))) { bv = ov; bm = om; }
        }
        int16_t* own = out_owner + (size_t)sc * n_max;
        for (int i = lane; i < n_max; i += 32) own[i] = -1;
        __syncwarp();
        if (lane == 0) {
            if (bm >= 0) {
                int j = n;
                int M = (int)bm;
                while (j > 0) {
                    const int32_t bb = back[j * S + M];
                    const int i = bb >> 8, wi = bb & 0xff;
                    for (int s2 = i; s2 < j; ++s2) own[s2] = (int16_t)wi;
                    M &= ~(1 << wi);
                    j = i;
                }
                out_mk[sc] = bv;
                out_found[sc] = 1;
            } else {
                out_mk[sc] = __longlong_as_double(0x7ff0000000000000LL);
                out_found[sc] = 0;
            }
        }
    }
}

// ---- small fleets, latency form: one CTA of kDpCtaWarps warps per scenario
//      (the same tables and pull-form key as subset_dp_warp_kernel), so a
//      batch that does not fill the GPU (the C1 link grid: 1024 DPs) finishes
//      each DP with 4x the lanes: chunk costs and _fits break points one
//      (i, worker) pair per thread, each warp reducing a quarter of the target
//      masks of a level, one __syncthreads between levels.
constexpr int kDpCtaWarps = 4;

__global__ void __launch_bounds__(32 * kDpCtaWarps) subset_dp_cta_kernel(const dm_tables* __restrict__ tables,
                                                                         int32_t n_scen, int32_t n_max,
                                                                         int32_t p_max, int32_t e_max,
                                                                         int16_t* out_owner, double* out_mk,
                                                                         int32_t* out_found) {
    extern __shared__ __align__(16) unsigned char dsm[];
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5, T = blockDim.x;
    for (int sc = blockIdx.x; sc < n_scen; sc += gridDim.x) {
        __syncthreads();
        const dm_tables tg = tables[sc];
        const int n = tg.n, p = tg.p, S = 1 << p, n1 = n + 1, E = tg.n_edges;
        unsigned char* b = dsm;
        double* cc = reinterpret_cast<double*>(b); b += align_up((size_t)n * n1 / 2 * p * 8);
        double* mk = reinterpret_cast<double*>(b); b += align_up((size_t)n1 * S * 8);
        int32_t* back = reinterpret_cast<int32_t*>(b); b += align_up((size_t)n1 * S * 4);
        int16_t* jlim = reinterpret_cast<int16_t*>(b); b += align_up((size_t)n1 * p * 2);
        // stage the columns (as dpw_stage, CTA-wide)
        dm_tables t = tg;
        {
            int64_t* pre = reinterpret_cast<int64_t*>(b); b += align_up(4 * (size_t)n1 * 8);
            double* col = reinterpret_cast<double*>(b); b += align_up(4 * (size_t)n * 8);
            int32_t* eptr = reinterpret_cast<int32_t*>(b); b += align_up((size_t)n1 * 4);
            int32_t* esrc = reinterpret_cast<int32_t*>(b); b += align_up((size_t)e_max * 4);
            double* em = reinterpret_cast<double*>(b); b += align_up((size_t)e_max * 8);
            double* peer = reinterpret_cast<double*>(b);
            for (int i = tid; i < n1; i += T) {
                pre[i] = tg.pre_flops[i]; pre[n1 + i] = tg.pre_gpu[i]; pre[2 * n1 + i] = tg.pre_cpu[i];
                pre[3 * n1 + i] = tg.pre_disk[i]; eptr[i] = tg.edge_ptr[i];
            }
            for (int i = tid; i < n; i += T) {
                col[i] = tg.flops[i]; col[n + i] = tg.gpu[i]; col[2 * n + i] = tg.cpu[i]; col[3 * n + i] = tg.disk[i];
            }
            const bool stage_edges = E <= e_max;
            if (stage_edges)
                for (int e = tid; e < E; e += T) { esrc[e] = tg.edge_src[e]; em[e] = tg.edge_m[e]; }
            for (int w = tid; w < p; w += T) {
                peer[w] = tg.speed[w]; peer[p + w] = tg.cap_gpu[w]; peer[2 * p + w] = tg.cap_cpu[w];
                peer[3 * p + w] = tg.cap_disk[w];
            }
            t.pre_flops = pre; t.pre_gpu = pre + n1; t.pre_cpu = pre + 2 * n1; t.pre_disk = pre + 3 * n1;
            t.flops = col; t.gpu = col + n; t.cpu = col + 2 * n; t.disk = col + 3 * n;
            t.edge_ptr = eptr;
            if (stage_edges) { t.edge_src = esrc; t.edge_m = em; }
            t.speed = peer; t.cap_gpu = peer + p; t.cap_cpu = peer + 2 * p; t.cap_disk = peer + 3 * p;
        }
        __syncthreads();
        for (int it = tid; it < n * p; it += T) {              // _fits break points (:313-315)
            const int i = it / p, wi = it % p;
            int j = i + 1;
            while (j <= n && fits_range(t, wi, i, j)) ++j;
            jlim[i * p + wi] = (int16_t)j;
        }
        for (int it = tid; it < n * p; it += T) {              // chunk_cost (:294-302) per (i, worker)
            const int i = it / p, wi = it % p;
            const double speed = t.speed[wi];
            double rd = 0.0;                                    // the read grows stage by stage, in the
            for (int j = i + 1; j <= n; ++j) {                  // reference's (stage, edge) order
                if (include_comm(t))
                    for (int e = t.edge_ptr[j - 1]; e < t.edge_ptr[j]; ++e)
                        if (t.edge_src[e] < i) rd = __dadd_rn(rd, comm_time(t.def_alpha, t.def_beta, t.edge_m[e]));
                const double fl = col_range(t.flops, t.pre_flops, flops_exact(t), i, j, np_flops(t));
                cc[(size_t)dpw_pair(i, j, n) * p + wi] = fl / speed + rd;
            }
        }
        for (int it = tid; it < n1 * S; it += T) back[it] = -1;
        __syncthreads();
        if (tid == 0) { mk[0] = 0.0; back[0] = 0; }
        __syncthreads();
        // levels: warp w owns masks w*MPW .. w*MPW + MPW - 1, G lanes per mask
        const int W = T >> 5;
        const int MPW = S >= W ? S / W : 1;
        const int G = 32 / MPW;
        const int M = wid * MPW + lane / G, g = lane % G;
        const bool mvalid = M < S;
        const int pc = mvalid ? __popc(M) : 0;
        for (int j = 1; j <= n; ++j) {
            double bv = __longlong_as_double(0x7ff0000000000000LL);
            int bsec = 0x7fffffff, bsrc = -1;
            if (mvalid && pc >= 1 && pc <= j) {
                // a lane visits its sources in key order (i ascending, then
                // worker descending), so within the lane the first strict
                // minimum of the value alone is the key minimum; source values
                // are finite, so the +inf start admits the first valid one
                for (int i = g; i < j; i += G) {
                    const double* crow = cc + (size_t)dpw_pair(i, j, n) * p;
                    for (uint32_t mm = (uint32_t)M; mm; ) {
                        const int wi = 31 - __clz(mm);
                        mm ^= 1u << wi;
                        const int src = i * S + (M ^ (1 << wi));
                        const int32_t bk = back[src];
                        const int jl = jlim[i * p + wi];
                        const double m0 = mk[src], c = crow[wi];
                        const double v = c > m0 ? c : m0;      // max(mk, chunk_cost) :316
                        if (bk >= 0 && j < jl && v < bv) { bv = v; bsrc = (i << 8) | wi; }
                    }
                }
                if (bsrc >= 0) bsec = (bsrc >> 8) * 64 + (63 - (bsrc & 0xff));
            }
            for (int off = 1; off < G; off <<= 1) {             // combine the G lanes of this mask
                const double ov = __shfl_xor_sync(0xffffffffu, bv, off);
                const int osec = __shfl_xor_sync(0xffffffffu, bsec, off);
                const int osrc = __shfl_xor_sync(0xffffffffu, bsrc, off);
                if (osrc >= 0 && (bsrc < 0 || key_less(ov, osec, bv, bsec))) { bv = ov; bsec = osec; bsrc = osrc; }
            }
            if (mvalid && g == 0 && bsrc >= 0) { mk[j * S + M] = bv; back[j * S + M] = bsrc; }
            __syncthreads();
        }
        if (wid == 0) {                                      // finals (:321-325), traceback
            double bv = 0.0;
            long long bm = -1;
            if (lane < S && back[n * S + lane] >= 0) { bv = mk[n * S + lane]; bm = lane; }
            for (int off = 16; off > 0; off >>= 1) {
                const double ov = __shfl_down_sync(0xffffffffu, bv, off);
                const long long om = __shfl_down_sync(0xffffffffu, bm, off);
                if (om >= 0 && (bm < 0 || ov < bv || (ov == bv && om < bm))) { bv = ov; bm = om; }
            }
            int16_t* own = out_owner + (size_t)sc * n_max;
            for (int i = lane; i < n_max; i += 32) own[i] = -1;
            __syncwarp();
            if (lane == 0) {
                if (bm >= 0) {
                    int j = n;
                    int Mm = (int)bm;
                    while (j > 0) {
                        const int32_t bb = back[j * S + Mm];
                        const int i = bb >> 8, wi = bb & 0xff;
                        for (int s2 = i; s2 < j; ++s2) own[s2] = (int16_t)wi;
                        Mm &= ~(1 << wi);
                        j = i;
                    }
                    out_mk[sc] = bv;
                    out_found[sc] = 1;
                } else {
                    out_mk[sc] = __longlong_as_double(0x7ff0000000000000LL);
                    out_found[sc] = 0;
                }
            }
        }
    }
}

}  // namespace dm

extern "C" {

int64_t dm_subset_dp_scratch_bytes(int32_t n_max, int32_t p_max, int32_t n_scen) {
    if (n_max <= 0 || p_max <= 0 || p_max > 24) return -1;
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    int64_t grid = (int64_t)sms * 4;
    if (grid > n_scen) grid = n_scen;
    return (int64_t)dm::dp_scratch_bytes(n_max, p_max) * grid;
}

int dm_subset_dp(const dm_tables* tables, int32_t n_scen, int32_t n_max, int32_t p_max, int16_t* out_owner,
                 double* out_makespan, int32_t* out_found, void* scratch, void* stream) {
    if (!tables || n_scen < 0 || n_max <= 0 || p_max <= 0 || !out_owner || !out_makespan || !out_found || !scratch)
        return dmabi::fail(DM_E_ARG, "dm_subset_dp: bad arguments");
    if (p_max > 24) return dmabi::fail(DM_E_TOO_LARGE, "dm_subset_dp: at most 24 workers");
    if (n_scen == 0) return DM_OK;
    {   // small fleets: one warp per scenario
        const int e_max = 4 * n_max;      // staged edge capacity (larger DAGs read edges from global)
        const size_t per_cta = dm::dpw_bytes(n_max, p_max, e_max) * dm::kDpWarps;
        const char* dis = std::getenv("DM_DISABLE_DP_WARP");
        if (p_max <= 5 && per_cta <= 100 * 1024 && !(dis && dis[0] && dis[0] != '0')) {
            int dev = 0, sms = 148;
            cudaGetDevice(&dev);
            cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);

            // a batch too small to fill the GPU with one warp per DP (the C1
            // link grid) runs one 4-warp CTA per DP: shorter per-DP latency
            const size_t per_dp = dm::dpw_bytes(n_max, p_max, e_max);
            const char* cta = std::getenv("DM_DP_CTA");
            const bool use_cta = cta ? cta[0] == '1' : (int64_t)n_scen * dm::kDpCtaWarps <= (int64_t)sms * 32;
            if (use_cta) {
                const int per_sm_c = (int)((220 * 1024) / (per_dp + 1024));
                int64_t gridc = n_scen;
                if (gridc > (int64_t)sms * per_sm_c) gridc = (int64_t)sms * per_sm_c;
                cudaFuncSetAttribute(dm::subset_dp_cta_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)per_dp);
                dm::subset_dp_cta_kernel<<<(int)gridc, 32 * dm::kDpCtaWarps, per_dp, (cudaStream_t)stream>>>(
                    tables, n_scen, n_max, p_max, e_max, out_owner, out_makespan, out_found);
                DM_CHECK_LAUNCH();
                return DM_OK;
            }
            int64_t grid = (n_scen + dm::kDpWarps - 1) / dm::kDpWarps;
            const int per_sm = (int)((220 * 1024) / (per_cta + 1024));
            if (grid > (int64_t)sms * per_sm * 4) grid = (int64_t)sms * per_sm * 4;
            cudaFuncSetAttribute(dm::subset_dp_warp_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)per_cta);
            dm::subset_dp_warp_kernel<<<(int)grid, 32 * dm::kDpWarps, per_cta, (cudaStream_t)stream>>>(
                tables, n_scen, n_max, p_max, e_max, out_owner, out_makespan, out_found);
            DM_CHECK_LAUNCH();
            return DM_OK;
        }
    }
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    {   // mid-size fleets: one thread per (target mask, worker)
        const char* dis = std::getenv("DM_DISABLE_DP_LANE");
        const int e_max_l = 4 * n_max;
        const size_t smem_p = dm::dpp_smem(n_max, e_max_l);
        if (p_max <= dm::kDpLaneMaxP && p_max >= 2 && n_max < 128 && smem_p <= 220 * 1024 &&
            !(dis && dis[0] && dis[0] != '0')) {
            int64_t grid = (int64_t)sms;
            if (grid > n_scen) grid = n_scen;
            cudaFuncSetAttribute(dm::subset_dp_pair_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_p);
            dm::subset_dp_pair_kernel<<<(int)grid, dm::kDpPairThreads, smem_p, (cudaStream_t)stream>>>(
                tables, n_scen, n_max, e_max_l, out_owner, out_makespan, out_found, (unsigned char*)scratch,
                dm::dp_scratch_bytes(n_max, p_max));
            DM_CHECK_LAUNCH();
            return DM_OK;
        }
    }
    const size_t n1 = (size_t)n_max + 1;
    const size_t st = dm::align_up((n1 << p_max) * 8) + dm::align_up((n1 << p_max) * 4) + dm::align_up(n1 * p_max * 2);
    const size_t cc = n1 * n1 * p_max * 8;
    int mode = 0;
    size_t smem = 0;
    if (st + cc <= 110 * 1024) { mode = 2; smem = st + cc; }   // >= 2 CTAs per SM with every table on chip
    int per_sm = mode == 0 ? 4 : (int)((220 * 1024) / (smem + 2048));
    if (per_sm < 1) per_sm = 1;
    if (per_sm > 4) per_sm = 4;
    int64_t grid = (int64_t)sms * per_sm;
    if (grid > n_scen) grid = n_scen;
    size_t per = dm::dp_scratch_bytes(n_max, p_max);
    if (smem) cudaFuncSetAttribute(dm::subset_dp_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    dm::subset_dp_kernel<<<(int)grid, 256, smem, (cudaStream_t)stream>>>(tables, n_scen, n_max, p_max, out_owner,
                                                                          out_makespan, out_found,
                                                                          (unsigned char*)scratch, per, mode);
    DM_CHECK_LAUNCH();
    return DM_OK;
}

}  // extern "C"
