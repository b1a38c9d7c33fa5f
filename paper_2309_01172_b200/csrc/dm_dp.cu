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
        // ---- chunk_cost (:294-302): default link, edges with src < i only
        for (int it = threadIdx.x; it < n * n; it += blockDim.x) {
            int i = it / n, j = it % n + 1;
            if (j <= i) continue;
            double fl = col_range(t.flops, t.pre_flops, flops_exact(t), i, j, np_flops(t));
            double rd = 0.0;
            if (include_comm(t)) {
                for (int s = i; s < j; ++s)
                    for (int e = t.edge_ptr[s]; e < t.edge_ptr[s + 1]; ++e)
                        if (t.edge_src[e] < i) rd = __dadd_rn(rd, comm_time(t.def_alpha, t.def_beta, t.edge_m[e]));
            }
            double* row = d.cc + ((size_t)i * n1 + j) * p;
            for (int wi = 0; wi < p; ++wi) {
                double compute = fl / t.speed[wi];
                row[wi] = compute + rd;
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
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
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
