// dm_mitm.cu — the exhaustive identity-split sweep (the split population of
// brute_force_schedule, scheduling.py:245-278, run q on worker q) as a
// meet-in-the-middle cross product, in ONE cooperative kernel.
//
// Splits with m cuts are grouped into blocks by the position c of cut
// j = ceil(m/2) (m = 0: one block).  Within a block a split is a pair
// (left, right) of the cuts before and after c, and
//     makespan = max(L, R)   L = max over runs 0..j-1 of T, R = max over runs j..m
//     rank     = RL + RR     the lexicographic rank is a sum of per-cut terms
//                            term_i = C(W - c_{i-1}, m-i+1) - C(W - c_i + 1, m-i+1)
// with T the memoised run-cost table (dm_memo.cuh).  max is exact and
// associative, so every makespan is bit-identical to the reference's max over
// runs; the winner key (makespan, rank) is the reference's first strict
// minimum in itertools order.
//
// Phases (grid-wide barriers between them):
//  0. T once for the grid into a global image (one entry per thread);
//  1. every CTA copies T into shared memory (+ row offsets, binomials);
//  2. side tables, one level (number of cuts) per barrier.  Left sides: the
//     k = j-1 left cuts as a colex-ordered subset of positions 1.. form
//     table L_k, and the left side of block (m, c) is its first C(c-1, j-1)
//     entries; an entry holds PV = max over the runs ending at one of its
//     cuts and its top cut, so L = max(PV, T[j-1][top][c]).  Right sides:
//     table R(m, j) over the m-j right cuts in colex order of MIRRORED
//     positions (W, W-1, ...), prefix C(W-c, m-j) for block c; an entry holds
//     SV = max over the runs starting at one of its cuts and its lowest cut,
//     so R = max(T[j][c][first], SV).  Each entry is one step of a dynamic
//     program over its top bit: L_k[e] = max(L_{k-1}[e'], T[k-1][top'][c+1]),
//     R(m, j')[e] = max(R(m, j'+1)[e'], T[j'+1][v][first']), with e' = e minus
//     the colex weight of the removed bit;
//  3. tiles of the cross products: TX elements of the larger side (registers,
//     8 per thread, compacted to the feasible ones) x TY elements of the
//     smaller side (shared memory, compacted).  Each candidate costs one fp64
//     max and its checksum add.  The tile's minimum and first rank follow in
//     closed form: the minimum over the tile is tm = max(min X, min Y), every
//     pair with X_x <= tm and Y_y <= tm has makespan exactly tm, so the
//     smallest rank at tm is min RX + min RY over those elements (ranks are
//     derived from the elements' cut masks, only for tiles that can hold the
//     incumbent).  Infeasible pairs (a run that does not fit: T = +inf) are
//     counted and their +inf contributions removed from the checksum.
#include <cooperative_groups.h>

#include "dm_common.cuh"
#include "dm_memo.cuh"
#include "dm_mitm.cuh"
#include "dm_abi_util.cuh"

namespace cg = cooperative_groups;

namespace dm {

constexpr int kMitmThreads = 256;
constexpr int kMitmNR = 8;                           // X elements per thread (register slots)
constexpr int kMitmNY = 4;                           // Y elements built per thread
constexpr int kMitmTX = kMitmThreads * kMitmNR;      // 2048
constexpr int kMitmTY = kMitmThreads * kMitmNY;      // 1024
constexpr int kMitmCtasPerSm = 2;
constexpr int kMitmMaxM = 64;
constexpr int kTableChunk = 8;
constexpr uint64_t kInfBits = 0x7ff0000000000000ULL;

__host__ __device__ inline int mitm_j(int m) { return (m + 1) >> 1; }
__host__ __device__ inline int mitm_blocks_of(int m, int W) { return m == 0 ? 1 : W - m + 1; }
// table levels k = 0 .. floor((rmax-1)/2); left tables exist for k <= j(rmax-1) - 1
__host__ __device__ inline int tab_levels(int rmax) { return rmax >= 2 ? (rmax - 1) / 2 + 1 : 0; }
__host__ __device__ inline int tab_kl(int rmax) { return rmax >= 2 ? mitm_j(rmax - 1) - 1 : -1; }

// Relative double index of T[q][a][0] in the memo layout (dm_memo.cuh).
__host__ __device__ inline int memo_row(int q, int a, int n) {
    int base = 0;
    for (int qq = 0; qq < q; ++qq) { const int Lq = n - qq; base += Lq * (Lq + 1) / 2; }
    return base + (a - q) * n - ((a - q) * (a + q - 1)) / 2 - (a + 1);
}

// Shared memory: the memo tables, the block plan (mbase[m], per-block m and
// c, tile prefix tstart), the compacted X and Y values, reduction space.
struct MitmLayout {
    MemoLayout M;
    int n_blocks;
    size_t off_mbase, off_bm, off_bc, off_tstart, off_bx, off_by, off_red, bytes;
};

__host__ __device__ inline MitmLayout mitm_layout(int n, int p) {
    MitmLayout L;
    L.M = memo_layout(n, p);
    const int rmax = L.M.rmax, W = n - 1;
    int nb = 0;
    for (int m = 0; m < rmax; ++m) nb += mitm_blocks_of(m, W);
    L.n_blocks = nb;
    size_t off = L.M.off_tail;
    L.off_mbase = off; off += (size_t)(rmax + 1) * 4;
    L.off_tstart = off; off += (size_t)(nb + 1) * 4;
    L.off_bm = off; off += (size_t)nb;
    L.off_bc = off; off += (size_t)nb;
    off = (off + 15) & ~(size_t)15;
    L.off_bx = off; off += (size_t)kMitmTX * 8;
    L.off_by = off; off += (size_t)kMitmTY * 8;
    L.off_red = off; off += 64 * 8;
    L.bytes = off;
    return L;
}

// Global workspace: T image, then the side-table values and boundary bytes.
struct MitmWorkspace {
    size_t off_val, off_bnd, bytes;
    int64_t entries;
};

__host__ inline bool mitm_workspace(int n, int p, MitmWorkspace& ws) {
    const int W = n - 1, rmax = n < p ? n : p;
    if (rmax > kMitmMaxM) return false;
    auto C = [](int a, int b) -> unsigned __int128 {
        if (b < 0 || b > a) return 0;
        unsigned __int128 r = 1;
        for (int i = 1; i <= b; ++i) r = r * (unsigned __int128)(a - b + i) / (unsigned __int128)i;
        return r;
    };
    unsigned __int128 e = 0;
    const int NL = tab_levels(rmax), KL = tab_kl(rmax);
    for (int k = 0; k < NL; ++k) {
        if (k <= KL) e += C(W - k - 1, k);
        for (int m = 1; m < rmax; ++m)
            if (k <= m - mitm_j(m)) e += C(W - m + k, k);
    }
    if (e > ((unsigned __int128)1 << 36)) return false;
    ws.entries = (int64_t)e;
    const size_t timg = (size_t)memo_layout(n, p).t_elems * 8;
    ws.off_val = (timg + 255) & ~(size_t)255;
    ws.off_bnd = ws.off_val + (((size_t)ws.entries * 8 + 255) & ~(size_t)255);
    ws.bytes = ws.off_bnd + (((size_t)ws.entries + 255) & ~(size_t)255);
    return true;
}

// One side of a block for rank derivation: k cuts among positions lo..hi
// (bit b <-> position lo + b), rank terms i0.. between the boundaries start,
// cuts..., end.
struct Side {
    int lo, hi, k;
    int q0, i0;
    int start, end;
    bool end_term;     // the end boundary is itself a cut (left side: c)
    bool empty;        // no cuts and no runs (left side of the m = 0 block)
    int64_t base;      // rank offset (right side: first rank with m cuts)
};

struct MitmCtx {
    int n, W, S, R1;
    const int64_t* binom;
    const int32_t* rowoff;
};

__device__ __forceinline__ double tval(const MitmCtx& x, int q, int a, int b) {
    return lds_f64((uint32_t)x.rowoff[q * x.S + a] + 8u * (uint32_t)b);
}

// colex unrank of element idx among the k-subsets of bit positions 0..P-1:
// the largest c with C(c, z) <= idx, z = k..1.
__device__ __forceinline__ uint64_t colex_unrank(const MitmCtx& x, int k, int P, int64_t idx) {
    uint64_t mask = 0;
    int c = P - 1;
    for (int z = k; z >= 1; --z) {
        int64_t b;
        while ((b = x.binom[c * x.R1 + z]) > idx) --c;
#ifdef DM_MITM_CHECK
        if (c < z - 1) { printf("MITM colex unrank oob c=%d z=%d\n", c, z); __trap(); }
#endif
        mask |= 1ull << c;
        idx -= b;
        --c;
    }
    return mask;
}

// the side's share of the global rank: sum of term_i over its cuts
__device__ __forceinline__ int64_t side_rank(const MitmCtx& x, int m, const Side& d, uint64_t mk) {
    int64_t r = d.base;
    if (d.empty) return r;
    int prev = d.start, i = d.i0;
    while (mk) {
        const int v = d.lo + __ffsll((long long)mk) - 1;
        mk &= mk - 1;
        const int kk = m - i + 1;
        r += x.binom[(x.W - prev) * x.R1 + kk] - x.binom[(x.W - v + 1) * x.R1 + kk];
        prev = v;
        ++i;
    }
    if (d.end_term) {
        const int kk = m - i + 1;
        r += x.binom[(x.W - prev) * x.R1 + kk] - x.binom[(x.W - d.end + 1) * x.R1 + kk];
    }
    return r;
}

// Warp-aggregated append of v to buf when keep (shared counter *cnt).
__device__ __forceinline__ void append_if(bool keep, double v, double* buf, int* cnt) {
    const unsigned bal = __ballot_sync(0xffffffffu, keep);
    if (!bal) return;
    const int lane = threadIdx.x & 31;
    int base = 0;
    if (lane == __ffs(bal) - 1) base = atomicAdd(cnt, __popc(bal));
    base = __shfl_sync(0xffffffffu, base, __ffs(bal) - 1);
    if (keep) buf[base + __popc(bal & ((1u << lane) - 1u))] = v;
}



// largest b in [k-1, maxb] with C(b, k) <= e (k >= 1)
__device__ __forceinline__ int top_bit(const MitmCtx& x, int k, int maxb, int64_t e) {
    int lo = k - 1, hi = maxb;
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (x.binom[mid * x.R1 + k] <= e) lo = mid; else hi = mid - 1;
    }
    return lo;
}

// ---- phase 0: T entry i of the flat (q, a, b) range into the global image
__device__ __forceinline__ void memo_image_entry(const dm_tables& t, int rmax, int64_t i, double* timg) {
    const int n = t.n;
    const int q = (int)(i / ((int64_t)n * n)), a = (int)((i / n) % n), b = (int)(i % n) + 1;
    if (q >= rmax || a < q || b <= a) return;
    double v = __longlong_as_double(0x7ff0000000000000LL);
    if ((q > 0 || a == 0) && fits_range(t, q, a, b)) {
        double c, rd;
        if (chain(t)) run_cost_contig(t, a, b, q, [&](int) { return q - 1; }, c, rd);
        else run_cost_contig(t, a, b, q, [&](int s) { return s < a ? -1 : q + 1; }, c, rd);
        v = c + rd;
    }
    timg[memo_row(q, a, n) + b] = v;
}

// ---- phase 1: shared copy of T, row offsets, the -inf row, binomials
//      (Pascal's triangle in warp 0: exact for n <= 64) and cum.
__device__ inline void memo_load(const MemoLayout& L, const double* __restrict__ timg, unsigned char* sm) {
    const int n = L.n, rmax = L.rmax, S = L.S, R1 = rmax + 1;
    double* T = reinterpret_cast<double*>(sm);
    for (int i = threadIdx.x; i < L.t_elems; i += blockDim.x) T[i] = timg[i];
    int32_t* rowoff = reinterpret_cast<int32_t*>(sm + L.off_rowoff);
    const uint32_t sm_base = (uint32_t)__cvta_generic_to_shared(sm);
    for (int i = threadIdx.x; i < (rmax + 4) * S; i += blockDim.x) {
        const int q = i / S, a = i % S;
        const int32_t v = (q < rmax && a >= q && a < n) ? memo_row(q, a, n) * 8 : (int32_t)L.off_dummy;
        rowoff[i] = (int32_t)(sm_base + (uint32_t)v);
    }
    for (int i = threadIdx.x; i <= n; i += blockDim.x)
        reinterpret_cast<double*>(sm + L.off_dummy)[i] = -__longlong_as_double(0x7ff0000000000000LL);
    if (threadIdx.x < 32) {
        int64_t* binom = reinterpret_cast<int64_t*>(sm + L.off_binom);
        const int lane = threadIdx.x;
        int64_t v0 = lane == 0, v1 = 0, v2 = 0;      // row 0 at b = lane, lane + 32, lane + 64
        for (int a = 0; a < n; ++a) {
            if (a > 0) {
                const int64_t u0 = __shfl_up_sync(0xffffffffu, v0, 1), u1 = __shfl_up_sync(0xffffffffu, v1, 1),
                              u2 = __shfl_up_sync(0xffffffffu, v2, 1);
                const int64_t t0 = __shfl_sync(0xffffffffu, v0, 31), t1 = __shfl_sync(0xffffffffu, v1, 31);
                v2 += lane ? u2 : t1;
                v1 += lane ? u1 : t0;
                v0 += lane ? u0 : 0;
            }
            if (lane < R1) binom[a * R1 + lane] = v0;
            if (lane + 32 < R1) binom[a * R1 + lane + 32] = v1;
            if (lane + 64 < R1) binom[a * R1 + lane + 64] = v2;
        }
        __syncwarp();
        if (lane == 0) {
            int64_t* cum = reinterpret_cast<int64_t*>(sm + L.off_cum);
            cum[0] = 0;
            for (int m = 1; m <= rmax; ++m) cum[m] = cum[m - 1] + binom[(n - 1) * R1 + (m - 1)];
        }
    }
    __syncthreads();
}

// ---- phase 2 helpers: the tables of level k in order (L_k first when it
//      exists, then R(m, m-k) by m): sizes and chunk prefix (thread 0).
struct LevelPlan {
    int n_tab;
    int8_t tm[kMitmMaxM + 1];        // -1: L_k, else m
    int64_t ent[kMitmMaxM + 2];      // entry prefix
    int64_t chk[kMitmMaxM + 2];      // chunk prefix
};

__device__ inline void level_plan(const MitmCtx& x, int rmax, int k, LevelPlan& P) {
    const int W = x.W, KL = tab_kl(rmax);
    int nt = 0;
    P.ent[0] = P.chk[0] = 0;
    auto add = [&](int m, int64_t sz) {
        P.tm[nt] = (int8_t)m;
        P.ent[nt + 1] = P.ent[nt] + sz;
        P.chk[nt + 1] = P.chk[nt] + (sz + kTableChunk - 1) / kTableChunk;
        ++nt;
    };
    if (k <= KL) add(-1, x.binom[(W - k - 1) * x.R1 + k]);
    for (int m = 1; m < rmax; ++m)
        if (k <= m - mitm_j(m)) add(m, x.binom[(W - m + k) * x.R1 + k]);
    P.n_tab = nt;
}

// ------------------------------------------------------------- the sweep
// A block's two sides: m, c, j and table offsets; element values from the
// side tables (m = 0: the single split [0, n) as an empty left side and a
// right side without cuts).
struct Blk {
    int m, j, c;
    int64_t nl, nr, offl, offr;
    uint32_t rbase;    // shared address of T[j][c][0] (right sides)
};

__device__ __forceinline__ double left_val(const MitmCtx& x, const Blk& B, const double* val, const uint8_t* bnd,
                                           int64_t e) {
    if (B.m == 0) return -__longlong_as_double(0x7ff0000000000000LL);
    const double pv = val[B.offl + e];
    const double tv = tval(x, B.j - 1, bnd[B.offl + e], B.c);
    return tv > pv ? tv : pv;
}

__device__ __forceinline__ double right_val(const MitmCtx& x, const Blk& B, const double* val, const uint8_t* bnd,
                                            int64_t e) {
    if (B.m == 0) return lds_f64(B.rbase + 8u * (uint32_t)x.n);
    const double sv = val[B.offr + e];
    const double tv = lds_f64(B.rbase + 8u * (uint32_t)bnd[B.offr + e]);
    return tv > sv ? tv : sv;
}

// Global rank share of element e of the left / right side of B.
__device__ __forceinline__ int64_t left_rank(const MitmCtx& x, const Blk& B, int64_t e) {
    if (B.m == 0) return 0;
    const Side d{1, B.c - 1, B.j - 1, 0, 1, 0, B.c, true, false, 0};
    return side_rank(x, B.m, d, colex_unrank(x, d.k, B.c - 1, e));
}

__device__ __forceinline__ int64_t right_rank(const MitmCtx& x, const Blk& B, const int64_t* cum, int64_t e) {
    const int k = B.m - B.j, P = x.W - B.c;
    const Side d{B.c + 1, x.W, k, B.j, B.j + 1, B.c, x.n, false, false, cum[B.m]};
    uint64_t mk = k ? colex_unrank(x, k, P, e) : 0;            // mirrored: bit b <-> position W - b
    if (k) mk = __brevll(mk) >> (64 - P);                       // -> bit b <-> position c + 1 + b
    return side_rank(x, B.m, d, mk);
}

__device__ __forceinline__ double side_value(const MitmCtx& x, const Blk& B, bool left, const double* val,
                                             const uint8_t* bnd, int64_t e) {
    return left ? left_val(x, B, val, bnd, e) : right_val(x, B, val, bnd, e);
}

// The same from an element's already loaded table value and boundary cut.
__device__ __forceinline__ double side_finish(const MitmCtx& x, const Blk& B, bool left, double raw, int b) {
    if (B.m == 0) return left ? -__longlong_as_double(0x7ff0000000000000LL) : lds_f64(B.rbase + 8u * (uint32_t)x.n);
    const double tv = left ? tval(x, B.j - 1, b, B.c) : lds_f64(B.rbase + 8u * (uint32_t)b);
    return tv > raw ? tv : raw;
}

__device__ __forceinline__ double block_min_f64(double v, double* red) {
    for (int off = 16; off > 0; off >>= 1) {
        const double o = __shfl_xor_sync(0xffffffffu, v, off);
        v = o < v ? o : v;
    }
    __syncthreads();
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
    __syncthreads();
    v = red[0];
    for (int i = 1; i < (int)(blockDim.x >> 5); ++i) v = red[i] < v ? red[i] : v;
    return v;
}

__device__ __forceinline__ int64_t block_min_i64(int64_t v, double* red) {
    int64_t* r = reinterpret_cast<int64_t*>(red);
    for (int off = 16; off > 0; off >>= 1) {
        const int64_t o = __shfl_xor_sync(0xffffffffu, v, off);
        v = o < v ? o : v;
    }
    __syncthreads();
    if ((threadIdx.x & 31) == 0) r[threadIdx.x >> 5] = v;
    __syncthreads();
    v = r[0];
    for (int i = 1; i < (int)(blockDim.x >> 5); ++i) v = r[i] < v ? r[i] : v;
    return v;
}

__device__ __forceinline__ int block_sum_i32(int v, double* red) {
    int* r = reinterpret_cast<int*>(red);
    for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
    __syncthreads();
    if ((threadIdx.x & 31) == 0) r[threadIdx.x >> 5] = v;
    __syncthreads();
    v = 0;
    for (int i = 0; i < (int)(blockDim.x >> 5); ++i) v += r[i];
    return v;
}

// Cross product of NS register slots with the feasible Y values in shared
// memory (pairs; the pad is +inf): one max and one checksum add per pair.
template <int NS>
__device__ __forceinline__ void mitm_cross(const double (&xv)[kMitmNR], const double* by, int nyf,
                                           uint64_t (&cs)[kMitmNR]) {
    const double2* y2 = reinterpret_cast<const double2*>(by);
#pragma unroll 2
    for (int y = 0; y < (nyf >> 1); ++y) {
        const double2 yy = y2[y];
#pragma unroll
        for (int u = 0; u < NS; ++u) {
            const double a = xv[u] > yy.x ? xv[u] : yy.x;
            const double b = xv[u] > yy.y ? xv[u] : yy.y;
            cs[u] += (uint64_t)__double_as_longlong(a) + (uint64_t)__double_as_longlong(b);
        }
    }
    if (nyf & 1) {
        const double yl = by[nyf - 1];
#pragma unroll
        for (int u = 0; u < NS; ++u) cs[u] += (uint64_t)__double_as_longlong(xv[u] > yl ? xv[u] : yl);
    }
}

__global__ void __launch_bounds__(kMitmThreads, kMitmCtasPerSm) splits_sweep_kernel(
        const dm_tables tp, double* __restrict__ timg, double* __restrict__ val, uint8_t* __restrict__ bnd, int part,
        int nparts, dm_winner* partial) {
    const dm_tables t = tp;   // register copy (no param-space references)
    cg::grid_group grid = cg::this_grid();
    extern __shared__ __align__(16) unsigned char sm[];
    __shared__ int s_cnt[2][2];       // [tile parity][X, Y] feasible counts
    __shared__ int s_flag[2];         // [tile parity] bit 0: an X <= best, bit 1: a Y <= best
    __shared__ double s_best;
    __shared__ LevelPlan s_lp;
    __shared__ int64_t s_lvl;                      // first entry of the current level
    __shared__ int64_t s_roff[2][kMitmMaxM];       // R(m, m-k) entry offsets, [level parity][m]
    __shared__ int64_t s_offL[kMitmMaxM], s_offR[kMitmMaxM];
    const int n = t.n;
    const MitmLayout L = mitm_layout(n, t.p);
    const int rmax = L.M.rmax, nb = L.n_blocks;
    const MitmCtx x{n, n - 1, L.M.S, rmax + 1, reinterpret_cast<const int64_t*>(sm + L.M.off_binom),
                    reinterpret_cast<const int32_t*>(sm + L.M.off_rowoff)};
    const int64_t* cum = reinterpret_cast<const int64_t*>(sm + L.M.off_cum);
    int32_t* mbase = reinterpret_cast<int32_t*>(sm + L.off_mbase);
    int32_t* tstart = reinterpret_cast<int32_t*>(sm + L.off_tstart);
    uint8_t* bm = sm + L.off_bm;
    uint8_t* bc = sm + L.off_bc;
    double* bx = reinterpret_cast<double*>(sm + L.off_bx);
    double* by = reinterpret_cast<double*>(sm + L.off_by);
    double* red = reinterpret_cast<double*>(sm + L.off_red);
    const double inf = __longlong_as_double(0x7ff0000000000000LL);
    const int64_t gtid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t gthreads = (int64_t)gridDim.x * blockDim.x;

    // ---- phase 0: T image
    for (int64_t i = gtid; i < (int64_t)rmax * n * n; i += gthreads) memo_image_entry(t, rmax, i, timg);
    grid.sync();
    // ---- phase 1: shared T, binomials
    memo_load(L.M, timg, sm);

    // ---- phase 2: side tables, level by level
    const int NL = tab_levels(rmax), KL = tab_kl(rmax);
    int64_t lvl_base = 0, prev_base = 0;   // first entries of levels k and k-1
    for (int k = 0; k < NL; ++k) {
        if (threadIdx.x == 0) {
            level_plan(x, rmax, k, s_lp);
            s_lvl = lvl_base;
            for (int i = 0; i < s_lp.n_tab; ++i) {
                const int m = s_lp.tm[i];
                const int64_t off = lvl_base + s_lp.ent[i];
                if (m < 0) {
                    for (int mm = 1; mm < rmax; ++mm) if (mitm_j(mm) - 1 == k) s_offL[mm] = off;
                } else {
                    s_roff[k & 1][m] = off;
                    if (k == m - mitm_j(m)) s_offR[m] = off;
                }
            }
        }
        __syncthreads();
        const int64_t nchunks = s_lp.chk[s_lp.n_tab];
        for (int64_t ch = gtid; ch < nchunks; ch += gthreads) {
            int lo = 0, hi = s_lp.n_tab - 1;
            while (lo < hi) {
                const int mid = (lo + hi + 1) >> 1;
                if (s_lp.chk[mid] <= ch) lo = mid; else hi = mid - 1;
            }
            const int m = s_lp.tm[lo];
            const int64_t e0 = (ch - s_lp.chk[lo]) * kTableChunk;
            const int64_t size = s_lp.ent[lo + 1] - s_lp.ent[lo];
            const int cnt = (int)(size - e0 < kTableChunk ? size - e0 : kTableChunk);
            const int64_t dst = s_lvl + s_lp.ent[lo];
            if (k == 0) {                                   // no cuts: L_0 = (-inf, 0), R(m, m) = (-inf, n)
                val[dst] = -inf;
                bnd[dst] = (uint8_t)(m < 0 ? 0 : n);
                continue;
            }
            const int jp = m < 0 ? 0 : m - k;              // R(m, jp)
            const int maxb = m < 0 ? x.W - k - 2 : x.W - jp - 1;
            // the chunk's entries: top bits and source indices, then all
            // source loads in flight, then the T lookups and stores
            const int64_t sbase = m < 0 ? prev_base : s_roff[(k - 1) & 1][m];
            int bs[kTableChunk];
            int64_t src[kTableChunk];
            int b = top_bit(x, k, maxb, e0);
#pragma unroll
            for (int u = 0; u < kTableChunk; ++u) {
                const int64_t e = e0 + u;
                if (u < cnt) while (b < maxb && x.binom[(b + 1) * x.R1 + k] <= e) ++b;
                bs[u] = b;
                src[u] = sbase + (e - x.binom[b * x.R1 + k]);
            }
            double sv[kTableChunk];
            int sb[kTableChunk];
#pragma unroll
            for (int u = 0; u < kTableChunk; ++u) {
                if (u < cnt) { sv[u] = val[src[u]]; sb[u] = bnd[src[u]]; }
            }
#pragma unroll
            for (int u = 0; u < kTableChunk; ++u) {
                if (u >= cnt) break;
                double tv;
                int nb8;
                if (m < 0) {                    // L_k: the top cut (position b + 1) extends L_{k-1}
                    nb8 = bs[u] + 1;
                    tv = tval(x, k - 1, sb[u], nb8);
                } else {                        // R(m, jp): the first cut (position W - b) extends R(m, jp+1)
                    nb8 = x.W - bs[u];
                    tv = tval(x, jp + 1, nb8, sb[u]);
                }
                val[dst + e0 + u] = tv > sv[u] ? tv : sv[u];
                bnd[dst + e0 + u] = (uint8_t)nb8;
            }
        }
        prev_base = lvl_base;
        lvl_base += s_lp.ent[s_lp.n_tab];
        __syncthreads();        // s_lp reuse
        grid.sync();
    }

    // ---- phase 3: tiles
    if (threadIdx.x == 0) {
        int b = 0;
        for (int m = 0; m < rmax; ++m) { mbase[m] = b; b += mitm_blocks_of(m, x.W); }
        mbase[rmax] = b;
        s_best = inf;
        s_cnt[0][0] = s_cnt[0][1] = s_cnt[1][0] = s_cnt[1][1] = 0;
        s_flag[0] = s_flag[1] = 0;
    }
    __syncthreads();
    auto block_of = [&](int b, int m, int c) {
        Blk B;
        B.m = m; B.c = c; B.j = m == 0 ? 0 : mitm_j(m);
        if (m == 0) { B.nl = 1; B.nr = 1; B.offl = B.offr = 0; }
        else {
            B.nl = x.binom[(c - 1) * x.R1 + (B.j - 1)];
            B.nr = x.binom[(x.W - c) * x.R1 + (m - B.j)];
            B.offl = s_offL[m]; B.offr = s_offR[m];
        }
        B.rbase = (uint32_t)x.rowoff[B.j * x.S + c];
        return B;
    };
    // ---- plan: (m, c) and tiles per block, inclusive prefix in tstart[1..nb]
    for (int b = threadIdx.x; b < nb; b += blockDim.x) {
        int m = 0;
        while (m + 1 < rmax && mbase[m + 1] <= b) ++m;
        const int c = m == 0 ? 0 : mitm_j(m) + (b - mbase[m]);
        bm[b] = (uint8_t)m;
        bc[b] = (uint8_t)c;
        const Blk B = block_of(b, m, c);
        const int64_t nX = B.nl >= B.nr ? B.nl : B.nr, nY = B.nl >= B.nr ? B.nr : B.nl;
        tstart[b + 1] = (int32_t)(((nX + kMitmTX - 1) / kMitmTX) * ((nY + kMitmTY - 1) / kMitmTY));
    }
    __syncthreads();
    if (threadIdx.x < 32) {
        const int lane = threadIdx.x, per = (nb + 31) / 32;
        const int b0 = lane * per, b1 = b0 + per < nb ? b0 + per : nb;
        int s = 0;
        for (int b = b0; b < b1; ++b) s += tstart[b + 1];
        int incl = s;
        for (int off = 1; off < 32; off <<= 1) {
            const int o = __shfl_up_sync(0xffffffffu, incl, off);
            if (lane >= off) incl += o;
        }
        int run = incl - s;
        for (int b = b0; b < b1; ++b) { run += tstart[b + 1]; tstart[b + 1] = run; }
        if (lane == 0) tstart[0] = 0;
    }
    __syncthreads();
    const int n_tiles = tstart[nb];

    Win w;
    win_init(w);
    uint64_t cs[kMitmNR];
#pragma unroll
    for (int u = 0; u < kMitmNR; ++u) cs[u] = 0;
    uint64_t corr = 0;   // +inf contributions to remove (counted in units of kInfBits)

    int par = 0;
    for (int g = part + nparts * blockIdx.x; g < n_tiles; g += nparts * gridDim.x, par ^= 1) {
        int lo = 0, hi = nb - 1;
        while (lo < hi) {
            const int mid = (lo + hi + 1) >> 1;
            if (tstart[mid] <= g) lo = mid; else hi = mid - 1;
        }
        const Blk B = block_of(lo, bm[lo], bc[lo]);
        const bool xl = B.nl >= B.nr;
        const int64_t nX = xl ? B.nl : B.nr, nY = xl ? B.nr : B.nl;
        const int64_t nty = (nY + kMitmTY - 1) / kMitmTY;
        const int64_t local = g - tstart[lo];
        const int64_t x0 = (local / nty) * kMitmTX, y0 = (local % nty) * kMitmTY;
        const int nXr = (int)(nX - x0 < kMitmTX ? nX - x0 : kMitmTX);
        const int nYr = (int)(nY - y0 < kMitmTY ? nY - y0 : kMitmTY);

        // ---- both sides' feasible elements, compacted into shared memory
        const double best = s_best;
        // element raw data (table value, boundary cut) for every slot first,
        // so all global loads are in flight together
        const int64_t xoff = xl ? B.offl : B.offr, yoff = xl ? B.offr : B.offl;
        double xr[kMitmNR], yr[kMitmNY];
        int xb[kMitmNR], yb[kMitmNY];
#pragma unroll
        for (int u = 0; u < kMitmNR; ++u) {
            const int e = u * kMitmThreads + threadIdx.x;
            if (e < nXr && B.m) { xr[u] = val[xoff + x0 + e]; xb[u] = bnd[xoff + x0 + e]; }
        }
#pragma unroll
        for (int u = 0; u < kMitmNY; ++u) {
            const int e = u * kMitmThreads + threadIdx.x;
            if (e < nYr && B.m) { yr[u] = val[yoff + y0 + e]; yb[u] = bnd[yoff + y0 + e]; }
        }
        double xmin = inf, ymin = inf;
#pragma unroll
        for (int u = 0; u < kMitmNR; ++u) {
            const int e = u * kMitmThreads + threadIdx.x;
            double v = inf;
            if (e < nXr) { v = side_finish(x, B, xl, xr[u], xb[u]); xmin = v < xmin ? v : xmin; }
            append_if(v != inf, v, bx, &s_cnt[par][0]);
        }
#pragma unroll
        for (int u = 0; u < kMitmNY; ++u) {
            const int e = u * kMitmThreads + threadIdx.x;
            double v = inf;
            if (e < nYr) { v = side_finish(x, B, !xl, yr[u], yb[u]); ymin = v < ymin ? v : ymin; }
            append_if(v != inf, v, by, &s_cnt[par][1]);
        }
        const int fl = (xmin <= best ? 1 : 0) | (ymin <= best ? 2 : 0);
        if (fl) atomicOr(&s_flag[par], fl);
        __syncthreads();
        const int nxf_tot = s_cnt[par][0], nyf = s_cnt[par][1];
        const bool maybe_best = s_flag[par] == 3;
        if (threadIdx.x == 0) {       // the other parity's slots are free until the end barrier
            s_cnt[par ^ 1][0] = s_cnt[par ^ 1][1] = 0;
            s_flag[par ^ 1] = 0;
            w.n_eval += (int64_t)nXr * nYr;
            w.n_feas += (int64_t)nxf_tot * nyf;
        }
        if (nxf_tot > 0 && nyf > 0) {     // uniform
            const int nsl = (nxf_tot + kMitmThreads - 1) / kMitmThreads;
            double xv[kMitmNR];
            int nxf = 0;
#pragma unroll
            for (int u = 0; u < kMitmNR; ++u) {
                const int e = u * kMitmThreads + threadIdx.x;
                xv[u] = e < nxf_tot ? bx[e] : inf;
                nxf += e < nxf_tot;
            }
            // ---- cross product: one max + checksum add per candidate
            switch (nsl) {
                case 1: mitm_cross<1>(xv, by, nyf, cs); break;
                case 2: mitm_cross<2>(xv, by, nyf, cs); break;
                case 3: mitm_cross<3>(xv, by, nyf, cs); break;
                case 4: mitm_cross<4>(xv, by, nyf, cs); break;
                case 5: mitm_cross<5>(xv, by, nyf, cs); break;
                case 6: mitm_cross<6>(xv, by, nyf, cs); break;
                case 7: mitm_cross<7>(xv, by, nyf, cs); break;
                default: mitm_cross<8>(xv, by, nyf, cs); break;
            }
            corr += (uint64_t)(nsl - nxf) * (uint64_t)nyf;
            // ---- rare: the tile can hold the incumbent. Its minimum is
            //      tm = max(min X, min Y); the first rank at tm is the sum of
            //      the smallest ranks of the elements at or below tm.
            if (maybe_best) {
                const double txmin = block_min_f64(xmin, red);
                const double tymin = block_min_f64(ymin, red);
                const double tm = txmin > tymin ? txmin : tymin;
                if (tm <= best) {
                    int64_t rx = INT64_MAX, ry = INT64_MAX;
                    for (int e = threadIdx.x; e < nXr; e += kMitmThreads) {
                        if (side_value(x, B, xl, val, bnd, x0 + e) <= tm) {
                            const int64_t r = xl ? left_rank(x, B, x0 + e) : right_rank(x, B, cum, x0 + e);
                            rx = r < rx ? r : rx;
                        }
                    }
                    for (int e = threadIdx.x; e < nYr; e += kMitmThreads) {
                        if (side_value(x, B, !xl, val, bnd, y0 + e) <= tm) {
                            const int64_t r = xl ? right_rank(x, B, cum, y0 + e) : left_rank(x, B, y0 + e);
                            ry = r < ry ? r : ry;
                        }
                    }
                    rx = block_min_i64(rx, red);
                    ry = block_min_i64(ry, red);
                    if (threadIdx.x == 0 && win_better(tm, rx + ry, w.mk, w.rank)) {
                        w.mk = tm;
                        w.rank = rx + ry;
                        s_best = tm;
                    }
                }
            }
        }
        __syncthreads();   // buffers, counters and s_best for the next tile
    }
    uint64_t c = 0;
#pragma unroll
    for (int u = 0; u < kMitmNR; ++u) c += cs[u];
    w.csum = c - corr * kInfBits;
    block_reduce_win_store(w, partial);
}

// Roofline denominator of the sweep: the cross-product inner loop alone
// (mitm_cross<kMitmNR> over kMitmTY shared-memory values, same grid shape and
// occupancy as the sweep, no element construction, barriers or tile
// bookkeeping).  pairs = grid * threads * kMitmNR * kMitmTY * iters.
__global__ void __launch_bounds__(kMitmThreads, kMitmCtasPerSm) cross_peak_kernel(int iters, uint64_t* sink) {
    __shared__ __align__(16) double ys[kMitmTY];
    for (int i = threadIdx.x; i < kMitmTY; i += blockDim.x) ys[i] = 1.0 + 1e-3 * ((i * 37) % 101);
    __syncthreads();
    double xv[kMitmNR];
    uint64_t cs[kMitmNR];
#pragma unroll
    for (int u = 0; u < kMitmNR; ++u) { xv[u] = 1.0 + 1e-3 * ((threadIdx.x + 13 * u) % 101); cs[u] = 0; }
    for (int it = 0; it < iters; ++it) mitm_cross<kMitmNR>(xv, ys, kMitmTY, cs);
    uint64_t c = 0;
#pragma unroll
    for (int u = 0; u < kMitmNR; ++u) c += cs[u];
    if (c == 42) sink[0] = c;
}

int mitm_grid(int sms) { return sms * kMitmCtasPerSm; }

int64_t mitm_workspace_bytes(const dm_tables& t) {
    if (t.n < 1 || t.n > 64 || t.p < 1 || !memo_valid(t)) return -1;
    const MitmLayout L = mitm_layout(t.n, t.p);
    if (L.bytes > 108 * 1024) return -1;
    MitmWorkspace ws;
    if (!mitm_workspace(t.n, t.p, ws)) return -1;
    return (int64_t)ws.bytes;
}

int launch_splits_mitm(const dm_tables& t, int part, int nparts, dm_winner* partial, int sms, void* ws,
                       int64_t ws_bytes, int* n_partials, cudaStream_t s) {
    const int64_t need = mitm_workspace_bytes(t);
    if (need < 0) return DM_E_TOO_LARGE;
    const MitmLayout L = mitm_layout(t.n, t.p);
    {   // tile count must fit the kernel's int32 tile indices
        const int W = t.n - 1, rmax = t.n < t.p ? t.n : t.p;
        auto C = [](int a, int b) -> unsigned __int128 {
            if (b < 0 || b > a) return 0;
            unsigned __int128 r = 1;
            for (int i = 1; i <= b; ++i) r = r * (unsigned __int128)(a - b + i) / (unsigned __int128)i;
            return r;
        };
        unsigned __int128 tiles = 1;
        for (int m = 1; m < rmax; ++m) {
            const int j = mitm_j(m);
            for (int c = j; c <= W - (m - j); ++c) {
                const unsigned __int128 nl = C(c - 1, j - 1), nr = C(W - c, m - j);
                const unsigned __int128 nX = nl >= nr ? nl : nr, nY = nl >= nr ? nr : nl;
                tiles += ((nX + kMitmTX - 1) / kMitmTX) * ((nY + kMitmTY - 1) / kMitmTY);
            }
        }
        if (tiles > (unsigned __int128)(INT32_MAX / 2)) return DM_E_TOO_LARGE;
    }
    MitmWorkspace W;
    mitm_workspace(t.n, t.p, W);
    void* buf = ws;
    const bool own = !ws || ws_bytes < need;
    if (own) DM_CUDA(cudaMallocAsync(&buf, (size_t)need, s));
    double* timg = static_cast<double*>(buf);
    double* val = reinterpret_cast<double*>(static_cast<unsigned char*>(buf) + W.off_val);
    uint8_t* bnd = static_cast<uint8_t*>(buf) + W.off_bnd;
    DM_CUDA(cudaFuncSetAttribute(splits_sweep_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)L.bytes));
    int per_sm = 0;
    DM_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, splits_sweep_kernel, kMitmThreads, L.bytes));
    if (per_sm < 1) return DM_E_TOO_LARGE;
    int grid = sms * (per_sm < kMitmCtasPerSm ? per_sm : kMitmCtasPerSm);
    dm_tables tv = t;
    void* args[] = {&tv, &timg, &val, &bnd, &part, &nparts, &partial};
    DM_CUDA(cudaLaunchCooperativeKernel((void*)splits_sweep_kernel, grid, kMitmThreads, args, L.bytes, s));
    if (own) DM_CUDA(cudaFreeAsync(buf, s));
    *n_partials = grid;
    return DM_OK;
}

}  // namespace dm

extern "C" int dm_microbench_cross(int64_t iters, uint64_t* sink, int64_t* pairs, void* stream) {
    if (iters <= 0 || iters > INT32_MAX || !sink) return dmabi::fail(DM_E_ARG, "dm_microbench_cross: bad arguments");
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int grid = dm::mitm_grid(sms);
    dm::cross_peak_kernel<<<grid, dm::kMitmThreads, 0, (cudaStream_t)stream>>>((int)iters, sink);
    DM_CHECK_LAUNCH();
    if (pairs) *pairs = (int64_t)grid * dm::kMitmThreads * dm::kMitmNR * dm::kMitmTY * iters;
    return DM_OK;
}
