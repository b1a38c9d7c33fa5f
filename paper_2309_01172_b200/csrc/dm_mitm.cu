// dm_mitm.cu — the exhaustive identity-split sweep (the split population of
// brute_force_schedule, scheduling.py:245-278, run q on worker q) as a
// meet-in-the-middle cross product.
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
// A block is the cross product of its left and right sets, cut into tiles of
// TX elements of the larger side (8 per thread, in registers) x TY elements of
// the smaller side (shared memory, compacted to the feasible ones).  Each
// candidate of a tile costs one fp64 max and its checksum add.  The tile's
// minimum and first rank follow in closed form: the minimum over the tile is
// tm = max(min X, min Y), every pair with X_x <= tm and Y_y <= tm has
// makespan exactly tm, so the smallest rank at tm is min RX + min RY over
// those elements (ranks are recomputed only for tiles that can improve the
// incumbent).  Infeasible pairs (a run that does not fit: T = +inf) are
// counted and their +inf contributions removed from the checksum per tile.
#include "dm_common.cuh"
#include "dm_memo.cuh"
#include "dm_mitm.cuh"
#include "dm_abi_util.cuh"

namespace dm {

constexpr int kMitmThreads = 256;
constexpr int kMitmNR = 8;                           // X elements per thread (register slots)
constexpr int kMitmNY = 4;                           // Y elements built per thread
constexpr int kMitmTX = kMitmThreads * kMitmNR;      // 2048
constexpr int kMitmTY = kMitmThreads * kMitmNY;      // 1024
constexpr int kMitmCtasPerSm = 2;
constexpr uint64_t kInfBits = 0x7ff0000000000000ULL;

// Shared memory: the memo tables, then the block plan (mbase[m], per-block
// m and c, tile prefix tstart), the compacted X and Y values, reduction space.
struct MitmLayout {
    MemoLayout M;
    int n_blocks;
    size_t off_mbase, off_bm, off_bc, off_tstart, off_bx, off_by, off_red, bytes;
};

__host__ __device__ inline int mitm_j(int m) { return (m + 1) >> 1; }
__host__ __device__ inline int mitm_blocks_of(int m, int W) { return m == 0 ? 1 : W - m + 1; }

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

// One side of a block: k cuts among positions lo..hi, runs q0.. between the
// boundaries start, cuts..., end.
struct Side {
    int lo, hi, k;
    int q0, i0;        // first run index, first rank-term index
    int start, end;
    bool end_term;     // the end boundary is itself a cut (left side: c)
    bool empty;        // no runs at all (left side of the m = 0 block)
    int64_t base;      // rank offset (right side: first rank with m cuts)
};

struct MitmCtx {
    int n, W, S, R1;
    const int64_t* binom;
    const int32_t* rowoff;
};

// Side elements are cut masks (bit b <-> cut at position lo + b), enumerated
// in colex order (increasing mask value): the element order inside a side is
// free because every candidate's rank is derived from its cuts.
//
// colex unrank of element idx: the largest c with C(c, z) <= idx, z = k..1.
__device__ __forceinline__ uint64_t side_first(const MitmCtx& x, const Side& d, int64_t idx) {
    uint64_t mask = 0;
    int c = d.hi - d.lo;
    for (int z = d.k; z >= 1; --z) {
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

// colex successor (Gosper): the next mask with the same popcount.
__device__ __forceinline__ uint64_t side_next(uint64_t mk) {
    const uint64_t low = mk & (0ull - mk);
    const uint64_t r = mk + low;
    return r | (((mk ^ r) >> 2) >> (__ffsll((long long)mk) - 1));
}

// max over the side's runs of T
__device__ __forceinline__ double side_val(const MitmCtx& x, const Side& d, uint64_t mk) {
    double mx = -__longlong_as_double(0x7ff0000000000000LL);
    if (d.empty) return mx;
    int prev = d.start, q = d.q0;
    while (mk) {
        const int v = d.lo + __ffsll((long long)mk) - 1;
        mk &= mk - 1;
        const double tv = lds_f64((uint32_t)x.rowoff[q * x.S + prev] + 8u * (uint32_t)v);
        mx = tv > mx ? tv : mx;
        prev = v;
        ++q;
    }
    const double tv = lds_f64((uint32_t)x.rowoff[q * x.S + prev] + 8u * (uint32_t)d.end);
    return tv > mx ? tv : mx;
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

// Elements [e0, e0 + cnt) of side d (cnt <= CNT consecutive colex indices
// per thread, warp-uniform loop): feasible values appended to buf; returns
// the minimum value.
template <int CNT>
__device__ __forceinline__ double side_chunk(const MitmCtx& x, const Side& d, int64_t e0, int cnt, double* buf,
                                             int* counter) {
    const double inf = __longlong_as_double(0x7ff0000000000000LL);
    double mn = inf;
    uint64_t mk = cnt > 0 ? side_first(x, d, e0) : 0;
#pragma unroll 1
    for (int u = 0; u < CNT; ++u) {
        const bool act = u < cnt;
        double v = inf;
        if (act) {
            if (u) mk = side_next(mk);
            v = side_val(x, d, mk);
            mn = v < mn ? v : mn;
        }
        append_if(act && v != inf, v, buf, counter);
    }
    return mn;
}

// Smallest rank among the chunk's elements with value <= tm.
__device__ __forceinline__ int64_t side_chunk_rank(const MitmCtx& x, int m, const Side& d, int64_t e0, int cnt,
                                                   double tm) {
    int64_t best = INT64_MAX;
    if (cnt <= 0) return best;
    uint64_t mk = side_first(x, d, e0);
    for (int u = 0; u < cnt; ++u) {
        if (u) mk = side_next(mk);
        if (side_val(x, d, mk) <= tm) {
            const int64_t r = side_rank(x, m, d, mk);
            best = r < best ? r : best;
        }
    }
    return best;
}

// Block (m, c) -> its two sides: left = cuts before c (the left side of the
// m = 0 block is empty), right = cuts after c.
__device__ __forceinline__ void mitm_sides(int m, int c, const int64_t* cum, const MitmCtx& x, Side& sl, Side& sr,
                                           int64_t& nl, int64_t& nr) {
    const int W = x.W;
    if (m == 0) {
        sl = Side{1, 0, 0, 0, 1, 0, 0, false, true, 0};
        sr = Side{1, W, 0, 0, 1, 0, x.n, false, false, cum[0]};
        nl = 1; nr = 1;
        return;
    }
    const int j = mitm_j(m);
    sl = Side{1, c - 1, j - 1, 0, 1, 0, c, true, false, 0};
    sr = Side{c + 1, W, m - j, j, j + 1, c, x.n, false, false, cum[m]};
    nl = x.binom[(c - 1) * x.R1 + (j - 1)];
    nr = x.binom[(W - c) * x.R1 + (m - j)];
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

__global__ void __launch_bounds__(kMitmThreads, kMitmCtasPerSm) splits_mitm_kernel(const dm_tables tp, int part,
                                                                                  int nparts, dm_winner* partial) {
    const dm_tables t = tp;   // register copy (no param-space references)
    extern __shared__ __align__(16) unsigned char sm[];
    __shared__ int s_cnt[2][2];       // [tile parity][X, Y] feasible counts
    __shared__ int s_flag[2];         // [tile parity] bit 0: an X <= best, bit 1: a Y <= best
    __shared__ double s_best;
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

    memo_build(t, L.M, sm);
    if (threadIdx.x == 0) {
        int b = 0;
        for (int m = 0; m < rmax; ++m) { mbase[m] = b; b += mitm_blocks_of(m, x.W); }
        mbase[rmax] = b;
        s_best = inf;
        s_cnt[0][0] = s_cnt[0][1] = s_cnt[1][0] = s_cnt[1][1] = 0;
        s_flag[0] = s_flag[1] = 0;
    }
    __syncthreads();
    // ---- plan: (m, c) and tiles per block, inclusive prefix in tstart[1..nb]
    for (int b = threadIdx.x; b < nb; b += blockDim.x) {
        int m = 0;
        while (m + 1 < rmax && mbase[m + 1] <= b) ++m;
        const int c = m == 0 ? 0 : mitm_j(m) + (b - mbase[m]);
        bm[b] = (uint8_t)m;
        bc[b] = (uint8_t)c;
        Side sl, sr;
        int64_t nl, nr;
        mitm_sides(m, c, cum, x, sl, sr, nl, nr);
        const int64_t nX = nl >= nr ? nl : nr, nY = nl >= nr ? nr : nl;
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
        const int m = bm[lo];
        Side sl, sr;
        int64_t nl, nr;
        mitm_sides(m, bc[lo], cum, x, sl, sr, nl, nr);
        const bool xl = nl >= nr;
        const Side sx = xl ? sl : sr, sy = xl ? sr : sl;
        const int64_t nX = xl ? nl : nr, nY = xl ? nr : nl;
        const int64_t nty = (nY + kMitmTY - 1) / kMitmTY;
        const int64_t local = g - tstart[lo];
        const int64_t x0 = (local / nty) * kMitmTX, y0 = (local % nty) * kMitmTY;
        const int nXr = (int)(nX - x0 < kMitmTX ? nX - x0 : kMitmTX);
        const int nYr = (int)(nY - y0 < kMitmTY ? nY - y0 : kMitmTY);

        // ---- both sides' feasible elements, compacted into shared memory
        const double best = s_best;
        // consecutive elements per thread, spread over as many threads as possible
        const int px = (nXr + kMitmThreads - 1) / kMitmThreads, py = (nYr + kMitmThreads - 1) / kMitmThreads;
        const int ex = threadIdx.x * px, ey = threadIdx.x * py;
        const int cx = nXr - ex < px ? nXr - ex : px;
        const int cy = nYr - ey < py ? nYr - ey : py;
        const double xmin = side_chunk<kMitmNR>(x, sx, x0 + ex, cx, bx, &s_cnt[par][0]);
        const double ymin = side_chunk<kMitmNY>(x, sy, y0 + ey, cy, by, &s_cnt[par][1]);
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
                    int64_t rx = side_chunk_rank(x, m, sx, x0 + ex, cx, tm);
                    int64_t ry = side_chunk_rank(x, m, sy, y0 + ey, cy, tm);
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

int launch_splits_mitm(const dm_tables& t, int part, int nparts, dm_winner* partial, int sms, cudaStream_t s) {
    if (t.n < 1 || t.n > 64 || t.p < 1) return DM_E_TOO_LARGE;
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
    if (L.bytes > 112 * 1024) return DM_E_TOO_LARGE;
    DM_CUDA(cudaFuncSetAttribute(splits_mitm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)L.bytes));
    splits_mitm_kernel<<<mitm_grid(sms), kMitmThreads, L.bytes, s>>>(t, part, nparts, partial);
    DM_CHECK_LAUNCH();
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
