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
// Launches per sweep (phase 1: 1-2, phase 2: 3-5 — or 4: 3 and 8: 4-5;
// dm_enum_splits_phase):
//  1. memo_image_kernel: T once into a global image (one entry per thread);
//  2. side_tables_kernel: the side tables, every entry evaluated directly from
//     its cut mask at full occupancy (T read through L1).  Left sides: the
//     k = j-1 left cuts as a colex-ordered subset of positions 1.. form table
//     L_k, and the left side of block (m, c) is its first C(c-1, j-1)
//     entries; an entry holds PV = max over the runs ending at one of its
//     cuts and its top cut, so L = max(PV, T[j-1][top][c]).  Right sides:
//     table R(m) over the m-j right cuts in colex order of MIRRORED positions
//     (W, W-1, ...), prefix C(W-c, m-j) for block c; an entry holds SV = max
//     over the runs starting at one of its cuts and its lowest cut, so
//     R = max(T[j][c][first], SV).  A side element then costs two loads and a
//     max in the sweep.  It also counts the finite entries per (table,
//     boundary position);
//  3. plan_kernel (one CTA): the tile order — blocks ranked by the feasible
//     pairs per tile those counts predict (an upper bound) plus the element
//     builds, so the longest tiles start first;
//  4. splits_sweep_kernel: tiles of the cross products from a dynamic queue
//     in that order: TX elements of the larger side (registers, 8 per
//     thread, compacted to the feasible ones) x TY elements of the smaller
//     side (shared memory, compacted).  Each candidate costs one fp64 max and
//     its checksum add.  The tile's minimum and first rank follow in closed
//     form: the minimum over the tile is tm = max(min X, min Y), every pair
//     with X_x <= tm and Y_y <= tm has makespan exactly tm, so the smallest
//     rank at tm is min RX + min RY over those elements (ranks are derived
//     from the elements' cut masks, only for tiles that can hold the
//     incumbent, which the CTAs share through a global atomic min).
//     Infeasible pairs (a run that does not fit: T = +inf) are counted and
//     their +inf contributions removed from the checksum;
//  5. finalize_kernel (dm_enum.cu): the CTAs' partial winners merged.
#include "dm_common.cuh"
#include "dm_memo.cuh"
#include "dm_mitm.cuh"
#include "dm_abi_util.cuh"

namespace dm {

#ifdef DM_MITM_TIMING
// phase timestamps of every CTA (globaltimer ns): debug builds only
__device__ unsigned long long g_mitm_times[1024][12];
#define MITM_MARK(i)                                                                               \
    do {                                                                                           \
        if (threadIdx.x == 0) {                                                                    \
            unsigned long long t_;                                                                 \
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                                 \
            g_mitm_times[blockIdx.x][i] = t_;                                                      \
        }                                                                                          \
    } while (0)
#define MITM_COUNT(i, v) atomicAdd(&g_mitm_times[blockIdx.x][i], (unsigned long long)(v))
// thread 0's clock in each phase of a tile: [6] elements + barrier, [7] cross
// product, [8] winner check + end barrier, [9] tiles, [10] thin tiles
#define MITM_CLK(v) long long v = clock64()
// per tile: block, clocks of thread 0 from the tile's start to its end barrier, X and Y elements
__device__ unsigned int g_mitm_tiles[1 << 16][4];
#define MITM_TILE(g, blk, a, b, nx, ny)                                                                \
    do {                                                                                           \
        if (threadIdx.x == 0 && (g) < (1 << 16)) {                                                 \
            g_mitm_tiles[g][0] = (unsigned)(blk); g_mitm_tiles[g][1] = (unsigned)((b) - (a));       \
            g_mitm_tiles[g][2] = (unsigned)(nx); g_mitm_tiles[g][3] = (unsigned)(ny);               \
        }                                                                                          \
    } while (0)
#define MITM_ACC(i, a, b) do { if (threadIdx.x == 0) g_mitm_times[blockIdx.x][i] += (unsigned long long)((b) - (a)); } while (0)
#else
#define MITM_CLK(v) do { } while (0)
#define MITM_TILE(g, blk, a, b, nx, ny) do { } while (0)
#define MITM_ACC(i, a, b) do { } while (0)
#define MITM_MARK(i) do { } while (0)
#define MITM_COUNT(i, v) do { } while (0)
#endif

constexpr int kMitmThreads = 256;
constexpr int kMitmNR = 8;                           // X elements per thread (register slots)
constexpr int kMitmNY = 8;                           // Y elements built per thread
constexpr int kMitmTX = kMitmThreads * kMitmNR;      // 2048
constexpr int kMitmTY = kMitmThreads * kMitmNY;      // 1024
constexpr int kMitmCtasPerSm = 2;
constexpr int kMitmMaxM = 64;
constexpr int kMitmMaxBlocks = 2048;                 // blocks of one sweep (size order in the launch parameters)
constexpr int kTabPass = 16;                         // side-table entries per thread and pass
constexpr int kThinY = 256;                          // blocks with a smaller side below this are "thin":
constexpr int kThinPairs = 1 << 21;                  // their tiles span ~kThinPairs pairs in rounds of kMitmTX
constexpr int kThinRounds = 8;                       // X elements, at most this many rounds per tile
constexpr int kThinRing = 512;                       // per-warp ring of a thin tile's feasible X (>= 2 x 256)
constexpr uint64_t kInfBits = 0x7ff0000000000000ULL;

__host__ __device__ inline int mitm_j(int m) { return (m + 1) >> 1; }
__host__ __device__ inline int mitm_blocks_of(int m, int W) { return m == 0 ? 1 : W - m + 1; }

// Relative double index of T[q][a][0] in the memo layout (dm_memo.cuh):
// rows of q start after sum_{qq<q} (n-qq)(n-qq+1)/2 = S3(n) - S3(n-q),
// S3(N) = N(N+1)(N+2)/6.
__host__ __device__ inline int memo_row(int q, int a, int n) {
    const int N = n - q;
    const int base = (n * (n + 1) * (n + 2) - N * (N + 1) * (N + 2)) / 6;
    return base + (a - q) * n - ((a - q) * (a + q - 1)) / 2 - (a + 1);
}

// Shared memory of the sweep: binomials and cum (the rank terms), the block
// plan (mbase[m], per block m and c, size-order position -> block, tile
// prefix tstart), the compacted X and Y values, reduction space.  The run
// costs T stay in the global image (57 KB for n = 34, L1-resident).
struct MitmLayout {
    MemoLayout M;      // sizes of the T image (rmax, t_elems); its shared offsets are not used
    int n_blocks;
    size_t off_binom, off_cum, off_mbase, off_bm, off_bc, off_pos, off_tstart, off_bx, off_by, off_red, bytes;
};

__host__ __device__ inline MitmLayout mitm_layout(int n, int p) {
    MitmLayout L;
    L.M = memo_layout(n, p);
    const int rmax = L.M.rmax, W = n - 1;
    int nb = 0;
    for (int m = 0; m < rmax; ++m) nb += mitm_blocks_of(m, W);
    L.n_blocks = nb;
    size_t off = 0;
    L.off_binom = off; off += (size_t)n * (rmax + 1) * 8;
    L.off_cum = off; off += (size_t)(rmax + 2) * 8;
    off = (off + 15) & ~(size_t)15;
    L.off_mbase = off; off += (size_t)(rmax + 1) * 4;
    L.off_tstart = off; off += (size_t)(nb + 1) * 4;
    L.off_bm = off; off += (size_t)nb;
    L.off_bc = off; off += (size_t)nb;
    off = (off + 1) & ~(size_t)1;
    L.off_pos = off; off += (size_t)nb * 2;
    off = (off + 15) & ~(size_t)15;
    L.off_bx = off; off += (size_t)(kMitmTX > kThinRing * (kMitmThreads / 32) ? kMitmTX : kThinRing * (kMitmThreads / 32)) * 8;
    L.off_by = off; off += (size_t)kMitmTY * 8;
    L.off_red = off; off += 64 * 8;
    L.bytes = off;
    return L;
}

// Side tables of one sweep (host-computed, passed by value): L_k for
// k = 0..KL, then R(m) for m = 1..rmax-1; tables the tiles read by m.
struct SideTables {
    int n_tab;
    int8_t kind[2 * kMitmMaxM];       // 0: L_k, 1: R(m)
    int8_t km[2 * kMitmMaxM];         // k for L_k, m for R(m)
    int8_t pos[2 * kMitmMaxM];        // positions the table's cuts range over
    int64_t start[2 * kMitmMaxM + 1]; // entry prefix
    int64_t offL[kMitmMaxM], offR[kMitmMaxM];
};

// Launch parameters of the sweep: table offsets by m and the block order by
// decreasing number of candidates.
struct SweepParams {
    int64_t offL[kMitmMaxM], offR[kMitmMaxM];
    int8_t tabL[kMitmMaxM], tabR[kMitmMaxM];   // histogram row of L_k / R(m) (-1: not built by this part)
    int nbp;                          // blocks of this part
    int16_t order[kMitmMaxBlocks];    // the part's blocks, largest tiles first
};

// Feasibility histogram of the side tables: finite entries per (table,
// boundary position); the sweep orders its tiles by the feasible pairs this
// predicts (an upper bound) instead of the raw tile size.
constexpr int kHistRow = 72;          // boundary positions 0..64

// Global workspace: tile counter, T image, side-table values, boundary bytes.
struct MitmWorkspace {
    size_t off_hist, off_plan, off_timg, off_val, off_bnd, bytes;
    int64_t entries;
};

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
    int n, W, R1;
    const int64_t* binom;
    const double* timg;    // the global T image (memo_row layout)
};

__device__ __forceinline__ double tval(const MitmCtx& x, int q, int a, int b) {
    return __ldg(x.timg + memo_row(q, a, x.n) + b);
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

// colex successor (Gosper): the next mask with the same popcount.
__device__ __forceinline__ uint64_t side_next(uint64_t mk) {
    const uint64_t low = mk & (0ull - mk);
    const uint64_t r = mk + low;
    return r | (((mk ^ r) >> 2) >> (__ffsll((long long)mk) - 1));
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


// ------------------------------------------------------------- the sweep
// A block's two sides: m, c, j and table offsets; element values from the
// side tables (m = 0: the single split [0, n) as an empty left side and a
// right side without cuts).
struct Blk {
    int m, j, c, R;    // R: rounds of kMitmTX X elements per tile (thin blocks)
    int64_t nl, nr, offl, offr;
    int32_t rrow;      // image index of T[j][c][0] (right sides)
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
    if (B.m == 0) return __ldg(x.timg + B.rrow + x.n);
    const double sv = val[B.offr + e];
    const double tv = __ldg(x.timg + B.rrow + bnd[B.offr + e]);
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

// A side element finished from its loaded table value and boundary cut, the
// tile's finishing runs staged in shared memory:
// col[a] = T[j-1][a][c] (left sides), row[b] = T[j][c][b] (right sides).
__device__ __forceinline__ double side_finish_s(const Blk& B, bool left, double raw, int b, const double* col,
                                                const double* row, int n) {
    if (B.m == 0) return left ? -__longlong_as_double(0x7ff0000000000000LL) : row[n];
    const double tv = left ? col[b] : row[b];
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


}  // namespace dm

#include <algorithm>
#include <array>
#include <memory>
#include <utility>
#include <vector>

namespace dm {

namespace {
unsigned __int128 binom128(int a, int b) {
    if (b < 0 || b > a) return 0;
    unsigned __int128 r = 1;
    for (int i = 1; i <= b; ++i) r = r * (unsigned __int128)(a - b + i) / (unsigned __int128)i;
    return r;
}
}  // namespace

// Positions the left table L_k ranges over: the largest left prefix any block
// reading it needs (cuts below c <= cmax(m) = W - (m - j), j = k + 1).
inline int left_positions(int W, int rmax, int k) {
    int P = 0;
    for (int m = 1; m < rmax; ++m)
        if (mitm_j(m) - 1 == k) P = std::max(P, W - (m - mitm_j(m)) - 1);
    return P;
}

// The sweep's plan for part `part` of `nparts` and its workspace layout;
// false when the sweep does not apply (more than kMitmMaxBlocks blocks, 2^36
// table entries or 2^30 tiles).
//
// Parts own whole blocks, dealt largest first to the part where the block
// adds the least load: its tiles plus the tables it reads (R(m), L_{j-1})
// when the part does not hold them yet.  Each part builds only the tables of
// its blocks, so the table phase splits across GPUs with the tiles.  Within a
// part, blocks are ordered by the estimated duration of one of their tiles
// (its pairs plus ~256 pair-equivalents per element it builds), largest
// first, for the dynamic tile queue.
inline bool mitm_plan(int n, int p, int part, int nparts, SideTables& st, MitmWorkspace& ws, SweepParams* sp) {
    const int W = n - 1, rmax = n < p ? n : p;
    if (n < 1 || n > 64 || p < 1 || rmax > kMitmMaxM || nparts < 1 || part < 0 || part >= nparts) return false;
    const MitmLayout L = mitm_layout(n, p);
    if (L.n_blocks > kMitmMaxBlocks || L.bytes > 108 * 1024) return false;
    const int nb = L.n_blocks;
    struct BlockCost { double tile, total; int m, b; };
    std::vector<BlockCost> blk(nb);
    unsigned __int128 tiles = 0;
    for (int m = 0, b = 0; m < rmax; ++m)
        for (int i = 0; i < mitm_blocks_of(m, W); ++i, ++b) {
            const int j = mitm_j(m), c = m == 0 ? 0 : j + i;
            const unsigned __int128 nl = m == 0 ? 1 : binom128(c - 1, j - 1), nr = m == 0 ? 1 : binom128(W - c, m - j);
            const unsigned __int128 nX = nl >= nr ? nl : nr, nY = nl >= nr ? nr : nl;
            unsigned __int128 R = 1;                     // thin blocks: rounds of kMitmTX X elements per tile
            if (nY < (unsigned __int128)kThinY) {
                R = (unsigned __int128)kThinPairs / ((unsigned __int128)kMitmTX * nY);
                R = R < 1 ? 1 : (R > (unsigned __int128)kThinRounds ? kThinRounds : R);
            }
            const unsigned __int128 txs = (unsigned __int128)kMitmTX * R;
            const unsigned __int128 tx = nX < txs ? nX : txs, ty = nY < kMitmTY ? nY : kMitmTY;
            const unsigned __int128 nt = ((nX + txs - 1) / txs) * ((nY + kMitmTY - 1) / kMitmTY);
            tiles += nt;
            const double tc = (double)(tx * ty + 256 * (tx + ty));
            blk[b] = {tc, tc * (double)nt, m, b};
        }
    if (tiles > ((unsigned __int128)1 << 30)) return false;
    // ---- blocks of this part
    std::vector<int> mine;
    if (nparts == 1) {
        for (int b = 0; b < nb; ++b) mine.push_back(b);
    } else {
        // m-groups (a group shares R(m) and L_{j-1}) whole to the least-loaded
        // part, largest first; a group above 3/4 of a part's share is dealt
        // block by block (LPT) and its tables are built by every part it
        // touches.  Costs: tiles plus ~270 pair-equivalents per table entry.
        std::vector<double> load(nparts, 0.0), gcost(rmax, 0.0), gtab(rmax, 0.0);
        double total = 0;
        for (const auto& x : blk) { gcost[x.m] += x.total; total += x.total; }
        for (int m = 1; m < rmax; ++m) {
            const int k = mitm_j(m) - 1;
            gtab[m] = 270.0 * (double)(binom128(W - mitm_j(m), m - mitm_j(m)) +
                                       binom128(left_positions(W, rmax, k), k));
            total += gtab[m];
        }
        std::vector<int> ms(rmax);
        for (int m = 0; m < rmax; ++m) ms[m] = m;
        std::stable_sort(ms.begin(), ms.end(),
                         [&](int a, int b) { return gcost[a] + gtab[a] > gcost[b] + gtab[b]; });
        auto least = [&]() { return (int)(std::min_element(load.begin(), load.end()) - load.begin()); };
        std::vector<int> owner(nb, 0);
        for (int m : ms) {
            std::vector<int> bs;
            for (int b = 0; b < nb; ++b) if (blk[b].m == m) bs.push_back(b);
            if (gcost[m] + gtab[m] <= 0.75 * total / nparts) {
                const int q = least();
                for (int b : bs) owner[b] = q;
                load[q] += gcost[m] + gtab[m];
            } else {
                std::vector<char> has(nparts, 0);
                std::stable_sort(bs.begin(), bs.end(), [&](int a, int b) { return blk[a].total > blk[b].total; });
                for (int b : bs) {
                    int best = 0;
                    double bl = 0;
                    for (int q = 0; q < nparts; ++q) {
                        const double l = load[q] + blk[b].total + (has[q] ? 0.0 : gtab[m]);
                        if (q == 0 || l < bl) { best = q; bl = l; }
                    }
                    owner[b] = best;
                    load[best] = bl;
                    has[best] = 1;
                }
            }
        }
        for (int b = 0; b < nb; ++b) if (owner[b] == part) mine.push_back(b);
    }
    // ---- the tables those blocks read
    std::vector<char> needR(rmax, 0), needL(rmax, 0);
    for (int b : mine) if (blk[b].m >= 1) { needR[blk[b].m] = 1; needL[mitm_j(blk[b].m) - 1] = 1; }
    unsigned __int128 e = 0;
    st.n_tab = 0;
    for (int m = 0; m < kMitmMaxM; ++m) st.offL[m] = st.offR[m] = 0;
    for (int k = 0; k < rmax; ++k) {
        if (!needL[k]) continue;
        const int Pk = left_positions(W, rmax, k);
        st.kind[st.n_tab] = 0; st.km[st.n_tab] = (int8_t)k; st.pos[st.n_tab] = (int8_t)Pk;
        st.start[st.n_tab++] = (int64_t)e;
        for (int m = 1; m < rmax; ++m) if (mitm_j(m) - 1 == k) st.offL[m] = (int64_t)e;
        e += binom128(Pk, k);
        if (e > ((unsigned __int128)1 << 36)) return false;
    }
    for (int m = 1; m < rmax; ++m) {
        if (!needR[m]) continue;
        st.kind[st.n_tab] = 1; st.km[st.n_tab] = (int8_t)m; st.pos[st.n_tab] = (int8_t)(W - mitm_j(m));
        st.start[st.n_tab++] = (int64_t)e;
        st.offR[m] = (int64_t)e;
        e += binom128(W - mitm_j(m), m - mitm_j(m));
        if (e > ((unsigned __int128)1 << 36)) return false;
    }
    st.start[st.n_tab] = (int64_t)e;
    ws.entries = (int64_t)e;
    ws.off_hist = 256;
    ws.off_plan = ws.off_hist + (((size_t)2 * kMitmMaxM * kHistRow * 4 + 255) & ~(size_t)255);
    ws.off_timg = ws.off_plan + (((size_t)kMitmMaxBlocks * 2 + (size_t)(kMitmMaxBlocks + 1) * 4 + 255) & ~(size_t)255);
    ws.off_val = ws.off_timg + ((((size_t)L.M.t_elems * 8) + 255) & ~(size_t)255);
    ws.off_bnd = ws.off_val + (((size_t)ws.entries * 8 + 255) & ~(size_t)255);
    ws.bytes = ws.off_bnd + (((size_t)ws.entries + 255) & ~(size_t)255);
    if (sp) {
        std::stable_sort(mine.begin(), mine.end(), [&](int a, int b) { return blk[a].tile > blk[b].tile; });
        sp->nbp = (int)mine.size();
        for (int i = 0; i < sp->nbp; ++i) sp->order[i] = (int16_t)mine[i];
        for (int m = 0; m < kMitmMaxM; ++m) {
            sp->offL[m] = st.offL[m]; sp->offR[m] = st.offR[m];
            sp->tabL[m] = sp->tabR[m] = -1;
        }
        for (int i = 0; i < st.n_tab; ++i) (st.kind[i] ? sp->tabR : sp->tabL)[st.km[i]] = (int8_t)i;
    }
    return true;
}

// ------------------------------------------------------------ 1. T image
__global__ void __launch_bounds__(256) memo_image_kernel(const dm_tables tp, double* __restrict__ timg,
                                                         int* __restrict__ hist) {
    const dm_tables t = tp;
    const int n = t.n, rmax = n < t.p ? n : t.p;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < 2 * kMitmMaxM * kHistRow; i += gridDim.x * blockDim.x)
        hist[i] = 0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < (int64_t)rmax * n * n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int q = (int)(i / ((int64_t)n * n)), a = (int)((i / n) % n), b = (int)(i % n) + 1;
        if (a < q || b <= a) continue;
        double v = __longlong_as_double(0x7ff0000000000000LL);
        if ((q > 0 || a == 0) && fits_range(t, q, a, b)) {
            double c, rd;
            if (chain(t)) run_cost_contig(t, a, b, q, [&](int) { return q - 1; }, c, rd);
            else run_cost_contig(t, a, b, q, [&](int s) { return s < a ? -1 : q + 1; }, c, rd);
            v = c + rd;
        }
        timg[memo_row(q, a, n) + b] = v;
    }
}

// -------------------------------------------------------- 2. side tables
// One thread per kTabPass consecutive entries of the concatenated tables:
// colex unrank of the first, Gosper successor for the rest, then the runs
// the entry covers (T from the global image through L1).  Binomials in
// shared memory (Pascal's triangle).  CTA 0 also resets the tile counter.
template <typename Mask>   // uint32_t when every cut position fits 32 bits (n <= 34), else uint64_t
__global__ void __launch_bounds__(256) side_tables_kernel(const dm_tables tp, const double* __restrict__ timg,
                                                          const __grid_constant__ SideTables st,
                                                          double* __restrict__ val, uint8_t* __restrict__ bnd,
                                                          int* __restrict__ counter, int* __restrict__ hist) {
    extern __shared__ __align__(16) int64_t binom_s[];
    const int n = tp.n, W = n - 1, rmax = n < tp.p ? n : tp.p, R1 = rmax + 1;
    int32_t* rowrel = reinterpret_cast<int32_t*>(binom_s + n * R1);       // memo_row(q, a) for a < n
    for (int i = threadIdx.x; i < rmax * n; i += blockDim.x) {
        const int q = i / n, a = i % n;
        rowrel[i] = a >= q ? memo_row(q, a, n) : 0;
    }
    if (threadIdx.x < 32) {                      // Pascal's triangle, exact for n <= 64
        const int lane = threadIdx.x;
        int64_t v0 = lane == 0, v1 = 0, v2 = 0;
        for (int a = 0; a < n; ++a) {
            if (a > 0) {
                const int64_t u0 = __shfl_up_sync(0xffffffffu, v0, 1), u1 = __shfl_up_sync(0xffffffffu, v1, 1),
                              u2 = __shfl_up_sync(0xffffffffu, v2, 1);
                const int64_t t0 = __shfl_sync(0xffffffffu, v0, 31), t1 = __shfl_sync(0xffffffffu, v1, 31);
                v2 += lane ? u2 : t1;
                v1 += lane ? u1 : t0;
                v0 += lane ? u0 : 0;
            }
            if (lane < R1) binom_s[a * R1 + lane] = v0;
            if (lane + 32 < R1) binom_s[a * R1 + lane + 32] = v1;
            if (lane + 64 < R1) binom_s[a * R1 + lane + 64] = v2;
        }
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        counter[0] = 0;                                                          // tile queue
        reinterpret_cast<unsigned long long*>(counter)[1] = 0x7ff0000000000000ull;   // shared incumbent (+inf)
    }
    __syncthreads();
    const MitmCtx x{n, W, R1, binom_s, nullptr};
    const double* __restrict__ tim = timg;
    auto T = [=](int q, int a, int b) { return __ldg(tim + (uint32_t)(rowrel[q * n + a] + b)); };
    auto hi_bit = [](Mask m) {           // index of the highest set bit, -1 for 0
        if constexpr (sizeof(Mask) == 4) return 31 - __clz((int)m); else return 63 - __clzll((long long)m);
    };
    const double ninf = -__longlong_as_double(0x7ff0000000000000LL);
    const int64_t E = st.start[st.n_tab];
    for (int64_t e0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * kTabPass; e0 < E;
         e0 += (int64_t)gridDim.x * blockDim.x * kTabPass) {
        int ti;
        {
            int lo = 0, hi = st.n_tab - 1;
            while (lo < hi) {
                const int mid = (lo + hi + 1) >> 1;
                if (st.start[mid] <= e0) lo = mid; else hi = mid - 1;
            }
            ti = lo;
        }
        Mask mk = 0;
        int key0 = -1, cnt0 = 0;        // histogram bucket of the pass's first entry, its finite count
        for (int u = 0; u < kTabPass; ++u) {
            const int64_t e = e0 + u;
            if (e >= E) break;
            bool fresh = u == 0;
            while (st.start[ti + 1] <= e) { ++ti; fresh = true; }
            const bool right = st.kind[ti];
            const int km = st.km[ti];
            const int k = right ? km - mitm_j(km) : km;               // cuts per entry
            const int P = st.pos[ti];                                  // positions
            if (fresh) mk = (Mask)colex_unrank(x, k, P, e - st.start[ti]);
            else mk = (Mask)side_next((uint64_t)mk);
            // runs visited from the highest cut bit down (FLO per cut, no
            // bit reversal): cut bit b sits at position b + 1 in L_k and
            // W - b in R(m); the run below bit hb ends at the next lower cut
            // (position 0 / n past the last one — b = -1 in both formulas)
            double v = ninf;
            int hb = hi_bit(mk);
            const int prev = right ? W - hb : hb + 1;          // the entry's boundary cut
            Mask r = mk;
            if (!right) {                // L_k: run i = [c_{i-1}, c_i), row i
                for (int i = k - 1; hb >= 0; --i) {
                    r ^= (Mask)1 << hb;
                    const int lb = hi_bit(r);
                    const double tv = T(i, lb + 1, hb + 1);
                    v = tv > v ? tv : v;
                    hb = lb;
                }
            } else {                     // R(m): run i = [c_i, c_{i-1}) (mirrored), row km - i
                for (int i = k - 1; hb >= 0; --i) {
                    r ^= (Mask)1 << hb;
                    const int lb = hi_bit(r);
                    const double tv = T(km - i, W - hb, W - lb);
                    v = tv > v ? tv : v;
                    hb = lb;
                }
            }
            val[e] = v;
            bnd[e] = (uint8_t)prev;
            const int key = ti * kHistRow + prev;
            const bool fin = v < __longlong_as_double(0x7ff0000000000000LL);
            if (key0 < 0) key0 = key;
            if (key == key0) cnt0 += fin;
            else if (fin) atomicAdd(hist + key, 1);          // rare: the pass crosses a boundary position
        }
        // warp-aggregated flush of the first buckets
        const unsigned act = __activemask();
        const unsigned grp = __match_any_sync(act, key0);
        const int sum = __reduce_add_sync(grp, cnt0);
        if (key0 >= 0 && sum > 0 && (threadIdx.x & 31) == __ffs(grp) - 1) atomicAdd(hist + key0, sum);
    }
}

// ------------------------------------------------------------ 2b. tile plan
// One CTA: the part's blocks ordered by the predicted duration of one of
// their tiles, longest first — feasible pairs bounded by the side tables'
// finite entries (the histogram by boundary position) plus ~50
// pair-equivalents per element built; ties keep the host order (largest
// tiles first).  Writes the order and the inclusive tile prefix.
constexpr int kPlanThreads = 1024;
// Shared memory of plan_kernel sized to the sweep (so it fits the carveout
// the table and sweep kernels use): keys, tile counts and sort indices for
// np2 >= nbp blocks, the histogram rows of the hrows tables, Pascal's triangle.
__host__ __device__ inline size_t plan_smem(int np2, int hrows, int n, int rmax) {
    return (size_t)np2 * 8 + (size_t)np2 * 4 + (size_t)hrows * kHistRow * 4 + (size_t)n * (rmax + 1) * 8 +
           (((size_t)np2 * 2 + 15) & ~(size_t)15);
}
__global__ void __launch_bounds__(kPlanThreads) plan_kernel(const dm_tables tp, const __grid_constant__ SweepParams P,
                                                            const int* __restrict__ hist, int hrows,
                                                            int16_t* __restrict__ pos, int32_t* __restrict__ tstart) {
    extern __shared__ __align__(16) unsigned char psm[];   // plan_smem bytes
    const int n = tp.n, W = n - 1, rmax = n < tp.p ? n : tp.p, nbp = P.nbp, R1 = rmax + 1;
    int np2 = 2;
    while (np2 < nbp) np2 <<= 1;
    double* key = reinterpret_cast<double*>(psm);                                          // [np2]
    int64_t* binom = reinterpret_cast<int64_t*>(key + np2);                                // [n][rmax + 1]
    int32_t* ntl = reinterpret_cast<int32_t*>(binom + n * R1);                             // [np2]
    int32_t* hp = ntl + np2;                         // [hrows][kHistRow]: per-row inclusive prefix
    int16_t* sidx = reinterpret_cast<int16_t*>(hp + hrows * kHistRow);                    // [np2]
    __shared__ int32_t wsum[kPlanThreads / 32];
    for (int i = threadIdx.x; i < hrows * kHistRow; i += blockDim.x) hp[i] = hist[i];
    if (threadIdx.x < 32) {                      // Pascal's triangle, exact for n <= 64
        const int lane = threadIdx.x;
        int64_t v0 = lane == 0, v1 = 0, v2 = 0;
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
    }
    __syncthreads();
    for (int r = threadIdx.x; r < hrows; r += blockDim.x) {
        int acc = 0;
        for (int xpos = 0; xpos < kHistRow; ++xpos) { acc += hp[r * kHistRow + xpos]; hp[r * kHistRow + xpos] = acc; }
    }
    __syncthreads();
    for (int i = threadIdx.x; i < np2; i += blockDim.x) {
        if (i >= nbp) { key[i] = -__longlong_as_double(0x7ff0000000000000LL); sidx[i] = (int16_t)i; continue; }
        const int b = P.order[i];
        int m = 0, base = 0;
        while (m + 1 < rmax && base + mitm_blocks_of(m, W) <= b) { base += mitm_blocks_of(m, W); ++m; }
        const int j = m == 0 ? 0 : mitm_j(m), c = m == 0 ? 0 : j + (b - base);
        const int64_t nl = m == 0 ? 1 : binom[(c - 1) * R1 + (j - 1)], nr = m == 0 ? 1 : binom[(W - c) * R1 + (m - j)];
        const int64_t nX = nl >= nr ? nl : nr, nY = nl >= nr ? nr : nl;
        int64_t R = nY >= kThinY ? 1 : kThinPairs / (kMitmTX * nY);
        R = R < 1 ? 1 : (R > kThinRounds ? kThinRounds : R);
        const int64_t txs = (int64_t)kMitmTX * R;
        const int64_t nt = ((nX + txs - 1) / txs) * ((nY + kMitmTY - 1) / kMitmTY);
        double fl = 1.0, fr = 1.0;
        if (m > 0 && P.tabL[j - 1] >= 0 && P.tabR[m] >= 0) {
            const int* hl = hp + P.tabL[j - 1] * kHistRow;
            const int* hr = hp + P.tabR[m] * kHistRow;
            fl = (double)hl[c - 1];                              // boundary positions < c
            fr = (double)(hr[kHistRow - 1] - hr[c]);             // boundary positions > c
        }
        const double ex = (double)(nX < txs ? nX : txs), ey = (double)(nY < kMitmTY ? nY : kMitmTY);
        key[i] = fl * fr / (double)nt + 50.0 * (ex + ey);
        sidx[i] = (int16_t)i;
        ntl[i] = (int32_t)nt;
    }
    __syncthreads();
    // bitonic sort: descending key, ties by ascending host position
    if (np2 <= kPlanThreads) {
        // one element per thread: strides below 32 exchange through
        // shuffles, wider strides through shared memory
        const int tI = threadIdx.x;
        double kv = tI < np2 ? key[tI] : 0.0;
        int iv = tI < np2 ? sidx[tI] : tI;
        for (int k = 2; k <= np2; k <<= 1)
            for (int jj = k >> 1; jj > 0; jj >>= 1) {
                double pk;
                int pi;
                if (jj >= 32) {
                    __syncthreads();
                    if (tI < np2) { key[tI] = kv; sidx[tI] = (int16_t)iv; }
                    __syncthreads();
                    pk = tI < np2 ? key[tI ^ jj] : kv;
                    pi = tI < np2 ? sidx[tI ^ jj] : iv;
                } else {
                    pk = __shfl_xor_sync(0xffffffffu, kv, jj);
                    pi = __shfl_xor_sync(0xffffffffu, iv, jj);
                }
                const bool p_first = pk > kv || (pk == kv && pi < iv);
                const bool up = (tI & k) == 0, lower = (tI & jj) == 0;
                if (tI < np2 && (lower == up ? p_first : !p_first)) { kv = pk; iv = pi; }
            }
        __syncthreads();
        if (tI < np2) { key[tI] = kv; sidx[tI] = (int16_t)iv; }
        __syncthreads();
    } else
    for (int k = 2; k <= np2; k <<= 1)
        for (int jj = k >> 1; jj > 0; jj >>= 1) {
            for (int i = threadIdx.x; i < np2; i += blockDim.x) {
                const int ixj = i ^ jj;
                if (ixj > i) {
                    const double ka = key[i], kb = key[ixj];
                    const int ia = sidx[i], ib = sidx[ixj];
                    const bool b_first = kb > ka || (kb == ka && ib < ia);
                    const bool a_first = ka > kb || (ka == kb && ia < ib);
                    if (((i & k) == 0) ? b_first : a_first) {
                        key[i] = kb; key[ixj] = ka;
                        sidx[i] = (int16_t)ib; sidx[ixj] = (int16_t)ia;
                    }
                }
            }
            __syncthreads();
        }
    // order and inclusive tile prefix in position order
    const int per = (nbp + kPlanThreads - 1) / kPlanThreads;
    const int b0 = threadIdx.x * per, b1 = b0 + per < nbp ? b0 + per : nbp;
    int sum = 0;
    for (int r = b0; r < b1; ++r) { pos[r] = (int16_t)P.order[sidx[r]]; sum += ntl[sidx[r]]; }
    int incl = sum;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    for (int off = 1; off < 32; off <<= 1) {
        const int o = __shfl_up_sync(0xffffffffu, incl, off);
        if (lane >= off) incl += o;
    }
    if (lane == 31) wsum[wid] = incl;
    __syncthreads();
    int wbase = 0;
    for (int w2 = 0; w2 < wid; ++w2) wbase += wsum[w2];
    int run = wbase + incl - sum;
    for (int r = b0; r < b1; ++r) { run += ntl[sidx[r]]; tstart[r + 1] = run; }
    if (threadIdx.x == 0) tstart[0] = 0;
}

// ------------------------------------------------------------- 3. sweep
// binomials (Pascal's triangle in warp 0) and cum in shared memory.
__device__ inline void sweep_prologue(const MitmLayout& L, unsigned char* sm) {
    const int n = L.M.n, rmax = L.M.rmax, R1 = rmax + 1;
    if (threadIdx.x < 32) {
        int64_t* binom = reinterpret_cast<int64_t*>(sm + L.off_binom);
        const int lane = threadIdx.x;
        int64_t v0 = lane == 0, v1 = 0, v2 = 0;
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

__global__ void __launch_bounds__(kMitmThreads, kMitmCtasPerSm) splits_sweep_kernel(
        const dm_tables tp, const __grid_constant__ SweepParams P, int* __restrict__ ctl,
        const double* __restrict__ timg, const double* __restrict__ val, const uint8_t* __restrict__ bnd,
        dm_winner* partial, const int16_t* __restrict__ plan_pos, const int32_t* __restrict__ plan_tstart) {
    const dm_tables t = tp;   // register copy (no param-space references)
    extern __shared__ __align__(16) unsigned char sm[];
    __shared__ int s_cnt[2][2];       // [tile parity][X, Y] feasible counts
    __shared__ int s_flag[2];         // [tile parity] bit 0: an X <= best, bit 1: a Y <= best
    __shared__ int s_g[2];            // [tile parity] tile index
    __shared__ double s_best;
    const int n = t.n;
    const MitmLayout L = mitm_layout(n, t.p);
    const int rmax = L.M.rmax, nb = L.n_blocks;
    const MitmCtx x{n, n - 1, rmax + 1, reinterpret_cast<const int64_t*>(sm + L.off_binom), timg};
    const int64_t* cum = reinterpret_cast<const int64_t*>(sm + L.off_cum);
    int32_t* mbase = reinterpret_cast<int32_t*>(sm + L.off_mbase);
    int32_t* tstart = reinterpret_cast<int32_t*>(sm + L.off_tstart);
    uint8_t* bm = sm + L.off_bm;
    uint8_t* bc = sm + L.off_bc;
    int16_t* pos_blk = reinterpret_cast<int16_t*>(sm + L.off_pos);
    double* bx = reinterpret_cast<double*>(sm + L.off_bx);
    double* by = reinterpret_cast<double*>(sm + L.off_by);
    double* red = reinterpret_cast<double*>(sm + L.off_red);
    const double inf = __longlong_as_double(0x7ff0000000000000LL);

    MITM_MARK(0);
#ifdef DM_MITM_TIMING
    if (threadIdx.x == 0) for (int i_ = 4; i_ < 12; ++i_) g_mitm_times[blockIdx.x][i_] = 0;
#endif
    sweep_prologue(L, sm);
    MITM_MARK(1);
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
            B.offl = P.offL[m]; B.offr = P.offR[m];
        }
        B.rrow = memo_row(B.j, c, x.n);
        const int64_t nY = B.nl >= B.nr ? B.nr : B.nl;
        const int R = nY >= kThinY ? 1 : (int)((unsigned)kThinPairs / (unsigned)(kMitmTX * (int)nY));   // 32-bit: nY < kThinY
        B.R = R < 1 ? 1 : (R > kThinRounds ? kThinRounds : R);
        return B;
    };
    // ---- plan: (m, c) per block; tiles per position of the size order,
    //      inclusive prefix in tstart[1..nb] (positions)
    for (int b = threadIdx.x; b < nb; b += blockDim.x) {
        int m = 0;
        while (m + 1 < rmax && mbase[m + 1] <= b) ++m;
        bm[b] = (uint8_t)m;
        bc[b] = (uint8_t)(m == 0 ? 0 : mitm_j(m) + (b - mbase[m]));
    }
    __syncthreads();
    // ---- tile order and tile prefix from plan_kernel
    const int nbp = P.nbp;
    for (int i = threadIdx.x; i < nbp; i += blockDim.x) pos_blk[i] = plan_pos[i];
    for (int i = threadIdx.x; i <= nbp; i += blockDim.x) tstart[i] = plan_tstart[i];
    if (threadIdx.x == 0) s_g[0] = atomicAdd(ctl, 1);   // dynamic tile queue over the part's blocks
    // the best makespan any CTA of the sweep has found so far (bits of a
    // non-negative double): tiles whose minimum exceeds it skip the rank
    // derivation.  Stale reads only make the test more permissive.
    unsigned long long* gbest = reinterpret_cast<unsigned long long*>(ctl) + 1;
    unsigned long long gb = 0x7ff0000000000000ull;
    __syncthreads();
    const int n_tiles = tstart[nbp];
    // the finishing runs of a tile, staged one tile ahead by warp 1 into the
    // other parity's buffers (visible after the tile's end barrier)
    __shared__ double s_col[2][kMitmMaxM + 1], s_row[2][kMitmMaxM + 2];
    __shared__ int s_lo[2];            // the tile's position in the block order
    auto stage = [&](int buf, int gn) {
        if (gn >= n_tiles) return;
        int lo = 0, hi = nbp - 1;
        while (lo < hi) {
            const int mid = (lo + hi + 1) >> 1;
            if (tstart[mid] <= gn) lo = mid; else hi = mid - 1;
        }
        const int b = pos_blk[lo], m = bm[b], c = bc[b], j = m == 0 ? 0 : mitm_j(m);
        const int lane = threadIdx.x & 31;
        if (lane == 0) s_lo[buf] = lo;
        if (m > 0)
            for (int a = j - 1 + lane; a < c; a += 32) s_col[buf][a] = tval(x, j - 1, a, c);
        const int rr = memo_row(j, c, n);
        for (int bb = c + 1 + lane; bb <= n; bb += 32) s_row[buf][bb] = __ldg(timg + rr + bb);
    };
    if ((threadIdx.x >> 5) == 1) stage(0, s_g[0]);
    __syncthreads();
    MITM_MARK(2);

    Win w;
    win_init(w);
    uint64_t cs[kMitmNR];
#pragma unroll
    for (int u = 0; u < kMitmNR; ++u) cs[u] = 0;
    uint64_t corr = 0;   // +inf contributions to remove (counted in units of kInfBits)

    for (int par = 0;; par ^= 1) {
        const int g = s_g[par];
        if (g >= n_tiles) break;           // uniform
        MITM_CLK(c_t0);
        // the next tile's index: the atomic is issued now, its result stored
        // only before the element barrier (the round trip overlaps this
        // tile's element loads)
        int nxt = 0;
        if (threadIdx.x == 0) {
            nxt = atomicAdd(ctl, 1);
            gb = *reinterpret_cast<volatile unsigned long long*>(gbest);
        }
        const int lo = s_lo[par];          // staged with the tile's finishing runs
        const int blk = pos_blk[lo];
        const Blk B = block_of(blk, bm[blk], bc[blk]);
        const bool xl = B.nl >= B.nr;
        const int64_t nX = xl ? B.nl : B.nr, nY = xl ? B.nr : B.nl;
        const int64_t nty = (nY + kMitmTY - 1) / kMitmTY;
        const int64_t local = g - tstart[lo];
        const int64_t txs = (int64_t)kMitmTX * B.R;
        const int64_t x0 = (local / nty) * txs, y0 = (local % nty) * kMitmTY;
        const int nXr = (int)(nX - x0 < txs ? nX - x0 : txs);
        const int nYr = (int)(nY - y0 < kMitmTY ? nY - y0 : kMitmTY);
        const double best = s_best;
        const int64_t xoff = xl ? B.offl : B.offr, yoff = xl ? B.offr : B.offl;
        bool maybe_best = false;
        double xmin = inf, ymin = inf;
        int nyf = 0;
        if (B.R > 1) {
            // ---- thin tile: the few feasible Y once in shared memory, then
            //      rounds of kMitmTX X elements straight into registers
            //      (infeasible X slots stay +inf and are counted)
            static_assert(kThinY <= kMitmThreads, "a thin tile's Y fits one element per thread");
            {
                const int e = threadIdx.x;
                double v = inf;
                if (e < nYr) {
                    v = side_finish_s(B, !xl, B.m ? __ldcg(val + yoff + y0 + e) : 0.0, B.m ? __ldcg(bnd + yoff + y0 + e) : 0, s_col[par], s_row[par], n);
                    ymin = v < ymin ? v : ymin;
                }
                append_if(v != inf, v, by, &s_cnt[par][1]);
            }
            if (ymin <= best) atomicOr(&s_flag[par], 2);
            if (threadIdx.x == 0) s_g[par ^ 1] = nxt;
            __syncthreads();
            if ((threadIdx.x >> 5) == 1) stage(par ^ 1, s_g[par ^ 1]);
            MITM_CLK(c_t1);
            MITM_ACC(6, c_t0, c_t1);
            MITM_ACC(10, 0, 1);
            nyf = s_cnt[par][1];
            const bool yb_ok = s_flag[par] & 2;
            if (threadIdx.x == 0) {
                s_cnt[par ^ 1][0] = s_cnt[par ^ 1][1] = 0;
                s_flag[par ^ 1] = 0;
                w.n_eval += (int64_t)nXr * nYr;
            }
            int64_t nxf_all = 0;
            if (nyf > 0) {
                // warp-private compaction of each round's feasible X into a
                // ring of kThinRing values; a cross pass takes full batches
                // of 256 (8 slots per lane) as they fill and the remainder
                // after the last round, so sparse rounds are not padded to
                // whole slots one round at a time
                double* wbuf = bx + (threadIdx.x >> 5) * kThinRing;
                const int lane = threadIdx.x & 31;
                double xr[kMitmNR];
                int xb[kMitmNR];
#pragma unroll
                for (int u = 0; u < kMitmNR; ++u) {
                    const int e = u * kMitmThreads + threadIdx.x;
                    if (e < nXr && B.m) { xr[u] = __ldcg(val + xoff + x0 + e); xb[u] = __ldcg(bnd + xoff + x0 + e); }
                }
                int head = 0, fill = 0;       // warp-uniform ring state
                for (int r0 = 0; r0 < nXr; r0 += kMitmTX) {
#pragma unroll
                    for (int u = 0; u < kMitmNR; ++u) {
                        const int e = r0 + u * kMitmThreads + threadIdx.x;
                        const double v = e < nXr ? side_finish_s(B, xl, xr[u], xb[u], s_col[par], s_row[par], n) : inf;
                        xmin = v < xmin ? v : xmin;
                        const unsigned bal = __ballot_sync(0xffffffffu, v != inf);
                        if (v != inf) wbuf[(head + fill + __popc(bal & ((1u << lane) - 1u))) & (kThinRing - 1)] = v;
                        fill += __popc(bal);
                    }
                    // the next round's elements are in flight during this round's cross product
#pragma unroll
                    for (int u = 0; u < kMitmNR; ++u) {
                        const int e = r0 + kMitmTX + u * kMitmThreads + threadIdx.x;
                        if (e < nXr && B.m) { xr[u] = __ldcg(val + xoff + x0 + e); xb[u] = __ldcg(bnd + xoff + x0 + e); }
                    }
                    const bool last = r0 + kMitmTX >= nXr;
                    if (fill < kMitmNR * 32 && !(last && fill > 0)) continue;
                    __syncwarp();
                    const int take = fill < kMitmNR * 32 ? fill : kMitmNR * 32;
                    const int nsl = (take + 31) >> 5;
                    double xv[kMitmNR];
                    int nxf = 0;
#pragma unroll
                    for (int u = 0; u < kMitmNR; ++u) {
                        const int e = u * 32 + lane;
                        xv[u] = e < take ? wbuf[(head + e) & (kThinRing - 1)] : inf;
                        nxf += e < take;
                    }
                    switch (nsl) {
                        case 0: break;
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
                    nxf_all += nxf;
                    MITM_COUNT(5, nsl * nyf);
                    head = (head + take) & (kThinRing - 1);
                    fill -= take;
                    __syncwarp();
                    // a full batch on the last round can leave a remainder
                    if (last && fill > 0) {
                        const int nsl2 = (fill + 31) >> 5;
                        int nxf2 = 0;
#pragma unroll
                        for (int u = 0; u < kMitmNR; ++u) {
                            const int e = u * 32 + lane;
                            xv[u] = e < fill ? wbuf[(head + e) & (kThinRing - 1)] : inf;
                            nxf2 += e < fill;
                        }
                        switch (nsl2) {
                            case 1: mitm_cross<1>(xv, by, nyf, cs); break;
                            case 2: mitm_cross<2>(xv, by, nyf, cs); break;
                            case 3: mitm_cross<3>(xv, by, nyf, cs); break;
                            case 4: mitm_cross<4>(xv, by, nyf, cs); break;
                            case 5: mitm_cross<5>(xv, by, nyf, cs); break;
                            case 6: mitm_cross<6>(xv, by, nyf, cs); break;
                            case 7: mitm_cross<7>(xv, by, nyf, cs); break;
                            default: mitm_cross<8>(xv, by, nyf, cs); break;
                        }
                        corr += (uint64_t)(nsl2 - nxf2) * (uint64_t)nyf;
                        nxf_all += nxf2;
                        MITM_COUNT(5, nsl2 * nyf);
                        fill = 0;
                        __syncwarp();
                    }
                }
            }
            w.n_feas += nxf_all * nyf;
            MITM_CLK(c_t2);
            MITM_ACC(7, c_t1, c_t2);
            maybe_best = __syncthreads_or(xmin <= best) && yb_ok && nyf > 0;
        } else {
            // ---- both sides' feasible elements, compacted into shared memory;
            //      element raw data (table value, boundary cut) for every slot
            //      first, so all global loads are in flight together
            constexpr int kYc = kMitmNY < 8 ? kMitmNY : 8;    // Y elements per load batch
            double xr[kMitmNR], yr[kYc];
            int xb[kMitmNR], yb[kYc];
    #pragma unroll
            for (int u = 0; u < kMitmNR; ++u) {
                const int e = u * kMitmThreads + threadIdx.x;
                if (e < nXr && B.m) { xr[u] = __ldcg(val + xoff + x0 + e); xb[u] = __ldcg(bnd + xoff + x0 + e); }
            }
    #pragma unroll
            for (int u = 0; u < kYc; ++u) {
                const int e = u * kMitmThreads + threadIdx.x;
                if (e < nYr && B.m) { yr[u] = __ldcg(val + yoff + y0 + e); yb[u] = __ldcg(bnd + yoff + y0 + e); }
            }
    #pragma unroll
            for (int u = 0; u < kMitmNR; ++u) {
                const int e = u * kMitmThreads + threadIdx.x;
                double v = inf;
                if (e < nXr) { v = side_finish_s(B, xl, xr[u], xb[u], s_col[par], s_row[par], n); xmin = v < xmin ? v : xmin; }
                append_if(v != inf, v, bx, &s_cnt[par][0]);
            }
    #pragma unroll 1
            for (int h = 0; h < kMitmNY; h += kYc) {
                if (h > 0) {
    #pragma unroll
                    for (int u = 0; u < kYc; ++u) {
                        const int e = (h + u) * kMitmThreads + threadIdx.x;
                        if (e < nYr && B.m) { yr[u] = __ldcg(val + yoff + y0 + e); yb[u] = __ldcg(bnd + yoff + y0 + e); }
                    }
                }
    #pragma unroll
                for (int u = 0; u < kYc; ++u) {
                    const int e = (h + u) * kMitmThreads + threadIdx.x;
                    double v = inf;
                    if (e < nYr) { v = side_finish_s(B, !xl, yr[u], yb[u], s_col[par], s_row[par], n); ymin = v < ymin ? v : ymin; }
                    append_if(v != inf, v, by, &s_cnt[par][1]);
                }
            }
            const int fl = (xmin <= best ? 1 : 0) | (ymin <= best ? 2 : 0);
            if (fl) atomicOr(&s_flag[par], fl);
            if (threadIdx.x == 0) s_g[par ^ 1] = nxt;
            __syncthreads();
            if ((threadIdx.x >> 5) == 1) stage(par ^ 1, s_g[par ^ 1]);
            MITM_CLK(c_t1);
            MITM_ACC(6, c_t0, c_t1);
            const int nxf_tot = s_cnt[par][0];
            nyf = s_cnt[par][1];
            maybe_best = s_flag[par] == 3;
            if (threadIdx.x == 0) {       // the other parity's slots are free until the end barrier
                s_cnt[par ^ 1][0] = s_cnt[par ^ 1][1] = 0;
                s_flag[par ^ 1] = 0;
                w.n_eval += (int64_t)nXr * nYr;
                w.n_feas += (int64_t)nxf_tot * nyf;
            }
            if (nxf_tot > 0 && nyf > 0) {     // uniform
                // ---- slot layout: G warp-aligned thread groups, each taking
                //      every X against 1/G of the Y (fewer padded slots when
                //      the feasible X do not fill kMitmNR slots per thread);
                //      cost per thread ~ Y pairs x (slots + 1 per-Y overhead)
                int G = 1, nsl = (nxf_tot + kMitmThreads - 1) / kMitmThreads;
                int best_cost = nyf * (nsl + 1);
                for (int g2 = 2; g2 <= 8; g2 <<= 1) {
                    const int per2 = kMitmThreads / g2, ns2 = (nxf_tot + per2 - 1) / per2;
                    if (ns2 > kMitmNR) break;
                    const int yc2 = ((nyf + g2 - 1) / g2 + 1) & ~1;
                    const int cost = yc2 * (ns2 + 1);
                    if (cost < best_cost) { best_cost = cost; G = g2; nsl = ns2; }
                }
                const int per = kMitmThreads / G, gi = threadIdx.x / per, l = threadIdx.x - gi * per;
                const int yc = G == 1 ? nyf : (((nyf + G - 1) / G + 1) & ~1);
                const int ylo = gi * yc < nyf ? gi * yc : nyf;
                const int nyg = (ylo + yc < nyf ? ylo + yc : nyf) - ylo;
                double xv[kMitmNR];
                int nxf = 0;
#pragma unroll
                for (int u = 0; u < kMitmNR; ++u) {
                    const int e = l + u * per;
                    const bool in = u < nsl && e < nxf_tot;
                    xv[u] = in ? bx[e] : inf;
                    nxf += in;
                }
                // ---- cross product: one max + checksum add per candidate
                const double* byg = by + ylo;
                switch (nsl) {
                    case 1: mitm_cross<1>(xv, byg, nyg, cs); break;
                    case 2: mitm_cross<2>(xv, byg, nyg, cs); break;
                    case 3: mitm_cross<3>(xv, byg, nyg, cs); break;
                    case 4: mitm_cross<4>(xv, byg, nyg, cs); break;
                    case 5: mitm_cross<5>(xv, byg, nyg, cs); break;
                    case 6: mitm_cross<6>(xv, byg, nyg, cs); break;
                    case 7: mitm_cross<7>(xv, byg, nyg, cs); break;
                    default: mitm_cross<8>(xv, byg, nyg, cs); break;
                }
                corr += (uint64_t)(nsl - nxf) * (uint64_t)nyg;
                MITM_COUNT(4, nsl * nyg);
            }
            MITM_CLK(c_t2);
            MITM_ACC(7, c_t1, c_t2);
            maybe_best = maybe_best && nxf_tot > 0 && nyf > 0;
        }
        // ---- rare: the tile can hold the incumbent. Its minimum is
        //      tm = max(min X, min Y); the first rank at tm is the sum of
        //      the smallest ranks of the elements at or below tm.
        if (maybe_best) {
            const double txmin = block_min_f64(xmin, red);
            const double tymin = block_min_f64(ymin, red);
            const double tm = txmin > tymin ? txmin : tymin;
            if (tm <= best && tm < inf) {
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
                    atomicMin(gbest, (unsigned long long)__double_as_longlong(tm));
                }
            }
        }
        if (threadIdx.x == 0 && __longlong_as_double((long long)gb) < s_best) s_best = __longlong_as_double((long long)gb);
        __syncthreads();   // buffers, counters and s_best for the next tile
        MITM_CLK(c_t3);
        MITM_ACC(8, c_t0, c_t3);
        MITM_TILE(g, blk, c_t0, c_t3, nXr, nYr);
        MITM_ACC(9, 0, 1);
    }
    uint64_t c = 0;
#pragma unroll
    for (int u = 0; u < kMitmNR; ++u) c += cs[u];
    w.csum = c - corr * kInfBits;
    MITM_MARK(3);
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

// Plans depend only on (n, p, part, nparts): computed once per thread and
// shape, then reused (host-side combinatorics, no instance data).
struct PlanEntry {
    bool ok;
    SideTables st;
    MitmWorkspace ws;
    SweepParams sp;
};

inline const PlanEntry& cached_plan(int n, int p, int part, int nparts) {
    static thread_local std::vector<std::pair<std::array<int, 4>, std::unique_ptr<PlanEntry>>> cache;
    const std::array<int, 4> key{n, p, part, nparts};
    for (auto& kv : cache)
        if (kv.first == key) return *kv.second;
    auto e = std::make_unique<PlanEntry>();
    e->ok = mitm_plan(n, p, part, nparts, e->st, e->ws, &e->sp);
    if (cache.size() > 64) cache.erase(cache.begin());
    cache.emplace_back(key, std::move(e));
    return *cache.back().second;
}

int64_t mitm_workspace_bytes(const dm_tables& t) {
    if (!memo_valid(t)) return -1;
    const PlanEntry& pe = cached_plan(t.n, t.p, 0, 1);
    return pe.ok ? (int64_t)pe.ws.bytes : -1;
}

// Optional per-launch event timing of the sweep's kernels (dm_sweep_timing).
struct SweepTiming {
    bool on = false;
    bool pending = false;
    cudaEvent_t ev[3] = {nullptr, nullptr, nullptr};
};
inline SweepTiming& sweep_timing() {
    static thread_local SweepTiming st;
    return st;
}

int launch_splits_mitm(const dm_tables& t, int part, int nparts, dm_winner* partial, int sms, void* ws,
                       int64_t ws_bytes, int* n_partials, cudaStream_t s, int phase) {
    if (!memo_valid(t)) return DM_E_TOO_LARGE;
    const PlanEntry& pe = cached_plan(t.n, t.p, part, nparts);
    if (!pe.ok) return DM_E_TOO_LARGE;
    const SideTables& st = pe.st;
    const MitmWorkspace& W = pe.ws;
    const SweepParams& sp = pe.sp;
    const MitmLayout L = mitm_layout(t.n, t.p);
    void* buf = ws;
    const bool own = !ws || ws_bytes < (int64_t)W.bytes;
    if (own && phase != 3) return DM_E_ARG;     // split phases keep the tables in the caller's workspace
    if (own) DM_CUDA(cudaMallocAsync(&buf, W.bytes, s));
    unsigned char* b8 = static_cast<unsigned char*>(buf);
    int* ctl = reinterpret_cast<int*>(b8);
    int* hist = reinterpret_cast<int*>(b8 + W.off_hist);
    int16_t* plan_pos = reinterpret_cast<int16_t*>(b8 + W.off_plan);
    int32_t* plan_tstart = reinterpret_cast<int32_t*>(b8 + W.off_plan + (size_t)kMitmMaxBlocks * 2);
    double* timg = reinterpret_cast<double*>(b8 + W.off_timg);
    double* val = reinterpret_cast<double*>(b8 + W.off_val);
    uint8_t* bnd = b8 + W.off_bnd;
    const int rmax = t.n < t.p ? t.n : t.p;
    SweepTiming& tm = sweep_timing();
    if (tm.on) for (auto& e : tm.ev) if (!e) DM_CUDA(cudaEventCreate(&e));
    if (tm.on && (phase & 1)) DM_CUDA(cudaEventRecord(tm.ev[0], s));
    if (phase & 1) {
        const int64_t work = (int64_t)rmax * t.n * t.n;
        int blocks = (int)((work + 255) / 256);
        memo_image_kernel<<<blocks, 256, 0, s>>>(t, timg, hist);
        DM_CHECK_LAUNCH();
    }
    if (phase & 1) {
        const size_t smem = (size_t)t.n * (rmax + 1) * 8 + (size_t)rmax * t.n * 4;
        const int64_t per = (int64_t)256 * kTabPass;
        int64_t blocks = (W.entries + per - 1) / per;
        if (blocks > (int64_t)sms * 8) blocks = (int64_t)sms * 8;
        if (blocks < 1) blocks = 1;
        if (t.n <= 34) side_tables_kernel<uint32_t><<<(int)blocks, 256, smem, s>>>(t, timg, st, val, bnd, ctl, hist);
        else side_tables_kernel<uint64_t><<<(int)blocks, 256, smem, s>>>(t, timg, st, val, bnd, ctl, hist);
        DM_CHECK_LAUNCH();
    }
    const int grid = mitm_grid(sms);
    // phase 2 = plan + sweep; 4 = the plan alone, 8 = the sweep alone (a
    // batch runs each plan on its own stream, off the sweeps' critical path)
    const bool do_plan = phase & (2 | 4), do_sweep = phase & (2 | 8);
    if (do_plan) {
        // the tile order from the tables' histogram: a one-CTA kernel (on
        // the sweep's stream, or its own — queued behind the next tables on
        // theirs it would hold them until a running sweep's tail)
        int np2 = 2;
        while (np2 < sp.nbp) np2 <<= 1;
        const size_t psmem = plan_smem(np2, st.n_tab, t.n, rmax);
        DM_CUDA(cudaFuncSetAttribute(plan_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)psmem));
        plan_kernel<<<1, kPlanThreads, psmem, s>>>(t, sp, hist, st.n_tab, plan_pos, plan_tstart);
        DM_CHECK_LAUNCH();
    }
    if (do_sweep) {
        DM_CUDA(cudaFuncSetAttribute(splits_sweep_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)L.bytes));
        if (tm.on) DM_CUDA(cudaEventRecord(tm.ev[1], s));
        splits_sweep_kernel<<<grid, kMitmThreads, L.bytes, s>>>(t, sp, ctl, timg, val, bnd, partial, plan_pos,
                                                                plan_tstart);
        DM_CHECK_LAUNCH();
        if (tm.on) {
            DM_CUDA(cudaEventRecord(tm.ev[2], s));
            tm.pending = true;
        }
    }
    if (own) DM_CUDA(cudaFreeAsync(buf, s));
    *n_partials = grid;
    return DM_OK;
}

}  // namespace dm

extern "C" int dm_sweep_timing(int32_t enable, float* ms_tables, float* ms_sweep) {
    dm::SweepTiming& tm = dm::sweep_timing();
    if (ms_tables || ms_sweep) {
        if (!tm.pending) return dmabi::fail(DM_E_ARG, "dm_sweep_timing: no timed sweep since it was enabled");
        DM_CUDA(cudaEventSynchronize(tm.ev[2]));
        float a = 0, b = 0;
        DM_CUDA(cudaEventElapsedTime(&a, tm.ev[0], tm.ev[1]));
        DM_CUDA(cudaEventElapsedTime(&b, tm.ev[1], tm.ev[2]));
        if (ms_tables) *ms_tables = a;
        if (ms_sweep) *ms_sweep = b;
    }
    if (enable >= 0) tm.on = enable != 0;
    return DM_OK;
}

#ifdef DM_MITM_TIMING
extern "C" __attribute__((visibility("default"))) int dm_debug_mitm_tiles(unsigned int* host) {
    return (int)cudaMemcpyFromSymbol(host, dm::g_mitm_tiles, sizeof(dm::g_mitm_tiles));
}

extern "C" __attribute__((visibility("default"))) int dm_debug_mitm_times(unsigned long long* host) {
    return (int)cudaMemcpyFromSymbol(host, dm::g_mitm_times, sizeof(dm::g_mitm_times));
}
#endif

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
