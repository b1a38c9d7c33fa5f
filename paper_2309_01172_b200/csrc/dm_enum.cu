// dm_enum.cu — Mode B candidate streams generated in-kernel from a rank or a
// counter, scored with the reference cost model and reduced to the first
// strict minimum (brute_force_schedule, scheduling.py:245-278).
//
// Work decomposition: a persistent grid (a multiple of the SM count), each
// thread owns a contiguous rank range, unranks its first candidate once and
// then walks the reference's itertools order with O(1)-amortised successor
// steps.  The winner is reduced warp -> block -> one partial per CTA; a final
// single-CTA pass merges the partials (deterministic: the key is
// (makespan, global rank), independent of grid shape and GPU count).
#include "dm_common.cuh"
#include "dm_memo.cuh"
#include "dm_mitm.cuh"

namespace dm {

// ----------------------------------------------------------- combinatorics

__device__ inline int64_t perm_sat(int p, int r) {
    unsigned __int128 v = 1;
    for (int i = 0; i < r; ++i) {
        v *= (unsigned __int128)(p - i);
        if (v > (unsigned __int128)INT64_MAX) return INT64_MAX;
    }
    return (int64_t)v;
}

// Lexicographic unrank of combination c of m cut positions from {1..n-1}
// (itertools.combinations(range(1, n), m) order).
__device__ inline void unrank_comb(int n, int m, int64_t c, int32_t* cuts) {
    int lo = 1;
    for (int q = 0; q < m; ++q) {
        for (int v = lo; v <= n - 1; ++v) {
            int64_t cnt = binom_sat((n - 1) - v, m - q - 1);
            if (c < cnt) { cuts[q] = v; lo = v + 1; break; }
            c -= cnt;
        }
    }
}

// successor in lexicographic order; false when c was the last combination
__device__ inline bool next_comb(int n, int m, int32_t* cuts) {
    for (int q = m - 1; q >= 0; --q) {
        if (cuts[q] < n - m + q) {
            int v = cuts[q] + 1;
            for (int z = q; z < m; ++z) cuts[z] = v + (z - q);
            return true;
        }
    }
    return false;
}

// Partial permutations of r workers out of p, itertools.permutations order.
struct PermSet {  // used-worker bitmap for p <= 1024
    uint32_t w[32];
    __device__ void clear(int p) { for (int i = 0; i < ((p + 31) >> 5); ++i) w[i] = 0; }
    __device__ bool get(int v) const { return (w[v >> 5] >> (v & 31)) & 1u; }
    __device__ void set(int v) { w[v >> 5] |= 1u << (v & 31); }
    __device__ void unset(int v) { w[v >> 5] &= ~(1u << (v & 31)); }
    // smallest free value > v (v = -1 for the smallest), -1 if none
    __device__ int next_free(int v, int p) const {
        for (int x = v + 1; x < p; ) {
            int wi = x >> 5;
            uint32_t free_bits = ~w[wi] & (0xffffffffu << (x & 31));
            if (free_bits) {
                int c = (wi << 5) + __ffs(free_bits) - 1;
                return c < p ? c : -1;
            }
            x = (wi + 1) << 5;
        }
        return -1;
    }
};

__device__ inline void unrank_perm(int p, int r, int64_t pi, int32_t* out, PermSet& used) {
    used.clear(p);
    for (int q = 0; q < r; ++q) {
        int64_t blk = perm_sat(p - q - 1, r - q - 1);
        int64_t d = pi / blk;
        pi -= d * blk;
        int v = used.next_free(-1, p);
        while (d-- > 0) v = used.next_free(v, p);
        out[q] = v;
        used.set(v);
    }
}

__device__ inline bool next_perm(int p, int r, int32_t* a, PermSet& used) {
    for (int i = r - 1; i >= 0; --i) {
        used.unset(a[i]);
        int c = used.next_free(a[i], p);
        if (c >= 0) {
            a[i] = c; used.set(c);
            for (int j = i + 1; j < r; ++j) { int f = used.next_free(-1, p); a[j] = f; used.set(f); }
            return true;
        }
    }
    return false;
}

// --------------------------------------------------- contiguous candidate
// Inner body of brute_force_schedule (scheduling.py:266-270): skip when a run
// fails _fits; else max over runs of compute + read.
template <int RMAX>
__device__ __forceinline__ bool score_contig(const dm_tables& t, int r, const int32_t* bounds,
                                             const int32_t* peers, double& mk) {
    for (int q = 0; q < r; ++q)
        if (!fits_range(t, peers[q], bounds[q], bounds[q + 1])) return false;
    double best = 0.0;
    for (int q = 0; q < r; ++q) {
        double c, rd;
        int a = bounds[q];
        if (chain(t)) {
            int prev = q > 0 ? peers[q - 1] : -1;
            run_cost_contig(t, a, bounds[q + 1], peers[q], [&](int) { return prev; }, c, rd);
        } else {
            BoundsOwner own{bounds, peers, r};
            run_cost_contig(t, a, bounds[q + 1], peers[q], own, c, rd);
        }
        double load = c + rd;
        if (q == 0 || load > best) best = load;
    }
    mk = best;
    return true;
}

__device__ __forceinline__ void win_add(Win& w, double mk, int64_t rank) {
    w.n_feas++;
    w.csum += (uint64_t)__double_as_longlong(mk);
    if (w.rank < 0 || mk < w.mk) { w.mk = mk; w.rank = rank; }
}

// MODE 0: full brute-force order; MODE 1: identity-order splits.
template <int MODE, int RMAX>
__global__ void __launch_bounds__(256) enum_kernel(dm_tables t, int64_t k0, int64_t k1, int part, int nparts,
                                                   int64_t per_thread, dm_winner* partial) {
    Win w; win_init(w);
    int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    int64_t kb = k0 + (tid * nparts + part) * per_thread;
    int64_t ke = kb + per_thread < k1 ? kb + per_thread : k1;
    if (kb < ke) {
        const int n = t.n, p = t.p, rmax = n < p ? n : p;
        int32_t cuts[RMAX + 1], bounds[RMAX + 2], peers[RMAX + 1];
        PermSet used;
        // locate r and the in-block offset of kb
        int r = 1;
        int64_t off = kb;
        for (; r <= rmax; ++r) {
            int64_t nc = binom_sat(n - 1, r - 1);
            int64_t np = MODE == 0 ? perm_sat(p, r) : 1;
            unsigned __int128 blk = (unsigned __int128)nc * (unsigned __int128)np;
            if ((unsigned __int128)off < blk) break;
            off -= (int64_t)blk;
        }
        int64_t np = MODE == 0 ? perm_sat(p, r) : 1;
        unrank_comb(n, r - 1, off / np, cuts);
        if (MODE == 0) unrank_perm(p, r, off % np, peers, used);
        else for (int q = 0; q < r; ++q) peers[q] = q;
        for (int64_t k = kb; k < ke; ++k) {
            bounds[0] = 0;
            for (int q = 0; q < r - 1; ++q) bounds[q + 1] = cuts[q];
            bounds[r] = n;
            double mk;
            w.n_eval++;
            if (score_contig<RMAX>(t, r, bounds, peers, mk)) win_add(w, mk, k);
            // successor in the reference's itertools order
            if (MODE == 0 && next_perm(p, r, peers, used)) continue;
            if (next_comb(n, r - 1, cuts)) {
                if (MODE == 0) { used.clear(p); for (int q = 0; q < r; ++q) { peers[q] = q; used.set(q); } }
                continue;
            }
            ++r;
            if (r > rmax) break;
            for (int q = 0; q < r - 1; ++q) cuts[q] = q + 1;
            used.clear(p);
            for (int q = 0; q < r; ++q) { peers[q] = q; if (MODE == 0) used.set(q); }
        }
    }
    block_reduce_win_store(w, partial);
}

// ------------------------------------------- direct identity-split scoring
// Per-candidate cost model for the identity-order population (run q on
// worker q) with exact integral columns and chain stages or a uniform link —
// the generic evaluator's work (brute_force_schedule's inner body,
// scheduling.py:266-270) with the tables staged in shared memory: per run the
// exact prefix differences at its two boundaries, three capacity compares,
// compute = flops / speed and the crossing read.  The quotient uses
// Markstein's correction q1 = q0 + (a - q0*b)*y with y = RN(1/b), q0 = RN(a*y)
// — within one ulp before the correction, so the result is the correctly
// rounded a / b (the parity tests compare it with div.rn bit for bit).
struct __align__(8) DStage { double pf, pg, pc, pd, R; };
struct __align__(8) DPeer { double speed, rcp, cg, cc, cd; };

__device__ __forceinline__ double div_markstein(double a, double b, double y) {
    const double q0 = __dmul_rn(a, y);
    const double rem = __fma_rn(-q0, b, a);
    return __fma_rn(rem, y, q0);
}

template <int RMAX>
__global__ void __launch_bounds__(256) splits_direct_kernel(dm_tables t, int64_t k0, int64_t k1, int part, int nparts,
                                                            int64_t per_thread, dm_winner* partial) {
    extern __shared__ __align__(16) unsigned char dsm[];
    const int n = t.n, p = t.p, rmax = n < p ? n : p;
    DStage* S = reinterpret_cast<DStage*>(dsm);
    DPeer* Pr = reinterpret_cast<DPeer*>(S + n + 1);
    const bool comm = include_comm(t);
    for (int i = threadIdx.x; i <= n; i += blockDim.x) {
        DStage d;
        d.pf = (double)t.pre_flops[i]; d.pg = (double)t.pre_gpu[i];
        d.pc = (double)t.pre_cpu[i]; d.pd = (double)t.pre_disk[i];
        double rd = 0.0;
        if (comm && i < n)                       // run starting at i reads stage i's in-edges (default link)
            for (int e = t.edge_ptr[i]; e < t.edge_ptr[i + 1]; ++e)
                rd = __dadd_rn(rd, comm_time(t.def_alpha, t.def_beta, t.edge_m[e]));
        d.R = rd;
        S[i] = d;
    }
    for (int w = threadIdx.x; w < rmax; w += blockDim.x) {
        DPeer d;
        d.speed = t.speed[w]; d.rcp = 1.0 / d.speed;
        d.cg = t.cap_gpu[w]; d.cc = t.cap_cpu[w]; d.cd = t.cap_disk[w];
        Pr[w] = d;
    }
    __syncthreads();
    Win w; win_init(w);
    int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    int64_t kb = k0 + (tid * nparts + part) * per_thread;
    int64_t ke = kb + per_thread < k1 ? kb + per_thread : k1;
    if (kb < ke) {
        int32_t cuts[RMAX + 1];
        int r = 1;
        int64_t off = kb;
        for (; r <= rmax; ++r) {
            int64_t nc = binom_sat(n - 1, r - 1);
            if (off < nc) break;
            off -= nc;
        }
        unrank_comb(n, r - 1, off, cuts);
        for (int64_t k = kb; k < ke; ++k) {
            // one pass over the runs: fits (all must hold) and the max load
            bool ok = true;
            double mk = 0.0;
            int a = 0;
            DStage A = S[0];
            for (int q = 0; q < r; ++q) {
                const int b = q + 1 < r ? cuts[q] : n;
                const DStage B = S[b];
                const DPeer P = Pr[q];
                ok &= (B.pg - A.pg <= P.cg) & (B.pc - A.pc <= P.cc) & (B.pd - A.pd <= P.cd);
                double load = div_markstein(B.pf - A.pf, P.speed, P.rcp);
                if (comm && a > 0) load = load + A.R;
                mk = load > mk ? load : mk;
                a = b; A = B;
            }
            w.n_eval++;
            if (ok) win_add(w, mk, k);
            if (next_comb(n, r - 1, cuts)) continue;
            ++r;
            if (r > rmax) break;
            for (int q = 0; q < r - 1; ++q) cuts[q] = q + 1;
        }
    }
    block_reduce_win_store(w, partial);
}

// ------------------------------------------------ memoised identity splits
// Rank-range form (any [k0, k1)): every candidate is scored from scratch as
// the max over its r runs of the memo table T (dm_memo.cuh).
//
// Each thread keeps its current combination as cut bytes in shared memory
// (column-major per thread, 4 cuts per 32-bit word, the final boundary n
// stored as a sentinel), so the run loop costs one LDS.32 per four runs, a
// row-offset LDS, the table LDS.64 and the max.  The lexicographic successor
// (itertools.combinations order) rewrites only the changed suffix.  Lanes of
// a warp own ADJACENT rank chunks, so they share long run prefixes and most
// table reads are shared-memory broadcasts.
constexpr int kMemoThreads = 512;
constexpr int kMemoChunk = 64;

__host__ __device__ inline size_t memo_cut_bytes(const MemoLayout& L) {
    return (size_t)((L.rmax + 4) / 4 + 2) * kMemoThreads * 4;
}

template <int S>
__global__ void __launch_bounds__(kMemoThreads, 2) splits_memo_kernel(dm_tables t, int64_t k0, int64_t k1,
                                                                      int part, int nparts, dm_winner* partial) {
    extern __shared__ __align__(16) unsigned char sm[];
    const int n = t.n;
    const MemoLayout L = memo_layout(n, t.p);
    const int rmax = L.rmax, W = L.W, R1 = rmax + 1;
    int32_t* rowoff = reinterpret_cast<int32_t*>(sm + L.off_rowoff);
    int64_t* binom = reinterpret_cast<int64_t*>(sm + L.off_binom);   // C(a, b), a < n, b <= rmax
    int64_t* cum = reinterpret_cast<int64_t*>(sm + L.off_cum);       // cum[m] = first rank with m cuts
    unsigned char* cutb = sm + L.off_tail;                            // byte z of thread t: ((z>>2)*BS+t)*4+(z&3)
    const double inf = __longlong_as_double(0x7ff0000000000000LL);
    memo_build(t, L, sm);

    const int BS = blockDim.x, tid = threadIdx.x;
    uint32_t* cutw = reinterpret_cast<uint32_t*>(cutb) + tid;   // word j at cutw[j * BS]
    const int n_words = (rmax + 4) / 4;
    Win w; win_init(w);
    const int lane = tid & 31;
    const int64_t warps_total = (int64_t)gridDim.x * (BS >> 5);
    const int64_t gw = (int64_t)blockIdx.x * (BS >> 5) + (tid >> 5);
    const int64_t span = k1 - k0, task_ranks = 32LL * kMemoChunk;
    const int64_t n_tasks = (span + task_ranks - 1) / task_ranks;
    const uint32_t npad = (uint32_t)n * 0x01010101u;
    const unsigned long long FULL = (W >= 64) ? ~0ull : ((1ull << W) - 1ull);
    // write the cut bytes of mask x (m cuts, bit v-1 <-> position v) + sentinel n
    auto write_all = [&](unsigned long long x, int m) {
        for (int j = 0; j < n_words + 2; ++j) cutw[j * BS] = npad;
        unsigned long long y = x;
        for (int z = 0; z < m; ++z) {
            int hb = __ffsll((long long)y) - 1;
            y &= y - 1;
            uint32_t& wd = cutw[(z >> 2) * BS];
            int sh = 8 * (z & 3);
            wd = (wd & ~(0xffu << sh)) | ((uint32_t)(hb + 1) << sh);
        }
    };
    for (int64_t task = gw * nparts + part; task < n_tasks; task += warps_total * nparts) {
        int64_t kb = k0 + task * task_ranks + (int64_t)lane * kMemoChunk;
        int64_t ke = kb + kMemoChunk < k1 ? kb + kMemoChunk : k1;
        if (kb >= ke) continue;
        w.n_eval += ke - kb;
        // ---- unrank kb: m cuts, lexicographic combination of positions 1..W
        int m = 0;
        while (m + 1 < rmax && cum[m + 1] <= kb) ++m;
        int64_t c = kb - cum[m];
        unsigned long long x = 0;
        int lo = 1;
        for (int z = 0; z < m; ++z) {
            for (int v = lo; v <= W; ++v) {
                int64_t cnt = binom[(W - v) * R1 + (m - z - 1)];
                if (c < cnt) { x |= 1ull << (v - 1); lo = v + 1; break; }
                c -= cnt;
            }
        }
        write_all(x, m);
        for (int64_t k = kb; k < ke; ++k) {
            // ---- score: max over the m + 1 runs of T (from scratch), in
            //      unconditional groups of four (padding runs read -inf)
            double mk = -inf;
            uint32_t a8 = 0;  // 4 * a
            const unsigned char* rq = reinterpret_cast<const unsigned char*>(rowoff);
            for (int z4 = 0; z4 <= m; z4 += 4, rq += 4 * 4 * S) {
                uint32_t wd = cutw[(z4 >> 2) * BS];
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    uint32_t b = __byte_perm(wd, 0u, 0x4440u + u);
                    uint32_t ro = *reinterpret_cast<const uint32_t*>(rq + u * 4 * S + a8);
                    double v = lds_f64(ro + 8 * b);
                    mk = v > mk ? v : mk;
                    a8 = 4 * b;
                }
            }
            if (mk < inf) {
                w.n_feas++;
                w.csum += (uint64_t)__double_as_longlong(mk);
                if (w.rank < 0 || mk < w.mk) { w.mk = mk; w.rank = k; }
            }
            // ---- lexicographic successor in O(1) on the mask: the top L cuts
            //      sit at positions W-L+1..W; the pivot cut (index z = m-1-L,
            //      position hb+1) moves up by one and the L cuts after it
            //      follow consecutively.
            unsigned long long t0 = ~x & FULL;
            int hz = 63 - __clzll((long long)t0);          // highest non-cut position - 1 (-1: none)
            int L = W - 1 - hz;                             // saturated cuts at the top
            int z = m - 1 - L;                              // pivot index
            if (z < 0) {                                    // block exhausted: one more cut
                ++m;
                if (m >= rmax) break;
                x = (1ull << m) - 1ull;
                write_all(x, m);
                continue;
            }
            unsigned long long below = x & ((1ull << hz) - 1ull);
            int hb = 63 - __clzll((long long)below);       // pivot bit
            x = (x & ((1ull << hb) - 1ull)) | ((((1ull << (L + 1)) - 1ull)) << (hb + 1));
            // bytes z..m-1 <- hb+2, hb+3, ...: predicated rewrite of three words
            const int base = hb + 2 - z;                    // value of byte index i is base + i
            const int jz = z >> 2;
#pragma unroll
            for (int dj = 0; dj < 3; ++dj) {
                int j = jz + dj;
                int lo_b = z - 4 * j, hi_b = m - 1 - 4 * j;
                lo_b = lo_b < 0 ? 0 : lo_b;
                if (hi_b > 3) hi_b = 3;
                if (hi_b >= lo_b) {
                    uint32_t msk = (0xffffffffu << (8 * lo_b)) & (0xffffffffu >> (8 * (3 - hi_b)));
                    uint32_t pat = (uint32_t)((base + 4 * j) & 0xff) * 0x01010101u + 0x03020100u;
                    uint32_t& wd = cutw[j * BS];
                    wd = (wd & ~msk) | (pat & msk);
                }
            }
            for (int j = jz + 3; 4 * j <= m - 1; ++j) {      // L >= 9: rare
                int hi_b = m - 1 - 4 * j;
                if (hi_b > 3) hi_b = 3;
                uint32_t msk = 0xffffffffu >> (8 * (3 - hi_b));
                uint32_t pat = (uint32_t)((base + 4 * j) & 0xff) * 0x01010101u + 0x03020100u;
                uint32_t& wd = cutw[j * BS];
                wd = (wd & ~msk) | (pat & msk);
            }
        }
    }
    block_reduce_win_store(w, partial);
}

// -------------------------------------------------- candidate materialiser
// Writes candidates [k0, k0 + count) of the brute-force (MODE 0) or
// identity-split (MODE 1) order as owner vectors (worker index per stage):
// the Mode A scoring stream's input, and a cross-check of the Mode B walk.
template <typename OT, int MODE, int RMAX>
__global__ void __launch_bounds__(256) materialize_kernel(int n, int p, int64_t k0, int64_t count,
                                                          int64_t per_thread, OT* __restrict__ out) {
    int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    int64_t kb = tid * per_thread;
    int64_t ke = kb + per_thread < count ? kb + per_thread : count;
    if (kb >= ke) return;
    const int rmax = n < p ? n : p;
    int32_t cuts[RMAX + 1], peers[RMAX + 1];
    PermSet used;
    int r = 1;
    int64_t off = k0 + kb;
    for (; r <= rmax; ++r) {
        int64_t nc = binom_sat(n - 1, r - 1);
        int64_t np = MODE == 0 ? perm_sat(p, r) : 1;
        unsigned __int128 blk = (unsigned __int128)nc * (unsigned __int128)np;
        if ((unsigned __int128)off < blk) break;
        off -= (int64_t)blk;
    }
    int64_t np = MODE == 0 ? perm_sat(p, r) : 1;
    unrank_comb(n, r - 1, off / np, cuts);
    if (MODE == 0) unrank_perm(p, r, off % np, peers, used);
    else for (int q = 0; q < r; ++q) peers[q] = q;
    for (int64_t k = kb; k < ke; ++k) {
        OT* row = out + k * n;
        int a = 0;
        for (int q = 0; q < r; ++q) {
            int b = q + 1 < r ? cuts[q] : n;
            for (int i = a; i < b; ++i) row[i] = (OT)peers[q];
            a = b;
        }
        if (MODE == 0 && next_perm(p, r, peers, used)) continue;
        if (next_comb(n, r - 1, cuts)) {
            if (MODE == 0) { used.clear(p); for (int q = 0; q < r; ++q) { peers[q] = q; used.set(q); } }
            continue;
        }
        ++r;
        if (r > rmax) break;
        for (int q = 0; q < r - 1; ++q) cuts[q] = q + 1;
        used.clear(p);
        for (int q = 0; q < r; ++q) { peers[q] = q; if (MODE == 0) used.set(q); }
    }
}

// ------------------------------------------------------------ final merge
__global__ void finalize_kernel(const dm_winner* partial, int n_parts, dm_winner* out) {
    Win w; win_init(w);
    for (int i = threadIdx.x; i < n_parts; i += blockDim.x) {
        Win o;
        o.mk = partial[i].makespan; o.rank = partial[i].rank; o.n_eval = partial[i].n_evaluated;
        o.n_feas = partial[i].n_feasible; o.csum = partial[i].checksum;
        win_merge(w, o);
    }
    __shared__ dm_winner tmp[1];
    block_reduce_win_store(w, tmp);  // writes tmp[blockIdx.x == 0]
    __syncthreads();
    if (threadIdx.x == 0) *out = tmp[0];
}

}  // namespace dm

// ================================================================== C ABI
#include "dm_abi_util.cuh"
#include <cstdlib>

namespace {
constexpr int kThreads = 256;

bool getenv_flag(const char* name) {
    const char* v = std::getenv(name);
    return v && v[0] && v[0] != '0';
}

int enum_grid() {
    static thread_local int sms = 0;
    if (!sms) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        if (sms <= 0) sms = 148;
    }
    return sms * 8;  // 8 CTAs x 256 threads per SM resident
}

template <int MODE>
int launch_enum(const dm_tables* t, int64_t k0, int64_t k1, int part, int nparts, dm_winner* out, void* scratch,
                cudaStream_t s) {
    {   // ranks beyond the population do not exist: clamp [k0, k1) to it
        const int rmax_ = t->n < t->p ? t->n : t->p;
        unsigned __int128 tot = 0;
        for (int r = 1; r <= rmax_; ++r) {
            unsigned __int128 nc = 1, np = 1;
            for (int i = 1; i <= r - 1; ++i) nc = nc * (unsigned __int128)(t->n - r + i) / (unsigned __int128)i;
            if (MODE == 0) for (int i = 0; i < r; ++i) np *= (unsigned __int128)(t->p - i);
            tot += nc * np;
            if (tot > (unsigned __int128)INT64_MAX) break;
        }
        if (tot < (unsigned __int128)INT64_MAX && (unsigned __int128)k1 > tot) k1 = (int64_t)tot;
        if (k0 > k1) k0 = k1;
    }
    int grid = enum_grid();
    dm_winner* partial = (dm_winner*)scratch;
    int64_t total_threads = (int64_t)grid * kThreads * nparts;
    int64_t span = k1 > k0 ? k1 - k0 : 0;
    int64_t per = (span + total_threads - 1) / total_threads;
    if (per < 1) per = 1;
    int rmax = t->n < t->p ? t->n : t->p;
    const uint32_t f = t->flags;
    const bool direct = MODE == 1 && (f & DM_F_FLOPS_EXACT) && (f & DM_F_BYTES_EXACT) &&
                        (!(f & DM_F_INCLUDE_COMM) || ((f & DM_F_CHAIN) && !(f & DM_F_PAIR_LINKS))) &&
                        !getenv_flag("DM_DISABLE_DIRECT");
    if (direct && rmax <= 64) {
        const size_t smem = (size_t)(t->n + 1) * sizeof(dm::DStage) + (size_t)rmax * sizeof(dm::DPeer);
        if (smem <= 48 * 1024) {
            dm::splits_direct_kernel<64><<<grid, kThreads, smem, s>>>(*t, k0, k1, part, nparts, per, partial);
            DM_CHECK_LAUNCH();
            dm::finalize_kernel<<<1, 1024, 0, s>>>(partial, grid, out);
            DM_CHECK_LAUNCH();
            return DM_OK;
        }
    }
    if (rmax <= 16) dm::enum_kernel<MODE, 16><<<grid, kThreads, 0, s>>>(*t, k0, k1, part, nparts, per, partial);
    else if (rmax <= 64) dm::enum_kernel<MODE, 64><<<grid, kThreads, 0, s>>>(*t, k0, k1, part, nparts, per, partial);
    else if (rmax <= 256) dm::enum_kernel<MODE, 256><<<grid, kThreads, 0, s>>>(*t, k0, k1, part, nparts, per, partial);
    else return dmabi::fail(DM_E_TOO_LARGE, "enumeration supports at most 256 runs");
    DM_CHECK_LAUNCH();
    dm::finalize_kernel<<<1, 1024, 0, s>>>(partial, grid, out);
    DM_CHECK_LAUNCH();
    return DM_OK;
}

// The meet-in-the-middle sweep covers whole populations only: [k0, k1) must
// be every split of the instance (its parts are tile sets, not rank ranges).
bool nparts_full_range(const dm_tables* t, int64_t k0, int64_t k1) {
    if (k0 != 0) return false;
    const int n = t->n, rmax = t->n < t->p ? t->n : t->p;
    unsigned __int128 tot = 0, c = 1;   // C(n-1, m) for m = 0..rmax-1
    for (int m = 0; m < rmax; ++m) {
        tot += c;
        if (tot > (unsigned __int128)INT64_MAX) return false;
        c = c * (unsigned __int128)(n - 1 - m) / (unsigned __int128)(m + 1);
    }
    return (unsigned __int128)k1 == tot;
}

int enum_splits_impl(const dm_tables* t, int64_t k0, int64_t k1, int part, int nparts, dm_winner* out,
                     void* scratch, void* ws, int64_t ws_bytes, void* stream, int phase = 3) {
    if (!t || !out || !scratch || t->n <= 0 || t->p <= 0 || nparts < 1 || part < 0 || part >= nparts ||
        phase < 1 || phase > 15)
        return dmabi::fail(DM_E_ARG, "bad arguments");
    cudaStream_t s = (cudaStream_t)stream;
    const bool memo_ok = dm::memo_valid(*t) && !getenv_flag("DM_DISABLE_MEMO");
    if (memo_ok && nparts_full_range(t, k0, k1) && !getenv_flag("DM_DISABLE_MITM")) {
        int n_partials = 0;
        int rc = dm::launch_splits_mitm(*t, part, nparts, (dm_winner*)scratch, enum_grid() / 8, ws, ws_bytes,
                                        &n_partials, s, phase);
        if (rc == DM_E_ARG) return dmabi::fail(DM_E_ARG, "split phases need a workspace of dm_splits_workspace_bytes");
        if (rc != DM_E_TOO_LARGE) {
            if (rc != DM_OK) return rc;
            if (phase & (2 | 8)) {
                dm::finalize_kernel<<<1, 1024, 0, s>>>((dm_winner*)scratch, n_partials, out);
                DM_CHECK_LAUNCH();
            }
            return DM_OK;
        }
    }
    if (!(phase & (2 | 8))) return DM_OK;     // the rank-range kernels have no table or plan phase
    dm::MemoLayout L = dm::memo_layout(t->n, t->p);
    const size_t memo_bytes = L.off_tail + dm::memo_cut_bytes(L);
    if (memo_ok && t->n <= 64 && memo_bytes <= 110 * 1024) {
        int grid = enum_grid() / 8 * 2;  // 2 CTAs x 512 threads per SM
        if (L.S == 64) {
            cudaFuncSetAttribute(dm::splits_memo_kernel<64>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)memo_bytes);
            dm::splits_memo_kernel<64><<<grid, dm::kMemoThreads, memo_bytes, s>>>(*t, k0, k1, part, nparts,
                                                                              (dm_winner*)scratch);
        } else {
            cudaFuncSetAttribute(dm::splits_memo_kernel<256>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)memo_bytes);
            dm::splits_memo_kernel<256><<<grid, dm::kMemoThreads, memo_bytes, s>>>(*t, k0, k1, part, nparts,
                                                                               (dm_winner*)scratch);
        }
        DM_CHECK_LAUNCH();
        dm::finalize_kernel<<<1, 1024, 0, s>>>((dm_winner*)scratch, grid, out);
        DM_CHECK_LAUNCH();
        return DM_OK;
    }
    return launch_enum<1>(t, k0, k1, part, nparts, out, scratch, s);
}
}  // namespace

extern "C" {

int64_t dm_enum_scratch_bytes(void) { return (int64_t)sizeof(dm_winner) * enum_grid(); }

int dm_enum_bruteforce(const dm_tables* t, int64_t k0, int64_t k1, dm_winner* out,
                       void* scratch, void* stream) {
    if (!t || !out || !scratch || t->n <= 0 || t->p <= 0) return dmabi::fail(DM_E_ARG, "bad arguments");
    if (t->p > 1024) return dmabi::fail(DM_E_TOO_LARGE, "brute force supports at most 1024 workers");
    return launch_enum<0>(t, k0, k1, 0, 1, out, scratch, (cudaStream_t)stream);
}

int dm_enum_splits(const dm_tables* t, int64_t k0, int64_t k1, dm_winner* out,
                   void* scratch, void* stream) {
    return enum_splits_impl(t, k0, k1, 0, 1, out, scratch, nullptr, 0, stream);
}

int dm_enum_splits_part(const dm_tables* t, int64_t k0, int64_t k1, int32_t part, int32_t nparts,
                        dm_winner* out, void* scratch, void* stream) {
    return enum_splits_impl(t, k0, k1, part, nparts, out, scratch, nullptr, 0, stream);
}

int64_t dm_splits_workspace_bytes(const dm_tables* t) {
    if (!t) return -1;
    return dm::mitm_workspace_bytes(*t);
}

int dm_enum_splits_ws(const dm_tables* t, int64_t k0, int64_t k1, int32_t part, int32_t nparts, dm_winner* out,
                      void* scratch, void* workspace, int64_t workspace_bytes, void* stream) {
    return enum_splits_impl(t, k0, k1, part, nparts, out, scratch, workspace, workspace_bytes, stream);
}

int dm_enum_splits_phase(const dm_tables* t, int64_t k0, int64_t k1, int32_t part, int32_t nparts, dm_winner* out,
                         void* scratch, void* workspace, int64_t workspace_bytes, int32_t phase, void* stream) {
    return enum_splits_impl(t, k0, k1, part, nparts, out, scratch, workspace, workspace_bytes, stream, phase);
}

int dm_materialize(int32_t n, int32_t p, int32_t mode, int64_t k0, int64_t count, void* owner, int32_t owner_bytes,
                   void* stream) {
    if (n <= 0 || p <= 0 || count < 0 || !owner || (owner_bytes != 1 && owner_bytes != 2) || (mode != 0 && mode != 1))
        return dmabi::fail(DM_E_ARG, "dm_materialize: bad arguments");
    int rmax = n < p ? n : p;
    if (rmax > 64) return dmabi::fail(DM_E_TOO_LARGE, "dm_materialize: at most 64 runs");
    if (count == 0) return DM_OK;
    const int64_t per = 64;
    int64_t threads = (count + per - 1) / per;
    int blocks = (int)((threads + 255) / 256);
    cudaStream_t s = (cudaStream_t)stream;
#define DM_MAT(OT, M) dm::materialize_kernel<OT, M, 64><<<blocks, 256, 0, s>>>(n, p, k0, count, per, (OT*)owner)
    if (owner_bytes == 1) { if (mode == 0) DM_MAT(uint8_t, 0); else DM_MAT(uint8_t, 1); }
    else { if (mode == 0) DM_MAT(uint16_t, 0); else DM_MAT(uint16_t, 1); }
#undef DM_MAT
    DM_CHECK_LAUNCH();
    return DM_OK;
}

int dm_finalize_winners(void* scratch, int32_t n_parts, dm_winner* out, void* stream) {
    if (!scratch || !out || n_parts <= 0) return dmabi::fail(DM_E_ARG, "bad arguments");
    dm::finalize_kernel<<<1, 1024, 0, (cudaStream_t)stream>>>((dm_winner*)scratch, n_parts, out);
    DM_CHECK_LAUNCH();
    return DM_OK;
}

}  // extern "C"
