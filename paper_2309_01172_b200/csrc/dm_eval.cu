// dm_eval.cu — candidate scoring.
//
//  * eval_runs_kernel: the general evaluate_runs (scheduling.py:210-239) for
//    arbitrary Runs (overlaps, gaps, repeated or unknown peers), one thread per
//    candidate, restating verify_assignment (:179-207) and _run_cost (:156-169)
//    step by step.  Used by the API calls that score a handful of assignments
//    (evaluate_runs, pinned runs, final reports, backup ranking).
//  * eval_owner_kernel: Mode A scoring stream.  A CTA stages a tile of owner
//    vectors through shared memory with 16-byte coalesced loads, then each
//    thread walks its vector run by run (contiguous fast path); a candidate
//    whose peer reappears falls back to the grouped general evaluation.
//  * argmin kernels: block/warp arg-min over (makespan, rank).
#include "dm_common.cuh"
#include "dm_abi_util.cuh"
#include <cstdio>
#include <cstdlib>
#include <type_traits>

namespace dm {

// ------------------------------------------------------- general evaluate
// Indices inside each run arrive sorted ascending (the reference only ever
// uses sorted(indices): verify :191, _evaluate :217); duplicates may remain.
__device__ inline bool in_run(const int32_t* idx, int k, int s) {
    int lo = 0, hi = k - 1;
    while (lo <= hi) {
        int mid = (lo + hi) >> 1;
        int v = idx[mid];
        if (v == s) return true;
        if (v < s) lo = mid + 1; else hi = mid - 1;
    }
    return false;
}

__device__ inline double col_items(const double* col, const int64_t* pre, bool exact,
                                   const int32_t* idx, int k, bool np_items) {
    if (exact) {
        int64_t s = 0;
        for (int q = 0; q < k; ++q) s += pre[idx[q] + 1] - pre[idx[q]];
        return (double)s;
    }
    PySum acc;
    for (int q = 0; q < k; ++q) acc.add(col[idx[q]], !np_items);
    return acc.value();
}

__global__ void eval_runs_kernel(dm_tables t, int32_t n_cand, const int32_t* __restrict__ cand_ptr,
                                 const int32_t* __restrict__ run_peer, const int32_t* __restrict__ run_ptr,
                                 const int32_t* __restrict__ run_idx, double* out_compute, double* out_read,
                                 double* out_makespan, int32_t* out_code, int32_t* out_code_run,
                                 int32_t* out_status, int32_t* ws_owner, uint8_t* ws_seen, int32_t* ws_order) {
    int c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= n_cand) return;
    const int n = t.n;
    int32_t* peer_of = ws_owner + (int64_t)c * n;
    uint8_t* seen = ws_seen + (int64_t)c * n;
    int r0 = cand_ptr[c], r1 = cand_ptr[c + 1];
    bool ex = bytes_exact(t);

    // ---- verify_assignment (:179-207), runs in the given order
    for (int i = 0; i < n; ++i) { seen[i] = 0; peer_of[i] = -1; }
    int code = DM_V_OK, bad = -1, n_seen = 0;
    for (int r = r0; r < r1 && code == DM_V_OK; ++r) {
        const int32_t* idx = run_idx + run_ptr[r];
        int k = run_ptr[r + 1] - run_ptr[r];
        if (!k) continue;
        int pe = run_peer[r];
        for (int u = r0; u < r; ++u)
            if (run_ptr[u + 1] > run_ptr[u] && run_peer[u] == pe) { code = DM_V_TWO_RUNS; break; }
        if (code) { bad = r - r0; break; }
        if (pe < 0 || pe >= t.P) { code = DM_V_UNKNOWN_PEER; bad = r - r0; break; }
        for (int q = 1; q < k; ++q)
            if (idx[q] != idx[0] + q) { code = DM_V_NOT_CONTIGUOUS; break; }
        if (code) { bad = r - r0; break; }
        for (int q = 0; q < k; ++q) {
            if (seen[idx[q]]) { code = DM_V_ASSIGNED_TWICE; break; }
            seen[idx[q]] = 1; ++n_seen;
        }
        if (code) { bad = r - r0; break; }
        const bool nb = np_bytes(t);
        if (col_items(t.gpu, t.pre_gpu, ex, idx, k, nb) > t.cap_gpu[pe]) code = DM_V_GPU;
        else if (col_items(t.cpu, t.pre_cpu, ex, idx, k, nb) > t.cap_cpu[pe]) code = DM_V_CPU;
        else if (col_items(t.disk, t.pre_disk, ex, idx, k, nb) > t.cap_disk[pe]) code = DM_V_DISK;
        if (code) bad = r - r0;
    }
    if (code == DM_V_OK && n_seen != n) code = DM_V_UNASSIGNED;
    out_code[c] = code;
    out_code_run[c] = bad;

    // ---- peer_of: last writer in runs order (:213)
    for (int r = r0; r < r1; ++r)
        for (int q = run_ptr[r]; q < run_ptr[r + 1]; ++q) peer_of[run_idx[q]] = run_peer[r];

    // ---- ordered_runs: non-empty runs stably sorted by first index (:217-218)
    int32_t* order = ws_order + r0;
    int no = 0;
    for (int r = r0; r < r1; ++r) {
        out_compute[r] = 0.0; out_read[r] = 0.0;
        if (run_ptr[r + 1] == run_ptr[r]) continue;
        int fr = run_idx[run_ptr[r]];
        int pos = no++;
        while (pos > 0 && run_idx[run_ptr[order[pos - 1]]] > fr) { order[pos] = order[pos - 1]; --pos; }
        order[pos] = r;
    }

    // ---- cost every run in that order (:219-222)
    double makespan = 0.0;
    int status = DM_OK;
    for (int o = 0; o < no; ++o) {
        int r = order[o];
        const int32_t* idx = run_idx + run_ptr[r];
        int k = run_ptr[r + 1] - run_ptr[r];
        int pe = run_peer[r];
        if (pe < 0 || pe >= t.P) { status = DM_E_UNKNOWN_PEER; break; }  // fleet.peer :158
        double fl = col_items(t.flops, t.pre_flops, flops_exact(t), idx, k, np_flops(t));
        double compute = fl / t.speed[pe];
        double rd = 0.0;
        if (include_comm(t)) {
            for (int q = 0; q < k && status == DM_OK; ++q) {
                int i = idx[q];
                for (int e = t.edge_ptr[i]; e < t.edge_ptr[i + 1]; ++e) {
                    int src = t.edge_src[e];
                    if (in_run(idx, k, src)) continue;
                    int own = peer_of[src];
                    if (own == -1) { status = DM_E_UNASSIGNED; break; }
                    double al, be;
                    link_of(t, own, pe, al, be);
                    rd = __dadd_rn(rd, comm_time(al, be, t.edge_m[e]));
                }
            }
            if (status != DM_OK) break;
        }
        out_compute[r] = compute;
        out_read[r] = rd;
        double load = compute + rd;
        if (load > makespan) makespan = load;
    }
    out_makespan[c] = makespan;
    out_status[c] = status;
}

// ------------------------------------------------------------ Mode A stream
constexpr int kTile = 128;          // candidates per CTA tile (= threads)

template <typename OT>
__device__ __forceinline__ int owner_at(const OT* row, int i) { return (int)row[i]; }

// Grouped general evaluation of one owner vector (non-contiguous case):
// Runs = stages of each peer in first-appearance order (verify order), each
// costed over its sorted indices with peer_of = the owner vector.
template <typename OT>
__device__ void eval_owner_grouped(const dm_tables& t, const OT* row, double& mk_out, int& code_out) {
    const int n = t.n;
    bool ex = bytes_exact(t), fex = flops_exact(t);
    int code = DM_V_OK;
    double mk = 0.0;
    for (int i0 = 0; i0 < n; ++i0) {
        int pe = owner_at(row, i0);
        bool first = true;
        for (int z = 0; z < i0; ++z) if (owner_at(row, z) == pe) { first = false; break; }
        if (!first) continue;
        // stages of pe, ascending; contiguity, capacities (verify :191-203)
        int last = -1, k = 0;
        bool contig = true;
        int64_t sg = 0, sc = 0, sd = 0, sf = 0;
        PySum pg, pc, pd, pf;
        for (int i = i0; i < n; ++i) {
            if (owner_at(row, i) != pe) continue;
            if (last >= 0 && i != last + 1) contig = false;
            last = i; ++k;
            if (ex) { sg += t.pre_gpu[i + 1] - t.pre_gpu[i]; sc += t.pre_cpu[i + 1] - t.pre_cpu[i];
                      sd += t.pre_disk[i + 1] - t.pre_disk[i]; }
            else { pg.add(t.gpu[i], !np_bytes(t)); pc.add(t.cpu[i], !np_bytes(t)); pd.add(t.disk[i], !np_bytes(t)); }
            if (fex) sf += t.pre_flops[i + 1] - t.pre_flops[i]; else pf.add(t.flops[i], !np_flops(t));
        }
        if (code == DM_V_OK) {
            if (!contig) code = DM_V_NOT_CONTIGUOUS;
            else if ((ex ? (double)sg : pg.value()) > t.cap_gpu[pe]) code = DM_V_GPU;
            else if ((ex ? (double)sc : pc.value()) > t.cap_cpu[pe]) code = DM_V_CPU;
            else if ((ex ? (double)sd : pd.value()) > t.cap_disk[pe]) code = DM_V_DISK;
        }
        double compute = (fex ? (double)sf : pf.value()) / t.speed[pe];
        double rd = 0.0;
        if (include_comm(t)) {
            for (int i = i0; i < n; ++i) {
                if (owner_at(row, i) != pe) continue;
                for (int e = t.edge_ptr[i]; e < t.edge_ptr[i + 1]; ++e) {
                    int src = t.edge_src[e];
                    int own = owner_at(row, src);
                    if (own == pe) continue;  // src inside this peer's run
                    double al, be;
                    link_of(t, own, pe, al, be);
                    rd = __dadd_rn(rd, comm_time(al, be, t.edge_m[e]));
                }
            }
        }
        double load = compute + rd;
        if (load > mk) mk = load;
    }
    mk_out = mk;
    code_out = code;
}

template <typename OT>
__global__ void __launch_bounds__(kTile) eval_owner_kernel(dm_tables t, int64_t n_cand,
                                                           const OT* __restrict__ owner,
                                                           double* __restrict__ out_mk,
                                                           uint8_t* __restrict__ out_code) {
    extern __shared__ __align__(16) unsigned char smem[];
    const int n = t.n;
    OT* tile = reinterpret_cast<OT*>(smem);
    uint32_t* seen = reinterpret_cast<uint32_t*>(smem + (((size_t)kTile * n * sizeof(OT) + 15) & ~(size_t)15));
    const int seen_words = (t.P + 31) >> 5;
    const int64_t n_tiles = (n_cand + kTile - 1) / kTile;
    for (int64_t tl = blockIdx.x; tl < n_tiles; tl += gridDim.x) {
        int64_t c0 = tl * kTile;
        int cnt = (int)((n_cand - c0) < kTile ? (n_cand - c0) : kTile);
        // ---- stage the tile: 16-byte loads when the tile is 16-byte aligned
        size_t bytes = (size_t)cnt * n * sizeof(OT);
        const unsigned char* src = reinterpret_cast<const unsigned char*>(owner + c0 * n);
        __syncthreads();
        if ((((uintptr_t)src) & 15) == 0) {
            size_t nv = bytes >> 4;
            for (size_t v = threadIdx.x; v < nv; v += blockDim.x)
                reinterpret_cast<uint4*>(smem)[v] = __ldcs(reinterpret_cast<const uint4*>(src) + v);
            for (size_t b = (nv << 4) + threadIdx.x; b < bytes; b += blockDim.x) smem[b] = src[b];
        } else {
            for (size_t b = threadIdx.x; b < bytes; b += blockDim.x) smem[b] = src[b];
        }
        __syncthreads();
        if (threadIdx.x >= cnt) continue;
        const OT* row = tile + (size_t)threadIdx.x * n;
        // ---- contiguous fast path
        for (int w = 0; w < seen_words; ++w) seen[w * kTile + threadIdx.x] = 0u;
        bool unknown = false, grouped = false;
        int code = DM_V_OK;
        double mk = 0.0;
        int a = 0, pe = owner_at(row, 0), prev = -1;
        for (int i = 1; i <= n; ++i) {
            int o = i < n ? owner_at(row, i) : -2;
            if (o == pe) continue;
            // run [a, i) on pe
            if (pe >= t.P) { unknown = true; break; }
            uint32_t& sw = seen[(pe >> 5) * kTile + threadIdx.x];
            uint32_t bit = 1u << (pe & 31);
            if (sw & bit) { grouped = true; break; }
            sw |= bit;
            if (code == DM_V_OK) code = cap_violation(t, pe, a, i);
            double c, rd;
            if (chain(t)) {
                run_cost_contig(t, a, i, pe, [&](int) { return prev; }, c, rd);
            } else {
                run_cost_contig(t, a, i, pe, [&](int s) { return owner_at(row, s); }, c, rd);
            }
            double load = c + rd;
            if (load > mk) mk = load;
            prev = pe; pe = o; a = i;
        }
        if (!unknown && grouped) {
            for (int i = 0; i < n; ++i) if (owner_at(row, i) >= t.P) { unknown = true; break; }
            if (!unknown) eval_owner_grouped(t, row, mk, code);
        }
        int64_t c = c0 + threadIdx.x;
        out_mk[c] = unknown ? __longlong_as_double(0x7ff8000000000000LL) : mk;
        out_code[c] = unknown ? (uint8_t)0xFF : (uint8_t)code;
    }
}

// ----------------------------------------------- Mode A, memoised stream
// Owner-vector stream for uint8 owners, n <= 64, P <= 64 when the load of a
// contiguous run [a, b) on peer w depends only on (a, b, w) (uniform link or
// include_comm off), or additionally on the previous run's peer for
// chain-structured stages with pairwise links (then the table holds the
// compute term and the crossing read alpha + beta*M is added per run).
// Per-(a, b, w) loads and violation codes are tabulated once per CTA in
// shared memory with the reference's arithmetic; candidate tiles stream in
// through a ring of 1-D TMA bulk copies (cp.async.bulk + mbarrier), one
// elected thread issuing, while every thread scores one candidate:
// SIMD byte compares build the run-boundary mask, then each run costs a
// table lookup.  A candidate whose peer reappears (non-contiguous) or whose
// owner index is out of range takes the general grouped path.
constexpr int kStreamThreads = 256;

// shared-memory layout; every segment 16-byte aligned (TMA destinations).
// The load table is square T[(a*(n+1) + b)*P + w] when it fits (no row-offset
// lookup per run), else triangular T[(rowidx[a] + b)*P + w].
struct StreamLayout {
    int n, P, stages, cpt, nt;
    bool square;
    size_t t_elems, off_T, off_code, off_rowidx, off_tiles, off_bar, bytes, tile_bytes;
};

__host__ __device__ inline size_t al16(size_t x) { return (x + 15) & ~(size_t)15; }

__host__ __device__ inline StreamLayout stream_layout(int n, int P, int stages, int cpt, bool square,
                                                     int nt = kStreamThreads) {
    StreamLayout L;
    L.n = n; L.P = P; L.stages = stages; L.cpt = cpt; L.square = square; L.nt = nt;
    L.t_elems = square ? (size_t)n * (n + 1) * P : (size_t)n * (n + 1) / 2 * P;
    size_t off = 0;
    L.off_T = off; off = al16(off + L.t_elems * 8);
    L.off_code = off; off = al16(off + L.t_elems);          // first failing capacity of the run (0: fits)
    L.off_rowidx = off; off = al16(off + (size_t)(n + 1) * 4);
    L.tile_bytes = al16((size_t)nt * cpt * n);
    L.off_tiles = off; off = al16(off + L.tile_bytes * stages + 16);
    L.off_bar = off; off += 8 * stages;
    // + 2 KB: a run on an owner index >= P (rerouted to the general path
    // afterwards) may address up to 255 entries past the end of T / codes
    L.bytes = al16(off) + 2048;
    return L;
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void tma_load_1d(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 :: "r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile("{\n\t.reg .pred p;\n"
                 "WAIT_%=:\n\t"
                 "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
                 "@!p bra WAIT_%=;\n}" :: "r"(smem_u32(bar)), "r"(parity) : "memory");
}

__device__ __forceinline__ uint32_t lds_u8(uint32_t a) {
    uint32_t v;
    asm volatile("ld.shared.u8 %0, [%1];" : "=r"(v) : "r"(a));
    return v;
}
__device__ __forceinline__ uint32_t lds_u32(uint32_t a) {
    uint32_t v;
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a));
    return v;
}
__device__ __forceinline__ double lds_f64s(uint32_t a) {
    double v;
    asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(a));
    return v;
}

// Run-boundary mask of one owner row (NW 32-bit words, row starting `sh`
// bits into the first aligned word): bit i <=> owner[i] != owner[i-1] (bit 0
// is always clear).
// Fully unrolled per word count so every shift is a compile-time constant.
template <int NW>
__device__ __forceinline__ unsigned long long boundary_mask(uint32_t waddr, int sh) {
    uint32_t m0 = 0, m1 = 0, prevw = 0, cur = lds_u32(waddr);
#pragma unroll
    for (int j = 0; j < NW; ++j) {
        uint32_t nxt = lds_u32(waddr + 4 * (j + 1));
        uint32_t wd = __funnelshift_r(cur, nxt, sh);
        cur = nxt;
        uint32_t x = wd ^ __byte_perm(prevw, wd, 0x6543);    // byte k vs byte k-1
        uint32_t nz = (x | ((x & 0x7f7f7f7fu) + 0x7f7f7f7fu)) & 0x80808080u;
        // bit k <=> byte k differs: the four flags gathered by one multiply
        // (high word; the product's terms are disjoint, so no carries), and
        // accumulated with multiply-adds — both on the FMA pipe, the ALU pipe
        // being the kernel's busiest
        const uint32_t nib = __umulhi(nz, 0x02040810u) & 0xFu;
        if (j < 8) m0 = nib * (1u << (4 * j)) + m0; else m1 = nib * (1u << (4 * j - 32)) + m1;
        prevw = wd;
    }
    return ((unsigned long long)m1 << 32) | m0;           // bit i <=> owner[i] != owner[i-1]
}

// Per-launch constants of the stream kernel's candidate loop.
struct StreamCtx {
    int n;
    uint32_t uP, rowstride, T_s, C_s, mask_lo, mask_hi, tri_k, pmask;
};

// Lean per-candidate arg-min state: n_evaluated is the number of candidates
// the thread saw (derived at the end), the feasible count fits 32 bits per
// thread and launch.
struct StreamWin {
    double mk;
    int64_t rank;
    uint32_t n_feas;
    uint64_t csum;
};

// Score this thread's candidates of one resident tile (NW: boundary-mask
// words).  Runs are visited from the last boundary down (FLO gives the
// highest set bit in one instruction); per run: the owner byte, its bit in
// `seen`, the table address, one 8-byte table load, the running maximum of
// |T| and the address of the last failing run visited (T's sign bit) —
// runs are visited by decreasing first stage and table addresses grow with
// it, so that is the first failing run in verify order
// (scheduling.py:184-203), whose violation code is read once after the loop.  A peer seen twice
// (non-contiguous owner vector) or an owner index >= P (bit outside the
// fleet) sends the candidate to the grouped general path.
template <bool PAIR, bool SQUARE, int NT, int NW>
__device__ __forceinline__ void stream_tile(const dm_tables& t, const StreamCtx& X, uint32_t tile_s,
                                            const unsigned char* tile, int cnt, int64_t c0,
                                            double* __restrict__ out_mk, uint8_t* __restrict__ out_code,
                                            int64_t rank_base, bool fuse, StreamWin& win, uint32_t& n_seen) {
    const int n = X.n;
    // the table's shared address as an opaque register value: otherwise the
    // compiler rematerialises it (CTA id + window offset, four uniform
    // instructions) at every run
    uint32_t T_s;
    asm volatile("mov.b32 %0, %1;" : "=r"(T_s) : "r"(X.T_s));
    // per-thread bases, advanced per candidate (no per-candidate address rebuild)
    double* omk = out_mk + c0 + threadIdx.x;
    uint8_t* ocode = out_code + c0 + threadIdx.x;
    int64_t rank = rank_base + c0 + threadIdx.x;
    uint32_t row_s = tile_s + (uint32_t)threadIdx.x * n;          // shared address of this thread's row
    const uint32_t row_step = (uint32_t)NT * n;
#pragma unroll 1
    for (int ci = threadIdx.x; ci < cnt; ci += NT, row_s += row_step, omk += NT, ocode += NT, rank += NT) {
        ++n_seen;
        const unsigned long long bm = boundary_mask<NW>(row_s & ~3u, (int)(row_s & 3u) * 8);
        double mk = 0.0;
        uint32_t end = (uint32_t)n, seen = 0, bad = 0xffffffffu;
        int prev_w = -1;
        auto run = [&](uint32_t b) {                             // run [b, end)
            const uint32_t w = lds_u8(row_s + b);
            seen |= 1u << w;                                     // shl clamps: w >= 32 leaves no bit
            uint32_t idx;
            if (SQUARE) idx = b * X.rowstride + end * X.uP + w;
            else idx = ((b * (X.tri_k - b)) >> 1) * X.uP + (end - b - 1) * X.uP + w;
            const uint32_t addr = T_s + 8u * idx;
            double v = lds_f64s(addr);
            if (PAIR) {
                // chain stages: the crossing read of run [b, end) is priced with
                // the link from the owner of stage b-1 (the next run visited)
                if (b > 0) {
                    const int pw = (int)lds_u8(row_s + b - 1);
                    double al, be;
                    link_of(t, pw, (int)w, al, be);
                    double rd = 0.0;
                    for (int e = t.edge_ptr[b]; e < t.edge_ptr[b + 1]; ++e)
                        rd = __dadd_rn(rd, comm_time(al, be, t.edge_m[e]));
                    v = copysign(fabs(v) + rd, v);
                }
            }
            mk = fabs(v) > fabs(mk) ? v : mk;                    // sign cleared after the loop
            bad = __double2hiint(v) < 0 ? addr : bad;           // runs visited by decreasing address
            end = b;
        };
        if (NW > 8)
            for (uint32_t y = (uint32_t)(bm >> 32) & X.mask_hi; y; ) {
                const uint32_t k = 31u - __clz(y);
                y ^= 1u << k;
                run(32u + k);
            }
        if (PAIR) {
            for (uint32_t y = (uint32_t)bm & X.mask_lo; y; ) {
                const uint32_t k = 31u - __clz(y);
                y ^= 1u << k;
                run(k);
            }
        } else {
            // two runs per step: both owner-byte and table loads in flight
            // before either is folded into the maximum (ILP for the few warps
            // a large table leaves resident)
            auto fetch = [&](uint32_t b, uint32_t e, uint32_t& w, uint32_t& addr, double& v) {
                w = lds_u8(row_s + b);
                uint32_t idx;
                if (SQUARE) idx = b * X.rowstride + e * X.uP + w;
                else idx = ((b * (X.tri_k - b)) >> 1) * X.uP + (e - b - 1) * X.uP + w;
                addr = T_s + 8u * idx;
                v = lds_f64s(addr);
            };
            auto fold = [&](uint32_t w, uint32_t addr, double v) {
                seen |= 1u << w;
                mk = fabs(v) > fabs(mk) ? v : mk;
                bad = __double2hiint(v) < 0 ? addr : bad;
            };
            for (uint32_t y = (uint32_t)bm & X.mask_lo; y; ) {
                const uint32_t k1 = 31u - __clz(y);
                y ^= 1u << k1;
                const uint32_t b1 = k1;
                uint32_t w1, a1;
                double v1;
                if (y) {
                    const uint32_t k2 = 31u - __clz(y);
                    y ^= 1u << k2;
                    const uint32_t b2 = k2;
                    uint32_t w2, a2;
                    double v2;
                    fetch(b1, end, w1, a1, v1);
                    fetch(b2, b1, w2, a2, v2);
                    fold(w1, a1, v1);
                    fold(w2, a2, v2);
                    end = b2;
                } else {
                    fetch(b1, end, w1, a1, v1);
                    fold(w1, a1, v1);
                    end = b1;
                }
            }
        }
        run(0u);
        (void)prev_w;
        mk = __hiloint2double(__double2hiint(mk) & 0x7fffffff, __double2loint(mk));   // |mk| without the fp64 pipe
        const int nruns = __popcll(bm & (((unsigned long long)X.mask_hi << 32) | X.mask_lo)) + 1;
        int code = bad != 0xffffffffu ? (int)lds_u8(X.C_s + ((bad - T_s) >> 3)) : DM_V_OK;
        bool unknown = false;
        if (__popc(seen) != nruns || (seen & X.pmask)) {        // repeated peer or owner >= P
            const unsigned char* row = tile + (size_t)ci * n;
            for (int i = 0; i < n; ++i) if (row[i] >= X.uP) { unknown = true; break; }
            if (!unknown) eval_owner_grouped(t, row, mk, code);
        }
        *omk = unknown ? __longlong_as_double(0x7ff8000000000000LL) : mk;
        *ocode = unknown ? (uint8_t)0xFF : (uint8_t)code;
        if (fuse && !unknown && code == DM_V_OK) {      // fused arg-min (first strict minimum by rank)
            win.n_feas++;
            win.csum += (uint64_t)__double_as_longlong(mk);
            if (win.rank < 0 || mk < win.mk) { win.mk = mk; win.rank = rank; }
        }
    }
}

template <bool PAIR, bool SQUARE, int NT, int MINB>
__global__ void __launch_bounds__(NT, MINB) eval_owner_stream_kernel(dm_tables t, int64_t n_cand,
                                                                              const uint8_t* __restrict__ owner,
                                                                              double* __restrict__ out_mk,
                                                                              uint8_t* __restrict__ out_code,
                                                                              int64_t rank_base, dm_winner* partial,
                                                                              int stages, int cpt) {
    extern __shared__ __align__(128) unsigned char sm[];
    const int n = t.n, P = t.P;
    const StreamLayout L = stream_layout(n, P, stages, cpt, SQUARE, NT);
    // T: load of run (a, b) on w (compute only when PAIR); sign bit set when
    // the run fails _fits (|T| is the value; -0.0 keeps the flag)
    double* T = reinterpret_cast<double*>(sm + L.off_T);
    uint8_t* C8 = sm + L.off_code;
    int32_t* rowidx = reinterpret_cast<int32_t*>(sm + L.off_rowidx);
    unsigned char* tiles = sm + L.off_tiles;
    uint64_t* bars = reinterpret_cast<uint64_t*>(sm + L.off_bar);
    const int tile_cand = NT * cpt;
    const int64_t n_tiles = (n_cand + tile_cand - 1) / tile_cand;
    const int64_t full_tiles = n_cand / tile_cand;
    const uint32_t tile_load = (uint32_t)(tile_cand * n);

    if (threadIdx.x == 0) {
        for (int st = 0; st < stages; ++st) mbar_init(&bars[st], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        for (int st = 0; st < stages; ++st) {
            int64_t tl = blockIdx.x + (int64_t)st * gridDim.x;
            if (tl < full_tiles) {
                mbar_expect_tx(&bars[st], tile_load);
                tma_load_1d(tiles + st * L.tile_bytes, owner + tl * tile_cand * n, tile_load, &bars[st]);
            }
        }
    }
    for (int a = threadIdx.x; a <= n; a += blockDim.x) rowidx[a] = a * n - a * (a - 1) / 2 - a - 1;
    __syncthreads();
    // ---- tables (reference arithmetic, once per CTA)
    const int npairs = n * (n + 1) / 2;
    for (int it = threadIdx.x; it < npairs * P; it += blockDim.x) {
        int pr = it / P, w = it % P;
        int a = 0;
        while (a + 1 < n && rowidx[a + 1] + (a + 2) <= pr) ++a;
        int b = pr - rowidx[a];
        double v, c, rd;
        if (PAIR) {
            v = col_range(t.flops, t.pre_flops, flops_exact(t), a, b, np_flops(t)) / t.speed[w];
        } else {
            run_cost_contig(t, a, b, w, [&](int) { return -1; }, c, rd);  // uniform link: every source is remote
            v = c + rd;
        }
        const int code = cap_violation(t, w, a, b);
        if (code) v = -v;
        const size_t ti = SQUARE ? ((size_t)a * (n + 1) + b) * P + w : (size_t)it;
        T[ti] = v;
        C8[ti] = (uint8_t)code;
    }
    __syncthreads();

    const int tid = threadIdx.x;
    const int nw = (n + 3) >> 2;
    const uint32_t sm_s = (uint32_t)__cvta_generic_to_shared(sm);
    const uint32_t T_s = sm_s + (uint32_t)L.off_T;
    const uint32_t C_s = sm_s + (uint32_t)L.off_code;
    StreamCtx X;
    X.n = n; X.uP = (uint32_t)P; X.rowstride = (uint32_t)(n + 1) * X.uP;
    X.T_s = T_s; X.C_s = C_s; X.tri_k = 2u * (uint32_t)n + 1u;
    X.pmask = P >= 32 ? 0u : ~((1u << P) - 1u);
    // boundary positions 1..n-1: bits 1..min(n-1, 31) of the low word, bits
    // 0..n-33 of the high word
    X.mask_lo = n >= 32 ? 0xfffffffeu : (((1u << n) - 1u) & ~1u);
    X.mask_hi = n - 32 >= 32 ? 0xffffffffu : (n > 32 ? ((1u << (n - 32)) - 1u) : 0u);
    StreamWin win;
    win.mk = __longlong_as_double(0x7ff0000000000000LL); win.rank = -1; win.n_feas = 0; win.csum = 0;
    uint32_t n_seen = 0;
    // the boundary-mask width is fixed per launch: one dispatch per CTA, the
    // tile loop (TMA ring) instantiated per width
    auto loop = [&](auto nw_tag) {
        constexpr int W = decltype(nw_tag)::value;
        int st = 0;
        uint32_t parity = 0;
        for (int64_t tl = blockIdx.x; tl < n_tiles; tl += gridDim.x) {
            const int64_t c0 = tl * tile_cand;
            const int cnt = (int)((n_cand - c0) < tile_cand ? (n_cand - c0) : tile_cand);
            unsigned char* tile = tiles + st * L.tile_bytes;
            if (tl < full_tiles) {
                mbar_wait(&bars[st], parity);
            } else {  // ragged last tile: plain loads
                for (int b = tid; b < cnt * n; b += blockDim.x) tile[b] = owner[c0 * n + b];
                __syncthreads();
            }
            const uint32_t tile_s = sm_s + (uint32_t)(tile - sm);
            stream_tile<PAIR, SQUARE, NT, W>(t, X, tile_s, tile, cnt, c0, out_mk, out_code, rank_base,
                                             partial != nullptr, win, n_seen);
            __syncthreads();  // every thread is done with this slot
            if (tid == 0) {
                int64_t nt = tl + (int64_t)stages * gridDim.x;
                if (nt < full_tiles) {
                    mbar_expect_tx(&bars[st], tile_load);
                    tma_load_1d(tile, owner + nt * tile_cand * n, tile_load, &bars[st]);
                }
            }
            if (++st == stages) { st = 0; parity ^= 1u; }
        }
    };
    switch (nw) {
#define DM_STREAM_LOOP(W) case W: loop(std::integral_constant<int, W>{}); break;
        DM_STREAM_LOOP(1) DM_STREAM_LOOP(2) DM_STREAM_LOOP(3) DM_STREAM_LOOP(4) DM_STREAM_LOOP(5)
        DM_STREAM_LOOP(6) DM_STREAM_LOOP(7) DM_STREAM_LOOP(8) DM_STREAM_LOOP(9) DM_STREAM_LOOP(10)
        DM_STREAM_LOOP(11) DM_STREAM_LOOP(12) DM_STREAM_LOOP(13) DM_STREAM_LOOP(14) DM_STREAM_LOOP(15)
        default: loop(std::integral_constant<int, 16>{}); break;
#undef DM_STREAM_LOOP
    }
    if (partial) {
        Win w;
        w.mk = win.mk; w.rank = win.rank; w.n_eval = n_seen; w.n_feas = win.n_feas; w.csum = win.csum;
        block_reduce_win_store(w, partial);
    }
}

// ---------------------------------------------------------------- arg-min
__global__ void __launch_bounds__(256) argmin_kernel(const double* __restrict__ mk, const uint8_t* __restrict__ code,
                                                     int64_t n, int64_t rank_base, dm_winner* partial) {
    Win w; win_init(w);
    int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
        w.n_eval++;
        if (code[i] != 0) continue;
        double v = mk[i];
        w.n_feas++;
        w.csum += (uint64_t)__double_as_longlong(v);
        if (win_better(v, rank_base + i, w.mk, w.rank)) { w.mk = v; w.rank = rank_base + i; }
    }
    block_reduce_win_store(w, partial);
}

__global__ void finalize_argmin_kernel(const dm_winner* partial, int n_parts, dm_winner* out) {
    Win w; win_init(w);
    for (int i = threadIdx.x; i < n_parts; i += blockDim.x) {
        Win o;
        o.mk = partial[i].makespan; o.rank = partial[i].rank; o.n_eval = partial[i].n_evaluated;
        o.n_feas = partial[i].n_feasible; o.csum = partial[i].checksum;
        win_merge(w, o);
    }
    __shared__ dm_winner tmp[1];
    block_reduce_win_store(w, tmp);
    __syncthreads();
    if (threadIdx.x == 0) *out = tmp[0];
}

}  // namespace dm

namespace {
int sm_count() {
    static thread_local int sms = 0;
    if (!sms) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        if (sms <= 0) sms = 148;
    }
    return sms;
}
}  // namespace

extern "C" {

int dm_abi_version(void) { return DM_ABI_VERSION; }
const char* dm_last_error(void) { return dmabi::last_error_buf(); }

int dm_eval_runs(const dm_tables* t, int32_t n_cand, const int32_t* cand_ptr, const int32_t* run_peer,
                 const int32_t* run_ptr, const int32_t* run_idx, double* out_compute, double* out_read,
                 double* out_makespan, int32_t* out_code, int32_t* out_code_run, int32_t* out_status,
                 void* stream) {
    if (!t || n_cand < 0 || !cand_ptr || !run_peer || !run_ptr || t->n <= 0)
        return dmabi::fail(DM_E_ARG, "dm_eval_runs: bad arguments");
    if (n_cand == 0) return DM_OK;
    cudaStream_t s = (cudaStream_t)stream;
    // per-candidate workspace: peer_of (int32 x n), seen (u8 x n), run order
    int32_t n_runs_total = 0;
    DM_CUDA(cudaMemcpyAsync(&n_runs_total, cand_ptr + n_cand, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
    DM_CUDA(cudaStreamSynchronize(s));
    size_t b_owner = (size_t)n_cand * t->n * sizeof(int32_t);
    size_t b_seen = ((size_t)n_cand * t->n + 15) & ~(size_t)15;
    size_t b_order = (size_t)(n_runs_total + 1) * sizeof(int32_t);
    void* ws = nullptr;
    DM_CUDA(cudaMallocAsync(&ws, b_owner + b_seen + b_order, s));
    int32_t* ws_owner = (int32_t*)ws;
    uint8_t* ws_seen = (uint8_t*)ws + b_owner;
    int32_t* ws_order = (int32_t*)((uint8_t*)ws + b_owner + b_seen);
    int threads = 128, blocks = (n_cand + threads - 1) / threads;
    dm::eval_runs_kernel<<<blocks, threads, 0, s>>>(*t, n_cand, cand_ptr, run_peer, run_ptr, run_idx, out_compute,
                                                    out_read, out_makespan, out_code, out_code_run, out_status,
                                                    ws_owner, ws_seen, ws_order);
    cudaError_t le = cudaGetLastError();
    cudaFreeAsync(ws, s);
    if (le != cudaSuccess) return dmabi::cuda_fail(le, "eval_runs_kernel");
    return DM_OK;
}

int64_t dm_eval_runs_ws_bytes(int32_t n, int32_t n_cand, int32_t n_runs_total) {
    if (n <= 0 || n_cand < 0 || n_runs_total < 0) return -1;
    const size_t b_owner = (size_t)n_cand * n * sizeof(int32_t);
    const size_t b_seen = ((size_t)n_cand * n + 15) & ~(size_t)15;
    return (int64_t)(b_owner + b_seen + (size_t)(n_runs_total + 1) * sizeof(int32_t));
}

int dm_eval_runs_ws(const dm_tables* t, int32_t n_cand, const int32_t* cand_ptr, const int32_t* run_peer,
                    const int32_t* run_ptr, const int32_t* run_idx, int32_t n_runs_total, double* out_compute,
                    double* out_read, double* out_makespan, int32_t* out_code, int32_t* out_code_run,
                    int32_t* out_status, void* workspace, void* stream) {
    if (!t || n_cand < 0 || !cand_ptr || !run_peer || !run_ptr || t->n <= 0 || n_runs_total < 0 || !workspace)
        return dmabi::fail(DM_E_ARG, "dm_eval_runs_ws: bad arguments");
    if (n_cand == 0) return DM_OK;
    const size_t b_owner = (size_t)n_cand * t->n * sizeof(int32_t);
    const size_t b_seen = ((size_t)n_cand * t->n + 15) & ~(size_t)15;
    int32_t* ws_owner = (int32_t*)workspace;
    uint8_t* ws_seen = (uint8_t*)workspace + b_owner;
    int32_t* ws_order = (int32_t*)((uint8_t*)workspace + b_owner + b_seen);
    const int threads = 128, blocks = (n_cand + threads - 1) / threads;
    dm::eval_runs_kernel<<<blocks, threads, 0, (cudaStream_t)stream>>>(*t, n_cand, cand_ptr, run_peer, run_ptr,
                                                                       run_idx, out_compute, out_read, out_makespan,
                                                                       out_code, out_code_run, out_status, ws_owner,
                                                                       ws_seen, ws_order);
    DM_CHECK_LAUNCH();
    return DM_OK;
}

static int eval_owner_impl(const dm_tables* t, int64_t n_cand, const void* owner, int32_t owner_bytes,
                           double* out_makespan, uint8_t* out_code, int64_t rank_base, dm_winner* out,
                           void* scratch, void* stream);

int dm_eval_owner(const dm_tables* t, int64_t n_cand, const void* owner, int32_t owner_bytes,
                  double* out_makespan, uint8_t* out_code, void* stream) {
    return eval_owner_impl(t, n_cand, owner, owner_bytes, out_makespan, out_code, 0, nullptr, nullptr, stream);
}

int dm_eval_owner_argmin(const dm_tables* t, int64_t n_cand, const void* owner, int32_t owner_bytes,
                         double* out_makespan, uint8_t* out_code, int64_t rank_base, dm_winner* out,
                         void* scratch, void* stream) {
    if (!out || !scratch) return dmabi::fail(DM_E_ARG, "dm_eval_owner_argmin: bad arguments");
    return eval_owner_impl(t, n_cand, owner, owner_bytes, out_makespan, out_code, rank_base, out, scratch, stream);
}

static int eval_owner_impl(const dm_tables* t, int64_t n_cand, const void* owner, int32_t owner_bytes,
                           double* out_makespan, uint8_t* out_code, int64_t rank_base, dm_winner* out,
                           void* scratch, void* stream) {
    if (!t || n_cand < 0 || !owner || !out_makespan || !out_code || t->n <= 0 ||
        (owner_bytes != 1 && owner_bytes != 2))
        return dmabi::fail(DM_E_ARG, "dm_eval_owner: bad arguments");
    if (owner_bytes == 1 && t->P > 256) return dmabi::fail(DM_E_ARG, "uint8 owners need P <= 256");
    if (n_cand == 0) return DM_OK;
    cudaStream_t s = (cudaStream_t)stream;
    {
        const uint32_t f = t->flags;
        bool memo_ok = !(f & DM_F_INCLUDE_COMM) || !(f & DM_F_PAIR_LINKS) || (f & DM_F_CHAIN);
        // pick a configuration (threads, CTAs per SM, candidates per thread
        // per tile, ring stages, table shape): the square table when it fits
        // with several CTAs per SM (no row-offset arithmetic per run), else
        // the triangular table with one large CTA per SM.  DM_MODEA_CFG =
        // "nt,minb,cpt,stages,square" overrides (experiments).
        struct Cfg { int nt, minb, cpt, stages, square; };
        static const Cfg kCfgs[] = {{256, 2, 4, 3, 1}, {256, 4, 2, 2, 1}, {256, 3, 2, 3, 1}, {256, 2, 2, 2, 1},
                                    {768, 1, 1, 2, 0}, {512, 1, 1, 2, 0}, {512, 1, 1, 1, 0}};
        const size_t smem_sm = 227 * 1024;
        dm::StreamLayout L{};
        Cfg cfg{0, 0, 0, 0, 0};
        bool found = false;
        for (const Cfg& c : kCfgs) {
            L = dm::stream_layout(t->n, t->P, c.stages, c.cpt, c.square == 1, c.nt);
            if ((L.bytes + 1024) * c.minb <= smem_sm) { cfg = c; found = true; break; }
        }
        if (const char* env = std::getenv("DM_MODEA_CFG")) {
            Cfg c{};
            if (std::sscanf(env, "%d,%d,%d,%d,%d", &c.nt, &c.minb, &c.cpt, &c.stages, &c.square) == 5) {
                dm::StreamLayout L2 = dm::stream_layout(t->n, t->P, c.stages, c.cpt, c.square == 1, c.nt);
                if ((L2.bytes + 1024) * c.minb <= smem_sm) { L = L2; cfg = c; found = true; }
            }
        }
        const char* dis = std::getenv("DM_DISABLE_MEMO");
        bool aligned = (((uintptr_t)owner) & 15) == 0;
        if (found && owner_bytes == 1 && memo_ok && aligned && t->n <= 64 && t->P <= 32 &&
            !(dis && dis[0] && dis[0] != '0')) {
            const int tile_cand = L.nt * L.cpt;
            int64_t n_tiles = (n_cand + tile_cand - 1) / tile_cand;
            int64_t grid = (int64_t)sm_count() * cfg.minb;
            if (grid > n_tiles) grid = n_tiles;
            if (out && grid > 8 * sm_count()) grid = 8 * sm_count();   // partial slots in scratch
            const bool pair = (t->flags & DM_F_INCLUDE_COMM) && (t->flags & DM_F_PAIR_LINKS);
            using KernT = void (*)(dm_tables, int64_t, const uint8_t*, double*, uint8_t*, int64_t, dm_winner*, int, int);
            KernT kern = nullptr;
#define DM_PICK(NT, MB, SQ)                                                                               \
            if (cfg.nt == NT && cfg.minb == MB && cfg.square == SQ)                                       \
                kern = pair ? dm::eval_owner_stream_kernel<true, SQ == 1, NT, MB>                         \
                            : dm::eval_owner_stream_kernel<false, SQ == 1, NT, MB>;
            DM_PICK(256, 4, 1) DM_PICK(256, 3, 1) DM_PICK(256, 2, 1) DM_PICK(512, 2, 1) DM_PICK(128, 8, 1)
            DM_PICK(768, 1, 0) DM_PICK(512, 1, 0) DM_PICK(1024, 1, 0) DM_PICK(256, 2, 0) DM_PICK(256, 3, 0)
            DM_PICK(384, 1, 0) DM_PICK(256, 1, 0)
#undef DM_PICK
            if (!kern) return dmabi::fail(DM_E_ARG, "dm_eval_owner: unsupported DM_MODEA_CFG");
            cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)L.bytes);
            kern<<<(int)grid, L.nt, L.bytes, s>>>(*t, n_cand, (const uint8_t*)owner, out_makespan, out_code, rank_base,
                                                  out ? (dm_winner*)scratch : nullptr, L.stages, L.cpt);
            DM_CHECK_LAUNCH();
            if (out) {
                dm::finalize_argmin_kernel<<<1, 1024, 0, s>>>((dm_winner*)scratch, (int)grid, out);
                DM_CHECK_LAUNCH();
            }
            return DM_OK;
        }
    }
    size_t tile_bytes = (((size_t)dm::kTile * t->n * owner_bytes) + 15) & ~(size_t)15;
    size_t seen_bytes = (size_t)((t->P + 31) / 32) * dm::kTile * sizeof(uint32_t);
    size_t smem = tile_bytes + seen_bytes;
    if (smem > 200 * 1024) return dmabi::fail(DM_E_TOO_LARGE, "dm_eval_owner: tile exceeds shared memory");
    int64_t n_tiles = (n_cand + dm::kTile - 1) / dm::kTile;
    int per_sm = (int)((220 * 1024) / (smem + 1024));
    if (per_sm < 1) per_sm = 1;
    if (per_sm > 16) per_sm = 16;
    int64_t grid = (int64_t)sm_count() * per_sm;
    if (grid > n_tiles) grid = n_tiles;
    if (owner_bytes == 1) {
        cudaFuncSetAttribute(dm::eval_owner_kernel<uint8_t>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        dm::eval_owner_kernel<uint8_t><<<(int)grid, dm::kTile, smem, s>>>(*t, n_cand, (const uint8_t*)owner,
                                                                           out_makespan, out_code);
    } else {
        cudaFuncSetAttribute(dm::eval_owner_kernel<uint16_t>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        dm::eval_owner_kernel<uint16_t><<<(int)grid, dm::kTile, smem, s>>>(*t, n_cand, (const uint16_t*)owner,
                                                                            out_makespan, out_code);
    }
    DM_CHECK_LAUNCH();
    if (out) return dm_argmin_scores(out_makespan, out_code, n_cand, rank_base, out, scratch, stream);
    return DM_OK;
}

int dm_argmin_scores(const double* makespan, const uint8_t* code, int64_t n, int64_t rank_base, dm_winner* out,
                     void* scratch, void* stream) {
    if (!makespan || !code || !out || !scratch || n < 0) return dmabi::fail(DM_E_ARG, "dm_argmin_scores: bad arguments");
    cudaStream_t s = (cudaStream_t)stream;
    int grid = sm_count() * 8;
    dm::argmin_kernel<<<grid, 256, 0, s>>>(makespan, code, n, rank_base, (dm_winner*)scratch);
    DM_CHECK_LAUNCH();
    dm::finalize_argmin_kernel<<<1, 1024, 0, s>>>((dm_winner*)scratch, grid, out);
    DM_CHECK_LAUNCH();
    return DM_OK;
}

}  // extern "C"
