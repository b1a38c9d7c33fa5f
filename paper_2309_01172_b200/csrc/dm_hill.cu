// dm_hill.cu — batched proportional split + boundary hill climb, and the
// pipeline epilogue.  One warp per scenario:
//   * _proportional_runs (scheduling.py:328-351) runs on lane 0 (O(n + p),
//     order-sensitive sums restated exactly);
//   * _hill_climb (:354-388): the reference takes the first improving move
//     (a, dir) in order, and until one improves every move is scored from the
//     same state — so when a move changes only the two runs at its boundary
//     (chain stages, no comm, or no pair links) the lanes score 32 moves at
//     once (the two new run loads + prefix / suffix maxima of the others),
//     apply the first improving one and resume after it; otherwise each
//     score() (:357-362) is parallelised over runs (lanes cost runs, a warp
//     max-reduce combines them);
//   * the epilogue scores the final runs (_evaluate :210-232) and applies
//     Eq. 3 / Eq. 4 (pipeline.py:41-62).
#include "dm_common.cuh"
#include "dm_abi_util.cuh"

namespace dm {

constexpr int kWarpsPerCta = 4;

__device__ __forceinline__ double warp_max(double v) {
    for (int off = 16; off > 0; off >>= 1) {
        double o = __shfl_xor_sync(0xffffffffu, v, off);
        v = o > v ? o : v;
    }
    return v;
}

// score() of _hill_climb over contiguous runs bounds[0..r] / peers[0..r)
// held in shared memory: inf if verify_assignment fails (only capacities can
// fail for these runs), else max over runs of compute + read.
// Load of run q (compute + read) and whether it fails _fits.
__device__ __forceinline__ double run_load(const dm_tables& t, int q, int r, const int32_t* bounds,
                                           const int32_t* peers, bool& bad) {
    int a = bounds[q], b = bounds[q + 1], w = peers[q];
    bad = cap_violation(t, w, a, b) != 0;
    if (bad) return 0.0;
    double c, rd;
    if (chain(t)) {
        int prev = q > 0 ? peers[q - 1] : -1;
        run_cost_contig(t, a, b, w, [&](int) { return prev; }, c, rd);
    } else {
        BoundsOwner own{bounds, peers, r};
        run_cost_contig(t, a, b, w, own, c, rd);
    }
    return c + rd;
}

// score() over all runs; when lr/bd are given, every run's load and fit
// flag are kept there for the incremental scores below.
__device__ double hill_score(const dm_tables& t, int r, const int32_t* bounds, const int32_t* peers, int lane,
                             double* lr = nullptr, uint8_t* bd = nullptr) {
    const double inf = __longlong_as_double(0x7ff0000000000000LL);
    bool bad = false;
    double best = 0.0;
    for (int q = lane; q < r; q += 32) {
        bool b;
        const double load = run_load(t, q, r, bounds, peers, b);
        if (lr) { lr[q] = load; bd[q] = b; }
        if (b) { bad = true; continue; }
        best = load > best ? load : best;
    }
    if (lr) __syncwarp();
    if (__any_sync(0xffffffffu, bad)) return inf;
    return warp_max(best);
}

// Load of the run [a, b) on worker w whose predecessor run is on prev, when
// reads do not depend on which run owns a source: chain stages, no comm, or
// no pair links (every source outside the run is on another peer).
__device__ __forceinline__ double run_load_ab(const dm_tables& t, int a, int b, int w, int prev, bool& bad) {
    bad = cap_violation(t, w, a, b) != 0;
    if (bad) return 0.0;
    double c, rd;
    run_cost_contig(t, a, b, w, [&](int) { return prev; }, c, rd);
    return c + rd;
}

// Staged scenario tables for the fast path (exact integral columns, chain
// stages or a uniform link, <= kHillPeers workers): per boundary i the exact
// prefix sums as doubles and R[i], the read of a run starting at i (stage i's
// in-edges priced with the default link, summed like run_cost_contig); per
// worker speed and capacities.  Every run load in the hill climb then costs
// shared-memory reads instead of dependent global loads.
constexpr int kHillPeers = 64;
struct HillStage { double pf, pg, pc, pd, R; };
struct HillPeer { double speed, cg, cc, cd; };

// Per-warp shared memory of prop_hill_kernel: stage flops, run loads and
// their prefix / suffix maxima, bounds/peers, run fit flags, staged tables.
__host__ __device__ inline size_t hill_core_bytes(int n_max) {
    return ((size_t)(4 * n_max + 3) * 8 + (size_t)2 * (n_max + 2) * 4 + (size_t)(n_max + 1) + 15) & ~(size_t)15;
}
__host__ __device__ inline size_t hill_warp_bytes(int n_max) {
    return hill_core_bytes(n_max) + (size_t)(n_max + 1) * sizeof(HillStage) + (size_t)kHillPeers * sizeof(HillPeer);
}

// run load on the staged tables (fast path); read of the run = R[a] when it
// has a predecessor run (chain stages: the previous run is on another worker)
__device__ __forceinline__ double run_load_staged(const HillStage* hs, const HillPeer* hp, int a, int b, int w,
                                                  bool comm, bool& bad) {
    const HillStage& A = hs[a];
    const HillStage& B = hs[b];
    const HillPeer& P = hp[w];
    bad = !((B.pg - A.pg <= P.cg) & (B.pc - A.pc <= P.cc) & (B.pd - A.pd <= P.cd));
    const double c = (B.pf - A.pf) / P.speed;
    const double rd = (comm && a > 0) ? A.R : 0.0;
    return c + rd;
}

// _proportional_runs on lane 0; returns r and fills bounds/peers.
__device__ int proportional(const dm_tables& t, int32_t* bounds, int32_t* peers, const double* fls) {
    const int n = t.n, p = t.p;
    PySum ts;
    for (int w = 0; w < p; ++w) ts.add(t.speed[w], !(t.peer_np && t.peer_np[w]));
    double total_speed = ts.value();                                     // :332
    double total_flops = col_range(t.flops, t.pre_flops, flops_exact(t), 0, n, np_flops(t));  // :333
    if (total_flops == 0.0) total_flops = 1.0;
    int start = 0, nr = 0;
    double acc = 0.0, pf = fls[0];       // pf = prefix[end-1] (itertools.accumulate :334), flops staged in smem
    int pf_at = 0;
    bounds[0] = 0;
    for (int wi = 0; wi < p; ++wi) {                                     // :337
        if (start >= n) break;
        int end;
        if (wi == p - 1) end = n;
        else {
            acc = acc + (total_flops * t.speed[wi]) / total_speed;        // :343
            end = start + 1;
            while (true) {                                               // :345-346
                if (end >= n) break;
                while (pf_at < end - 1) { ++pf_at; pf = pf + fls[pf_at]; }
                if (!(pf < acc)) break;
                ++end;
            }
            int remaining = p - wi - 1;
            int lim = n - remaining;
            end = end < lim ? end : lim;
            end = end > start + 1 ? end : start + 1;                     // :348
        }
        peers[nr] = wi;
        bounds[++nr] = end;
        start = end;
    }
    return nr;
}

// The same, warp-cooperative, when the stage flops are exact integers (then
// prefix[k] = pre_flops[k+1] exactly, whatever the summation order): the
// boundary of worker wi is max(start + 1, e*) clamped as at :348, where
// e* = min{end : end == n or prefix[end-1] >= acc_wi} — a binary search per
// worker on the lanes; acc (:343) and the clamps stay sequential on lane 0.
// acc: scratch of n_max + 1 doubles.  Returns r on every lane.
__device__ int proportional_warp(const dm_tables& t, int32_t* bounds, int32_t* peers, double* acc, int lane) {
    const int n = t.n, p = t.p;
    const int nw = (p - 1 < n ? p - 1 : n);      // workers that can need a search (each run takes >= 1 stage)
    double total_speed = 0.0, total_flops = 0.0;
    if (lane == 0) {
        PySum ts;
        for (int w = 0; w < p; ++w) ts.add(t.speed[w], !(t.peer_np && t.peer_np[w]));
        total_speed = ts.value();                                        // :332
        total_flops = (double)(t.pre_flops[n] - t.pre_flops[0]);         // :333
        if (total_flops == 0.0) total_flops = 1.0;
    }
    total_speed = __shfl_sync(0xffffffffu, total_speed, 0);
    total_flops = __shfl_sync(0xffffffffu, total_flops, 0);
    for (int w = lane; w < nw; w += 32) acc[w] = (total_flops * t.speed[w]) / total_speed;
    __syncwarp();
    if (lane == 0) {
        double a = 0.0;
        for (int w = 0; w < nw; ++w) { a = a + acc[w]; acc[w] = a; }    // :343, in order
    }
    __syncwarp();
    for (int w = lane; w < nw; w += 32) {
        const double aw = acc[w];
        int lo = 1, hi = n;
        while (lo < hi) {
            const int mid = (lo + hi) >> 1;
            if ((double)t.pre_flops[mid] >= aw) hi = mid; else lo = mid + 1;
        }
        bounds[w + 1] = lo;                                              // e*, overwritten in order below
    }
    __syncwarp();
    int nr = 0;
    if (lane == 0) {
        int start = 0;
        bounds[0] = 0;
        for (int wi = 0; wi < p; ++wi) {                                 // :337
            if (start >= n) break;
            int end;
            if (wi == p - 1) end = n;
            else {
                end = bounds[wi + 1] > start + 1 ? bounds[wi + 1] : start + 1;   // :344-346
                const int lim = n - (p - wi - 1);
                end = end < lim ? end : lim;
                end = end > start + 1 ? end : start + 1;                 // :348
            }
            peers[nr] = wi;
            bounds[++nr] = end;
            start = end;
        }
    }
    return __shfl_sync(0xffffffffu, nr, 0);
}

// _evaluate + Eq. 3/4 (scheduling.py:210-232, pipeline.py:41-62) over runs
// bounds[0..r] / peers[0..r) in shared memory, one warp; `loads` is r
// doubles of scratch.  hs/hp (optional): the scenario's staged tables (the
// hill climb's fast path) — then run costs come from shared memory.
__device__ void epilogue_runs(const dm_tables& t, int r, const int32_t* bounds, const int32_t* peers, double* loads,
                              int lane, int64_t n_batches, int64_t spb, double* ob, const HillStage* hs,
                              const HillPeer* hp) {
    int first_bad = 0x7fffffff, bad_code = 0;
    double mk = 0.0, bn = 0.0;
    for (int q = lane; q < r; q += 32) {
        int a = bounds[q], b = bounds[q + 1], w = peers[q];
        double c, rd;
        int v;
        if (hs) {
            const HillStage& A = hs[a];
            const HillStage& B = hs[b];
            const HillPeer& P = hp[w];
            v = (B.pg - A.pg > P.cg) ? DM_V_GPU : (B.pc - A.pc > P.cc) ? DM_V_CPU : (B.pd - A.pd > P.cd) ? DM_V_DISK : 0;
            c = (B.pf - A.pf) / P.speed;
            rd = (include_comm(t) && a > 0) ? A.R : 0.0;
        } else {
            v = cap_violation(t, w, a, b);
            int prev = q > 0 ? peers[q - 1] : -1;
            if (chain(t)) run_cost_contig(t, a, b, w, [&](int) { return prev; }, c, rd);
            else { BoundsOwner own{bounds, peers, r}; run_cost_contig(t, a, b, w, own, c, rd); }
        }
        if (v && q < first_bad) { first_bad = q; bad_code = v; }
        double load = c + rd;
        // Python type of p.compute_s + p.read_s: numpy when the speed, the
        // FLOPs or (for a run with a crossing read) the link values are
        // (sum() over them then turns naive, see PySum)
        bool np_load = (t.peer_np && t.peer_np[w]) || np_flops(t);
        if (np_comm(t) && include_comm(t)) {
            if (chain(t)) np_load |= a > 0 && t.edge_ptr[a + 1] > t.edge_ptr[a];
            else for (int i = a; i < b && !np_load; ++i)
                for (int e = t.edge_ptr[i]; e < t.edge_ptr[i + 1]; ++e)
                    if (t.edge_src[e] < a || t.edge_src[e] >= b) { np_load = true; break; }
        }
        loads[q] = np_load ? -load : load;    // loads are >= 0 (or NaN): the sign bit flags a numpy item
        mk = load > mk ? load : mk;
        double m = c >= rd ? c : rd;          // max(p.compute_s, p.read_s) pipeline.py:50
        bn = m > bn ? m : bn;
    }
    mk = warp_max(mk);
    bn = warp_max(bn);
    for (int off = 16; off > 0; off >>= 1) {
        int of = __shfl_xor_sync(0xffffffffu, first_bad, off);
        int oc = __shfl_xor_sync(0xffffffffu, bad_code, off);
        if (of < first_bad) { first_bad = of; bad_code = oc; }
    }
    __syncwarp();
    if (lane == 0) {
        PySum lat;                                 // fp_latency, builtin sum :43
        for (int q = 0; q < r; ++q) {
            const double v = loads[q];
            lat.add(fabs(v), !signbit(v));
        }
        double latency = lat.value();
        double fill = (double)(n_batches - 1) * bn;   // (n_b - 1) * bottleneck :56
        double pipe = latency + fill;
        double thr = (double)(n_batches * spb) / pipe; // :62
        ob[0] = mk; ob[1] = latency; ob[2] = bn; ob[3] = pipe; ob[4] = thr; ob[5] = (double)bad_code;
    }
}

__global__ void __maxnreg__(168) prop_hill_kernel(
        const dm_tables* __restrict__ tables, int32_t n_scen, int32_t n_max, const int16_t* __restrict__ init_owner,
        const uint8_t* __restrict__ do_hill, int16_t* out_owner, double* out_score, int32_t* out_moves,
        double* epi_out, int64_t n_batches, int64_t spb) {
    extern __shared__ __align__(16) unsigned char shb[];
    const int lane = threadIdx.x & 31, wl = threadIdx.x >> 5;
    unsigned char* mine = shb + (size_t)wl * hill_warp_bytes(n_max);
    HillStage* hs = reinterpret_cast<HillStage*>(mine + hill_core_bytes(n_max));
    HillPeer* hp = reinterpret_cast<HillPeer*>(hs + n_max + 1);
    double* fls = reinterpret_cast<double*>(mine);                   // [n_max] the scenario's stage flops
    double* lr = fls + n_max;                                         // [n_max + 1] run loads
    double* pm = lr + n_max + 1;                                      // [n_max + 1] prefix max of the loads
    double* sm = pm + n_max + 1;                                      // [n_max + 1] suffix max
    int32_t* bounds = reinterpret_cast<int32_t*>(sm + n_max + 1);     // [n_max + 2]
    int32_t* peers = bounds + (n_max + 2);                            // [n_max + 2]
    uint8_t* bd = reinterpret_cast<uint8_t*>(peers + (n_max + 2));    // [n_max + 1] run fails _fits
    const int gw = blockIdx.x * kWarpsPerCta + wl, nw = gridDim.x * kWarpsPerCta;
    for (int sc = gw; sc < n_scen; sc += nw) {
        const dm_tables t = tables[sc];
        const int n = t.n;
        __syncwarp();
        const bool comm = include_comm(t);
        const bool fast = flops_exact(t) && bytes_exact(t) && chain(t) && !(comm && pair_links(t)) &&
                          t.p <= kHillPeers && !np_comm(t);
        if (fast) {                                   // stage the scenario's tables for the hill climb
            for (int i = lane; i <= n; i += 32) {
                HillStage h;
                h.pf = (double)t.pre_flops[i]; h.pg = (double)t.pre_gpu[i];
                h.pc = (double)t.pre_cpu[i]; h.pd = (double)t.pre_disk[i];
                double rd = 0.0;
                if (comm && i < n)
                    for (int e = t.edge_ptr[i]; e < t.edge_ptr[i + 1]; ++e)
                        rd = __dadd_rn(rd, comm_time(t.def_alpha, t.def_beta, t.edge_m[e]));
                h.R = rd;
                hs[i] = h;
            }
            for (int w = lane; w < t.p; w += 32) {
                HillPeer h;
                h.speed = t.speed[w]; h.cg = t.cap_gpu[w]; h.cc = t.cap_cpu[w]; h.cd = t.cap_disk[w];
                hp[w] = h;
            }
        }
        int r = 0;
        const bool pwarp = !init_owner && flops_exact(t);
        if (!init_owner && !pwarp) for (int i = lane; i < n; i += 32) fls[i] = t.flops[i];
        __syncwarp();
        if (pwarp) r = proportional_warp(t, bounds, peers, pm, lane);
        else if (lane == 0) {
            if (init_owner) {
                const int16_t* o = init_owner + (size_t)sc * n_max;
                bounds[0] = 0; peers[0] = o[0];
                for (int i = 1; i < n; ++i) if (o[i] != o[i - 1]) { bounds[++r] = i; peers[r] = o[i]; }
                bounds[++r] = n;
            } else {
                r = proportional(t, bounds, peers, fls);
            }
        }
        r = __shfl_sync(0xffffffffu, r, 0);
        __syncwarp();
        // only the two runs at a moved boundary change unless reads depend on
        // which run owns a source (pair links on DAG stages)
        const bool incr = chain(t) || !include_comm(t) || !pair_links(t);
        double cur;
        if (fast) {                                                        // :365 on the staged tables
            const double inf = __longlong_as_double(0x7ff0000000000000LL);
            bool anybad = false;
            double best = 0.0;
            for (int q = lane; q < r; q += 32) {
                bool b_;
                const double load = run_load_staged(hs, hp, bounds[q], bounds[q + 1], peers[q], comm, b_);
                lr[q] = load; bd[q] = b_;
                anybad |= b_;
                if (!b_) best = load > best ? load : best;
            }
            __syncwarp();
            cur = __any_sync(0xffffffffu, anybad) ? inf : warp_max(best);
        } else {
            cur = incr ? hill_score(t, r, bounds, peers, lane, lr, bd) : hill_score(t, r, bounds, peers, lane);
        }
        int moves = 0;
        if ((!do_hill || do_hill[sc]) && incr) {
            // The reference walks moves (a, dir) in order and takes the first
            // that improves (:366-387); until one does, every move is scored
            // from the same state, so the lanes score 32 moves at a time:
            // score = max(0, loads before a, loads after a+1, the two new
            // loads) from prefix / suffix maxima (+inf marks a run failing
            // _fits), the first improving move in order is applied and the
            // walk resumes after it from the new state.
            const double inf = __longlong_as_double(0x7ff0000000000000LL);
            const int Lend = 2 * (r - 1);
            int round = 0, L0 = 0;
            bool improved = false;
            while (true) {
                {   // warp max-scans, 32 runs at a time (max is exact in any order)
                    double carry = 0.0;
                    for (int base = 0; base < r; base += 32) {
                        const int q = base + lane;
                        double v = q < r ? (bd[q] ? inf : lr[q]) : 0.0;
                        for (int off = 1; off < 32; off <<= 1) {
                            const double o = __shfl_up_sync(0xffffffffu, v, off);
                            if (lane >= off) v = o > v ? o : v;
                        }
                        v = carry > v ? carry : v;
                        if (q < r) pm[q] = v;
                        carry = __shfl_sync(0xffffffffu, v, 31);
                    }
                    carry = 0.0;
                    for (int top = r - 1; top >= 0; top -= 32) {
                        const int q = top - lane;
                        double v = q >= 0 ? (bd[q] ? inf : lr[q]) : 0.0;
                        for (int off = 1; off < 32; off <<= 1) {
                            const double o = __shfl_up_sync(0xffffffffu, v, off);
                            if (lane >= off) v = o > v ? o : v;
                        }
                        v = carry > v ? carry : v;
                        if (q >= 0) sm[q] = v;
                        carry = __shfl_sync(0xffffffffu, v, 31);
                    }
                }
                __syncwarp();
                int found = -1, fnb = 0;
                double fcs = 0.0, fva = 0.0, fvb = 0.0;
                bool fba = false, fbb = false;
                for (int base = L0; base < Lend && found < 0; base += 32) {
                    const int L = base + lane;
                    bool imp = false, ba = false, bb = false;
                    double cs = inf, va = 0.0, vb = 0.0;
                    int nb = 0;
                    if (L < Lend) {
                        const int a = L >> 1, dir = L & 1;
                        const int la = bounds[a + 1] - bounds[a], lb = bounds[a + 2] - bounds[a + 1];
                        if ((dir == 0 && la > 1) || (dir == 1 && lb > 1)) {                      // :373-376
                            nb = dir == 0 ? bounds[a + 1] - 1 : bounds[a + 1] + 1;
                            if (fast) {
                                va = run_load_staged(hs, hp, bounds[a], nb, peers[a], comm, ba);
                                vb = run_load_staged(hs, hp, nb, bounds[a + 2], peers[a + 1], comm, bb);
                            } else {
                                va = run_load_ab(t, bounds[a], nb, peers[a], a > 0 ? peers[a - 1] : -1, ba);
                                vb = run_load_ab(t, nb, bounds[a + 2], peers[a + 1], peers[a], bb);
                            }
                            double sc2 = 0.0;
                            if (a > 0) sc2 = pm[a - 1] > sc2 ? pm[a - 1] : sc2;
                            if (a + 2 < r) sc2 = sm[a + 2] > sc2 ? sm[a + 2] : sc2;
                            const double xa = ba ? inf : va, xb = bb ? inf : vb;
                            sc2 = xa > sc2 ? xa : sc2;
                            sc2 = xb > sc2 ? xb : sc2;
                            cs = sc2;
                            imp = cs < cur - 1e-15;                                              // :383
                        }
                    }
                    const unsigned bal = __ballot_sync(0xffffffffu, imp);
                    if (bal) {
                        const int src = __ffs(bal) - 1;
                        found = base + src;
                        fcs = __shfl_sync(0xffffffffu, cs, src);
                        fva = __shfl_sync(0xffffffffu, va, src);
                        fvb = __shfl_sync(0xffffffffu, vb, src);
                        fba = __shfl_sync(0xffffffffu, (int)ba, src);
                        fbb = __shfl_sync(0xffffffffu, (int)bb, src);
                        fnb = __shfl_sync(0xffffffffu, nb, src);
                    }
                }
                if (found >= 0) {                                                                // :384-385
                    const int a = found >> 1;
                    __syncwarp();
                    if (lane == 0) { bounds[a + 1] = fnb; lr[a] = fva; lr[a + 1] = fvb; bd[a] = fba; bd[a + 1] = fbb; }
                    __syncwarp();
                    cur = fcs; improved = true; ++moves;
                    L0 = found + 1;
                    continue;
                }
                ++round;                                                                         // :386-387
                if (!improved || round >= 200) break;
                improved = false;
                L0 = 0;
            }
        } else if (!do_hill || do_hill[sc]) {
            for (int round = 0; round < 200; ++round) {                   // :366
                bool improved = false;
                for (int a = 0; a + 1 < r; ++a) {                         // :368-369
                    for (int dir = 0; dir < 2; ++dir) {                   // :370
                        int la = bounds[a + 1] - bounds[a], lb = bounds[a + 2] - bounds[a + 1];
                        int nb;
                        if (dir == 0 && la > 1) nb = bounds[a + 1] - 1;   // :373-374
                        else if (dir == 1 && lb > 1) nb = bounds[a + 1] + 1;  // :375-376
                        else continue;
                        int old = bounds[a + 1];
                        __syncwarp();
                        if (lane == 0) bounds[a + 1] = nb;
                        __syncwarp();
                        double cs = hill_score(t, r, bounds, peers, lane);
                        if (cs < cur - 1e-15) { cur = cs; improved = true; ++moves; }  // :383-385
                        else {
                            __syncwarp();
                            if (lane == 0) bounds[a + 1] = old;
                            __syncwarp();
                        }
                    }
                }
                if (!improved) break;                                     // :386-387
            }
        }
        __syncwarp();
        int16_t* o = out_owner + (size_t)sc * n_max;
        for (int i = lane; i < n; i += 32) {          // each stage's run by binary search over the bounds
            int lo = 0, hi = r - 1;
            while (lo < hi) {
                const int mid = (lo + hi + 1) >> 1;
                if (bounds[mid] <= i) lo = mid; else hi = mid - 1;
            }
            o[i] = (int16_t)peers[lo];
        }
        for (int i = n + lane; i < n_max; i += 32) o[i] = -1;
        if (lane == 0) { out_score[sc] = cur; if (out_moves) out_moves[sc] = moves; }
        if (epi_out)                                  // fused epilogue on the final runs (pm is free scratch now)
            epilogue_runs(t, r, bounds, peers, pm, lane, n_batches, spb, epi_out + (size_t)sc * 6,
                          fast ? hs : nullptr, hp);
    }
}

// ------------------------------------------------------------- epilogue
__global__ void __launch_bounds__(32 * kWarpsPerCta) epilogue_kernel(
        const dm_tables* __restrict__ tables, int32_t n_scen, int32_t n_max, const int16_t* __restrict__ owner,
        int64_t n_batches, int64_t spb, double* out) {
    extern __shared__ int32_t sh[];
    const int lane = threadIdx.x & 31, wl = threadIdx.x >> 5;
    int32_t* bounds = sh + (size_t)wl * 2 * (n_max + 2);
    int32_t* peers = bounds + (n_max + 2);
    double* loads = reinterpret_cast<double*>(sh + (size_t)kWarpsPerCta * 2 * (n_max + 2)) + (size_t)wl * (n_max + 1);
    const int gw = blockIdx.x * kWarpsPerCta + wl, nw = gridDim.x * kWarpsPerCta;
    for (int sc = gw; sc < n_scen; sc += nw) {
        const dm_tables t = tables[sc];
        const int n = t.n;
        const int16_t* o = owner + (size_t)sc * n_max;
        if (n <= 0 || o[0] < 0 || o[0] >= t.P) {       // no assignment (unscheduled / DP-infeasible row)
            if (lane == 0) {
                double* ob = out + (size_t)sc * 6;
                const double nan = __longlong_as_double(0x7ff8000000000000LL);
                ob[0] = nan; ob[1] = nan; ob[2] = nan; ob[3] = nan; ob[4] = nan; ob[5] = -1.0;
            }
            continue;
        }
        __syncwarp();
        int r = 0;                                     // runs from the owner row, 32 stages at a time
        for (int base = 0; base < n; base += 32) {
            const int i = base + lane;
            const int oi = i < n ? o[i] : -1;
            const bool start = i < n && (i == 0 || oi != o[i - 1]);
            const unsigned bal = __ballot_sync(0xffffffffu, start);
            if (start) {
                const int k = r + __popc(bal & ((1u << lane) - 1u));
                bounds[k] = i;
                peers[k] = oi;
            }
            r += __popc(bal);
        }
        if (lane == 0) bounds[r] = n;
        __syncwarp();
        epilogue_runs(t, r, bounds, peers, loads, lane, n_batches, spb, out + (size_t)sc * 6, nullptr, nullptr);
    }
}

}  // namespace dm

namespace {
int hill_grid(int32_t n_scen) {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    int64_t g = (int64_t)sms * 16;
    int64_t need = (n_scen + dm::kWarpsPerCta - 1) / dm::kWarpsPerCta;
    return (int)(g < need ? g : need);
}
}  // namespace

extern "C" {

int dm_prop_hill(const dm_tables* tables, int32_t n_scen, int32_t n_max, const int16_t* init_owner,
                 const uint8_t* do_hill, int16_t* out_owner, double* out_score, int32_t* out_moves, void* stream) {
    if (!tables || n_scen < 0 || n_max <= 0 || !out_owner || !out_score) return dmabi::fail(DM_E_ARG, "dm_prop_hill: bad arguments");
    if (n_scen == 0) return DM_OK;
    size_t smem = (size_t)dm::kWarpsPerCta * dm::hill_warp_bytes(n_max);
    if (smem > 200 * 1024) return dmabi::fail(DM_E_TOO_LARGE, "dm_prop_hill: too many stages");
    cudaFuncSetAttribute(dm::prop_hill_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    dm::prop_hill_kernel<<<hill_grid(n_scen), 32 * dm::kWarpsPerCta, smem, (cudaStream_t)stream>>>(
        tables, n_scen, n_max, init_owner, do_hill, out_owner, out_score, out_moves, nullptr, 1, 1);
    DM_CHECK_LAUNCH();
    return DM_OK;
}

int dm_prop_hill_epilogue(const dm_tables* tables, int32_t n_scen, int32_t n_max, const int16_t* init_owner,
                          const uint8_t* do_hill, int16_t* out_owner, double* out_score, int32_t* out_moves,
                          int64_t n_batches, int64_t samples_per_batch, double* out, void* stream) {
    if (!tables || n_scen < 0 || n_max <= 0 || !out_owner || !out_score || !out)
        return dmabi::fail(DM_E_ARG, "dm_prop_hill_epilogue: bad arguments");
    if (n_scen == 0) return DM_OK;
    size_t smem = (size_t)dm::kWarpsPerCta * dm::hill_warp_bytes(n_max);
    if (smem > 200 * 1024) return dmabi::fail(DM_E_TOO_LARGE, "dm_prop_hill_epilogue: too many stages");
    cudaFuncSetAttribute(dm::prop_hill_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    dm::prop_hill_kernel<<<hill_grid(n_scen), 32 * dm::kWarpsPerCta, smem, (cudaStream_t)stream>>>(
        tables, n_scen, n_max, init_owner, do_hill, out_owner, out_score, out_moves, out, n_batches,
        samples_per_batch);
    DM_CHECK_LAUNCH();
    return DM_OK;
}

int dm_pipeline_epilogue(const dm_tables* tables, int32_t n_scen, int32_t n_max, const int16_t* owner,
                         int64_t n_batches, int64_t samples_per_batch, double* out, void* stream) {
    if (!tables || n_scen < 0 || n_max <= 0 || !owner || !out) return dmabi::fail(DM_E_ARG, "dm_pipeline_epilogue: bad arguments");
    if (n_scen == 0) return DM_OK;
    size_t smem = (size_t)dm::kWarpsPerCta * 2 * (n_max + 2) * sizeof(int32_t) +
                  (size_t)dm::kWarpsPerCta * (n_max + 1) * sizeof(double) + 16;
    if (smem > 200 * 1024) return dmabi::fail(DM_E_TOO_LARGE, "dm_pipeline_epilogue: too many stages");
    cudaFuncSetAttribute(dm::epilogue_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    dm::epilogue_kernel<<<hill_grid(n_scen), 32 * dm::kWarpsPerCta, smem, (cudaStream_t)stream>>>(
        tables, n_scen, n_max, owner, n_batches, samples_per_batch, out);
    DM_CHECK_LAUNCH();
    return DM_OK;
}

}  // extern "C"
