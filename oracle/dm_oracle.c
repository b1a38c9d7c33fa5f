/*
 * dm_oracle.c — CPU restatement of the dagmesh scheduling hot path.
 *
 *   *** TEST INFRASTRUCTURE ONLY ***
 *   Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 *   --impl reference leg may load this library, and only as the checker or
 *   the timed CPU baseline.  The product (paper_2309_01172_b200) never links
 *   or calls it.
 *
 * Every function restates one reference function of
 * /root/reference/pkg/src/dagmesh/scheduling.py (or hardware.py / pipeline.py)
 * with the same loop order, the same rounding sequence (IEEE binary64, no FMA
 * contraction: build with -ffp-contract=off) and the same tie-break rules.
 * Parity of this restatement is pinned by tests/test_oracle_golden.py against
 * fixtures produced by the reference itself (tests/golden/make_golden.py).
 *
 * Stage/fleet data come in the dm_tables layout of include/dagmesh_b200.h
 * (host pointers here).
 */
#include "../include/dagmesh_b200.h"

#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define EXPORT __attribute__((visibility("default")))

/* ------------------------------------------------------------------ sums */

/* CPython 3.12 builtin sum() over float items (Python/bltinmodule.c,
 * builtin_sum_impl): the int start 0 is promoted by the first float item
 * (0 + x0), then Neumaier-compensated accumulation; the compensation is added
 * at the end when it is non-zero and finite.  Used where the reference calls
 * sum() over Python floats: scheduling.py:160,174-176,200,295,332-333,
 * pipeline.py:43. */
/* The same sum() when some items are not exact `float` objects
 * (numpy.float64; np_item[i] != 0): builtin_sum_impl leaves its float fast
 * path at the first such item, adding the compensation gathered so far, and
 * adds every later item with plain `+`.  np_item == NULL: all exact floats. */
EXPORT double or_py_sum_items(const double* x, const uint8_t* np_item, int64_t k) {
    if (k <= 0) return 0.0;
    double f = 0.0 + x[0];
    double c = 0.0;
    int naive = np_item && np_item[0];
    for (int64_t i = 1; i < k; ++i) {
        double v = x[i];
        if (!naive && np_item && np_item[i]) {
            if (c != 0.0 && isfinite(c)) f += c;
            naive = 1;
        }
        if (naive) { f = f + v; continue; }
        double t = f + v;
        if (fabs(f) >= fabs(v)) c += (f - t) + v;
        else c += (v - t) + f;
        f = t;
    }
    if (!naive && c != 0.0 && isfinite(c)) f += c;
    return f;
}

EXPORT double or_py_sum(const double* x, int64_t k) {
    return or_py_sum_items(x, NULL, k);
}

/* Python sum over the items col[idx[0..k)] (in that order). */
static double col_sum_idx(const double* col, const int64_t* pre, int exact,
                          const int32_t* idx, int k, int np_items) {
    if (exact) {
        int64_t s = 0;
        for (int q = 0; q < k; ++q) s += (pre[idx[q] + 1] - pre[idx[q]]);
        return (double)s;
    }
    if (k <= 0) return 0.0;
    if (np_items) {                       /* sum() over numpy items: plain + */
        double f = 0.0 + col[idx[0]];
        for (int q = 1; q < k; ++q) f = f + col[idx[q]];
        return f;
    }
    double f = 0.0 + col[idx[0]], c = 0.0;
    for (int q = 1; q < k; ++q) {
        double v = col[idx[q]], t = f + v;
        if (fabs(f) >= fabs(v)) c += (f - t) + v; else c += (v - t) + f;
        f = t;
    }
    if (c != 0.0 && isfinite(c)) f += c;
    return f;
}

/* Python sum over col[a..b) in index order. */
static double col_sum_range(const double* col, const int64_t* pre, int exact,
                            int a, int b, int np_items) {
    if (exact) return (double)(pre[b] - pre[a]);
    if (b <= a) return 0.0;
    if (np_items) {
        double f = 0.0 + col[a];
        for (int i = a + 1; i < b; ++i) f = f + col[i];
        return f;
    }
    return or_py_sum(col + a, b - a);
}

static inline int flops_exact(const dm_tables* t) { return (t->flags & DM_F_FLOPS_EXACT) != 0; }
static inline int bytes_exact(const dm_tables* t) { return (t->flags & DM_F_BYTES_EXACT) != 0; }
static inline int np_flops(const dm_tables* t) { return (t->flags & DM_F_NP_FLOPS) != 0; }
static inline int np_bytes(const dm_tables* t) { return (t->flags & DM_F_NP_BYTES) != 0; }

/* hardware.Fleet.link_between (hardware.py:136-140) resolved to indices;
 * owner indices outside [0, P) are peers unknown to the fleet (default link). */
static inline void link_of(const dm_tables* t, int a, int b, double* al, double* be) {
    if (a == b) { *al = 0.0; *be = 0.0; return; }
    if ((t->flags & DM_F_PAIR_LINKS) && a >= 0 && a < t->P && b >= 0 && b < t->P) {
        *al = t->link_alpha[(int64_t)a * t->P + b];
        *be = t->link_beta[(int64_t)a * t->P + b];
        return;
    }
    *al = t->def_alpha; *be = t->def_beta;
}

/* hardware.comm_time (hardware.py:147-150): alpha + beta*M, two roundings. */
static inline double comm_time(double al, double be, double m) {
    return al + be * m;   /* built with -ffp-contract=off: no FMA */
}

/* ------------------------------------------------------------- _run_cost */

/* scheduling._run_cost (scheduling.py:156-169) for one run whose stage
 * indices idx[0..k) are iterated in the given order.  peer_of[i] is the owner
 * of stage i (-1 = unassigned, >= P = unknown peer). */
static int run_cost(const dm_tables* t, const int32_t* peer_of, int peer,
                    const int32_t* idx, int k, uint8_t* inside,
                    double* compute, double* read) {
    if (peer < 0 || peer >= t->P) return DM_E_UNKNOWN_PEER;  /* fleet.peer :158 */
    double speed = t->speed[peer];                              /* :159 */
    double fl = col_sum_idx(t->flops, t->pre_flops, flops_exact(t), idx, k, np_flops(t));
    *compute = fl / speed;                                      /* :160 */
    double rd = 0.0;
    if (t->flags & DM_F_INCLUDE_COMM) {                         /* :162 */
        for (int q = 0; q < k; ++q) inside[idx[q]] = 1;         /* :163 */
        for (int q = 0; q < k; ++q) {                           /* :164 */
            int i = idx[q];
            for (int e = t->edge_ptr[i]; e < t->edge_ptr[i + 1]; ++e) {  /* :165 */
                int src = t->edge_src[e];
                if (!inside[src]) {                             /* :166 */
                    int own = peer_of[src];
                    if (own == -1) {                            /* peer_of[src] KeyError */
                        for (int z = 0; z < k; ++z) inside[idx[z]] = 0;
                        return DM_E_UNASSIGNED;
                    }
                    double al, be;
                    link_of(t, own, peer, &al, &be);            /* :167 */
                    rd += comm_time(al, be, t->edge_m[e]);      /* :168 */
                }
            }
        }
        for (int q = 0; q < k; ++q) inside[idx[q]] = 0;
    }
    *read = rd;
    return DM_OK;
}

/* scheduling._fits (scheduling.py:172-176) over the contiguous range [a, b). */
static int fits_range(const dm_tables* t, int peer, int a, int b) {
    int ex = bytes_exact(t);
    return col_sum_range(t->gpu, t->pre_gpu, ex, a, b, np_bytes(t)) <= t->cap_gpu[peer]
        && col_sum_range(t->cpu, t->pre_cpu, ex, a, b, np_bytes(t)) <= t->cap_cpu[peer]
        && col_sum_range(t->disk, t->pre_disk, ex, a, b, np_bytes(t)) <= t->cap_disk[peer];
}

/* ------------------------------------------------------ verify_assignment */

static int cmp_i32(const void* a, const void* b) {
    int32_t x = *(const int32_t*)a, y = *(const int32_t*)b;
    return (x > y) - (x < y);
}

/* scheduling.verify_assignment (scheduling.py:179-207).  Runs in CSR form
 * (run_peer[r], run_idx[run_ptr[r]..run_ptr[r+1])).  Returns DM_V_* and the
 * offending run in *bad_run. */
EXPORT int or_verify_runs(const dm_tables* t, int nr, const int32_t* run_peer,
                          const int32_t* run_ptr, const int32_t* run_idx,
                          int32_t* bad_run) {
    int n = t->n;
    int32_t* seen = (int32_t*)calloc((size_t)n, sizeof(int32_t));
    int32_t* used = (int32_t*)calloc((size_t)(nr > 0 ? nr : 1), sizeof(int32_t));
    int32_t* sorted = (int32_t*)malloc(sizeof(int32_t) * (size_t)(run_ptr[nr] + 1));
    int n_used = 0, n_seen = 0, code = DM_V_OK;
    *bad_run = -1;
    for (int r = 0; r < nr && code == DM_V_OK; ++r) {
        int k = run_ptr[r + 1] - run_ptr[r];
        if (k == 0) continue;                                    /* :184 */
        int peer = run_peer[r];
        for (int u = 0; u < n_used; ++u)
            if (used[u] == peer) { code = DM_V_TWO_RUNS; break; } /* :186 */
        if (code) { *bad_run = r; break; }
        used[n_used++] = peer;
        if (peer < 0 || peer >= t->P) { code = DM_V_UNKNOWN_PEER; *bad_run = r; break; }
        memcpy(sorted, run_idx + run_ptr[r], sizeof(int32_t) * (size_t)k);
        qsort(sorted, (size_t)k, sizeof(int32_t), cmp_i32);      /* :191 */
        for (int q = 0; q < k; ++q)
            if (sorted[q] != sorted[0] + q) { code = DM_V_NOT_CONTIGUOUS; break; }
        if (code) { *bad_run = r; break; }
        for (int q = 0; q < k; ++q) {                            /* :194-197 */
            if (seen[sorted[q]]) { code = DM_V_ASSIGNED_TWICE; break; }
            seen[sorted[q]] = 1; ++n_seen;
        }
        if (code) { *bad_run = r; break; }
        int ex = bytes_exact(t);                                  /* :199-203 */
        if (col_sum_idx(t->gpu, t->pre_gpu, ex, sorted, k, np_bytes(t)) > t->cap_gpu[peer]) code = DM_V_GPU;
        else if (col_sum_idx(t->cpu, t->pre_cpu, ex, sorted, k, np_bytes(t)) > t->cap_cpu[peer]) code = DM_V_CPU;
        else if (col_sum_idx(t->disk, t->pre_disk, ex, sorted, k, np_bytes(t)) > t->cap_disk[peer]) code = DM_V_DISK;
        if (code) *bad_run = r;
    }
    if (code == DM_V_OK && n_seen != n) code = DM_V_UNASSIGNED;  /* :204-206 */
    free(seen); free(used); free(sorted);
    return code;
}

/* ------------------------------------------------------------- _evaluate */

/* scheduling._evaluate (scheduling.py:210-232): verify, then cost every
 * non-empty run in first-stage order with sorted indices.  Per-run outputs
 * are written at the run's given position.  Returns DM_OK or the error the
 * reference raises while costing. */
EXPORT int or_eval_runs(const dm_tables* t, int nr, const int32_t* run_peer,
                        const int32_t* run_ptr, const int32_t* run_idx,
                        double* out_compute, double* out_read,
                        double* out_makespan, int32_t* out_code,
                        int32_t* out_code_run) {
    int n = t->n;
    *out_code = or_verify_runs(t, nr, run_peer, run_ptr, run_idx, out_code_run);
    int32_t* peer_of = (int32_t*)malloc(sizeof(int32_t) * (size_t)n);
    for (int i = 0; i < n; ++i) peer_of[i] = -1;
    for (int r = 0; r < nr; ++r)                                  /* :213 */
        for (int q = run_ptr[r]; q < run_ptr[r + 1]; ++q) peer_of[run_idx[q]] = run_peer[r];
    /* ordered_runs: non-empty runs stably sorted by first (min) index :217-218 */
    int32_t* order = (int32_t*)malloc(sizeof(int32_t) * (size_t)(nr + 1));
    int32_t* first = (int32_t*)malloc(sizeof(int32_t) * (size_t)(nr + 1));
    int no = 0;
    for (int r = 0; r < nr; ++r) {
        int k = run_ptr[r + 1] - run_ptr[r];
        out_compute[r] = 0.0; out_read[r] = 0.0;
        if (!k) continue;
        int mn = run_idx[run_ptr[r]];
        for (int q = run_ptr[r]; q < run_ptr[r + 1]; ++q) if (run_idx[q] < mn) mn = run_idx[q];
        int pos = no++;
        while (pos > 0 && first[pos - 1] > mn) { first[pos] = first[pos - 1]; order[pos] = order[pos - 1]; --pos; }
        first[pos] = mn; order[pos] = r;
    }
    int32_t* sorted = (int32_t*)malloc(sizeof(int32_t) * (size_t)(run_ptr[nr] + 1));
    uint8_t* inside = (uint8_t*)calloc((size_t)n, 1);
    double makespan = 0.0;
    int st = DM_OK;
    for (int o = 0; o < no && st == DM_OK; ++o) {
        int r = order[o], k = run_ptr[r + 1] - run_ptr[r];
        memcpy(sorted, run_idx + run_ptr[r], sizeof(int32_t) * (size_t)k);
        qsort(sorted, (size_t)k, sizeof(int32_t), cmp_i32);
        double c, rd;
        st = run_cost(t, peer_of, run_peer[r], sorted, k, inside, &c, &rd);
        if (st != DM_OK) break;
        out_compute[r] = c; out_read[r] = rd;
        double load = c + rd;                                     /* :221 */
        if (load > makespan) makespan = load;                     /* :222 */
    }
    *out_makespan = makespan;
    free(peer_of); free(order); free(first); free(sorted); free(inside);
    return st;
}

/* Mode A scoring: owner vector -> Runs grouped by peer in first-appearance
 * order, then _evaluate.  Returns the violation code, 0xFF for an owner index
 * outside [0, P) (FleetError in the reference). */
EXPORT int or_eval_owner(const dm_tables* t, const int32_t* owner, double* out_makespan) {
    int n = t->n;
    for (int i = 0; i < n; ++i) if (owner[i] < 0 || owner[i] >= t->P) { *out_makespan = NAN; return 0xFF; }
    int32_t* run_peer = (int32_t*)malloc(sizeof(int32_t) * (size_t)n);
    int32_t* run_ptr = (int32_t*)malloc(sizeof(int32_t) * (size_t)(n + 1));
    int32_t* run_idx = (int32_t*)malloc(sizeof(int32_t) * (size_t)n);
    int nr = 0, w = 0;
    for (int i = 0; i < n; ++i) {
        int pe = owner[i], seen = 0;
        for (int r = 0; r < nr; ++r) if (run_peer[r] == pe) { seen = 1; break; }
        if (!seen) run_peer[nr++] = pe;
    }
    for (int r = 0; r < nr; ++r) {
        run_ptr[r] = w;
        for (int i = 0; i < n; ++i) if (owner[i] == run_peer[r]) run_idx[w++] = i;
    }
    run_ptr[nr] = w;
    double* c = (double*)malloc(sizeof(double) * (size_t)(nr + 1));
    double* rd = (double*)malloc(sizeof(double) * (size_t)(nr + 1));
    int32_t code, bad;
    or_eval_runs(t, nr, run_peer, run_ptr, run_idx, c, rd, out_makespan, &code, &bad);
    free(run_peer); free(run_ptr); free(run_idx); free(c); free(rd);
    return code;
}

/* --------------------------------------------------- brute-force family */

/* Score of a contiguous assignment given as bounds[0..r] and peers[0..r):
 * the inner body of brute_force_schedule (scheduling.py:266-270).
 * Returns 0 if some run fails _fits, else 1 with *mk = max over runs of
 * sum(_run_cost) (sum of the 2-tuple equals compute + read exactly). */
static int score_contiguous(const dm_tables* t, int r, const int32_t* bounds,
                            const int32_t* peers, int32_t* peer_of,
                            int32_t* idxbuf, uint8_t* inside, double* mk) {
    for (int q = 0; q < r; ++q)                                   /* :266 */
        if (!fits_range(t, peers[q], bounds[q], bounds[q + 1])) return 0;
    for (int q = 0; q < r; ++q)                                   /* :268 */
        for (int i = bounds[q]; i < bounds[q + 1]; ++i) peer_of[i] = peers[q];
    double best = 0.0; int have = 0;
    for (int q = 0; q < r; ++q) {                                 /* :269-270 */
        int k = bounds[q + 1] - bounds[q];
        for (int z = 0; z < k; ++z) idxbuf[z] = bounds[q] + z;
        double c, rd;
        run_cost(t, peer_of, peers[q], idxbuf, k, inside, &c, &rd);
        double load = c + rd;
        if (!have || load > best) { best = load; have = 1; }
    }
    *mk = best;
    return 1;
}

static double binom_d(int n, int k) {
    if (k < 0 || k > n) return 0.0;
    double r = 1.0;
    for (int i = 1; i <= k; ++i) r = r * (double)(n - k + i) / (double)i;
    return floor(r + 0.5);
}
static int64_t binom(int n, int k) { return (int64_t)binom_d(n, k); }
static int64_t perm(int p, int r) { int64_t v = 1; for (int i = 0; i < r; ++i) v *= (p - i); return v; }

/* Lexicographic unranking of combination c of (r-1) cut positions from
 * {1..n-1} (itertools.combinations order). */
static void unrank_comb(int n, int m, int64_t c, int32_t* cuts) {
    int lo = 1;
    for (int q = 0; q < m; ++q) {
        for (int v = lo; v <= n - 1; ++v) {
            int64_t cnt = binom((n - 1) - v, m - q - 1);
            if (c < cnt) { cuts[q] = v; lo = v + 1; break; }
            c -= cnt;
        }
    }
}

/* Lexicographic unranking of partial permutation pi of r items from p
 * (itertools.permutations order). */
static void unrank_perm(int p, int r, int64_t pi, int32_t* out) {
    uint8_t used[1024];
    memset(used, 0, (size_t)p);
    for (int q = 0; q < r; ++q) {
        int64_t blk = perm(p - q - 1, r - q - 1);
        int64_t d = pi / blk; pi -= d * blk;
        for (int v = 0; v < p; ++v) {
            if (used[v]) continue;
            if (d == 0) { out[q] = v; used[v] = 1; break; }
            --d;
        }
    }
}

typedef struct { double mk; int64_t rank; int64_t n_eval, n_feas; uint64_t csum; } or_win;

static void win_update(or_win* w, double mk, int64_t k) {
    w->n_feas++;
    uint64_t bits; memcpy(&bits, &mk, 8);
    w->csum += bits;
    if (w->rank < 0 || mk < w->mk) { w->mk = mk; w->rank = k; }  /* :271 strict < */
}

/* brute_force_schedule (scheduling.py:245-278) restricted to global ranks
 * [k0, k1); mode 0 = full order (permutations), mode 1 = identity-order
 * splits (run q on worker q). */
EXPORT void or_enum(const dm_tables* t, int mode, int64_t k0, int64_t k1, dm_winner* out) {
    int n = t->n, p = t->p, rmax = n < p ? n : p;
    int32_t bounds[1100], peers[1100], cuts[1100];
    int32_t* peer_of = (int32_t*)malloc(sizeof(int32_t) * (size_t)n);
    int32_t* idxbuf = (int32_t*)malloc(sizeof(int32_t) * (size_t)n);
    uint8_t* inside = (uint8_t*)calloc((size_t)n, 1);
    or_win w = {INFINITY, -1, 0, 0, 0};
    int64_t base = 0;
    for (int r = 1; r <= rmax; ++r) {
        int64_t nc = binom(n - 1, r - 1), np = mode == 0 ? perm(p, r) : 1, blk = nc * np;
        if (k1 <= base) break;
        if (k0 >= base + blk) { base += blk; continue; }
        int64_t lo = k0 > base ? k0 - base : 0, hi = (k1 < base + blk ? k1 : base + blk) - base;
        int64_t have_c = -1;
        for (int64_t kk = lo; kk < hi; ++kk) {
            int64_t c = kk / np, pi = kk % np;
            if (have_c < 0) unrank_comb(n, r - 1, c, cuts);
            else if (c != have_c) {
                /* itertools.combinations successor: bump the rightmost cut
                 * that can move, reset the ones after it */
                int m = r - 1, i = m - 1;
                while (i >= 0 && cuts[i] == n - 1 - (m - 1 - i)) --i;
                cuts[i]++;
                for (int j = i + 1; j < m; ++j) cuts[j] = cuts[j - 1] + 1;
            }
            have_c = c;
            bounds[0] = 0;
            for (int q = 0; q < r - 1; ++q) bounds[q + 1] = cuts[q];
            bounds[r] = n;
            if (mode == 0) unrank_perm(p, r, pi, peers);
            else for (int q = 0; q < r; ++q) peers[q] = q;
            double mk;
            w.n_eval++;
            if (score_contiguous(t, r, bounds, peers, peer_of, idxbuf, inside, &mk))
                win_update(&w, mk, base + kk);
        }
        base += blk;
    }
    out->makespan = w.mk; out->rank = w.rank; out->n_evaluated = w.n_eval;
    out->n_feasible = w.n_feas; out->checksum = w.csum;
    free(peer_of); free(idxbuf); free(inside);
}

/* Decode global rank k of mode (0 full, 1 splits) into bounds/peers; returns r. */
EXPORT int or_unrank(const dm_tables* t, int mode, int64_t k, int32_t* bounds, int32_t* peers) {
    int n = t->n, p = t->p, rmax = n < p ? n : p;
    int32_t cuts[1100];
    for (int r = 1; r <= rmax; ++r) {
        int64_t nc = binom(n - 1, r - 1), np = mode == 0 ? perm(p, r) : 1, blk = nc * np;
        if (k >= blk) { k -= blk; continue; }
        unrank_comb(n, r - 1, k / np, cuts);
        bounds[0] = 0;
        for (int q = 0; q < r - 1; ++q) bounds[q + 1] = cuts[q];
        bounds[r] = n;
        if (mode == 0) unrank_perm(p, r, k % np, peers);
        else for (int q = 0; q < r; ++q) peers[q] = q;
        return r;
    }
    return 0;
}

/* ---------------------------------------------------- random placements */

/* Candidate k of the random-placement stream (configs C3/C5; the recipe is
 * documented in paper_2309_01172_b200/rng.py and restated in
 * csrc/dm_random.cu): xoshiro128** seeded from (seed, k), r ~ U{1..rmax},
 * Knuth's selection sampling for the r-1 cut positions, a keyed 4-round
 * Feistel permutation (cycle walking) of the online peers. */
static inline uint64_t fmix64(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}
static inline uint32_t rotl32(uint32_t x, int r) { return (x << r) | (x >> (32 - r)); }
typedef struct { uint32_t s[4]; } xo128;
static void xo_seed(xo128* g, uint64_t key, int64_t k) {
    uint64_t za = fmix64(key + 2ULL * (uint64_t)k + 1ULL), zb = fmix64(key + 2ULL * (uint64_t)k + 2ULL);
    g->s[0] = (uint32_t)za; g->s[1] = (uint32_t)(za >> 32); g->s[2] = (uint32_t)zb; g->s[3] = (uint32_t)(zb >> 32);
    if (!(g->s[0] | g->s[1] | g->s[2] | g->s[3])) g->s[0] = 1;
}
static inline uint32_t xo_next(xo128* g) {
    uint32_t* s = g->s;
    uint32_t res = rotl32(s[1] * 5u, 7) * 9u, t = s[1] << 9;
    s[2] ^= s[0]; s[3] ^= s[1]; s[1] ^= s[2]; s[0] ^= s[3]; s[2] ^= t; s[3] = rotl32(s[3], 11);
    return res;
}
static inline uint32_t mulhi32(uint32_t u, uint32_t m) { return (uint32_t)(((uint64_t)u * m) >> 32); }
static int feistel_h(int32_t n_online) {
    int bits = 0; uint32_t v = (uint32_t)(n_online > 1 ? n_online - 1 : 1);
    while (v) { ++bits; v >>= 1; }
    int h = (bits + 1) / 2;
    return h < 1 ? 1 : h;
}
static int32_t feistel_perm(int32_t q, int32_t n_online, const uint32_t kr[4]) {
    int h = feistel_h(n_online);
    uint32_t mask = (1u << h) - 1u, x = (uint32_t)q;
    do {
        uint32_t L = x >> h, R = x & mask;
        for (int i = 0; i < 4; ++i) { uint32_t nl = R; R = L ^ (((R ^ kr[i]) * 0x9E3779B1u) >> (32 - h)); L = nl; }
        x = (L << h) | R;
    } while (x >= (uint32_t)n_online);
    return (int32_t)x;
}

/* bounds[0..r], run q -> online index peer_idx[q]; returns r */
EXPORT int or_random_candidate(int n, int32_t n_online, uint64_t seed, int64_t k,
                               int32_t* bounds, int32_t* peer_idx) {
    uint64_t key = fmix64(seed + 0x9E3779B97F4A7C15ULL);
    xo128 g; xo_seed(&g, key, k);
    uint32_t rmax = (uint32_t)(n < n_online ? n : n_online);
    int r = 1 + (int)mulhi32(xo_next(&g), rmax), need = r - 1, nb = 0;
    bounds[nb++] = 0;
    for (int pos = 1; pos < n && need > 0; ++pos)
        if (mulhi32(xo_next(&g), (uint32_t)(n - pos)) < (uint32_t)need) { bounds[nb++] = pos; --need; }
    bounds[nb] = n;
    uint32_t kr[4];
    for (int i = 0; i < 4; ++i) kr[i] = xo_next(&g);
    for (int q = 0; q < r; ++q) peer_idx[q] = feistel_perm(q, n_online, kr);
    return r;
}

EXPORT void or_enum_random(const dm_tables* t, int32_t n_online, const int32_t* online, uint64_t seed,
                           int64_t k0, int64_t k1, dm_winner* out) {
    int n = t->n;
    int32_t* bounds = (int32_t*)malloc(sizeof(int32_t) * (size_t)(n + 2));
    int32_t* pidx = (int32_t*)malloc(sizeof(int32_t) * (size_t)(n + 1));
    int32_t* peers = (int32_t*)malloc(sizeof(int32_t) * (size_t)(n + 1));
    int32_t* peer_of = (int32_t*)malloc(sizeof(int32_t) * (size_t)n);
    int32_t* idxbuf = (int32_t*)malloc(sizeof(int32_t) * (size_t)n);
    uint8_t* inside = (uint8_t*)calloc((size_t)n, 1);
    or_win w = {INFINITY, -1, 0, 0, 0};
    for (int64_t k = k0; k < k1; ++k) {
        int r = or_random_candidate(n, n_online, seed, k, bounds, pidx);
        for (int q = 0; q < r; ++q) peers[q] = online[pidx[q]];
        double mk;
        w.n_eval++;
        if (score_contiguous(t, r, bounds, peers, peer_of, idxbuf, inside, &mk)) win_update(&w, mk, k);
    }
    out->makespan = w.mk; out->rank = w.rank; out->n_evaluated = w.n_eval;
    out->n_feasible = w.n_feas; out->checksum = w.csum;
    free(bounds); free(pidx); free(peers); free(peer_of); free(idxbuf); free(inside);
}

/* ------------------------------------------------------------ _subset_dp */

/* scheduling._subset_dp (scheduling.py:288-325), push form exactly as the
 * reference: layers i ascending, states of a layer by mask ascending, workers
 * ascending, j ascending with the _fits break; strict < updates; final state =
 * smallest (makespan, mask).  Costs price reads with the default link and
 * only count edges with src < i (:299-301).  Writes owner[i] = worker index and
 * returns 1, or 0 when no final state exists. */
EXPORT int or_subset_dp(const dm_tables* t, int32_t* owner, double* out_mk) {
    int n = t->n, p = t->p;
    int64_t S = (int64_t)1 << p;
    int64_t nst = (int64_t)(n + 1) * S;
    double* mk = (double*)malloc(sizeof(double) * (size_t)nst);
    uint8_t* has = (uint8_t*)calloc((size_t)nst, 1);
    int16_t* bi = (int16_t*)malloc(sizeof(int16_t) * (size_t)nst);
    int16_t* bw = (int16_t*)malloc(sizeof(int16_t) * (size_t)nst);
    has[0] = 1; mk[0] = 0.0;                                        /* :304 */
    int inc = (t->flags & DM_F_INCLUDE_COMM) != 0;
    for (int i = 0; i < n; ++i) {                                    /* :305 */
        for (int64_t mask = 0; mask < S; ++mask) {                   /* :306 sorted layer */
            int64_t key = (int64_t)i * S + mask;
            if (!has[key]) continue;
            double m0 = mk[key];
            for (int wi = 0; wi < p; ++wi) {                         /* :310 */
                if (mask & ((int64_t)1 << wi)) continue;
                for (int j = i + 1; j <= n; ++j) {                   /* :313 */
                    if (!fits_range(t, wi, i, j)) break;             /* :314-315 */
                    /* chunk_cost :294-302 */
                    double fl = col_sum_range(t->flops, t->pre_flops, flops_exact(t), i, j, np_flops(t));
                    double compute = fl / t->speed[wi];
                    double rd = 0.0;
                    if (inc) {
                        for (int s = i; s < j; ++s)
                            for (int e = t->edge_ptr[s]; e < t->edge_ptr[s + 1]; ++e)
                                if (t->edge_src[e] < i) rd += comm_time(t->def_alpha, t->def_beta, t->edge_m[e]);
                    }
                    double cc = compute + rd;
                    double nm = cc > m0 ? cc : m0;                   /* :316 max(mk, cc) */
                    int64_t nk = (int64_t)j * S + (mask | ((int64_t)1 << wi));
                    if (!has[nk] || nm < mk[nk]) {                   /* :318-320 */
                        has[nk] = 1; mk[nk] = nm; bi[nk] = (int16_t)i; bw[nk] = (int16_t)wi;
                    }
                }
            }
        }
    }
    int64_t bestmask = -1; double bestv = INFINITY;                  /* :321-325 */
    for (int64_t mask = 0; mask < S; ++mask) {
        int64_t key = (int64_t)n * S + mask;
        if (!has[key]) continue;
        if (bestmask < 0 || mk[key] < bestv) { bestv = mk[key]; bestmask = mask; }
    }
    int found = bestmask >= 0;
    if (found) {
        int j = n; int64_t mask = bestmask;
        while (j > 0) {
            int64_t key = (int64_t)j * S + mask;
            int i = bi[key], wi = bw[key];
            for (int s = i; s < j; ++s) owner[s] = wi;
            mask &= ~((int64_t)1 << wi); j = i;
        }
    }
    *out_mk = bestv;
    free(mk); free(has); free(bi); free(bw);
    return found;
}

/* ----------------------------------------------------- proportional split */

/* scheduling._proportional_runs (scheduling.py:328-351).  Writes bounds of
 * the runs (run q on worker q) and returns the number of runs. */
EXPORT int or_proportional(const dm_tables* t, int32_t* bounds) {
    int n = t->n, p = t->p;
    double total_speed = or_py_sum_items(t->speed, t->peer_np, p);                     /* :332 */
    double total_flops = col_sum_range(t->flops, t->pre_flops, flops_exact(t), 0, n, np_flops(t)); /* :333 */
    if (total_flops == 0.0) total_flops = 1.0;
    double* prefix = (double*)malloc(sizeof(double) * (size_t)n);   /* :334 accumulate */
    prefix[0] = t->flops[0];
    for (int i = 1; i < n; ++i) prefix[i] = prefix[i - 1] + t->flops[i];
    int start = 0, nr = 0; double acc = 0.0;
    bounds[0] = 0;
    for (int wi = 0; wi < p; ++wi) {                                 /* :337 */
        if (start >= n) break;
        int end;
        if (wi == p - 1) end = n;
        else {
            double num = total_flops * t->speed[wi];
            acc += num / total_speed;                                /* :343 */
            end = start + 1;
            while (end < n && prefix[end - 1] < acc) ++end;          /* :345-346 */
            int remaining = p - wi - 1;
            int lim = n - remaining;
            end = end < lim ? end : lim;
            end = end > start + 1 ? end : start + 1;                 /* :348 */
        }
        bounds[++nr] = end;
        start = end;
    }
    free(prefix);
    return nr;
}

/* ------------------------------------------------------------ _hill_climb */

/* score() inside _hill_climb (scheduling.py:357-362) for contiguous runs
 * given by bounds[0..r], peers[0..r): inf if verify fails, else max load with
 * pairwise links. */
static double hill_score(const dm_tables* t, int r, const int32_t* bounds, const int32_t* peers,
                         int32_t* peer_of, int32_t* idxbuf, uint8_t* inside) {
    /* verify_assignment: runs are contiguous, distinct, cover all stages;
       only the capacity checks can fail, in run order :199-203 */
    int ex = bytes_exact(t);
    for (int q = 0; q < r; ++q) {
        int a = bounds[q], b = bounds[q + 1], pe = peers[q];
        if (b == a) continue;
        if (col_sum_range(t->gpu, t->pre_gpu, ex, a, b, np_bytes(t)) > t->cap_gpu[pe]) return INFINITY;
        if (col_sum_range(t->cpu, t->pre_cpu, ex, a, b, np_bytes(t)) > t->cap_cpu[pe]) return INFINITY;
        if (col_sum_range(t->disk, t->pre_disk, ex, a, b, np_bytes(t)) > t->cap_disk[pe]) return INFINITY;
    }
    for (int q = 0; q < r; ++q)
        for (int i = bounds[q]; i < bounds[q + 1]; ++i) peer_of[i] = peers[q];
    double best = 0.0; int have = 0;
    for (int q = 0; q < r; ++q) {
        int k = bounds[q + 1] - bounds[q];
        if (!k) continue;
        for (int z = 0; z < k; ++z) idxbuf[z] = bounds[q] + z;
        double c, rd;
        run_cost(t, peer_of, peers[q], idxbuf, k, inside, &c, &rd);
        double load = c + rd;
        if (!have || load > best) { best = load; have = 1; }
    }
    return best;
}

/* scheduling._hill_climb (scheduling.py:354-388) on contiguous runs in
 * stage order: bounds[0..r], peers[0..r) updated in place.  Returns the
 * number of accepted moves; *score_out = final score. */
EXPORT int or_hill_climb(const dm_tables* t, int r, int32_t* bounds, const int32_t* peers,
                         int rounds, double* score_out) {
    int n = t->n;
    int32_t* peer_of = (int32_t*)malloc(sizeof(int32_t) * (size_t)n);
    int32_t* idxbuf = (int32_t*)malloc(sizeof(int32_t) * (size_t)n);
    uint8_t* inside = (uint8_t*)calloc((size_t)n, 1);
    int moves = 0;
    double cur = hill_score(t, r, bounds, peers, peer_of, idxbuf, inside);  /* :365 */
    for (int round = 0; round < rounds; ++round) {                   /* :366 */
        int improved = 0;
        for (int a = 0; a + 1 < r; ++a) {                            /* :368-369 all runs non-empty */
            int b = a + 1;
            for (int dir = 0; dir < 2; ++dir) {                      /* :370 (+1, -1) */
                int la = bounds[a + 1] - bounds[a], lb = bounds[b + 1] - bounds[b];
                int nb;
                if (dir == 0 && la > 1) nb = bounds[a + 1] - 1;      /* :373-374 */
                else if (dir == 1 && lb > 1) nb = bounds[a + 1] + 1; /* :375-376 */
                else continue;
                int old = bounds[a + 1];
                bounds[a + 1] = nb;
                double cs = hill_score(t, r, bounds, peers, peer_of, idxbuf, inside);
                if (cs < cur - 1e-15) { cur = cs; improved = 1; ++moves; }   /* :383-385 */
                else bounds[a + 1] = old;
            }
        }
        if (!improved) break;                                        /* :386-387 */
    }
    *score_out = cur;
    free(peer_of); free(idxbuf); free(inside);
    return moves;
}

/* ------------------------------------------------------------- schedule() */

/* scheduling.schedule (scheduling.py:391-423) without the pinned branch
 * (pinned runs are scored with or_eval_runs).  Writes owner[i] (worker index),
 * returns path: 1 = exact subset search, 2 = proportional + hill climb,
 * negative = infeasible (-1 DP found nothing, -2 hill result infeasible).
 * has_links: fleet.links non-empty (:412). */
EXPORT int or_schedule(const dm_tables* t, int has_links, int32_t* owner) {
    int n = t->n, p = t->p;
    int32_t bounds[1100], peers[1100];
    double sc;
    double gate = (double)n * (double)n * (double)p * ldexp(1.0, p);
    if (gate <= 3000000.0) {                                          /* :406 */
        double mk;
        if (!or_subset_dp(t, owner, &mk)) return -1;                  /* :408-411 */
        if (has_links) {                                              /* :412-413 */
            int r = 0; bounds[0] = 0; peers[0] = owner[0];
            for (int i = 1; i < n; ++i) if (owner[i] != owner[i - 1]) { bounds[++r] = i; peers[r] = owner[i]; }
            bounds[++r] = n;
            or_hill_climb(t, r, bounds, peers, 200, &sc);
            for (int q = 0; q < r; ++q) for (int i = bounds[q]; i < bounds[q + 1]; ++i) owner[i] = peers[q];
        }
        return 1;
    }
    int r = or_proportional(t, bounds);                               /* :416 */
    for (int q = 0; q < r; ++q) peers[q] = q;
    or_hill_climb(t, r, bounds, peers, 200, &sc);                     /* :417 */
    for (int q = 0; q < r; ++q) for (int i = bounds[q]; i < bounds[q + 1]; ++i) owner[i] = peers[q];
    return isinf(sc) ? -2 : 2;
}

/* ------------------------------------------- meet-in-the-middle sweep (CPU) */

/* The identity-split population (brute_force_schedule's order with run q on
 * worker q, scheduling.py:260-272) swept with the GPU headline's algorithm
 * (csrc/dm_mitm.cu) on the CPU: the algorithm-matched CPU baseline of the
 * bench, and an independent check of the sweep.  Valid when the load of run
 * q over [a, b) depends on (q, a, b) only (no comm, a uniform link, or chain
 * stages) — the same condition as the GPU path.
 *
 * T[(q*(n+1) + a)*(n+1) + b] = load of run [a, b) on worker q, +inf when the
 * run fails _fits.  A split with m cuts is grouped by its middle cut
 * j = ceil(m/2) at position c: left sets (j-1 cuts below c) x right sets
 * (m-j cuts above c); makespan = max(L, R) (exact), lexicographic rank =
 * RL + RR (a sum of per-cut terms).  Per feasible pair: one max, one
 * checksum add, one compare — the GPU's per-pair work. */
EXPORT void or_mitm_table(const dm_tables* t, double* T) {
    int n = t->n, p = t->p;
    int32_t* peer_of = (int32_t*)malloc(sizeof(int32_t) * (size_t)n);
    int32_t* idx = (int32_t*)malloc(sizeof(int32_t) * (size_t)n);
    uint8_t* inside = (uint8_t*)calloc((size_t)n, 1);
    for (int q = 0; q < p; ++q)
        for (int a = 0; a <= n; ++a)
            for (int b = 0; b <= n; ++b) {
                double v = INFINITY;
                if (b > a && fits_range(t, q, a, b)) {
                    for (int i = 0; i < n; ++i) peer_of[i] = i < a ? (q > 0 ? q - 1 : q + 1) : (i < b ? q : q + 1);
                    for (int z = 0; z < b - a; ++z) idx[z] = a + z;
                    double c, rd;
                    run_cost(t, peer_of, q, idx, b - a, inside, &c, &rd);
                    v = c + rd;
                }
                T[((size_t)q * (n + 1) + a) * (n + 1) + b] = v;
            }
    free(peer_of); free(idx); free(inside);
}

typedef struct { double v; int64_t rank; } mitm_side;

/* Lexicographic rank term of cut i (1-based) at position ci after c_{i-1} =
 * prev, for m cuts over positions 1..N: sum over v in (prev, ci) of
 * C(N - v, m - i). */
static int64_t cut_term(int N, int m, int i, int prev, int ci) {
    int64_t s = 0;
    for (int v = prev + 1; v < ci; ++v) s += binom(N - v, m - i);
    return s;
}

/* Left sets of block (m, c): cuts 1..j-1 below c; runs 0..j-1. */
static void mitm_left(const double* T, int n, int m, int j, int c, int q, int prev, double acc, int64_t rk,
                      mitm_side* out, int64_t* cnt) {
    int N = n - 1;
    if (q == j - 1) {                          /* last left run ends at c */
        double v = T[((size_t)q * (n + 1) + prev) * (n + 1) + c];
        if (v == INFINITY) return;
        out[*cnt].v = v > acc ? v : acc;
        out[*cnt].rank = rk + cut_term(N, m, j, prev, c);
        ++*cnt;
        return;
    }
    for (int x = prev + 1; x <= c - (j - 1 - q); ++x) {
        double v = T[((size_t)q * (n + 1) + prev) * (n + 1) + x];
        if (v == INFINITY) continue;
        mitm_left(T, n, m, j, c, q + 1, x, v > acc ? v : acc, rk + cut_term(N, m, q + 1, prev, x), out, cnt);
    }
}

/* Right sets of block (m, c): cuts j+1..m above c; runs j..m. */
static void mitm_right(const double* T, int n, int m, int q, int prev, double acc, int64_t rk,
                       mitm_side* out, int64_t* cnt) {
    int N = n - 1;
    if (q == m) {                              /* last run ends at n */
        double v = T[((size_t)q * (n + 1) + prev) * (n + 1) + n];
        if (v == INFINITY) return;
        out[*cnt].v = v > acc ? v : acc;
        out[*cnt].rank = rk;
        ++*cnt;
        return;
    }
    for (int x = prev + 1; x <= n - 1 - (m - 1 - q); ++x) {
        double v = T[((size_t)q * (n + 1) + prev) * (n + 1) + x];
        if (v == INFINITY) continue;
        mitm_right(T, n, m, q + 1, x, v > acc ? v : acc, rk + cut_term(N, m, q + 1, prev, x), out, cnt);
    }
}

/* Sweep the blocks (m, c) with m in [m_lo, m_hi) (c over every middle
 * position) and merge into *out (first strict minimum by rank).  `T` from
 * or_mitm_table.  Returns the number of feasible pairs visited. */
EXPORT int64_t or_splits_mitm(const dm_tables* t, const double* T, int m_lo, int m_hi, dm_winner* out) {
    int n = t->n, p = t->p, rmax = n < p ? n : p, N = n - 1;
    or_win w = {INFINITY, -1, 0, 0, 0};
    int64_t base = 0;
    for (int m = 0; m < m_lo && m < rmax; ++m) base += binom(N, m);
    for (int m = m_lo; m < m_hi && m < rmax; ++m) {
        int64_t nc = binom(N, m);
        w.n_eval += nc;
        if (m == 0) {
            double v = T[(size_t)0 * (n + 1) * (n + 1) + n];
            if (v != INFINITY) win_update(&w, v, base);
            base += nc;
            continue;
        }
        int j = (m + 1) / 2;
        for (int c = j; c <= N - (m - j); ++c) {
            int64_t nl = binom(c - 1, j - 1), nr = binom(N - c, m - j), cl = 0, cr = 0;
            mitm_side* L = (mitm_side*)malloc(sizeof(mitm_side) * (size_t)(nl > 0 ? nl : 1));
            mitm_side* R = (mitm_side*)malloc(sizeof(mitm_side) * (size_t)(nr > 0 ? nr : 1));
            mitm_left(T, n, m, j, c, 0, 0, 0.0, 0, L, &cl);
            mitm_right(T, n, m, j, c, 0.0, 0, R, &cr);
            for (int64_t a = 0; a < cl; ++a) {
                double lv = L[a].v;
                int64_t lr = base + L[a].rank;
                for (int64_t b = 0; b < cr; ++b) {
                    double mk = R[b].v > lv ? R[b].v : lv;
                    uint64_t bits; memcpy(&bits, &mk, 8);
                    w.csum += bits;
                    if (mk <= w.mk) {
                        int64_t rk = lr + R[b].rank;
                        if (w.rank < 0 || mk < w.mk || rk < w.rank) { w.mk = mk; w.rank = rk; }
                    }
                }
            }
            w.n_feas += cl * cr;
            free(L); free(R);
        }
        base += nc;
    }
    out->makespan = w.mk; out->rank = w.rank; out->n_evaluated = w.n_eval;
    out->n_feasible = w.n_feas; out->checksum = w.csum;
    return w.n_feas;
}

/* -------------------------------------------------------------- epilogue */

/* pipeline.fp_latency / bottleneck / pipeline_time / throughput
 * (pipeline.py:41-62) over profiles given in first-stage order.  np_load[q]
 * != 0 when profile q's compute_s + read_s is a numpy float (NULL: none). */
EXPORT void or_epilogue(int r, const double* compute, const double* read, const uint8_t* np_load,
                        int64_t n_batches, int64_t samples_per_batch, double* out4) {
    double* tot = (double*)malloc(sizeof(double) * (size_t)(r + 1));
    double bn = 0.0;
    for (int q = 0; q < r; ++q) {
        tot[q] = compute[q] + read[q];
        double m = compute[q] >= read[q] ? compute[q] : read[q];
        if (q == 0 || m > bn) bn = m;
    }
    double lat = or_py_sum_items(tot, np_load, r);
    double fill = (double)(n_batches - 1) * bn;
    double pipe = lat + fill;
    double thr = (double)(n_batches * samples_per_batch) / pipe;
    out4[0] = lat; out4[1] = bn; out4[2] = pipe; out4[3] = thr;
    free(tot);
}

/* ----------------------------------------------------------- op costs */

/* hardware.op_time (hardware.py:190-206) for every op of one placement:
 * read = naive sum over args on other peers of comm_time(link_between, M),
 * compute = op_flops / effective_speed, write = M / write_bandwidth when any
 * user sits on another peer. */
EXPORT void or_op_costs(const dm_tables* t, int n_ops, const double* flops, const double* mbytes,
                        const int32_t* aptr, const int32_t* aidx, const int32_t* uptr, const int32_t* uidx,
                        const double* write_bw, const int32_t* place, double* out,
                        int np_links, const uint8_t* write_np, uint8_t* out_np) {
    for (int i = 0; i < n_ops; ++i) {
        int me = place[i];
        double* o = out + 3 * i;
        if (me < 0 || me >= t->P) { o[0] = o[1] = o[2] = NAN; if (out_np) out_np[i] = 0; continue; }
        int is_np = t->peer_np && t->peer_np[me];              /* compute_s type */
        double rd = 0.0;
        for (int e = aptr[i]; e < aptr[i + 1]; ++e) {
            int src = place[aidx[e]];
            if (src != me) {
                double al, be;
                link_of(t, src, me, &al, &be);
                rd += comm_time(al, be, mbytes[aidx[e]]);
                is_np |= np_links;
            }
        }
        double wr = 0.0;
        for (int e = uptr[i]; e < uptr[i + 1]; ++e)
            if (place[uidx[e]] != me) { wr = mbytes[i] / write_bw[me]; is_np |= write_np && write_np[me]; break; }
        o[0] = rd; o[1] = flops[i] / t->speed[me]; o[2] = wr;
        if (out_np) out_np[i] = (uint8_t)is_np;
    }
}

/* hardware.subgraph_time (hardware.py:219-226): max and CPython sum of the
 * per-op totals read + compute + write. */
EXPORT void or_subgraph(int k, const int32_t* idx, const double* op_out, const uint8_t* op_np, double* out3) {
    if (k == 0) { out3[0] = out3[1] = out3[2] = 0.0; return; }
    double* tot = (double*)malloc(sizeof(double) * (size_t)k);
    uint8_t* npv = (uint8_t*)malloc((size_t)k);
    double mx = 0.0;
    for (int q = 0; q < k; ++q) {
        const double* o = op_out + 3 * idx[q];
        tot[q] = o[0] + o[1] + o[2];
        npv[q] = op_np ? op_np[idx[q]] : 0;
        if (q == 0 || tot[q] > mx) mx = tot[q];
    }
    double seq = or_py_sum_items(tot, npv, k);
    free(npv);
    out3[0] = mx; out3[1] = seq; out3[2] = seq;
    free(tot);
}

EXPORT int or_abi_version(void) { return DM_ABI_VERSION; }
