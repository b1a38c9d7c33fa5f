// dm_memo.cuh — the memoised run-cost table of the identity-order split
// population, shared by the split-sweep kernels (dm_enum.cu, dm_mitm.cu).
//
// For run q on worker q the load of a run over stages [a, b) depends only on
// (q, a, b) whenever the crossing read does not depend on which run owns a
// source stage: include_comm off, a uniform link (no pair overrides: every
// crossing source sits on another worker), or chain-structured stages (the
// source of run q's crossing edges is stage a-1, owned by worker q-1).  Each
// CTA tabulates
//     T[q][a][b] = _fits(q, a..b) ? compute + read : +inf
// (scheduling.py:156-176, exactly the reference's arithmetic) once in shared
// memory: n(n+1)(n+2)/6 doubles at most, 57 KB for n = 34.
#pragma once

#include "dm_common.cuh"

namespace dm {

__device__ inline int64_t binom_sat(int a, int b);

// Shared-memory layout.  rowoff[q * S + a] is the ABSOLUTE shared address of
// T[q][a][0] (so &T[q][a][b] = rowoff + 8b); rows that no valid run uses
// (q >= rmax, a < q, a = n) point at a row of -inf.  binom[a * R1 + b] =
// C(a, b) for a < n, b <= rmax; cum[m] = number of splits with fewer than m
// cuts (the first global rank with m cuts).  off_cuts/off_tail: kernel-owned
// space after the tables.
struct MemoLayout {
    int n, rmax, W, S;
    int t_elems;
    size_t off_dummy, off_rowoff, off_binom, off_cum, off_tail;
};

__host__ __device__ inline MemoLayout memo_layout(int n, int p) {
    MemoLayout L;
    L.n = n; L.rmax = n < p ? n : p; L.W = n - 1; L.S = n < 64 ? 64 : 256;
    int tot = 0;
    for (int q = 0; q < L.rmax; ++q) { int Lq = n - q; tot += Lq * (Lq + 1) / 2; }
    L.t_elems = tot;
    size_t off = (size_t)tot * 8;
    L.off_dummy = off; off += (size_t)(n + 1) * 8;
    off = (off + 15) & ~(size_t)15;
    L.off_rowoff = off; off += (size_t)(L.rmax + 4) * L.S * 4;
    L.off_binom = off; off += (size_t)n * (L.rmax + 1) * 8;
    L.off_cum = off; off += (size_t)(L.rmax + 2) * 8;
    off = (off + 15) & ~(size_t)15;
    L.off_tail = off;
    return L;
}

// Whether the memoised table is exact for this instance (see header).
__host__ __device__ inline bool memo_valid(const dm_tables& t) {
    const uint32_t f = t.flags;
    return !(f & DM_F_INCLUDE_COMM) || !(f & DM_F_PAIR_LINKS) || (f & DM_F_CHAIN);
}

__device__ __forceinline__ double lds_f64(uint32_t addr) {
    double v;
    asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(addr));
    return v;
}

// Fill rowoff, the -inf row, binom, cum and T (all threads of the CTA; ends
// with __syncthreads).
__device__ inline void memo_build(const dm_tables& t, const MemoLayout& L, unsigned char* sm) {
    const int n = t.n, rmax = L.rmax, S = L.S, R1 = rmax + 1;
    int32_t* rowoff = reinterpret_cast<int32_t*>(sm + L.off_rowoff);
    int64_t* binom = reinterpret_cast<int64_t*>(sm + L.off_binom);
    int64_t* cum = reinterpret_cast<int64_t*>(sm + L.off_cum);
    const double inf = __longlong_as_double(0x7ff0000000000000LL);
    const uint32_t sm_base = (uint32_t)__cvta_generic_to_shared(sm);
    for (int i = threadIdx.x; i < (rmax + 4) * S; i += blockDim.x) {
        int q = i / S, a = i % S;
        int32_t v = (int32_t)L.off_dummy;
        if (q < rmax && a >= q && a < n) {
            int base = 0;
            for (int qq = 0; qq < q; ++qq) { int Lq = n - qq; base += Lq * (Lq + 1) / 2; }
            int within = (a - q) * n - ((a - q) * (a + q - 1)) / 2;
            v = (base + within - (a + 1)) * 8;
        }
        rowoff[i] = (int32_t)(sm_base + (uint32_t)v);
    }
    for (int i = threadIdx.x; i <= n; i += blockDim.x) reinterpret_cast<double*>(sm + L.off_dummy)[i] = -inf;
    for (int i = threadIdx.x; i < n * R1; i += blockDim.x) binom[i] = binom_sat(i / R1, i % R1);
    __syncthreads();
    if (threadIdx.x == 0) {
        cum[0] = 0;
        for (int m = 1; m <= rmax; ++m) cum[m] = cum[m - 1] + binom[(n - 1) * R1 + (m - 1)];
    }
    for (int row = threadIdx.x; row < rmax * n; row += blockDim.x) {
        int q = row / n, a = row % n;
        if (a < q) continue;
        double* Trow = reinterpret_cast<double*>(sm + ((uint32_t)rowoff[q * S + a] - sm_base));
        for (int b = a + 1; b <= n; ++b) {
            double v = inf;
            if ((q > 0 || a == 0) && fits_range(t, q, a, b)) {
                double c, rd;
                if (chain(t)) run_cost_contig(t, a, b, q, [&](int) { return q - 1; }, c, rd);
                else run_cost_contig(t, a, b, q, [&](int s) { return s < a ? -1 : q + 1; }, c, rd);
                v = c + rd;
            }
            Trow[b] = v;
        }
    }
    __syncthreads();
}

// Saturating binomial C(a, b) (int64 max on overflow).
__device__ inline int64_t binom_sat(int a, int b) {
    if (b < 0 || b > a) return 0;
    if (b > a - b) b = a - b;
    unsigned __int128 r = 1;
    for (int i = 1; i <= b; ++i) {
        r = r * (unsigned __int128)(a - b + i) / (unsigned __int128)i;
        if (r > (unsigned __int128)INT64_MAX) return INT64_MAX;
    }
    return (int64_t)r;
}

}  // namespace dm
