/*
 * dagmesh_b200.h — C ABI of the B200 placement-cost / partition-search engine.
 *
 * This is the drop-in boundary for the hot path of the reference planner
 * `dagmesh` (FusionAI, arXiv 2309.01172).  The reference has no FFI of its
 * own: its boundary is the Python API of `dagmesh.scheduling` and
 * `dagmesh.pipeline`.  Every entry point below replaces one reference
 * function (cited as pkg/src/dagmesh/<file>:<line>, relative to the
 * reference tree) and is bound from Python with ctypes by
 * `paper_2309_01172_b200/_lib.py` (see INTEGRATION.md for the binding a
 * maintainer adds to the reference package itself).
 *
 * Conventions
 *   - plain pointers and sizes only; no torch types.  Pointers inside the
 *     structs passed to dm_* calls are DEVICE pointers (caller-owned).
 *   - every call is stream-ordered (`stream` is a cudaStream_t, NULL = legacy
 *     default stream), reentrant, and keeps no global mutable state except a
 *     thread-local last-error string (dm_last_error()).
 *   - functions return DM_OK (0) or a negative DM_E_* status; they never
 *     throw across the ABI.
 *   - all arithmetic is IEEE-754 binary64 with the reference's rounding
 *     sequence (no FMA contraction: the library is built with -fmad=false,
 *     division is correctly rounded), so results are bit-identical to the
 *     CPython reference.
 *
 * The same struct layout is consumed by the CPU oracle under oracle/ (host
 * pointers there); the oracle is test infrastructure only.
 */
#ifndef DAGMESH_B200_H
#define DAGMESH_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define DM_ABI_VERSION 1

#if defined(__GNUC__)
#define DM_API __attribute__((visibility("default")))
#else
#define DM_API
#endif

/* ---------------------------------------------------------------- status */
#define DM_OK              0
#define DM_E_ARG          -1   /* bad argument (sizes, null pointers)            */
#define DM_E_CUDA         -2   /* CUDA runtime error; see dm_last_error()        */
#define DM_E_UNKNOWN_PEER -3   /* FleetError("unknown peer")  hardware.py:122-126 */
#define DM_E_UNASSIGNED   -4   /* KeyError: crossing edge from an unowned stage
                                  (peer_of[src] in scheduling.py:167)            */
#define DM_E_TOO_LARGE    -5   /* instance exceeds a device-side size limit      */

/* ------------------------------------------------------ violation codes
 * First violation found by verify_assignment (scheduling.py:179-207), in the
 * reference's check order.  The Python layer rebuilds the reason string. */
#define DM_V_OK             0
#define DM_V_TWO_RUNS       1  /* "peer X holds two runs"          :186-187 */
#define DM_V_UNKNOWN_PEER   2  /* "unknown peer X"                 :189-190 */
#define DM_V_NOT_CONTIGUOUS 3  /* "peer X run [...] is not contiguous" :191-193 */
#define DM_V_ASSIGNED_TWICE 4  /* "stage i assigned twice"         :194-196 */
#define DM_V_GPU            5  /* "peer X exceeds gpu capacity"    :199-203 */
#define DM_V_CPU            6  /*                  cpu                      */
#define DM_V_DISK           7  /*                  disk                     */
#define DM_V_UNASSIGNED     8  /* "stages [...] unassigned"        :204-206 */

/* ------------------------------------------------------------ table flags */
#define DM_F_FLOPS_EXACT  1u   /* flops integral, every prefix < 2^53: pre_flops valid */
#define DM_F_BYTES_EXACT  2u   /* gpu/cpu/disk integral, prefixes < 2^53: pre_* valid  */
#define DM_F_PAIR_LINKS   4u   /* link_alpha/link_beta (P x P) hold link_between()    */
#define DM_F_CHAIN        8u   /* every in-edge of stage i has src == i-1             */
#define DM_F_BACKWARD    16u   /* some in-edge has src >= its own stage               */
#define DM_F_INCLUDE_COMM 32u  /* include_comm=True (scheduling.py:162)               */
/* CPython's sum() runs its compensated fast path only over exact `float`
 * items; numpy.float64 inputs make it a naive left-to-right sum from the first
 * such item on (with the compensation gathered so far applied at the switch).
 * These flags record which inputs are not exact Python floats. */
#define DM_F_NP_FLOPS    64u   /* stage flops column            */
#define DM_F_NP_COMM    128u   /* msg_ratio or link alpha/beta  */
#define DM_F_NP_BYTES   256u   /* gpu/cpu/disk byte columns      */

/*
 * One scheduling instance: the stage table (scheduling.Stage, :32-42) and the
 * fleet (hardware.Fleet, hardware.py:103-144) in structure-of-arrays form.
 *
 * Peer indexing: 0..p-1 are fleet.worker_ids() in order (hardware.py:131-134,
 * ir.peer_sort_key ordering); p..P-1 are the remaining peers (backups) in
 * peer_ids() order.  Worker order defines brute-force permutation order,
 * subset-DP masks and pinned-run mapping.
 */
typedef struct dm_tables {
    int32_t n;          /* stages                                     */
    int32_t p;          /* schedulable workers                        */
    int32_t P;          /* all addressable peers (workers + backups)  */
    int32_t n_edges;    /* CSR length                                  */
    uint32_t flags;     /* DM_F_*                                      */
    int32_t pad_;
    double def_alpha;   /* fleet.default_link.alpha  (s)               */
    double def_beta;    /* fleet.default_link.beta   (s/B)             */
    /* stage columns, length n */
    const double* flops;
    const double* gpu;
    const double* cpu;
    const double* disk;
    /* exact prefix sums, length n+1 (valid per DM_F_*_EXACT) */
    const int64_t* pre_flops;
    const int64_t* pre_gpu;
    const int64_t* pre_cpu;
    const int64_t* pre_disk;
    /* in-edges in stored order: stage i owns edge_ptr[i] .. edge_ptr[i+1]-1 */
    const int32_t* edge_ptr;   /* [n+1] */
    const int32_t* edge_src;   /* [n_edges] source stage                     */
    const double* edge_m;      /* [n_edges] nbytes * fleet.msg_ratio (>= 0)   */
    /* peer columns, length P */
    const double* speed;       /* effective_speed = peak_flops * lam (hardware.py:153-154) */
    const double* cap_gpu;
    const double* cap_cpu;
    const double* cap_disk;
    /* resolved link_between(a, b) (hardware.py:136-140), row a = source owner,
       column b = reading peer, diagonal = ZERO_LINK; only with DM_F_PAIR_LINKS */
    const double* link_alpha;  /* [P*P] */
    const double* link_beta;   /* [P*P] */
    /* peer_np[w] = 1 when effective_speed(peer w) is not an exact Python float
       (numpy.float64 peak or lambda): CPython's sum() then leaves its
       compensated fast path at that item (bltinmodule.c) — see dm_common.cuh */
    const uint8_t* peer_np;    /* [P] */
} dm_tables;

/* Arg-min record shared by every enumeration: first strict minimum in rank
 * order (brute_force_schedule, scheduling.py:269-272). */
typedef struct dm_winner {
    double   makespan;     /* +inf if no candidate was feasible           */
    int64_t  rank;         /* global rank of the winner, -1 if none       */
    int64_t  n_evaluated;  /* candidates scored                           */
    int64_t  n_feasible;   /* candidates that passed _fits                */
    uint64_t checksum;     /* sum (mod 2^64) of makespan bit patterns of
                              all feasible candidates — order independent  */
} dm_winner;

/* --------------------------------------------------------------- general */
DM_API int         dm_abi_version(void);
DM_API const char* dm_last_error(void);
/* bytes of device scratch the enumeration calls need (per-CTA partials) */
DM_API int64_t     dm_enum_scratch_bytes(void);

/*
 * dm_eval_runs — replaces scheduling._evaluate / evaluate_runs
 * (scheduling.py:210-239) including verify_assignment (:179-207) and
 * _run_cost (:156-169), for arbitrary Runs in CSR form:
 *   candidate c owns runs cand_ptr[c] .. cand_ptr[c+1]-1 (runs order as given);
 *   run r is (run_peer[r], stage indices run_idx[run_ptr[r] .. run_ptr[r+1]-1]).
 * run_peer[r] < 0 or >= P encodes a peer unknown to the fleet.
 * Outputs: per run compute_s / read_s (only for non-empty runs; the order is the
 * given order, the Python layer sorts by first stage as :217-218 does),
 * per candidate makespan (max(0.0, loads)), violation code and the index of the
 * run that triggered it.  Status DM_E_UNKNOWN_PEER / DM_E_UNASSIGNED mirror the
 * FleetError / KeyError the reference raises while costing; out_status[c] holds
 * the per-candidate status.
 */
DM_API int dm_eval_runs(const dm_tables* t, int32_t n_cand,
                 const int32_t* cand_ptr, const int32_t* run_peer,
                 const int32_t* run_ptr, const int32_t* run_idx,
                 double* out_compute, double* out_read,
                 double* out_makespan, int32_t* out_code,
                 int32_t* out_code_run, int32_t* out_status, void* stream);

/* dm_eval_runs_ws — dm_eval_runs with the total run count known to the
 * caller and a caller workspace of dm_eval_runs_ws_bytes(n, n_cand,
 * n_runs_total) bytes: stream-ordered with no host synchronisation and no
 * allocation (the one-call API path). */
DM_API int64_t dm_eval_runs_ws_bytes(int32_t n, int32_t n_cand, int32_t n_runs_total);
DM_API int dm_eval_runs_ws(const dm_tables* t, int32_t n_cand, const int32_t* cand_ptr, const int32_t* run_peer,
                           const int32_t* run_ptr, const int32_t* run_idx, int32_t n_runs_total,
                           double* out_compute, double* out_read, double* out_makespan, int32_t* out_code,
                           int32_t* out_code_run, int32_t* out_status, void* workspace, void* stream);

/*
 * dm_eval_owner — Mode A scoring stream (the scoring-service form of
 * evaluate_runs).  Candidate c is the owner vector owner[c*n .. c*n+n-1]
 * (uint8 when owner_bytes == 1, uint16 when 2) whose Runs are the stages of
 * each peer grouped in first-appearance order.  Writes makespan (f64) and
 * violation code (u8, DM_V_*; 0xFF = owner index >= P, i.e. FleetError).
 */
DM_API int dm_eval_owner(const dm_tables* t, int64_t n_cand, const void* owner,
                  int32_t owner_bytes, double* out_makespan,
                  uint8_t* out_code, void* stream);

/* dm_eval_owner_argmin — dm_eval_owner with the arg-min fused into the
 * scoring kernel (ranks = rank_base + index; scratch as dm_enum_scratch_bytes). */
DM_API int dm_eval_owner_argmin(const dm_tables* t, int64_t n_cand, const void* owner,
                                int32_t owner_bytes, double* out_makespan, uint8_t* out_code,
                                int64_t rank_base, dm_winner* out, void* scratch, void* stream);

/*
 * dm_argmin_scores — block/warp arg-min over (makespan, rank) of a scored
 * stream (codes != 0 are skipped), ranks = rank_base + index.
 * out is a device dm_winner.
 */
DM_API int dm_argmin_scores(const double* makespan, const uint8_t* code, int64_t n,
                     int64_t rank_base, dm_winner* out, void* scratch,
                     void* stream);

/*
 * dm_enum_bruteforce — brute_force_schedule's exhaustive order
 * (scheduling.py:245-278): global rank k in [k0, k1) over
 * r = 1..min(n,p); cut sets = combinations(range(1,n), r-1) (lexicographic);
 * peer tuples = permutations(workers, r) (lexicographic by worker index).
 * Candidates failing _fits (:172-176) are skipped; winner = first strict min.
 */
DM_API int dm_enum_bruteforce(const dm_tables* t, int64_t k0, int64_t k1,
                       dm_winner* out, void* scratch, void* stream);

/*
 * dm_enum_splits — the identity-order subset of the brute-force order: run q
 * goes to worker q.  Rank order: r ascending, then cut sets lexicographic.
 * Total Σ_{r=1..min(n,p)} C(n-1, r-1).
 */
DM_API int dm_enum_splits(const dm_tables* t, int64_t k0, int64_t k1,
                   dm_winner* out, void* scratch, void* stream);

/*
 * dm_enum_splits_part — the share of dm_enum_splits owned by part `part` of
 * `nparts` (multi-GPU): rank tasks are interleaved across parts so every GPU
 * gets the same mix of run counts; the union over parts is [k0, k1) exactly.
 */
DM_API int dm_enum_splits_part(const dm_tables* t, int64_t k0, int64_t k1, int32_t part,
                               int32_t nparts, dm_winner* out, void* scratch, void* stream);

/* Whole-population split sweeps (k0 = 0, k1 = every split) run as a
 * meet-in-the-middle cross product over per-sweep side tables held in a
 * device workspace.  dm_splits_workspace_bytes: bytes that workspace needs
 * (-1: the instance takes the rank-range kernels).  dm_enum_splits_ws: as
 * dm_enum_splits_part with a caller-provided workspace (NULL or smaller than
 * required: allocated stream-ordered inside the call, as dm_enum_splits and
 * dm_enum_splits_part do).  Replaces the same brute_force_schedule loop
 * (scheduling.py:245-278) for the identity worker order. */
DM_API int64_t dm_splits_workspace_bytes(const dm_tables* t);
DM_API int dm_enum_splits_ws(const dm_tables* t, int64_t k0, int64_t k1, int32_t part, int32_t nparts,
                             dm_winner* out, void* scratch, void* workspace, int64_t workspace_bytes,
                             void* stream);

/* dm_enum_splits_phase — dm_enum_splits_ws in two stream-ordered halves so a
 * batch of sweeps can overlap one instance's table phase with another's
 * sweep: phase 1 builds the side tables into `workspace` (required, at least
 * dm_splits_workspace_bytes), phase 2 sweeps them and writes `out`; phase 3
 * does both.  Phase 1 then phase 2 on the same workspace equals phase 3.
 * Phase 2 itself splits into 4 (the tile plan, a one-CTA kernel a batch can
 * run on a stream of its own) then 8 (the sweep kernel and `out`).
 * Instances that take the rank-range kernels do all their work in phase 2. */
DM_API int dm_enum_splits_phase(const dm_tables* t, int64_t k0, int64_t k1, int32_t part, int32_t nparts,
                                dm_winner* out, void* scratch, void* workspace, int64_t workspace_bytes,
                                int32_t phase, void* stream);

/*
 * dm_enum_random — random contiguous placements scored on chip (configs C3,
 * C5; replaces scoring a sampled candidate list with evaluate_runs,
 * scheduling.py:235-239, and keeps brute_force_schedule's arg-min rule :271):
 * candidate k (k0 <= k < k1) of the stream keyed by `seed` draws
 * r ~ U{1..min(n, n_online)}, a uniform (r-1)-subset of the cut positions
 * 1..n-1 (selection sampling) and r distinct online peers (a keyed Feistel
 * permutation of online[0..n_online)); runs failing _fits make the candidate
 * infeasible, the winner is the first strict minimum by k.  Recipe:
 * paper_2309_01172_b200/rng.py (shared bit for bit with the oracle).
 * Requires chain-structured stages (DM_F_CHAIN) when include_comm is set and
 * n <= 257.  `scratch` >= dm_enum_scratch_bytes().
 */
DM_API int dm_enum_random(const dm_tables* t, const int32_t* online, int32_t n_online, uint64_t seed,
                          int64_t k0, int64_t k1, dm_winner* out, void* scratch, void* stream);

/* dm_materialize — write candidates [k0, k0+count) of the brute-force
 * (mode 0) or identity-split (mode 1) order as owner vectors (uint8/uint16
 * worker indices, count x n): the input stream of dm_eval_owner. */
DM_API int dm_materialize(int32_t n, int32_t p, int32_t mode, int64_t k0, int64_t count,
                          void* owner, int32_t owner_bytes, void* stream);

/* dm_finalize_winners — reduce per-CTA partials left in scratch by the
 * enumeration calls into out (called internally; exposed for multi-stream use) */
DM_API int dm_finalize_winners(void* scratch, int32_t n_parts, dm_winner* out,
                        void* stream);

/*
 * dm_subset_dp — batched _subset_dp (scheduling.py:288-325): one CTA per
 * scenario, tables[s] is a device array of dm_tables (device pointers).
 * Output per scenario: out_owner[s*n_max + i] = worker index of stage i
 * (-1 beyond n), out_makespan[s] = DP value of the chosen final state
 * (+inf and out_found[s] = 0 when no final state exists → schedule() marks
 * the instance infeasible, :408-411).
 * scratch: device bytes for DP tables that do not fit shared memory; query
 * dm_subset_dp_scratch_bytes(n_max, p_max, n_scen).
 */
DM_API int64_t dm_subset_dp_scratch_bytes(int32_t n_max, int32_t p_max, int32_t n_scen);
DM_API int dm_subset_dp(const dm_tables* tables, int32_t n_scen, int32_t n_max,
                 int32_t p_max, int16_t* out_owner, double* out_makespan,
                 int32_t* out_found, void* scratch, void* stream);

/*
 * dm_prop_hill — batched _proportional_runs (:328-351) followed by
 * _hill_climb (:354-388) when do_hill[s] != 0 (one warp per scenario).
 * When init_owner != NULL the hill climb starts from those runs instead of
 * the proportional split (schedule()'s DP + pairwise-links polish, :412-413).
 * Output: final owner vectors and the hill-climb score (inf when infeasible).
 */
DM_API int dm_prop_hill(const dm_tables* tables, int32_t n_scen, int32_t n_max,
                 const int16_t* init_owner, const uint8_t* do_hill,
                 int16_t* out_owner, double* out_score, int32_t* out_moves,
                 void* stream);

/*
 * dm_schedule_report — the _evaluate half of one schedule() call
 * (scheduling.py:210-232, :391-423) on the device: from the owner vector a
 * search kernel left in `owner` (int16[n], worker indices; `found` = the DP's
 * found flag or NULL) derive the runs, per run compute / read (_run_cost
 * :156-169), the first capacity violation in run order (verify_assignment
 * :199-203) and the makespan, into one record of dm_sched_out_bytes(n) bytes:
 * int32 {found, n_runs, code, bad_run}, float64 makespan at offset 16,
 * int32 bounds[n+1] at 32, then int32 peers[n], float64 compute[n] and
 * float64 read[n], each 8-byte aligned.  `tables` is a device dm_tables.
 * found == 0 scores ((workers[0], all stages),) as the reference does (:408).
 */
DM_API int64_t dm_sched_out_bytes(int32_t n);
DM_API int dm_schedule_report(const dm_tables* tables, int32_t n, const int16_t* owner, const int32_t* found,
                              void* out, void* stream);

/*
 * dm_prop_hill_epilogue — dm_prop_hill followed, in the same kernel, by the
 * dm_pipeline_epilogue values of each scenario's final runs (out[s*6 + ...]
 * as below): batched schedule() + Eq. 3/4 in one launch.
 */
DM_API int dm_prop_hill_epilogue(const dm_tables* tables, int32_t n_scen, int32_t n_max,
                                 const int16_t* init_owner, const uint8_t* do_hill,
                                 int16_t* out_owner, double* out_score, int32_t* out_moves,
                                 int64_t n_batches, int64_t samples_per_batch, double* out, void* stream);

/*
 * dm_pipeline_epilogue — per scenario, from an owner vector with contiguous
 * runs: _evaluate's makespan and feasibility (:210-232), then
 * fp_latency (Neumaier sum, pipeline.py:41-43), bottleneck (:46-50),
 * pipeline_time (:53-56) and throughput (:59-62).
 * out[s*6 + {0..5}] = makespan, latency, bottleneck, pipe_time, throughput,
 * violation code (as double).
 */
DM_API int dm_pipeline_epilogue(const dm_tables* tables, int32_t n_scen, int32_t n_max,
                         const int16_t* owner, int64_t n_batches,
                         int64_t samples_per_batch, double* out, void* stream);

/*
 * Operator-level PALEO cost (hardware.op_time, hardware.py:190-206) over a
 * DAG of operators, batched over placements.  dm_ops holds, per operator i:
 * op_flops(node) (as f64), message_bytes(node, msg_ratio) (int-valued f64),
 * its args and users (CSR).  place[b*n_ops + i] = peer index of op i in
 * placement b (dm_tables indexing; >= P for peers unknown to the fleet).
 * out[(b*n_ops + i)*3 + {0,1,2}] = read_s, compute_s, write_s; out_np (optional)
 * [b*n_ops + i] = 1 when OpCost.total_s is a numpy float in the reference
 * (numpy speed, or a crossing read / write priced with numpy link values or
 * write bandwidth — flags DM_OPS_NP_LINKS, write_np[peer]).
 */
#define DM_OPS_NP_LINKS 1

typedef struct dm_ops {
    int32_t n_ops;
    int32_t flags;             /* DM_OPS_* */
    const double* flops;
    const double* mbytes;
    const int32_t* arg_ptr;    /* [n_ops+1] */
    const int32_t* arg_idx;
    const int32_t* user_ptr;   /* [n_ops+1] */
    const int32_t* user_idx;
    const uint8_t* write_np;   /* [P] write_bandwidth is a numpy value (NULL: none) */
} dm_ops;

DM_API int dm_op_costs(const dm_ops* ops, const dm_tables* t, const double* write_bw,
                       int32_t n_place, const int32_t* place, double* out, uint8_t* out_np,
                       void* stream);

/* hardware.subgraph_time (hardware.py:219-226) for cells sub_idx[sub_ptr[s]..]
 * over op costs from dm_op_costs: out[(b*n_sub + s)*3] = lower, upper, sequential.
 * op_np: dm_op_costs' out_np (NULL: every total an exact float). */
DM_API int dm_subgraph_times(int32_t n_ops, int32_t n_place, const double* op_out, const uint8_t* op_np,
                             int32_t n_sub, const int32_t* sub_ptr, const int32_t* sub_idx,
                             double* out, void* stream);

/* dm_microbench_fp64 — FP64 DMUL+DADD issue-rate microbenchmark (the
 * roofline denominator of the generated-candidate kernels).  *ops receives
 * the number of fp64 operations the launch performs; time it with events. */
DM_API int dm_microbench_fp64(int64_t iters, double* sink, int64_t* ops, void* stream);

/* dm_microbench_alu — ALU-pipe (LOP3) issue-rate microbenchmark: lane-ops
 * executed by `iters` iterations of 8 independent chains per thread, full
 * grid.  The independent roofline denominator of the split sweep. */
DM_API int dm_microbench_alu(int64_t iters, uint32_t* sink, int64_t* ops, void* stream);

/* dm_microbench_cross — the whole-population split sweep's inner loop alone
 * (one fp64 max + checksum add per candidate pair, register x shared-memory
 * operands, the sweep's grid and occupancy): the issue-bound roofline of the
 * sweep.  *pairs receives the candidate pairs the launch evaluates. */
DM_API int dm_microbench_cross(int64_t iters, uint64_t* sink, int64_t* pairs, void* stream);

/* dm_sweep_timing — CUDA-event timing of the whole-population split sweep's
 * kernels on the calling thread: enable = 1 / 0 switches it (-1: unchanged);
 * when ms_tables / ms_sweep are given, waits for the last timed sweep and
 * returns its table phase (T image + side tables) and sweep kernel times. */
DM_API int dm_sweep_timing(int32_t enable, float* ms_tables, float* ms_sweep);

#ifdef __cplusplus
}
#endif

#endif /* DAGMESH_B200_H */
