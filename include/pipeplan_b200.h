/*
 * pipeplan_b200.h — C ABI of libpipeplan_b200.so, the sm_100a planning path
 * of arXiv 2204.10562 ("pipeplan" reference package).
 *
 * The reference has no FFI: its boundary is the Python library API exported
 * by pipeplan/__init__.py:96-174.  Every entry point below replaces the
 * inside of one reference function and is bound by the Python drop-in
 * package (paper_2204_10562_b200/_lib.py, ctypes); INTEGRATION.md shows the
 * binding.  Conventions:
 *   - plain C types, caller-allocated DEVICE memory for every array (the
 *     library never allocates long-lived memory and never frees caller memory;
 *     scratch comes from the caller's fp64 workspace `ws`);
 *   - every launch goes to the caller's stream (cudaStream_t passed as void*);
 *   - status: 0 ok, negative PP_E* on error, message via pp_last_error()
 *     (thread-local).  Planning infeasibility is a VALUE (+inf / flag 0), as in
 *     the reference (partition.py:115-121); simulation stalls are reported per
 *     plan in pp_sim_batch.status (scheduler.py:207-214).
 *   - device indices are positions in the ascending-sorted GPU id list; the
 *     bandwidth matrix bw is V*V, symmetric, row-major over those positions.
 *   - fp64 everywhere, IEEE round-to-nearest, no FMA contraction
 *     (nvcc -fmad=false): results are bit-identical to the reference's
 *     Python float arithmetic on the same inputs.
 */
#ifndef PIPEPLAN_B200_H
#define PIPEPLAN_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PP_OK 0
#define PP_EINVAL (-1)   /* bad argument / size beyond the build's limits   */
#define PP_ECUDA (-3)    /* CUDA runtime error (message has the CUDA text)   */

/* pp_instance.flags */
#define PP_ALLOW_REPLICATION 1   /* PartitionSolver(allow_replication=True) (partition.py:49-51) */
#define PP_SUM_NAIVE 2           /* CPython <= 3.11 float sum(); default is the 3.12+ Neumaier sum */
#define PP_GIVEN_ORDER 4         /* order[] is an input (caller's DeviceOrdering); else RDO fills it */

/* Build limits (checked by pp_layout). */
#define PP_MAX_LAYERS 4096
#define PP_MAX_GPUS 512

/* One planning instance: spp(profile, cluster, M) (planner.py:57).  All
 * *_off fields are element offsets into the pp_batch arrays; pp_layout()
 * fills them. */
typedef struct {
    int32_t L, V, M, flags;
    int64_t layer_off;   /* fwd/bwd/param[layer_off + l-1]; efwd/ebwd[layer_off + l-1], l < L      */
    int64_t bw_off;      /* bw[bw_off + a*V + b]                                                    */
    int64_t order_off;   /* order[order_off + rank-1] = device index                                */
    int64_t sweep_off;   /* sweep_*[sweep_off + xi-1], xi = 1..V                                     */
    int64_t stage_off;   /* stage_*[stage_off + xi(xi-1)/2 + n-1]: stage n of the best xi-stage plan */
    int64_t ws_off;      /* fp64 scratch: tables, DP slices W_i, expansion X (pp_layout sizes it)    */
    int64_t ev_off;      /* ev_start/ev_end[ev_off + (m-1)*(4N-3) + pos-1] for the selected plan    */
    int64_t ar_off;      /* ar_start/ar_end[ar_off + n-1], selected plan                            */
} pp_instance;

/* A batch of planning instances and every array they use (device pointers). */
typedef struct {
    int32_t n_inst;
    int32_t max_L, max_V;             /* host copies: maxima over the batch                       */
    const pp_instance *inst;          /* device [n_inst]                                          */
    const double *fwd, *bwd, *param;  /* profile (model.py:24-30)                                 */
    const double *efwd, *ebwd;        /* edges (model.py:33-39)                                   */
    const double *bw;                 /* cluster (model.py:62-81)                                 */
    int32_t *order;                   /* device order (ordering.py:94-113)                        */
    /* per-xi sweep (planner.py:30-37, SweepEntry) */
    double *sweep_w;                  /* W: best workload, +inf if infeasible                     */
    double *sweep_mk;                 /* simulated makespan (simulate_pe)                         */
    double *sweep_bound;              /* lemma1_bound                                             */
    int32_t *sweep_r;                 /* last-stage width of the best plan, 0 if infeasible       */
    /* best plan per xi (partition.py:144-162): layer interval and device-rank interval */
    int32_t *stage_ls, *stage_le, *stage_dlo, *stage_dhi;
    /* selection (planner.py:66-77) */
    int32_t *best_xi;                 /* [n_inst]                                                 */
    double *best_mk;                  /* [n_inst]                                                 */
    double *phi;                      /* [n_inst] cost.py:131-142                                 */
    /* schedule of the selected plan (optional: NULL skips event capture) */
    double *ev_start, *ev_end;
    double *ar_start, *ar_end;
    double *ws;                       /* fp64 workspace, pp_layout() doubles.  May be NULL for a
                                         batch used only with pp_phi / pp_simulate (caller plans
                                         need no DP tables); every other entry point then fails
                                         with PP_EINVAL instead of touching it                  */
    double *gamma;                    /* [n_inst] cost.py:126-128, written by pp_phi; NULL skips  */
    /* schedule order of the selected plan's events (optional, needs ev_start):
     * ev_order[ev_off + k] = (m-1)*(4N-3) + pos-1 of the k-th event of the
     * reference's Schedule.events order (start, resource key, microbatch,
     * position; scheduler.py:227-231); NULL skips */
    int32_t *ev_order;
    int32_t max_M;                    /* host copy: max microbatch count over the batch (0 = unknown;
                                         sizes the event-order launch)                        */
    int64_t ws_doubles;               /* size of ws in doubles; > 0: pp_rdo / pp_prm / pp_spp check
                                         every instance's workspace range (L, V limits and
                                         ws_off + pp_layout's per-instance size <= ws_doubles)
                                         against it first (one small D2H of the instance table +
                                         a stream sync) and return PP_EINVAL; 0 = unchecked   */
} pp_batch;

/* ---- host helpers (no device work) ------------------------------------ */
const char *pp_version(void);
const char *pp_last_error(void);
int pp_device_count(void);

/* Fill inst[k] offsets for n instances of sizes L[k], V[k] (M[k], flags[k]
 * copied).  Returns totals through the out-pointers: layer, bw, order, sweep,
 * stage, event, allreduce element counts and workspace doubles.  Host only. */
int pp_layout(int32_t n, const int32_t *L, const int32_t *V, const int32_t *M, const int32_t *flags,
              pp_instance *inst, int64_t *n_layer, int64_t *n_bw, int64_t *n_order, int64_t *n_sweep,
              int64_t *n_stage, int64_t *n_ev, int64_t *n_ar, int64_t *n_ws);

/* ---- planning path -------------------------------------------------------
 * Each call enqueues kernels on `stream` and returns without synchronising. */

/* rdo(cluster) for every instance without PP_GIVEN_ORDER (ordering.py:94-113). */
int pp_rdo(const pp_batch *b, void *stream);

/* Number of speculative rounds pp_rdo runs before its sequential finisher
 * (default 1; 0 = the sequential recursion only).  The order is the
 * reference's either way; this is a performance / test knob.  Returns the
 * previous value, or PP_EINVAL outside 0..64.  Process-wide. */
int pp_rdo_set_rounds(int32_t rounds);

/* PartitionSolver over all cells + best_partition(xi) for every xi
 * (partition.py:41-162): fills sweep_w, sweep_r, stage_*. */
int pp_prm(const pp_batch *b, void *stream);
/* (The per-step schedule replays a CUDA graph cached per batch shape, per host
 * thread; each cache entry owns 2.3 KB of device memory for the batch
 * descriptors its kernels read.  Up to 8 shapes are cached.) */

/* DP schedule for batches inside the shared-memory limits (L, V <= 128):
 * 0 = one launch pair per wavefront step (replayed as a cached CUDA graph),
 * 3 = one CTA per instance, 2 (default) = auto (one CTA per instance for
 * >= 2 x SMs instances with L * V <= 2048, else per step).  Other values:
 * PP_EINVAL.  Bit-identical results; a performance / test knob.  Returns the
 * previous mode.  Process-wide. */
int pp_dp_set_persistent(int32_t mode);

/* Combine early exit (default 1): for stage-term triangles certified
 * non-increasing in l', the (min, max) fold scans l' downward and stops once no
 * remaining candidate can lower a cell.  Identical results; a test knob.
 * Returns the previous value (needs a device: the flag is device state). */
int pp_dp_set_early_exit(int32_t on);

/* Combine kernel of the per-step DP schedule: 1 = crossing search
 * (combine_bis.cu: bisection for the valley of max(X, S) under a certified
 * monotone stage-term triangle), 0 = exhaustive register tiles, 2 (default) =
 * auto (crossing search for single-instance batches, where the wavefront is
 * latency-bound; tiles above).  Identical results; a performance / test knob.
 * Returns the previous kind. */
int pp_dp_set_combine(int32_t kind);

/* RDO deduplication across a batch (instances with bitwise-equal bandwidth
 * matrices share one RDO run): 0 off, 1 (default) auto = only for batches of
 * more than 2 x SMs instances (RDO is latency-bound below that), 2 always.
 * Identical results; a performance / test knob.  Returns the previous mode. */
int pp_rdo_set_dedup(int32_t mode);

/* Debug: per-CTA timeline of the per-step expand / combine kernels (4 x u64 per
 * CTA: kind << 56 | j << 40 | smid << 32 | block id, start, end, 0); NULL
 * disables.  Not on the planning path. */
int pp_step_trace(uint64_t *d_buf, int32_t cap);

/* simulate_pe + lemma1_bound for every feasible xi plan (scheduler.py:75-238):
 * fills sweep_mk, sweep_bound. */
int pp_pe_sweep(const pp_batch *b, void *stream);

/* spp selection (planner.py:66-88): best_xi, best_mk, phi; then replays the
 * selected plan into ev_start/ev_end and ar_start/ar_end when ev_start != NULL. */
int pp_select(const pp_batch *b, void *stream);

/* phi(profile, cluster) per instance into phi[] (cost.py:126-142). */
int pp_phi(const pp_batch *b, void *stream);

/* The whole spp(): pp_phi, pp_rdo, pp_prm, pp_pe_sweep, pp_select. */
int pp_spp(const pp_batch *b, void *stream);

/* DP table access for PartitionSolver.solve(l, xi, r, i) (partition.py:95-142):
 * for each query q (device arrays, 1-based arguments already range-checked by
 * the caller) write W to w[q] and the realizing fragments (ls, le, dlo, dhi)
 * to frag[q*4*max_xi ...]; feasible[q] = 1/0.  Requires a prior pp_prm on the
 * same batch and workspace. */
int pp_prm_query(const pp_batch *b, int32_t n_query, const int32_t *q_inst, const int32_t *q_l,
                 const int32_t *q_xi, const int32_t *q_r, const int32_t *q_i, int32_t max_xi,
                 double *w, int32_t *frag, int32_t *feasible, void *stream);

/* ---- simulation of caller plans (simulate_with_order / simulate_pe) -----
 * One pp_plan per plan; resources are numbered in chain order
 * (0 = stage1, 1 = chan1, 2 = stage2, ...), R = 2N-1 of them. */
#define PP_SIM_FORWARD_BARRIER 1   /* simulate_with_order(forward_barrier=True)          */
#define PP_SIM_PE_ORDER 2          /* queues = compute_execution_order(plan) (closed form) */
#define PP_SIM_CYCLE 4             /* simulate_cycle_schedule (scheduler.py:241-296)       */
#define PP_SIM_COSTS_ONLY 8        /* per-lane costs + workload + bound, no simulation    */

/* per-lane cost record (lane_cost[(lane_off + r) * PP_LANE_COST_FIELDS + f]) */
#define PP_LANE_COST_FIELDS 7
/* stage lane: F (FB for the last stage) duration, B duration, stage_compute_time,
 *             allreduce_time (0 unless replicated), split F duration and split B
 *             duration (stage_*_time / k, also for the last stage),
 *             min pairwise bandwidth (+inf for one device)
 * chan lane : X duration (c_fwd), Y duration (c_bwd), c_fwd + c_bwd, 0, 0, 0,
 *             min cross bandwidth                                          */

typedef struct {
    int32_t inst;        /* instance (profile + bw) in the pp_batch            */
    int32_t N, M, flags;
    int64_t stage_off;   /* ls/le[stage_off + n-1]                              */
    int64_t devoff_off;  /* dev_off[devoff_off + 0..N] into devs                */
    int64_t queue_off;   /* q_off[queue_off + 0..R] into q_items pairs          */
    int64_t lane_off;    /* head[lane_off + 0..R-1]                             */
    int64_t ev_off;      /* ev_start, ev_end, scratch [ev_off + (m-1)*(4N-3) + pos-1]         */
    int64_t ar_off;      /* ar_*[ar_off + n-1]                                  */
} pp_plan;

typedef struct {
    int32_t n_plan, max_N;
    const pp_plan *plan;              /* device [n_plan]                        */
    const int32_t *ls, *le;           /* stage layer intervals (1-based)         */
    const int32_t *dev_off;           /* per plan N+1 offsets into devs          */
    const int32_t *devs;              /* device indices                          */
    const int32_t *q_off;             /* per plan R+1 offsets (pairs)            */
    const int32_t *q_items;           /* (m, pos) pairs                          */
    double *makespan, *bound;         /* [n_plan]                                */
    int32_t *status;                  /* [n_plan] 0 ok, 1 stalled                */
    int64_t *n_done;                  /* [n_plan] executions finished            */
    int32_t *head;                    /* per resource: next unserved queue index */
    double *ev_start, *ev_end;        /* per (m,pos); NULL skips event capture   */
    double *ar_start, *ar_end;        /* per stage                               */
    double *scratch;                  /* per (m,pos) completion times (generic queues) */
    double *lane_cost;                /* per resource PP_LANE_COST_FIELDS doubles; NULL skips */
    double *workload;                 /* [n_plan] cost_summary workload; NULL skips          */
    int32_t *cycles;                  /* [n_plan] cycle count (PP_SIM_CYCLE); NULL skips      */
} pp_sim_batch;

/* simulate_with_order / simulate_pe (scheduler.py:121-231) + lemma1_bound
 * (scheduler.py:234-238) for every plan.  Queue items must be unique, with
 * 1 <= m <= M and 1 <= pos <= 4N-3, each on its own block's resource (the
 * Python layer checks this). */
int pp_simulate(const pp_batch *inst_batch, const pp_sim_batch *s, void *stream);

/* Kernel launches issued by this library since load (evidence counter). */
int64_t pp_launch_count(void);

/* Measurement only (bench.py roofline denominator): launch a kernel that
 * saturates the fp64 min/max pipe; *n_ops receives the DMNMX count it
 * issues.  d_out: one device double (never written in practice). */
int pp_peak_minmax(double *d_out, int32_t iters, int64_t *n_ops, void *stream);

/* ---- ordering primitives ------------------------------------------------ */
/* global_min_cut (ordering.py:30-91) over a vertex subset of instance `k`:
 * verts (device, ascending, n of them); in_a[v] = 1 for side_a; weight[0]. */
int pp_min_cut(const pp_batch *b, int32_t k, const int32_t *verts, int32_t n, uint8_t *in_a,
               double *weight, void *stream);

/* ---- schedule validation (validate_schedule, scheduler.py:303-452) -------
 * Expected blocks of an N-stage plan, "expected index" e (scheduler.py:322-338):
 *   stages n = 1..N : fwd n, bwd n  (the last stage: fwdbwd N alone when merged_last)
 *   channels n = 1..N-1 : comm_fwd n, comm_bwd n
 * The host maps every event's label to e (-1 = not an expected block) and
 * its resource string to res_ok.  Slots are (m-1) * n_exp + e.
 * Phase 1 (structural, pp_validate_schedule with phase = 1):
 *   ev_flags[k] : 1 duplicate (not the first event of its slot), 2 ends
 *                 before it starts, 4 unexpected block, 8 unknown microbatch
 *   slot_flags  : 1 missing, 2 wrong resource, 4 wrong duration
 *                 (the LAST event of a slot is the one checked, as by_key keeps it)
 * Phase 2 (ordering; only meaningful when phase 1 found nothing):
 *   mn_flags[(m-1)*N + n-1] : bits 0..5 the six channel-n checks of
 *                 scheduler.py:376-391 in order, bit 6 the last-stage check (:392-393)
 *   ar_flags[n-1] : 1 missing, 2 starts early, 4 wrong duration, 8 unexpected
 *   ov_idx / ov_flags : per resource, its events sorted by (start, end, k);
 *                 ov_flags[j] = 1 when sorted item j overlaps item j-1
 *   scal[0..3] : expected makespan, forward max, backward min, f_start(1,1)
 *   stat[0..2] : first-start violated, barrier violated, makespan mismatch
 * Resources are stage n (lane 2n-2) / chan n (lane 2n-1); res_off[lane] is the
 * start of the lane's block in ov_idx (M items per expected label it hosts). */
#define PP_VAL_MERGED_LAST 1
#define PP_VAL_FORWARD_BARRIER 2

typedef struct {
    int32_t N, M, flags, n_exp;
    int64_t n_ev;
    const int32_t *ev_m, *ev_e;       /* microbatch, expected index (-1 unknown)  */
    const uint8_t *ev_res_ok;         /* resource string matches e's resource     */
    const double *ev_start, *ev_end;
    const double *lane_cost;          /* the plan's PP_LANE_COST_FIELDS records   */
    const uint8_t *win_has;           /* [N] AllReduce window given for stage n   */
    const double *win_start, *win_end;/* [N] (the last window given per stage)    */
    int32_t n_win_all;                /* every window's end enters the makespan   */
    const double *win_all_end;        /* [n_win_all]                              */
    double makespan;
    /* scratch + outputs (device) */
    int32_t *slot_first, *slot_last, *slot_count;   /* [M*n_exp] */
    uint8_t *ev_flags, *slot_flags, *mn_flags, *ar_flags, *ov_flags;
    int32_t *ov_idx;                  /* [M*n_exp] */
    const int32_t *res_off;           /* [2N] */
    double *part;                     /* [3*M + N] per-microbatch partials scratch  */
    double *scal;                     /* [4] */
    int32_t *stat;                    /* [3] */
    /* overlap-check sort scratch, needed only when 2*M > 8192 (the shared-memory
     * sort's capacity): per resource lane sort_cap keys, i.e. (2N-1)*sort_cap
     * doubles in each of sort_ks / sort_ke and int32 in sort_ki, sort_cap = the
     * next power of two >= 2*M.  NULL / 0 otherwise. */
    double *sort_ks;
    double *sort_ke;
    int32_t *sort_ki;
    int64_t sort_cap;
} pp_validate_args;

int pp_validate_schedule(const pp_validate_args *a, int32_t phase, void *stream);

/* ---- trace writer (host) ------------------------------------------------ */
/* write_trace text (fileio.py:170-188; numbers as format_number, fileio.py:32-38)
 * from event arrays: row k = res_names[ev_pos[k]], ev_m[k], labels[ev_pos[k]],
 * ev_start[k], ev_end[k]; then one "allreduce" row per window.  Host memory
 * only; formats on up to nthreads threads.  *out_len = bytes needed; PP_EINVAL
 * with "non-finite number in output: <x>" at the first inf/nan, or when the
 * text exceeds cap (out is then unspecified). */
int pp_format_trace(int64_t n_events, const int32_t *ev_m, const int32_t *ev_pos, const double *ev_start,
                    const double *ev_end, const char *const *res_names, const char *const *labels,
                    int32_t n_names, int32_t n_ar, const int32_t *ar_stage, const double *ar_start,
                    const double *ar_end, double makespan, char *out, int64_t cap, int64_t *out_len,
                    int32_t nthreads);

#ifdef __cplusplus
}
#endif
#endif /* PIPEPLAN_B200_H */
