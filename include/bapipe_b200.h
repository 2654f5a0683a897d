/*
 * bapipe_b200.h -- C ABI of the B200-native BaPipe explorer (drop-in for the
 * reference's explore() candidate-evaluation path).
 *
 * The reference is a header-only C++20 library; its hot path is
 *   bapipe::explore(const NetworkProfile&, const ClusterSpec&, const TrainingConfig&)
 *   (/root/reference/proj/include/bapipe/explorer.hpp:80-155)
 * which, per (schedule kind x micro-batch count M) candidate, runs
 *   balance_partition   (partition.hpp:441-474)
 *   estimate            (cost_models.hpp:124-166)
 *   simulate            (simulator.hpp:264-274)
 * and ranks the survivors (explorer.hpp:142-152).
 *
 * This header is the thin, torch-free C boundary between the C++ host side
 * (include/bapipe_b200/explorer.hpp, the drop-in for explorer.hpp) and the
 * sm_100a kernels.  Inputs are structure-of-arrays copies of the reference's
 * value types with the std::map<string,int64> lookups resolved to integer
 * accelerator-type ids; outputs are fixed-size records whose rationals cross
 * the boundary as (int64 num, int64 den) pairs exactly as bapipe::Rat stores
 * them (rational.hpp:108-109, always reduced, den > 0).
 *
 * Ownership: every pointer argument is caller-owned host memory, read or
 * written only for the duration of the call.  A context owns its device
 * buffers.  One context per (host thread, device).  Calls are synchronous.
 */
#ifndef BAPIPE_B200_H
#define BAPIPE_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define BP_ABI_VERSION 1

/* ---- return codes of every entry point -------------------------------- */
enum {
    BP_OK = 0,
    BP_BAD_INPUT = 1,     /* malformed arguments (see bp_last_error) */
    BP_CUDA_ERROR = 2,    /* a CUDA call failed (see bp_last_error) */
    BP_NO_DEVICE = 3,     /* no CUDA device / extension cannot run */
    BP_OUT_OF_MEMORY = 4
};

/* ---- schedule kinds: order of enum ScheduleKind, schedule_kind.hpp:15 ---- */
enum { BP_KIND_1F1B_AS = 0, BP_KIND_FBP_AS = 1, BP_KIND_1F1B_SNO = 2, BP_KIND_1F1B_SO = 3 };
/* ---- execution modes: enum ExecutionMode, schedule_kind.hpp:11 ---------- */
enum { BP_MODE_SYNC = 0, BP_MODE_ASYNC = 1 };

/* ---- inputs ------------------------------------------------------------ */

/* NetworkProfile (profiles.hpp:24-51).  Accelerator types are global ids
 * 0..n_types-1; fp_us/bp_us are type-major [n_types][n_layers].  A value of 0
 * means "the layer has no time for this type" (the reference's map has no
 * entry); validate_pair (profiles.hpp:121-132) rejects a query whose chain
 * uses such a type. */
typedef struct {
    int32_t n_layers;
    int32_t n_types;
    const int64_t* fp_us;          /* [n_types * n_layers] */
    const int64_t* bp_us;          /* [n_types * n_layers] */
    const int64_t* weight_bytes;   /* [n_layers] */
    const int64_t* out_act_bytes;  /* [n_layers] */
} bp_network;

/* ClusterSpec (profiles.hpp:53-73).  min_micro_batch is [n_accels][4] in
 * ScheduleKind order; the reference's default for a missing kind is 1
 * (profiles.hpp:61-64). */
typedef struct {
    int32_t n_accels;
    int32_t exec_mode;             /* BP_MODE_* */
    const int32_t* type_id;        /* [n_accels] */
    const int64_t* mem_capacity;   /* [n_accels], bytes */
    const int64_t* min_micro;      /* [n_accels * 4] */
    const int64_t* link_bw;        /* [n_accels - 1], bytes/us */
} bp_cluster;

/* One explore() call: (network, the first n_stages accelerators and
 * n_stages-1 links of a cluster, TrainingConfig (profiles.hpp:75-78)).
 * Candidates are numbered kind-major in feasible_kinds order
 * (explorer.hpp:17-21), then in base-M-list order (explorer.hpp:90-96):
 * index = kind_slot * n_base + m_slot.  cand_offset / stage_offset locate the
 * query's records in the output arrays; bp_layout() fills them. */
typedef struct {
    int32_t network;
    int32_t cluster;
    int32_t n_stages;              /* chain prefix length; 0 = whole cluster */
    int32_t n_m;                   /* explicit micro_batch_candidates count; 0 = all divisors */
    int64_t mini_batch;
    const int64_t* m_list;         /* [n_m] or NULL */
    int64_t cand_offset;           /* first bp_candidate of this query */
    int64_t stage_offset;          /* first bp_stage of this query */
} bp_query;

/* ---- outputs ------------------------------------------------------------ */

typedef struct { int64_t num, den; } bp_rat;

/* Per-query outcome of explore(). */
enum {
    BP_Q_OK = 0,            /* returned normally; best = ranked.front() */
    BP_Q_NO_FEASIBLE = 1,   /* NoFeasiblePlan (explorer.hpp:135-141) */
    BP_Q_OVERFLOW = 2,      /* std::overflow_error("Rat: overflow") escaped (rational.hpp:90-91) */
    BP_Q_INVALID_PLAN = 3,  /* InvalidPlan escaped from simulate() (plan.hpp:41-85) */
    BP_Q_DOMAIN = 4,        /* std::domain_error escaped (rational.hpp:37,84) */
    BP_Q_REF_UB = 5,        /* the reference reads net.layers out of bounds here
                               (memory_fine_tune collapse, partition.hpp:359-373);
                               its result is undefined, ours is not compared */
    BP_Q_SCHEMA = 6         /* SchemaError before any candidate (explorer.hpp:82-83,
                               candidate_Ms 32-35, validate_pair) */
};

/* Per-candidate outcome: one pass of explorer.hpp:96-132 for one (kind, M). */
enum {
    BP_C_OK = 0,
    BP_C_REJ_MIN_MICRO = 1,        /* "min_micro_batch": "micro-batch size <mini/M> below minimum" */
    BP_C_REJ_COARSEN = 2,          /* "memory": "infeasible: coarsening for communication leaves <detail> blocks for <N> stages" */
    BP_C_REJ_FINETUNE = 3,         /* "memory": "infeasible: no contiguous plan satisfies memory for <kind>, M=<M>" */
    BP_C_REJ_FINETUNE_NOCONV = 4,  /* "memory": "infeasible: memory fine-tune did not converge" */
    BP_C_REJ_SHAPE = 5,            /* "partition": "infeasible shape: <detail> partition units for <N> stages" */
    BP_C_REJ_MEM_POST = 6,         /* "memory": "plan exceeds capacity" */
    BP_C_ERR_OVERFLOW = 7,         /* overflow_error escapes explore() */
    BP_C_ERR_INVALID_PLAN = 8,     /* InvalidPlan escapes; detail = BP_IP_* code, detail2 = stage/layer */
    BP_C_ERR_DOMAIN = 9,           /* domain_error escapes */
    BP_C_REF_UB = 10,              /* reference undefined behaviour (out-of-bounds layer read) */
    BP_C_PRUNED_LB = 11            /* BP_OPT_PRUNE_LB only: feasible and ranked, but not simulated --
                                      its makespan lower bound exceeds its query's best
                                      (SPEC.md:320); makespan {0, 0}, rank -1 */
};

/* InvalidPlan message codes (plan.hpp:42-83). */
enum {
    BP_IP_RANGE = 1,          /* "stage <d2>: layer range [lo,hi] out of bounds" */
    BP_IP_FRACTION = 2,       /* "stage <d2>: fractions must lie in (0, 1]" */
    BP_IP_FIRST = 3,          /* "stage 1 must start at layer 1 with full ownership" */
    BP_IP_CONTIG = 4,         /* "stage <d2>: not contiguous with previous stage" */
    BP_IP_SHARED_FULL = 5,    /* "stage <d2>: shared boundary layer must be fractional" */
    BP_IP_LEAD_UNSHARED = 6,  /* "stage <d2>: fractional lead without shared layer" */
    BP_IP_LAST = 7,           /* "last stage must end at layer L with full ownership" */
    BP_IP_COVERAGE = 8,       /* "layer <d2> coverage sums to <aux>, expected 1" */
    BP_IP_STAGE_COUNT = 9,    /* "plan stage count != cluster size" (simulator.hpp:271-272) */
    BP_IP_M = 10              /* "M >= 1 required" (simulator.hpp:83) */
};

typedef struct {
    int32_t status;          /* BP_Q_* */
    int32_t n_candidates;
    int32_t n_ranked;
    int32_t best;            /* candidate index of ranked.front(), or -1 */
    int32_t first_error;     /* candidate whose escaping error decides status, or -1 */
    int32_t best_kind;
    int64_t best_M;
    int64_t best_micro;
    bp_rat best_makespan;
    bp_rat best_peak_memory;
    bp_rat best_max_bw;
} bp_query_result;

typedef struct {
    int32_t kind;            /* BP_KIND_* */
    int32_t status;          /* BP_C_* */
    int64_t M;
    int64_t micro;           /* mini_batch / M (explorer.hpp:104) */
    int64_t detail;          /* see BP_C_* / BP_IP_* */
    int64_t detail2;
    int32_t rank;            /* position in ExplorationResult::ranked, or -1 */
    int32_t n_stages;
    int32_t heuristic;       /* CostEstimate::heuristic */
    int32_t plan_fractional; /* 1 if any stage owns a fractional layer */
    bp_rat makespan;         /* Candidate::simulated_makespan */
    bp_rat est_minibatch;    /* CostEstimate::minibatch_time */
    bp_rat bubble;           /* CostEstimate::bubble_fraction */
    bp_rat peak_memory;      /* Candidate::peak_memory */
    bp_rat max_bw_demand;    /* Candidate::max_bandwidth_demand */
    bp_rat aux;              /* coverage sum for BP_IP_COVERAGE */
} bp_candidate;

/* One stage of a ranked candidate's plan (plan.hpp:16-22) with its estimate
 * (cost_models.hpp:26-44).  bw_demand is link k = stage k -> k+1 and is {0,1}
 * on the last stage. */
typedef struct {
    int64_t lo, hi;          /* 1-based layer range */
    bp_rat lead, trail;      /* leading_fraction, trailing_fraction */
    bp_rat features;         /* features_mem[i] */
    bp_rat weights;          /* weights_mem[i] */
    bp_rat bw_demand;        /* bandwidth_demand[i] */
} bp_stage;

/* Compact per-query best record for multi-GPU sweeps (exchanged with one
 * allgather; ordered by bp_best_less()). */
typedef struct {
    bp_rat makespan;
    bp_rat peak_memory;
    bp_rat max_bw;
    int64_t M;
    int32_t kind;
    int32_t valid;           /* 0: no feasible candidate in this shard */
    int64_t query_id;        /* global query index (final tie-break) */
    int64_t pad;
} bp_best_record;

/* ---- entry points ------------------------------------------------------- */

typedef struct bp_ctx bp_ctx;
typedef struct bp_batch bp_batch;

/* Context on a CUDA device.  Returns NULL (and sets the global error) when the
 * device cannot be used: the product path never falls back to the CPU. */
bp_ctx* bp_create(int device);
void bp_destroy(bp_ctx* ctx);
const char* bp_last_error(const bp_ctx* ctx);   /* ctx may be NULL */
int bp_abi_version(void);

/* Upload (replace) the network / cluster tables.  Arrays are copied before
 * the call returns; the device copy completes asynchronously, after every run
 * this context enqueued before the call and before any run enqueued after it
 * (and before a bp_simulate_plan / bp_estimate_plan reads the tables). */
int bp_set_networks(bp_ctx* ctx, const bp_network* nets, int n);
int bp_set_clusters(bp_ctx* ctx, const bp_cluster* cls, int n);

/* Fill cand_offset / stage_offset of each query (dense, in order) and return
 * the totals the output arrays must hold. */
int bp_layout(bp_ctx* ctx, bp_query* q, int nq, int64_t* total_candidates,
              int64_t* total_stages);

/* explore() for a batch of queries: host in, host out.  cand / stages may be
 * NULL (best-only mode).  stream is a cudaStream_t (NULL = legacy stream). */
int bp_explore_batch(bp_ctx* ctx, const bp_query* q, int nq, bp_query_result* res,
                     bp_candidate* cand, bp_stage* stages, void* stream);

/* Split form for device-resident timing: prepare uploads the queries once,
 * run launches only the kernels (inputs already in HBM), fetch copies back.
 * A prepared batch refers to the context's current network / cluster tables:
 * after a later bp_set_networks / bp_set_clusters, run / fetch / best return
 * BP_BAD_INPUT for it (prepare it again). */
bp_batch* bp_batch_prepare(bp_ctx* ctx, const bp_query* q, int nq, int want_details,
                           void* stream);
int bp_batch_run(bp_ctx* ctx, bp_batch* b, void* stream);
int bp_batch_fetch(bp_ctx* ctx, bp_batch* b, bp_query_result* res, bp_candidate* cand,
                   bp_stage* stages, void* stream);
/* Reduce the batch's per-query bests to one bp_best_record written to DEVICE
 * memory dev_out (e.g. a tensor handed to an NCCL allgather). query_base is
 * added to local query indices. */
int bp_batch_best(bp_ctx* ctx, bp_batch* b, void* dev_out, int64_t query_base,
                  void* stream);
void bp_batch_free(bp_ctx* ctx, bp_batch* b);

/* Instrumentation: number of kernels launched since creation, and per-kernel
 * device time (CUDA events on the launching stream) when enabled. */
int64_t bp_launch_count(const bp_ctx* ctx);
int bp_set_profiling(bp_ctx* ctx, int enable);

/* Engine options (results never depend on them).
 *   BP_OPT_DEDUP (default 1): solve identical subproblems of a batch once --
 *   the whole-layer DP and refine per (network, stage count, type chain), the
 *   comm-coarsened DP per (that, a_th), simulations per identical inputs --
 *   and share the results; 0 evaluates every query and candidate
 *   independently. */
enum { BP_OPT_DEDUP = 1, BP_OPT_PLAN_ONLY = 2, BP_OPT_PRUNE_LB = 3, BP_OPT_SPLIT = 4 };
/*   BP_OPT_PLAN_ONLY (default 0): each candidate stops after balance_partition,
 *   its estimate and the memory check -- the reference's `bapipe plan`
 *   (tools/bapipe.cpp:152-170), which calls balance_partition for one
 *   (kind, M) with no min-micro filter and no simulation.  Feasible candidates
 *   get BP_C_OK with makespan 0/1; want_details gives their plans. */
/*   BP_OPT_PRUNE_LB (default 0): estimate-based pruning, the reference's
 *   SPEC.md:320 promise (its explore() simulates every candidate).  A
 *   candidate whose simulation provably cannot raise (the scaled-integer
 *   simulator class) is simulated only if its makespan lower bound
 *   max_b [sum_{s<b} (F_s + B_s + 2 SR_s [sync]) + M (F_b + B_b)] does not
 *   exceed its query's best simulated makespan; the others get
 *   BP_C_PRUNED_LB.  Every bp_query_result is byte-identical to the
 *   unpruned run (status, n_ranked, best, first_error and the best's
 *   values); only per-candidate records of pruned candidates differ. */
/*   BP_OPT_SPLIT (default 1 = up to four parts): a batch of at least 4096
 *   queries runs as concurrent parts on their own streams -- the queries of
 *   each of the batch's largest stage counts (the longest refine walks), then
 *   the rest; a part needs 512 queries.  A value k >= 2 asks for up to k
 *   parts; 0 turns it off.  Results are identical either way. */
int bp_set_option(bp_ctx* ctx, int option, int64_t value);

/* ---- one plan: full-timeline simulate and estimate ----------------------
 * simulate(kind, plan, net, cluster, M, micro, mini_batches)
 * (simulator.hpp:264-274, 81-246) and estimate(kind, plan, net, cluster, M,
 * micro) (cost_models.hpp:124-166) for a caller-given plan on network
 * `network` and the first n_stages accelerators of cluster `cluster`.  The
 * caller checks the kind against the cluster's mode (check_mode) first. */
typedef struct {
    int32_t network;
    int32_t cluster;
    int32_t kind;                  /* BP_KIND_* */
    int32_t n_stages;              /* the plan's stage count */
    int64_t M;
    int64_t micro;                 /* micro-batch size */
    int64_t mini_batches;          /* simulate only; the CLI uses 1 */
    const int32_t* lo;             /* [n_stages], 1-based layers */
    const int32_t* hi;
    const bp_rat* lead;            /* leading / trailing fractions */
    const bp_rat* trail;
} bp_plan_request;

/* Timeline event (simulator.hpp:16-36); kind: 0 FP, 1 BP, 2 SEND_F,
 * 3 RECV_F, 4 SEND_B, 5 RECV_B. */
typedef struct {
    int64_t stage;                 /* 1-based */
    int32_t kind;
    int32_t pad;
    int64_t micro_batch;           /* 1-based, numbered across mini-batches */
    bp_rat start;
    bp_rat end;
} bp_event;

typedef struct {
    int32_t status;                /* BP_C_OK, BP_C_ERR_OVERFLOW, BP_C_ERR_DOMAIN,
                                      BP_C_ERR_INVALID_PLAN, BP_C_REF_UB */
    int32_t pad;
    int64_t detail;                /* BP_IP_* for BP_C_ERR_INVALID_PLAN */
    int64_t detail2;               /* stage / layer */
    bp_rat aux;                    /* coverage sum for BP_IP_COVERAGE */
    bp_rat makespan;               /* Timeline::makespan */
    int64_t n_events;
} bp_timeline_result;

/* events: [cap] in the reference's order (stage, start, kind, micro-batch);
 * cap >= mini_batches * (2*n*M + 4*(n-1)*M) always suffices.  highwater,
 * weight_static: [n_stages]; busy: [n_stages - 1] (per_stage_feature_highwater,
 * per_stage_weight_static, per_link_busy_fraction).  Returns BP_OK when the
 * device ran (the outcome is in res->status), else an error code. */
int bp_simulate_plan(bp_ctx* ctx, const bp_plan_request* req, bp_timeline_result* res, bp_event* events,
                     int64_t cap, bp_rat* highwater, bp_rat* weight_static, bp_rat* busy);

typedef struct {
    int32_t status;                /* BP_C_OK, BP_C_ERR_OVERFLOW, BP_C_ERR_DOMAIN, BP_C_REF_UB */
    int32_t heuristic;
    bp_rat minibatch_time;
    bp_rat bubble_fraction;
} bp_estimate_result;

/* stages: [n_stages]; echoes the plan and fills features, weights and
 * bw_demand (link k in stages[k-1]); mem_infeasible: [n_stages], 1 where
 * features + weights exceed the accelerator's capacity. */
int bp_estimate_plan(bp_ctx* ctx, const bp_plan_request* req, bp_estimate_result* res, bp_stage* stages,
                     int32_t* mem_infeasible);
/* Copies up to cap entries: names (NUL-separated, 48 bytes each), total ms,
 * launch counts and algorithmic work units.  Returns the entry count. */
int bp_kernel_stats(const bp_ctx* ctx, char* names48, double* ms, int64_t* launches,
                    double* work, int cap);
/* Bytes copied host->device and device->host since creation. */
int bp_transfer_stats(const bp_ctx* ctx, int64_t* h2d_bytes, int64_t* d2h_bytes);

/* Deterministic argmin order for bp_best_record (makespan, peak_memory,
 * max_bw, M, kind, query_id); the first five keys are explorer.hpp:144-151. */
int bp_best_less(const bp_best_record* a, const bp_best_record* b);

#ifdef __cplusplus
}
#endif
#endif /* BAPIPE_B200_H */
