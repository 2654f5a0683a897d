// batch.cuh -- per-batch device state shared by the kernels.
#pragma once
#include <stdint.h>

#include "../../include/bapipe_b200.h"
#include "common.cuh"

namespace bpk {

// One explore() query as the kernels see it.
struct QDesc {
    int32_t net, cl, N, nbase;
    int64_t mini;
    int64_t m_off;        // into Mpool (base micro-batch list)
    int64_t cand_off;     // first candidate (global index)
    int64_t stage_off;    // first bp_stage / candidate plan slot of this query
    int64_t qstage_off;   // per-query stage arrays (DP / refined plan, F/B/W)
    int64_t mslot_off;    // per-(query, M slot) arrays
    int32_t schema_ok;    // host-side validation (explorer.hpp:82-83, candidate_Ms)
    int32_t pad;
};

// Per-query device state.
struct QState {
    int32_t need_refine;
    int32_t grp_refine;    // some query sharing this one's class needs refine (rep only)
    int32_t dp_shape;      // 1 = InfeasibleShape (U < N) for the whole-layer DP
    int32_t refine_err;    // Err code of refine + refined-plan stage sums
    int32_t refined;       // refine ran
    int64_t target;        // max stage compute time of the DP plan (integer)
    int64_t refine_iters, refine_evals, refine_moves, refine_exact;
    // validate_plan (plan.hpp:41-85) of the refined plan, raised at simulate()
    int32_t vcode;         // BP_IP_* or 0
    int32_t verr;          // Err code of the coverage Rat sums
    int64_t vwhere;
    Rat vaux;
    // exact simulator scaling for the refined plan
    int64_t D;             // lcm of F/B denominators, 0 if >= 2^62
    int64_t sumFB_D;       // sum over stages of (F+B)*D, saturated at 2^62
};

// Per (query, M slot) bottleneck analysis (partition.hpp:454-466).
struct MState {
    int32_t bott;          // detect_comm_bottleneck().bottleneck
    int32_t err;           // overflow in Rat(min_bw) * target
    int64_t a_th;
    int64_t K;             // coarse block count
    int32_t coarse_ok;     // coarse DP done
    int32_t want;          // a coarse DP is needed (bottleneck, K >= N)
    int32_t q;             // owning query
    int32_t crep;          // mslot whose identical coarse DP this one shares, -1 = own
};

// Per-candidate plan kinds.
enum { PLAN_NONE = 0, PLAN_REFINED = 1, PLAN_WHOLE = 2 };

// Simulator classes: 0..4 = lanes per candidate 2, 4, 8, 16, 32 (one stage
// per lane); 5, 6, 7 = 32 lanes with 2, 4, 8 stages per lane; 8 = exact
// (Rat) path, thread per candidate; 9, 10 = exact (Rat) dataflow, block per
// candidate, thread per stage (xwave.cu), for the heavy exact candidates with
// N <= 32 / N <= 64.
enum { SIM_CLASSES = 11, SIM_EXACT = 8, SIM_FLOW = 9, SIM_FLOW_CLASSES = 2 };
// exact candidates with at least this many events (and FLOW_MIN_N <= N <= 64)
// go to the dataflow kernel: their serial walk would otherwise set the kernel
// time (measured on C5: 256 / 4 take the simulator phase from 15.2 to 14.3 ms
// against 1024 / 8)
constexpr int64_t FLOW_MIN_EVENTS = 256;
constexpr int64_t FLOW_MIN_N = 4;
// instrumentation slots of BatchDev::work (algorithmic work of one run)
// refine: boundary steps evaluated (and the longest query's count: the serial
// critical path); prune: candidate-stages estimated
enum { WORK_DP_WHOLE = 0, WORK_DP_COARSE = 1, WORK_REFINE = 2, WORK_PRUNE = 3, WORK_REFINE_MAX = 4,
       WORK_PRUNE_TRIALS = 5, WORK_PRUNE_MAX = 6, WORK_REFINE_MOVES = 7, WORK_REFINE_EXACT = 8,
       WORK_SIM_EVENTS = 9, WORK_SLOTS = WORK_SIM_EVENTS + SIM_CLASSES };
enum { XBUCKETS = 32768, XSIM_WARPS_PER_SM = 32 };

// Per-candidate device state (beyond the bp_candidate output record).
struct CState {
    int32_t plan_kind;
    int32_t sim_ready;     // 1: passed estimate + memory check, needs simulate
    int64_t D;             // simulator scale for this candidate's plan
    int32_t sim_cls;       // simulator class, -1 = not simulated
    int32_t sim_rep;       // candidate whose identical simulation this one shares, -1 = none
    int32_t pshare;        // prune: first estimate may be shared (see k_prune_key)
    int32_t est_first;     // prune: 1 = first estimate feasible, 2 = it raised (shareable outcomes)
    int32_t ft_trials;     // prune: memory_fine_tune trial moves (instrumentation)
    int32_t mem0_from;     // prune member: representative whose first-estimate memory it starts from, -1 = none
    int32_t mem0_buf;      // 0: that memory is in sMem (estimate was feasible), 1: in sMem0
    int64_t lb;            // BP_OPT_PRUNE_LB: makespan lower bound * D (scaled-integer class), -1 = none
    int32_t lbstate;       // LB_* below
    // a simulated candidate's outcome before its link busy fractions (the
    // only part of an asynchronous simulation that depends on the links):
    // 1 = the events and feature high-water fit (sim_mk is the makespan),
    // 2 = one of them overflowed; 0 = not simulated
    int32_t sim_core;
    Rat sim_mk;
    int32_t est_fbbal;     // prune: the first estimate's fb_balanced (asynchronous members form their heuristic)
    int32_t pad2;
};

// BP_OPT_PRUNE_LB states of a simulation representative: simulated normally,
// deferred (not simulated yet), simulated in round 1 (its query's seed) or
// round 2 (its bound did not exceed a best)
enum { LB_NONE = 0, LB_DEFERRED = 1, LB_ROUND1 = 2, LB_ROUND2 = 3 };

// DP work item: a (query, a_th) pair; a_th < 0 = whole-layer partition.
struct DPItem {
    int32_t q;
    int32_t mslot;         // -1 for the whole-layer DP
    int64_t a_th;
};

struct BatchDev {
    Pools P;
    int nq;
    int64_t ncand;
    const QDesc* q;
    const int64_t* Mpool;
    QState* qs;
    MState* ms;
    CState* cs;
    bp_candidate* cand;       // output records (device)
    bp_stage* stages;         // output stages (device), null in best-only mode
    bp_query_result* res;     // output per query (device)
    // per-query stage arrays (qstage_off)
    int32_t *qlo, *qhi;       // DP plan, then refined plan
    Rat *qlead, *qtrail;
    Rat *qF, *qB, *qW, *qT;
    uint8_t* qdirty;
    // per-candidate plan slots (stage_off + local*N)
    int32_t *clo, *chi;
    // per-candidate estimate scratch (stage_off + local*N), 6 arrays
    Rat *sF, *sB, *sW, *sMem;
    Rat* sMem0;               // first-estimate memory of infeasible prune-sharing candidates (null: none)
    int64_t *sA, *sSR;
    Rat* simbuf;              // exact simulator state, 9 Rats per stage slot
    int32_t* cq;              // candidate -> query
    int32_t* corder;          // ranking scratch, one slot per candidate
    // scheduling orders, built on the device each run (k_sched_*): queries by
    // (stage count, layers, network, chain type signature) so that a warp's
    // lanes run similar instruction streams; candidates follow their query
    int32_t* qorder;          // [nq]
    int32_t* cperm;           // [ncand]
    unsigned long long *okey, *okey2;   // [nq] order sort keys (in / out)
    int32_t *oval, *ocnt, *ocoff, *owfl, *owoff;   // [nq] sort values, counts, offsets
    void* otemp;              // CUB temporary storage
    size_t otemp_bytes;
    int32_t* sim_list;        // [SIM_CLASSES][ncand] candidate lists per simulator class
    int32_t* sim_count;       // [2 * SIM_CLASSES]: list lengths, then hand-out counters (k_sim_flow)
    int32_t* flow_tmp;        // [ncand] scratch of k_flow_sort
    // exact-simulator scheduling: counting sort of its list by (N, log2 M)
    int32_t* xkey;            // [ncand]
    int32_t* xsorted;         // [ncand]
    int32_t* xhist;           // [XBUCKETS] counts, then running offsets; [XBUCKETS] = chunk counter
    int max_N;                // largest stage count in the batch (exact-sim state sizing)
    int max_nbase;            // largest M-slot count of a query (k_bottleneck's grid)
    // batch-level deduplication of the whole-layer DP + refine (kernels.cu):
    // qrep[q] = the query whose results q shares (q itself if none); NULL in
    // the host emulation (no sharing)
    int32_t* qrep;
    unsigned long long* dkey; // [dmask+1] open-addressing table of class hashes
    int32_t* drep;            // [dmask+1] smallest query index per hash
    int32_t dmask;
    unsigned long long* skey; // [smask+1] simulation-input hashes (sim.cu)
    int32_t* srep;            // [smask+1] smallest candidate index per hash
    int32_t smask;
    unsigned long long* ckey; // [cmask+1] coarse-DP (class, a_th) hashes
    int32_t* crep;            // [cmask+1] smallest mslot index per hash
    int32_t cmask;
    int32_t dedup;            // BP_OPT_DEDUP: share identical subproblems
    int32_t plan_only;        // BP_OPT_PLAN_ONLY: stop after balance_partition + estimate
    int32_t prune_lb;         // BP_OPT_PRUNE_LB: simulate dominated scaled-integer candidates only if needed
    unsigned long long* qseed;// [nq] BP_OPT_PRUNE_LB: packed (lower bound, local index) minimum per query
    bp_rat* qinc;             // [nq] BP_OPT_PRUNE_LB: best simulated makespan per query ({0,0}: none)
    int32_t* rlist;           // [nq] queries to refine this run (compacted)
    int32_t* rcount;          // [2] list length, next entry
    int32_t* plist;           // [ncand] candidates to prune this run (compacted)
    int32_t* pctr;            // [3] list length, next chunk, (members' list) light entries at the back
    unsigned long long* pkey; // [pmask+1] estimate-input hashes (prune dedup)
    unsigned long long* pbest;// [pmask+1] max (capacity score, -index) per hash
    int32_t pmask;
    int details;              // write bp_stage records
    // DP work lists
    DPItem* dp_items;
    int32_t* dp_count;        // [0] whole-layer items, [1] coarse items
    unsigned long long* work; // instrumentation counters
};

}  // namespace bpk
