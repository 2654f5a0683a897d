// phases.cuh -- per-thread bodies of the explore() pipeline kernels.
//
//   setup_query       K0  candidate records (explorer.hpp:87-108)
//   bottleneck_slot   K1b detect_comm_bottleneck + a_th + coarse block count
//                         per (query, micro-batch) (partition.hpp:454-465)
//   refine_query      K3a intra_layer_refine once per query (partition.hpp:469)
//                         + the refined plan's stage sums and validation
//   prune_candidate   K3b balance_partition's branch logic, estimate, memory
//                         fine-tune, explore's estimate (explorer.hpp:389-402)
//   sim_exact         K4  simulate() with exact Rat events (simulator.hpp:81-246)
//   rank_query        K5  ranking + query outcome (explorer.hpp:133-155)
// All are __host__ __device__ so tests/emu can replay them on the CPU.
#pragma once
#include "batch.cuh"
#include "model.cuh"

namespace bpk {

enum { C_PENDING = -1 };

BPK_HD int kind_of_slot(int mode, int k) {   // feasible_kinds, explorer.hpp:17-21
    return mode == MODE_ASYNC ? (k == 0 ? KIND_AS : KIND_FBP) : (k == 0 ? KIND_SNO : KIND_SO);
}

BPK_HD int status_of_err(uint32_t code) { return (int)code; }   // ERR_* == BP_C_*

// ---------------------------------------------------------------- K0
// lane / nlanes: the candidates of the query are shared among nlanes
// cooperating threads (a warp on the device, 1 in the host emulation)
BPK_HDNI void setup_query(const BatchDev& B, int qi, int lane = 0, int nlanes = 1) {
    const QDesc Q = B.q[qi];
    if (lane == 0) {
        B.qs[qi] = QState{};
        bp_query_result r = bp_query_result{};
        r.best = -1;
        r.first_error = -1;
        r.status = Q.schema_ok ? 0 : BP_Q_SCHEMA;
        r.n_candidates = Q.schema_ok ? 2 * Q.nbase : 0;
        B.res[qi] = r;
    }
    if (!Q.schema_ok) return;
    ChainView c = chain_view(B.P, Q.cl, Q.N);
    for (int64_t local = lane; local < 2 * (int64_t)Q.nbase; local += nlanes) {
        const int k = (int)(local / Q.nbase), m = (int)(local - (int64_t)k * Q.nbase);
        const int kind = kind_of_slot(c.mode, k);
        int64_t min_micro = 1;   // candidate_Ms, explorer.hpp:42-47
        for (int a = 0; a < Q.N; ++a) {
            int64_t mm = c.minm[4 * a + kind];
            if (mm > min_micro) min_micro = mm;
        }
        const int64_t ci = Q.cand_off + local;
        bp_candidate cd = bp_candidate{};
        cd.kind = kind;
        cd.M = B.Mpool[Q.m_off + m];
        cd.micro = Q.mini / cd.M;
        cd.rank = -1;
        cd.n_stages = Q.N;
        // (`bapipe plan` calls balance_partition with no min-micro filter)
        cd.status = (B.plan_only || Q.mini / cd.M >= min_micro) ? (int32_t)C_PENDING : (int32_t)BP_C_REJ_MIN_MICRO;
        B.cand[ci] = cd;
        B.cs[ci] = CState{};
        B.cq[ci] = qi;
    }
    for (int m = lane; m < Q.nbase; m += nlanes) B.ms[Q.mslot_off + m] = MState{};
}

// ---------------------------------------------------------------- K1b
// Returns 1 when a coarse DP item must be queued for (qi, m).
BPK_HDNI int bottleneck_slot(const BatchDev& B, int qi, int m) {
    const QDesc Q = B.q[qi];
    if (!Q.schema_ok || Q.N == 1 || m >= Q.nbase) return 0;
    QState& qs = B.qs[qi];
    if (qs.dp_shape) return 0;
    bool alive = B.cand[Q.cand_off + m].status == C_PENDING ||
                 B.cand[Q.cand_off + Q.nbase + m].status == C_PENDING;
    if (!alive) return 0;
    NetView v = net_view(B.P, Q.net);
    ChainView c = chain_view(B.P, Q.cl, Q.N);
    const int64_t micro = Q.mini / B.Mpool[Q.m_off + m];
    const int64_t target = qs.target;
    const int32_t* hi = B.qhi + Q.qstage_off;
    MState& ms = B.ms[Q.mslot_off + m];
    bool bott = false;
    for (int k = 0; k + 1 < Q.N; ++k) {           // detect_comm_bottleneck (228-241)
        int64_t a = v.a[hi[k] - 1] * micro;
        int64_t sr = a == 0 ? 0 : ceil_div64(a, c.bw[k]);
        if (sr > target) bott = true;
    }
    ms.bott = bott ? 1 : 0;
    if (!bott) {
        qs.need_refine = 1;
        return 0;
    }
    int64_t min_bw = c.bw[0];
    for (int k = 1; k + 1 < Q.N; ++k)
        if (c.bw[k] < min_bw) min_bw = c.bw[k];
    // a_th = (Rat(min_bw) * target / Rat(micro)).floor()  (460)
    i128 prod = (i128)min_bw * target;
    if (prod > (i128)INT64_MAX) { ms.err = ERR_OVERFLOW; return 0; }
    int64_t a_th = (int64_t)prod / micro;
    ms.a_th = a_th;
    // coarsen_by_comm block count: layers j < L with a_j <= a_th, plus L
    const int64_t n_sorted = v.L - 1;
    int64_t lo = 0, hi2 = n_sorted;                 // upper_bound in asort
    while (lo < hi2) {
        int64_t mid = (lo + hi2) >> 1;
        if (v.asort[mid] <= a_th) lo = mid + 1;
        else hi2 = mid;
    }
    ms.K = lo + 1;
    return ms.K >= Q.N ? 1 : 0;
}

// ---------------------------------------------------------------- K3a
// lcm accumulation for the simulator scale; returns 0 once above 2^62.
BPK_HD int64_t lcm_sat(int64_t D, int64_t d) {
    if (D == 0) return 0;
    uint64_t g = gcd_u64((uint64_t)D, (uint64_t)d);
    u128 l = (u128)(D / (int64_t)g) * (u128)d;
    if (l >= ((u128)1 << 62)) return 0;
    return (int64_t)l;
}

// Per-stage working arrays of one refine (the plan and the stage-time
// caches).  The kernel keeps them in shared memory (k_refine_smem); NULL =
// work in the query's global arrays.
struct RefineScratch {
    int32_t *lo, *hi;
    Rat *lead, *trail, *tF, *tB, *tT;
    uint8_t* dirty;
};

BPK_HD bool refine_wanted(const BatchDev& B, int qi) {
    const QDesc Q = B.q[qi];
    const QState& qs = B.qs[qi];
    // with batch dedup only the class representative refines (for its whole
    // class); the emulation (qrep == NULL) refines every query that needs it
    const bool need = B.qrep ? (B.qrep[qi] == qi && qs.grp_refine) : qs.need_refine;
    return Q.schema_ok && need && !qs.dp_shape && Q.N >= 2;
}

BPK_HD void refine_commit(const BatchDev& B, int qi, const NetView& v, const ChainView& c, const int32_t* lo,
                          const int32_t* hi, const Rat* lead, const Rat* trail, const int64_t* rs, bool copy, Err e);

// vo (nullable): the query's network view with its tables staged elsewhere
// (shared memory in k_refine_smem)
BPK_HDNI void refine_query_at(const BatchDev& B, int qi, const RefineScratch* sc, const NetView* vo = nullptr) {
    const QDesc Q = B.q[qi];
    if (!refine_wanted(B, qi)) return;
    NetView v = vo ? *vo : net_view(B.P, Q.net);
    ChainView c = chain_view(B.P, Q.cl, Q.N);
    const int64_t o = Q.qstage_off;
    int32_t* lo = sc ? sc->lo : B.qlo + o;
    int32_t* hi = sc ? sc->hi : B.qhi + o;
    Rat* lead = sc ? sc->lead : B.qlead + o;
    Rat* trail = sc ? sc->trail : B.qtrail + o;
    for (int s = 0; s < Q.N; ++s) {
        lead[s] = R(1);
        trail[s] = R(1);
        if (sc) { lo[s] = B.qlo[o + s]; hi[s] = B.qhi[o + s]; }
    }
    Err e{ERR_NONE};
    int64_t rs[4];
    if (sc) refine(v, c, lo, hi, lead, trail, sc->tF, sc->tB, sc->tT, sc->dirty, rs, e);
    else refine(v, c, lo, hi, lead, trail, B.qF + o, B.qB + o, B.qT + o, B.qdirty + o, rs, e);
    refine_commit(B, qi, v, c, lo, hi, lead, trail, rs, sc != nullptr, e);
}

// The refined plan (lo/hi/lead/trail, wherever the walk kept it) into the
// query's arrays, with the walk's stats and its error, then the plan's stage
// sums, simulator scale and validate_plan outcome.  Also the host emulation's
// tail after refine_fast_walk (tests/emu); k_refine_fast has a warp version.
BPK_HD void refine_commit(const BatchDev& B, int qi, const NetView& v, const ChainView& c, const int32_t* lo,
                          const int32_t* hi, const Rat* lead, const Rat* trail, const int64_t* rs, bool copy, Err e) {
    const QDesc Q = B.q[qi];
    QState& qs = B.qs[qi];
    const int64_t o = Q.qstage_off;
    if (copy) {
        for (int s = 0; s < Q.N; ++s) {
            B.qlo[o + s] = lo[s];
            B.qhi[o + s] = hi[s];
            B.qlead[o + s] = lead[s];
            B.qtrail[o + s] = trail[s];
        }
    }
    qs.refined = 1;
    qs.refine_iters = rs[0];
    qs.refine_evals = rs[1];
    qs.refine_moves = rs[2];
    qs.refine_exact = rs[3];
    // The refined plan's stage sums in estimate's order (stage_costs 103-119).
    int64_t D = 1;
    u128 sumFB = 0;
    for (int s = 0; s < Q.N && !e.bad(); ++s) {
        int32_t t = c.type[s];
        Rat F = stage_sum_frac(lo[s], hi[s], lead[s], trail[s], v.Pfp + (int64_t)t * (v.L + 1), e);
        Rat Bt = stage_sum_frac(lo[s], hi[s], lead[s], trail[s], v.Pbp + (int64_t)t * (v.L + 1), e);
        Rat W = stage_sum_frac(lo[s], hi[s], lead[s], trail[s], v.Pw, e);
        B.qF[o + s] = F;
        B.qB[o + s] = Bt;
        B.qW[o + s] = W;
        D = lcm_sat(lcm_sat(D, F.d), Bt.d);
    }
    qs.refine_err = e.code;
    if (e.bad()) return;
    qs.D = D;
    if (D) {
        for (int s = 0; s < Q.N; ++s) {
            sumFB += (u128)((i128)B.qF[o + s].n * (D / B.qF[o + s].d));
            sumFB += (u128)((i128)B.qB[o + s].n * (D / B.qB[o + s].d));
        }
        qs.sumFB_D = sumFB >= ((u128)1 << 62) ? -1 : (int64_t)sumFB;
    }
    // validate_plan of the refined plan (raised only when simulate() runs)
    Err ve{ERR_NONE};
    int64_t where = 0;
    Rat aux{0, 1};
    qs.vcode = validate_frac(lo, hi, lead, trail, Q.N, v.L, &where, &aux, ve);
    qs.verr = ve.code;
    qs.vwhere = where;
    qs.vaux = aux;
}

BPK_HDNI void refine_query(const BatchDev& B, int qi) { refine_query_at(B, qi, nullptr); }

// ---------------------------------------------------------------- K3b
BPK_HD EstScratch cand_scratch(const BatchDev& B, int64_t slot) {
    EstScratch s;
    s.F = B.sF + slot;
    s.B = B.sB + slot;
    s.W = B.sW + slot;
    s.Mem = B.sMem + slot;
    s.A = B.sA + slot;
    s.SR = B.sSR + slot;
    return s;
}

BPK_HD void fail(bp_candidate& cd, const Err& e) { cd.status = status_of_err(e.code); }

// pass: -1 = every candidate; 0 = candidates that do not use the refined plan
// (N = 1, InfeasibleShape, comm-bottleneck M slots: they can run while refine
// is still going); 1 = the refined-plan candidates.
BPK_HDNI void prune_candidate(const BatchDev& B, int64_t ci, int pass = -1) {
    bp_candidate& cd = B.cand[ci];
    if (cd.status != C_PENDING) return;
    const int qi = B.cq[ci];
    const QDesc Q = B.q[qi];
    const QState& qs = B.qs[qi];
    const int64_t local = ci - Q.cand_off;
    const int m = (int)(local % Q.nbase);
    const int N = Q.N;
    if (pass >= 0) {
        const bool refined_path = N > 1 && !qs.dp_shape && !B.ms[Q.mslot_off + m].bott;
        if (refined_path != (pass == 1)) return;
    }
    const int kind = cd.kind;
    const int64_t M = cd.M, micro = cd.micro;
    NetView v = net_view(B.P, Q.net);
    ChainView c = chain_view(B.P, Q.cl, N);
    const int64_t slot = Q.stage_off + local * N;
    int32_t* lo = B.clo + slot;
    int32_t* hi = B.chi + slot;
    EstScratch S = cand_scratch(B, slot);
    CState& cs = B.cs[ci];
    Err e{ERR_NONE};
    EstOut o;
    int plan_kind = PLAN_WHOLE;
    int ft = FT_OK;
    // A prune-sharing member whose representative's first estimate (same
    // inputs, hence same values and no error) is infeasible for it starts
    // from that estimate's memory (k_prune_members); memory_fine_tune reads
    // nothing else of it.  Representatives keep theirs for the members.
    const Rat* mem0 = nullptr;
    if (cs.pshare && cs.mem0_from >= 0) {
        const QDesc Qr = B.q[B.cq[cs.mem0_from]];
        mem0 = (cs.mem0_buf ? B.sMem0 : B.sMem) + Qr.stage_off + (cs.mem0_from - Qr.cand_off) * N;
    }
    auto first_estimate = [&](const auto& plan) {
        if (mem0) {
            for (int s = 0; s < N; ++s) S.Mem[s] = mem0[s];
            o.feasible = 0;
        } else {
            estimate(plan, v, c, kind, M, micro, S, o, nullptr, e);
            cs.est_fbbal = o.fb_balanced;
            if (cs.pshare && B.sMem0 && !e.bad() && !o.feasible)
                for (int s = 0; s < N; ++s) B.sMem0[slot + s] = S.Mem[s];
        }
        cs.est_first = e.bad() ? 2 : o.feasible ? 1 : 0;
    };
    if (N == 1) {                                                  // 447-451
        lo[0] = 1;
        hi[0] = (int32_t)v.L;
        WholePlan wp{&v, &c, lo, hi};
        estimate(wp, v, c, kind, M, micro, S, o, nullptr, e);
        if (!e.bad()) ft = memory_fine_tune(v, c, kind, M, micro, lo, hi, nullptr, nullptr, S, o, e);
    } else if (qs.dp_shape) {                                      // 115-117
        cd.status = BP_C_REJ_SHAPE;
        cd.detail = v.L;
        return;
    } else {
        const MState ms = B.ms[Q.mslot_off + m];
        if (ms.bott) {                                             // 456-467
            if (ms.err) { cd.status = status_of_err(ms.err); return; }
            if (ms.K < N) { cd.status = BP_C_REJ_COARSEN; cd.detail = ms.K; return; }
            first_estimate(WholePlan{&v, &c, lo, hi});
            if (!e.bad()) ft = memory_fine_tune(v, c, kind, M, micro, lo, hi, nullptr, nullptr, S, o, e);
        } else {                                                   // 469-473
            if (qs.refine_err) { cd.status = status_of_err(qs.refine_err); return; }
            const int64_t qo = Q.qstage_off;
            first_estimate(CachedPlan{B.qhi + qo, B.qF + qo, B.qB + qo, B.qW + qo});
            if (!e.bad() && !o.feasible) {
                for (int s = 0; s < N; ++s) { lo[s] = B.qlo[qo + s]; hi[s] = B.qhi[qo + s]; }
                ft = memory_fine_tune(v, c, kind, M, micro, lo, hi, B.qlead + qo, B.qtrail + qo, S, o, e);
            } else {
                plan_kind = PLAN_REFINED;
            }
        }
    }
    cs.ft_trials = o.trials;
    if (e.bad()) { fail(cd, e); return; }
    if (ft == FT_REJ) { cd.status = BP_C_REJ_FINETUNE; return; }
    if (ft == FT_NOCONV) { cd.status = BP_C_REJ_FINETUNE_NOCONV; return; }
    // explore's estimate on the final plan (explorer.hpp:398-402).  The last
    // estimate computed above (balance_partition's, or the one memory_fine_tune
    // accepted its final plan on) is of this very plan: same values, same
    // (absent) errors, so o and the scratch S are reused as is.
    bp_stage* st = B.details ? B.stages + slot : nullptr;
    if (!o.feasible) { cd.status = BP_C_REJ_MEM_POST; return; }
    cd.est_minibatch = bp_rat{o.minibatch.n, o.minibatch.d};
    cd.bubble = bp_rat{o.bubble.n, o.bubble.d};
    cd.heuristic = o.heuristic;
    cd.peak_memory = bp_rat{o.peak_mem.n, o.peak_mem.d};
    cd.max_bw_demand = bp_rat{o.max_bw.n, o.max_bw.d};
    cd.plan_fractional = 0;
    cs.plan_kind = plan_kind;
    cs.sim_ready = 1;
    if (st || plan_kind == PLAN_REFINED) {
        const int64_t qo = Q.qstage_off;
        const bool dbl = (kind == KIND_FBP || kind == KIND_SO);
        for (int s = 0; s < N; ++s) {
            Rat ld = plan_kind == PLAN_REFINED ? B.qlead[qo + s] : R(1);
            Rat tr = plan_kind == PLAN_REFINED ? B.qtrail[qo + s] : R(1);
            if (ld.n != ld.d || tr.n != tr.d) cd.plan_fractional = 1;
            if (!st) continue;
            st[s].lo = plan_kind == PLAN_REFINED ? B.qlo[qo + s] : lo[s];
            st[s].hi = plan_kind == PLAN_REFINED ? B.qhi[qo + s] : hi[s];
            st[s].lead = bp_rat{ld.n, ld.d};
            st[s].trail = bp_rat{tr.n, tr.d};
            // features / weights exactly as estimate formed them (no new ops)
            Err dummy{ERR_NONE};
            Rat fm = rat_mul(R(N - s), R(S.A[s]), dummy);
            if (dbl) fm = rat_mul(R(2), fm, dummy);
            Rat wm = rat_mul(R(2), S.W[s], dummy);
            st[s].features = bp_rat{fm.n, fm.d};
            st[s].weights = bp_rat{wm.n, wm.d};
            if (s + 1 < N) {
                // bandwidth_demand of link s: the cut activation = A[s+1]
                Rat d = (kind == KIND_FBP) ? rat_div(rat_mul(R(2), R(S.A[s + 1]), dummy), rat_add(o.Fm, o.Bm, dummy), dummy)
                                           : rat_div(R(S.A[s + 1]), o.Fm, dummy);
                st[s].bw_demand = bp_rat{d.n, d.d};
            } else {
                st[s].bw_demand = bp_rat{0, 1};
            }
        }
    }
}

// ---------------------------------------------------------------- K4 (exact)
// simulate(): validate_plan, chain_instance, simulate_chain with exact Rat
// values for every event.  Ops are visited position by position: all F ops
// at a position in ascending stage order, then all B ops in descending stage
// order -- a topological order of the reference's sorted op list
// (simulator.hpp:107-125), so every value equals the reference's.
// Per link a 4-slot ring keyed by micro-batch carries arrivals.
struct StageOp {
    int is_f;
    int64_t m;
};

BPK_HD StageOp op_at(int64_t p, int64_t w, int64_t M) {
    if (p < w) return StageOp{1, p + 1};
    int64_t r = p - w;
    if (r < 2 * (M - w)) {
        if ((r & 1) == 0) return StageOp{0, r / 2 + 1};
        return StageOp{1, w + (r + 1) / 2};
    }
    return StageOp{0, (M - w) + (r - 2 * (M - w)) + 1};
}

// simulate() entry: validate_plan (plan.hpp:41-85), then choose the
// simulator.  Returns the class (see SIM_CLASSES) or -1 when the candidate
// is finished (InvalidPlan / error).
//   Fast path: every event time is an exact multiple of 1/D, D = lcm of the
//   stage F/B denominators; if D * (M * sum(F+B) + 2M * sum(SR)) < 2^61 --
//   an upper bound on every path length, hence on every event -- all events
//   are int64 multiples of 1/D, and no reduced numerator/denominator can
//   exceed int64, so the reference cannot overflow there (rational.hpp:90).
//   Otherwise the exact Rat simulator decides (slow path).
BPK_HDNI int sim_classify(const BatchDev& B, int64_t ci) {
    CState& cs = B.cs[ci];
    if (!cs.sim_ready) return -1;
    bp_candidate& cd = B.cand[ci];
    const int qi = B.cq[ci];
    const QDesc Q = B.q[qi];
    const QState& qs = B.qs[qi];
    const int64_t local = ci - Q.cand_off;
    const int N = Q.N;
    const int64_t M = cd.M, micro = cd.micro;
    NetView v = net_view(B.P, Q.net);
    ChainView c = chain_view(B.P, Q.cl, N);
    const int64_t slot = Q.stage_off + local * N;
    const int64_t qo = Q.qstage_off;
    const int32_t* hi = cs.plan_kind == PLAN_REFINED ? B.qhi + qo : B.chi + slot;
    const int32_t* lo = cs.plan_kind == PLAN_REFINED ? B.qlo + qo : B.clo + slot;
    if (cs.plan_kind == PLAN_REFINED) {
        if (qs.vcode) {
            cd.status = BP_C_ERR_INVALID_PLAN;
            cd.detail = qs.vcode;
            cd.detail2 = qs.vwhere;
            cd.aux = bp_rat{qs.vaux.n, qs.vaux.d};
            return -1;
        }
        if (qs.verr) { cd.status = status_of_err(qs.verr); return -1; }
    } else {
        int64_t where = 0;
        int vc = validate_whole(lo, hi, N, v.L, &where);
        if (vc) {
            cd.status = BP_C_ERR_INVALID_PLAN;
            cd.detail = vc;
            cd.detail2 = where;
            return -1;
        }
    }
    int64_t D;
    u128 sumFB;
    if (cs.plan_kind == PLAN_REFINED) {
        D = qs.D;
        if (D == 0 || qs.sumFB_D < 0) return SIM_EXACT;
        sumFB = (u128)qs.sumFB_D;
    } else {
        D = 1;
        sumFB = 0;
        for (int s = 0; s < N; ++s) {
            int32_t t = c.type[s];
            sumFB += (u128)stage_sum_whole(lo[s], hi[s], v.Pc + (int64_t)t * (v.L + 1));
        }
    }
    u128 sumSR = 0;
    for (int k = 0; k + 1 < N; ++k) {
        int64_t a = v.a[hi[k] - 1] * micro;
        sumSR += (u128)(a == 0 ? 0 : ceil_div64(a, c.bw[k]));
    }
    u128 bound = (u128)M * sumFB + (u128)(2 * M) * (u128)D * sumSR;
    cs.D = D;
    if (bound >= ((u128)1 << 61)) return SIM_EXACT;
    if (N <= 2) return 0;
    if (N <= 4) return 1;
    if (N <= 8) return 2;
    if (N <= 16) return 3;
    if (N <= 32) return 4;
    if (N <= 64) return 5;
    if (N <= 128) return 6;
    if (N <= 256) return 7;
    return SIM_EXACT;
}

// Per-stage state of the exact simulator, element s at base[s * stride]
// (stride 32 on the GPU interleaves a warp's lanes for coalescing).
struct SimState {
    Rat *fr, *pF, *pB, *F, *B;
    int64_t *SR, *A;
    int stride;
    BPK_HD Rat& f(int s) const { return fr[(int64_t)s * stride]; }
    BPK_HD Rat& mf(int s) const { return pF[(int64_t)s * stride]; }
    BPK_HD Rat& mb(int s) const { return pB[(int64_t)s * stride]; }
    BPK_HD Rat& dF(int s) const { return F[(int64_t)s * stride]; }
    BPK_HD Rat& dB(int s) const { return B[(int64_t)s * stride]; }
    BPK_HD int64_t& sr(int s) const { return SR[(int64_t)s * stride]; }
    BPK_HD int64_t& act(int s) const { return A[(int64_t)s * stride]; }
};

// Exact simulator body.  Positions are walked in order; at each position
// the F ops run in ascending stage order and the B ops in descending order
// (a topological order of the reference's sorted op list).  An arrival goes
// into the receiving stage's one-slot mailbox unless the receiver consumes it
// at the same position (a chain); the carry register defers the mailbox
// write until the receiver has read its own input, which is what keeps one
// slot sufficient (at most one arrival is outstanding per link direction).
BPK_HDNI void sim_exact(const BatchDev& B, int64_t ci, const SimState& S_in) {
    // a register copy: through the reference every access reloaded the
    // seven base pointers from local memory (the Rat calls may alias them)
    const SimState S = S_in;
    CState& cs = B.cs[ci];
    bp_candidate& cd = B.cand[ci];
    const int qi = B.cq[ci];
    const QDesc Q = B.q[qi];
    const int64_t local = ci - Q.cand_off;
    const int N = Q.N;
    const int kind = cd.kind;
    const int64_t M = cd.M, micro = cd.micro;
    NetView v = net_view(B.P, Q.net);
    ChainView c = chain_view(B.P, Q.cl, N);
    const int64_t slot = Q.stage_off + local * N;
    const int64_t qo = Q.qstage_off;
    const int32_t* hi = cs.plan_kind == PLAN_REFINED ? B.qhi + qo : B.chi + slot;
    Err e{ERR_NONE};
    // chain_instance (simulator.hpp:248-262): F, B per stage; SR per link.
    for (int s = 0; s < N; ++s) {
        if (cs.plan_kind == PLAN_REFINED) { S.dF(s) = B.qF[qo + s]; S.dB(s) = B.qB[qo + s]; }
        else {
            int32_t t = c.type[s];
            S.dF(s) = R(stage_sum_whole(B.clo[slot + s], B.chi[slot + s], v.Pfp + (int64_t)t * (v.L + 1)));
            S.dB(s) = R(stage_sum_whole(B.clo[slot + s], B.chi[slot + s], v.Pbp + (int64_t)t * (v.L + 1)));
        }
        S.act(s) = (s >= 1 ? v.a[hi[s - 1] - 1] : v.a[hi[0] - 1]) * micro;
        int64_t sr = 0;
        if (s + 1 < N) {
            int64_t a = v.a[hi[s] - 1] * micro;
            sr = a == 0 ? 0 : ceil_div64(a, c.bw[s]);
        }
        S.sr(s) = sr;
        S.f(s) = Rat{0, 1};
    }
    const bool async = kind_async(kind);
    for (int64_t p = 0; p < 2 * M && !e.bad(); ++p) {
        bool carry = false;
        int64_t cm = 0;
        Rat cv{0, 1};
        for (int s = 0; s < N; ++s) {             // F ops, ascending
            int64_t w = warmup_depth(kind, N, s + 1);
            if (w > M) w = M;
            StageOp op = op_at(p, w, M);
            bool chain = carry && op.is_f && op.m == cm;
            bool out = false;
            Rat ov{0, 1};
            if (op.is_f) {
                Rat ready = S.f(s);
                if (s > 0) {
                    Rat arr = chain ? cv : S.mf(s);
                    if (rat_gt(arr, ready)) ready = arr;
                }
                Rat end = rat_addsub_body(ready, S.dF(s), +1, e);
                S.f(s) = end;
                if (s + 1 < N) {
                    ov = async ? end : rat_addsub_body(end, R(S.sr(s)), +1, e);
                    out = true;
                }
            }
            if (carry && !chain) S.mf(s) = cv;    // deliver s-1's output to the mailbox
            carry = out;
            cm = op.m;
            cv = ov;
        }
        carry = false;
        for (int s = N - 1; s >= 0; --s) {        // B ops, descending
            int64_t w = warmup_depth(kind, N, s + 1);
            if (w > M) w = M;
            StageOp op = op_at(p, w, M);
            bool chain = carry && !op.is_f && op.m == cm;
            bool out = false;
            Rat ov{0, 1};
            if (!op.is_f) {
                Rat ready = S.f(s);   // >= endF(m, s): F(m, s) ran earlier on this stage
                if (s + 1 < N) {
                    Rat arr = chain ? cv : S.mb(s);
                    if (rat_gt(arr, ready)) ready = arr;
                }
                Rat end = rat_addsub_body(ready, S.dB(s), +1, e);
                S.f(s) = end;
                if (s > 0) {
                    ov = async ? end : rat_addsub_body(end, R(S.sr(s - 1)), +1, e);
                    out = true;
                }
            }
            if (carry && !chain) S.mb(s) = cv;
            carry = out;
            cm = op.m;
            cv = ov;
        }
    }
    if (e.bad()) { cs.sim_core = 2; fail(cd, e); return; }
    Rat mk{0, 1};
    for (int s = 0; s < N; ++s)
        if (rat_gt(S.f(s), mk)) mk = S.f(s);
    // feature high-water = min(M, depth) * a (simulator.hpp:219-238): the
    // in-flight count on a 1F1B stage peaks right after its warm-up.
    for (int s = 0; s < N; ++s) {
        int64_t w = warmup_depth(kind, N, s + 1);
        if (w > M) w = M;
        if ((i128)w * S.act(s) > (i128)INT64_MAX) { e.set(ERR_OVERFLOW); break; }
    }
    cs.sim_core = e.bad() ? 2 : 1;   // shared with asynchronous members (sim_copy)
    cs.sim_mk = mk;
    // link busy fraction Rat(M * SR) / makespan (239-244)
    for (int k = 0; k + 1 < N && !e.bad(); ++k)
        if (!rat_eq(mk, Rat{0, 1})) (void)rat_div(R(M * S.sr(k)), mk, e);
    if (e.bad()) { fail(cd, e); return; }
    cd.makespan = bp_rat{mk.n, mk.d};
    cd.status = BP_C_OK;
}

// ---------------------------------------------------------------- K5
BPK_HD bool cand_less(const bp_candidate& a, const bp_candidate& b) {   // explorer.hpp:142-152
    Rat am{a.makespan.num, a.makespan.den}, bm{b.makespan.num, b.makespan.den};
    if (!rat_eq(am, bm)) return rat_lt(am, bm);
    Rat ap{a.peak_memory.num, a.peak_memory.den}, bpm{b.peak_memory.num, b.peak_memory.den};
    if (!rat_eq(ap, bpm)) return rat_lt(ap, bpm);
    Rat aw{a.max_bw_demand.num, a.max_bw_demand.den}, bw{b.max_bw_demand.num, b.max_bw_demand.den};
    if (!rat_eq(aw, bw)) return rat_lt(aw, bw);
    if (a.M != b.M) return a.M < b.M;
    return a.kind < b.kind;
}

BPK_HD bool escaping(int st) {
    return st == BP_C_ERR_OVERFLOW || st == BP_C_ERR_INVALID_PLAN || st == BP_C_ERR_DOMAIN || st == BP_C_REF_UB;
}

BPK_HD int q_status_of(int st) {
    return st == BP_C_ERR_OVERFLOW ? BP_Q_OVERFLOW
           : st == BP_C_ERR_INVALID_PLAN ? BP_Q_INVALID_PLAN
           : st == BP_C_ERR_DOMAIN ? BP_Q_DOMAIN
                                    : BP_Q_REF_UB;
}

BPK_HDNI void rank_query(const BatchDev& B, int qi) {
    const QDesc Q = B.q[qi];
    bp_query_result& r = B.res[qi];
    if (!Q.schema_ok) return;
    int32_t* order = B.corder + Q.cand_off;
    const int nc = 2 * Q.nbase;
    bp_candidate* cand = B.cand + Q.cand_off;
    int nr = 0;
    int npruned = 0;
    for (int i = 0; i < nc; ++i) {
        int st = cand[i].status;
        if (st == BP_C_PRUNED_LB) {   // BP_OPT_PRUNE_LB: ranked, never first (its bound exceeds the best)
            cand[i].rank = -1;
            ++npruned;
            continue;
        }
        if (st != BP_C_OK) {
            // a candidate that failed after its estimate (simulate) carries
            // no values, like the reference's rejected/aborted candidates
            bp_candidate& cd = cand[i];
            cd.heuristic = 0;
            cd.plan_fractional = 0;
            cd.makespan = cd.est_minibatch = cd.bubble = cd.peak_memory = cd.max_bw_demand = bp_rat{0, 0};
            if (B.details && B.cs[Q.cand_off + i].sim_ready) {
                bp_stage* stg = B.stages + Q.stage_off + (int64_t)i * Q.N;
                for (int s = 0; s < Q.N; ++s) stg[s] = bp_stage{};
            }
        }
        if (escaping(st) && r.first_error < 0) {
            r.first_error = i;
            r.status = q_status_of(st);
        }
        if (st == BP_C_OK) {
            // stable insertion by the 5 keys
            int k = nr - 1;
            while (k >= 0 && cand_less(cand[i], cand[order[k]])) { order[k + 1] = order[k]; --k; }
            order[k + 1] = i;
            ++nr;
        }
    }
    if (r.first_error >= 0) return;
    if (nr == 0) { r.status = BP_Q_NO_FEASIBLE; return; }
    for (int i = 0; i < nr; ++i) cand[order[i]].rank = i;
    const bp_candidate& b = cand[order[0]];
    r.status = BP_Q_OK;
    r.n_ranked = nr + npruned;
    r.best = order[0];
    r.best_kind = b.kind;
    r.best_M = b.M;
    r.best_micro = b.micro;
    r.best_makespan = b.makespan;
    r.best_peak_memory = b.peak_memory;
    r.best_max_bw = b.max_bw_demand;
}

}  // namespace bpk
