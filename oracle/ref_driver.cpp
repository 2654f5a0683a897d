// oracle/ref_driver.cpp -- TEST INFRASTRUCTURE ONLY (never on the product path).
//
// Builds the UNMODIFIED reference headers (/root/reference/proj/include/bapipe,
// compiled where they lie by oracle/Makefile) into oracle/_ref/libbapipe_ref.so
// behind the same SoA structs as include/bapipe_b200.h, so that tests, smoke()
// and bench.py's reference arm can run the reference's own explore() on exactly
// the inputs the CUDA path sees.
//
// Two entry points:
//   bpref_explore_batch  -- parity mode.  Calls bapipe::explore()
//       (explorer.hpp:80-155) per query for the query-level outcome and the
//       ranking, then replays explorer.hpp:96-132 per (kind, M) candidate
//       through the public balance_partition / estimate / simulate calls, each
//       candidate wrapped separately so one overflow does not hide the rest
//       (SURVEY.md 8c "parity harness design").
//   bpref_explore_timed  -- timing mode.  Only bapipe::explore() per query,
//       on a std::thread pool (one worker per requested thread).
//
// Undefined behaviour: the library is compiled with
// -D_GLIBCXX_ASSERTIONS so the out-of-bounds net.layers[-1] read that
// memory_fine_tune's collapse step can trigger (partition.hpp:359-373 ->
// plan.hpp:136-139) lands in std::__glibcxx_assert_fail, which we interpose
// and longjmp out of; the candidate/query is reported as REF_UB.
#include <atomic>
#include <csetjmp>
#include <cstdio>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "bapipe/explorer.hpp"
#include "bapipe_b200.h"

using namespace bapipe;

static thread_local jmp_buf* g_ub_jump = nullptr;

namespace std {
// Interposes libstdc++'s assertion handler (c++config.h) for bounds checks.
void __glibcxx_assert_fail(const char*, int, const char*, const char*) noexcept {
    if (g_ub_jump) longjmp(*g_ub_jump, 1);
    std::fprintf(stderr, "bapipe_ref: libstdc++ assertion outside a guarded region\n");
    std::abort();
}
}  // namespace std

namespace {

NetworkProfile to_network(const bp_network& n) {
    NetworkProfile net;
    net.name = "net";
    for (int j = 0; j < n.n_layers; ++j) {
        LayerProfile l;
        l.name = "l" + std::to_string(j);
        for (int t = 0; t < n.n_types; ++t) {
            int64_t f = n.fp_us[(size_t)t * n.n_layers + j];
            int64_t b = n.bp_us[(size_t)t * n.n_layers + j];
            if (f != 0) l.fp_time["t" + std::to_string(t)] = f;
            if (b != 0) l.bp_time["t" + std::to_string(t)] = b;
        }
        l.weight_bytes = n.weight_bytes[j];
        l.out_activation_bytes = n.out_act_bytes[j];
        net.layers.push_back(std::move(l));
    }
    return net;
}

ClusterSpec to_cluster(const bp_cluster& c, int n_stages) {
    ClusterSpec cl;
    cl.execution_mode =
        c.exec_mode == BP_MODE_ASYNC ? ExecutionMode::Asynchronous : ExecutionMode::Synchronous;
    int N = n_stages > 0 ? n_stages : c.n_accels;
    for (int k = 0; k < N; ++k) {
        AcceleratorSpec a;
        a.id = "d" + std::to_string(k);
        a.accel_type = "t" + std::to_string(c.type_id[k]);
        a.mem_capacity_bytes = c.mem_capacity[k];
        for (int kind = 0; kind < 4; ++kind)
            a.min_micro_batch[all_schedule_kinds[kind]] = c.min_micro[(size_t)k * 4 + kind];
        cl.accelerators.push_back(std::move(a));
    }
    for (int k = 0; k + 1 < N; ++k) cl.link_bandwidth.push_back(c.link_bw[k]);
    return cl;
}

TrainingConfig to_config(const bp_query& q) {
    TrainingConfig cfg;
    cfg.mini_batch_size = q.mini_batch;
    if (q.n_m > 0 && q.m_list) cfg.micro_batch_candidates = std::vector<int64_t>(q.m_list, q.m_list + q.n_m);
    return cfg;
}

bp_rat R(const Rat& r) { return bp_rat{r.num(), r.den()}; }

std::vector<int64_t> base_list(const TrainingConfig& cfg) {
    std::vector<int64_t> base;
    if (cfg.micro_batch_candidates) return *cfg.micro_batch_candidates;
    for (int64_t m = 1; m <= cfg.mini_batch_size; ++m)
        if (cfg.mini_batch_size % m == 0) base.push_back(m);
    return base;
}

int64_t parse_after(const std::string& s, const char* key) {
    auto p = s.find(key);
    if (p == std::string::npos) return -1;
    return std::atoll(s.c_str() + p + std::strlen(key));
}

// InvalidPlan message -> (code, index, aux) following plan.hpp:42-83.
void classify_invalid(const std::string& m, bp_candidate& c) {
    c.status = BP_C_ERR_INVALID_PLAN;
    c.detail2 = parse_after(m, "stage ");
    if (m.find("out of bounds") != std::string::npos) c.detail = BP_IP_RANGE;
    else if (m.find("fractions must lie") != std::string::npos) c.detail = BP_IP_FRACTION;
    else if (m.find("stage 1 must start") != std::string::npos) { c.detail = BP_IP_FIRST; c.detail2 = 1; }
    else if (m.find("not contiguous") != std::string::npos) c.detail = BP_IP_CONTIG;
    else if (m.find("must be fractional") != std::string::npos) c.detail = BP_IP_SHARED_FULL;
    else if (m.find("fractional lead") != std::string::npos) c.detail = BP_IP_LEAD_UNSHARED;
    else if (m.find("last stage must end") != std::string::npos) { c.detail = BP_IP_LAST; c.detail2 = 0; }
    else if (m.find("coverage sums to") != std::string::npos) {
        c.detail = BP_IP_COVERAGE;
        c.detail2 = parse_after(m, "layer ");
        auto p = m.find("sums to ") + 8;
        auto e = m.find(',', p);
        c.aux = R(rat_from_string(m.substr(p, e - p)));
    } else if (m.find("stage count != cluster size") != std::string::npos) {
        c.detail = BP_IP_STAGE_COUNT;
        c.detail2 = 0;
    } else if (m.find("M >= 1 required") != std::string::npos) {
        c.detail = BP_IP_M;
        c.detail2 = 0;
    } else c.detail = 0;
}

PartitionPlan to_plan(const bp_plan_request& q) {
    PartitionPlan p;
    for (int s = 0; s < q.n_stages; ++s)
        p.stages.push_back({"d" + std::to_string(s), q.lo[s], q.hi[s], Rat(q.lead[s].num, q.lead[s].den),
                            Rat(q.trail[s].num, q.trail[s].den)});
    return p;
}

// outcome of a reference call on one plan, as the ABI status codes
template <class F>
int32_t run_plan_call(F&& f, bp_candidate& c) {
    try {
        f();
        return BP_C_OK;
    } catch (const InvalidPlan& e) {
        classify_invalid(e.what(), c);
        return BP_C_ERR_INVALID_PLAN;
    } catch (const std::overflow_error&) {
        return BP_C_ERR_OVERFLOW;
    } catch (const std::domain_error&) {
        return BP_C_ERR_DOMAIN;
    }
}

struct QueryCtx {
    const bp_network* nets;
    const bp_cluster* cls;
};

// One explore() call; classifies its outcome.  Returns the result when OK.
int run_explore(const NetworkProfile& net, const ClusterSpec& cl, const TrainingConfig& cfg,
                ExplorationResult* out) {
    jmp_buf jb;
    g_ub_jump = &jb;
    if (setjmp(jb)) { g_ub_jump = nullptr; return BP_Q_REF_UB; }
    int st = BP_Q_OK;
    try {
        *out = explore(net, cl, cfg);
    } catch (const NoFeasiblePlan&) { st = BP_Q_NO_FEASIBLE; }
    catch (const SchemaError&) { st = BP_Q_SCHEMA; }
    catch (const InvalidPlan&) { st = BP_Q_INVALID_PLAN; }
    catch (const std::overflow_error&) { st = BP_Q_OVERFLOW; }
    catch (const std::domain_error&) { st = BP_Q_DOMAIN; }
    g_ub_jump = nullptr;
    return st;
}

// explorer.hpp:104-131 for one candidate, wrapped on its own.
void replay_candidate(const NetworkProfile& net, const ClusterSpec& cl, ScheduleKind kind,
                      int64_t M, int64_t micro, bp_candidate& c, bp_stage* st) {
    jmp_buf jb;
    g_ub_jump = &jb;
    if (setjmp(jb)) { g_ub_jump = nullptr; c.status = BP_C_REF_UB; return; }
    try {
        PartitionPlan plan;
        try {
            plan = balance_partition(net, cl, kind, M, micro);
        } catch (const Infeasible& e) {
            std::string m = e.what();
            if (m.find("coarsening") != std::string::npos) {
                c.status = BP_C_REJ_COARSEN;
                c.detail = parse_after(m, "leaves ");
            } else if (m.find("did not converge") != std::string::npos) {
                c.status = BP_C_REJ_FINETUNE_NOCONV;
            } else {
                c.status = BP_C_REJ_FINETUNE;
            }
            g_ub_jump = nullptr;
            return;
        } catch (const InfeasibleShape& e) {
            c.status = BP_C_REJ_SHAPE;
            c.detail = parse_after(std::string(e.what()), "shape: ");
            g_ub_jump = nullptr;
            return;
        }
        CostEstimate est = estimate(kind, plan, net, cl, M, micro);
        if (!est.memory_feasible()) {
            c.status = BP_C_REJ_MEM_POST;
            g_ub_jump = nullptr;
            return;
        }
        Timeline t = simulate(kind, plan, net, cl, M, micro);
        Rat peak(0), maxbw(0);
        for (int64_t i = 0; i < plan.n_stages(); ++i) {
            Rat mem = est.features_mem[i] + est.weights_mem[i];
            if (mem > peak) peak = mem;
        }
        for (const Rat& d : est.bandwidth_demand)
            if (d > maxbw) maxbw = d;
        c.status = BP_C_OK;
        c.makespan = R(t.makespan);
        c.est_minibatch = R(est.minibatch_time);
        c.bubble = R(est.bubble_fraction);
        c.peak_memory = R(peak);
        c.max_bw_demand = R(maxbw);
        c.heuristic = est.heuristic ? 1 : 0;
        c.n_stages = (int32_t)plan.n_stages();
        c.plan_fractional = 0;
        for (int64_t i = 0; i < plan.n_stages(); ++i) {
            const StageAssignment& s = plan.stages[i];
            if (s.leading_fraction != Rat(1) || s.trailing_fraction != Rat(1)) c.plan_fractional = 1;
            if (!st) continue;
            st[i].lo = s.lo;
            st[i].hi = s.hi;
            st[i].lead = R(s.leading_fraction);
            st[i].trail = R(s.trailing_fraction);
            st[i].features = R(est.features_mem[i]);
            st[i].weights = R(est.weights_mem[i]);
            st[i].bw_demand = i + 1 < plan.n_stages() ? R(est.bandwidth_demand[i]) : bp_rat{0, 1};
        }
    } catch (const InvalidPlan& e) {
        classify_invalid(e.what(), c);
    } catch (const std::overflow_error&) {
        c.status = BP_C_ERR_OVERFLOW;
    } catch (const std::domain_error&) {
        c.status = BP_C_ERR_DOMAIN;
    }
    g_ub_jump = nullptr;
}

void one_query(const QueryCtx& qc, const bp_query& q, bp_query_result& r, bp_candidate* cand,
               bp_stage* stages) {
    std::memset(&r, 0, sizeof(r));
    r.best = -1;
    r.first_error = -1;
    NetworkProfile net = to_network(qc.nets[q.network]);
    ClusterSpec cl = to_cluster(qc.cls[q.cluster], q.n_stages);
    TrainingConfig cfg = to_config(q);
    ExplorationResult res;
    r.status = run_explore(net, cl, cfg, &res);
    std::vector<int64_t> base = base_list(cfg);
    auto kinds = feasible_kinds(cl.execution_mode);
    r.n_candidates = (int32_t)(kinds.size() * base.size());
    if (r.status == BP_Q_SCHEMA) { r.n_candidates = 0; return; }
    int64_t N = cl.N();
    if (cand) {
        for (size_t ki = 0; ki < kinds.size(); ++ki) {
            std::vector<int64_t> allowed = candidate_Ms(cfg, cl, kinds[ki]);
            for (size_t mi = 0; mi < base.size(); ++mi) {
                size_t idx = ki * base.size() + mi;
                bp_candidate& c = cand[q.cand_offset + idx];
                std::memset(&c, 0, sizeof(c));
                c.kind = (int32_t)kinds[ki];
                c.M = base[mi];
                c.micro = cfg.mini_batch_size / c.M;
                c.rank = -1;
                c.n_stages = (int32_t)N;
                if (std::find(allowed.begin(), allowed.end(), c.M) == allowed.end()) {
                    c.status = BP_C_REJ_MIN_MICRO;
                    continue;
                }
                replay_candidate(net, cl, kinds[ki], c.M, c.micro, c,
                                 stages ? stages + q.stage_offset + (int64_t)idx * N : nullptr);
                if (r.first_error < 0 && (c.status == BP_C_ERR_OVERFLOW ||
                                          c.status == BP_C_ERR_INVALID_PLAN ||
                                          c.status == BP_C_ERR_DOMAIN || c.status == BP_C_REF_UB))
                    r.first_error = (int32_t)idx;
            }
        }
    }
    if (r.status != BP_Q_OK) return;
    r.n_ranked = (int32_t)res.ranked.size();
    // Map ranked candidates back to candidate indices by (kind, M, occurrence).
    std::vector<int> used(r.n_candidates, 0);
    for (size_t rk = 0; rk < res.ranked.size(); ++rk) {
        const Candidate& c = res.ranked[rk];
        int found = -1;
        for (size_t ki = 0; ki < kinds.size() && found < 0; ++ki) {
            if (kinds[ki] != c.kind) continue;
            for (size_t mi = 0; mi < base.size(); ++mi) {
                size_t idx = ki * base.size() + mi;
                if (base[mi] == c.M && !used[idx]) { found = (int)idx; break; }
            }
        }
        if (found < 0) continue;
        used[found] = 1;
        if (cand) cand[q.cand_offset + found].rank = (int32_t)rk;
        if (rk == 0) r.best = found;
    }
    r.best_kind = (int32_t)res.best.kind;
    r.best_M = res.best.M;
    r.best_micro = res.best.micro_batch_size;
    r.best_makespan = R(res.best.simulated_makespan);
    r.best_peak_memory = R(res.best.peak_memory);
    r.best_max_bw = R(res.best.max_bandwidth_demand);
}

}  // namespace

extern "C" {

int bpref_abi_version(void) { return BP_ABI_VERSION; }

int bpref_explore_batch(const bp_network* nets, int n_nets, const bp_cluster* cls, int n_cls,
                        const bp_query* q, int nq, bp_query_result* res, bp_candidate* cand,
                        bp_stage* stages, int threads) {
    if (!nets || !cls || !q || !res || n_nets < 1 || n_cls < 1) return BP_BAD_INPUT;
    QueryCtx qc{nets, cls};
    if (threads <= 1) {
        for (int i = 0; i < nq; ++i) one_query(qc, q[i], res[i], cand, stages);
        return BP_OK;
    }
    std::atomic<int> next{0};
    std::vector<std::thread> pool;
    for (int t = 0; t < threads; ++t)
        pool.emplace_back([&] {
            for (int i; (i = next.fetch_add(1)) < nq;) one_query(qc, q[i], res[i], cand, stages);
        });
    for (auto& th : pool) th.join();
    return BP_OK;
}

// Timing mode: the reference's public explore() only, per query.
int bpref_explore_timed(const bp_network* nets, int n_nets, const bp_cluster* cls, int n_cls,
                        const bp_query* q, int nq, bp_query_result* res, int threads) {
    if (!nets || !cls || !q || !res || n_nets < 1 || n_cls < 1) return BP_BAD_INPUT;
    // Convert inputs up front (the reference API takes value types).
    std::vector<NetworkProfile> N(n_nets);
    for (int i = 0; i < n_nets; ++i) N[i] = to_network(nets[i]);
    std::atomic<int> next{0};
    auto work = [&] {
        for (int i; (i = next.fetch_add(1)) < nq;) {
            ClusterSpec cl = to_cluster(cls[q[i].cluster], q[i].n_stages);
            TrainingConfig cfg = to_config(q[i]);
            ExplorationResult er;
            bp_query_result& r = res[i];
            std::memset(&r, 0, sizeof(r));
            r.best = -1;
            r.first_error = -1;
            r.status = run_explore(N[q[i].network], cl, cfg, &er);
            if (r.status == BP_Q_OK) {
                r.n_ranked = (int32_t)er.ranked.size();
                r.n_candidates = (int32_t)(er.ranked.size() + er.rejected.size());
                r.best_kind = (int32_t)er.best.kind;
                r.best_M = er.best.M;
                r.best_micro = er.best.micro_batch_size;
                r.best_makespan = R(er.best.simulated_makespan);
                r.best_peak_memory = R(er.best.peak_memory);
                r.best_max_bw = R(er.best.max_bandwidth_demand);
            }
        }
    };
    if (threads <= 1) work();
    else {
        std::vector<std::thread> pool;
        for (int t = 0; t < threads; ++t) pool.emplace_back(work);
        for (auto& th : pool) th.join();
    }
    return BP_OK;
}

// simulate() / estimate() of one plan (simulator.hpp:264-274,
// cost_models.hpp:124-166): the reference side of bp_simulate_plan /
// bp_estimate_plan.  The caller guarantees a mode-compatible kind.
int bpref_simulate_plan(const bp_network* nets, int, const bp_cluster* cls, int, const bp_plan_request* q,
                        bp_timeline_result* res, bp_event* ev, int64_t cap, bp_rat* hw, bp_rat* ws, bp_rat* busy) {
    NetworkProfile net = to_network(nets[q->network]);
    ClusterSpec cl = to_cluster(cls[q->cluster], 0);
    PartitionPlan plan = to_plan(*q);
    Timeline t;
    bp_candidate c{};
    std::memset(res, 0, sizeof(*res));
    res->status = run_plan_call(
        [&] { t = simulate((ScheduleKind)q->kind, plan, net, cl, q->M, q->micro, q->mini_batches); }, c);
    if (res->status == BP_C_ERR_INVALID_PLAN) {
        res->detail = c.detail;
        res->detail2 = c.detail2;
        res->aux = c.aux;
    }
    if (res->status != BP_C_OK) return BP_OK;
    res->makespan = R(t.makespan);
    res->n_events = (int64_t)t.events.size();
    for (int64_t i = 0; i < res->n_events && i < cap; ++i) {
        const Event& e = t.events[(size_t)i];
        ev[i] = bp_event{e.stage, (int32_t)e.kind, 0, e.micro_batch, R(e.start), R(e.end)};
    }
    for (size_t s = 0; s < t.per_stage_feature_highwater.size(); ++s) {
        hw[s] = R(t.per_stage_feature_highwater[s]);
        ws[s] = R(t.per_stage_weight_static[s]);
    }
    for (size_t k = 0; k < t.per_link_busy_fraction.size(); ++k) busy[k] = R(t.per_link_busy_fraction[k]);
    return BP_OK;
}

int bpref_estimate_plan(const bp_network* nets, int, const bp_cluster* cls, int, const bp_plan_request* q,
                        bp_estimate_result* res, bp_stage* st, int32_t* inf) {
    NetworkProfile net = to_network(nets[q->network]);
    ClusterSpec cl = to_cluster(cls[q->cluster], 0);
    PartitionPlan plan = to_plan(*q);
    CostEstimate e;
    bp_candidate c{};
    std::memset(res, 0, sizeof(*res));
    res->status = run_plan_call([&] { e = estimate((ScheduleKind)q->kind, plan, net, cl, q->M, q->micro); }, c);
    if (res->status != BP_C_OK) return BP_OK;
    res->heuristic = e.heuristic ? 1 : 0;
    res->minibatch_time = R(e.minibatch_time);
    res->bubble_fraction = R(e.bubble_fraction);
    for (int s = 0; s < q->n_stages; ++s) {
        st[s] = bp_stage{};
        st[s].lo = q->lo[s];
        st[s].hi = q->hi[s];
        st[s].lead = q->lead[s];
        st[s].trail = q->trail[s];
        st[s].features = R(e.features_mem[(size_t)s]);
        st[s].weights = R(e.weights_mem[(size_t)s]);
        st[s].bw_demand = s + 1 < q->n_stages ? R(e.bandwidth_demand[(size_t)s]) : bp_rat{0, 1};
        inf[s] = e.mem_infeasible[(size_t)s] ? 1 : 0;
    }
    return BP_OK;
}

}  // extern "C"
