// bapipe_b200/interop.hpp -- call the B200 explorer with the REFERENCE's own
// types, for code that keeps using the reference headers for everything else
// (JSON I/O, reports, the CLI).  Duck-typed templates: this header does not
// include the reference; it copies the fields the two APIs share by name
// (profiles.hpp:24-78, plan.hpp:16-28, cost_models.hpp:26-44,
// explorer.hpp:51-76) and maps the enums by value (schedule_kind.hpp:11-16
// declares them in the same order as bapipe_b200).
//
//   // tools/bapipe.cpp:219, the one line a maintainer changes:
//   ExplorationResult res = bapipe_b200::explore_as<bapipe::ExplorationResult,
//       bapipe::NoFeasiblePlan, bapipe::InvalidPlan, bapipe::SchemaError>(net, cluster, cfg);
//
// Exceptions are re-thrown as the reference's types with the reference's
// messages, so the CLI's exit-code mapping (tools/bapipe.cpp:257-269) holds.
#pragma once

#include <string>
#include <utility>

#include "explorer.hpp"

namespace bapipe_b200 {
namespace interop {

template <class RefNet>
NetworkProfile network(const RefNet& n) {
    NetworkProfile out;
    out.name = n.name;
    out.layers.reserve(n.layers.size());
    for (const auto& l : n.layers) {
        LayerProfile x;
        x.name = l.name;
        x.fp_time.insert(l.fp_time.begin(), l.fp_time.end());
        x.bp_time.insert(l.bp_time.begin(), l.bp_time.end());
        x.weight_bytes = l.weight_bytes;
        x.out_activation_bytes = l.out_activation_bytes;
        out.layers.push_back(std::move(x));
    }
    return out;
}

template <class RefCluster>
ClusterSpec cluster(const RefCluster& c) {
    ClusterSpec out;
    for (const auto& a : c.accelerators) {
        AcceleratorSpec x;
        x.id = a.id;
        x.accel_type = a.accel_type;
        x.mem_capacity_bytes = a.mem_capacity_bytes;
        for (const auto& [k, v] : a.min_micro_batch) x.min_micro_batch[(ScheduleKind)(int)k] = v;
        out.accelerators.push_back(std::move(x));
    }
    out.link_bandwidth.assign(c.link_bandwidth.begin(), c.link_bandwidth.end());
    out.execution_mode = (ExecutionMode)(int)c.execution_mode;
    return out;
}

template <class RefCfg>
TrainingConfig config(const RefCfg& c) {
    TrainingConfig out;
    out.mini_batch_size = c.mini_batch_size;
    if (c.micro_batch_candidates)
        out.micro_batch_candidates.emplace(c.micro_batch_candidates->begin(), c.micro_batch_candidates->end());
    return out;
}

// Reference Rat from an already-reduced value (Rat(n, d) re-normalises: no-op).
template <class RefRat>
RefRat rat(const Rat& r) {
    return RefRat(r.num(), r.den());
}

template <class RefCandidate>
RefCandidate candidate(const Candidate& c) {
    using RefRat = decltype(RefCandidate{}.simulated_makespan);
    using RefKind = decltype(RefCandidate{}.kind);
    RefCandidate out;
    out.kind = (RefKind)(int)c.kind;
    out.M = c.M;
    out.micro_batch_size = c.micro_batch_size;
    for (const StageAssignment& s : c.plan.stages) {
        typename decltype(out.plan.stages)::value_type x;
        x.accelerator_id = s.accelerator_id;
        x.lo = s.lo;
        x.hi = s.hi;
        x.leading_fraction = rat<RefRat>(s.leading_fraction);
        x.trailing_fraction = rat<RefRat>(s.trailing_fraction);
        out.plan.stages.push_back(std::move(x));
    }
    out.simulated_makespan = rat<RefRat>(c.simulated_makespan);
    out.est.schedule = (RefKind)(int)c.est.schedule;
    out.est.M = c.est.M;
    out.est.N = c.est.N;
    out.est.minibatch_time = rat<RefRat>(c.est.minibatch_time);
    out.est.bubble_fraction = rat<RefRat>(c.est.bubble_fraction);
    for (const Rat& r : c.est.features_mem) out.est.features_mem.push_back(rat<RefRat>(r));
    for (const Rat& r : c.est.weights_mem) out.est.weights_mem.push_back(rat<RefRat>(r));
    for (const Rat& r : c.est.bandwidth_demand) out.est.bandwidth_demand.push_back(rat<RefRat>(r));
    out.est.mem_infeasible.assign(c.est.mem_infeasible.begin(), c.est.mem_infeasible.end());
    out.est.heuristic = c.est.heuristic;
    out.peak_memory = rat<RefRat>(c.peak_memory);
    out.max_bandwidth_demand = rat<RefRat>(c.max_bandwidth_demand);
    return out;
}

template <class RefResult>
RefResult result(const ExplorationResult& r) {
    using RefCandidate = decltype(RefResult{}.best);
    using RefKind = decltype(RefCandidate{}.kind);
    RefResult out;
    out.best = candidate<RefCandidate>(r.best);
    for (const Candidate& c : r.ranked) out.ranked.push_back(candidate<RefCandidate>(c));
    for (const Rejection& j : r.rejected) {
        typename decltype(out.rejected)::value_type x;
        x.kind = (RefKind)(int)j.kind;
        x.M = j.M;
        x.reason = j.reason;
        x.detail = j.detail;
        out.rejected.push_back(std::move(x));
    }
    out.mini_batch_size = r.mini_batch_size;
    out.dp_baseline_minibatch_time = r.dp_baseline_minibatch_time;
    return out;
}

// what() minus our prefix: the reference constructors add their own.
inline std::string strip(const char* what, const char* prefix) {
    std::string s(what), p(prefix);
    return s.compare(0, p.size(), p) == 0 ? s.substr(p.size()) : s;
}

}  // namespace interop

// explore() with the reference's input and result types.
template <class RefResult, class RefNoFeasiblePlan, class RefInvalidPlan, class RefSchemaError, class RefNet,
          class RefCluster, class RefCfg>
RefResult explore_as(const RefNet& net, const RefCluster& cl, const RefCfg& cfg) {
    try {
        return interop::result<RefResult>(explore(interop::network(net), interop::cluster(cl), interop::config(cfg)));
    } catch (const NoFeasiblePlan& e) {
        throw RefNoFeasiblePlan(interop::strip(e.what(), "no feasible plan: "));
    } catch (const InvalidPlan& e) {
        throw RefInvalidPlan(interop::strip(e.what(), "invalid plan: "));
    } catch (const SchemaError& e) {
        throw RefSchemaError(interop::strip(e.what(), "schema error: "));
    }
}

}  // namespace bapipe_b200
