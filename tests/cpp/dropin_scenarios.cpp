// dropin_scenarios.cpp -- one source, two builds:
//   -DUSE_REFERENCE  against the reference headers (/root/reference/proj/include),
//                    run in the dev container to produce tests/golden/dropin_expected.txt
//   (default)        against include/bapipe_b200/explorer.hpp + libbapipe_b200.so,
//                    run on the B200 by tests/test_dropin.py and diffed with the golden.
// The scenarios and the dump format are in scenarios.inc.
#include <cstdint>
#include <cstdio>
#include <iostream>
#include <sstream>
#include <string>
#include <vector>

#ifdef USE_REFERENCE
#include "bapipe/explorer.hpp"
#include "bapipe/gantt.hpp"
namespace api = bapipe;
#else
#include "bapipe_b200/explorer.hpp"
#include "bapipe_b200/gantt.hpp"
namespace api = bapipe_b200;
#endif

#include "scenarios.inc"

// For every ranked candidate of a scenario: balance_partition for its (kind,
// M, micro), estimate on that plan and the full-timeline simulate, as the
// reference's `bapipe plan` / `bapipe simulate` call them (SURVEY.md 8f F2,
// F3).  The timeline is printed as its event count and an FNV-1a digest of its
// gantt_csv text, with makespan, high-water marks and busy fractions.
std::string one_plan_checks(const Scenario& s) {
    std::ostringstream os;
    api::ExplorationResult r;
    try {
        r = api::explore(s.net, s.cl, s.cfg);
    } catch (const std::exception&) {
        return "";
    }
    for (const auto& c : r.ranked) {
        os << "plan " << api::to_string(c.kind) << " M=" << c.M << " micro=" << c.micro_batch_size << ":";
        try {
            api::PartitionPlan p = api::balance_partition(s.net, s.cl, c.kind, c.M, c.micro_batch_size);
            for (const auto& st : p.stages)
                os << " [" << st.lo << "," << st.hi << " " << st.leading_fraction.str() << " "
                   << st.trailing_fraction.str() << "]";
            api::CostEstimate e = api::estimate(c.kind, p, s.net, s.cl, c.M, c.micro_batch_size);
            os << " est " << e.minibatch_time.str() << " " << e.bubble_fraction.str() << " h" << e.heuristic
               << " feasible" << e.memory_feasible();
            api::Timeline t = api::simulate(c.kind, p, s.net, s.cl, c.M, c.micro_batch_size);
            const std::string csv = api::gantt_csv(t);
            std::uint64_t h = 0xcbf29ce484222325ull;
            for (unsigned char ch : csv) h = (h ^ ch) * 0x100000001b3ull;
            os << " sim " << t.makespan.str() << " events " << t.events.size() << " digest " << std::hex << h
               << std::dec << " hw";
            for (const auto& x : t.per_stage_feature_highwater) os << " " << x.str();
            os << " busy";
            for (const auto& x : t.per_link_busy_fraction) os << " " << x.str();
        } catch (const std::exception& e) {
            os << " EXC " << e.what();
        }
        os << "\n";
    }
    return os.str();
}

// estimate / simulate on caller-given plans at their edges: a plan stage over
// a layer without a time for its accelerator type (SchemaError from
// LayerProfile::at, profiles.hpp:38-43, after check_mode / validate_plan /
// the stage count), an invalid plan that also misses a type (InvalidPlan
// first, simulator.hpp:268-273), and mini_batches < 1 (no events, makespan
// Rat(mini_batches) * makespan, simulator.hpp:182-216).
std::string edge_plan_checks() {
    std::ostringstream os;
    auto plan_of = [](std::vector<std::pair<std::int64_t, std::int64_t>> r) {
        api::PartitionPlan p;
        for (size_t i = 0; i < r.size(); ++i) {
            api::StageAssignment st;
            st.accelerator_id = "g" + std::to_string(i);
            st.lo = r[i].first;
            st.hi = r[i].second;
            p.stages.push_back(st);
        }
        return p;
    };
    auto run = [&](const std::string& name, auto&& f) {
        os << "== edge " << name << ":";
        try {
            os << " " << f();
        } catch (const api::SchemaError& e) {
            os << " EXC SchemaError " << e.what();
        } catch (const api::InvalidPlan& e) {
            os << " EXC InvalidPlan " << e.what();
        } catch (const std::exception& e) {
            os << " EXC " << e.what();
        }
        os << "\n";
    };
    const auto K = api::ScheduleKind::OneFOneB_SNO;
    api::NetworkProfile net = tri_net();
    net.layers[1].fp_time.erase("gpu");
    const ClusterSpec cl = tri_cluster(ExecutionMode::Synchronous, {1000000, 1000000, 1000000});
    const api::PartitionPlan whole = plan_of({{1, 1}, {2, 2}, {3, 3}});
    auto est_str = [&](const api::NetworkProfile& n, const ClusterSpec& c, const api::PartitionPlan& p) {
        api::CostEstimate e = api::estimate(K, p, n, c, 4, 1);
        return "est " + e.minibatch_time.str() + " " + e.bubble_fraction.str();
    };
    auto sim_str = [&](const api::NetworkProfile& n, const ClusterSpec& c, const api::PartitionPlan& p,
                       std::int64_t mb) {
        api::Timeline t = api::simulate(K, p, n, c, 4, 1, mb);
        std::string r = "sim " + t.makespan.str() + " events " + std::to_string(t.events.size()) + " hw";
        for (const auto& x : t.per_stage_feature_highwater) r += " " + x.str();
        r += " busy";
        for (const auto& x : t.per_link_busy_fraction) r += " " + x.str();
        return r;
    };
    run("estimate missing fp type", [&] { return est_str(net, cl, whole); });
    run("simulate missing fp type", [&] { return sim_str(net, cl, whole, 1); });
    {
        api::NetworkProfile n2 = tri_net();
        n2.layers[2].bp_time.erase("gpu");
        run("estimate missing bp type", [&] { return est_str(n2, cl, whole); });
    }
    {
        ClusterSpec c2 = cl;
        c2.accelerators[1].accel_type = "tpu";
        run("estimate stage type absent", [&] { return est_str(tri_net(), c2, whole); });
        run("simulate stage type absent", [&] { return sim_str(tri_net(), c2, whole, 1); });
    }
    run("simulate invalid plan and missing type", [&] { return sim_str(net, cl, plan_of({{1, 1}, {3, 3}, {3, 3}}), 1); });
    run("simulate mini_batches 0", [&] { return sim_str(tri_net(), cl, whole, 0); });
    run("simulate mini_batches -2", [&] { return sim_str(tri_net(), cl, whole, -2); });
    run("simulate mini_batches 3", [&] { return sim_str(tri_net(), cl, whole, 3); });
    return os.str();
}

int main() {
    for (const Scenario& s : scenarios()) {
        std::cout << run_one(s, [](const auto& n, const auto& c, const auto& g) { return api::explore(n, c, g); });
        std::cout << one_plan_checks(s);
    }
    std::cout << edge_plan_checks();
    return 0;
}
