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

int main() {
    for (const Scenario& s : scenarios()) {
        std::cout << run_one(s, [](const auto& n, const auto& c, const auto& g) { return api::explore(n, c, g); });
        std::cout << one_plan_checks(s);
    }
    return 0;
}
