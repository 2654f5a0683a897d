// interop_check.cpp -- include/bapipe_b200/interop.hpp against the reference
// headers themselves: every scenario of scenarios.inc is built with the
// REFERENCE's types, explored once by bapipe::explore and once by
// bapipe_b200::explore_as (reference types in and out, B200 explorer inside),
// and the two canonical dumps must be identical.  Needs /root/reference
// (dev container); linked with emu_abi_shim.cpp on the CPU or with
// libbapipe_b200.so on a B200.
#include <cstdint>
#include <cstdio>
#include <iostream>
#include <sstream>
#include <string>
#include <vector>

#include "bapipe/explorer.hpp"
#include "bapipe_b200/interop.hpp"
namespace api = bapipe;

#include "scenarios.inc"

int main() {
    int bad = 0, n = 0;
    for (const Scenario& s : scenarios()) {
        const std::string want =
            run_one(s, [](const auto& a, const auto& b, const auto& c) { return bapipe::explore(a, b, c); });
        const std::string got = run_one(s, [](const auto& a, const auto& b, const auto& c) {
            return bapipe_b200::explore_as<bapipe::ExplorationResult, bapipe::NoFeasiblePlan, bapipe::InvalidPlan,
                                           bapipe::SchemaError>(a, b, c);
        });
        ++n;
        if (got != want) {
            ++bad;
            std::cout << "MISMATCH\n--- reference\n" << want << "--- b200\n" << got;
        }
    }
    std::cout << n << " scenarios, " << bad << " mismatches\n";
    return bad ? 1 : 0;
}
