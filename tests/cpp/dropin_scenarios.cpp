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
namespace api = bapipe;
#else
#include "bapipe_b200/explorer.hpp"
namespace api = bapipe_b200;
#endif

#include "scenarios.inc"

int main() {
    for (const Scenario& s : scenarios())
        std::cout << run_one(s, [](const auto& n, const auto& c, const auto& g) { return api::explore(n, c, g); });
    return 0;
}
