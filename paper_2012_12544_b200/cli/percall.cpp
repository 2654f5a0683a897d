// percall -- per-call latency of explore() on single queries (bench.py's
// per_call block; BASELINE.md's CPU plan: C1-C3 with >= 20 repetitions, C4
// in its variants).
//
//   percall [--threads T] REPS MINI NET.json CLUSTER.json [MINI NET CLUSTER ...]
//
// Each case is one (network, cluster, mini-batch): two warm-up calls, then
// REPS timed calls of explore() (explorer.hpp:80-155 -- here the drop-in's,
// include/bapipe_b200/explorer.hpp, every candidate on the GPU), one JSON
// line per case with every call's wall time in ms, the median and minimum,
// the outcome and the best candidate.  --threads T (reference build only)
// also runs T concurrent callers and reports their aggregate calls/s.  Built
// with -DUSE_REFERENCE against the reference headers (oracle/Makefile) the
// same source times the reference's own explore().
#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <string>
#include <thread>
#include <vector>

#ifdef USE_REFERENCE
#include "bapipe/explorer.hpp"
using namespace bapipe;
#else
#include "bapipe_b200/io.hpp"
using namespace bapipe_b200;
#endif

namespace {

using Clock = std::chrono::steady_clock;

struct Outcome {
    std::string status = "ok";
    std::string best;
};

Outcome call(const NetworkProfile& net, const ClusterSpec& cl, const TrainingConfig& cfg) {
    Outcome o;
    try {
        ExplorationResult r = explore(net, cl, cfg);
        o.best = std::string(to_string(r.best.kind)) + " M=" + std::to_string(r.best.M) + " makespan=" +
                 r.best.simulated_makespan.str();
    } catch (const NoFeasiblePlan&) {
        o.status = "no_feasible_plan";
    } catch (const std::overflow_error&) {
        o.status = "overflow";
    } catch (const std::exception& e) {
        o.status = std::string("error: ") + e.what();
    }
    return o;
}

double ms_since(Clock::time_point t) { return std::chrono::duration<double, std::milli>(Clock::now() - t).count(); }

}  // namespace

int main(int argc, char** argv) {
    int a = 1, threads = 0;
    if (a + 1 < argc && std::string(argv[a]) == "--threads") {
        threads = std::atoi(argv[a + 1]);
        a += 2;
    }
    if (argc - a < 4 || (argc - a - 1) % 3 != 0) {
        std::fprintf(stderr, "usage: percall [--threads T] REPS MINI NET.json CLUSTER.json [...]\n");
        return 1;
    }
    const int reps = std::atoi(argv[a++]);
    for (int c = 0; a + 2 < argc; ++c, a += 3) {
        TrainingConfig cfg;
        cfg.mini_batch_size = std::atoll(argv[a]);
        const NetworkProfile net = load_network(argv[a + 1], false);
        const ClusterSpec cl = load_cluster(argv[a + 2], false);
        Outcome o;
        for (int w = 0; w < 2; ++w) o = call(net, cl, cfg);
        std::vector<double> ms;
        for (int r = 0; r < reps; ++r) {
            const auto t = Clock::now();
            o = call(net, cl, cfg);
            ms.push_back(ms_since(t));
        }
        std::vector<double> s = ms;
        std::sort(s.begin(), s.end());
        std::printf("{\"case\": %d, \"status\": \"%s\", \"best\": \"%s\", \"reps\": %d, \"median_ms\": %.4f, "
                    "\"min_ms\": %.4f, \"ms\": [",
                    c, o.status.c_str(), o.best.c_str(), reps, s[s.size() / 2], s[0]);
        for (size_t i = 0; i < ms.size(); ++i) std::printf("%s%.4f", i ? ", " : "", ms[i]);
        std::printf("]");
        if (threads > 1) {
            // T independent callers (explore() is reentrant),
            // each on its own copy of the inputs
            std::atomic<int> next{0};
            const int total = reps * threads;
            const auto t = Clock::now();
            std::vector<std::thread> pool;
            for (int k = 0; k < threads; ++k)
                pool.emplace_back([&] {
                    const NetworkProfile n2 = net;
                    const ClusterSpec c2 = cl;
                    while (next.fetch_add(1) < total) call(n2, c2, cfg);
                });
            for (auto& th : pool) th.join();
            std::printf(", \"pool_threads\": %d, \"pool_calls_per_s\": %.3f", threads, total / (ms_since(t) / 1e3));
        }
        std::printf("}\n");
        std::fflush(stdout);
    }
    return 0;
}
