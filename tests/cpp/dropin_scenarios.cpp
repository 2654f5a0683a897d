// dropin_scenarios.cpp -- one source, two builds:
//   -DUSE_REFERENCE  against the reference headers (/root/reference/proj/include),
//                    run in the dev container to produce tests/golden/dropin_expected.txt
//   (default)        against include/bapipe_b200/explorer.hpp + libbapipe_b200.so,
//                    run on the B200 by tests/test_dropin.py and diffed with the golden.
// Scenarios: every explore() case of the reference's tests/test_explorer.cpp
// (tri_net / tri_cluster, 25-185), its error paths, and seeded heterogeneous
// chains.  The dump is canonical text: every field of ExplorationResult, or the
// exception type and what() string.
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

using api::ClusterSpec;
using api::ExecutionMode;
using api::NetworkProfile;
using api::ScheduleKind;
using api::TrainingConfig;

namespace {

NetworkProfile tri_net() { return api::synth_uniform_network(3, 10, 20, 100, 50, {"gpu"}); }

ClusterSpec tri_cluster(ExecutionMode mode, std::vector<std::int64_t> caps) {
    ClusterSpec cl;
    for (int i = 0; i < 3; ++i) {
        api::AcceleratorSpec a;
        a.id = "g" + std::to_string(i);
        a.accel_type = "gpu";
        a.mem_capacity_bytes = caps[i];
        cl.accelerators.push_back(a);
    }
    cl.link_bandwidth = {50, 50};
    cl.execution_mode = mode;
    return cl;
}

// splitmix64: deterministic, identical in both builds
struct Rng {
    std::uint64_t s;
    std::uint64_t next() {
        std::uint64_t z = (s += 0x9E3779B97F4A7C15ull);
        z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
        z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
        return z ^ (z >> 31);
    }
    std::int64_t in(std::int64_t lo, std::int64_t hi) { return lo + (std::int64_t)(next() % (std::uint64_t)(hi - lo + 1)); }
};

struct Scenario {
    std::string name;
    NetworkProfile net;
    ClusterSpec cl;
    TrainingConfig cfg;
};

// big = true: times, sizes and bandwidths near the int64 limits, where
// Rat: overflow escapes from some candidates
Scenario random_scenario(std::uint64_t seed, bool big = false) {
    Rng r{seed};
    Scenario s;
    s.name = (big ? "random-big/" : "random/") + std::to_string(seed);
    const int tb = big ? 44 : 0, sb = big ? 18 : 0;
    const char* types[3] = {"fpga", "gpu", "tpu"};
    int n_types = (int)r.in(1, 3);
    std::int64_t L = r.in(4, 40);
    s.net.name = "net" + std::to_string(seed);
    for (std::int64_t j = 0; j < L; ++j) {
        api::LayerProfile l;
        l.name = "l" + std::to_string(j);
        for (int t = 0; t < n_types; ++t) {
            l.fp_time[types[t]] = r.in(1, 400ll << tb);
            l.bp_time[types[t]] = r.in(1, 800ll << tb);
        }
        l.weight_bytes = r.in(0, 1ll << (20 + sb));
        l.out_activation_bytes = r.in(0, 1ll << (18 + sb));
        s.net.layers.push_back(l);
    }
    std::int64_t N = r.in(1, std::min<std::int64_t>(8, L));
    s.cl.execution_mode = r.in(0, 1) ? ExecutionMode::Asynchronous : ExecutionMode::Synchronous;
    for (std::int64_t i = 0; i < N; ++i) {
        api::AcceleratorSpec a;
        a.id = "acc" + std::to_string(i);
        a.accel_type = types[r.in(0, n_types - 1)];
        a.mem_capacity_bytes = r.in(1, 4) << r.in(22 + sb, 31 + sb);
        if (r.in(0, 3) == 0) a.min_micro_batch[api::all_schedule_kinds[r.in(0, 3)]] = r.in(1, 8);
        s.cl.accelerators.push_back(a);
        if (i + 1 < N) s.cl.link_bandwidth.push_back(r.in(1, 4096ll << sb));
    }
    s.cfg.mini_batch_size = std::int64_t(1) << r.in(0, 7);
    if (r.in(0, 4) == 0) s.cfg.micro_batch_candidates = std::vector<std::int64_t>{1, s.cfg.mini_batch_size};
    return s;
}

std::vector<Scenario> scenarios() {
    std::vector<Scenario> v;
    auto add = [&](std::string name, NetworkProfile net, ClusterSpec cl, std::int64_t mini,
                   std::optional<std::vector<std::int64_t>> ms = std::nullopt) {
        Scenario s{std::move(name), std::move(net), std::move(cl), {}};
        s.cfg.mini_batch_size = mini;
        s.cfg.micro_batch_candidates = ms;
        v.push_back(std::move(s));
    };
    add("memory-tight sync selects 1f1b-sno", tri_net(), tri_cluster(ExecutionMode::Synchronous, {400, 1000000, 1000000}), 4,
        std::vector<std::int64_t>{4});
    add("abundant memory M>2 selects 1f1b-so", tri_net(),
        tri_cluster(ExecutionMode::Synchronous, {1000000, 1000000, 1000000}), 4, std::vector<std::int64_t>{4});
    add("M=1 tie broken by memory", tri_net(), tri_cluster(ExecutionMode::Synchronous, {1000000, 1000000, 1000000}), 1);
    {
        ClusterSpec cl = tri_cluster(ExecutionMode::Asynchronous, {600, 600, 600});
        for (auto& a : cl.accelerators) a.min_micro_batch[ScheduleKind::OneFOneB_AS] = 4;
        add("async per-kind floors select fbp-as", tri_net(), cl, 8);
    }
    add("tight", tri_net(), tri_cluster(ExecutionMode::Synchronous, {400, 1000000, 1000000}), 4);
    add("roomy", tri_net(), tri_cluster(ExecutionMode::Synchronous, {1000000000, 1000000000, 1000000000}), 4);
    add("ranking ascending", api::synth_uniform_network(6, 10, 20, 100, 40, {"gpu"}),
        tri_cluster(ExecutionMode::Synchronous, {1000000, 1000000, 1000000}), 8);
    add("everything rejected", tri_net(), tri_cluster(ExecutionMode::Synchronous, {1, 1, 1}), 2);
    // error paths
    add("non-divisor candidate", tri_net(), tri_cluster(ExecutionMode::Synchronous, {1000, 1000, 1000}), 128,
        std::vector<std::int64_t>{8, 3});
    add("empty candidate list", tri_net(), tri_cluster(ExecutionMode::Synchronous, {1000, 1000, 1000}), 4,
        std::vector<std::int64_t>{});
    add("mini-batch 0", tri_net(), tri_cluster(ExecutionMode::Synchronous, {1000, 1000, 1000}), 0);
    {
        ClusterSpec cl = tri_cluster(ExecutionMode::Synchronous, {1000, 1000, 1000});
        cl.accelerators[2].accel_type = "tpu";
        add("missing accelerator type", tri_net(), cl, 4);
    }
    {
        ClusterSpec cl = tri_cluster(ExecutionMode::Synchronous, {1000, 1000, 1000});
        cl.link_bandwidth = {50};
        add("wrong link count", tri_net(), cl, 4);
    }
    {
        NetworkProfile net = tri_net();
        net.layers[1].fp_time["gpu"] = 0;
        add("zero fp time", net, tri_cluster(ExecutionMode::Synchronous, {1000, 1000, 1000}), 4);
    }
    {
        ClusterSpec cl = tri_cluster(ExecutionMode::Asynchronous, {1000000, 1000000, 1000000});
        cl.accelerators.resize(1);
        cl.link_bandwidth.clear();
        add("single stage", api::synth_uniform_network(5, 7, 9, 100, 40, {"gpu"}), cl, 16);
    }
    // activations near 2^58: every candidate is rejected for memory
    add("huge activations", api::synth_uniform_network(3, 10, 20, 0, std::int64_t(1) << 58, {"gpu"}),
        tri_cluster(ExecutionMode::Synchronous, {INT64_MAX, INT64_MAX, INT64_MAX}), 4);
    for (std::uint64_t seed = 1; seed <= 40; ++seed) v.push_back(random_scenario(seed));
    for (std::uint64_t seed = 1; seed <= 40; ++seed) v.push_back(random_scenario(seed, true));
    return v;
}

void dump_result(std::ostream& os, const api::ExplorationResult& r) {
    os << "mini_batch " << r.mini_batch_size << " ranked " << r.ranked.size() << " rejected " << r.rejected.size()
       << "\n";
    auto cand = [&](const char* tag, const api::Candidate& c) {
        os << tag << " " << api::to_string(c.kind) << " M=" << c.M << " micro=" << c.micro_batch_size
           << " makespan=" << c.simulated_makespan.str() << " peak=" << c.peak_memory.str()
           << " maxbw=" << c.max_bandwidth_demand.str() << " est=" << c.est.minibatch_time.str()
           << " bubble=" << c.est.bubble_fraction.str() << " heur=" << c.est.heuristic << " N=" << c.est.N
           << " estM=" << c.est.M << " feasible=" << c.est.memory_feasible() << "\n";
        for (std::size_t i = 0; i < c.plan.stages.size(); ++i) {
            const auto& s = c.plan.stages[i];
            os << "  stage " << s.accelerator_id << " [" << s.lo << "," << s.hi << "] lead=" << s.leading_fraction.str()
               << " trail=" << s.trailing_fraction.str() << " feat=" << c.est.features_mem[i].str()
               << " w=" << c.est.weights_mem[i].str() << "\n";
        }
        os << "  bw";
        for (const auto& b : c.est.bandwidth_demand) os << " " << b.str();
        os << "\n";
    };
    cand("best", r.best);
    for (const auto& c : r.ranked) cand("ranked", c);
    for (const auto& j : r.rejected)
        os << "rejected " << api::to_string(j.kind) << " M=" << j.M << " " << j.reason << ": " << j.detail << "\n";
}

}  // namespace

int main() {
    for (const Scenario& s : scenarios()) {
        std::ostringstream os;
        os << "== " << s.name << "\n";
        try {
            api::ExplorationResult r = api::explore(s.net, s.cl, s.cfg);
            dump_result(os, r);
        } catch (const api::NoFeasiblePlan& e) {
            os << "EXC NoFeasiblePlan " << e.what() << "\n";
        } catch (const api::SchemaError& e) {
            os << "EXC SchemaError " << e.what() << "\n";
        } catch (const api::InvalidPlan& e) {
            os << "EXC InvalidPlan " << e.what() << "\n";
        } catch (const std::overflow_error& e) {
            os << "EXC overflow_error " << e.what() << "\n";
        } catch (const std::domain_error& e) {
            os << "EXC domain_error " << e.what() << "\n";
        } catch (const api::Error& e) {
            os << "EXC Error " << e.what() << "\n";
        }
        std::cout << os.str();
    }
    return 0;
}
