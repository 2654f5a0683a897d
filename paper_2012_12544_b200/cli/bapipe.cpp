// bapipe -- command-line front end of the B200 explorer.
//
// Mirrors the reference tool's `validate` and `explore` subcommands
// (tools/bapipe.cpp:100-232): same positional arguments and options, same
// JSON / table output (include/bapipe_b200/io.hpp), same run manifest
// (FNV-1a-64 input digests, tool_version 1.0.0, tools/bapipe.cpp:17-47) and
// the same exit codes: 0 success, 1 input or usage error, 2 infeasible
// (tools/bapipe.cpp:257-269).  `plan` and `simulate` evaluate a single
// candidate outside the explore path and are not part of this build.
//
// Every candidate is evaluated on the GPU through libbapipe_b200.so.  Built
// with -DUSE_REFERENCE against the reference headers instead, the same source
// is the checker that produced tests/golden/cli/expected.json.
#include <cctype>
#include <cstdint>
#include <cstdlib>
#include <fstream>
#include <iostream>
#include <sstream>
#include <string>
#include <vector>

#ifdef USE_REFERENCE
#include "bapipe/explorer.hpp"
using namespace bapipe;
#else
#include "bapipe_b200/io.hpp"
using namespace bapipe_b200;
#endif

namespace {

constexpr const char* kToolVersion = "1.0.0";

struct UsageError : std::runtime_error {
    explicit UsageError(const std::string& m) : std::runtime_error(m) {}
};

std::string read_bytes(const std::string& path) {
    std::ifstream in(path, std::ios::binary);
    if (!in) throw ParseError("cannot open '" + path + "'");
    std::ostringstream s;
    s << in.rdbuf();
    return s.str();
}

std::string fnv1a64_hex(const std::string& bytes) {
    std::uint64_t h = 0xcbf29ce484222325ull;
    for (unsigned char c : bytes) h = (h ^ c) * 0x100000001b3ull;
    char buf[17];
    std::snprintf(buf, sizeof(buf), "%016llx", (unsigned long long)h);
    return buf;
}

json manifest(const std::vector<std::string>& inputs, const std::vector<std::string>& argv) {
    json digests = json::object();
    for (const std::string& p : inputs) digests[p] = fnv1a64_hex(read_bytes(p));
    return json{{"tool_version", kToolVersion}, {"input_digests", digests}, {"command", argv}, {"seed_free", true}};
}

std::int64_t to_int(const std::string& opt, const std::string& v) {
    try {
        std::size_t used = 0;
        const long long x = std::stoll(v, &used);
        if (used == v.size()) return x;
    } catch (const std::exception&) {
    }
    throw UsageError(opt + ": '" + v + "' is not an integer");
}

struct Args {
    std::string cmd, net, cluster, format = "human", out;
    bool lenient = false, has_minibatch = false;
    std::int64_t minibatch = 0;
    std::vector<std::int64_t> micro_set;
    double dp_baseline = 0.0;
};

Args parse(int argc, char** argv) {
    Args a;
    std::vector<std::string> pos;
    for (int i = 1; i < argc; ++i) {
        std::string s = argv[i], val;
        const bool opt = s.size() > 1 && s[0] == '-' && !(s.size() > 1 && std::isdigit((unsigned char)s[1]));
        if (!opt) {
            pos.push_back(s);
            continue;
        }
        const auto eq = s.find('=');
        const bool inline_val = eq != std::string::npos && s.rfind("--", 0) == 0;
        if (inline_val) {
            val = s.substr(eq + 1);
            s = s.substr(0, eq);
        }
        auto next = [&]() -> std::string {
            if (inline_val) return val;
            if (i + 1 >= argc) throw UsageError(s + " requires a value");
            return argv[++i];
        };
        if (s == "--lenient") a.lenient = true;
        else if (s == "--format") {
            a.format = next();
            if (a.format != "human" && a.format != "json") throw UsageError("--format: must be human or json");
        } else if (s == "--minibatch") {
            a.minibatch = to_int(s, next());
            a.has_minibatch = true;
        } else if (s == "--micro-set") {
            if (inline_val) a.micro_set.push_back(to_int(s, val));
            else {
                bool any = false;
                while (i + 1 < argc && argv[i + 1][0] != '-') {
                    a.micro_set.push_back(to_int(s, argv[++i]));
                    any = true;
                }
                if (!any) throw UsageError(s + " requires a value");
            }
        } else if (s == "-o" || s == "--out") a.out = next();
        else if (s == "--dp-baseline") {
            const std::string v = next();
            char* end = nullptr;
            a.dp_baseline = std::strtod(v.c_str(), &end);
            if (end == v.c_str() || *end) throw UsageError("--dp-baseline: '" + v + "' is not a number");
        } else throw UsageError("unknown option " + s);
    }
    if (pos.empty()) throw UsageError("a subcommand is required (validate | explore)");
    a.cmd = pos[0];
    if (a.cmd == "plan" || a.cmd == "simulate")
        throw UsageError("'" + a.cmd + "' evaluates one candidate outside the explore path and is not part of this build");
    if (a.cmd != "validate" && a.cmd != "explore") throw UsageError("unknown subcommand '" + a.cmd + "'");
    if (pos.size() != 3) throw UsageError(a.cmd + ": expected <net> <cluster>");
    a.net = pos[1];
    a.cluster = pos[2];
    if (a.cmd == "explore" && !a.has_minibatch) throw UsageError("explore: --minibatch is required");
    return a;
}

}  // namespace

int main(int argc, char** argv) {
    const std::vector<std::string> raw(argv, argv + argc);
    Args a;
    try {
        a = parse(argc, argv);
    } catch (const UsageError& e) {
        std::cerr << "usage error: " << e.what() << "\n"
                  << "usage: bapipe validate|explore <net.json> <cluster.json> [--lenient] [--format human|json]\n"
                  << "       explore: --minibatch B [--micro-set M...] [-o plan.json] [--dp-baseline US]\n";
        return 1;
    }
    try {
        const NetworkProfile net = load_network(a.net, a.lenient);
        const ClusterSpec cluster = load_cluster(a.cluster, a.lenient);
        validate_pair(net, cluster);
        if (a.cmd == "validate") {
            if (a.format == "json")
                std::cout << dump_canonical(json{{"status", "ok"}, {"manifest", manifest({a.net, a.cluster}, raw)}});
            else
                std::cout << "ok: network '" << net.name << "' (" << net.L() << " layers), cluster of " << cluster.N()
                          << "\n";
            return 0;
        }
        TrainingConfig cfg;
        cfg.mini_batch_size = a.minibatch;
        if (!a.micro_set.empty()) cfg.micro_batch_candidates = a.micro_set;
        ExplorationResult res = explore(net, cluster, cfg);
        if (a.dp_baseline > 0.0) res.dp_baseline_minibatch_time = a.dp_baseline;
        if (!a.out.empty()) save_file(a.out, plan_to_json(res.best.plan));
        if (a.format == "json") {
            json j = exploration_to_json(res);
            j["manifest"] = manifest({a.net, a.cluster}, raw);
            std::cout << dump_canonical(j);
        } else {
            std::cout << exploration_table(res);
            if (!a.out.empty()) std::cout << "best plan written to " << a.out << "\n";
        }
        return 0;
    } catch (const Infeasible& e) {
        std::cerr << e.what() << "\n";
        return 2;
    } catch (const InfeasibleShape& e) {
        std::cerr << e.what() << "\n";
        return 2;
    } catch (const NoFeasiblePlan& e) {
        std::cerr << e.what() << "\n";
        return 2;
    } catch (const std::exception& e) {
        std::cerr << "error: " << e.what() << "\n";
        return 1;
    }
}
