// bapipe -- command-line front end of the B200 explorer.
//
// Mirrors the reference tool's four subcommands (tools/bapipe.cpp:100-256):
// `validate`, `explore`, `plan` (balance_partition + estimate for one
// schedule and M) and `simulate` (the full event timeline of a plan file,
// with --gantt .csv/.svg export and --trace) -- same positional arguments and
// options, same JSON / table / human output (include/bapipe_b200/io.hpp,
// gantt.hpp), same run manifest (FNV-1a-64 input digests, tool_version 1.0.0,
// tools/bapipe.cpp:17-47) and the same exit codes: 0 success, 1 input or
// usage error, 2 infeasible (tools/bapipe.cpp:257-269).
//
// Every candidate, plan and timeline is evaluated on the GPU through
// libbapipe_b200.so.  Built
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
#include "bapipe/gantt.hpp"
using namespace bapipe;
#else
#include "bapipe_b200/gantt.hpp"
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
    std::string cmd, net, cluster, plan, format = "human", out, schedule, gantt;
    bool lenient = false, has_minibatch = false, has_micro = false, has_schedule = false, trace = false;
    std::int64_t minibatch = 0, micro = 0;
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
        } else if (s == "--micro") {
            a.micro = to_int(s, next());
            a.has_micro = true;
        } else if (s == "--schedule") {
            a.schedule = next();
            a.has_schedule = true;
        } else if (s == "--gantt") a.gantt = next();
        else if (s == "--trace") a.trace = true;
        else if (s == "-o" || s == "--out") a.out = next();
        else if (s == "--dp-baseline") {
            const std::string v = next();
            char* end = nullptr;
            a.dp_baseline = std::strtod(v.c_str(), &end);
            if (end == v.c_str() || *end) throw UsageError("--dp-baseline: '" + v + "' is not a number");
        } else throw UsageError("unknown option " + s);
    }
    if (pos.empty()) throw UsageError("a subcommand is required (validate | plan | explore | simulate)");
    a.cmd = pos[0];
    if (a.cmd != "validate" && a.cmd != "explore" && a.cmd != "plan" && a.cmd != "simulate")
        throw UsageError("unknown subcommand '" + a.cmd + "'");
    const std::size_t want = a.cmd == "simulate" ? 4 : 3;
    if (pos.size() != want)
        throw UsageError(a.cmd + (a.cmd == "simulate" ? ": expected <net> <cluster> <plan>" : ": expected <net> <cluster>"));
    a.net = pos[1];
    a.cluster = pos[2];
    if (a.cmd == "simulate") a.plan = pos[3];
    // which options each subcommand takes (tools/bapipe.cpp:113-142)
    const bool plan_like = a.cmd == "plan" || a.cmd == "simulate";
    if (a.cmd == "explore" && !a.has_minibatch) throw UsageError("explore: --minibatch is required");
    if (plan_like && !a.has_schedule) throw UsageError(a.cmd + ": --schedule is required");
    if (a.cmd == "simulate" && !a.has_micro) throw UsageError("simulate: --micro is required");
    if (a.cmd == "validate" && (a.has_minibatch || !a.out.empty())) throw UsageError("validate takes no such option");
    if (!plan_like && (a.has_micro || a.has_schedule)) throw UsageError(a.cmd + ": unknown option --micro/--schedule");
    if (a.cmd != "explore" && (!a.micro_set.empty() || a.dp_baseline != 0.0))
        throw UsageError(a.cmd + ": unknown option --micro-set/--dp-baseline");
    if (a.cmd != "simulate" && (!a.gantt.empty() || a.trace)) throw UsageError(a.cmd + ": unknown option --gantt/--trace");
    if (a.cmd == "simulate" && !a.out.empty()) throw UsageError("simulate: unknown option -o");
    return a;
}

ScheduleKind require_kind(const std::string& s) {
    auto k = parse_schedule_kind(s);
    if (!k) throw SchemaError("unknown schedule kind '" + s + "'");
    return *k;
}

void write_text(const std::string& path, const std::string& text) {
    std::ofstream out(path, std::ios::binary);
    if (!out) throw Error("cannot write '" + path + "'");
    out << text;
}

// SimReport (tools/bapipe.cpp:61-77)
json sim_json(const Timeline& t, const CostEstimate& est) {
    json feat = json::array(), wt = json::array(), busy = json::array();
    for (const Rat& r : t.per_stage_feature_highwater) feat.push_back(r.str());
    for (const Rat& r : t.per_stage_weight_static) wt.push_back(r.str());
    for (const Rat& r : t.per_link_busy_fraction) busy.push_back(r.str());
    return {{"makespan_us", t.makespan.str()},
            {"bubble_fraction", est.bubble_fraction.str()},
            {"estimate_minibatch_us", est.minibatch_time.str()},
            {"estimate_is_heuristic", est.heuristic},
            {"feature_highwater_bytes", feat},
            {"weight_static_bytes", wt},
            {"link_busy_fraction", busy},
            {"events", (std::int64_t)t.events.size()}};
}

// print_sim_human (tools/bapipe.cpp:79-90)
void sim_human(const Timeline& t, const CostEstimate& est) {
    std::cout << "makespan: " << t.makespan.str() << " us\n";
    std::cout << "bubble:   " << est.bubble_fraction.str() << (est.heuristic ? " (heuristic)" : "") << "\n";
    for (std::size_t i = 0; i < t.per_stage_feature_highwater.size(); ++i)
        std::cout << "stage " << i + 1 << ": features " << t.per_stage_feature_highwater[i].str() << " B, weights "
                  << t.per_stage_weight_static[i].str() << " B\n";
    for (std::size_t k = 0; k < t.per_link_busy_fraction.size(); ++k)
        std::cout << "link " << k + 1 << ": busy " << t.per_link_busy_fraction[k].str() << "\n";
}

// `plan` (tools/bapipe.cpp:152-190)
int run_plan(const Args& a, const NetworkProfile& net, const ClusterSpec& cluster,
             const std::vector<std::string>& raw) {
    const ScheduleKind kind = require_kind(a.schedule);
    if (a.micro <= 0 && a.minibatch <= 0) throw SchemaError("plan: give --micro and/or --minibatch");
    const std::int64_t M = a.micro > 0 ? a.micro : a.minibatch;
    const std::int64_t mini = a.minibatch > 0 ? a.minibatch : M;
    if (mini % M != 0) throw SchemaError("--minibatch must be divisible by --micro");
    const std::int64_t mu = mini / M;
    const PartitionPlan p = balance_partition(net, cluster, kind, M, mu);
    const CostEstimate est = estimate(kind, p, net, cluster, M, mu);
    if (!est.memory_feasible()) throw Infeasible("memory");
    const json pj = plan_to_json(p);
    if (!a.out.empty()) save_file(a.out, pj);
    if (a.format == "json") {
        json mem = json::array(), bw = json::array();
        for (std::size_t i = 0; i < est.features_mem.size(); ++i)
            mem.push_back((est.features_mem[i] + est.weights_mem[i]).str());
        for (const Rat& d : est.bandwidth_demand) bw.push_back(d.str());
        std::cout << dump_canonical(json{{"schedule", to_string(kind)},
                                         {"M", M},
                                         {"micro_batch_size", mu},
                                         {"minibatch_time_us", est.minibatch_time.str()},
                                         {"bubble_fraction", est.bubble_fraction.str()},
                                         {"estimate_is_heuristic", est.heuristic},
                                         {"stage_memory_bytes", mem},
                                         {"bandwidth_demand_bytes_per_us", bw},
                                         {"plan", pj},
                                         {"manifest", manifest({a.net, a.cluster}, raw)}});
    } else {
        std::cout << "schedule " << to_string(kind) << ", M=" << M << ", micro-batch size " << mu << "\n";
        for (std::size_t i = 0; i < p.stages.size(); ++i) {
            const StageAssignment& s = p.stages[i];
            std::cout << "stage " << i + 1 << " (" << s.accelerator_id << "): layers [" << s.lo << "," << s.hi
                      << "] lead " << s.leading_fraction.str() << " trail " << s.trailing_fraction.str() << ", mem "
                      << (est.features_mem[i] + est.weights_mem[i]).str() << " B\n";
        }
        std::cout << "estimated mini-batch time " << est.minibatch_time.str() << " us, bubble "
                  << est.bubble_fraction.str() << (est.heuristic ? " (heuristic)" : "") << "\n";
        if (!a.out.empty()) std::cout << "plan written to " << a.out << "\n";
    }
    return 0;
}

// `simulate` (tools/bapipe.cpp:234-256)
int run_simulate(const Args& a, const NetworkProfile& net, const ClusterSpec& cluster,
                 const std::vector<std::string>& raw) {
    const ScheduleKind kind = require_kind(a.schedule);
    const PartitionPlan p = load_plan(a.plan, a.lenient);
    if (a.micro == 0) throw SchemaError("--micro must be nonzero");   // the reference divides by it
    const std::int64_t mini = a.minibatch > 0 ? a.minibatch : a.micro;
    if (mini % a.micro != 0) throw SchemaError("--minibatch must be divisible by --micro");
    const std::int64_t mu = mini / a.micro;
    const Timeline t = simulate(kind, p, net, cluster, a.micro, mu);
    const CostEstimate est = estimate(kind, p, net, cluster, a.micro, mu);
    if (!a.gantt.empty()) {
        const bool svg = a.gantt.size() >= 4 && a.gantt.compare(a.gantt.size() - 4, 4, ".svg") == 0;
        write_text(a.gantt, export_gantt(t, svg ? GanttFormat::Svg : GanttFormat::Csv));
    }
    if (a.format == "json") {
        json j = sim_json(t, est);
        j["manifest"] = manifest({a.net, a.cluster, a.plan}, raw);
        std::cout << dump_canonical(j);
    } else {
        sim_human(t, est);
    }
    if (a.trace) std::cout << gantt_csv(t);
    return 0;
}

}  // namespace

int main(int argc, char** argv) {
    const std::vector<std::string> raw(argv, argv + argc);
    Args a;
    try {
        a = parse(argc, argv);
    } catch (const UsageError& e) {
        std::cerr << "usage error: " << e.what() << "\n"
                  << "usage: bapipe validate|plan|explore <net.json> <cluster.json> [--lenient] [--format human|json]\n"
                  << "       bapipe simulate <net.json> <cluster.json> <plan.json> [--lenient] [--format human|json]\n"
                  << "       plan: --schedule K [--micro M] [--minibatch B] [-o plan.json]\n"
                  << "       explore: --minibatch B [--micro-set M...] [-o plan.json] [--dp-baseline US]\n"
                  << "       simulate: --schedule K --micro M [--minibatch B] [--gantt out.csv|out.svg] [--trace]\n";
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
        if (a.cmd == "plan") return run_plan(a, net, cluster, raw);
        if (a.cmd == "simulate") return run_simulate(a, net, cluster, raw);
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
