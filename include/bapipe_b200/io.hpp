// bapipe_b200/io.hpp -- the reference's file formats for the explore path
// (SURVEY.md 8f row F1): profile / cluster / plan JSON ingest with the same
// strict schema checks and messages, the canonical writers, and the explore
// report (JSON and table).  Mirrors
//   profiles.hpp:134-311   check_keys, get_int/get_str/get_time_map,
//                          parse_file, network/cluster_from_json, load_*,
//                          network/cluster_to_json, dump_canonical, save_file
//   plan.hpp:160-214       rat_from_string, plan_to_json, plan_from_json
//   explorer.hpp:160-217   exploration_to_json, exploration_table
// Needs nlohmann/json ("json.hpp", as profiles.hpp:11 includes it; the image
// ships 3.11.3 under cudnn_frontend/thirdparty/nlohmann).
#pragma once

#include <cstdio>
#include <fstream>
#include <initializer_list>
#include <sstream>
#include <string>

#include "explorer.hpp"
#include "json.hpp"

namespace bapipe_b200 {

using json = nlohmann::ordered_json;   // insertion-ordered keys (profiles.hpp:18)

namespace io_detail {

// Unknown keys are a SchemaError unless lenient (profiles.hpp:139-148).
inline void only_keys(const json& j, std::initializer_list<const char*> allowed, bool lenient,
                      const std::string& where) {
    if (lenient) return;
    for (const auto& kv : j.items()) {
        bool known = false;
        for (const char* a : allowed) known = known || kv.key() == a;
        if (!known) throw SchemaError(where + ": unknown key '" + kv.key() + "'");
    }
}

inline const json& field(const json& j, const char* key, const std::string& where) {
    if (!j.contains(key)) throw SchemaError(where + ": missing '" + key + "'");
    return j.at(key);
}

inline std::int64_t int_field(const json& j, const char* key, const std::string& where) {
    const json& v = field(j, key, where);
    if (!v.is_number_integer()) throw SchemaError(where + ": '" + key + "' must be an integer");
    return v.get<std::int64_t>();
}

inline std::string str_field(const json& j, const char* key, const std::string& where) {
    const json& v = field(j, key, where);
    if (!v.is_string()) throw SchemaError(where + ": '" + key + "' must be a string");
    return v.get<std::string>();
}

inline std::map<std::string, std::int64_t> int_map_field(const json& j, const char* key, const std::string& where) {
    const json& v = field(j, key, where);
    if (!v.is_object()) throw SchemaError(where + ": '" + key + "' must be an object");
    std::map<std::string, std::int64_t> out;
    for (const auto& kv : v.items()) {
        if (!kv.value().is_number_integer())
            throw SchemaError(where + ": '" + key + "." + kv.key() + "' must be an integer");
        out[kv.key()] = kv.value().get<std::int64_t>();
    }
    return out;
}

inline json read_object(const std::string& path) {
    std::ifstream in(path);
    if (!in) throw ParseError("cannot open '" + path + "'");
    json j;
    try {
        j = json::parse(in);
    } catch (const nlohmann::json::exception& e) {
        throw ParseError(path + ": " + e.what());
    }
    if (!j.is_object()) throw ParseError(path + ": top-level value must be an object");
    return j;
}

inline const json& array_field(const json& j, const char* key, const std::string& missing_msg) {
    if (!j.contains(key) || !j.at(key).is_array()) throw SchemaError(missing_msg);
    return j.at(key);
}

}  // namespace io_detail

// ---- ingest (profiles.hpp:192-282)
inline NetworkProfile network_from_json(const json& j, bool lenient = false) {
    using namespace io_detail;
    only_keys(j, {"name", "layers"}, lenient, "network");
    NetworkProfile net;
    net.name = str_field(j, "name", "network");
    const json& layers = array_field(j, "layers", "network: missing 'layers' array");
    for (std::size_t i = 0; i < layers.size(); ++i) {
        const json& lj = layers[i];
        const std::string where = "layer " + std::to_string(i);
        only_keys(lj, {"name", "fp_us", "bp_us", "weight_bytes", "out_activation_bytes"}, lenient, where);
        LayerProfile l;
        l.name = str_field(lj, "name", where);
        l.fp_time = int_map_field(lj, "fp_us", where);
        l.bp_time = int_map_field(lj, "bp_us", where);
        l.weight_bytes = int_field(lj, "weight_bytes", where);
        l.out_activation_bytes = int_field(lj, "out_activation_bytes", where);
        net.layers.push_back(std::move(l));
    }
    validate_network(net);
    return net;
}

inline ClusterSpec cluster_from_json(const json& j, bool lenient = false) {
    using namespace io_detail;
    only_keys(j, {"execution_mode", "accelerators", "link_bandwidth_bytes_per_us"}, lenient, "cluster");
    ClusterSpec c;
    const std::string mode = str_field(j, "execution_mode", "cluster");
    if (mode != "sync" && mode != "async") throw SchemaError("cluster: execution_mode must be 'sync' or 'async'");
    c.execution_mode = mode == "sync" ? ExecutionMode::Synchronous : ExecutionMode::Asynchronous;
    const json& accels = array_field(j, "accelerators", "cluster: missing 'accelerators' array");
    for (std::size_t i = 0; i < accels.size(); ++i) {
        const json& aj = accels[i];
        const std::string where = "accelerator " + std::to_string(i);
        only_keys(aj, {"id", "type", "mem_capacity_bytes", "min_micro_batch"}, lenient, where);
        AcceleratorSpec a;
        a.id = str_field(aj, "id", where);
        a.accel_type = str_field(aj, "type", where);
        a.mem_capacity_bytes = int_field(aj, "mem_capacity_bytes", where);
        if (aj.contains("min_micro_batch")) {
            for (const auto& [name, v] : int_map_field(aj, "min_micro_batch", where)) {
                const auto kind = parse_schedule_kind(name);
                if (!kind) throw SchemaError(where + ": unknown schedule kind '" + name + "' in min_micro_batch");
                a.min_micro_batch[*kind] = v;
            }
        }
        c.accelerators.push_back(std::move(a));
    }
    const json& links =
        array_field(j, "link_bandwidth_bytes_per_us", "cluster: missing 'link_bandwidth_bytes_per_us' array");
    for (const json& b : links) {
        if (!b.is_number_integer()) throw SchemaError("cluster: link bandwidths must be integers (bytes per us)");
        c.link_bandwidth.push_back(b.get<std::int64_t>());
    }
    validate_cluster(c);
    return c;
}

inline NetworkProfile load_network(const std::string& path, bool lenient = false) {
    return network_from_json(io_detail::read_object(path), lenient);
}
inline ClusterSpec load_cluster(const std::string& path, bool lenient = false) {
    return cluster_from_json(io_detail::read_object(path), lenient);
}

// ---- canonical writers (profiles.hpp:284-311): fixed key order, 2-space
// indent, trailing newline
inline json network_to_json(const NetworkProfile& net) {
    json layers = json::array();
    for (const LayerProfile& l : net.layers) {
        json fp(l.fp_time), bp(l.bp_time);
        layers.push_back(json{{"name", l.name}, {"fp_us", fp}, {"bp_us", bp}, {"weight_bytes", l.weight_bytes},
                              {"out_activation_bytes", l.out_activation_bytes}});
    }
    return json{{"name", net.name}, {"layers", layers}};
}

inline json cluster_to_json(const ClusterSpec& c) {
    json accels = json::array();
    for (const AcceleratorSpec& a : c.accelerators) {
        json aj{{"id", a.id}, {"type", a.accel_type}, {"mem_capacity_bytes", a.mem_capacity_bytes}};
        if (!a.min_micro_batch.empty()) {
            json mm = json::object();
            for (const auto& [k, v] : a.min_micro_batch) mm[to_string(k)] = v;
            aj["min_micro_batch"] = mm;
        }
        accels.push_back(aj);
    }
    return json{{"execution_mode", to_string(c.execution_mode)},
                {"accelerators", accels},
                {"link_bandwidth_bytes_per_us", c.link_bandwidth}};
}

inline std::string dump_canonical(const json& j) { return j.dump(2) + "\n"; }

inline void save_file(const std::string& path, const json& j) {
    std::ofstream out(path, std::ios::binary);
    if (!out) throw Error("cannot write '" + path + "'");
    out << dump_canonical(j);
}

// ---- plans (plan.hpp:163-214)
inline Rat rat_from_string(const std::string& s) {
    const auto slash = s.find('/');
    try {
        return slash == std::string::npos ? Rat(std::stoll(s))
                                          : Rat(std::stoll(s.substr(0, slash)), std::stoll(s.substr(slash + 1)));
    } catch (const std::exception&) {
        throw ParseError("bad rational '" + s + "'");
    }
}

inline json plan_to_json(const PartitionPlan& plan) {
    json stages = json::array();
    for (const StageAssignment& s : plan.stages)
        stages.push_back(json{{"accelerator", s.accelerator_id},
                              {"layers", {s.lo, s.hi}},
                              {"leading_fraction", s.leading_fraction.str()},
                              {"trailing_fraction", s.trailing_fraction.str()}});
    return json{{"stages", stages}};
}

inline PartitionPlan plan_from_json(const json& j, bool lenient = false) {
    using namespace io_detail;
    only_keys(j, {"stages"}, lenient, "plan");
    const json& stages = array_field(j, "stages", "plan: missing 'stages' array");
    PartitionPlan plan;
    for (std::size_t i = 0; i < stages.size(); ++i) {
        const json& sj = stages[i];
        const std::string where = "plan stage " + std::to_string(i);
        only_keys(sj, {"accelerator", "layers", "leading_fraction", "trailing_fraction"}, lenient, where);
        StageAssignment s;
        s.accelerator_id = str_field(sj, "accelerator", where);
        if (!sj.contains("layers") || !sj.at("layers").is_array() || sj.at("layers").size() != 2)
            throw SchemaError(where + ": 'layers' must be [lo, hi]");
        s.lo = sj.at("layers")[0].get<std::int64_t>();
        s.hi = sj.at("layers")[1].get<std::int64_t>();
        if (sj.contains("leading_fraction")) s.leading_fraction = rat_from_string(str_field(sj, "leading_fraction", where));
        if (sj.contains("trailing_fraction"))
            s.trailing_fraction = rat_from_string(str_field(sj, "trailing_fraction", where));
        plan.stages.push_back(std::move(s));
    }
    return plan;
}

inline PartitionPlan load_plan(const std::string& path, bool lenient = false) {
    return plan_from_json(io_detail::read_object(path), lenient);
}

// ---- explore report (explorer.hpp:160-217)
inline json candidate_to_json(const Candidate& c) {
    json demand = json::array(), mem = json::array();
    for (const Rat& d : c.est.bandwidth_demand) demand.push_back(d.str());
    // features + weights: a Rat addition, which (like the reference's) may throw
    for (std::size_t i = 0; i < c.est.features_mem.size(); ++i)
        mem.push_back((c.est.features_mem[i] + c.est.weights_mem[i]).str());
    return json{{"schedule", to_string(c.kind)},
                {"M", c.M},
                {"micro_batch_size", c.micro_batch_size},
                {"simulated_makespan_us", c.simulated_makespan.str()},
                {"estimate_minibatch_us", c.est.minibatch_time.str()},
                {"bubble_fraction", c.est.bubble_fraction.str()},
                {"peak_memory_bytes", c.peak_memory.str()},
                {"stage_memory_bytes", mem},
                {"bandwidth_demand_bytes_per_us", demand},
                {"plan", plan_to_json(c.plan)}};
}

inline json exploration_to_json(const ExplorationResult& res) {
    json ranked = json::array(), rejected = json::array();
    for (const Candidate& c : res.ranked) ranked.push_back(candidate_to_json(c));
    for (const Rejection& r : res.rejected)
        rejected.push_back(json{{"schedule", to_string(r.kind)}, {"M", r.M}, {"reason", r.reason}, {"detail", r.detail}});
    json out{{"mini_batch_size", res.mini_batch_size},
             {"best", candidate_to_json(res.best)},
             {"ranked", ranked},
             {"rejected", rejected}};
    if (res.dp_baseline_minibatch_time) out["dp_baseline_minibatch_time_us"] = *res.dp_baseline_minibatch_time;
    return out;
}

inline std::string exploration_table(const ExplorationResult& res) {
    std::ostringstream s;
    char line[256];
    s << "schedule   M     makespan_us   bubble      peak_mem_B   max_bw_B/us\n";
    for (const Candidate& c : res.ranked) {
        std::snprintf(line, sizeof(line), "%-9s %5lld %13s %-11s %12s %12s\n", to_string(c.kind), (long long)c.M,
                      c.simulated_makespan.str().c_str(), c.est.bubble_fraction.str().c_str(),
                      c.peak_memory.str().c_str(), c.max_bandwidth_demand.str().c_str());
        s << line;
    }
    for (const Rejection& r : res.rejected) {
        std::snprintf(line, sizeof(line), "%-9s %5lld rejected: %s\n", to_string(r.kind), (long long)r.M,
                      r.reason.c_str());
        s << line;
    }
    s << "best: " << to_string(res.best.kind) << " M=" << res.best.M << " makespan "
      << res.best.simulated_makespan.str() << " us\n";
    if (res.dp_baseline_minibatch_time) s << "dp baseline (reported only): " << *res.dp_baseline_minibatch_time << " us\n";
    return s.str();
}

}  // namespace bapipe_b200
