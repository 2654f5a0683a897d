// bapipe_b200/explorer.hpp -- C++ drop-in for the reference's explore() path.
//
// Mirrors the public interface of /root/reference/proj/include/bapipe/
//   rational.hpp     Rat                                   (14-114)
//   errors.hpp       Error and the 7 typed exceptions       (8-46)
//   schedule_kind.hpp ScheduleKind, ExecutionMode, ...      (11-64)
//   profiles.hpp     LayerProfile ... TrainingConfig, validate_*  (24-132)
//   plan.hpp         StageAssignment, PartitionPlan         (16-28)
//   cost_models.hpp  CostEstimate                           (26-44)
//   explorer.hpp     Candidate, Rejection, ExplorationResult, explore()  (51-155)
// with the same names, fields, exception types and what() strings, in
// namespace bapipe_b200 (define BAPIPE_B200_AS_BAPIPE to alias it as
// `bapipe` for a source-level drop-in).  explore() validates exactly as the
// reference does, flattens the inputs into the SoA records of
// include/bapipe_b200.h and evaluates every candidate on the B200 through the
// C ABI (libbapipe_b200.so); results are rebuilt into the reference's types.
//
// Escaping errors are re-thrown as the reference throws them:
// std::overflow_error("Rat: overflow"), std::domain_error, InvalidPlan(<same
// message>), NoFeasiblePlan("all K candidates rejected; ...").  Where the
// reference has undefined behaviour (an out-of-bounds layer read after
// memory_fine_tune's collapse step, partition.hpp:359-373), this throws
// UndefinedInReference instead of reproducing garbage.
#pragma once

#include <algorithm>
#include <cstdint>
#include <map>
#include <numeric>
#include <optional>
#include <ostream>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

#include "../bapipe_b200.h"

namespace bapipe_b200 {

// ------------------------------------------------------------------ Rat
class Rat {
public:
    constexpr Rat() : num_(0), den_(1) {}
    constexpr Rat(std::int64_t v) : num_(v), den_(1) {}
    Rat(std::int64_t n, std::int64_t d) : num_(n), den_(d) { normalize(); }
    static Rat raw(std::int64_t n, std::int64_t d) { Rat r; r.num_ = n; r.den_ = d; return r; }

    std::int64_t num() const { return num_; }
    std::int64_t den() const { return den_; }
    bool is_integer() const { return den_ == 1; }
    double to_double() const { return double(num_) / double(den_); }
    std::string str() const { return den_ == 1 ? std::to_string(num_) : std::to_string(num_) + "/" + std::to_string(den_); }

    friend Rat operator+(const Rat& a, const Rat& b) {
        return from128((__int128)a.num_ * b.den_ + (__int128)b.num_ * a.den_, (__int128)a.den_ * b.den_);
    }
    friend Rat operator-(const Rat& a, const Rat& b) {
        return from128((__int128)a.num_ * b.den_ - (__int128)b.num_ * a.den_, (__int128)a.den_ * b.den_);
    }
    friend Rat operator*(const Rat& a, const Rat& b) { return from128((__int128)a.num_ * b.num_, (__int128)a.den_ * b.den_); }
    friend Rat operator/(const Rat& a, const Rat& b) {
        if (b.num_ == 0) throw std::domain_error("Rat: division by zero");
        return from128((__int128)a.num_ * b.den_, (__int128)a.den_ * b.num_);
    }
    Rat operator-() const { return raw(-num_, den_); }
    Rat& operator+=(const Rat& o) { return *this = *this + o; }
    Rat& operator-=(const Rat& o) { return *this = *this - o; }
    Rat& operator*=(const Rat& o) { return *this = *this * o; }
    Rat& operator/=(const Rat& o) { return *this = *this / o; }
    friend bool operator==(const Rat& a, const Rat& b) { return a.num_ == b.num_ && a.den_ == b.den_; }
    friend bool operator!=(const Rat& a, const Rat& b) { return !(a == b); }
    friend bool operator<(const Rat& a, const Rat& b) { return (__int128)a.num_ * b.den_ < (__int128)b.num_ * a.den_; }
    friend bool operator>(const Rat& a, const Rat& b) { return b < a; }
    friend bool operator<=(const Rat& a, const Rat& b) { return !(b < a); }
    friend bool operator>=(const Rat& a, const Rat& b) { return !(a < b); }
    std::int64_t floor() const { std::int64_t q = num_ / den_; return (num_ % den_ != 0 && num_ < 0) ? q - 1 : q; }
    std::int64_t ceil() const { std::int64_t q = num_ / den_; return (num_ % den_ != 0 && num_ > 0) ? q + 1 : q; }
    friend std::ostream& operator<<(std::ostream& os, const Rat& r) { return os << r.str(); }

private:
    static Rat from128(__int128 n, __int128 d) {
        if (d == 0) throw std::domain_error("Rat: zero denominator");
        if (d < 0) { n = -n; d = -d; }
        __int128 a = n < 0 ? -n : n, b = d;
        while (b != 0) { __int128 t = a % b; a = b; b = t; }
        if (a > 1) { n /= a; d /= a; }
        if (n > INT64_MAX || n < INT64_MIN || d > INT64_MAX) throw std::overflow_error("Rat: overflow");
        return raw((std::int64_t)n, (std::int64_t)d);
    }
    void normalize() {
        if (den_ == 0) throw std::domain_error("Rat: zero denominator");
        if (den_ < 0) { num_ = -num_; den_ = -den_; }
        std::int64_t g = std::gcd(num_ < 0 ? -num_ : num_, den_);
        if (g > 1) { num_ /= g; den_ /= g; }
    }
    std::int64_t num_, den_;
};

// ------------------------------------------------------------------ errors
struct Error : std::runtime_error { explicit Error(const std::string& m) : std::runtime_error(m) {} };
struct ParseError : Error { explicit ParseError(const std::string& m) : Error("parse error: " + m) {} };
struct SchemaError : Error { explicit SchemaError(const std::string& m) : Error("schema error: " + m) {} };
struct IncompatibleSchedule : Error { explicit IncompatibleSchedule(const std::string& m) : Error("incompatible schedule: " + m) {} };
struct InfeasibleShape : Error { explicit InfeasibleShape(const std::string& m) : Error("infeasible shape: " + m) {} };
struct Infeasible : Error { explicit Infeasible(const std::string& m) : Error("infeasible: " + m) {} };
struct InvalidPlan : Error { explicit InvalidPlan(const std::string& m) : Error("invalid plan: " + m) {} };
struct NoFeasiblePlan : Error { explicit NoFeasiblePlan(const std::string& m) : Error("no feasible plan: " + m) {} };
// Not in the reference: raised where the reference reads out of bounds.
struct UndefinedInReference : Error {
    explicit UndefinedInReference(const std::string& m) : Error("undefined in reference: " + m) {}
};
// Not in the reference: the CUDA path could not run (no B200, CUDA error).
struct DeviceError : Error { explicit DeviceError(const std::string& m) : Error("device error: " + m) {} };

// ------------------------------------------------------------------ schedule kinds
enum class ExecutionMode { Synchronous, Asynchronous };
enum class ScheduleKind { OneFOneB_AS, FBP_AS, OneFOneB_SNO, OneFOneB_SO };
constexpr ScheduleKind all_schedule_kinds[4] = {ScheduleKind::OneFOneB_AS, ScheduleKind::FBP_AS,
                                                ScheduleKind::OneFOneB_SNO, ScheduleKind::OneFOneB_SO};

inline const char* to_string(ScheduleKind k) {
    switch (k) {
        case ScheduleKind::OneFOneB_AS: return "1f1b-as";
        case ScheduleKind::FBP_AS: return "fbp-as";
        case ScheduleKind::OneFOneB_SNO: return "1f1b-sno";
        case ScheduleKind::OneFOneB_SO: return "1f1b-so";
    }
    return "?";
}
inline const char* to_string(ExecutionMode m) { return m == ExecutionMode::Synchronous ? "sync" : "async"; }
inline std::optional<ScheduleKind> parse_schedule_kind(const std::string& s) {
    for (ScheduleKind k : all_schedule_kinds)
        if (s == to_string(k)) return k;
    return std::nullopt;
}
inline ExecutionMode mode_of(ScheduleKind k) {
    return (k == ScheduleKind::OneFOneB_AS || k == ScheduleKind::FBP_AS) ? ExecutionMode::Asynchronous
                                                                         : ExecutionMode::Synchronous;
}
// schedule_kind.hpp:59-64
inline void check_mode(ScheduleKind k, ExecutionMode mode) {
    if (mode_of(k) != mode)
        throw IncompatibleSchedule(std::string(to_string(k)) + " requires " + to_string(mode_of(k)) +
                                   " execution, cluster is " + to_string(mode));
}
inline std::int64_t warmup_depth(ScheduleKind k, std::int64_t n_stages, std::int64_t stage) {
    std::int64_t d = n_stages - stage + 1;
    return (k == ScheduleKind::FBP_AS || k == ScheduleKind::OneFOneB_SO) ? 2 * d : d;
}
inline std::vector<ScheduleKind> feasible_kinds(ExecutionMode mode) {
    if (mode == ExecutionMode::Asynchronous) return {ScheduleKind::OneFOneB_AS, ScheduleKind::FBP_AS};
    return {ScheduleKind::OneFOneB_SNO, ScheduleKind::OneFOneB_SO};
}

// ------------------------------------------------------------------ inputs
struct LayerProfile {
    std::string name;
    std::map<std::string, std::int64_t> fp_time;
    std::map<std::string, std::int64_t> bp_time;
    std::int64_t weight_bytes = 0;
    std::int64_t out_activation_bytes = 0;
};
struct NetworkProfile {
    std::string name;
    std::vector<LayerProfile> layers;
    std::int64_t L() const { return (std::int64_t)layers.size(); }
};
struct AcceleratorSpec {
    std::string id;
    std::string accel_type;
    std::int64_t mem_capacity_bytes = 0;
    std::map<ScheduleKind, std::int64_t> min_micro_batch;
    std::int64_t min_micro(ScheduleKind k) const {
        auto it = min_micro_batch.find(k);
        return it == min_micro_batch.end() ? 1 : it->second;
    }
};
struct ClusterSpec {
    std::vector<AcceleratorSpec> accelerators;
    std::vector<std::int64_t> link_bandwidth;
    ExecutionMode execution_mode = ExecutionMode::Synchronous;
    std::int64_t N() const { return (std::int64_t)accelerators.size(); }
};
struct TrainingConfig {
    std::int64_t mini_batch_size = 1;
    std::optional<std::vector<std::int64_t>> micro_batch_candidates;
};

// synthetic fixture (profiles.hpp:316-336)
inline NetworkProfile synth_uniform_network(std::int64_t L, std::int64_t fp, std::int64_t bp, std::int64_t w,
                                            std::int64_t a, const std::vector<std::string>& accel_types,
                                            const std::string& name = "uniform") {
    if (L < 1) throw SchemaError("synth_uniform_network: L >= 1 required");
    if (fp < 1 || bp < 1) throw SchemaError("synth_uniform_network: fp, bp >= 1 required");
    NetworkProfile net;
    net.name = name;
    net.layers.resize((std::size_t)L);
    for (std::int64_t i = 0; i < L; ++i) {
        LayerProfile& l = net.layers[(std::size_t)i];
        l.name = "layer" + std::to_string(i);
        for (const std::string& t : accel_types) l.fp_time[t] = fp, l.bp_time[t] = bp;
        l.weight_bytes = w;
        l.out_activation_bytes = a;
    }
    return net;
}

// validation with the reference's messages (profiles.hpp:83-132)
inline void validate_network(const NetworkProfile& net) {
    if (net.layers.empty()) throw SchemaError("network '" + net.name + "': L >= 1 required");
    for (std::size_t i = 0; i < net.layers.size(); ++i) {
        const LayerProfile& l = net.layers[i];
        auto where = [&] { return "layer " + std::to_string(i) + " ('" + l.name + "')"; };
        if (l.fp_time.empty() || l.bp_time.empty()) throw SchemaError(where() + ": fp/bp time maps must be non-empty");
        for (auto& [t, v] : l.fp_time)
            if (v < 1) throw SchemaError(where() + ": fp time for '" + t + "' must be >= 1");
        for (auto& [t, v] : l.bp_time)
            if (v < 1) throw SchemaError(where() + ": bp time for '" + t + "' must be >= 1");
        if (l.weight_bytes < 0) throw SchemaError(where() + ": weight_bytes must be >= 0");
        if (l.out_activation_bytes < 0) throw SchemaError(where() + ": out_activation_bytes must be >= 0");
    }
}
inline void validate_cluster(const ClusterSpec& c) {
    if (c.accelerators.empty()) throw SchemaError("cluster: N >= 1 required");
    if ((std::int64_t)c.link_bandwidth.size() != c.N() - 1)
        throw SchemaError("cluster: expected N-1 links (" + std::to_string(c.N() - 1) + "), got " +
                          std::to_string(c.link_bandwidth.size()));
    for (std::size_t k = 0; k < c.link_bandwidth.size(); ++k)
        if (c.link_bandwidth[k] <= 0) throw SchemaError("link " + std::to_string(k) + ": bandwidth must be > 0");
    for (std::size_t i = 0; i < c.accelerators.size(); ++i) {
        const AcceleratorSpec& a = c.accelerators[i];
        if (a.mem_capacity_bytes <= 0)
            throw SchemaError("accelerator " + std::to_string(i) + " ('" + a.id + "'): mem_capacity_bytes must be > 0");
        for (auto& [k, v] : a.min_micro_batch)
            if (v < 1)
                throw SchemaError("accelerator '" + a.id + "': min_micro_batch[" + to_string(k) + "] must be >= 1");
    }
}
inline void validate_pair(const NetworkProfile& net, const ClusterSpec& cluster) {
    validate_network(net);
    validate_cluster(cluster);
    for (const AcceleratorSpec& a : cluster.accelerators)
        for (std::size_t i = 0; i < net.layers.size(); ++i) {
            const LayerProfile& l = net.layers[i];
            if (!l.fp_time.count(a.accel_type) || !l.bp_time.count(a.accel_type))
                throw SchemaError("layer " + std::to_string(i) + " ('" + l.name + "') lacks times for accelerator type '" +
                                  a.accel_type + "'");
        }
}
inline std::vector<std::int64_t> candidate_Ms(const TrainingConfig& cfg, const ClusterSpec& cluster, ScheduleKind kind) {
    std::vector<std::int64_t> base;
    if (cfg.micro_batch_candidates) {
        for (std::int64_t m : *cfg.micro_batch_candidates) {
            if (m < 1 || cfg.mini_batch_size % m != 0)
                throw SchemaError("micro-batch candidate " + std::to_string(m) + " does not divide mini-batch " +
                                  std::to_string(cfg.mini_batch_size));
            base.push_back(m);
        }
    } else {
        for (std::int64_t m = 1; m <= cfg.mini_batch_size; ++m)
            if (cfg.mini_batch_size % m == 0) base.push_back(m);
    }
    std::int64_t mm = 1;
    for (const AcceleratorSpec& a : cluster.accelerators) mm = std::max(mm, a.min_micro(kind));
    std::vector<std::int64_t> out;
    for (std::int64_t m : base)
        if (cfg.mini_batch_size / m >= mm) out.push_back(m);
    return out;
}

// ------------------------------------------------------------------ results
struct StageAssignment {
    std::string accelerator_id;
    std::int64_t lo = 1, hi = 1;
    Rat leading_fraction{1}, trailing_fraction{1};
};
struct PartitionPlan {
    std::vector<StageAssignment> stages;
    std::int64_t n_stages() const { return (std::int64_t)stages.size(); }
};
struct CostEstimate {
    ScheduleKind schedule = ScheduleKind::OneFOneB_AS;
    std::int64_t M = 1, N = 1;
    Rat minibatch_time{0}, bubble_fraction{0};
    std::vector<Rat> features_mem, weights_mem, bandwidth_demand;
    std::vector<bool> mem_infeasible;
    bool heuristic = false;
    bool memory_feasible() const { return std::none_of(mem_infeasible.begin(), mem_infeasible.end(), [](bool b) { return b; }); }
};
struct Candidate {
    ScheduleKind kind = ScheduleKind::OneFOneB_AS;
    std::int64_t M = 1, micro_batch_size = 1;
    PartitionPlan plan;
    Rat simulated_makespan{0};
    CostEstimate est;
    Rat peak_memory{0}, max_bandwidth_demand{0};
};
struct Rejection {
    ScheduleKind kind = ScheduleKind::OneFOneB_AS;
    std::int64_t M = 0;
    std::string reason, detail;
};
struct ExplorationResult {
    Candidate best;
    std::vector<Candidate> ranked;
    std::vector<Rejection> rejected;
    std::int64_t mini_batch_size = 1;
    std::optional<double> dp_baseline_minibatch_time;
};

// simulator.hpp:16-44
enum class EventKind { FP, BP, SEND_F, RECV_F, SEND_B, RECV_B };
inline const char* to_string(EventKind k) {
    switch (k) {
        case EventKind::FP: return "FP";
        case EventKind::BP: return "BP";
        case EventKind::SEND_F: return "SEND_F";
        case EventKind::RECV_F: return "RECV_F";
        case EventKind::SEND_B: return "SEND_B";
        case EventKind::RECV_B: return "RECV_B";
    }
    return "?";
}
struct Event {
    std::int64_t stage = 1;
    EventKind kind = EventKind::FP;
    std::int64_t micro_batch = 1;
    Rat start{0};
    Rat end{0};
};
struct Timeline {
    std::vector<Event> events;
    Rat makespan{0};
    std::vector<Rat> per_stage_feature_highwater;
    std::vector<Rat> per_stage_weight_static;
    std::vector<Rat> per_link_busy_fraction;
};

// ------------------------------------------------------------------ device context
class Explorer {
public:
    explicit Explorer(int device = 0) : ctx_(bp_create(device)) {
        if (!ctx_) throw DeviceError(bp_last_error(nullptr));
    }
    ~Explorer() { if (ctx_) bp_destroy(ctx_); }
    Explorer(const Explorer&) = delete;
    Explorer& operator=(const Explorer&) = delete;

    ExplorationResult explore(const NetworkProfile& net, const ClusterSpec& cluster, const TrainingConfig& cfg);
    // partition.hpp:441-474 for one (kind, M, micro) -- `bapipe plan`
    PartitionPlan balance_partition(const NetworkProfile& net, const ClusterSpec& cluster, ScheduleKind kind,
                                    std::int64_t M, std::int64_t micro_batch_size = 1);
    // cost_models.hpp:124-166 on a given plan
    CostEstimate estimate(ScheduleKind kind, const PartitionPlan& plan, const NetworkProfile& net,
                          const ClusterSpec& cluster, std::int64_t M, std::int64_t micro_batch_size = 1);
    // simulator.hpp:264-274: the full event timeline of a plan
    Timeline simulate(ScheduleKind kind, const PartitionPlan& plan, const NetworkProfile& net,
                      const ClusterSpec& cluster, std::int64_t M, std::int64_t micro_batch_size = 1,
                      std::int64_t mini_batches = 1);

private:
    // SoA tables of (net, cluster) on the device: network 0, cluster 0.  The
    // host copies stay alive until the next upload (an ABI implementation may
    // read them until the evaluating call returns).
    void upload(const NetworkProfile& net, const ClusterSpec& cluster);
    struct Tables {
        std::vector<std::int64_t> fp, bp, w, a, caps, mm, bw;
        std::vector<std::int32_t> types;
    } tables_;
    struct PlanBuf {
        std::vector<std::int32_t> lo, hi;
        std::vector<bp_rat> lead, trail;
    };
    static bp_plan_request plan_request(const PartitionPlan& plan, PlanBuf& buf, ScheduleKind kind,
                                        std::int64_t M, std::int64_t micro, std::int64_t mini);
    void check(int rc, const char* what) {
        if (rc != BP_OK) throw DeviceError(std::string(what) + ": " + bp_last_error(ctx_));
    }
    bp_ctx* ctx_;
};

inline Explorer& default_explorer() {
    thread_local Explorer ex(0);
    return ex;
}

// explore (explorer.hpp:80-155) on the B200.
inline ExplorationResult explore(const NetworkProfile& net, const ClusterSpec& cluster, const TrainingConfig& cfg) {
    return default_explorer().explore(net, cluster, cfg);
}
inline PartitionPlan balance_partition(const NetworkProfile& net, const ClusterSpec& cluster, ScheduleKind kind,
                                       std::int64_t M, std::int64_t micro_batch_size = 1) {
    return default_explorer().balance_partition(net, cluster, kind, M, micro_batch_size);
}
inline CostEstimate estimate(ScheduleKind kind, const PartitionPlan& plan, const NetworkProfile& net,
                             const ClusterSpec& cluster, std::int64_t M, std::int64_t micro_batch_size = 1) {
    return default_explorer().estimate(kind, plan, net, cluster, M, micro_batch_size);
}
inline Timeline simulate(ScheduleKind kind, const PartitionPlan& plan, const NetworkProfile& net,
                         const ClusterSpec& cluster, std::int64_t M, std::int64_t micro_batch_size = 1,
                         std::int64_t mini_batches = 1) {
    return default_explorer().simulate(kind, plan, net, cluster, M, micro_batch_size, mini_batches);
}
inline std::vector<Rat> memory_highwater(const Timeline& t) { return t.per_stage_feature_highwater; }

namespace detail {
inline Rat R(const bp_rat& r) { return Rat::raw(r.num, r.den); }

inline std::string invalid_plan_message(const bp_candidate& c) {
    const std::string st = "stage " + std::to_string(c.detail2);
    switch (c.detail) {
        case BP_IP_RANGE:   // the ABI carries the stage, not its [lo,hi]
            return st + ": layer range out of bounds";
        case BP_IP_FRACTION: return st + ": fractions must lie in (0, 1]";
        case BP_IP_FIRST: return "stage 1 must start at layer 1 with full ownership";
        case BP_IP_CONTIG: return st + ": not contiguous with previous stage";
        case BP_IP_SHARED_FULL: return st + ": shared boundary layer must be fractional";
        case BP_IP_LEAD_UNSHARED: return st + ": fractional lead without shared layer";
        case BP_IP_LAST: return "last stage must end at layer L with full ownership";
        case BP_IP_COVERAGE:
            return "layer " + std::to_string(c.detail2) + " coverage sums to " + R(c.aux).str() + ", expected 1";
        case BP_IP_STAGE_COUNT: return "plan stage count != cluster size";
        case BP_IP_M: return "M >= 1 required";
        default: return "invalid plan";
    }
}

// The accelerator-type lookups of stage_fp_time / stage_bp_time (plan.hpp:
// 90-108) in stage_costs / chain_instance order (cost_models.hpp:103-119,
// simulator.hpp:248-262): stage by stage, F's layers then B's.  The first
// layer without a time for its stage's type throws the reference's
// SchemaError (profiles.hpp:38-43).  The device tables hold such an entry as
// 0 and clamp non-positive times, so a plan over a layer time <= 0 (which
// validate_network rejects, profiles.hpp:83-98, but estimate / simulate do
// not check) is refused instead of computed on the wrong value.
inline void check_stage_times(const PartitionPlan& plan, const NetworkProfile& net, const ClusterSpec& cluster) {
    const std::int64_t L = net.L();
    for (std::size_t i = 0; i < plan.stages.size() && i < cluster.accelerators.size(); ++i) {
        const StageAssignment& st = plan.stages[i];
        const std::string& type = cluster.accelerators[i].accel_type;
        const std::int64_t lo = std::max<std::int64_t>(st.lo, 1), hi = std::min<std::int64_t>(st.hi, L);
        for (int which = 0; which < 2; ++which)
            for (std::int64_t j = lo; j <= hi; ++j) {
                const LayerProfile& l = net.layers[(std::size_t)j - 1];
                const auto& m = which == 0 ? l.fp_time : l.bp_time;
                auto it = m.find(type);
                if (it == m.end())
                    throw SchemaError("layer '" + l.name + "' has no " + (which == 0 ? "fp" : "bp") +
                                      " time for accelerator type '" + type + "'");
                if (it->second <= 0)
                    throw DeviceError("layer '" + l.name + "' has a non-positive " + (which == 0 ? "fp" : "bp") +
                                      " time: outside the device library's domain (validate_network requires >= 1)");
            }
    }
}

// an escaping device status as the reference throws it
[[noreturn]] inline void throw_status(int status, const std::string& invalid_plan_msg) {
    switch (status) {
        case BP_C_ERR_OVERFLOW: throw std::overflow_error("Rat: overflow");
        case BP_C_ERR_DOMAIN: throw std::domain_error("Rat: division by zero");
        case BP_C_ERR_INVALID_PLAN: throw InvalidPlan(invalid_plan_msg);
        case BP_C_REF_UB:
            throw UndefinedInReference("a plan stage reads a layer outside net.layers (plan.hpp:90-158)");
        default: throw SchemaError("plan rejected by the device library");
    }
}
}  // namespace detail

inline void Explorer::upload(const NetworkProfile& net, const ClusterSpec& cluster) {
    // SoA: global accelerator-type ids over the cluster's types and the
    // network's map keys; 0 marks a missing entry.
    std::map<std::string, int> tid;
    for (const auto& a : cluster.accelerators) tid.emplace(a.accel_type, (int)tid.size());
    for (const auto& l : net.layers) {
        for (auto& kv : l.fp_time) tid.emplace(kv.first, (int)tid.size());
        for (auto& kv : l.bp_time) tid.emplace(kv.first, (int)tid.size());
    }
    const int T = (int)tid.size(), L = (int)net.L(), N = (int)cluster.N();
    Tables& tb = tables_;
    tb.fp.assign((std::size_t)T * L, 0);
    tb.bp.assign((std::size_t)T * L, 0);
    tb.w.assign(L, 0);
    tb.a.assign(L, 0);
    auto &fp = tb.fp, &bp = tb.bp, &w = tb.w, &a = tb.a;
    for (int j = 0; j < L; ++j) {
        const LayerProfile& l = net.layers[j];
        for (auto& [t, v] : l.fp_time) fp[(std::size_t)tid[t] * L + j] = v;
        for (auto& [t, v] : l.bp_time) bp[(std::size_t)tid[t] * L + j] = v;
        w[j] = l.weight_bytes;
        a[j] = l.out_activation_bytes;
    }
    tb.types.assign(N, 0);
    tb.caps.assign(N, 0);
    tb.mm.assign((std::size_t)N * 4, 0);
    tb.bw = cluster.link_bandwidth;
    auto &types = tb.types;
    auto &caps = tb.caps, &mm = tb.mm, &bw = tb.bw;
    for (int i = 0; i < N; ++i) {
        types[i] = tid[cluster.accelerators[i].accel_type];
        caps[i] = cluster.accelerators[i].mem_capacity_bytes;
        for (int k = 0; k < 4; ++k) mm[(std::size_t)i * 4 + k] = cluster.accelerators[i].min_micro(all_schedule_kinds[k]);
    }
    if (bw.empty()) bw.push_back(1);
    bp_network bn{L, T, fp.data(), bp.data(), w.data(), a.data()};
    bp_cluster bc{N, cluster.execution_mode == ExecutionMode::Asynchronous ? BP_MODE_ASYNC : BP_MODE_SYNC,
                  types.data(), caps.data(), mm.data(), bw.data()};
    check(bp_set_networks(ctx_, &bn, 1), "bp_set_networks");
    check(bp_set_clusters(ctx_, &bc, 1), "bp_set_clusters");
}

inline ExplorationResult Explorer::explore(const NetworkProfile& net, const ClusterSpec& cluster,
                                           const TrainingConfig& cfg) {
    // the reference's own validation order (explorer.hpp:82-83, 87-89)
    validate_pair(net, cluster);
    if (cfg.mini_batch_size < 1) throw SchemaError("mini_batch_size >= 1 required");
    for (ScheduleKind k : feasible_kinds(cluster.execution_mode)) (void)candidate_Ms(cfg, cluster, k);
    // an explicit empty list yields no candidates (the ABI reads n_m == 0 as
    // "all divisors", so this case is answered here, as explorer.hpp:135-141)
    if (cfg.micro_batch_candidates && cfg.micro_batch_candidates->empty())
        throw NoFeasiblePlan("all 0 candidates rejected");
    upload(net, cluster);
    const int N = (int)cluster.N();
    std::vector<std::int64_t> mlist;
    bp_query q{};
    q.network = 0;
    q.cluster = 0;
    q.n_stages = N;
    q.mini_batch = cfg.mini_batch_size;
    if (cfg.micro_batch_candidates) {
        mlist = *cfg.micro_batch_candidates;
        q.n_m = (std::int32_t)mlist.size();
        q.m_list = mlist.data();
    }
    std::int64_t ncand = 0, nst = 0;
    check(bp_layout(ctx_, &q, 1, &ncand, &nst), "bp_layout");
    bp_query_result res{};
    std::vector<bp_candidate> cand((std::size_t)std::max<std::int64_t>(ncand, 1));
    std::vector<bp_stage> stg((std::size_t)std::max<std::int64_t>(nst, 1));
    check(bp_explore_batch(ctx_, &q, 1, &res, cand.data(), stg.data(), nullptr), "bp_explore_batch");

    ExplorationResult out;
    out.mini_batch_size = cfg.mini_batch_size;
    std::vector<std::pair<int, Candidate>> ranked;
    for (std::int64_t i = 0; i < ncand; ++i) {
        const bp_candidate& c = cand[(std::size_t)i];
        const ScheduleKind kind = all_schedule_kinds[c.kind];
        if (c.status == BP_C_OK) {
            Candidate x;
            x.kind = kind;
            x.M = c.M;
            x.micro_batch_size = c.micro;
            x.simulated_makespan = detail::R(c.makespan);
            x.peak_memory = detail::R(c.peak_memory);
            x.max_bandwidth_demand = detail::R(c.max_bw_demand);
            x.est.schedule = kind;
            x.est.M = c.M;
            x.est.N = N;
            x.est.minibatch_time = detail::R(c.est_minibatch);
            x.est.bubble_fraction = detail::R(c.bubble);
            x.est.heuristic = c.heuristic != 0;
            const bp_stage* s = stg.data() + i * N;
            for (int k = 0; k < N; ++k) {
                StageAssignment sa;
                sa.accelerator_id = cluster.accelerators[k].id;
                sa.lo = s[k].lo;
                sa.hi = s[k].hi;
                sa.leading_fraction = detail::R(s[k].lead);
                sa.trailing_fraction = detail::R(s[k].trail);
                x.plan.stages.push_back(sa);
                x.est.features_mem.push_back(detail::R(s[k].features));
                x.est.weights_mem.push_back(detail::R(s[k].weights));
                x.est.mem_infeasible.push_back(false);   // every ranked candidate passed the memory check
                if (k + 1 < N) x.est.bandwidth_demand.push_back(detail::R(s[k].bw_demand));
            }
            ranked.emplace_back(c.rank, std::move(x));
            continue;
        }
        Rejection r;
        r.kind = kind;
        r.M = c.M;
        switch (c.status) {
            case BP_C_REJ_MIN_MICRO:
                r.reason = "min_micro_batch";
                r.detail = "micro-batch size " + std::to_string(c.micro) + " below minimum";
                break;
            case BP_C_REJ_COARSEN:
                r.reason = "memory";
                r.detail = Infeasible("coarsening for communication leaves " + std::to_string(c.detail) + " blocks for " +
                                      std::to_string(N) + " stages").what();
                break;
            case BP_C_REJ_FINETUNE:
                r.reason = "memory";
                r.detail = Infeasible(std::string("no contiguous plan satisfies memory for ") + to_string(kind) +
                                      ", M=" + std::to_string(c.M)).what();
                break;
            case BP_C_REJ_FINETUNE_NOCONV:
                r.reason = "memory";
                r.detail = Infeasible("memory fine-tune did not converge").what();
                break;
            case BP_C_REJ_SHAPE:
                r.reason = "partition";
                r.detail = InfeasibleShape(std::to_string(c.detail) + " partition units for " + std::to_string(N) +
                                           " stages").what();
                break;
            case BP_C_REJ_MEM_POST:
                r.reason = "memory";
                r.detail = "plan exceeds capacity";
                break;
            default:
                continue;   // escaping errors: decided by the query status below
        }
        out.rejected.push_back(std::move(r));
    }
    switch (res.status) {
        case BP_Q_OK: break;
        case BP_Q_OVERFLOW: throw std::overflow_error("Rat: overflow");
        case BP_Q_DOMAIN: throw std::domain_error("Rat: division by zero");
        case BP_Q_INVALID_PLAN: throw InvalidPlan(detail::invalid_plan_message(cand[(std::size_t)res.first_error]));
        case BP_Q_REF_UB:
            throw UndefinedInReference("memory_fine_tune's collapse step leaves a stage reading net.layers[-1] "
                                       "(partition.hpp:359-373, plan.hpp:136-139)");
        case BP_Q_NO_FEASIBLE: {
            std::ostringstream why;
            why << "all " << out.rejected.size() << " candidates rejected";
            for (const Rejection& r : out.rejected) why << "; " << to_string(r.kind) << " M=" << r.M << ": " << r.reason;
            throw NoFeasiblePlan(why.str());
        }
        default: throw SchemaError("query rejected by the device library");
    }
    std::sort(ranked.begin(), ranked.end(), [](const auto& x, const auto& y) { return x.first < y.first; });
    for (auto& kv : ranked) out.ranked.push_back(std::move(kv.second));
    out.best = out.ranked.front();
    return out;
}

inline bp_plan_request Explorer::plan_request(const PartitionPlan& plan, PlanBuf& buf, ScheduleKind kind,
                                              std::int64_t M, std::int64_t micro, std::int64_t mini) {
    for (const StageAssignment& st : plan.stages) {
        buf.lo.push_back((std::int32_t)std::max<std::int64_t>(INT32_MIN, std::min<std::int64_t>(INT32_MAX, st.lo)));
        buf.hi.push_back((std::int32_t)std::max<std::int64_t>(INT32_MIN, std::min<std::int64_t>(INT32_MAX, st.hi)));
        buf.lead.push_back(bp_rat{st.leading_fraction.num(), st.leading_fraction.den()});
        buf.trail.push_back(bp_rat{st.trailing_fraction.num(), st.trailing_fraction.den()});
    }
    bp_plan_request q{};
    q.network = 0;
    q.cluster = 0;
    q.kind = (std::int32_t)kind;
    q.n_stages = (std::int32_t)plan.stages.size();
    q.M = M;
    q.micro = micro;
    q.mini_batches = mini;
    q.lo = buf.lo.data();
    q.hi = buf.hi.data();
    q.lead = buf.lead.data();
    q.trail = buf.trail.data();
    return q;
}

inline PartitionPlan Explorer::balance_partition(const NetworkProfile& net, const ClusterSpec& cluster,
                                                 ScheduleKind kind, std::int64_t M, std::int64_t micro) {
    check_mode(kind, cluster.execution_mode);   // partition.hpp:443-444
    validate_pair(net, cluster);
    // the device enumerates (kind, M) candidates of a mini-batch M * micro
    if (M < 1 || micro < 1) throw SchemaError("balance_partition: M >= 1 and micro-batch size >= 1 required");
    upload(net, cluster);
    const int N = (int)cluster.N();
    std::int64_t mlist[1] = {M};
    bp_query q{};
    q.n_stages = N;
    q.mini_batch = M * micro;
    q.n_m = 1;
    q.m_list = mlist;
    std::int64_t ncand = 0, nst = 0;
    check(bp_layout(ctx_, &q, 1, &ncand, &nst), "bp_layout");
    bp_query_result res{};
    std::vector<bp_candidate> cand((std::size_t)std::max<std::int64_t>(ncand, 1));
    std::vector<bp_stage> stg((std::size_t)std::max<std::int64_t>(nst, 1));
    check(bp_set_option(ctx_, BP_OPT_PLAN_ONLY, 1), "bp_set_option");
    const int rc = bp_explore_batch(ctx_, &q, 1, &res, cand.data(), stg.data(), nullptr);
    bp_set_option(ctx_, BP_OPT_PLAN_ONLY, 0);
    check(rc, "bp_explore_batch");
    const std::vector<ScheduleKind> kinds = feasible_kinds(cluster.execution_mode);
    const std::size_t slot = (std::size_t)(std::find(kinds.begin(), kinds.end(), kind) - kinds.begin());
    const bp_candidate& c = cand[slot];
    switch (c.status) {
        case BP_C_OK: {
            PartitionPlan plan;
            const bp_stage* st = stg.data() + slot * (std::size_t)N;
            for (int k = 0; k < N; ++k) {
                StageAssignment sa;
                sa.accelerator_id = cluster.accelerators[k].id;
                sa.lo = st[k].lo;
                sa.hi = st[k].hi;
                sa.leading_fraction = detail::R(st[k].lead);
                sa.trailing_fraction = detail::R(st[k].trail);
                plan.stages.push_back(sa);
            }
            return plan;
        }
        case BP_C_REJ_COARSEN:
            throw Infeasible("coarsening for communication leaves " + std::to_string(c.detail) + " blocks for " +
                             std::to_string(N) + " stages");
        case BP_C_REJ_FINETUNE:
            throw Infeasible(std::string("no contiguous plan satisfies memory for ") + to_string(kind) +
                             ", M=" + std::to_string(M));
        case BP_C_REJ_FINETUNE_NOCONV: throw Infeasible("memory fine-tune did not converge");
        case BP_C_REJ_SHAPE:
            throw InfeasibleShape(std::to_string(c.detail) + " partition units for " + std::to_string(N) + " stages");
        case BP_C_REJ_MEM_POST:
            // a balanced plan whose final estimate is over capacity: memory_fine_tune
            // only returns plans within capacity, so this is not reached
            throw Infeasible("memory");
        default: detail::throw_status(c.status, detail::invalid_plan_message(c));
    }
}

inline CostEstimate Explorer::estimate(ScheduleKind kind, const PartitionPlan& plan, const NetworkProfile& net,
                                       const ClusterSpec& cluster, std::int64_t M, std::int64_t micro) {
    check_mode(kind, cluster.execution_mode);   // cost_models.hpp:127-129
    if (plan.n_stages() != cluster.N()) throw InvalidPlan("plan stage count != cluster size");
    detail::check_stage_times(plan, net, cluster);   // stage_costs' lookups (cost_models.hpp:103-119)
    upload(net, cluster);
    PlanBuf buf;
    const bp_plan_request q = plan_request(plan, buf, kind, M, micro, 1);
    const std::size_t N = plan.stages.size();
    bp_estimate_result r{};
    std::vector<bp_stage> st(N);
    std::vector<std::int32_t> inf(N);
    check(bp_estimate_plan(ctx_, &q, &r, st.data(), inf.data()), "bp_estimate_plan");
    if (r.status != BP_C_OK) detail::throw_status(r.status, "");
    CostEstimate e;
    e.schedule = kind;
    e.M = M;
    e.N = (std::int64_t)N;
    e.minibatch_time = detail::R(r.minibatch_time);
    e.bubble_fraction = detail::R(r.bubble_fraction);
    e.heuristic = r.heuristic != 0;
    for (std::size_t i = 0; i < N; ++i) {
        e.features_mem.push_back(detail::R(st[i].features));
        e.weights_mem.push_back(detail::R(st[i].weights));
        e.mem_infeasible.push_back(inf[i] != 0);
        if (i + 1 < N) e.bandwidth_demand.push_back(detail::R(st[i].bw_demand));
    }
    return e;
}

inline Timeline Explorer::simulate(ScheduleKind kind, const PartitionPlan& plan, const NetworkProfile& net,
                                   const ClusterSpec& cluster, std::int64_t M, std::int64_t micro,
                                   std::int64_t mini_batches) {
    check_mode(kind, cluster.execution_mode);   // simulator.hpp:268
    if (plan.stages.empty()) throw InvalidPlan("plan has no stages");
    upload(net, cluster);
    PlanBuf buf;
    // mini_batches < 1: the reference simulates one mini-batch, emits no
    // events and reports Rat(mini_batches) * makespan (simulator.hpp:182-216)
    const std::int64_t mb = std::max<std::int64_t>(mini_batches, 1);
    const bp_plan_request q = plan_request(plan, buf, kind, M, micro, mb);
    const std::int64_t N = plan.n_stages(), Mp = std::max<std::int64_t>(M, 0);
    const std::int64_t cap = mb * (2 * N * Mp + 4 * (N - 1) * Mp);
    std::vector<bp_event> ev((std::size_t)std::max<std::int64_t>(cap, 1));
    std::vector<bp_rat> hw((std::size_t)N), ws((std::size_t)N), busy((std::size_t)std::max<std::int64_t>(N - 1, 1));
    bp_timeline_result r{};
    check(bp_simulate_plan(ctx_, &q, &r, ev.data(), cap, hw.data(), ws.data(), busy.data()), "bp_simulate_plan");
    // chain_instance's type lookups come after validate_plan and the stage
    // count check (simulator.hpp:268-273)
    if (r.status != BP_C_ERR_INVALID_PLAN) detail::check_stage_times(plan, net, cluster);
    if (r.status != BP_C_OK) {
        std::string msg;
        if (r.status == BP_C_ERR_INVALID_PLAN) {
            bp_candidate c{};
            c.detail = r.detail;
            c.detail2 = r.detail2;
            c.aux = r.aux;
            msg = detail::invalid_plan_message(c);
            if (r.detail == BP_IP_RANGE) {   // the plan is at hand: the reference's full message
                const StageAssignment& st = plan.stages[(std::size_t)r.detail2 - 1];
                msg = "stage " + std::to_string(r.detail2) + ": layer range [" + std::to_string(st.lo) + "," +
                      std::to_string(st.hi) + "] out of bounds";
            }
        }
        detail::throw_status(r.status, msg);
    }
    Timeline t;
    t.makespan = detail::R(r.makespan);
    if (mini_batches < 1) {
        t.makespan = Rat(mini_batches) * t.makespan;
        r.n_events = 0;
    }
    t.events.reserve((std::size_t)r.n_events);
    for (std::int64_t i = 0; i < r.n_events; ++i) {
        const bp_event& x = ev[(std::size_t)i];
        t.events.push_back({x.stage, (EventKind)x.kind, x.micro_batch, detail::R(x.start), detail::R(x.end)});
    }
    for (std::int64_t s = 0; s < N; ++s) {
        t.per_stage_feature_highwater.push_back(detail::R(hw[(std::size_t)s]));
        t.per_stage_weight_static.push_back(detail::R(ws[(std::size_t)s]));
    }
    for (std::int64_t k = 0; k + 1 < N; ++k) t.per_link_busy_fraction.push_back(detail::R(busy[(std::size_t)k]));
    return t;
}

}  // namespace bapipe_b200

#ifdef BAPIPE_B200_AS_BAPIPE
namespace bapipe = bapipe_b200;
#endif
