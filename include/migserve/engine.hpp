// Discrete-event simulation of a MIG-partitioned inference server — the same
// API as the reference's engine.hpp (engine.hpp:23-313). run() executes on the
// device (msv_run_replay -> the K2 simulation kernel): one warp simulates the trace
// with one partition per lane slot, reproducing the reference's event order,
// placements and timings bit for bit. Report formatting (CSV/JSON) stays on the host.
#pragma once

#include <algorithm>
#include <charconv>
#include <cmath>
#include <cstdint>
#include <numeric>
#include <ostream>
#include <string>
#include <utility>
#include <vector>

#include <json.hpp>

#include "device.hpp"
#include "errors.hpp"
#include "paris.hpp"
#include "profile.hpp"
#include "sched.hpp"
#include "workload.hpp"

namespace migserve {

enum class SchedulerKind { Fifs, Elsa };

inline const char* to_string(SchedulerKind s) { return s == SchedulerKind::Fifs ? "fifs" : "elsa"; }

inline SchedulerKind scheduler_from_string(const std::string& name) {
    if (name == "fifs") return SchedulerKind::Fifs;
    if (name == "elsa") return SchedulerKind::Elsa;
    throw ValidationError("unknown scheduler '" + name + "' (expected fifs or elsa)");
}

struct EngineOptions {
    double warmup_fraction = 0.1;
    double noise_sigma = 0.0;  // lognormal execution noise, 0 = exact (engine.hpp:37-38)
    uint64_t noise_seed = 1;
    bool check_wait_consistency = false;
    bool segment_routing = false;
    std::vector<BatchSegment> routing_segments;
};

struct QueryRecord {
    int64_t id = 0;
    double arrival_ms = 0.0;
    int batch = 1;
    int partition_id = -1;
    double start_ms = 0.0;
    double finish_ms = 0.0;
    double latency_ms = 0.0;
    bool sla_met = true;
    DispatchKind kind = DispatchKind::SlackSatisfying;
};

struct PartitionUsage {
    int id = 0;
    int k = 0;
    double busy_ms = 0.0;
    double weighted_busy_ms = 0.0;
    int64_t queries = 0;
};

struct SimReport {
    std::vector<QueryRecord> queries;  // trace order
    std::vector<PartitionUsage> partitions;
    double duration_ms = 0.0;
    double horizon_ms = 0.0;
    double warmup_ms = 0.0;
    SlaConfig sla;
    SchedulerKind scheduler = SchedulerKind::Fifs;
    uint64_t trace_seed = 0;
    double noise_sigma = 0.0;
    int64_t total_queries = 0;
    int64_t violations = 0;
    int64_t measured_queries = 0;
    int64_t measured_violations = 0;
    double max_wait_estimate_diff = 0.0;

    std::vector<double> latency_samples() const {
        std::vector<double> out;
        out.reserve(queries.size());
        for (const QueryRecord& q : queries)
            if (q.arrival_ms >= warmup_ms) out.push_back(q.latency_ms);
        return out;
    }
};

namespace detail {

// Plan upload for the current context (plans are plain structs, uploaded per call).
inline int upload_plan(msv_ctx* ctx, const PartitionPlan& plan) {
    std::vector<int32_t> counts, flat;
    for (const auto& g : plan.gpus) {
        counts.push_back(static_cast<int32_t>(g.size()));
        flat.insert(flat.end(), g.begin(), g.end());
    }
    int32_t h = -1;
    device::check(msv_upload_plan(ctx, plan.num_gpus, plan.gpcs_per_gpu, counts.data(), flat.data(), &h),
                  "msv_upload_plan");
    return h;
}

inline int upload_routing(msv_ctx* ctx, const std::vector<BatchSegment>& segs) {
    std::vector<int32_t> k, first, last;
    for (const BatchSegment& s : segs) {
        k.push_back(s.k.gpcs);
        first.push_back(s.first);
        last.push_back(s.last);
    }
    int32_t h = -1;
    device::check(msv_upload_routing(ctx, static_cast<int>(segs.size()), k.data(), first.data(), last.data(), &h),
                  "msv_upload_routing");
    return h;
}

// The reference's up-front argument checks, in its order (engine.hpp:118-124).
inline void check_run_args(const PartitionPlan& plan, const SlaConfig& cfg, const EngineOptions& options) {
    plan.validate();
    cfg.validate();
    if (plan.total_instances() == 0) throw ParamError("run: plan has no partition instances");
    if (options.warmup_fraction < 0.0 || options.warmup_fraction >= 1.0)
        throw ParamError("run: warmup_fraction must be in [0,1)");
    if (options.segment_routing && options.routing_segments.empty())
        throw ParamError("run: segment_routing enabled without segments");
}

}  // namespace detail

// One deterministic simulation of (plan, scheduler, trace) on the device.
inline SimReport run(const PartitionPlan& plan, SchedulerKind scheduler, const QueryTrace& trace,
                     const ProfileTable& table, const SlaConfig& cfg, const EngineOptions& options = {}) {
    detail::check_run_args(plan, cfg, options);
    msv_ctx* ctx = device::context().get();
    const std::size_t n = trace.queries.size();
    // The reference's event heap serves arrivals by (time, trace index); a stable sort
    // reproduces that order for traces that are not already sorted.
    std::vector<std::size_t> order(n);
    std::iota(order.begin(), order.end(), std::size_t{0});
    bool sorted = true;
    for (std::size_t i = 1; i < n; ++i)
        if (trace.queries[i].arrival_ms < trace.queries[i - 1].arrival_ms) sorted = false;
    if (!sorted)
        std::stable_sort(order.begin(), order.end(), [&](std::size_t a, std::size_t b) {
            return trace.queries[a].arrival_ms < trace.queries[b].arrival_ms;
        });
    std::vector<double> arr(n);
    std::vector<int32_t> bat(n);
    for (std::size_t j = 0; j < n; ++j) {
        arr[j] = trace.queries[order[j]].arrival_ms;
        bat[j] = trace.queries[order[j]].batch;
    }
    msv_scenario s{};
    s.profile = table.device_handle();
    s.dist = -1;
    s.plan = detail::upload_plan(ctx, plan);
    s.scheduler = scheduler == SchedulerKind::Elsa ? MSV_ELSA : MSV_FIFS;
    s.routing = options.segment_routing ? detail::upload_routing(ctx, options.routing_segments) : -1;
    s.flags = options.check_wait_consistency ? MSV_FLAG_CHECK_WAIT : 0;
    s.sla_ms = cfg.sla_target_ms;
    s.alpha = cfg.alpha;
    s.beta = cfg.beta;
    s.rate_qps = 0.0;
    s.duration_ms = trace.duration_ms;
    s.warmup_fraction = options.warmup_fraction;
    s.seed = trace.seed;
    const int64_t offsets[2] = {0, static_cast<int64_t>(n)};
    msv_result res{};
    const std::vector<PartitionSize> sizes = plan.flatten();
    std::vector<msv_usage> usage(sizes.size());
    std::vector<msv_record> rec(std::max<std::size_t>(n, 1));
    if (options.noise_sigma > 0.0) {
        // Execution noise (engine.hpp:140-145): the j-th query started runs for
        // est * exp(sigma*z_j - sigma^2/2), z_j the j-th Rng(noise_seed).normal(). The
        // multipliers are an input stream (drawn here with the reference's Rng and libm,
        // n of them: every query starts once); the device starts queries in the global
        // event order, so query j-th-started takes multiplier j (msv_noise.cu).
        Rng noise_rng(options.noise_seed);
        std::vector<double> mult(std::max<std::size_t>(n, 1));
        for (std::size_t j = 0; j < n; ++j) {
            const double z = noise_rng.normal();
            mult[j] = std::exp(options.noise_sigma * z - 0.5 * options.noise_sigma * options.noise_sigma);
        }
        device::check(msv_run_noise(ctx, &s, static_cast<int64_t>(n), arr.data(), bat.data(), mult.data(), &res,
                                    usage.data(), rec.data()),
                      "run");
    } else {
        device::check(msv_run_replay(ctx, &s, 1, offsets, arr.data(), bat.data(), nullptr, 0, &res, usage.data(),
                                     rec.data()),
                      "run");
    }
    SimReport rep;
    rep.queries.resize(n);
    for (std::size_t j = 0; j < n; ++j) {
        const Query& q = trace.queries[order[j]];
        QueryRecord& r = rep.queries[order[j]];
        r.id = q.id;
        r.arrival_ms = q.arrival_ms;
        r.batch = q.batch;
        r.partition_id = rec[j].partition;
        r.start_ms = rec[j].start_ms;
        r.finish_ms = rec[j].finish_ms;
        r.latency_ms = r.finish_ms - r.arrival_ms;
        r.sla_met = r.latency_ms <= cfg.sla_target_ms;
        r.kind = static_cast<DispatchKind>(rec[j].kind);
    }
    for (std::size_t p = 0; p < sizes.size(); ++p)
        rep.partitions.push_back(PartitionUsage{static_cast<int>(p), sizes[p].gpcs, usage[p].busy_ms,
                                                usage[p].weighted_busy_ms, usage[p].queries});
    rep.duration_ms = trace.duration_ms;
    rep.horizon_ms = res.horizon_ms;
    rep.warmup_ms = res.warmup_ms;
    rep.sla = cfg;
    rep.scheduler = scheduler;
    rep.trace_seed = trace.seed;
    rep.noise_sigma = options.noise_sigma;
    rep.total_queries = res.total;
    rep.violations = res.violations;
    rep.measured_queries = res.measured;
    rep.measured_violations = res.measured_violations;
    rep.max_wait_estimate_diff = res.max_wait_estimate_diff;
    return rep;
}

// Utilisation-weighted busy time over the horizon (engine.hpp:257-262).
inline double busy_fraction(const SimReport& report, int partition_id) {
    for (const PartitionUsage& u : report.partitions)
        if (u.id == partition_id) return report.horizon_ms > 0.0 ? u.weighted_busy_ms / report.horizon_ms : 0.0;
    throw LookupError("busy_fraction: unknown partition " + std::to_string(partition_id));
}

inline double busy_time_fraction(const SimReport& report, int partition_id) {
    for (const PartitionUsage& u : report.partitions)
        if (u.id == partition_id) return report.horizon_ms > 0.0 ? u.busy_ms / report.horizon_ms : 0.0;
    throw LookupError("busy_time_fraction: unknown partition " + std::to_string(partition_id));
}

// Shortest round-trip decimal (std::to_chars), so CSVs are byte-stable.
inline std::string format_double(double v) {
    char buf[32];
    const auto r = std::to_chars(buf, buf + sizeof buf, v);
    return std::string(buf, r.ptr);
}

inline void write_query_csv(const SimReport& report, std::ostream& out) {
    out << "id,arrival_ms,partition,start_ms,finish_ms,latency_ms,sla_met\n";
    for (const QueryRecord& q : report.queries)
        out << q.id << ',' << format_double(q.arrival_ms) << ',' << q.partition_id << ','
            << format_double(q.start_ms) << ',' << format_double(q.finish_ms) << ','
            << format_double(q.latency_ms) << ',' << (q.sla_met ? 1 : 0) << '\n';
}

inline nlohmann::json report_to_json(const SimReport& report) {
    nlohmann::json parts = nlohmann::json::array();
    const double h = report.horizon_ms;
    for (const PartitionUsage& u : report.partitions)
        parts.push_back({{"id", u.id},
                         {"k", u.k},
                         {"queries", u.queries},
                         {"busy_time_fraction", h > 0.0 ? u.busy_ms / h : 0.0},
                         {"weighted_utilization", h > 0.0 ? u.weighted_busy_ms / h : 0.0}});
    return nlohmann::json{{"scheduler", to_string(report.scheduler)},
                          {"seed", report.trace_seed},
                          {"duration_ms", report.duration_ms},
                          {"horizon_ms", report.horizon_ms},
                          {"warmup_ms", report.warmup_ms},
                          {"noise_sigma", report.noise_sigma},
                          {"sla",
                           {{"target_ms", report.sla.sla_target_ms},
                            {"alpha", report.sla.alpha},
                            {"beta", report.sla.beta}}},
                          {"totals",
                           {{"queries", report.total_queries},
                            {"violations", report.violations},
                            {"measured_queries", report.measured_queries},
                            {"measured_violations", report.measured_violations}}},
                          {"partitions", parts}};
}

}  // namespace migserve
