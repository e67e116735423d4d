// Batch entry point of the B200 engine (new in this build; the reference runs one
// simulation per call): a grid of independent (plan x profile x dist x rate x seed
// x scheduler) cells, each = sample_trace -> run -> tail_latency(latency_samples())
// (workload.hpp:97-113, engine.hpp:115-253, metrics.hpp:22-29), executed by the
// device in one launch sequence (msv_run_grid). The reference's own search drivers
// (metrics.hpp) are rebuilt on top of it.
#pragma once

#include <cstdint>
#include <map>
#include <vector>

#include "device.hpp"
#include "engine.hpp"
#include "paris.hpp"
#include "profile.hpp"
#include "sched.hpp"
#include "workload.hpp"

namespace migserve {

struct GridCell {
    const PartitionPlan* plan = nullptr;
    SchedulerKind scheduler = SchedulerKind::Elsa;
    const ProfileTable* table = nullptr;
    const BatchDistribution* dist = nullptr;
    SlaConfig sla;
    double rate_qps = 0.0;
    double duration_ms = 0.0;
    uint64_t seed = 0;
    double warmup_fraction = 0.1;
};

struct GridCellResult {
    int64_t total_queries = 0;
    int64_t violations = 0;
    int64_t measured_queries = 0;
    int64_t measured_violations = 0;
    std::vector<double> tails;  // per requested percentile; NaN when nothing was measured
    double horizon_ms = 0.0;
    uint64_t placement_hash = 0;  // sum over queries of msv_query_digest(id, partition, start, finish)
};

inline std::vector<GridCellResult> run_grid(const std::vector<GridCell>& cells,
                                            const std::vector<double>& tail_ps = {0.95, 0.99}) {
    if (tail_ps.size() > 4) throw ParamError("run_grid: at most 4 tail percentiles");
    msv_ctx* ctx = device::context().get();
    std::map<const PartitionPlan*, int> plan_handles;
    std::vector<msv_scenario> sc(cells.size());
    for (std::size_t i = 0; i < cells.size(); ++i) {
        const GridCell& c = cells[i];
        if (!c.plan || !c.table || !c.dist) throw ParamError("run_grid: cell without plan/table/dist");
        auto it = plan_handles.find(c.plan);
        if (it == plan_handles.end()) it = plan_handles.emplace(c.plan, detail::upload_plan(ctx, *c.plan)).first;
        msv_scenario& s = sc[i];
        s.profile = c.table->device_handle();
        s.dist = c.dist->device_handle();
        s.plan = it->second;
        s.scheduler = c.scheduler == SchedulerKind::Elsa ? MSV_ELSA : MSV_FIFS;
        s.routing = -1;
        s.flags = 0;
        s.sla_ms = c.sla.sla_target_ms;
        s.alpha = c.sla.alpha;
        s.beta = c.sla.beta;
        s.rate_qps = c.rate_qps;
        s.duration_ms = c.duration_ms;
        s.warmup_fraction = c.warmup_fraction;
        s.seed = c.seed;
    }
    std::vector<msv_result> res(cells.size());
    if (!cells.empty())
        device::check(msv_run_grid(ctx, sc.data(), static_cast<int64_t>(sc.size()), tail_ps.data(),
                                   static_cast<int>(tail_ps.size()), res.data(), nullptr),
                      "run_grid");
    std::vector<GridCellResult> out(cells.size());
    for (std::size_t i = 0; i < cells.size(); ++i) {
        GridCellResult& o = out[i];
        o.total_queries = res[i].total;
        o.violations = res[i].violations;
        o.measured_queries = res[i].measured;
        o.measured_violations = res[i].measured_violations;
        o.tails.assign(res[i].tail, res[i].tail + tail_ps.size());
        o.horizon_ms = res[i].horizon_ms;
        o.placement_hash = res[i].placement_hash;
    }
    return out;
}

}  // namespace migserve
