// Tail latency and the latency-bounded-throughput searches (reference
// metrics.hpp:22-209). tail_latency() selects on the device; the LBT and
// GPU(max) drivers advance every design's bracket/bisection in lockstep and
// evaluate each round's (design x seed) simulations as one device grid, which
// reproduces the reference's per-design rate sequence exactly.
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <limits>
#include <map>
#include <numeric>
#include <string>
#include <vector>

#include "device.hpp"
#include "engine.hpp"
#include "errors.hpp"
#include "grid.hpp"
#include "paris.hpp"
#include "profile.hpp"
#include "sched.hpp"
#include "workload.hpp"

namespace migserve {

// Nearest rank: the ceil(p*n)-th smallest sample (metrics.hpp:22-29).
inline double tail_latency(std::vector<double> samples, double p = 0.95) {
    if (samples.empty()) throw ParamError("tail_latency: no samples");
    if (!(p > 0.0) || !(p < 1.0)) throw ParamError("tail_latency: percentile must be in (0,1)");
    double out = 0.0;
    device::check(msv_tail_latency(device::context().get(), samples.data(), static_cast<int64_t>(samples.size()),
                                   &p, 1, &out),
                  "tail_latency");
    return out;
}

inline double derive_sla_target(const ProfileTable& table, int b_max, double multiplier) {
    if (!(multiplier > 0.0)) throw ParamError("derive_sla_target: multiplier must be > 0");
    return multiplier * table.latency_ms(table.max_size(), b_max);
}

struct LbtOptions {
    double duration_ms = 20000.0;
    std::vector<uint64_t> seeds = {1, 2, 3};
    double rel_tol = 0.01;
    double tail_p = 0.95;
    double lambda_min = 1.0;
    double warmup_fraction = 0.1;
    int max_doublings = 24;
};

struct LbtResult {
    double qps = 0.0;
    bool infeasible_at_min = false;
    int sims_run = 0;
};

namespace detail {

// Grid cells of one rate probe: one per seed, in seed order.
inline void append_probe(std::vector<GridCell>& cells, const PartitionPlan& plan, SchedulerKind scheduler,
                         const ProfileTable& table, const SlaConfig& cfg, const BatchDistribution& dist, double rate,
                         const LbtOptions& opt) {
    for (uint64_t seed : opt.seeds) {
        GridCell c;
        c.plan = &plan;
        c.scheduler = scheduler;
        c.table = &table;
        c.dist = &dist;
        c.sla = cfg;
        c.rate_qps = rate;
        c.duration_ms = opt.duration_ms;
        c.seed = seed;
        c.warmup_fraction = opt.warmup_fraction;
        cells.push_back(c);
    }
}

// Mean of the per-seed tails, seeds with no measured query skipped (metrics.hpp:57-75).
inline double mean_of_probe(const std::vector<GridCellResult>& res, std::size_t first, std::size_t count) {
    double sum = 0.0;
    int used = 0;
    for (std::size_t j = 0; j < count; ++j) {
        const GridCellResult& r = res[first + j];
        if (r.measured_queries == 0) continue;
        sum += r.tails[0];
        ++used;
    }
    return used == 0 ? 0.0 : sum / static_cast<double>(used);
}

inline double mean_tail_at_rate(const PartitionPlan& plan, SchedulerKind scheduler, const ProfileTable& table,
                                const SlaConfig& cfg, const BatchDistribution& dist, double rate_qps,
                                const LbtOptions& opt, int& sims) {
    std::vector<GridCell> cells;
    append_probe(cells, plan, scheduler, table, cfg, dist, rate_qps, opt);
    const std::vector<GridCellResult> res = run_grid(cells, {opt.tail_p});
    sims += static_cast<int>(opt.seeds.size());
    return mean_of_probe(res, 0, opt.seeds.size());
}

// One design's latency_bounded_throughput (metrics.hpp:81-120) as a resumable state
// machine: pending() is the next rate to evaluate, feed() consumes its mean tail.
struct LbtSearch {
    enum Phase { Min, Double, Bisect, Done };
    const PartitionPlan* plan;
    SchedulerKind scheduler;
    const ProfileTable* table;
    SlaConfig cfg;
    const BatchDistribution* dist;
    LbtOptions opt;
    Phase phase = Min;
    double lo = 0.0, hi = 0.0, mid = 0.0, rate = 0.0;
    int doublings = 0;
    LbtResult result;

    void start() {
        if (!(cfg.sla_target_ms > 0.0)) throw ParamError("latency_bounded_throughput: sla must be > 0");
        if (opt.seeds.empty()) throw ParamError("latency_bounded_throughput: need at least one seed");
        phase = Min;
        rate = opt.lambda_min;
    }
    bool done() const { return phase == Done; }
    void next_double() {
        if (doublings < opt.max_doublings) {
            hi *= 2.0;
            rate = hi;
            phase = Double;
        } else {
            result.qps = lo;  // effectively unbounded within the probe range
            phase = Done;
        }
    }
    void next_bisect() {
        if ((hi - lo) / lo > opt.rel_tol) {
            mid = 0.5 * (lo + hi);
            rate = mid;
            phase = Bisect;
        } else {
            result.qps = lo;
            phase = Done;
        }
    }
    void feed(double tail) {
        result.sims_run += static_cast<int>(opt.seeds.size());
        const double sla = cfg.sla_target_ms;
        switch (phase) {
            case Min:
                if (tail > sla) {
                    result.infeasible_at_min = true;
                    phase = Done;
                    return;
                }
                lo = hi = opt.lambda_min;
                doublings = 0;
                next_double();
                return;
            case Double:
                if (tail > sla) {
                    next_bisect();
                    return;
                }
                lo = hi;
                ++doublings;
                next_double();
                return;
            case Bisect:
                if (tail <= sla) lo = mid;
                else hi = mid;
                next_bisect();
                return;
            case Done: return;
        }
    }
};

// Advance all searches together. Each round is one device grid over the rates of every
// active search's next kLbtLookahead steps — its outcome tree: node k's children are
// 2k+1 (the probe met the SLA) and 2k+2 (it did not) — all independent simulations;
// the tree is then walked with the measured tails, so each search takes exactly the
// reference's probes and rates (metrics.hpp:81-120) in kLbtLookahead times fewer rounds.
constexpr int kLbtLookahead = 3;

inline void run_lockstep(std::vector<LbtSearch>& searches) {
    for (LbtSearch& s : searches) s.start();
    for (;;) {
        std::vector<GridCell> cells;
        struct Probe {
            std::size_t search;
            int node;
            std::size_t first;
        };
        std::vector<Probe> probes;
        for (std::size_t i = 0; i < searches.size(); ++i) {
            if (searches[i].done()) continue;
            std::vector<std::pair<int, LbtSearch>> level{{0, searches[i]}};
            for (int d = 0; d < kLbtLookahead && !level.empty(); ++d) {
                std::vector<std::pair<int, LbtSearch>> next;
                for (auto& [k, st] : level) {
                    if (st.done()) continue;
                    probes.push_back({i, k, cells.size()});
                    append_probe(cells, *st.plan, st.scheduler, *st.table, st.cfg, *st.dist, st.rate, st.opt);
                    LbtSearch ok = st, bad = st;
                    ok.feed(-std::numeric_limits<double>::infinity());
                    bad.feed(std::numeric_limits<double>::infinity());
                    next.emplace_back(2 * k + 1, std::move(ok));
                    next.emplace_back(2 * k + 2, std::move(bad));
                }
                level = std::move(next);
            }
        }
        if (probes.empty()) return;
        // one grid per distinct tail_p
        std::vector<GridCellResult> res(cells.size());
        std::vector<double> ps;
        for (const Probe& pr : probes)
            if (std::find(ps.begin(), ps.end(), searches[pr.search].opt.tail_p) == ps.end())
                ps.push_back(searches[pr.search].opt.tail_p);
        for (double p : ps) {
            std::vector<GridCell> sub;
            std::vector<std::size_t> where;
            for (const Probe& pr : probes) {
                const LbtSearch& s = searches[pr.search];
                if (s.opt.tail_p != p) continue;
                for (std::size_t q = 0; q < s.opt.seeds.size(); ++q) {
                    sub.push_back(cells[pr.first + q]);
                    where.push_back(pr.first + q);
                }
            }
            const std::vector<GridCellResult> r = run_grid(sub, {p});
            for (std::size_t q = 0; q < r.size(); ++q) res[where[q]] = r[q];
        }
        std::map<std::pair<std::size_t, int>, std::size_t> at;
        for (const Probe& pr : probes) at[{pr.search, pr.node}] = pr.first;
        for (std::size_t i = 0; i < searches.size(); ++i) {
            LbtSearch& s = searches[i];
            int node = 0;
            while (!s.done()) {
                auto it = at.find({i, node});
                if (it == at.end()) break;
                const double tail = mean_of_probe(res, it->second, s.opt.seeds.size());
                const double sla = s.cfg.sla_target_ms;  // the branch feed() takes
                const bool bad = s.phase == LbtSearch::Bisect ? !(tail <= sla) : tail > sla;
                s.feed(tail);
                node = 2 * node + (bad ? 2 : 1);
            }
        }
    }
}

}  // namespace detail

// Largest arrival rate whose mean tail stays within the SLA: double from lambda_min,
// then bisect to rel_tol (metrics.hpp:81-120).
inline LbtResult latency_bounded_throughput(const PartitionPlan& plan, SchedulerKind scheduler,
                                            const ProfileTable& table, const SlaConfig& cfg,
                                            const BatchDistribution& dist, const LbtOptions& opt = {}) {
    std::vector<detail::LbtSearch> s(1);
    s[0].plan = &plan;
    s[0].scheduler = scheduler;
    s[0].table = &table;
    s[0].cfg = cfg;
    s[0].dist = &dist;
    s[0].opt = opt;
    detail::run_lockstep(s);
    return s[0].result;
}

struct DesignPoint {
    std::string label;
    SchedulerKind scheduler = SchedulerKind::Fifs;
    PartitionPlan plan;
    std::vector<uint64_t> seeds;
    LbtResult lbt;
    double tail_ms_at_rate = 0.0;
    double rate_qps = 0.0;
};

struct ComparisonRow {
    std::string label;
    double lbt_qps = 0.0;
    double tail_ms = 0.0;
    double norm_lbt = 0.0;
    double norm_tail = 0.0;
};

inline constexpr const char* kBaselineLabel = "gpu(7)+fifs";

// Normalise every design against gpu(7)+fifs (metrics.hpp:146-173).
inline std::vector<ComparisonRow> compare(const std::vector<DesignPoint>& designs) {
    if (designs.empty()) throw ParamError("compare: no designs");
    for (const DesignPoint& d : designs)
        if (d.seeds != designs.front().seeds) throw ValidationError("compare: designs ran different workload seeds");
    const auto base = std::find_if(designs.begin(), designs.end(),
                                   [](const DesignPoint& d) { return d.label == kBaselineLabel; });
    if (base == designs.end())
        throw ValidationError(std::string("compare: normalization baseline ") + kBaselineLabel + " absent");
    std::vector<ComparisonRow> rows;
    for (const DesignPoint& d : designs) {
        ComparisonRow r;
        r.label = d.label;
        r.lbt_qps = d.lbt.qps;
        r.tail_ms = d.tail_ms_at_rate;
        r.norm_lbt = base->lbt.qps > 0.0 ? d.lbt.qps / base->lbt.qps : 0.0;
        r.norm_tail = base->tail_ms_at_rate > 0.0 ? d.tail_ms_at_rate / base->tail_ms_at_rate : 0.0;
        rows.push_back(r);
    }
    return rows;
}

struct BestHomogeneous {
    int k = 0;
    PartitionPlan plan;
    LbtResult lbt;
};

// GPU(max): LBT of every homogeneous size under FIFS, all searches in lockstep on
// the device; the first strictly larger rate wins in ascending k (metrics.hpp:183-209).
inline BestHomogeneous best_homogeneous(const ProfileTable& table, const BatchDistribution& dist,
                                        const SlaConfig& cfg, int total_gpcs, int num_gpus, int gpcs_per_gpu,
                                        const LbtOptions& opt = {}) {
    std::vector<int> ks;
    std::vector<PartitionPlan> plans;
    for (int k : table.sizes()) {
        if (k > gpcs_per_gpu || k > total_gpcs) continue;
        ks.push_back(k);
        plans.push_back(homogeneous_plan(k, total_gpcs, num_gpus, gpcs_per_gpu));
    }
    if (ks.empty()) throw InfeasibleError("best_homogeneous: no size fits the server");
    std::vector<detail::LbtSearch> searches;
    std::vector<std::size_t> search_of(ks.size(), static_cast<std::size_t>(-1));
    for (std::size_t i = 0; i < ks.size(); ++i) {
        if (plans[i].total_instances() == 0) continue;
        detail::LbtSearch s;
        s.plan = &plans[i];
        s.scheduler = SchedulerKind::Fifs;
        s.table = &table;
        s.cfg = cfg;
        s.dist = &dist;
        s.opt = opt;
        search_of[i] = searches.size();
        searches.push_back(s);
    }
    detail::run_lockstep(searches);
    BestHomogeneous best;
    for (std::size_t i = 0; i < ks.size(); ++i) {
        const LbtResult r = search_of[i] == static_cast<std::size_t>(-1) ? LbtResult{} : searches[search_of[i]].result;
        if (best.k == 0 || r.qps > best.lbt.qps) {
            best.k = ks[i];
            best.plan = plans[i];
            best.lbt = r;
        }
    }
    return best;
}

}  // namespace migserve
