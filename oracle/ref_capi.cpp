// TEST INFRASTRUCTURE ONLY — the reference oracle.
//
// Compiles the reference's own headers, unmodified, from where they lie
// (/root/reference/proj/include/migserve, header-only C++20) and exposes them
// through the checker ABI in oracle_abi.h plus a few reference-only entry points
// (PARIS planning, LBT, GPU(max), single dispatch decisions) used to generate the
// golden fixtures under tests/golden/. Built by oracle/build_oracle.py into
// oracle/_ref/libmsv_ref.so (git-ignored, travels to the GPU box in the snapshot).
// Nothing in the product links this library.
#include <algorithm>
#include <atomic>
#include <cstring>
#include <exception>
#include <string>
#include <thread>
#include <vector>

// Everything the reference headers include, first, with normal access rules...
#include <charconv>
#include <cmath>
#include <compare>
#include <cstdint>
#include <deque>
#include <fstream>
#include <future>
#include <istream>
#include <limits>
#include <map>
#include <numeric>
#include <optional>
#include <ostream>
#include <queue>
#include <random>
#include <sstream>
#include <stdexcept>
#include <utility>

#include <json.hpp>
// ...then the reference headers themselves: BatchDistribution / ProfileTable keep
// their cdf and grids private and the fixtures need them verbatim.
#define private public
#include <migserve/engine.hpp>
#include <migserve/metrics.hpp>
#include <migserve/paris.hpp>
#include <migserve/profile.hpp>
#include <migserve/sched.hpp>
#include <migserve/workload.hpp>
#undef private

#include "oracle_abi.h"

using namespace migserve;

namespace {
thread_local std::string g_err;

int code_of_current_exception() {
    try {
        throw;
    } catch (const ParamError& e) {
        g_err = e.what();
        return 1;
    } catch (const FormatError& e) {
        g_err = e.what();
        return 2;
    } catch (const ValidationError& e) {
        g_err = e.what();
        return 3;
    } catch (const LookupError& e) {
        g_err = e.what();
        return 4;
    } catch (const InfeasibleError& e) {
        g_err = e.what();
        return 5;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 7;
    }
}

ProfileTable make_table(const ora_profile* p) {
    const size_t cells = static_cast<size_t>(p->n_sizes) * static_cast<size_t>(p->b_max);
    return ProfileTable("oracle", std::vector<int>(p->sizes, p->sizes + p->n_sizes), p->b_max,
                        std::vector<double>(p->lat, p->lat + cells), std::vector<double>(p->util, p->util + cells));
}

BatchDistribution make_dist(const ora_dist* d) {
    return BatchDistribution(std::vector<double>(d->weights, d->weights + d->b_max));
}

PartitionPlan make_plan(const ora_plan* p) {
    PartitionPlan plan;
    plan.num_gpus = p->num_gpus;
    plan.gpcs_per_gpu = p->gpcs_per_gpu;
    size_t off = 0;
    for (int g = 0; g < p->num_gpus; ++g) {
        plan.gpus.emplace_back(p->sizes_flat + off, p->sizes_flat + off + p->n_per_gpu[g]);
        off += static_cast<size_t>(p->n_per_gpu[g]);
    }
    return plan;
}

void fill_plan(const PartitionPlan& plan, int32_t* n_per_gpu, int32_t* flat) {
    size_t off = 0;
    for (size_t g = 0; g < plan.gpus.size(); ++g) {
        n_per_gpu[g] = static_cast<int32_t>(plan.gpus[g].size());
        for (int k : plan.gpus[g]) flat[off++] = k;
    }
}
}  // namespace

extern "C" {

const char* ora_last_error(void) { return g_err.c_str(); }
const char* ora_kind(void) { return "reference"; }

int ora_dist_tables(const ora_dist* d, double* pmf, double* cdf) {
    try {
        BatchDistribution bd = make_dist(d);
        std::copy(bd.pmf_.begin(), bd.pmf_.end(), pmf);
        std::copy(bd.cdf_.begin(), bd.cdf_.end(), cdf);
        return 0;
    } catch (...) {
        return code_of_current_exception();
    }
}

int64_t ora_sample_trace(const ora_dist* d, double rate_qps, double duration_ms, uint64_t seed, int64_t cap,
                         double* arrival, int32_t* batch) {
    try {
        QueryTrace t = sample_trace(make_dist(d), rate_qps, duration_ms, seed);
        const int64_t n = static_cast<int64_t>(t.queries.size());
        for (int64_t i = 0; i < n && i < cap; ++i) {
            arrival[i] = t.queries[static_cast<size_t>(i)].arrival_ms;
            batch[i] = t.queries[static_cast<size_t>(i)].batch;
        }
        return n;
    } catch (...) {
        return -code_of_current_exception();
    }
}

static int run_impl(const ora_plan* plan_in, int scheduler, const double* arrival, const int32_t* batch, int64_t n,
                    double duration_ms, const ora_profile* prof, double sla, double alpha, double beta,
                    double warmup_fraction, int check_wait, int n_route, const int32_t* route_k,
                    const int32_t* route_first, const int32_t* route_last, ora_records* rec, ora_report* rep,
                    double noise_sigma, uint64_t noise_seed) {
    try {
        PartitionPlan plan = make_plan(plan_in);
        ProfileTable table = make_table(prof);
        QueryTrace trace;
        trace.duration_ms = duration_ms;
        for (int64_t i = 0; i < n; ++i) trace.queries.push_back(Query{i, arrival[i], batch[i]});
        EngineOptions opt;
        opt.warmup_fraction = warmup_fraction;
        opt.check_wait_consistency = check_wait != 0;
        opt.noise_sigma = noise_sigma;
        opt.noise_seed = noise_seed;
        if (n_route > 0) {
            opt.segment_routing = true;
            for (int j = 0; j < n_route; ++j)
                opt.routing_segments.push_back(BatchSegment{PartitionSize{route_k[j]}, route_first[j], route_last[j]});
        } else if (n_route == 0 && route_k) {
            opt.segment_routing = true;  // enabled without segments: ParamError path
        }
        SimReport r = run(plan, scheduler ? SchedulerKind::Elsa : SchedulerKind::Fifs, trace, table,
                          SlaConfig{sla, alpha, beta}, opt);
        if (rec) {
            for (int64_t i = 0; i < n; ++i) {
                const QueryRecord& q = r.queries[static_cast<size_t>(i)];
                rec->partition[i] = q.partition_id;
                rec->start_ms[i] = q.start_ms;
                rec->finish_ms[i] = q.finish_ms;
                rec->kind[i] = static_cast<int32_t>(q.kind);
            }
        }
        if (rep) {
            rep->total = r.total_queries;
            rep->violations = r.violations;
            rep->measured = r.measured_queries;
            rep->measured_violations = r.measured_violations;
            rep->horizon_ms = r.horizon_ms;
            rep->warmup_ms = r.warmup_ms;
            rep->max_wait_estimate_diff = r.max_wait_estimate_diff;
            for (size_t p = 0; p < r.partitions.size(); ++p) {
                if (rep->busy_ms) rep->busy_ms[p] = r.partitions[p].busy_ms;
                if (rep->weighted_busy_ms) rep->weighted_busy_ms[p] = r.partitions[p].weighted_busy_ms;
                if (rep->queries) rep->queries[p] = r.partitions[p].queries;
            }
        }
        return 0;
    } catch (...) {
        return code_of_current_exception();
    }
}

int ora_run(const ora_plan* plan_in, int scheduler, const double* arrival, const int32_t* batch, int64_t n,
            double duration_ms, const ora_profile* prof, double sla, double alpha, double beta,
            double warmup_fraction, int check_wait, int n_route, const int32_t* route_k, const int32_t* route_first,
            const int32_t* route_last, ora_records* rec, ora_report* rep) {
    return run_impl(plan_in, scheduler, arrival, batch, n, duration_ms, prof, sla, alpha, beta, warmup_fraction,
                    check_wait, n_route, route_k, route_first, route_last, rec, rep, 0.0, 1);
}

// run() with EngineOptions::noise_sigma / noise_seed (engine.hpp:140-145): the reference only.
int oraref_run_noise(const ora_plan* plan_in, int scheduler, const double* arrival, const int32_t* batch, int64_t n,
                     double duration_ms, const ora_profile* prof, double sla, double alpha, double beta,
                     double warmup_fraction, int n_route, const int32_t* route_k, const int32_t* route_first,
                     const int32_t* route_last, double noise_sigma, uint64_t noise_seed, ora_records* rec,
                     ora_report* rep) {
    return run_impl(plan_in, scheduler, arrival, batch, n, duration_ms, prof, sla, alpha, beta, warmup_fraction, 0,
                    n_route, route_k, route_first, route_last, rec, rep, noise_sigma, noise_seed);
}

int ora_tail_latency(const double* samples, int64_t n, double p, double* out) {
    try {
        *out = tail_latency(std::vector<double>(samples, samples + n), p);
        return 0;
    } catch (...) {
        return code_of_current_exception();
    }
}

// CPU baseline / grid oracle: the reference's own sample_trace -> run ->
// latency_samples -> tail_latency per scenario, scenarios pulled from an atomic
// counter by n_threads std::threads (the reference itself only parallelises
// best_homogeneous, metrics.hpp:187-198).
int ora_run_grid(const ora_profile* profs, const ora_dist* dists, const ora_plan* plans, const ora_scenario* sc,
                 int64_t n, const double* ps, int n_p, int n_threads, ora_result* out) {
    int64_t max_prof = -1, max_dist = -1, max_plan = -1;
    for (int64_t i = 0; i < n; ++i) {
        max_prof = std::max<int64_t>(max_prof, sc[i].profile);
        max_dist = std::max<int64_t>(max_dist, sc[i].dist);
        max_plan = std::max<int64_t>(max_plan, sc[i].plan);
    }
    std::vector<ProfileTable> tables;
    std::vector<BatchDistribution> ds;
    std::vector<PartitionPlan> pls;
    try {
        for (int64_t i = 0; i <= max_prof; ++i) tables.push_back(make_table(&profs[i]));
        for (int64_t i = 0; i <= max_dist; ++i) ds.push_back(make_dist(&dists[i]));
        for (int64_t i = 0; i <= max_plan; ++i) pls.push_back(make_plan(&plans[i]));
    } catch (...) {
        return code_of_current_exception();
    }
    std::atomic<int64_t> next{0};
    auto worker = [&]() {
        for (;;) {
            const int64_t i = next.fetch_add(1);
            if (i >= n) return;
            const ora_scenario& s = sc[i];
            ora_result& r = out[i];
            std::memset(&r, 0, sizeof r);
            try {
                QueryTrace t = sample_trace(ds[static_cast<size_t>(s.dist)], s.rate_qps, s.duration_ms, s.seed);
                EngineOptions eng;
                eng.warmup_fraction = s.warmup_fraction;
                SimReport rep = run(pls[static_cast<size_t>(s.plan)], s.scheduler ? SchedulerKind::Elsa : SchedulerKind::Fifs,
                                    t, tables[static_cast<size_t>(s.profile)], SlaConfig{s.sla_ms, s.alpha, s.beta}, eng);
                r.total = rep.total_queries;
                r.violations = rep.violations;
                r.measured = rep.measured_queries;
                r.measured_violations = rep.measured_violations;
                r.horizon_ms = rep.horizon_ms;
                uint64_t h = 0;
                for (const QueryRecord& q : rep.queries)
                    h += ora_query_digest(static_cast<uint64_t>(q.id), q.partition_id, q.start_ms, q.finish_ms);
                r.placement_hash = h;
                std::vector<double> samples = rep.latency_samples();
                for (int j = 0; j < 4; ++j) r.tail[j] = __builtin_nan("");
                if (!samples.empty())
                    for (int j = 0; j < n_p && j < 4; ++j) r.tail[j] = tail_latency(samples, ps[j]);
            } catch (...) {
                r.status = code_of_current_exception();
            }
        }
    };
    if (n_threads <= 1) {
        worker();
    } else {
        std::vector<std::thread> pool;
        for (int t = 0; t < n_threads; ++t) pool.emplace_back(worker);
        for (std::thread& th : pool) th.join();
    }
    return 0;
}

// ---- reference-only entry points (fixtures for the host planning headers) ----

int oraref_synth_profile(double w, double f, double g, double u, const int32_t* sizes, int n_sizes, int b_max,
                         int32_t* sizes_out, int* n_out, double* lat, double* util) {
    try {
        ProfileTable t = synth_profile(SyntheticProfileParams{w, f, g, u}, std::vector<int>(sizes, sizes + n_sizes), b_max);
        *n_out = static_cast<int>(t.sizes().size());
        std::copy(t.sizes().begin(), t.sizes().end(), sizes_out);
        std::copy(t.latency_.begin(), t.latency_.end(), lat);
        std::copy(t.util_.begin(), t.util_.end(), util);
        return 0;
    } catch (...) {
        return code_of_current_exception();
    }
}

int oraref_lognormal_pdf(double mu, double sigma, int b_max, double* pmf, double* cdf) {
    try {
        BatchDistribution d = lognormal_batch_pdf(mu, sigma, b_max);
        std::copy(d.pmf_.begin(), d.pmf_.end(), pmf);
        std::copy(d.cdf_.begin(), d.cdf_.end(), cdf);
        return 0;
    } catch (...) {
        return code_of_current_exception();
    }
}

int oraref_paris_plan(const ora_profile* prof, const ora_dist* d, int total_gpcs, int num_gpus, int gpcs_per_gpu,
                      double knee_threshold, int32_t* knees, double* ratios, double* counts, int32_t* n_per_gpu,
                      int32_t* flat) {
    try {
        ParisResult r = paris_plan(make_table(prof), make_dist(d), total_gpcs, num_gpus, gpcs_per_gpu, knee_threshold);
        size_t i = 0;
        for (const auto& kv : r.knees) knees[i++] = kv.second;
        for (size_t j = 0; j < r.ratios.entries.size(); ++j) ratios[j] = r.ratios.entries[j].ratio;
        for (size_t j = 0; j < r.counts.counts.size(); ++j) counts[j] = r.counts.counts[j].second;
        fill_plan(r.plan, n_per_gpu, flat);
        return 0;
    } catch (...) {
        return code_of_current_exception();
    }
}

int oraref_homogeneous_plan(int k, int total_gpcs, int num_gpus, int gpcs_per_gpu, int32_t* n_per_gpu, int32_t* flat) {
    try {
        fill_plan(homogeneous_plan(k, total_gpcs, num_gpus, gpcs_per_gpu), n_per_gpu, flat);
        return 0;
    } catch (...) {
        return code_of_current_exception();
    }
}

int oraref_lbt(const ora_plan* plan, int scheduler, const ora_profile* prof, double sla, double alpha, double beta,
               const ora_dist* d, double duration_ms, const uint64_t* seeds, int n_seeds, double rel_tol, double tail_p,
               double lambda_min, double warmup_fraction, int max_doublings, double* qps, int* infeasible, int* sims) {
    try {
        LbtOptions opt;
        opt.duration_ms = duration_ms;
        opt.seeds.assign(seeds, seeds + n_seeds);
        opt.rel_tol = rel_tol;
        opt.tail_p = tail_p;
        opt.lambda_min = lambda_min;
        opt.warmup_fraction = warmup_fraction;
        opt.max_doublings = max_doublings;
        LbtResult r = latency_bounded_throughput(make_plan(plan), scheduler ? SchedulerKind::Elsa : SchedulerKind::Fifs,
                                                 make_table(prof), SlaConfig{sla, alpha, beta}, make_dist(d), opt);
        *qps = r.qps;
        *infeasible = r.infeasible_at_min ? 1 : 0;
        *sims = r.sims_run;
        return 0;
    } catch (...) {
        return code_of_current_exception();
    }
}

int oraref_best_homogeneous(const ora_profile* prof, const ora_dist* d, double sla, double alpha, double beta,
                            int total_gpcs, int num_gpus, int gpcs_per_gpu, double duration_ms, const uint64_t* seeds,
                            int n_seeds, int* k_out, double* qps) {
    try {
        LbtOptions opt;
        opt.duration_ms = duration_ms;
        opt.seeds.assign(seeds, seeds + n_seeds);
        BestHomogeneous b = best_homogeneous(make_table(prof), make_dist(d), SlaConfig{sla, alpha, beta}, total_gpcs,
                                             num_gpus, gpcs_per_gpu, opt);
        *k_out = b.k;
        *qps = b.lbt.qps;
        return 0;
    } catch (...) {
        return code_of_current_exception();
    }
}

// Single dispatch decisions: elsa_dispatch / fifs_dispatch / t_wait (sched.hpp:77-174).
int oraref_dispatch(const ora_profile* prof, int scheduler, int P, const int32_t* id, const int32_t* k,
                    const uint8_t* busy, const double* cur_est, const double* cur_start, const int64_t* q_off,
                    const int32_t* qbatch, int query_batch, double now, double sla, double alpha, double beta,
                    int32_t* chosen, int32_t* kind, double* t_wait_out) {
    try {
        ProfileTable table = make_table(prof);
        std::vector<PartitionState> parts;
        for (int j = 0; j < P; ++j) {
            PartitionState s;
            s.id = id[j];
            s.k = PartitionSize{k[j]};
            if (busy[j]) s.current = RunningQuery{1000 + j, 1, cur_est[j], cur_start[j]};
            for (int64_t q = q_off[j]; q < q_off[j + 1]; ++q)
                s.queued.push_back(QueuedQuery{2000 + q, qbatch[q], 0.0});
            parts.push_back(std::move(s));
        }
        Query qu{1, now, query_batch};
        Dispatch dsp = scheduler ? elsa_dispatch(qu, parts, table, SlaConfig{sla, alpha, beta}, now)
                                 : fifs_dispatch(qu, parts);
        *chosen = dsp.partition_id;
        *kind = static_cast<int32_t>(dsp.kind);
        if (t_wait_out)
            for (int j = 0; j < P; ++j) t_wait_out[j] = t_wait(parts[static_cast<size_t>(j)], table, now);
        return 0;
    } catch (...) {
        return code_of_current_exception();
    }
}

}  // extern "C"
