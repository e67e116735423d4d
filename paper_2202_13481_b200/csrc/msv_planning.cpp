// C ABI exports of the host-side planning headers (include/migserve/paris.hpp),
// for bindings that cannot include C++ headers (the Python package, bench.py).
#include <algorithm>
#include <cmath>
#include <exception>
#include <map>
#include <string>
#include <vector>

#include "../../include/migserve/paris.hpp"
#include "../../include/migserve/rng.hpp"
#include "../../include/msv.h"

namespace migserve_capi {
int set_error(int code, const char* what);
}

namespace {
thread_local std::string g_plan_err;

int map_exception() {
    try {
        throw;
    } catch (const migserve::ParamError& e) {
        return migserve_capi::set_error(MSV_PARAM, e.what());
    } catch (const migserve::FormatError& e) {
        return migserve_capi::set_error(MSV_FORMAT, e.what());
    } catch (const migserve::ValidationError& e) {
        return migserve_capi::set_error(MSV_VALIDATION, e.what());
    } catch (const migserve::LookupError& e) {
        return migserve_capi::set_error(MSV_LOOKUP, e.what());
    } catch (const migserve::InfeasibleError& e) {
        return migserve_capi::set_error(MSV_INFEASIBLE, e.what());
    } catch (const std::exception& e) {
        return migserve_capi::set_error(MSV_PARAM, e.what());
    }
}
}  // namespace

extern "C" int msv_paris_plan(int n_sizes, const int32_t* sizes, int b_max, const double* latency_ms,
                              const double* utilization, const double* dist_weights, int total_gpcs, int num_gpus,
                              int gpcs_per_gpu, double knee_threshold, int32_t* n_per_gpu, int32_t* sizes_flat) {
    try {
        if (n_sizes < 1 || b_max < 1 || !sizes || !latency_ms || !utilization || !dist_weights)
            throw migserve::ParamError("msv_paris_plan: empty profile");
        const std::size_t cells = static_cast<std::size_t>(n_sizes) * static_cast<std::size_t>(b_max);
        migserve::ProfileTable table("capi", std::vector<int>(sizes, sizes + n_sizes), b_max,
                                     std::vector<double>(latency_ms, latency_ms + cells),
                                     std::vector<double>(utilization, utilization + cells));
        migserve::BatchDistribution dist(std::vector<double>(dist_weights, dist_weights + b_max));
        const migserve::ParisResult r =
            migserve::paris_plan(table, dist, total_gpcs, num_gpus, gpcs_per_gpu, knee_threshold);
        std::size_t off = 0;
        for (int g = 0; g < num_gpus; ++g) {
            const std::vector<int>& gpu = r.plan.gpus[static_cast<std::size_t>(g)];
            n_per_gpu[g] = static_cast<int32_t>(gpu.size());
            for (int k : gpu) sizes_flat[off++] = k;
        }
        return MSV_OK;
    } catch (...) {
        return map_exception();
    }
}

// synth_profile (profile.hpp:183-215) through the C++ host headers. sizes_out /
// latency / utilization must hold n_sizes and n_sizes * b_max entries.
extern "C" int msv_synth_profile(double work_per_sample, double fixed_overhead, double parallelism_per_sample,
                                 double util_cap, int n_sizes, const int32_t* sizes, int b_max, int32_t* n_out,
                                 int32_t* sizes_out, double* latency_ms, double* utilization) {
    try {
        const migserve::ProfileTable t = migserve::synth_profile(
            migserve::SyntheticProfileParams{work_per_sample, fixed_overhead, parallelism_per_sample, util_cap},
            std::vector<int>(sizes, sizes + std::max(n_sizes, 0)), b_max);
        *n_out = static_cast<int32_t>(t.sizes().size());
        for (std::size_t i = 0; i < t.sizes().size(); ++i) sizes_out[i] = t.sizes()[i];
        for (std::size_t c = 0; c < t.latency_grid().size(); ++c) {
            latency_ms[c] = t.latency_grid()[c];
            utilization[c] = t.utilization_grid()[c];
        }
        return MSV_OK;
    } catch (...) {
        return map_exception();
    }
}

// lognormal_batch_pdf (workload.hpp:81-93): normalised pmf and cdf.
extern "C" int msv_lognormal_pdf(double mu, double sigma, int b_max, double* pmf, double* cdf) {
    try {
        const migserve::BatchDistribution d = migserve::lognormal_batch_pdf(mu, sigma, b_max);
        for (int b = 0; b < d.b_max(); ++b) {
            pmf[b] = d.pmf()[static_cast<std::size_t>(b)];
            cdf[b] = d.cdf()[static_cast<std::size_t>(b)];
        }
        return MSV_OK;
    } catch (...) {
        return map_exception();
    }
}

// The noise multiplier stream of run() (engine.hpp:140-145), drawn with the reference's
// Rng (rng.hpp) and this host's libm exp/log/cos/sqrt (the reference's own calls).
extern "C" int msv_noise_multipliers(uint64_t seed, double sigma, int64_t n, double* out) {
    if (n < 0 || (n > 0 && !out)) return migserve_capi::set_error(MSV_PARAM, "noise_multipliers: bad arguments");
    migserve::Rng rng(seed);
    for (int64_t j = 0; j < n; ++j) {
        const double z = rng.normal();
        out[j] = std::exp(sigma * z - 0.5 * sigma * sigma);
    }
    return MSV_OK;
}
