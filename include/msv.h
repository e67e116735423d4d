/*
 * msv.h — C ABI of the B200 scenario-grid engine (libmsv.so).
 *
 * The reference (arXiv 2202.13481's `migserve`, /root/reference/proj/include/migserve)
 * is a header-only C++20 library with no FFI layer. This header is the thin C boundary
 * its hot path crosses in this build: the C++ host headers in include/migserve/ (same
 * names and signatures as the reference) and the Python package call these entry points,
 * and everything behind them runs as sm_100a CUDA kernels. Each entry point names the
 * reference interface it replaces.
 *
 * Conventions
 *   - Every function returns an msv_status; 0 is success. Codes 1..5 mirror the
 *     reference's exception taxonomy (errors.hpp:16-40) one-to-one so wrappers can
 *     rethrow the same C++ type; 6 is a CUDA/NCCL failure. The message of the last
 *     failure on the calling thread is available from msv_last_error().
 *   - Plain C types only; buffers are caller-owned host memory unless stated.
 *   - A context owns one CUDA device, its device memory and its stream. Distinct
 *     contexts may be used concurrently from distinct threads; one context must not
 *     be used from two threads at once. Multi-GPU runs use one process (and one
 *     context) per GPU — see INTEGRATION.md.
 *   - Handles (profile, dist, plan, routing) are small non-negative ints, valid for
 *     the lifetime of the context.
 */
#ifndef MSV_H
#define MSV_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MSV_ABI_VERSION 1

typedef enum {
    MSV_OK = 0,
    MSV_PARAM = 1,      /* migserve::ParamError      (errors.hpp:16) */
    MSV_FORMAT = 2,     /* migserve::FormatError     (errors.hpp:22) */
    MSV_VALIDATION = 3, /* migserve::ValidationError (errors.hpp:28) */
    MSV_LOOKUP = 4,     /* migserve::LookupError     (errors.hpp:33) */
    MSV_INFEASIBLE = 5, /* migserve::InfeasibleError (errors.hpp:38) */
    MSV_CUDA = 6        /* device / driver / NCCL failure (no reference analogue) */
} msv_status;

typedef enum { MSV_FIFS = 0, MSV_ELSA = 1 } msv_scheduler; /* engine.hpp:23 SchedulerKind */

typedef enum { /* DispatchKind, sched.hpp:50-55 */
    MSV_SLACK_SATISFYING = 0,
    MSV_FASTEST_FALLBACK = 1,
    MSV_IDLE_LARGEST = 2,
    MSV_SHORTEST_QUEUE = 3
} msv_dispatch_kind;

typedef enum { MSV_LOG1P_AUTO = -1, MSV_LOG1P_GENERIC_BUILD = 0, MSV_LOG1P_FMA_BUILD = 1 } msv_log1p_variant;

/* Scenario flags */
#define MSV_FLAG_CHECK_WAIT 1 /* EngineOptions::check_wait_consistency (engine.hpp:39) */

typedef struct msv_ctx msv_ctx;

/* One simulation cell: (plan x profile x dist x rate x seed x scheduler).
 * Replaces the argument list of run() (engine.hpp:115-117) plus sample_trace()
 * (workload.hpp:97-98) when the trace is generated on the device. 80 bytes. */
typedef struct {
    int32_t profile;         /* msv_upload_profile handle (ProfileTable)           */
    int32_t dist;            /* msv_upload_dist handle (BatchDistribution); grid only */
    int32_t plan;            /* msv_upload_plan handle (PartitionPlan)             */
    int32_t scheduler;       /* msv_scheduler                                      */
    int32_t routing;         /* msv_upload_routing handle, or -1 (segment_routing off) */
    int32_t flags;           /* MSV_FLAG_*                                         */
    double sla_ms;           /* SlaConfig::sla_target_ms (sched.hpp:40)            */
    double alpha;            /* SlaConfig::alpha                                   */
    double beta;             /* SlaConfig::beta                                    */
    double rate_qps;         /* sample_trace rate (grid only)                      */
    double duration_ms;      /* QueryTrace::duration_ms                            */
    double warmup_fraction;  /* EngineOptions::warmup_fraction (engine.hpp:36)     */
    uint64_t seed;           /* sample_trace seed (grid only)                      */
} msv_scenario;

/* Per-scenario aggregate of SimReport (engine.hpp:45-89) + tail_latency(). */
typedef struct {
    int64_t total;               /* SimReport::total_queries                       */
    int64_t violations;          /* SimReport::violations                          */
    int64_t measured;            /* SimReport::measured_queries                    */
    int64_t measured_violations; /* SimReport::measured_violations                 */
    double tail[4];              /* tail_latency(latency_samples(), p_i); NaN if no samples */
    double horizon_ms;           /* SimReport::horizon_ms                          */
    double warmup_ms;            /* SimReport::warmup_ms                           */
    double max_wait_estimate_diff; /* SimReport::max_wait_estimate_diff            */
    double duration_ms;          /* SimReport::duration_ms                         */
    uint64_t placement_hash;     /* wrapping sum of msv_query_digest over queries  */
    int32_t status;              /* msv_status of this scenario                    */
    int32_t n_partitions;
} msv_result;

/* PartitionUsage (engine.hpp:57-63) without the redundant id/k. */
typedef struct {
    double busy_ms;
    double weighted_busy_ms;
    int64_t queries;
} msv_usage;

/* QueryRecord fields the engine decides (engine.hpp:45-55); arrival/batch/id are
 * the caller's trace, latency = finish - arrival, sla_met = latency <= sla. */
typedef struct {
    double start_ms;
    double finish_ms;
    int32_t partition;
    int32_t kind; /* msv_dispatch_kind */
} msv_record;

/* ---- context ----------------------------------------------------------- */
const char* msv_last_error(void);
int msv_abi_version(void);
int msv_create(int device, msv_ctx** out);
/* A context over several GPUs (member 0 = device_ids[0]; a device may repeat). Uploads
 * go to it as usual; msv_run_grid, msv_run_replay and the msv_grid_* calls cut their
 * scenarios into contiguous cost-balanced shards, run one per member concurrently and
 * gather the per-scenario results in scenario order (the reference's
 * best_homogeneous fans out with std::async, metrics.hpp:183-209). Timing,
 * synchronize and counters cover every member; single-scenario calls use member 0. */
int msv_create_multi(const int* device_ids, int n_devices, msv_ctx** out);
/* Devices of a context's members (returns the member count; fills up to cap ids). */
int msv_context_devices(msv_ctx* ctx, int* device_ids, int cap);
int msv_destroy(msv_ctx* ctx);
/* Which glibc log1p build the device mirrors for Rng::exponential (rng.hpp:20).
 * AUTO (default) probes the host libm at msv_create(). */
int msv_set_log1p_variant(msv_ctx* ctx, int variant);
int msv_get_log1p_variant(msv_ctx* ctx, int* variant);

/* ---- immutable inputs -------------------------------------------------- */
/* ProfileTable(model, sizes, b_max, latency_ms, utilization) (profile.hpp:54-61):
 * row-major [size_idx][batch-1]; validated exactly like ProfileTable::validate(). */
int msv_upload_profile(msv_ctx* ctx, int n_sizes, const int32_t* sizes, int b_max,
                       const double* latency_ms, const double* utilization, int32_t* handle);
/* BatchDistribution(weights) (workload.hpp:25-38): renormalised, cdf by partial sum. */
int msv_upload_dist(msv_ctx* ctx, int b_max, const double* weights, int32_t* handle);
/* Same, from an already-built BatchDistribution: its cdf (nondecreasing, last = 1.0)
 * is used verbatim so host and device sample identically. */
int msv_upload_cdf(msv_ctx* ctx, int b_max, const double* cdf, int32_t* handle);
/* PartitionPlan (paris.hpp:133-156): gpus[g] = sizes_flat[off_g .. off_g + n_per_gpu[g]). */
int msv_upload_plan(msv_ctx* ctx, int num_gpus, int gpcs_per_gpu, const int32_t* n_per_gpu,
                    const int32_t* sizes_flat, int32_t* handle);
/* EngineOptions::routing_segments (engine.hpp:41-42, BatchSegment paris.hpp:23-30). */
int msv_upload_routing(msv_ctx* ctx, int n_segments, const int32_t* k, const int32_t* first,
                       const int32_t* last, int32_t* handle);

/* ---- hot path ----------------------------------------------------------- */
/* Generated-trace grid: per scenario sample_trace(dist, rate, duration, seed)
 * (workload.hpp:97-113) -> run(...) (engine.hpp:115-253) -> tail_latency(
 * latency_samples(), p) (metrics.hpp:22-29) for each p in tail_p[0..n_tails).
 * usage (nullable) receives sum_i P_i entries, scenario-major, partition-id order. */
int msv_run_grid(msv_ctx* ctx, const msv_scenario* scenarios, int64_t n, const double* tail_p,
                 int n_tails, msv_result* results, msv_usage* usage);

/* Replay: host-supplied traces (QueryTrace, workload.hpp:59-63) concatenated with
 * offsets[n+1]; run() on each. records (nullable) is indexed like the traces. The
 * scenario's rate/seed/dist are ignored. */
int msv_run_replay(msv_ctx* ctx, const msv_scenario* scenarios, int64_t n, const int64_t* offsets,
                   const double* arrival_ms, const int32_t* batch, const double* tail_p,
                   int n_tails, msv_result* results, msv_usage* usage, msv_record* records);

/* run() with execution noise (EngineOptions::noise_sigma > 0, engine.hpp:140-145) on one
 * host trace (sorted by arrival), with per-query records. noise_mult[j] = exp(sigma*z_j -
 * 0.5*sigma*sigma), z_j the j-th Rng(noise_seed).normal() (rng.hpp:27-31), is the
 * multiplier of the j-th query started; the caller draws them (n of them: every query
 * starts once) with the reference's Rng and libm, and the device starts queries in the
 * reference's global event order. P <= 64. No tails (result->tail = NaN). */
int msv_run_noise(msv_ctx* ctx, const msv_scenario* scenario, int64_t n, const double* arrival_ms,
                  const int32_t* batch, const double* noise_mult, msv_result* result, msv_usage* usage,
                  msv_record* records);

/* sample_trace() on the device (workload.hpp:97-113). On MSV_PARAM with *n_out > cap
 * the trace did not fit; retry with cap >= *n_out. */
int msv_sample_trace(msv_ctx* ctx, int32_t dist, double rate_qps, double duration_ms,
                     uint64_t seed, int64_t cap, double* arrival_ms, int32_t* batch,
                     int64_t* n_out);

/* tail_latency(samples, p) (metrics.hpp:22-29), exact nearest-rank on the device. */
int msv_tail_latency(msv_ctx* ctx, const double* samples, int64_t n, const double* p,
                     int n_p, double* out);

/* Batched single-decision dispatch: elsa_dispatch / fifs_dispatch (sched.hpp:119-174)
 * and t_wait (sched.hpp:77-85) evaluated on the device for n independent trials.
 * Trial t has part_off[t+1]-part_off[t] partitions; partition j carries
 * id, k, busy, cur_est, cur_start and queue batches
 * qbatch[q_off[j] .. q_off[j+1]). All trials share one profile handle.
 * Outputs: chosen partition id, kind, and (optionally) t_wait per partition. */
int msv_dispatch_batch(msv_ctx* ctx, int32_t profile, int scheduler, int64_t n_trials,
                       const int64_t* part_off, const int32_t* part_id, const int32_t* part_k,
                       const uint8_t* busy, const double* cur_est, const double* cur_start,
                       const int64_t* q_off, const int32_t* qbatch, const int32_t* query_batch,
                       const double* now_ms, const double* sla_ms, const double* alpha,
                       const double* beta, int32_t* chosen, int32_t* kind, double* t_wait_out);

/* Batched PARIS planning (paris_plan, paris.hpp:329-345) on the device: knees
 * (profile.hpp:275-280) as a warp ballot over each size's utilization row, batch
 * segments (paris.hpp:34-49), instance ratios (paris.hpp:64-81, one lane per
 * segment folding its batches in order), instance counts (paris.hpp:92-105) and the
 * first-fit packing (paris.hpp:186-262), one warp per job. Job j's plan lands in
 * n_per_gpu[gpu_off_j ..] (num_gpus entries) and sizes_flat[inst_off_j ..]
 * (<= num_gpus * gpcs_per_gpu entries), the offsets being the running sums of those
 * two quantities over jobs 0..j-1 (jobs with num_gpus < 1 or gpcs_per_gpu < 1
 * contribute 0). Per-job errors are reported in msv_paris_out.status with the
 * exception paris_plan would throw; the call itself fails only on bad arguments. */
#define MSV_PARIS_MAX_SIZES 8
typedef struct {
    int32_t profile;        /* msv_upload_profile handle                           */
    int32_t dist;           /* msv_upload_dist handle (its normalised pmf)         */
    int32_t total_gpcs;
    int32_t num_gpus;
    int32_t gpcs_per_gpu;
    int32_t pad;
    double knee_threshold;  /* paris_plan default 0.8                              */
} msv_paris_job;            /* 32 bytes */

typedef struct {
    int32_t status;         /* msv_status of paris_plan for this job               */
    int32_t n_sizes;        /* profile sizes, ascending                             */
    int32_t n_instances;    /* placed instances (entries in this job's sizes_flat)  */
    int32_t err_k;          /* size / batch named by the error message, if any      */
    int32_t err_b;
    int32_t pad;
    int32_t k[MSV_PARIS_MAX_SIZES];
    int32_t knee[MSV_PARIS_MAX_SIZES];
    int32_t seg_first[MSV_PARIS_MAX_SIZES];
    int32_t seg_last[MSV_PARIS_MAX_SIZES];
    double ratio[MSV_PARIS_MAX_SIZES];         /* RatioEntry::ratio                 */
    double segment_mass[MSV_PARIS_MAX_SIZES];  /* RatioEntry::segment_mass          */
    double count[MSV_PARIS_MAX_SIZES];         /* InstanceCounts::counts (real)     */
    double weighted_sum;                       /* InstanceCounts::weighted_sum      */
    double normalizer;                         /* InstanceCounts::normalizer        */
} msv_paris_out;
int msv_paris_batch(msv_ctx* ctx, const msv_paris_job* jobs, int64_t n_jobs, msv_paris_out* out,
                    int32_t* n_per_gpu, int32_t* sizes_flat);

/* ---- device-resident grid (benchmarks; value = HBM-resident throughput) ---- */
typedef struct msv_grid msv_grid;
int msv_grid_create(msv_ctx* ctx, const msv_scenario* scenarios, int64_t n, const double* tail_p,
                    int n_tails, msv_grid** out);
/* Runs trace generation, simulation and tail selection for the whole grid on the
 * context stream; no host synchronisation, no host<->device copies. Back-to-back
 * launches of one single-wave grid overlap (each chunk waits only for its own previous
 * run); msv_event_record, or launching another grid in between, restores a full
 * barrier. msv_grid_results returns the last launch's results. */
int msv_grid_launch(msv_grid* grid);
int msv_grid_results(msv_grid* grid, msv_result* results, msv_usage* usage);
int msv_grid_destroy(msv_grid* grid);
/* Device time of the last launch: total and per stage (ms, CUDA events on the
 * context stream). */
int msv_grid_timing(msv_grid* grid, float* total_ms, float* trace_ms, float* sim_ms,
                    float* tail_ms);
int64_t msv_grid_queries(msv_grid* grid);   /* simulated queries of one launch */
/* Chunks of a large grid run on concurrent streams by default (on = 1); with on = 0
 * the stages run back to back and msv_grid_timing reports each stage. */
int msv_grid_set_overlap(msv_grid* grid, int on);
/* Per-partition usage (busy / weighted busy / queries, engine.hpp:57-62) is accumulated
 * by default (on = 1); with on = 0 the launch skips it and msv_grid_results must be
 * called with usage = NULL. msv_run_grid accumulates usage only when asked for it. */
int msv_grid_set_usage(msv_grid* grid, int on);
int msv_synchronize(msv_ctx* ctx);
int64_t msv_kernel_launches(msv_ctx* ctx); /* kernels launched by this context so far */
/* CUDA events on the context stream (slots 0..7) for timing loops of launches. */
int msv_event_record(msv_ctx* ctx, int slot);
int msv_event_elapsed(msv_ctx* ctx, int slot_start, int slot_end, float* ms);
/* Bytes this context copied host->device and device->host so far. */
int msv_transfer_bytes(msv_ctx* ctx, int64_t* h2d, int64_t* d2h);

/* ---- host-side planning helpers exported for bindings (paris.hpp) ------ */
/* paris_plan(table, dist, total_gpcs, num_gpus, gpcs_per_gpu, knee_threshold)
 * (paris.hpp:329-345), computed by the C++ host headers in include/migserve.
 * n_per_gpu[num_gpus] and sizes_flat[num_gpus * gpcs_per_gpu] receive the plan. */
int msv_paris_plan(int n_sizes, const int32_t* sizes, int b_max, const double* latency_ms,
                   const double* utilization, const double* dist_weights, int total_gpcs,
                   int num_gpus, int gpcs_per_gpu, double knee_threshold, int32_t* n_per_gpu,
                   int32_t* sizes_flat);

/* synth_profile(params, sizes, b_max) (profile.hpp:183-215): *n_out sorted unique
 * sizes, grids row-major [size_idx][batch-1]. */
int msv_synth_profile(double work_per_sample, double fixed_overhead, double parallelism_per_sample,
                      double util_cap, int n_sizes, const int32_t* sizes, int b_max, int32_t* n_out,
                      int32_t* sizes_out, double* latency_ms, double* utilization);
/* lognormal_batch_pdf(mu, sigma, b_max) (workload.hpp:81-93): pmf and cdf. */
int msv_lognormal_pdf(double mu, double sigma, int b_max, double* pmf, double* cdf);
/* Execution-noise multipliers (engine.hpp:140-145): out[j] = exp(sigma*z_j - 0.5*sigma*sigma),
 * z_j the j-th Rng(seed).normal() (rng.hpp:14-31: mt19937_64, Box-Muller, this host's libm),
 * the input stream of msv_run_noise. */
int msv_noise_multipliers(uint64_t seed, double sigma, int64_t n, double* out);

/* A grid of noisy scenarios (EngineOptions::noise_sigma / noise_seed per scenario,
 * engine.hpp:140-145): sample_trace -> run with execution noise -> tail_latency for every
 * scenario, like msv_run_grid. Traces are generated on the device (K1); each scenario's
 * multiplier stream exp(sigma*z_j - sigma^2/2), z_j = Rng(noise_seed).normal()
 * (rng.hpp:27-32), is drawn on the host with the reference's libm (one thread per core);
 * K5 runs one warp per scenario in the reference's global event order; K3 selects the
 * tails. P <= 64 per scenario (ParamError otherwise); noise_sigma must be > 0. */
int msv_run_grid_noise(msv_ctx* ctx, const msv_scenario* scenarios, int64_t n, const double* noise_sigma,
                       const uint64_t* noise_seed, const double* tail_p, int n_tails, msv_result* results,
                       msv_usage* usage);

/* Arithmetic self-checks (test support; no reference analogue). The parity tests
 * compare these with the host's libm directly (rng.hpp:20):
 *   msv_log1p_digest   per chunk of `chunk` inputs k in [0, n) of seed's stream
 *                      (msv_selftest_input in csrc/msv_math.h), the wrapping sum of
 *                      msv_selftest_digest(k, -log1p(-u_k)) computed with the device's
 *                      glibc-log1p transcription `variant`; digests[ceil(n/chunk)].
 *   msv_log1p_values   the device's -log1p(-u_k) for k in [first, first+count).
 *   msv_quotient_check K1's certified quotient (msv_trace.cuh gap_quotient) against
 *                      the IEEE division on n (gap, rate) pairs: counts[0] mismatches,
 *                      counts[1] certificate fallbacks. */
int msv_log1p_digest(msv_ctx* ctx, int variant, uint64_t seed, int64_t n, int64_t chunk, uint64_t* digests);
int msv_log1p_values(msv_ctx* ctx, int variant, uint64_t seed, int64_t first, int64_t count, double* out);
int msv_quotient_check(msv_ctx* ctx, uint64_t seed, int64_t n, int64_t* counts);

#ifdef __cplusplus
}
#endif
#endif /* MSV_H */
