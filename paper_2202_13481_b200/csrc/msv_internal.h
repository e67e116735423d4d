// Internal structures shared by the CUDA kernels (msv_kernels.cu) and the host
// runtime (msv_host.cpp). Not part of the public ABI (include/msv.h).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/msv.h"

namespace msv {

// Shared-memory ring capacity of each partition's FIFO (entries). Deeper queues
// continue as a singly linked list threaded through the scenario's query ids
// (DevScen::next), so queue depth is bounded only by the trace length.
constexpr int kQCap = 8;
// Profile cells (latency + utilisation, all uploaded profiles) staged in shared
// memory by the simulation kernel.
constexpr int kMaxSmemCells = 1024;
constexpr int kSimWarpsPerBlock = 4;
constexpr int kTraceWarpsPerBlock = 4;
constexpr int kTraceGroupMax = 16;    // traces sharing one random stream per K1 warp
constexpr int kTraceAccStride = 34;   // padded row (double2 reads by 16 lanes: 2 wavefronts)
constexpr int kTailThreads = 256;
constexpr int kTailSmemCap = 2048;  // values gathered for the final in-smem select
// Guide table of BatchDistribution::sample: u in [j/G, (j+1)/G) starts its lower_bound at guide[j].
constexpr int kGuide = 256;
// Internal status: generated trace exceeded its capacity, host re-runs with a larger one.
constexpr int kStatusRetryTrace = 101;

// One partition as the simulation sees it, in by_ascending_size order
// (sched.hpp:96-104): the warp lane of order index o = s*W + lane.
struct DevPart {
    int32_t pid;   // partition id = index in plan.flatten() (paris.hpp:134-139)
    int32_t k;     // partition size in GPCs
    int32_t row;   // offset of latency(k, 1) in the concatenated profile cells
    int32_t pad;
};

// Per-scenario inputs of the simulation kernel.
struct DevScen {
    const double* arrival;      // trace arrivals (device)
    const int32_t* batch;       // trace batches (device)
    const int64_t* n;           // queries in the trace (written by K1 or the host)
    double duration_ms;
    double warmup_ms;
    double lat_floor;           // lower bound of every latency (half the profile's smallest cell)
    double sla, alpha, beta;
    const DevPart* parts;       // P entries in (k, id) ascending order
    const uint64_t* route_mask; // P masks (bit b-1: segment of k covers batch b) or null
    uint32_t* next;             // per-query link of the overflow queues (capacity n)
    double* samples;            // measured latencies out: latency of query q >= m0 lands at
                                // samples[q] (the generated / uploaded arrival buffer itself:
                                // a query's arrival is dead once its window is retired)
    msv_record* records;        // per-query records out, or null
    int32_t P;
    int32_t b_max;              // profile b_max
    int32_t sched;
    int32_t flags;
    int32_t usage_off;          // first msv_usage slot of this scenario (or -1)
    int32_t pad;
};

// Per-scenario outputs of the simulation kernel (input of the tail kernel).
struct DevOut {
    int64_t violations;
    int64_t measured;
    int64_t measured_violations;
    int64_t n_samples;
    double horizon_ms;
    double max_wait_diff;
    uint64_t hash;
    uint64_t lat_min_bits;
    uint64_t lat_max_bits;
    int32_t status;
    int32_t m0;                 // first measured query: samples live at samples[m0, m0 + n_samples)
    int32_t planar;             // sample layout: 0 doubles, 1 K2 warp blocks (kPlanar below)
    int32_t pad;
};

// Planar sample layout (the one-warp K2 kernel): the latencies of queries 32b .. 32b + 31
// occupy the 256 bytes of their own arrivals as 32 high words followed by 32 low words,
// so K3's first passes read only the high halves (4 bytes per sample).
__host__ __device__ inline int64_t planar_hi_word(int64_t q) { return ((q >> 5) << 6) + (q & 31); }

struct SimParams {
    const DevScen* scen;
    DevOut* out;
    msv_usage* usage;
    const int32_t* work;  // scenario indices of this class, longest first
    int32_t n_work;
    int32_t* counter;     // work-stealing counter (device)
    const double* lat;    // all profile latency cells
    const double* util;   // all profile utilisation cells
    int32_t n_cells;
    // Launch-wide feature flags: when 0, the kernel skips the corresponding per-arrival
    // warp votes entirely.
    int32_t any_routing;     // some scenario uses segment routing
    int32_t any_bad;         // some plan has a size the profile lacks
    int32_t any_check_wait;  // some scenario sets MSV_FLAG_CHECK_WAIT
    int32_t any_usage;       // per-partition usage (PartitionUsage) requested
    int32_t lazy;            // warp kernel: lazy folds for long queues (overloaded scenarios)
    // Streamed launch (latency-bound generated grids): one 2-warp block per scenario, warp 0
    // generates the trace (stream_jobs[scenario index], K1's job) while warp 1 simulates it.
    int32_t stream;
    int32_t log1p_variant;
    const struct TraceJob* stream_jobs;
};

// Trace generation job (sample_trace, workload.hpp:97-113).
struct TraceJob {
    uint64_t seed;
    double rate_per_ms;   // rate_qps / 1000.0 (workload.hpp:103)
    double duration_ms;
    const double* cdf;    // BatchDistribution cdf (device)
    const int16_t* guide; // kGuide entries: first index with cdf >= j / kGuide
    int32_t b_max;
    int32_t pad;
    double* arrival;      // out
    int32_t* batch;       // out
    int64_t cap;
    int64_t* n_out;       // out: queries generated (min(n, cap))
    int32_t* overflow;    // out: 1 when the trace did not fit in cap
};

struct TailJob {
    const double* samples;
    const DevOut* src;  // n_samples / lat_min_bits / lat_max_bits / layout of the scenario
    double* out;        // n_p tails
    uint64_t* cand;     // candidate keys scratch (the scenario's dead overflow links), or null
    int64_t cand_cap;   // entries of cand
};

// Single-decision dispatch trials (msv_dispatch_batch).
struct DispatchParams {
    int64_t n_trials;
    const int64_t* part_off;
    const int32_t* part_id;
    const int32_t* part_k;
    const int32_t* part_row;
    const uint8_t* busy;
    const double* cur_est;
    const double* cur_start;
    const int64_t* q_off;
    const int32_t* qbatch;
    const int32_t* query_batch;
    const double* now_ms;
    const double* sla_ms;
    const double* alpha;
    const double* beta;
    const double* lat;
    int32_t b_max;        // shared profile's b_max
    int32_t scheduler;
    int32_t* chosen;
    int32_t* kind;
    double* t_wait_out;
    int32_t* error;  // LookupError flag per trial
};

// Batched paris_plan jobs (msv_paris_batch); offsets precomputed on the host.
struct ParisJobDev {
    int32_t row0;      // cell offset of the profile's first size row
    int32_t n_sizes;
    int32_t b_max;     // profile b_max
    int32_t dist_b_max;
    int64_t pmf_off;   // dist pmf offset
    int64_t gpu_off;   // into n_per_gpu
    int64_t inst_off;  // into sizes_flat
    const int32_t* sizes;
    int32_t total_gpcs, num_gpus, gpcs_per_gpu, pad;
    double knee_threshold;
};

struct ParisParams {
    const ParisJobDev* jobs;
    int64_t n_jobs;
    const double* lat;
    const double* util;
    const double* pmf;
    msv_paris_out* out;
    int32_t* n_per_gpu;
    int32_t* sizes_flat;
    int32_t* remaining;  // scratch: num_gpus ints per job at gpu_off
};

// K5: run() with execution noise (msv_noise.cu), one warp (one block) per job, P <= 64.
struct NoiseParams {
    const double* arrival;      // sorted trace (device)
    const int32_t* batch;
    int64_t n;
    const int64_t* n_ptr;       // trace length on the device (K1's count), or null: use n
    double* samples;            // measured latencies out at samples[q] (the arrival buffer), or null
    double duration_ms;         // horizon = max(duration, last finish) (engine.hpp:235)
    const double* mult;         // n noise multipliers exp(sigma*z_j - sigma^2/2), start order
    const double* lat;          // this profile's cells, row-major [size_idx][batch-1]
    const double* util;
    const DevPart* parts;       // P entries in (k, id) order; row relative to lat, -1 = size missing
    const uint64_t* route_mask; // P masks or null
    int32_t P, b_max, sched, n_cells;  // n_cells: entries of lat (and util)
    double sla, alpha, beta, warmup_ms;
    uint32_t* next;             // n: FIFO links through query indices
    msv_record* records;        // n, or null (grids keep only the aggregates and samples)
    msv_usage* usage;           // P, by partition id
    DevOut* out;                // violations, measured(+samples, m0), hash, horizon, status
};

// Kernel launchers (msv_kernels.cu). Return cudaGetLastError().
// One block (one warp) per job; max_cells = the largest job's profile cells.
cudaError_t launch_noise(const NoiseParams* d_jobs, int n_jobs, int max_cells, int max_parts, cudaStream_t stream);
cudaError_t launch_paris(const ParisParams& p, cudaStream_t stream);
// K1 over groups: group g covers jobs [first, first + count) (count <= kTraceGroupMax, one
// seed and distribution per group).
struct TraceGroup {
    int32_t first, count;
};
cudaError_t launch_trace_groups(const TraceJob* d_jobs, const TraceGroup* d_groups, int n_groups, int log1p_variant,
                                cudaStream_t stream);
cudaError_t launch_trace_gen(const TraceJob* d_jobs, int n_jobs, int log1p_variant,
                             cudaStream_t stream);
// Persistent simulation kernel for P <= W*S (W lanes per scenario, S slots per lane).
// sched is the scenario class's scheduler (all scenarios of one launch share it).
cudaError_t launch_sim(int W, int S, int sched, bool records, const SimParams& p, int blocks,
                       cudaStream_t stream);
size_t sim_smem_bytes(int W, int S, int n_cells);
int sim_max_blocks_per_sm(int W, int S, int sched, bool records, bool full, bool lazy, int n_cells);
// Raise a kernel's dynamic shared-memory limit on the current device (never lowers it;
// thread-safe: contexts on several threads launch the same kernels).
cudaError_t ensure_dyn_smem(const void* fn, size_t bytes);
// Arithmetic self-checks (msv_selftest.cu).
cudaError_t launch_log1p_digest(int variant, uint64_t seed, int64_t n, int64_t chunk, uint64_t* d_out,
                                cudaStream_t stream);
cudaError_t launch_log1p_values(int variant, uint64_t seed, int64_t first, int64_t count, double* d_out,
                                cudaStream_t stream);
cudaError_t launch_quotient_check(uint64_t seed, int64_t n, unsigned long long* d_counts, cudaStream_t stream);
cudaError_t launch_tail(const TailJob* d_jobs, int n_jobs, const double* d_p, int n_p,
                        cudaStream_t stream);
cudaError_t launch_dispatch(const DispatchParams& p, cudaStream_t stream);

}  // namespace msv
