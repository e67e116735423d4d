/*
 * TEST INFRASTRUCTURE ONLY. Checker ABI shared by the two CPU oracles:
 *   - oracle/_ref/libmsv_ref.so   the reference itself: /root/reference/proj/include
 *                                 compiled unmodified behind these C entry points
 *                                 (oracle/ref_capi.cpp);
 *   - oracle/libmsv_oracle.so     an independent plain-C restatement of the same
 *                                 path (oracle/port/msv_oracle.c), each function
 *                                 citing the reference file:line it follows.
 * Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline leg load them.
 * The product (paper_2202_13481_b200/libmsv.so) never links or calls either.
 */
#ifndef MSV_ORACLE_ABI_H
#define MSV_ORACLE_ABI_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct {
    int n_sizes;
    const int32_t* sizes;
    int b_max;
    const double* lat; /* [size_idx][batch-1] */
    const double* util;
} ora_profile;

typedef struct {
    int num_gpus;
    int gpcs_per_gpu;
    const int32_t* n_per_gpu;
    const int32_t* sizes_flat;
} ora_plan;

typedef struct {
    int b_max;
    const double* weights; /* BatchDistribution(weights) */
} ora_dist;

typedef struct {
    int32_t profile, dist, plan, scheduler; /* scheduler 0 FIFS, 1 ELSA */
    double sla_ms, alpha, beta, rate_qps, duration_ms, warmup_fraction;
    uint64_t seed;
} ora_scenario;

typedef struct {
    int64_t total, violations, measured, measured_violations;
    double tail[4];
    double horizon_ms;
    uint64_t placement_hash;
    int32_t status; /* 0 ok, 1..5 = reference exception type */
    int32_t pad;
} ora_result;

/* Per-query engine outputs of one run (QueryRecord, engine.hpp:45-55). */
typedef struct {
    int32_t* partition;
    double* start_ms;
    double* finish_ms;
    int32_t* kind;
} ora_records;

typedef struct {
    int64_t total, violations, measured, measured_violations;
    double horizon_ms, warmup_ms, max_wait_estimate_diff;
    double* busy_ms;          /* [P] */
    double* weighted_busy_ms; /* [P] */
    int64_t* queries;         /* [P] */
} ora_report;

/* Digest identical to the device engine's grid hash (msv_math.h msv_query_digest). */
static inline uint64_t ora_mix64(uint64_t z) {
    z += 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}
static inline uint64_t ora_bits(double x) {
    union {
        double d;
        uint64_t u;
    } v;
    v.d = x;
    return v.u;
}
static inline uint64_t ora_query_digest(uint64_t id, int32_t partition, double start, double finish) {
    const uint64_t sb = ora_bits(start), fb = ora_bits(finish);
    const uint32_t c = (uint32_t)id * 0x9E3779B1u + (uint32_t)partition;
    const uint32_t a = ((uint32_t)sb ^ (uint32_t)(fb >> 32) ^ c) * 0x85EBCA6Bu;
    const uint32_t b = ((uint32_t)(sb >> 32) ^ (uint32_t)fb ^ c) * 0x27D4EB2Fu + c;
    return ((uint64_t)a << 32) | b;
}

/* ---- entry points (same names in both oracles, prefix ora_) ---- */
const char* ora_last_error(void);
const char* ora_kind(void); /* "reference" or "port" */
/* BatchDistribution: normalised pmf and cdf (workload.hpp:25-38). */
int ora_dist_tables(const ora_dist* d, double* pmf, double* cdf);
/* sample_trace (workload.hpp:97-113). Returns the count; > cap means truncated. */
int64_t ora_sample_trace(const ora_dist* d, double rate_qps, double duration_ms, uint64_t seed, int64_t cap,
                         double* arrival, int32_t* batch);
/* run (engine.hpp:115-253) on a host trace. records / report arrays are caller-owned. */
int ora_run(const ora_plan* plan, int scheduler, const double* arrival, const int32_t* batch, int64_t n,
            double duration_ms, const ora_profile* prof, double sla, double alpha, double beta,
            double warmup_fraction, int check_wait, int n_route, const int32_t* route_k,
            const int32_t* route_first, const int32_t* route_last, ora_records* rec, ora_report* rep);
/* tail_latency (metrics.hpp:22-29). */
int ora_tail_latency(const double* samples, int64_t n, double p, double* out);
/* Grid of sample_trace -> run -> tail_latency, on n_threads host threads. */
int ora_run_grid(const ora_profile* profs, const ora_dist* dists, const ora_plan* plans, const ora_scenario* sc,
                 int64_t n, const double* ps, int n_p, int n_threads, ora_result* out);

#ifdef __cplusplus
}
#endif
#endif
