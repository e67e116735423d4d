// K1 trace_gen_kernel: sample_trace (workload.hpp:97-113) on the device — a
// warp-parallel std::mt19937_64 twist, Rng::uniform/exponential with the
// glibc-log1p transcription (msv_math.h) and BatchDistribution::sample.
#include "msv_device.cuh"

namespace msv {

namespace {
// BatchDistribution::sample's lower_bound (workload.hpp:48-53): first i with
// !(cdf[i] < u), clamped to the last bin. guide[floor(u*G)] is lower_bound(cdf, j/G)
// <= the answer (u >= j/G, cdf nondecreasing), so a forward scan from it is exact.
__device__ __forceinline__ int32_t cdf_sample(const double* __restrict__ cdf, const int16_t* __restrict__ guide,
                                              int n, double u) {
    int i = __ldg(guide + (int)(u * (double)kGuide));  // u*G is exact (G = 2^8, u on the 2^-53 grid)
    while (i < n && __ldg(cdf + i) < u) ++i;
    if (i == n) i = n - 1;
    return i + 1;
}

__global__ void __launch_bounds__(kTraceWarpsPerBlock * 32)
    trace_gen_kernel(const TraceJob* __restrict__ jobs, int n_jobs, int variant) {
    __shared__ uint64_t s_mt[kTraceWarpsPerBlock][MSV_MT_N];
    __shared__ __align__(16) double s_acc[kTraceWarpsPerBlock][32];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int job = blockIdx.x * kTraceWarpsPerBlock + warp;
    if (job >= n_jobs) return;
    const TraceJob J = jobs[job];
    uint64_t* mt = s_mt[warp];

    // mt19937_64(seed): x[0] = seed; x[i] = f*(x[i-1] ^ (x[i-1] >> 62)) + i.
    if (lane == 0) {
        uint64_t x = J.seed;
        mt[0] = x;
        for (uint32_t i = 1; i < MSV_MT_N; ++i) {
            x = msv_mt_next_seed(x, i);
            mt[i] = x;
        }
    }
    __syncwarp();

    double t = 0.0;  // last arrival so far (warp-uniform)
    int64_t n = 0;
    bool stop = false;
    while (!stop) {
        // Regenerate the 312-word block. Words [0,156) read only old words;
        // words [156,312) read new[i-156] (and word 311 reads new[0]). Within a
        // pass every lane reads before any lane writes.
        for (int base = 0; base < MSV_MT_M; base += 32) {
            const int i = base + lane;
            uint64_t v = 0;
            if (i < MSV_MT_M) v = msv_mt_twist(mt[i], mt[i + 1], mt[i + MSV_MT_M]);
            __syncwarp();
            if (i < MSV_MT_M) mt[i] = v;
            __syncwarp();
        }
        for (int base = MSV_MT_M; base < MSV_MT_N; base += 32) {
            const int i = base + lane;
            uint64_t v = 0;
            if (i < MSV_MT_N) v = msv_mt_twist(mt[i], mt[(i + 1 == MSV_MT_N) ? 0 : i + 1], mt[i - MSV_MT_M]);
            __syncwarp();
            if (i < MSV_MT_N) mt[i] = v;
            __syncwarp();
        }
        // Draw order (workload.hpp:104-111): gap_0, then (batch_p, gap_{p+1}) —
        // i.e. word 2p is query p's gap, word 2p+1 its batch. Pairs are handled in
        // rounds of 32 (lane = pair); the arrival times are the sequential sums
        // t_p = t_{p-1} + gap_p (workload.hpp:108-111, t_{-1} = 0.0 since 0.0 + g == g),
        // carried lane to lane by a shuffle chain so the rounding order is the
        // reference's.
        for (int r = 0; r * 32 < MSV_MT_M && !stop; ++r) {
            const int p = r * 32 + lane;
            const int nvalid = min(32, MSV_MT_M - r * 32);
            double g = 0.0;
            int32_t bt = 0;
            if (lane < nvalid) {
                const double ug = msv_uniform(msv_mt_temper(mt[2 * p]));
                g = -msv_log1p_neg(-ug, variant) / J.rate_per_ms;  // rng.hpp:20
                const double ub = msv_uniform(msv_mt_temper(mt[2 * p + 1]));
                bt = cdf_sample(J.cdf, J.guide, J.b_max, ub);
            }
            // the 32 sequential sums run in lane 0 out of shared memory (two gaps per
            // 16-byte load), then every lane picks its own arrival up again
            double* sa = s_acc[warp];
            sa[lane] = g;
            __syncwarp();
            if (lane == 0) {
                double a = t;
#pragma unroll
                for (int k = 0; k < 32; k += 2) {
                    double2 v = *reinterpret_cast<const double2*>(sa + k);
                    a = a + v.x;
                    v.x = a;
                    a = a + v.y;
                    v.y = a;
                    *reinterpret_cast<double2*>(sa + k) = v;
                }
            }
            __syncwarp();
            const double acc = sa[lane];  // lanes >= nvalid carry g = 0 and are masked below
            // `while (t < duration)`: arrivals are non-decreasing, so the kept ones are a prefix.
            const unsigned keep = __ballot_sync(kFull, lane < nvalid && acc < J.duration_ms);
            const int cnt = (keep == kFull) ? 32 : (__ffs(~keep) - 1);
            if (lane < cnt && n + lane < J.cap) {
                J.arrival[n + lane] = acc;
                J.batch[n + lane] = bt;
            }
            n += cnt;
            if (cnt < nvalid || n > J.cap) stop = true;
            t = __shfl_sync(kFull, acc, nvalid - 1);
        }
        __syncwarp();
    }
    if (lane == 0) {
        *J.n_out = (n > J.cap) ? J.cap : n;
        *J.overflow = (n > J.cap) ? 1 : 0;
    }
}


}  // namespace

cudaError_t launch_trace_gen(const TraceJob* d_jobs, int n_jobs, int log1p_variant,
                             cudaStream_t stream) {
    if (n_jobs <= 0) return cudaSuccess;
    const int blocks = (n_jobs + kTraceWarpsPerBlock - 1) / kTraceWarpsPerBlock;
    trace_gen_kernel<<<blocks, kTraceWarpsPerBlock * 32, 0, stream>>>(d_jobs, n_jobs, log1p_variant);
    return cudaGetLastError();
}

}  // namespace msv
