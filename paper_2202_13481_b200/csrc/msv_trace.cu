// K1 trace_gen_kernel: sample_trace (workload.hpp:97-113) on the device — a
// warp-parallel std::mt19937_64 twist, Rng::uniform/exponential with the
// glibc-log1p transcription (msv_math.h) and BatchDistribution::sample.
#include "msv_device.cuh"

namespace msv {

namespace {
// BatchDistribution::sample's lower_bound (workload.hpp:48-53).
__device__ __forceinline__ int32_t cdf_sample(const double* __restrict__ cdf, int n, double u) {
    int lo = 0, len = n;
    while (len > 0) {
        const int half = len >> 1;
        if (__ldg(cdf + lo + half) < u) {
            lo += half + 1;
            len -= half + 1;
        } else {
            len = half;
        }
    }
    if (lo == n) lo = n - 1;
    return lo + 1;
}

__global__ void __launch_bounds__(kTraceWarpsPerBlock * 32)
    trace_gen_kernel(const TraceJob* __restrict__ jobs, int n_jobs, int variant) {
    __shared__ uint64_t s_mt[kTraceWarpsPerBlock][MSV_MT_N];
    __shared__ double s_gap[kTraceWarpsPerBlock][MSV_MT_M];
    __shared__ double s_arr[kTraceWarpsPerBlock][MSV_MT_M];
    __shared__ int32_t s_bat[kTraceWarpsPerBlock][MSV_MT_M];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int job = blockIdx.x * kTraceWarpsPerBlock + warp;
    if (job >= n_jobs) return;
    const TraceJob J = jobs[job];
    uint64_t* mt = s_mt[warp];
    double* gap = s_gap[warp];
    double* arr = s_arr[warp];
    int32_t* bat = s_bat[warp];

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

    double t = 0.0;  // meaningful in lane 0 only
    int64_t n = 0;
    bool first = true, stop = false;
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
        // i.e. word 2p is query p's gap, word 2p+1 its batch.
        for (int p = lane; p < MSV_MT_M; p += 32) {
            const double ug = msv_uniform(msv_mt_temper(mt[2 * p]));
            gap[p] = -msv_log1p_neg(-ug, variant) / J.rate_per_ms;  // rng.hpp:20
            const double ub = msv_uniform(msv_mt_temper(mt[2 * p + 1]));
            bat[p] = cdf_sample(J.cdf, J.b_max, ub);
        }
        __syncwarp();
        // Sequential arrival accumulation, exactly `t += gap` (workload.hpp:111).
        int cnt = 0;
        if (lane == 0) {
            for (int p = 0; p < MSV_MT_M; ++p) {
                const double g = gap[p];
                t = first ? g : t + g;
                first = false;
                if (!(t < J.duration_ms)) {
                    stop = true;
                    break;
                }
                arr[p] = t;
                ++cnt;
            }
        }
        cnt = __shfl_sync(kFull, cnt, 0);
        stop = __shfl_sync(kFull, stop, 0);
        for (int p = lane; p < cnt; p += 32) {
            const int64_t idx = n + p;
            if (idx < J.cap) {
                J.arrival[idx] = arr[p];
                J.batch[idx] = bat[p];
            }
        }
        n += cnt;
        if (n > J.cap) stop = true;
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
