// K1: sample_trace (workload.hpp:97-113) on the device. trace_gen_kernel: one warp per
// trace (warp_sample_trace); trace_group_kernel: one warp per random stream, i.e. per
// group of traces with the same seed and batch distribution (warp_sample_trace_group);
// both in msv_trace.cuh.
#include "msv_trace.cuh"

namespace msv {

namespace {

__global__ void __launch_bounds__(kTraceWarpsPerBlock * 32)
    trace_gen_kernel(const TraceJob* __restrict__ jobs, int n_jobs, int variant) {
    __shared__ uint64_t s_mt[kTraceWarpsPerBlock][MSV_MT_N];
    __shared__ __align__(16) double s_acc[kTraceWarpsPerBlock][32];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int job = blockIdx.x * kTraceWarpsPerBlock + warp;
    if (job >= n_jobs) return;
    const TraceJob J = jobs[job];
    warp_sample_trace(J, s_mt[warp], s_acc[warp], lane, variant);
}

__global__ void __launch_bounds__(kTraceWarpsPerBlock * 32)
    trace_group_kernel(const TraceJob* __restrict__ jobs, const TraceGroup* __restrict__ groups, int n_groups,
                       int variant) {
    __shared__ TraceGroupSmem s_grp[kTraceWarpsPerBlock];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int g = blockIdx.x * kTraceWarpsPerBlock + warp;
    if (g >= n_groups) return;
    const TraceGroup G = groups[g];
    warp_sample_trace_group(jobs + G.first, G.count, s_grp[warp], lane, variant);
}

}  // namespace

cudaError_t launch_trace_gen(const TraceJob* d_jobs, int n_jobs, int log1p_variant,
                             cudaStream_t stream) {
    if (n_jobs <= 0) return cudaSuccess;
    const int blocks = (n_jobs + kTraceWarpsPerBlock - 1) / kTraceWarpsPerBlock;
    trace_gen_kernel<<<blocks, kTraceWarpsPerBlock * 32, 0, stream>>>(d_jobs, n_jobs, log1p_variant);
    return cudaGetLastError();
}

cudaError_t launch_trace_groups(const TraceJob* d_jobs, const TraceGroup* d_groups, int n_groups, int log1p_variant,
                                cudaStream_t stream) {
    if (n_groups <= 0) return cudaSuccess;
    const int blocks = (n_groups + kTraceWarpsPerBlock - 1) / kTraceWarpsPerBlock;
    trace_group_kernel<<<blocks, kTraceWarpsPerBlock * 32, 0, stream>>>(d_jobs, d_groups, n_groups, log1p_variant);
    return cudaGetLastError();
}

}  // namespace msv
