// K3 tail_kernel: tail_latency (metrics.hpp:22-29) — exact nearest-rank by an
// MSB-first radix select over order-preserving keys of the IEEE bit patterns,
// finished by an in-shared-memory bitonic sort of the final bin.
#include "msv_device.cuh"

namespace msv {

namespace {
__device__ void bitonic_sort_smem(uint64_t* buf, int n_pow2) {
    for (int k = 2; k <= n_pow2; k <<= 1) {
        for (int j = k >> 1; j > 0; j >>= 1) {
            for (int idx = threadIdx.x; idx < n_pow2; idx += blockDim.x) {
                const int ixj = idx ^ j;
                if (ixj > idx) {
                    const uint64_t a = buf[idx], c = buf[ixj];
                    const bool up = (idx & k) == 0;
                    if ((a > c) == up) {
                        buf[idx] = c;
                        buf[ixj] = a;
                    }
                }
            }
            __syncthreads();
        }
    }
}

__global__ void __launch_bounds__(kTailThreads)
    tail_kernel(const TailJob* __restrict__ jobs, int n_jobs, const double* __restrict__ ps, int n_p) {
    __shared__ unsigned int hist[2048];
    __shared__ uint64_t buf[kTailSmemCap];
    __shared__ long long s_r;
    __shared__ unsigned long long s_prefix, s_min, s_max;
    __shared__ unsigned int s_cnt;
    __shared__ unsigned int s_pos;
    for (int jb = blockIdx.x; jb < n_jobs; jb += gridDim.x) {
        const TailJob J = jobs[jb];
        const DevOut src = *J.src;
        const long long Jn = src.n_samples;
        uint64_t kmin = src.lat_min_bits, kmax = src.lat_max_bits;  // order keys
        if (Jn > 0 && kmin > kmax) {  // not supplied: one reduction pass
            if (threadIdx.x == 0) {
                s_min = ~0ull;
                s_max = 0;
            }
            __syncthreads();
            uint64_t lo = ~0ull, hi = 0;
            for (long long idx = threadIdx.x; idx < Jn; idx += blockDim.x) {
                const uint64_t v = order_key(msv_dbits(J.samples[idx]));
                lo = v < lo ? v : lo;
                hi = v > hi ? v : hi;
            }
            atomicMin(&s_min, (unsigned long long)lo);
            atomicMax(&s_max, (unsigned long long)hi);
            __syncthreads();
            kmin = s_min;
            kmax = s_max;
            __syncthreads();
        }
        for (int q = 0; q < n_p; ++q) {
            if (Jn == 0) {
                if (threadIdx.x == 0) J.out[q] = __longlong_as_double(0x7ff8000000000000ll);
                continue;
            }
            // metrics.hpp:26-28: rank = ceil(p * n), at least 1.
            long long r = (long long)ceil(ps[q] * (double)Jn);
            if (r < 1) r = 1;
            uint64_t answer;
            if (kmin == kmax) {
                answer = kmin;
            } else {
                // MSB-first radix select over order keys, 11 bits per pass, starting
                // at the highest bit where min and max differ.
                int pos = 64 - __clzll((long long)(kmin ^ kmax));  // unknown low bits
                uint64_t prefix = (pos == 64) ? 0ull : (kmin >> pos);
                while (true) {
                    const int d = pos < 11 ? pos : 11;
                    const int shift = pos - d;
                    const int nb = 1 << d;
                    for (int k = threadIdx.x; k < nb; k += blockDim.x) hist[k] = 0;
                    __syncthreads();
                    for (long long idx = threadIdx.x; idx < Jn; idx += blockDim.x) {
                        const uint64_t v = order_key(msv_dbits(J.samples[idx]));
                        if (pos == 64 || (v >> pos) == prefix) atomicAdd(&hist[(v >> shift) & (uint64_t)(nb - 1)], 1u);
                    }
                    __syncthreads();
                    if (threadIdx.x == 0) {
                        long long cum = 0;
                        int jbin = 0;
                        for (; jbin < nb; ++jbin) {
                            if (cum + hist[jbin] >= r) break;
                            cum += hist[jbin];
                        }
                        s_r = r - cum;
                        s_prefix = ((pos == 64) ? 0ull : (prefix << d)) | (uint64_t)jbin;
                        s_cnt = hist[jbin];
                    }
                    __syncthreads();
                    r = s_r;
                    prefix = s_prefix;
                    pos = shift;
                    const unsigned cnt = s_cnt;
                    __syncthreads();
                    if (pos == 0) {
                        answer = prefix;
                        break;
                    }
                    if (cnt <= (unsigned)kTailSmemCap) {
                        if (threadIdx.x == 0) s_pos = 0;
                        __syncthreads();
                        for (long long idx = threadIdx.x; idx < Jn; idx += blockDim.x) {
                            const uint64_t v = order_key(msv_dbits(J.samples[idx]));
                            if ((v >> pos) == prefix) buf[atomicAdd(&s_pos, 1u)] = v;
                        }
                        __syncthreads();
                        int np2 = 1;
                        while (np2 < (int)cnt) np2 <<= 1;
                        for (int k = cnt + threadIdx.x; k < np2; k += blockDim.x) buf[k] = ~0ull;
                        __syncthreads();
                        bitonic_sort_smem(buf, np2);
                        answer = buf[r - 1];
                        __syncthreads();
                        break;
                    }
                }
            }
            if (threadIdx.x == 0) J.out[q] = msv_bitsd(order_unkey(answer));
            __syncthreads();
        }
    }
}


}  // namespace

cudaError_t launch_tail(const TailJob* d_jobs, int n_jobs, const double* d_p, int n_p,
                        cudaStream_t stream) {
    if (n_jobs <= 0) return cudaSuccess;
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int blocks = n_jobs < sms * 4 ? n_jobs : sms * 4;
    tail_kernel<<<blocks, kTailThreads, 0, stream>>>(d_jobs, n_jobs, d_p, n_p);
    return cudaGetLastError();
}

}  // namespace msv
