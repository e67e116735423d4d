// Device self-checks of the two arithmetic kernels K1's bit-exactness rests on, so the
// parity tests can compare them directly with the host (not only through traces, where
// a libm mismatch surfaces ~1e-6 of the time):
//   * msv_log1p_digest: the device's -log1p(-u) (msv_log1p_neg, the glibc transcription
//     K1 evaluates for Rng::exponential, rng.hpp:20) on n counter-based inputs from the
//     uniform grid u = m * 2^-53 (msv_selftest_input, shared with the host checker);
//     per chunk of inputs a wrapping sum of mixed result bits, compared with the same
//     digest of the host libm's log1p;
//   * msv_quotient_check: gap_quotient (K1's certified division, msv_trace.cuh) against
//     the IEEE division on n (l, r) pairs — mismatches (must be 0) and how often the
//     certificate fell back to the division.
#include "msv_device.cuh"
#include "msv_trace.cuh"

namespace msv {

namespace {

__global__ void log1p_digest_kernel(int variant, uint64_t seed, int64_t n, int64_t chunk, uint64_t* out) {
    const int64_t n_chunks = (n + chunk - 1) / chunk;
    for (int64_t c = blockIdx.x; c < n_chunks; c += gridDim.x) {
        const int64_t lo = c * chunk, hi = min(n, lo + chunk);
        uint64_t acc = 0;
        for (int64_t k = lo + threadIdx.x; k < hi; k += blockDim.x) {
            const double u = msv_selftest_input(seed, (uint64_t)k);
            acc += msv_selftest_digest((uint64_t)k, -msv_log1p_neg(-u, variant));
        }
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) acc += __shfl_xor_sync(kFull, acc, off);
        __shared__ uint64_t part[32];
        if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = acc;
        __syncthreads();
        if (threadIdx.x == 0) {
            uint64_t s = 0;
            for (int w = 0; w < (int)(blockDim.x >> 5); ++w) s += part[w];
            out[c] = s;
        }
        __syncthreads();
    }
}

__global__ void log1p_values_kernel(int variant, uint64_t seed, int64_t first, int64_t count, double* out) {
    for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < count; j += (int64_t)gridDim.x * blockDim.x)
        out[j] = -msv_log1p_neg(-msv_selftest_input(seed, (uint64_t)(first + j)), variant);
}

__global__ void quotient_check_kernel(uint64_t seed, int64_t n, unsigned long long* mism,
                                      unsigned long long* fallback) {
    unsigned long long bad = 0, fb = 0;
    for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < n; k += (int64_t)gridDim.x * blockDim.x) {
        const uint64_t x = msv_splitmix64(seed ^ ((uint64_t)k * 0x9E3779B97F4A7C15ull));
        const uint64_t z = msv_splitmix64(x);
        // l: an exponential gap -log1p(-u) (the numerators K1 divides), r: a rate per ms
        // log-uniform over [2^-600, 2^600] on odd k, over [1e-3, 1e3] q/ms on even k
        const double l = -msv_log1p_neg(-msv_selftest_input(seed, (uint64_t)k), MSV_LOG1P_GENERIC);
        const int e = (k & 1) ? (int)(z % 1200) - 600 : (int)(z % 20) - 10;
        const double r = ldexp(1.0 + (double)(z >> 12) * 0x1.0p-52, e);
        const double q = gap_quotient(l, r, 1.0 / r);
        bad += msv_dbits(q) != msv_dbits(__ddiv_rn(l, r));
        bool ok;  // how often the certificate sends the quotient to the division
        (void)gap_quotient_candidate(l, r, 1.0 / r, ok);
        fb += ok ? 0 : 1;
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
        bad += __shfl_xor_sync(kFull, bad, off);
        fb += __shfl_xor_sync(kFull, fb, off);
    }
    if ((threadIdx.x & 31) == 0) {
        atomicAdd(mism, bad);
        atomicAdd(fallback, fb);
    }
}

}  // namespace

cudaError_t launch_log1p_digest(int variant, uint64_t seed, int64_t n, int64_t chunk, uint64_t* d_out,
                                cudaStream_t stream) {
    const int64_t n_chunks = (n + chunk - 1) / chunk;
    const int blocks = (int)(n_chunks < 148 * 16 ? n_chunks : 148 * 16);
    log1p_digest_kernel<<<blocks, 256, 0, stream>>>(variant, seed, n, chunk, d_out);
    return cudaGetLastError();
}

cudaError_t launch_log1p_values(int variant, uint64_t seed, int64_t first, int64_t count, double* d_out,
                                cudaStream_t stream) {
    log1p_values_kernel<<<148 * 4, 256, 0, stream>>>(variant, seed, first, count, d_out);
    return cudaGetLastError();
}

cudaError_t launch_quotient_check(uint64_t seed, int64_t n, unsigned long long* d_counts, cudaStream_t stream) {
    quotient_check_kernel<<<148 * 8, 256, 0, stream>>>(seed, n, d_counts, d_counts + 1);
    return cudaGetLastError();
}

}  // namespace msv
