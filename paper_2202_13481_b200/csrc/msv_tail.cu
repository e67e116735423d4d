// K3 tail_kernel: tail_latency (metrics.hpp:22-29) — exact nearest-rank by an
// MSB-first radix select over order-preserving keys of the IEEE bit patterns.
//
// One block per scenario (grid-stride). All requested percentiles advance together:
// each pass streams the scenario's samples once and builds one 2048-bin histogram
// per still-open percentile (warp-aggregated with __match_any_sync, since identical
// latencies are common); a block scan picks each percentile's bin. As soon as a
// bin holds <= kTailGather values they are gathered into shared memory (one more
// pass) and sorted there (bitonic), which settles the percentile exactly.
// The key range [lo, hi] comes from the sim kernel (coarse 32-bit bounds) or, when
// absent, from one reduction pass.
#include "msv_device.cuh"

namespace msv {

namespace {

constexpr int kBins = 2048;
constexpr int kDigit = 11;
// The first pass is shared by every percentile (same prefix): its histogram spans the
// whole kMaxTails x kBins area, i.e. 13-bit digits, so the bin holding a target rank is
// usually small enough to gather right away (2 passes instead of 3 on the bench grid).
constexpr int kDigit0 = 13;
constexpr int kMaxTails = 4;
constexpr int kTailGather = 1024;  // per percentile

struct TailSmem {
    unsigned int hist[kMaxTails][kBins];
    uint64_t buf[kMaxTails][kTailGather];
    unsigned long long prefix[kMaxTails];
    long long rank[kMaxTails];
    int pos[kMaxTails];
    unsigned int cnt[kMaxTails];
    unsigned int fill[kMaxTails];
    int state[kMaxTails];  // 0 radix pass, 1 gather, 2 done
    unsigned long long answer[kMaxTails];
    unsigned long long kmin, kmax;
    unsigned int warp_sum[kTailThreads / 32];
};

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

// Exclusive block scan of per-thread sums; returns the prefix before this thread.
__device__ unsigned int block_exclusive_scan(unsigned int v, unsigned int* warp_sum, unsigned int* total) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    unsigned int x = v;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
        const unsigned int y = __shfl_up_sync(kFull, x, off);
        if (lane >= off) x += y;
    }
    if (lane == 31) warp_sum[wid] = x;
    __syncthreads();
    unsigned int before = 0, all = 0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) {
        if (w < wid) before += warp_sum[w];
        all += warp_sum[w];
    }
    __syncthreads();
    *total = all;
    return before + x - v;
}

__global__ void __launch_bounds__(kTailThreads)
    tail_kernel(const TailJob* __restrict__ jobs, int n_jobs, const double* __restrict__ ps, int n_p) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    TailSmem& S = *reinterpret_cast<TailSmem*>(smem_raw);
    for (int jb = blockIdx.x; jb < n_jobs; jb += gridDim.x) {
        const TailJob J = jobs[jb];
        const DevOut src = *J.src;
        const long long n = src.n_samples;
        if (n == 0) {
            if (threadIdx.x < n_p) J.out[threadIdx.x] = __longlong_as_double(0x7ff8000000000000ll);
            continue;
        }
        const double* __restrict__ x = J.samples + src.m0;  // the measured suffix
        if (threadIdx.x == 0) {
            S.kmin = src.lat_min_bits;
            S.kmax = src.lat_max_bits;
        }
        __syncthreads();
        if (S.kmin > S.kmax) {  // bounds not supplied: one reduction pass
            uint64_t lo = ~0ull, hi = 0;
            for (long long i = threadIdx.x; i < n; i += blockDim.x) {
                const uint64_t v = order_key(msv_dbits(x[i]));
                lo = v < lo ? v : lo;
                hi = v > hi ? v : hi;
            }
            __syncthreads();
            if (threadIdx.x == 0) {
                S.kmin = ~0ull;
                S.kmax = 0;
            }
            __syncthreads();
            atomicMin(&S.kmin, (unsigned long long)lo);
            atomicMax(&S.kmax, (unsigned long long)hi);
            __syncthreads();
        }
        const uint64_t kmin = S.kmin, kmax = S.kmax;
        if (threadIdx.x < n_p) {
            const int q = threadIdx.x;
            long long r = (long long)ceil(ps[q] * (double)n);  // metrics.hpp:26-27
            if (r < 1) r = 1;
            S.rank[q] = r;
            const int top = (kmin == kmax) ? 0 : 64 - __clzll((long long)(kmin ^ kmax));
            S.pos[q] = top;  // number of unknown low key bits
            S.prefix[q] = top == 64 ? 0ull : (kmin >> top);
            S.state[q] = top == 0 ? 2 : 0;
            S.answer[q] = kmin;
        }
        __syncthreads();
        for (int pass = 0;; ++pass) {
            // ---- one streaming pass: radix histograms and/or gathers ----
            bool any_open = false;
            for (int q = 0; q < n_p; ++q) any_open |= S.state[q] != 2;
            if (!any_open) break;
            if (pass > 16) {  // at most ceil(64/11) radix passes + 1 gather: inconsistent input
                if (threadIdx.x < n_p) S.answer[threadIdx.x] = order_key(0x7ff8000000000000ull);  // NaN
                __syncthreads();
                break;
            }
            // Percentiles still in radix mode with the same (pos, prefix) share one
            // histogram (always the case in the first pass).
            int hsrc[kMaxTails];
            for (int q = 0; q < n_p; ++q) {
                hsrc[q] = q;
                if (S.state[q] == 0)
                    for (int q2 = 0; q2 < q; ++q2)
                        if (S.state[q2] == 0 && S.pos[q2] == S.pos[q] && S.prefix[q2] == S.prefix[q]) {
                            hsrc[q] = q2;
                            break;
                        }
            }
            // pass 0: every open percentile rides on histogram 0 -> one wide histogram
            bool shared0 = pass == 0;
            for (int q = 0; q < n_p; ++q) shared0 = shared0 && (S.state[q] != 0 || hsrc[q] == 0);
            const int dig = shared0 ? kDigit0 : kDigit;
            unsigned int* const hbase = &S.hist[0][0];
            for (int q = 0; q < n_p; ++q) {
                if (S.state[q] == 0 && hsrc[q] == q)
                    for (int k = threadIdx.x; k < (1 << dig); k += blockDim.x) hbase[q * kBins + k] = 0;
                if (S.state[q] == 1 && threadIdx.x == 0) S.fill[q] = 0;
            }
            __syncthreads();
            // pass parameters in registers (constant during the pass)
            int st_r[kMaxTails], pos_r[kMaxTails], sh_r[kMaxTails];
            uint64_t pre_r[kMaxTails];
            unsigned dmask_r[kMaxTails];
#pragma unroll
            for (int q = 0; q < kMaxTails; ++q) {
                const bool on = q < n_p;
                st_r[q] = on ? S.state[q] : 2;
                if (on && st_r[q] == 0 && hsrc[q] != q) st_r[q] = 3;  // rides on another histogram
                pos_r[q] = on ? S.pos[q] : 0;
                pre_r[q] = on ? S.prefix[q] : 0;
                const int d = pos_r[q] < dig ? pos_r[q] : dig;
                sh_r[q] = pos_r[q] - d;
                dmask_r[q] = (1u << d) - 1u;
            }
            constexpr int U = 4;  // independent loads in flight per thread
            const int lane = threadIdx.x & 31;
            for (long long base = 0; base < n; base += (long long)blockDim.x * U) {
                uint64_t v[U];
                bool valid[U];
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const long long i = base + (long long)u * blockDim.x + threadIdx.x;
                    valid[u] = i < n;
                    v[u] = valid[u] ? order_key(msv_dbits(__ldg(x + i))) : 0;
                }
#pragma unroll
                for (int u = 0; u < U; ++u) {
#pragma unroll
                    for (int q = 0; q < kMaxTails; ++q) {
                        if (st_r[q] >= 2) continue;
                        const bool hit = valid[u] && (pos_r[q] == 64 || (v[u] >> pos_r[q]) == pre_r[q]);
                        if (st_r[q] == 0) {
                            const unsigned bin = hit ? (unsigned)((v[u] >> sh_r[q]) & dmask_r[q]) : 0xffffffffu;
                            const unsigned peers = __match_any_sync(kFull, bin);
                            if (hit && lane == __ffs(peers) - 1) atomicAdd(&hbase[q * kBins + bin], (unsigned)__popc(peers));
                        } else {
                            const unsigned m = __ballot_sync(kFull, hit);
                            unsigned slot = 0;
                            if (lane == 0 && m) slot = atomicAdd(&S.fill[q], (unsigned)__popc(m));
                            slot = __shfl_sync(kFull, slot, 0);
                            if (hit) S.buf[q][slot + __popc(m & ((1u << lane) - 1u))] = v[u];
                        }
                    }
                }
            }
            __syncthreads();
            // ---- resolve every open percentile ----
            for (int q = 0; q < n_p; ++q) {
                const int st = S.state[q];
                if (st == 0) {
                    const int pos = S.pos[q];
                    const int d = pos < dig ? pos : dig;
                    const int nb = 1 << d;
                    const int per = (nb + blockDim.x - 1) / blockDim.x;
                    const int b0 = threadIdx.x * per;
                    unsigned int sum = 0;
                    const unsigned int* H = hbase + hsrc[q] * kBins;
                    for (int k = b0; k < b0 + per && k < nb; ++k) sum += H[k];
                    // read before the scan's barriers: the owning thread rewrites S.rank[q] below
                    const long long r = S.rank[q];
                    unsigned int total;
                    const unsigned int before = block_exclusive_scan(sum, S.warp_sum, &total);
                    if ((long long)before < r && r <= (long long)(before + sum)) {
                        unsigned int cum = before;
                        int k = b0;
                        for (; k < b0 + per; ++k) {
                            if ((long long)(cum + H[k]) >= r) break;
                            cum += H[k];
                        }
                        S.rank[q] = r - cum;
                        S.prefix[q] = ((pos == 64) ? 0ull : (S.prefix[q] << d)) | (uint64_t)k;
                        S.cnt[q] = H[k];
                        S.pos[q] = pos - d;
                    }
                    __syncthreads();
                    if (threadIdx.x == 0) {
                        if (S.pos[q] == 0) {
                            S.answer[q] = S.prefix[q];
                            S.state[q] = 2;
                        } else if (S.cnt[q] <= (unsigned)kTailGather) {
                            S.state[q] = 1;
                        }
                    }
                } else if (st == 1) {
                    const int cnt = (int)S.fill[q];
                    int np2 = 1;
                    while (np2 < cnt) np2 <<= 1;
                    for (int k = cnt + threadIdx.x; k < np2; k += blockDim.x) S.buf[q][k] = ~0ull;
                    __syncthreads();
                    bitonic_sort_smem(S.buf[q], np2);
                    if (threadIdx.x == 0) {
                        S.answer[q] = S.buf[q][S.rank[q] - 1];
                        S.state[q] = 2;
                    }
                }
                __syncthreads();
            }
        }
        if (threadIdx.x < n_p) J.out[threadIdx.x] = msv_bitsd(order_unkey(S.answer[threadIdx.x]));
        __syncthreads();
    }
}

}  // namespace

cudaError_t launch_tail(const TailJob* d_jobs, int n_jobs, const double* d_p, int n_p, cudaStream_t stream) {
    if (n_jobs <= 0) return cudaSuccess;
    if (n_p < 1 || n_p > kMaxTails) return cudaErrorInvalidValue;
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const size_t smem = sizeof(TailSmem);
    cudaError_t e = ensure_dyn_smem((const void*)tail_kernel, smem);
    if (e != cudaSuccess) return e;
    const int blocks = n_jobs < sms * 3 ? n_jobs : sms * 3;
    tail_kernel<<<blocks, kTailThreads, smem, stream>>>(d_jobs, n_jobs, d_p, n_p);
    return cudaGetLastError();
}

}  // namespace msv
