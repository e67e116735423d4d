// K3 tail_kernel: tail_latency (metrics.hpp:22-29) — exact nearest-rank selection over
// order-preserving keys of the IEEE bit patterns, one block per scenario.
//
//   0. key bounds [kmin, kmax]: given by the producer (K5: min / max of the high words;
//      the segmented K2: [floor, horizon]) or taken here in one pass — on the planar
//      layout of the one-warp K2 (msv_internal.h) a pass over the high words only;
//   1. histogram pass: 8,192 bins of equal key width spanning [kmin, kmax], again
//      reading only the high words on the planar layout (4 bytes per sample). The bin
//      totals are checked against n: a key outside the bounds re-derives them;
//   2. one block scan locates every requested rank's bin (all percentiles share it);
//   3. gather pass: the keys of the chosen bins (a few thousand at 10^6 samples) go to
//      the scenario's dead overflow-link buffer, low words loaded only for them;
//   4. each percentile is settled inside its bin by 8-bit digit passes over those
//      candidates (L2-resident), each pass also taking their min and max, so a bin
//      of equal latencies (common: queries that never waited) ends after one pass.
// A bin larger than the candidate buffer falls back to step 4 over the full samples.
// Planar layout: three passes of 4 bytes per sample; plain doubles: 8 bytes per pass.
#include <type_traits>

#include "msv_device.cuh"

namespace msv {

namespace {

constexpr int kBins = 8192;      // histogram pass: 13-bit bins over the key range
constexpr int kDigitBins = 256;  // candidate passes: 8-bit digits
constexpr int kMaxTails = 4;
constexpr int kWarps = kTailThreads / 32;

struct TailSmem {
    unsigned int hist[kBins];
    unsigned int warp_sum[kWarps];
    unsigned long long kmin, kmax;  // histogram pass: key bounds
    unsigned long long rmin, rmax;  // candidate passes: min / max of the keys in range
    unsigned int qbin[kMaxTails];   // per percentile: its bin and its rank inside it (1-based)
    long long qrank[kMaxTails];
    int list[kMaxTails];            // per percentile: its candidate list
    unsigned int lbin[kMaxTails];   // per list: bin, offset in the candidates, gathered so far
    long long off[kMaxTails];
    long long cnt[kMaxTails];       // (the histogram is reused by the candidate passes)
    unsigned int fill[kMaxTails];
    int n_lists;
    long long n_cand;
    unsigned int sel_bin;           // select_in_range: the digit holding the rank
    long long sel_rank;
    unsigned long long answer[kMaxTails];
};

// Keys of a scenario's samples on either layout.
struct PlainSrc {  // consecutive doubles
    const double* x;
    __device__ __forceinline__ uint64_t key(long long j) const { return order_key(msv_dbits(__ldg(x + j))); }
};
struct PlanarSrc {  // msv_internal.h planar_hi_word: per 32 queries, 32 high then 32 low words
    const uint32_t* w;
    long long m0;
    __device__ __forceinline__ long long hi_at(long long j) const { return planar_hi_word(m0 + j); }
    __device__ __forceinline__ uint64_t key(long long j) const {
        const long long h = hi_at(j);
        return order_key(((uint64_t)__ldg(w + h) << 32) | __ldg(w + h + 32));
    }
};
struct KeySrc {  // candidate keys
    const uint64_t* k;
    __device__ __forceinline__ uint64_t key(long long j) const { return k[j]; }
};

__device__ __forceinline__ uint32_t hi_key(uint32_t h) { return (h & 0x80000000u) ? ~h : (h | 0x80000000u); }
__device__ __forceinline__ uint32_t lo_key(uint32_t h, uint32_t l) { return (h & 0x80000000u) ? ~l : l; }

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
    for (int w = 0; w < kWarps; ++w) {
        if (w < wid) before += warp_sum[w];
        all += warp_sum[w];
    }
    __syncthreads();
    *total = all;
    return before + x - v;
}

// Block-wide min / max of per-thread values into S.rmin / S.rmax (initialised by the caller).
__device__ __forceinline__ void block_range(uint64_t lo, uint64_t hi, TailSmem& S) {
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
        const uint64_t a = __shfl_xor_sync(kFull, lo, off), b = __shfl_xor_sync(kFull, hi, off);
        lo = a < lo ? a : lo;
        hi = b > hi ? b : hi;
    }
    if ((threadIdx.x & 31) == 0) {
        atomicMin(&S.rmin, (unsigned long long)lo);
        atomicMax(&S.rmax, (unsigned long long)hi);
    }
}

// Key bounds of all samples (one pass), for scenarios without bounds.
template <class Src>
__device__ void derive_bounds(const Src& src, long long n, TailSmem& S) {
    if (threadIdx.x == 0) {
        S.rmin = ~0ull;
        S.rmax = 0;
    }
    __syncthreads();
    uint64_t lo = ~0ull, hi = 0;
    if constexpr (std::is_same<Src, PlanarSrc>::value) {  // high words only: [min:0, max:ffffffff]
        uint32_t hl = 0xffffffffu, hh = 0;
        constexpr int U = 8;
        for (long long b0 = 0; b0 < n; b0 += (long long)blockDim.x * U) {
            uint32_t h[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const long long j = b0 + (long long)u * blockDim.x + threadIdx.x;
                h[u] = j < n ? hi_key(__ldg(src.w + src.hi_at(j))) : 0u;
                hl = (j < n && h[u] < hl) ? h[u] : hl;
                hh = h[u] > hh ? h[u] : hh;
            }
        }
        lo = hl <= hh ? (uint64_t)hl << 32 : ~0ull;
        hi = ((uint64_t)hh << 32) | 0xffffffffull;
    } else {
        for (long long j = threadIdx.x; j < n; j += blockDim.x) {
            const uint64_t k = src.key(j);
            lo = k < lo ? k : lo;
            hi = k > hi ? k : hi;
        }
    }
    block_range(lo, hi, S);
    __syncthreads();
    if (threadIdx.x == 0) {
        S.kmin = S.rmin;
        S.kmax = S.rmax;
    }
    __syncthreads();
}

// Histogram pass: hist[(key >> sh) - base] for keys inside the bins; HI: planar source,
// sh >= 32, only the high words are read. Identical bins of a warp are combined before
// the shared atomic (equal latencies are common).
template <class Src, bool HI>
__device__ void hist_pass(const Src& src, long long n, int sh, uint64_t base, TailSmem& S) {
    constexpr int U = HI ? 8 : 4;
    const int lane = threadIdx.x & 31;
    for (long long b0 = 0; b0 < n; b0 += (long long)blockDim.x * U) {
        uint64_t top[U];
        bool valid[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const long long j = b0 + (long long)u * blockDim.x + threadIdx.x;
            valid[u] = j < n;
            if constexpr (HI) {
                const uint32_t h = valid[u] ? __ldg(src.w + src.hi_at(j)) : 0u;
                top[u] = (uint64_t)hi_key(h) >> (sh - 32);
            } else {
                top[u] = valid[u] ? src.key(j) >> sh : 0;
            }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const uint64_t d = top[u] - base;
            const bool hit = valid[u] && d < (uint64_t)kBins;
            const unsigned bin = hit ? (unsigned)d : 0xffffffffu;
            const unsigned peers = __match_any_sync(kFull, bin);
            if (hit && lane == __ffs(peers) - 1) atomicAdd(&S.hist[bin], (unsigned)__popc(peers));
        }
    }
}

// Gather pass: keys whose (key >> sh) - base equals a list's bin go to that list.
template <class Src, bool HI>
__device__ void gather_pass(const Src& src, long long n, int sh, uint64_t base, uint64_t* cand, TailSmem& S) {
    constexpr int U = HI ? 8 : 4;
    const int lane = threadIdx.x & 31;
    const int n_lists = S.n_lists;
    unsigned tgt[kMaxTails];
#pragma unroll
    for (int l = 0; l < kMaxTails; ++l) tgt[l] = l < n_lists ? S.lbin[l] : 0xffffffffu;
    for (long long b0 = 0; b0 < n; b0 += (long long)blockDim.x * U) {
        uint64_t top[U];
        uint32_t hw[U];
        bool valid[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const long long j = b0 + (long long)u * blockDim.x + threadIdx.x;
            valid[u] = j < n;
            if constexpr (HI) {
                hw[u] = valid[u] ? __ldg(src.w + src.hi_at(j)) : 0u;
                top[u] = (uint64_t)hi_key(hw[u]) >> (sh - 32);
            } else {
                top[u] = valid[u] ? src.key(j) : 0;  // the full key; binned below
            }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const long long j = b0 + (long long)u * blockDim.x + threadIdx.x;
            const uint64_t d = (HI ? top[u] : top[u] >> sh) - base;
            const unsigned bin = valid[u] && d < (uint64_t)kBins ? (unsigned)d : 0xfffffffeu;
#pragma unroll
            for (int l = 0; l < kMaxTails; ++l) {
                if (l >= n_lists) break;
                const bool hit = bin == tgt[l];
                const unsigned m = __ballot_sync(kFull, hit);
                if (m == 0) continue;
                unsigned slot = 0;
                if (lane == __ffs(m) - 1) slot = atomicAdd(&S.fill[l], (unsigned)__popc(m));
                slot = __shfl_sync(kFull, slot, __ffs(m) - 1);
                if (hit) {
                    uint64_t k;
                    if constexpr (HI) k = ((uint64_t)hi_key(hw[u]) << 32) | lo_key(hw[u], __ldg(src.w + src.hi_at(j) + 32));
                    else k = top[u];
                    cand[S.off[l] + slot + __popc(m & ((1u << lane) - 1u))] = k;
                }
            }
        }
    }
}

// The r-th smallest (1-based) of the keys in [lo, hi] of src[0, n): 8-bit digit passes,
// each also taking the min / max of the keys in range. Block-uniform; returns on every thread.
template <class Src>
__device__ uint64_t select_in_range(const Src& src, long long n, uint64_t lo, uint64_t hi, long long r, TailSmem& S) {
    for (;;) {
        if (lo == hi) return lo;
        const int t = 64 - __clzll((long long)(lo ^ hi));
        const int sh = t > 8 ? t - 8 : 0;
        const uint64_t base = lo >> sh;
        for (int k = threadIdx.x; k < kDigitBins; k += blockDim.x) S.hist[k] = 0;
        if (threadIdx.x == 0) {
            S.rmin = ~0ull;
            S.rmax = 0;
        }
        __syncthreads();
        uint64_t mn = ~0ull, mx = 0;
        for (long long j = threadIdx.x; j < n; j += blockDim.x) {
            const uint64_t k = src.key(j);
            if (k >= lo && k <= hi) {
                atomicAdd(&S.hist[(unsigned)((k >> sh) - base)], 1u);
                mn = k < mn ? k : mn;
                mx = k > mx ? k : mx;
            }
        }
        block_range(mn, mx, S);
        __syncthreads();
        const uint64_t rmin = S.rmin, rmax = S.rmax;
        if (rmin == rmax || rmin > rmax) return rmin;  // all keys in range equal (or inconsistent input)
        // bin holding rank r (one bin per thread: kDigitBins <= kTailThreads)
        const unsigned v = threadIdx.x < kDigitBins ? S.hist[threadIdx.x] : 0u;
        unsigned int total;
        const unsigned before = block_exclusive_scan(v, S.warp_sum, &total);
        if ((long long)before < r && r <= (long long)(before + v)) {
            S.sel_bin = threadIdx.x;
            S.sel_rank = r - before;
        }
        __syncthreads();
        const uint64_t b = base + S.sel_bin;
        r = S.sel_rank;
        const uint64_t blo = b << sh, bhi = sh == 0 ? blo : (blo | ((1ull << sh) - 1));
        lo = blo > rmin ? blo : rmin;
        hi = bhi < rmax ? bhi : rmax;
        __syncthreads();
    }
}

template <class Src>
__device__ void select_job(const Src& src, long long n, const double* ps, int n_p, uint64_t* cand,
                           long long cand_cap, TailSmem& S) {
    constexpr bool kPlanar = std::is_same<Src, PlanarSrc>::value;
    if (S.kmin > S.kmax) derive_bounds(src, n, S);
    for (int attempt = 0;; ++attempt) {
        const uint64_t kmin = S.kmin, kmax = S.kmax;
        int sh = 0;
        while ((kmax >> sh) - (kmin >> sh) >= (uint64_t)kBins) ++sh;
        const uint64_t base = kmin >> sh;
        for (int k = threadIdx.x; k < kBins; k += blockDim.x) S.hist[k] = 0;
        __syncthreads();
        if constexpr (kPlanar) {
            if (sh >= 32) hist_pass<Src, true>(src, n, sh, base, S);
            else hist_pass<Src, false>(src, n, sh, base, S);
        } else {
            hist_pass<Src, false>(src, n, sh, base, S);
        }
        __syncthreads();
        // one scan for every percentile: kBins / kTailThreads bins per thread
        constexpr int per = kBins / kTailThreads;
        const int b0 = threadIdx.x * per;
        unsigned sum = 0;
#pragma unroll
        for (int k = 0; k < per; ++k) sum += S.hist[b0 + k];
        unsigned int total;
        const unsigned before = block_exclusive_scan(sum, S.warp_sum, &total);
        if ((long long)total != n) {  // a key outside the bounds: derive them and start over
            if (attempt > 0) {        // cannot happen with derived bounds
                if (threadIdx.x < n_p) S.answer[threadIdx.x] = order_key(0x7ff8000000000000ull);
                __syncthreads();
                return;
            }
            derive_bounds(src, n, S);
            continue;
        }
        for (int q = 0; q < n_p; ++q) {
            long long r = (long long)ceil(ps[q] * (double)n);  // metrics.hpp:26-27
            if (r < 1) r = 1;
            if ((long long)before < r && r <= (long long)(before + sum)) {
                unsigned cum = before;
                int k = b0;
                while ((long long)(cum + S.hist[k]) < r) cum += S.hist[k++];
                S.qbin[q] = (unsigned)k;
                S.qrank[q] = r - cum;
            }
        }
        __syncthreads();
        if (threadIdx.x == 0) {  // one candidate list per distinct bin
            int nl = 0;
            long long off = 0;
            for (int q = 0; q < n_p; ++q) {
                int l = 0;
                while (l < nl && S.lbin[l] != S.qbin[q]) ++l;
                if (l == nl) {
                    S.lbin[nl] = S.qbin[q];
                    S.off[nl] = off;
                    S.cnt[nl] = S.hist[S.qbin[q]];
                    S.fill[nl] = 0;
                    off += S.cnt[nl];
                    ++nl;
                }
                S.list[q] = l;
            }
            S.n_lists = nl;
            S.n_cand = off;
        }
        __syncthreads();
        const bool gathered = cand != nullptr && S.n_cand <= cand_cap;
        if (gathered) {
            if constexpr (kPlanar) {
                if (sh >= 32) gather_pass<Src, true>(src, n, sh, base, cand, S);
                else gather_pass<Src, false>(src, n, sh, base, cand, S);
            } else {
                gather_pass<Src, false>(src, n, sh, base, cand, S);
            }
            __syncthreads();
        }
        for (int q = 0; q < n_p; ++q) {
            const unsigned bin = S.qbin[q];
            const uint64_t blo = (base + bin) << sh;
            const uint64_t bhi = sh == 0 ? blo : (blo | ((1ull << sh) - 1));
            const uint64_t lo = blo > kmin ? blo : kmin, hi = bhi < kmax ? bhi : kmax;
            const long long r = S.qrank[q];
            uint64_t a;
            const int l = S.list[q];
            if (gathered) a = select_in_range(KeySrc{cand + S.off[l]}, S.cnt[l], lo, hi, r, S);
            else a = select_in_range(src, n, lo, hi, r, S);
            if (threadIdx.x == 0) S.answer[q] = a;
            __syncthreads();
        }
        return;
    }
}

__global__ void __launch_bounds__(kTailThreads)
    tail_kernel(const TailJob* __restrict__ jobs, int n_jobs, const double* __restrict__ ps, int n_p) {
    __shared__ TailSmem S;
    for (int jb = blockIdx.x; jb < n_jobs; jb += gridDim.x) {
        const TailJob J = jobs[jb];
        const DevOut src = *J.src;
        const long long n = src.n_samples;
        if (n == 0) {
            if (threadIdx.x < n_p) J.out[threadIdx.x] = __longlong_as_double(0x7ff8000000000000ll);
            continue;
        }
        if (threadIdx.x == 0) {
            S.kmin = src.lat_min_bits;
            S.kmax = src.lat_max_bits;
        }
        __syncthreads();
        if (src.planar) {
            const PlanarSrc v{reinterpret_cast<const uint32_t*>(J.samples), (long long)src.m0};
            select_job(v, n, ps, n_p, J.cand, J.cand_cap, S);
        } else {
            const PlainSrc v{J.samples + src.m0};  // the measured suffix
            select_job(v, n, ps, n_p, J.cand, J.cand_cap, S);
        }
        if (threadIdx.x < n_p) J.out[threadIdx.x] = msv_bitsd(order_unkey(S.answer[threadIdx.x]));
        __syncthreads();
    }
}

}  // namespace

cudaError_t launch_tail(const TailJob* d_jobs, int n_jobs, const double* d_p, int n_p, cudaStream_t stream) {
    if (n_jobs <= 0) return cudaSuccess;
    if (n_p < 1 || n_p > kMaxTails) return cudaErrorInvalidValue;
    // one block per scenario: while the next wave's simulation holds most of the SMs, K3's
    // blocks take whatever slots free up (a small persistent grid would stretch in time)
    const int blocks = n_jobs;
    tail_kernel<<<blocks, kTailThreads, 0, stream>>>(d_jobs, n_jobs, d_p, n_p);
    return cudaGetLastError();
}

}  // namespace msv
