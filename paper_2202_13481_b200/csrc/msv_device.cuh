// Device helpers shared by the kernels. Every .cu of the engine is compiled with
// -fmad=false: decision and accumulation expressions must round exactly like the
// reference's x86-64 SSE2 build (no contraction).
#pragma once

#include <math.h>

#include "msv_internal.h"
#include "msv_math.h"

namespace msv {

constexpr unsigned kFull = 0xffffffffu;
constexpr uint64_t kSignBit = 1ull << 63;

// Explicit 32-bit shared-memory addressing. `opaque` hides a value's provenance from
// the compiler so a per-lane shared base stays in one register instead of being
// re-derived from special registers (SR_TID, SR_CgaCtaId) at every use.
__device__ __forceinline__ uint32_t opaque(uint32_t x) {
    asm volatile("" : "+r"(x));
    return x;
}
__device__ __forceinline__ uint32_t smem_addr(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ double lds_f64(uint32_t a) {
    double v;
    asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(a));
    return v;
}
__device__ __forceinline__ uint64_t lds_u64(uint32_t a) {
    uint64_t v;
    asm volatile("ld.shared.u64 %0, [%1];" : "=l"(v) : "r"(a));
    return v;
}
__device__ __forceinline__ int32_t lds_s32(uint32_t a) {
    int32_t v;
    asm volatile("ld.shared.s32 %0, [%1];" : "=r"(v) : "r"(a));
    return v;
}
__device__ __forceinline__ uint32_t lds_u32(uint32_t a) {
    uint32_t v;
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a));
    return v;
}
__device__ __forceinline__ void sts_f64(uint32_t a, double v) {
    asm volatile("st.shared.f64 [%0], %1;" ::"r"(a), "d"(v) : "memory");
}
__device__ __forceinline__ void sts_u64(uint32_t a, uint64_t v) {
    asm volatile("st.shared.u64 [%0], %1;" ::"r"(a), "l"(v) : "memory");
}
__device__ __forceinline__ void sts_u32(uint32_t a, uint32_t v) {
    asm volatile("st.shared.u32 [%0], %1;" ::"r"(a), "r"(v) : "memory");
}

// (0.0 < x) ? x : 0.0 — Eq. 1's max(0, est - (now - start)) as the reference writes it
// (std::max(0.0, x), sched.hpp:83): one compare and a 64-bit select (the compiler's own
// lowering of the pattern goes through fmax with NaN fix-ups and register moves).
__device__ __forceinline__ double pos_part(double x) {
    double r;
    asm("{\n\t.reg .pred p;\n\tsetp.gt.f64 p, %1, 0d0000000000000000;\n\tselp.f64 %0, %1, 0d0000000000000000, p;\n\t}"
        : "=d"(r)
        : "d"(x));
    return r;
}

// Eq. 1's current-query term (sched.hpp:82-83): max(0, est - (now - start)) if the
// partition is running a query at `now` (its finish > now; a finish <= now has
// completed, completions precede arrivals), else 0 — two compares, one 64-bit select.
__device__ __forceinline__ double running_part(double finish, double now, double x) {
    double r;
    asm("{\n\t.reg .pred p;\n\tsetp.gt.f64 p, %1, %2;\n\tsetp.gt.and.f64 p, %3, 0d0000000000000000, p;"
        "\n\tselp.f64 %0, %3, 0d0000000000000000, p;\n\t}"
        : "=d"(r)
        : "d"(finish), "d"(now), "d"(x));
    return r;
}

// c ? a : b on doubles as one predicated 64-bit select.
__device__ __forceinline__ double sel_f64(bool c, double a, double b) {
    double r;
    asm("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %3, 0;\n\tselp.f64 %0, %1, %2, p;\n\t}"
        : "=d"(r)
        : "d"(a), "d"(b), "r"((int)c));
    return r;
}

// Order-preserving map of IEEE doubles onto uint64 (total order of finite values).
__device__ __forceinline__ uint64_t order_key(uint64_t b) { return (b & kSignBit) ? ~b : (b | kSignBit); }
__device__ __forceinline__ uint64_t order_unkey(uint64_t k) { return (k & kSignBit) ? (k & ~kSignBit) : ~k; }

// Minimum over the W-lane segment of a warp; every lane of the warp must call it.
template <int W>
__device__ __forceinline__ uint32_t seg_min_u32(uint32_t v) {
    if constexpr (W == 32) {
        return __reduce_min_sync(kFull, v);
    } else {
#pragma unroll
        for (int off = W / 2; off > 0; off >>= 1) {
            const uint32_t o = __shfl_xor_sync(kFull, v, off);
            v = o < v ? o : v;
        }
        return v;
    }
}

// Minimum of non-negative IEEE bit patterns (or ~0 sentinels) over a segment.
template <int W>
__device__ __forceinline__ uint64_t seg_min_u64(uint64_t v) {
    if constexpr (W == 32) {
        const uint32_t hi = (uint32_t)(v >> 32);
        const uint32_t mh = __reduce_min_sync(kFull, hi);
        const uint32_t lo = (hi == mh) ? (uint32_t)v : 0xffffffffu;
        const uint32_t ml = __reduce_min_sync(kFull, lo);
        return ((uint64_t)mh << 32) | ml;
    } else {
#pragma unroll
        for (int off = W / 2; off > 0; off >>= 1) {
            const uint64_t o = __shfl_xor_sync(kFull, v, off);
            v = o < v ? o : v;
        }
        return v;
    }
}

// Segment-masked reductions for segment-uniform branches (only that segment's lanes).
template <int W>
__device__ __forceinline__ uint64_t seg_sum_u64(uint64_t v, unsigned mask) {
#pragma unroll
    for (int off = W / 2; off > 0; off >>= 1) v += __shfl_xor_sync(mask, v, off);
    return v;
}
template <int W>
__device__ __forceinline__ uint64_t seg_max_u64(uint64_t v, unsigned mask) {
#pragma unroll
    for (int off = W / 2; off > 0; off >>= 1) {
        const uint64_t o = __shfl_xor_sync(mask, v, off);
        v = o > v ? o : v;
    }
    return v;
}
template <int W>
__device__ __forceinline__ uint64_t seg_minm_u64(uint64_t v, unsigned mask) {
#pragma unroll
    for (int off = W / 2; off > 0; off >>= 1) {
        const uint64_t o = __shfl_xor_sync(mask, v, off);
        v = o < v ? o : v;
    }
    return v;
}
// Minimum and maximum of u32 values over a segment (segment-uniform branches).
template <int W>
__device__ __forceinline__ void seg_range_u32(uint32_t& lo, uint32_t& hi, unsigned mask) {
    if constexpr (W == 32) {
        lo = __reduce_min_sync(mask, lo);
        hi = __reduce_max_sync(mask, hi);
    } else {
#pragma unroll
        for (int off = W / 2; off > 0; off >>= 1) {
            const uint32_t a = __shfl_xor_sync(mask, lo, off), b = __shfl_xor_sync(mask, hi, off);
            lo = a < lo ? a : lo;
            hi = b > hi ? b : hi;
        }
    }
}

// K3 key bounds from the high words of a scenario's (non-negative) latencies: every
// latency's order key lies in [min_hi:00000000, max_hi:ffffffff]. With no latency
// (lo > hi) the bounds come out empty (min > max) and K3 derives them itself.
__device__ __forceinline__ void lat_key_bounds(uint32_t hmin, uint32_t hmax, uint64_t& kmin, uint64_t& kmax) {
    if (hmin > hmax) {
        kmin = ~0ull;
        kmax = 0;
        return;
    }
    kmin = (uint64_t)(hmin | 0x80000000u) << 32;
    kmax = ((uint64_t)(hmax | 0x80000000u) << 32) | 0xffffffffull;
}

// std::max on doubles as the reference writes it: (a < b) ? b : a.
template <int W>
__device__ __forceinline__ double seg_max_f64(double v, unsigned mask) {
#pragma unroll
    for (int off = W / 2; off > 0; off >>= 1) {
        const double o = __shfl_xor_sync(mask, v, off);
        v = (v < o) ? o : v;
    }
    return v;
}

}  // namespace msv
