// Bit-exact scalar pieces of the reference's trace generator, usable from CUDA
// device code and from host C/C++ (for the device-variant probe).
//
//   * std::mt19937_64 (libstdc++ / C++ standard) seeding, twist, tempering —
//     the engine behind migserve::Rng (rng.hpp:14, rng.hpp:35).
//   * Rng::uniform() = (x >> 11) * 2^-53                          (rng.hpp:17)
//   * glibc 2.39 log1p, both ifunc builds of sysdeps/ieee754/dbl-64/s_log1p.c
//     as shipped in Ubuntu's libm.so.6 (2.39-0ubuntu8.x):
//       - MSV_LOG1P_GENERIC: the SSE2 build (libm+0x2ef90), no FMA;
//       - MSV_LOG1P_FMA:     the FMA/AVX2 build (libm+0x7aff0), where gcc
//                            contracted six multiply-adds into vfmadd/vfmsub.
//     Rng::exponential() = -log1p(-u) / rate (rng.hpp:20) calls whichever build
//     the host's ifunc resolver (libm+0x2f300) picked, so the device carries both
//     and msv_create() probes the host libm to pick the matching one.
//   The op sequences below were transcribed from `objdump -d` of that libm (see
//   DESIGN.md "log1p"); every operation is a single IEEE-754 RN op, fused ops are
//   explicit fma() calls, and the translation units using this header are compiled
//   with contraction disabled (nvcc -fmad=false, gcc -ffp-contract=off).
#pragma once

#include <stdint.h>
#include <string.h>
#include <math.h>

#ifdef __CUDACC__
#define MSV_HD __host__ __device__ __forceinline__
#else
#define MSV_HD static inline
#endif

#define MSV_LOG1P_GENERIC 0
#define MSV_LOG1P_FMA 1

MSV_HD uint64_t msv_dbits(double x) {
#ifdef __CUDA_ARCH__
    return (uint64_t)__double_as_longlong(x);
#else
    uint64_t u;
    memcpy(&u, &x, 8);
    return u;
#endif
}

MSV_HD double msv_bitsd(uint64_t u) {
#ifdef __CUDA_ARCH__
    return __longlong_as_double((long long)u);
#else
    double x;
    memcpy(&x, &u, 8);
    return x;
#endif
}

MSV_HD double msv_fma(double a, double b, double c) {
#ifdef __CUDA_ARCH__
    return __fma_rn(a, b, c);
#else
    return fma(a, b, c);
#endif
}

// fdlibm constants (bit patterns read from libm's .rodata).
#define MSV_LN2_HI 6.93147180369123816490e-01   /* 3fe62e42 fee00000 */
#define MSV_LN2_LO 1.90821492927058770002e-10   /* 3dea39ef 35793c76 */
#define MSV_LP1 6.666666666666735130e-01        /* 3fe55555 55555593 */
#define MSV_LP2 3.999999999940941908e-01        /* 3fd99999 9997fa04 */
#define MSV_LP3 2.857142874366239149e-01        /* 3fd24924 94229359 */
#define MSV_LP4 2.222219843214978396e-01        /* 3fcc71c5 1d8e78af */
#define MSV_LP5 1.818357216161805012e-01        /* 3fc74664 96cb03de */
#define MSV_LP6 1.531383769920937332e-01        /* 3fc39a09 d078c69f */
#define MSV_LP7 1.479819860511658591e-01        /* 3fc2f112 df3e5244 */
#define MSV_TWO_THIRDS 6.6666666666666666e-01   /* 3fe55555 55555555 */

// log1p restricted to the domain the trace generator feeds it: x = -u with
// u = k * 2^-53, k in [0, 2^53), i.e. x in (-1, 0]. (|x| >= 1, +inf, NaN and
// x >= 0.41422 branches of the libm routine are unreachable from Rng.)
MSV_HD double msv_log1p_neg(double x, int variant) {
    const uint64_t bits = msv_dbits(x);
    const int32_t hx = (int32_t)(bits >> 32);
    const uint32_t ax = (uint32_t)hx & 0x7fffffffu;
    if (ax <= 0x3e1fffffu) {           // |x| < 2^-29
        if (ax <= 0x3c8fffffu) return x;  // |x| < 2^-54
        if (variant == MSV_LOG1P_FMA) return msv_fma(-(x * x), 0.5, x);
        return x - (x * x) * 0.5;
    }
    int k = 0;
    double f, c = 0.0;
    uint32_t hu = 1;
    if ((uint32_t)hx + 0x402d413cu <= 0x402d413cu) {  // x <= -0.2928932...: k path
        const double u = x + 1.0;
        const uint32_t hu0 = (uint32_t)(msv_dbits(u) >> 32);
        k = (int)(hu0 >> 20) - 1023;
        c = (k > 0) ? (1.0 - (u - x)) : (x - (u - 1.0));
        // c is often exactly +-0 (u = x + 1 exact) and 0 / u == c bit for bit; dividing
        // a stand-in 1.0 instead keeps the device division off its zero-operand slow path
        // (the select alone would still evaluate c / u)
        double cn = (c == 0.0) ? 1.0 : c;
#ifdef __CUDA_ARCH__
        asm("" : "+d"(cn));  // keep the compiler from folding the stand-in back into c / u
#endif
        const double cq = cn / u;
        c = (c == 0.0) ? c : cq;
        hu = hu0 & 0x000fffffu;
        const uint64_t lo = msv_dbits(u) & 0xffffffffull;
        double un;
        if (hu < 0x6a09eu) {
            un = msv_bitsd(((uint64_t)(hu | 0x3ff00000u) << 32) | lo);
        } else {
            k += 1;
            un = msv_bitsd(((uint64_t)(hu | 0x3fe00000u) << 32) | lo);
            hu = (0x00100000u - hu) >> 2;
        }
        f = un - 1.0;
    } else {
        f = x;
    }
    const double hfsq = (f * 0.5) * f;  // both builds: (0.5*f)*f
    if (hu == 0) {  // |f| < 2^-20
        if (f == 0.0) {
            if (k == 0) return 0.0;
            const double dk = (double)k;
            if (variant == MSV_LOG1P_FMA) return msv_fma(dk, MSV_LN2_HI, msv_fma(dk, MSV_LN2_LO, c));
            return (dk * MSV_LN2_LO + c) + dk * MSV_LN2_HI;
        }
        double R;
        if (variant == MSV_LOG1P_FMA)
            R = msv_fma(-f, MSV_TWO_THIRDS, 1.0) * hfsq;
        else
            R = (1.0 - MSV_TWO_THIRDS * f) * hfsq;
        if (k == 0) return f - R;
        const double dk = (double)k;
        if (variant == MSV_LOG1P_FMA)
            return msv_fma(dk, MSV_LN2_HI, -((R - msv_fma(dk, MSV_LN2_LO, c)) - f));
        return dk * MSV_LN2_HI - ((R - (dk * MSV_LN2_LO + c)) - f);
    }
    const double s = f / (f + 2.0);
    const double z = s * s;
    double R;
    if (variant == MSV_LOG1P_FMA) {
        const double R2 = msv_fma(z, MSV_LP3, MSV_LP2);
        const double R3 = msv_fma(z, MSV_LP5, MSV_LP4);
        const double R4 = msv_fma(z, MSV_LP7, MSV_LP6);
        const double z2 = z * z;
        const double z4 = z2 * z2;
        const double z6 = z2 * z4;
        const double t1 = msv_fma(z, MSV_LP1, z2 * R2);
        const double t2 = msv_fma(z4, R3, t1);
        R = msv_fma(z6, R4, t2);
    } else {
        const double R1 = z * MSV_LP1;
        const double z2 = z * z;
        const double R2 = MSV_LP2 + z * MSV_LP3;
        const double z4 = z2 * z2;
        const double z6 = z2 * z4;
        const double R3 = MSV_LP4 + z * MSV_LP5;
        const double R4 = MSV_LP6 + z * MSV_LP7;
        R = ((R1 + z2 * R2) + z4 * R3) + z6 * R4;
    }
    const double sv = (R + hfsq) * s;
    if (k == 0) return f - (hfsq - sv);
    const double dk = (double)k;
    if (variant == MSV_LOG1P_FMA)
        return msv_fma(dk, MSV_LN2_HI, -((hfsq - (msv_fma(dk, MSV_LN2_LO, c) + sv)) - f));
    return dk * MSV_LN2_HI - ((hfsq - (sv + (dk * MSV_LN2_LO + c))) - f);
}

// ---- std::mt19937_64 -------------------------------------------------------
#define MSV_MT_N 312
#define MSV_MT_M 156
#define MSV_MT_MATRIX 0xB5026F5AA96619E9ull
#define MSV_MT_UPPER 0xFFFFFFFF80000000ull
#define MSV_MT_LOWER 0x000000007FFFFFFFull

MSV_HD uint64_t msv_mt_next_seed(uint64_t prev, uint32_t i) {
    return 6364136223846793005ull * (prev ^ (prev >> 62)) + (uint64_t)i;
}

MSV_HD uint64_t msv_mt_twist(uint64_t cur, uint64_t nxt, uint64_t far) {
    const uint64_t y = (cur & MSV_MT_UPPER) | (nxt & MSV_MT_LOWER);
    return far ^ (y >> 1) ^ ((y & 1ull) ? MSV_MT_MATRIX : 0ull);
}

MSV_HD uint64_t msv_mt_temper(uint64_t y) {
    y ^= (y >> 29) & 0x5555555555555555ull;
    y ^= (y << 17) & 0x71D67FFFEDA60000ull;
    y ^= (y << 37) & 0xFFF7EEE000000000ull;
    y ^= (y >> 43);
    return y;
}

// Rng::uniform (rng.hpp:17)
MSV_HD double msv_uniform(uint64_t tempered) { return (double)(tempered >> 11) * 0x1.0p-53; }

// Order-independent per-query digest: the grid hash is the wrapping sum over all
// queries of mix(id, partition, start, finish), so the device (completion order)
// and the oracle (id order) agree without transferring per-query records.
MSV_HD uint64_t msv_mix64(uint64_t z) {
    z += 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

MSV_HD uint64_t msv_query_digest(uint64_t id, int32_t partition, double start, double finish) {
    // Checksum term of one query: both halves are odd-constant products of words that
    // mix the query's (id, partition) with its start/finish bits, so any change of one
    // query's placement or timing changes the grid's wrapping sum. 7 integer ops.
    const uint64_t sb = msv_dbits(start), fb = msv_dbits(finish);
    const uint32_t c = (uint32_t)id * 0x9E3779B1u + (uint32_t)partition;
    const uint32_t a = ((uint32_t)sb ^ (uint32_t)(fb >> 32) ^ c) * 0x85EBCA6Bu;
    const uint32_t b = ((uint32_t)(sb >> 32) ^ (uint32_t)fb ^ c) * 0x27D4EB2Fu + c;
    return ((uint64_t)a << 32) | b;
}

// ---- self-check inputs (msv_log1p_digest; the host checker tests/log1p_check.c) ----
MSV_HD uint64_t msv_splitmix64(uint64_t z) { return msv_mix64(z); }

// Input k of seed's stream on the generator's grid u = m * 2^-53 (Rng::uniform,
// rng.hpp:17): k mod 4 == 0/3 uniform m, 1 a right-shifted m (small u, log1p's tiny
// and intermediate ranges), 2 m close to 2^53 (u close to 1, large gaps).
MSV_HD double msv_selftest_input(uint64_t seed, uint64_t k) {
    const uint64_t x = msv_mix64(seed ^ (k * 0xD1B54A32D192ED03ull));
    uint64_t m = x >> 11;
    const uint64_t y = msv_mix64(x);
    if ((k & 3) == 1) m >>= (y & 63);
    if ((k & 3) == 2) m = (1ull << 53) - 1 - (m >> (y & 31));
    return (double)m * 0x1.0p-53;
}

// Digest term of result v of input k (wrapping sums of these are compared).
MSV_HD uint64_t msv_selftest_digest(uint64_t k, double v) { return msv_mix64(msv_dbits(v) ^ (k << 1)); }
