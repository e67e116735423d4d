/* Host-side check of the device's glibc-log1p transcription (csrc/msv_math.h)
 * against this process's libm log1p. Test infrastructure. */
#include <math.h>
#include "../paper_2202_13481_b200/csrc/msv_math.h"

static uint64_t xs(uint64_t* s) {
    *s ^= *s << 13;
    *s ^= *s >> 7;
    *s ^= *s << 17;
    return *s;
}

/* inputs spread over the generator's whole domain u = k * 2^-53 */
static double draw(uint64_t* s, long i) {
    uint64_t m = xs(s) >> 11;
    if (i % 4 == 1) m >>= (xs(s) & 63);
    if (i % 4 == 2) m = (1ull << 53) - 1 - (m >> (xs(s) & 31));
    return (double)m * 0x1.0p-53;
}

long check_log1p(int variant, long n, uint64_t seed) {
    long bad = 0;
    uint64_t s = seed | 1;
    for (long i = 0; i < n; ++i) {
        volatile double x = -draw(&s, i);
        if (msv_dbits(log1p(x)) != msv_dbits(msv_log1p_neg(x, variant))) ++bad;
    }
    return bad;
}

long variants_differ(long n, uint64_t seed) {
    long d = 0;
    uint64_t s = seed | 1;
    for (long i = 0; i < n; ++i) {
        double x = -draw(&s, i);
        if (msv_dbits(msv_log1p_neg(x, 0)) != msv_dbits(msv_log1p_neg(x, 1))) ++d;
    }
    return d;
}

int host_variant(void) {
    uint64_t s = 99;
    int f = 0, g = 0;
    for (long i = 0; i < 4000000 && f + g < 16; ++i) {
        double x = -draw(&s, i);
        double a = msv_log1p_neg(x, 1), b = msv_log1p_neg(x, 0);
        if (msv_dbits(a) == msv_dbits(b)) continue;
        volatile double xi = x;
        double h = log1p(xi);
        if (msv_dbits(h) == msv_dbits(a)) ++f;
        else if (msv_dbits(h) == msv_dbits(b)) ++g;
    }
    return g > f ? 0 : 1;
}
