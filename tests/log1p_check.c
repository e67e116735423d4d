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

/* Host side of msv_log1p_digest: the same per-chunk digests with this process's libm
 * log1p (whichever build the ifunc picked), on n_threads threads. */
#include <pthread.h>

typedef struct {
    uint64_t seed;
    long n, chunk, c0, c1;
    uint64_t* out;
} digest_job;

static void* digest_worker(void* arg) {
    digest_job* J = (digest_job*)arg;
    for (long c = J->c0; c < J->c1; ++c) {
        uint64_t acc = 0;
        long hi = (c + 1) * J->chunk < J->n ? (c + 1) * J->chunk : J->n;
        for (long k = c * J->chunk; k < hi; ++k) {
            volatile double x = -msv_selftest_input(J->seed, (uint64_t)k);
            acc += msv_selftest_digest((uint64_t)k, -log1p(x));
        }
        J->out[c] = acc;
    }
    return 0;
}

int host_log1p_digest(uint64_t seed, long n, long chunk, uint64_t* out, int n_threads) {
    long n_chunks = (n + chunk - 1) / chunk;
    pthread_t th[256];
    digest_job jobs[256];
    if (n_threads < 1) n_threads = 1;
    if (n_threads > 256) n_threads = 256;
    for (int t = 0; t < n_threads; ++t) {
        jobs[t].seed = seed;
        jobs[t].n = n;
        jobs[t].chunk = chunk;
        jobs[t].c0 = n_chunks * t / n_threads;
        jobs[t].c1 = n_chunks * (t + 1) / n_threads;
        jobs[t].out = out;
        if (pthread_create(&th[t], 0, digest_worker, &jobs[t])) return -1;
    }
    for (int t = 0; t < n_threads; ++t) pthread_join(th[t], 0);
    return 0;
}

double host_log1p_value(uint64_t seed, long k) {
    volatile double x = -msv_selftest_input(seed, (uint64_t)k);
    return -log1p(x);
}
