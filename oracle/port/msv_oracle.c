/*
 * TEST INFRASTRUCTURE ONLY — plain-C restatement of the reference's hot path,
 * used as an independent checker next to the compiled reference (oracle/_ref).
 * Never linked or called by the product. Build: oracle/build_oracle.py
 * (gcc -O2 -ffp-contract=off, glibc libm for log1p exactly like rng.hpp:20).
 *
 * Parity pin: tests/test_oracle.py checks this port against oracle/_ref (the
 * reference compiled from /root/reference) and against tests/golden/*.
 *
 * Restated functions (reference file:line):
 *   mt19937_64 + Rng::uniform/exponential ... rng.hpp:14-20 (libstdc++ <random>)
 *   BatchDistribution ctor / sample ........ workload.hpp:25-53
 *   sample_trace ............................ workload.hpp:97-113
 *   ProfileTable::cell lookups .............. profile.hpp:123-132
 *   t_wait .................................. sched.hpp:77-85
 *   elsa_dispatch ........................... sched.hpp:119-143
 *   fifs_dispatch ........................... sched.hpp:154-170
 *   run (event heap, EventAfter) ............ engine.hpp:93-253
 *   SimReport totals / latency_samples ...... engine.hpp:82-88, 233-252
 *   tail_latency ............................ metrics.hpp:22-29
 */
#include <math.h>
#include <pthread.h>
#include <stdatomic.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "../oracle_abi.h"

static _Thread_local char g_err[256];

static int set_err(int code, const char* msg) {
    snprintf(g_err, sizeof g_err, "%s", msg);
    return code;
}

const char* ora_last_error(void) { return g_err; }
const char* ora_kind(void) { return "port"; }

/* ---- std::mt19937_64 (C++ [rand.eng.mers]) ------------------------------ */
typedef struct {
    uint64_t x[312];
    int i;
} mt64;

static void mt_seed(mt64* m, uint64_t seed) {
    m->x[0] = seed;
    for (int i = 1; i < 312; ++i) m->x[i] = 6364136223846793005ull * (m->x[i - 1] ^ (m->x[i - 1] >> 62)) + (uint64_t)i;
    m->i = 312;
}

static uint64_t mt_next(mt64* m) {
    if (m->i >= 312) {
        for (int k = 0; k < 312; ++k) {
            uint64_t y = (m->x[k] & 0xFFFFFFFF80000000ull) | (m->x[(k + 1) % 312] & 0x7FFFFFFFull);
            m->x[k] = m->x[(k + 156) % 312] ^ (y >> 1) ^ ((y & 1ull) ? 0xB5026F5AA96619E9ull : 0ull);
        }
        m->i = 0;
    }
    uint64_t y = m->x[m->i++];
    y ^= (y >> 29) & 0x5555555555555555ull;
    y ^= (y << 17) & 0x71D67FFFEDA60000ull;
    y ^= (y << 37) & 0xFFF7EEE000000000ull;
    y ^= (y >> 43);
    return y;
}

static double rng_uniform(mt64* m) { return (double)(mt_next(m) >> 11) * 0x1.0p-53; } /* rng.hpp:17 */
static double rng_exponential(mt64* m, double rate) { return -log1p(-rng_uniform(m)) / rate; } /* rng.hpp:20 */

/* ---- BatchDistribution (workload.hpp:25-53) ----------------------------- */
int ora_dist_tables(const ora_dist* d, double* pmf, double* cdf) {
    if (d->b_max <= 0) return set_err(1, "batch distribution: empty support");
    double total = 0.0;
    for (int i = 0; i < d->b_max; ++i) {
        double w = d->weights[i];
        if (w < 0.0 || !isfinite(w)) return set_err(1, "batch distribution: weights must be finite and >= 0");
        total += w;
    }
    if (!(total > 0.0)) return set_err(1, "batch distribution: all weights are zero");
    double acc = 0.0;
    for (int i = 0; i < d->b_max; ++i) {
        pmf[i] = d->weights[i] / total;
        acc = (i == 0) ? pmf[0] : acc + pmf[i];
        cdf[i] = acc;
    }
    cdf[d->b_max - 1] = 1.0;
    return 0;
}

static int dist_sample(const double* cdf, int n, mt64* m) {
    double u = rng_uniform(m);
    int lo = 0; /* first index with !(cdf[i] < u) */
    while (lo < n && cdf[lo] < u) ++lo;
    if (lo == n) lo = n - 1;
    return lo + 1;
}

/* ---- sample_trace (workload.hpp:97-113) --------------------------------- */
int64_t ora_sample_trace(const ora_dist* d, double rate_qps, double duration_ms, uint64_t seed, int64_t cap,
                         double* arrival, int32_t* batch) {
    if (!(rate_qps > 0.0)) return -set_err(1, "sample_trace: rate must be > 0");
    if (duration_ms < 0.0) return -set_err(1, "sample_trace: duration must be >= 0");
    double* pmf = malloc(sizeof(double) * (size_t)d->b_max);
    double* cdf = malloc(sizeof(double) * (size_t)d->b_max);
    int rc = ora_dist_tables(d, pmf, cdf);
    if (rc) {
        free(pmf);
        free(cdf);
        return -rc;
    }
    mt64* m = malloc(sizeof(mt64));
    mt_seed(m, seed);
    const double rate_per_ms = rate_qps / 1000.0;
    double t = rng_exponential(m, rate_per_ms);
    int64_t n = 0;
    while (t < duration_ms) {
        int b = dist_sample(cdf, d->b_max, m);
        if (n < cap) {
            arrival[n] = t;
            batch[n] = b;
        }
        ++n;
        t += rng_exponential(m, rate_per_ms);
    }
    free(m);
    free(pmf);
    free(cdf);
    return n;
}

/* ---- profile lookups (profile.hpp:123-132) ------------------------------- */
static int cell(const ora_profile* p, int k, int b, size_t* out) {
    int lo = 0;
    while (lo < p->n_sizes && p->sizes[lo] < k) ++lo;
    if (lo == p->n_sizes || p->sizes[lo] != k) return set_err(4, "profile: unknown partition size");
    if (b < 1 || b > p->b_max) return set_err(4, "profile: batch outside grid");
    *out = (size_t)lo * (size_t)p->b_max + (size_t)(b - 1);
    return 0;
}

/* ---- engine state -------------------------------------------------------- */
typedef struct {
    int64_t q; /* query index */
    int batch;
    double est;
} qentry;

typedef struct {
    int id, k;
    qentry* ring;
    int64_t head, count, cap;
    int busy;
    int64_t cur_q;
    int cur_batch;
    double cur_est, cur_start;
} part;

static void q_push(part* p, qentry e) {
    if (p->count == p->cap) {
        int64_t nc = p->cap ? 2 * p->cap : 8;
        qentry* r = malloc(sizeof(qentry) * (size_t)nc);
        for (int64_t i = 0; i < p->count; ++i) r[i] = p->ring[(p->head + i) % p->cap];
        free(p->ring);
        p->ring = r;
        p->head = 0;
        p->cap = nc;
    }
    p->ring[(p->head + p->count) % p->cap] = e;
    p->count++;
}

static qentry q_pop(part* p) {
    qentry e = p->ring[p->head];
    p->head = (p->head + 1) % p->cap;
    p->count--;
    return e;
}

/* t_wait (sched.hpp:77-85): left fold over the FIFO, then the running remainder. */
static int t_wait(const part* p, const ora_profile* prof, double now, double* out) {
    double w = 0.0;
    for (int64_t i = 0; i < p->count; ++i) {
        size_t c;
        int rc = cell(prof, p->k, p->ring[(p->head + i) % p->cap].batch, &c);
        if (rc) return rc;
        w += prof->lat[c];
    }
    if (p->busy) {
        double elapsed = now - p->cur_start;
        double x = p->cur_est - elapsed;
        w += (0.0 < x) ? x : 0.0; /* std::max(0.0, x) */
    }
    *out = w;
    return 0;
}

/* Events ordered by EventAfter (engine.hpp:101-107): time, completion first, seq. */
typedef struct {
    double t;
    int type; /* 0 completion, 1 arrival */
    uint64_t seq;
    int pid;
    int64_t q;
} event;

static int ev_before(const event* a, const event* b) {
    if (a->t != b->t) return a->t < b->t;
    if (a->type != b->type) return a->type < b->type;
    return a->seq < b->seq;
}

typedef struct {
    event* v;
    int64_t n, cap;
} heap;

static void h_push(heap* h, event e) {
    if (h->n == h->cap) {
        h->cap = h->cap ? 2 * h->cap : 64;
        h->v = realloc(h->v, sizeof(event) * (size_t)h->cap);
    }
    int64_t i = h->n++;
    h->v[i] = e;
    while (i > 0) {
        int64_t par = (i - 1) / 2;
        if (!ev_before(&h->v[i], &h->v[par])) break;
        event tmp = h->v[i];
        h->v[i] = h->v[par];
        h->v[par] = tmp;
        i = par;
    }
}

static event h_pop(heap* h) {
    event top = h->v[0];
    h->v[0] = h->v[--h->n];
    int64_t i = 0;
    for (;;) {
        int64_t l = 2 * i + 1, r = l + 1, m = i;
        if (l < h->n && ev_before(&h->v[l], &h->v[m])) m = l;
        if (r < h->n && ev_before(&h->v[r], &h->v[m])) m = r;
        if (m == i) break;
        event tmp = h->v[i];
        h->v[i] = h->v[m];
        h->v[m] = tmp;
        i = m;
    }
    return top;
}

int ora_run(const ora_plan* plan, int scheduler, const double* arrival, const int32_t* batch, int64_t n,
            double duration_ms, const ora_profile* prof, double sla, double alpha, double beta,
            double warmup_fraction, int check_wait, int n_route, const int32_t* route_k,
            const int32_t* route_first, const int32_t* route_last, ora_records* rec, ora_report* rep) {
    /* argument checks, engine.hpp:118-124 / sched.hpp:44-47 / paris.hpp:141-156 */
    if (plan->num_gpus < 1) return set_err(3, "plan: num_gpus must be >= 1");
    if (plan->gpcs_per_gpu < 1) return set_err(3, "plan: gpcs_per_gpu must be >= 1");
    int P = 0;
    for (int g = 0; g < plan->num_gpus; ++g) {
        int used = 0;
        for (int j = 0; j < plan->n_per_gpu[g]; ++j) {
            int k = plan->sizes_flat[P + j];
            if (k < 1) return set_err(3, "plan: partition size must be positive");
            used += k;
        }
        if (used > plan->gpcs_per_gpu) return set_err(3, "plan: GPU over capacity");
        P += plan->n_per_gpu[g];
    }
    if (!(sla > 0.0)) return set_err(1, "sla: target must be > 0");
    if (alpha < 0.0 || beta < 0.0) return set_err(1, "sla: alpha/beta must be >= 0");
    if (P == 0) return set_err(1, "run: plan has no partition instances");
    if (warmup_fraction < 0.0 || warmup_fraction >= 1.0) return set_err(1, "run: warmup_fraction must be in [0,1)");
    if (n_route == 0 && route_k) return set_err(1, "run: segment_routing enabled without segments");

    part* ps = calloc((size_t)P, sizeof(part));
    for (int j = 0; j < P; ++j) {
        ps[j].id = j;
        ps[j].k = plan->sizes_flat[j];
    }
    /* static (k asc, id asc) order (sched.hpp:96-104) */
    int* order = malloc(sizeof(int) * (size_t)P);
    for (int j = 0; j < P; ++j) order[j] = j;
    for (int a = 1; a < P; ++a) {
        int x = order[a], b = a;
        while (b > 0 && (ps[order[b - 1]].k > ps[x].k || (ps[order[b - 1]].k == ps[x].k && ps[order[b - 1]].id > ps[x].id))) {
            order[b] = order[b - 1];
            --b;
        }
        order[b] = x;
    }
    double* busy_ms = calloc((size_t)P, sizeof(double));
    double* wbusy = calloc((size_t)P, sizeof(double));
    int64_t* nq = calloc((size_t)P, sizeof(int64_t));
    double* completion_at = calloc((size_t)P, sizeof(double));
    double* finish = malloc(sizeof(double) * (size_t)(n ? n : 1));
    double* start = malloc(sizeof(double) * (size_t)(n ? n : 1));
    int32_t* partition = malloc(sizeof(int32_t) * (size_t)(n ? n : 1));
    int32_t* kind = malloc(sizeof(int32_t) * (size_t)(n ? n : 1));
    int* cand = malloc(sizeof(int) * (size_t)P);
    heap h = {0};
    uint64_t seq = 0;
    for (int64_t i = 0; i < n; ++i) {
        event e = {arrival[i], 1, seq++, -1, i};
        h_push(&h, e);
    }
    double last_finish = 0.0, max_wait_diff = 0.0;
    int rc = 0;
    while (h.n > 0 && rc == 0) {
        event ev = h_pop(&h);
        const double now = ev.t;
        if (ev.type == 0) { /* completion, engine.hpp:167-187 */
            part* p = &ps[ev.pid];
            int64_t q = p->cur_q;
            finish[q] = now;
            double ran = now - p->cur_start;
            size_t c;
            rc = cell(prof, p->k, p->cur_batch, &c);
            if (rc) break;
            busy_ms[p->id] += ran;
            wbusy[p->id] += ran * prof->util[c];
            nq[p->id] += 1;
            last_finish = (last_finish < now) ? now : last_finish;
            p->busy = 0;
            if (p->count > 0) {
                qentry e = q_pop(p);
                p->busy = 1;
                p->cur_q = e.q;
                p->cur_batch = e.batch;
                p->cur_est = e.est;
                p->cur_start = now;
                completion_at[p->id] = now + e.est;
                start[e.q] = now;
                event ce = {now + e.est, 0, seq++, p->id, e.q};
                h_push(&h, ce);
            }
            continue;
        }
        /* arrival, engine.hpp:189-230 */
        const int64_t qi = ev.q;
        const int b = batch[qi];
        int nc = 0;
        if (n_route > 0) {
            for (int j = 0; j < P; ++j)
                for (int s = 0; s < n_route; ++s)
                    if (route_k[s] == ps[j].k && b >= route_first[s] && b <= route_last[s]) {
                        cand[nc++] = j;
                        break;
                    }
        }
        if (nc == 0)
            for (int j = 0; j < P; ++j) cand[nc++] = j;
        if (check_wait) { /* engine.hpp:208-217 */
            for (int c2 = 0; c2 < nc; ++c2) {
                part* p = &ps[cand[c2]];
                double gt = 0.0;
                for (int64_t i = 0; i < p->count; ++i) gt += p->ring[(p->head + i) % p->cap].est;
                if (p->busy) {
                    double y = completion_at[p->id] - now;
                    gt += (0.0 < y) ? y : 0.0;
                }
                double est;
                if ((rc = t_wait(p, prof, now, &est))) break;
                double d = fabs(gt - est);
                max_wait_diff = (max_wait_diff < d) ? d : max_wait_diff;
            }
            if (rc) break;
        }
        int chosen = -1, kd = 0;
        if (scheduler) { /* elsa_dispatch, sched.hpp:119-143 */
            for (int o = 0; o < P && chosen < 0; ++o) {
                int j = order[o];
                int is_c = 0;
                for (int c2 = 0; c2 < nc; ++c2) is_c |= cand[c2] == j;
                if (!is_c) continue;
                size_t c;
                if ((rc = cell(prof, ps[j].k, b, &c))) break;
                double est = prof->lat[c], w;
                if ((rc = t_wait(&ps[j], prof, now, &w))) break;
                if (sla > alpha * (w + beta * est)) {
                    chosen = j;
                    kd = 0;
                }
            }
            if (rc) break;
            if (chosen < 0) {
                double best = INFINITY;
                for (int o = 0; o < P; ++o) {
                    int j = order[o];
                    int is_c = 0;
                    for (int c2 = 0; c2 < nc; ++c2) is_c |= cand[c2] == j;
                    if (!is_c) continue;
                    if (chosen < 0) chosen = j; /* order.front() of the candidates */
                    size_t c;
                    double w;
                    if ((rc = cell(prof, ps[j].k, b, &c)) || (rc = t_wait(&ps[j], prof, now, &w))) break;
                    double fin = w + prof->lat[c];
                    if (fin < best) {
                        best = fin;
                        chosen = j;
                    }
                }
                if (rc) break;
                kd = 1;
            }
        } else { /* fifs_dispatch, sched.hpp:154-170 */
            int idle = -1;
            for (int c2 = 0; c2 < nc; ++c2) {
                part* p = &ps[cand[c2]];
                if (p->busy) continue;
                if (idle < 0 || p->k > ps[idle].k || (p->k == ps[idle].k && p->id < ps[idle].id)) idle = cand[c2];
            }
            if (idle >= 0) {
                chosen = idle;
                kd = 2;
            } else {
                int best = cand[0];
                for (int c2 = 0; c2 < nc; ++c2) {
                    part* p = &ps[cand[c2]];
                    if (p->count < ps[best].count || (p->count == ps[best].count && p->id < ps[best].id)) best = cand[c2];
                }
                chosen = best;
                kd = 3;
            }
        }
        partition[qi] = chosen;
        kind[qi] = kd;
        part* p = &ps[chosen];
        size_t c;
        if ((rc = cell(prof, p->k, b, &c))) break;
        qentry e = {qi, b, prof->lat[c]};
        if (p->busy) {
            q_push(p, e);
        } else {
            p->busy = 1;
            p->cur_q = qi;
            p->cur_batch = b;
            p->cur_est = e.est;
            p->cur_start = now;
            completion_at[p->id] = now + e.est;
            start[qi] = now;
            event ce = {now + e.est, 0, seq++, p->id, qi};
            h_push(&h, ce);
        }
    }
    if (rc == 0) {
        const double warmup_ms = warmup_fraction * duration_ms; /* engine.hpp:238 */
        int64_t viol = 0, meas = 0, mviol = 0;
        for (int64_t i = 0; i < n; ++i) {
            double lat = finish[i] - arrival[i];
            int met = lat <= sla;
            if (!met) ++viol;
            if (arrival[i] >= warmup_ms) {
                ++meas;
                if (!met) ++mviol;
            }
            if (rec) {
                rec->partition[i] = partition[i];
                rec->start_ms[i] = start[i];
                rec->finish_ms[i] = finish[i];
                rec->kind[i] = kind[i];
            }
        }
        if (rep) {
            rep->total = n;
            rep->violations = viol;
            rep->measured = meas;
            rep->measured_violations = mviol;
            rep->horizon_ms = (duration_ms < last_finish) ? last_finish : duration_ms;
            rep->warmup_ms = warmup_ms;
            rep->max_wait_estimate_diff = max_wait_diff;
            for (int j = 0; j < P; ++j) {
                if (rep->busy_ms) rep->busy_ms[j] = busy_ms[j];
                if (rep->weighted_busy_ms) rep->weighted_busy_ms[j] = wbusy[j];
                if (rep->queries) rep->queries[j] = nq[j];
            }
        }
    }
    for (int j = 0; j < P; ++j) free(ps[j].ring);
    free(ps);
    free(order);
    free(busy_ms);
    free(wbusy);
    free(nq);
    free(completion_at);
    free(finish);
    free(start);
    free(partition);
    free(kind);
    free(cand);
    free(h.v);
    return rc;
}

/* ---- tail_latency (metrics.hpp:22-29) ------------------------------------ */
static int cmp_double(const void* a, const void* b) {
    double x = *(const double*)a, y = *(const double*)b;
    return (x > y) - (x < y);
}

int ora_tail_latency(const double* samples, int64_t n, double p, double* out) {
    if (n <= 0) return set_err(1, "tail_latency: no samples");
    if (!(p > 0.0) || !(p < 1.0)) return set_err(1, "tail_latency: percentile must be in (0,1)");
    double* s = malloc(sizeof(double) * (size_t)n);
    memcpy(s, samples, sizeof(double) * (size_t)n);
    qsort(s, (size_t)n, sizeof(double), cmp_double);
    size_t rank = (size_t)ceil(p * (double)n);
    if (rank < 1) rank = 1;
    *out = s[rank - 1];
    free(s);
    return 0;
}

/* ---- grid: sample_trace -> run -> latency_samples -> tail_latency ---------- */
typedef struct {
    const ora_profile* profs;
    const ora_dist* dists;
    const ora_plan* plans;
    const ora_scenario* sc;
    int64_t n;
    const double* ps;
    int n_p;
    ora_result* out;
    atomic_llong next;
} grid_job;

static void grid_one(grid_job* J, int64_t i) {
    const ora_scenario* s = &J->sc[i];
    ora_result* r = &J->out[i];
    memset(r, 0, sizeof *r);
    for (int j = 0; j < 4; ++j) r->tail[j] = NAN;
    const ora_dist* d = &J->dists[s->dist];
    double mean = s->rate_qps * s->duration_ms / 1000.0;
    int64_t cap = (int64_t)(mean + 12.0 * sqrt(mean) + 256.0);
    double* arr = malloc(sizeof(double) * (size_t)cap);
    int32_t* bat = malloc(sizeof(int32_t) * (size_t)cap);
    int64_t n = ora_sample_trace(d, s->rate_qps, s->duration_ms, s->seed, cap, arr, bat);
    if (n > cap) {
        free(arr);
        free(bat);
        cap = n;
        arr = malloc(sizeof(double) * (size_t)cap);
        bat = malloc(sizeof(int32_t) * (size_t)cap);
        n = ora_sample_trace(d, s->rate_qps, s->duration_ms, s->seed, cap, arr, bat);
    }
    if (n < 0) {
        r->status = (int32_t)(-n);
        free(arr);
        free(bat);
        return;
    }
    size_t nn = (size_t)(n ? n : 1);
    ora_records rec = {malloc(sizeof(int32_t) * nn), malloc(sizeof(double) * nn), malloc(sizeof(double) * nn),
                       malloc(sizeof(int32_t) * nn)};
    ora_report rep;
    memset(&rep, 0, sizeof rep);
    int rc = ora_run(&J->plans[s->plan], s->scheduler, arr, bat, n, s->duration_ms, &J->profs[s->profile], s->sla_ms,
                     s->alpha, s->beta, s->warmup_fraction, 0, -1, NULL, NULL, NULL, &rec, &rep);
    if (rc) {
        r->status = rc;
    } else {
        r->total = rep.total;
        r->violations = rep.violations;
        r->measured = rep.measured;
        r->measured_violations = rep.measured_violations;
        r->horizon_ms = rep.horizon_ms;
        uint64_t h = 0;
        double* samples = malloc(sizeof(double) * nn);
        int64_t m = 0;
        for (int64_t q = 0; q < n; ++q) {
            h += ora_query_digest((uint64_t)q, rec.partition[q], rec.start_ms[q], rec.finish_ms[q]);
            if (arr[q] >= rep.warmup_ms) samples[m++] = rec.finish_ms[q] - arr[q];
        }
        r->placement_hash = h;
        for (int j = 0; j < J->n_p && j < 4 && m > 0; ++j) ora_tail_latency(samples, m, J->ps[j], &r->tail[j]);
        free(samples);
    }
    free(rec.partition);
    free(rec.start_ms);
    free(rec.finish_ms);
    free(rec.kind);
    free(arr);
    free(bat);
}

static void* grid_worker(void* arg) {
    grid_job* J = arg;
    for (;;) {
        int64_t i = atomic_fetch_add(&J->next, 1);
        if (i >= J->n) return NULL;
        grid_one(J, i);
    }
}

int ora_run_grid(const ora_profile* profs, const ora_dist* dists, const ora_plan* plans, const ora_scenario* sc,
                 int64_t n, const double* ps, int n_p, int n_threads, ora_result* out) {
    grid_job J = {profs, dists, plans, sc, n, ps, n_p, out, 0};
    if (n_threads <= 1) {
        grid_worker(&J);
        return 0;
    }
    pthread_t* th = malloc(sizeof(pthread_t) * (size_t)n_threads);
    for (int t = 0; t < n_threads; ++t) pthread_create(&th[t], NULL, grid_worker, &J);
    for (int t = 0; t < n_threads; ++t) pthread_join(th[t], NULL);
    free(th);
    return 0;
}
