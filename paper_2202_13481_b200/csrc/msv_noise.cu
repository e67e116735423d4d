// K5 sim_noise_kernel: run() (engine.hpp:115-253) with execution noise
// (EngineOptions::noise_sigma > 0, engine.hpp:140-145): every start draws the next
// Rng(noise_seed).normal() and runs for est * exp(sigma*z - sigma^2/2) instead of est.
//
// The noise-free kernels rely on the drain rule: completions on
// different partitions commute, so each lane retires its own chain. With noise they do
// not: the j-th start takes the j-th draw, so starts must happen in the reference's global
// event order — (time asc, completion before arrival, seq asc), seq = push order
// (engine.hpp:93-107, :134-137). This kernel keeps that order exactly:
//   * one warp per scenario, lane slot s of lane l = by_ascending_size index s*32 + l
//     (sched.hpp:96-104), P <= 128 (one, two or four slots per lane);
//   * before each arrival (and after the last) the warp repeatedly takes the global
//     minimum (completion time, seq) over the slots with completion <= t — a shuffle
//     argmin — and retires it; a queue head started there takes the next multiplier and
//     the next seq, so a chain of starts inside one drain keeps the heap's order;
//   * ELSA / FIFS decisions are msv_sim_warp.cu's (ballot Step A in scan order, shuffle
//     argmin Step B, FIFS key reductions), on the same exact left fold of Eq. 1;
//   * the multipliers exp(sigma*z_j - sigma^2/2) are an input stream drawn by the caller
//     with the reference's Rng (rng.hpp:27-31) and libm, like a replayed trace: the device
//     consumes multiplier j at the j-th start (est * m_j, one RN multiply, engine.hpp:144).
// Compiled with -fmad=false like every decision path (Appendix A.13).
#include <math_constants.h>

#include "msv_device.cuh"

namespace msv {

namespace {

// S slots per lane (P <= 32 * S); RING queued latencies per slot cached in shared memory:
// S = 1 (P <= 32) with a 128-entry ring, S = 2 with 64, S = 4 (P <= 128) with 32 — 32 KB each.
template <int S, int RING>
__global__ void __launch_bounds__(32, 1) sim_noise_kernel(const NoiseParams* __restrict__ jobs) {
    constexpr int kRing = RING;
    const NoiseParams& p = jobs[blockIdx.x];
    const int lane = threadIdx.x & 31;
    const double* __restrict__ arr = p.arrival;
    const int32_t* __restrict__ bat = p.batch;
    // the profile's latency / utilisation cells in shared memory (per-query lookups)
    extern __shared__ double s_tab[];
    for (int c = lane; c < p.n_cells; c += 32) {
        s_tab[c] = p.lat[c];
        s_tab[p.n_cells + c] = p.util[c];
    }
    __syncwarp();
    const double* lat = s_tab;
    const double* util = s_tab + p.n_cells;
    const int64_t n = p.n_ptr ? *p.n_ptr : p.n;
    const double sla = p.sla, alpha = p.alpha, beta = p.beta, warmup = p.warmup_ms;
    const bool route = p.route_mask != nullptr;
    const bool elsa = p.sched == MSV_ELSA;  // Eq. 1's fold is needed by ELSA only
    // The first kRing queued estimates of each slot in FIFO order (a ring at rh[s]); the
    // rest of a longer queue is walked through the query list from rq[s] (queue item kRing).
    __shared__ double ring[S][kRing][32];
    int rh[S];
    int64_t rq[S];
    // multipliers j in [mj, mj + 32) staged in shared memory; refilled at warp-uniform points
    __shared__ double mw[32];
    int64_t mj = -64;
    double c_arr[S];  // arrival of each slot's running query
    int32_t c_b[S];   // and its batch

    bool act[S], busy[S];
    int32_t row[S], pid[S], kk[S];
    uint64_t rmask[S];
    int64_t qh[S], qt[S], qn[S];
    double fold[S], c_start[S], c_est[S], c_comp[S], bms[S], wbms[S];
    uint64_t c_seq[S];
    int64_t cq[S], nq[S];
#pragma unroll
    for (int s = 0; s < S; ++s) {
        const int o = s * 32 + lane;
        act[s] = o < p.P;
        const DevPart dp = act[s] ? p.parts[o] : DevPart{0, 0, -1, 0};
        row[s] = dp.row;
        pid[s] = dp.pid;
        kk[s] = dp.k;
        rmask[s] = (act[s] && route) ? p.route_mask[o] : 0;
        busy[s] = false;
        qh[s] = qt[s] = -1;
        qn[s] = 0;
        fold[s] = c_start[s] = c_est[s] = c_comp[s] = bms[s] = wbms[s] = 0.0;
        c_seq[s] = 0;
        cq[s] = -1;
        nq[s] = 0;
        rh[s] = 0;
        rq[s] = -1;
        c_arr[s] = 0.0;
        c_b[s] = 1;
    }
    uint64_t seq = (uint64_t)n;  // arrivals hold seq 0..n-1 (engine.hpp:136-137)
    int64_t j = 0;               // next noise multiplier
    auto stage_mult = [&]() {
        if (j >= mj + 32) {
            mj = j;
            __syncwarp();
            mw[lane] = mj + lane < n ? p.mult[mj + lane] : 1.0;
            __syncwarp();
        }
    };
    int64_t viol = 0, meas = 0, mviol = 0, m0 = -1;
    uint32_t hmin = 0xffffffffu, hmax = 0;  // high words of the measured latencies (K3's key bounds)
    uint64_t hash = 0;
    double last_finish = 0.0;
    int status = 0;

    // Exact left fold of slot s's FIFO (sched.hpp:78-79): the cached ring, then the list.
    auto refold = [&](int s) {
        double acc = 0.0;
        const int nr = qn[s] < kRing ? (int)qn[s] : kRing;
        for (int k = 0; k < nr; ++k) acc = acc + ring[s][(rh[s] + k) & (kRing - 1)][lane];
        int64_t q = rq[s];
        for (int64_t i = kRing; i < qn[s]; ++i) {
            acc = acc + lat[row[s] + bat[q] - 1];
            q = p.next[q];
        }
        return acc;
    };

    // Retire, in global (time, seq) order, every completion with time <= t.
    auto drain = [&](double t) {
        for (;;) {
            bool due = false;
#pragma unroll
            for (int s = 0; s < S; ++s) due |= busy[s] && c_comp[s] <= t;
            const unsigned dm = __ballot_sync(kFull, due);
            if (dm == 0) return;  // nothing due by t
            stage_mult();
            double bt = CUDART_INF;
            uint64_t bs = ~0ull;
            int bsl = -1;
#pragma unroll
            for (int s = 0; s < S; ++s)
                if (busy[s] && c_comp[s] <= t && (c_comp[s] < bt || (c_comp[s] == bt && c_seq[s] < bs))) {
                    bt = c_comp[s];
                    bs = c_seq[s];
                    bsl = s;
                }
            int bl;
            if (__popc(dm) == 1) {
                bl = __ffs(dm) - 1;  // one lane has due completions: its own minimum is the global one
            } else {
                // the earliest (time, seq) over the due lanes: completion times are non-negative,
                // so their IEEE bits order like the values — two 32-bit warp reductions find
                // the minimum time, and only equal times fall back to the seq reduction
                const uint64_t tb = bsl >= 0 ? msv_dbits(bt) : ~0ull;
                const uint32_t mh = __reduce_min_sync(kFull, (uint32_t)(tb >> 32));
                const uint32_t ml = __reduce_min_sync(kFull, (uint32_t)(tb >> 32) == mh ? (uint32_t)tb : 0xffffffffu);
                const bool at_min = tb == (((uint64_t)mh << 32) | ml);
                const unsigned tie = __ballot_sync(kFull, at_min);
                if (__popc(tie) == 1) {
                    bl = __ffs(tie) - 1;
                } else {  // equal completion times: the smaller seq first (engine.hpp:101-107)
                    const uint64_t sk = at_min ? bs : ~0ull;
                    const uint32_t sh = __reduce_min_sync(kFull, (uint32_t)(sk >> 32));
                    const uint32_t sl = __reduce_min_sync(kFull, (uint32_t)(sk >> 32) == sh ? (uint32_t)sk : 0xffffffffu);
                    bl = __ffs(__ballot_sync(kFull, at_min && sk == (((uint64_t)sh << 32) | sl))) - 1;
                }
            }
            int started = 0;
            if (lane == bl) {
#pragma unroll
                for (int s = 0; s < S; ++s) {
                    if (s != bsl) continue;
                    const double now = c_comp[s];  // engine.hpp:167-187
                    const int64_t q = cq[s];
                    const double a = c_arr[s];
                    const double l = now - a;
                    const bool met = l <= sla;
                    const double ran = now - c_start[s];
                    bms[s] = bms[s] + ran;
                    wbms[s] = wbms[s] + ran * util[row[s] + c_b[s] - 1];
                    nq[s] += 1;
                    viol += met ? 0 : 1;
                    if (a >= warmup) {
                        meas += 1;
                        mviol += met ? 0 : 1;
                        if (p.samples) p.samples[q] = l;  // over its own (dead) arrival
                        const uint32_t lh = (uint32_t)(msv_dbits(l) >> 32);
                        hmin = lh < hmin ? lh : hmin;
                        hmax = lh > hmax ? lh : hmax;
                    }
                    last_finish = last_finish < now ? now : last_finish;
                    hash += msv_query_digest((uint64_t)q, pid[s], c_start[s], now);
                    if (p.records) p.records[q].finish_ms = now;
                    if (qn[s] > 0) {  // start the queue head now (engine.hpp:181-185)
                        const int64_t h = qh[s];
                        qh[s] = p.next[h];
                        // the head's latency comes from the ring (cached when it was queued), so
                        // the new finish does not wait for a global load of the head's batch
                        const int vac = rh[s];
                        const double est = ring[s][vac][lane];
                        rh[s] = (vac + 1) & (kRing - 1);  // the ring drops its head, takes item kRing
                        if (qn[s] > kRing) {
                            ring[s][vac][lane] = lat[row[s] + bat[rq[s]] - 1];
                            if (qn[s] > kRing + 1) rq[s] = p.next[rq[s]];
                        }
                        qn[s] -= 1;
                        if (qn[s] == 0) qt[s] = -1;
                        const int32_t hb = bat[h];  // needed at its completion (utilisation)
                        c_arr[s] = arr[h];
                        c_b[s] = hb;
                        c_start[s] = now;
                        c_est[s] = est;
                        c_comp[s] = now + est * mw[j - mj];
                        c_seq[s] = seq;
                        cq[s] = h;
                        if (p.records) p.records[h].start_ms = now;
                        if (elsa) fold[s] = refold(s);
                        started = 1;
                    } else {
                        busy[s] = false;
                        fold[s] = 0.0;
                    }
                }
            }
            if (__shfl_sync(kFull, started, bl)) {
                j += 1;
                seq += 1;
            }
        }
    };

    double w_t = lane < n ? arr[lane] : 0.0;  // arrivals [i & ~31, +32) one per lane
    int32_t w_b = lane < n ? bat[lane] : 0;
    double nx_t = 32 + lane < n ? arr[32 + lane] : 0.0;  // and the next window
    int32_t nx_b = 32 + lane < n ? bat[32 + lane] : 0;
    for (int64_t i = 0; i < n && status == 0; ++i) {
        if (i > 0 && (i & 31) == 0) {
            w_t = nx_t;
            w_b = nx_b;
            nx_t = i + 32 + lane < n ? arr[i + 32 + lane] : 0.0;
            nx_b = i + 32 + lane < n ? bat[i + 32 + lane] : 0;
        }
        const double t = __shfl_sync(kFull, w_t, (int)(i & 31));
        const int b = __shfl_sync(kFull, w_b, (int)(i & 31));
        if (m0 < 0 && t >= warmup) m0 = i;  // the measured suffix (arrivals are sorted)
        drain(t);  // completions at <= t precede the arrival (engine.hpp:101-107)
        stage_mult();
        if (b < 1 || b > p.b_max) {  // every lookup of this query fails (profile.hpp:123-132)
            status = MSV_LOOKUP;
            break;
        }
        // candidates (engine.hpp:197-206): routed partitions, else all
        bool cand[S];
        unsigned any = 0;
#pragma unroll
        for (int s = 0; s < S; ++s) {
            cand[s] = act[s] && route && ((rmask[s] >> (b - 1)) & 1ull);
            any |= __ballot_sync(kFull, cand[s]);
        }
        if (any == 0) {
#pragma unroll
            for (int s = 0; s < S; ++s) cand[s] = act[s];
        }
        int csl = -1, cl = 0, kind = 0;
        if (p.sched == MSV_ELSA) {
            double w[S], est[S];
            unsigned okb[S], badb[S];
#pragma unroll
            for (int s = 0; s < S; ++s) {
                const bool good = cand[s] && row[s] >= 0;
                est[s] = good ? lat[row[s] + b - 1] : 0.0;
                double x = fold[s];  // t_wait, Eq. 1 (sched.hpp:77-85)
                if (busy[s]) {
                    const double r = c_est[s] - (t - c_start[s]);
                    x = x + (0.0 < r ? r : 0.0);
                }
                w[s] = x;
                okb[s] = __ballot_sync(kFull, good && sla > alpha * (x + beta * est[s]));
                badb[s] = __ballot_sync(kFull, cand[s] && row[s] < 0);
            }
            // Step A: the first candidate in scan order that satisfies the SLA (or whose
            // lookup fails first) (sched.hpp:124-129)
#pragma unroll
            for (int s = 0; s < S; ++s) {
                if (csl >= 0 || status) continue;
                const unsigned m = okb[s] | badb[s];
                if (m) {
                    const int f = __ffs(m) - 1;
                    if ((badb[s] >> f) & 1u) {
                        status = MSV_LOOKUP;
                    } else {
                        csl = s;
                        cl = f;
                        kind = MSV_SLACK_SATISFYING;
                    }
                }
            }
            if (csl < 0 && !status) {  // Step B: argmin w + est, earliest in scan order (sched.hpp:131-141)
                unsigned bad = 0;
#pragma unroll
                for (int s = 0; s < S; ++s) bad |= badb[s];
                if (bad) {
                    status = MSV_LOOKUP;
                } else {
                    double bv = CUDART_INF;
                    int bo = 1 << 30;
#pragma unroll
                    for (int s = 0; s < S; ++s) {
                        const double v = w[s] + est[s];
                        if (cand[s] && v < bv) {  // slots ascend in scan order
                            bv = v;
                            bo = s * 32 + lane;
                        }
                    }
#pragma unroll
                    for (int off = 16; off > 0; off >>= 1) {
                        const double ov = __shfl_xor_sync(kFull, bv, off);
                        const int oo = __shfl_xor_sync(kFull, bo, off);
                        if (ov < bv || (ov == bv && oo < bo)) {
                            bv = ov;
                            bo = oo;
                        }
                    }
                    csl = bo >> 5;
                    cl = bo & 31;
                    kind = MSV_FASTEST_FALLBACK;
                }
            }
        } else {  // FIFS (sched.hpp:154-170): ties by partition id
            unsigned key = 0;  // idle: max k, then min id
#pragma unroll
            for (int s = 0; s < S; ++s)
                if (cand[s] && !busy[s]) {
                    const unsigned kv = ((unsigned)kk[s] << 10) | (unsigned)(1023 - pid[s]);
                    key = kv > key ? kv : key;
                }
            const unsigned best = __reduce_max_sync(kFull, key);
            if (best) {
                const int want = 1023 - (int)(best & 1023u);
#pragma unroll
                for (int s = 0; s < S; ++s) {
                    const unsigned hit = __ballot_sync(kFull, cand[s] && !busy[s] && pid[s] == want);
                    if (hit) {
                        csl = s;
                        cl = __ffs(hit) - 1;
                    }
                }
                kind = MSV_IDLE_LARGEST;
            } else {  // shortest queue by count, then min id
                unsigned long long qk = ~0ull;
#pragma unroll
                for (int s = 0; s < S; ++s)
                    if (cand[s]) {
                        const unsigned long long v = ((unsigned long long)qn[s] << 10) | (unsigned)pid[s];
                        qk = v < qk ? v : qk;
                    }
#pragma unroll
                for (int off = 16; off > 0; off >>= 1) {
                    const unsigned long long o = __shfl_xor_sync(kFull, qk, off);
                    qk = o < qk ? o : qk;
                }
                const int want = (int)(qk & 1023u);
#pragma unroll
                for (int s = 0; s < S; ++s) {
                    const unsigned hit = __ballot_sync(kFull, cand[s] && pid[s] == want);
                    if (hit) {
                        csl = s;
                        cl = __ffs(hit) - 1;
                    }
                }
                kind = MSV_SHORTEST_QUEUE;
            }
        }
        if (status) break;
        // the chosen partition: est lookup (engine.hpp:224-229), start or enqueue
        int started = 0, lookup_bad = 0;
        if (lane == cl) {
#pragma unroll
            for (int s = 0; s < S; ++s) {
                if (s != csl) continue;
                if (row[s] < 0) {
                    lookup_bad = 1;
                    continue;
                }
                const double est = lat[row[s] + b - 1];
                if (p.records) {
                    p.records[i].partition = pid[s];
                    p.records[i].kind = kind;
                }
                if (busy[s]) {  // queue it; the ring caches the first kRing latencies (both schedulers)
                    if (qn[s] < kRing) ring[s][(rh[s] + (int)qn[s]) & (kRing - 1)][lane] = est;
                    else if (qn[s] == kRing) rq[s] = i;
                    if (qn[s] == 0) {
                        qh[s] = i;
                    } else {
                        p.next[qt[s]] = (uint32_t)i;
                    }
                    qt[s] = i;
                    qn[s] += 1;
                    fold[s] = fold[s] + est;  // the left fold extends exactly on append
                } else {
                    busy[s] = true;
                    c_start[s] = t;
                    c_est[s] = est;
                    c_comp[s] = t + est * mw[j - mj];
                    c_seq[s] = seq;
                    cq[s] = i;
                    c_arr[s] = t;
                    c_b[s] = b;
                    fold[s] = 0.0;
                    if (p.records) p.records[i].start_ms = t;
                    started = 1;
                }
            }
        }
        if (__shfl_sync(kFull, lookup_bad, cl)) {
            status = MSV_LOOKUP;
            break;
        }
        if (__shfl_sync(kFull, started, cl)) {
            j += 1;
            seq += 1;
        }
    }
    if (status == 0) drain(CUDART_INF);  // run to completion (no horizon cut-off)

    // per-partition usage by id, totals
#pragma unroll
    for (int s = 0; s < S; ++s)
        if (act[s] && p.usage) {
            p.usage[pid[s]].busy_ms = bms[s];
            p.usage[pid[s]].weighted_busy_ms = wbms[s];
            p.usage[pid[s]].queries = nq[s];
        }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
        viol += __shfl_xor_sync(kFull, viol, off);
        meas += __shfl_xor_sync(kFull, meas, off);
        mviol += __shfl_xor_sync(kFull, mviol, off);
        hash += __shfl_xor_sync(kFull, hash, off);
        const double o = __shfl_xor_sync(kFull, last_finish, off);
        last_finish = last_finish < o ? o : last_finish;
    }
    seg_range_u32<32>(hmin, hmax, kFull);
    if (lane == 0) {
        p.out->violations = viol;
        p.out->measured = meas;
        p.out->measured_violations = mviol;
        p.out->hash = hash;
        p.out->horizon_ms = (p.duration_ms < last_finish) ? last_finish : p.duration_ms;  // engine.hpp:235
        p.out->status = status;
        p.out->n_samples = meas;
        p.out->m0 = m0 >= 0 ? (int32_t)m0 : 0;
        uint64_t kmin, kmax;
        lat_key_bounds(hmin, hmax, kmin, kmax);
        p.out->lat_min_bits = kmin;
        p.out->lat_max_bits = kmax;
        p.out->planar = 0;
        p.out->pad = 0;
    }
}

}  // namespace

cudaError_t launch_noise(const NoiseParams* d_jobs, int n_jobs, int max_cells, int max_parts, cudaStream_t stream) {
    if (max_parts > 128) return cudaErrorInvalidValue;
    // Always opt in: the kernel's ~33 KB of static shared memory (ring, multiplier
    // window) already eats most of the default 48 KB, so the default dynamic limit is
    // only ~15 KB (profiles of ~1,000 cells failed to launch).
    const size_t smem = (size_t)2 * max_cells * sizeof(double);
    const void* fn = max_parts > 64   ? (const void*)sim_noise_kernel<4, 32>
                     : max_parts > 32 ? (const void*)sim_noise_kernel<2, 64>
                                      : (const void*)sim_noise_kernel<1, 128>;
    const cudaError_t e = ensure_dyn_smem(fn, smem);
    if (e != cudaSuccess) return e;
    if (n_jobs <= 0) return cudaSuccess;
    if (max_parts > 64) sim_noise_kernel<4, 32><<<n_jobs, 32, smem, stream>>>(d_jobs);
    else if (max_parts > 32) sim_noise_kernel<2, 64><<<n_jobs, 32, smem, stream>>>(d_jobs);
    else sim_noise_kernel<1, 128><<<n_jobs, 32, smem, stream>>>(d_jobs);
    return cudaGetLastError();
}

}  // namespace msv
