// K2 sim_kernel: run() (engine.hpp:115-253) with ELSA (sched.hpp:119-143) or FIFS
// (sched.hpp:154-170), segmented variant: a warp runs G = 32/W scenarios side by
// side, one segment of W lanes each, every lane holding S partition slots, so a plan
// of P <= W*S partitions fits one segment (W in {4, 8, 16}; instantiated with S = 1:
// two slots per lane for 16 < P <= 32 measured slower than the warp kernel). Slot s of
// segment lane l owns by_ascending_size order index s*W + l (sched.hpp:96-104). All
// segments advance one arrival per iteration (lockstep): every warp instruction of
// the per-arrival path serves G scenarios.
//
// Per arrival (every kernel of K2 follows this protocol):
//   1. every lane advances its own partitions to `now`: a running query with finish
//      <= now has completed and the queue head starts at that finish, in chain order,
//      with no warp collective (completions on different partitions commute and a
//      completion precedes an arrival at equal time, engine.hpp:101-107). A
//      completion's bookkeeping is not done here: with noise off a query's start and
//      finish are known when it is placed (step 3);
//   2. every lane evaluates Eq. 1 (t_wait, kept as an exact FIFO fold) and Eq. 2 for
//      its slots; Step A = first set bit of the segment's ballot bits over the slots in
//      order, Step B = a shuffle-tree argmin over the segment with order tie-break;
//      FIFS = (k, id) / (queue length, id) key minima;
//   3. the chosen slot starts the query or appends it to its FIFO (shared-memory
//      ring, overflow list threaded through query ids in global memory); its start is
//      the arrival (idle) or the finish of the query placed before it, its finish =
//      start + est (the same RN add the completion event performs), and the chosen lane
//      books the completion at once: latency, SLA, measured sample, placement digest,
//      record, usage (in the partition's completion = FIFO order).
// Each segment keeps a double-buffered 32-arrival window in shared memory, refilled
// by cp.async one window ahead. Measured latencies overwrite their own arrivals
// (samples[q] with samples == the arrival buffer: a placed query's arrival is never
// read again); arrivals are sorted, so the measured set is the suffix from the first
// arrival >= warmup, m0, ready for K3. The plain variant (no routing / missing sizes /
// wait check / usage / records in the launch) carries none of those features' work.
#include <cuda_pipeline.h>

#include <map>
#include <mutex>
#include <utility>

#include "msv_device.cuh"

namespace msv {

namespace {


template <int W, int S>
struct SegCfg {
    static constexpr int G = 32 / W;
    static constexpr int qcap = S == 1 ? kQCap : 4;  // shared ring entries per slot
    static constexpr int min_blocks = S == 1 ? 6 : 5;
};

template <int W, int S>
struct SegSmem {
    static constexpr int G = SegCfg<W, S>::G;
    static constexpr int QC = SegCfg<W, S>::qcap;
    double q_est[S][QC][32];  // queued latencies (starts / finishes follow from them)
    double win_t[2][32][G];  // [buffer][entry][segment]
    int32_t win_b[2][32][G];
    uint32_t g_head[S][32];  // overflow list head / tail per lane slot
    uint32_t g_tail[S][32];
};

template <int W, int S, int SCHED, bool REC, bool FULL>
__global__ void __launch_bounds__(kSimWarpsPerBlock * 32, (SegCfg<W, S>::min_blocks))
    sim_kernel(const SimParams p) {
    constexpr int QC = SegCfg<W, S>::qcap;
    constexpr bool kFold = (SCHED == MSV_ELSA) || FULL;
    extern __shared__ __align__(16) unsigned char smem[];
    double* s_lat = reinterpret_cast<double*>(smem);
    double* s_util = s_lat + p.n_cells;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const size_t tab_bytes = ((size_t)2 * p.n_cells * sizeof(double) + 15) & ~(size_t)15;
    SegSmem<W, S>& M = reinterpret_cast<SegSmem<W, S>*>(smem + tab_bytes)[warp];
    for (int c = threadIdx.x; c < p.n_cells; c += blockDim.x) {
        s_lat[c] = p.lat[c];
        s_util[c] = p.util[c];
    }
    __syncthreads();

    const int seg = lane / W, seg_base = seg * W, sl = lane - seg_base;
    const unsigned seg_mask = (W == 32) ? kFull : (((1u << W) - 1u) << seg_base);

    // ---- segment state (identical in the lanes of a segment) ----
    int32_t sidx = -1;
    bool done = false;
    int n = 0, i = 0, win_base = 0, buf = 0, m0 = -1, status = 0;
    const DevScen* d = nullptr;
    const double* g_arr = nullptr;
    const int32_t* g_bat = nullptr;
    double* samples = nullptr;
    double sla = 0.0, warmup = 0.0, alpha = 1.0, beta = 1.0;
    bool unit = true, check_wait = false;
    int bmax = 0;
    // ---- per-lane partition slots ----
    // c_* = the query placed last to start; tail = finish of the query placed last; the
    // slot is busy at t iff c_comp > t (msv_sim_warp.cu).
    bool act[S];
    int32_t row[S], pk[S], qh[S], qn[S];
    uint32_t gn[S], nq[S];
    double c_start[S], c_est[S], c_comp[S], tail[S], fold[S], bms[S], wbms[S];
    uint32_t viol = 0, mviol = 0;
    uint64_t hash = 0;
    double wdiff = 0.0;
#pragma unroll
    for (int s = 0; s < S; ++s) {
        act[s] = false;
        row[s] = pk[s] = qh[s] = qn[s] = 0;
        gn[s] = nq[s] = 0;
        c_start[s] = c_est[s] = 0.0;
        c_comp[s] = -INFINITY;  // idle: busy at t iff c_comp > t
        tail[s] = fold[s] = bms[s] = wbms[s] = 0.0;
    }

    // Async copy of arrivals [from, from+32) into the segment's window buffer b.
    auto prefetch = [&](int from, int b) {
        for (int e = sl; e < 32; e += W) {
            const int q = from + e;
            if (q < n) {
                __pipeline_memcpy_async(&M.win_t[b][e][seg], g_arr + q, sizeof(double));
                __pipeline_memcpy_async(&M.win_b[b][e][seg], g_bat + q, sizeof(int32_t));
            }
        }
        __pipeline_commit();
    };
    // Exact left fold of slot s's FIFO (sched.hpp:78-79), starting from the head entry
    // (0.0 + e == e); an overflow list implies a full ring.
    auto refold = [&](int s) {
        if (qn[s] == 0) return 0.0;
        double acc = M.q_est[s][qh[s]][lane];
#pragma unroll 1
        for (int k = 1; k < qn[s]; ++k) acc = acc + M.q_est[s][(qh[s] + k) & (QC - 1)][lane];
        if (gn[s] > 0) {
            uint32_t g = M.g_head[s][lane];
#pragma unroll 1
            for (uint32_t k = 0; k < gn[s]; ++k) {
                acc = acc + s_lat[row[s] + g_bat[g] - 1];
                g = d->next[g];
            }
        }
        return acc;
    };

    while (true) {
        // ---- acquire a scenario (segment-uniform, rare) ----
        if (sidx < 0 && !done) {
            int w = 0;
            if (sl == 0) w = atomicAdd(p.counter, 1);
            w = __shfl_sync(seg_mask, w, seg_base);
            if (w >= p.n_work) {
                done = true;
            } else {
                sidx = p.work[w];
                d = p.scen + sidx;
                n = (int)*d->n;
                g_arr = d->arrival;
                g_bat = d->batch;
                samples = d->samples;
                __builtin_assume(__isGlobal(g_arr));
                __builtin_assume(__isGlobal(g_bat));
                __builtin_assume(__isGlobal(samples));
                sla = d->sla;
                warmup = d->warmup_ms;
                alpha = d->alpha;
                beta = d->beta;
                unit = alpha == 1.0 && beta == 1.0;  // 1*x == x: identical bits
                check_wait = FULL && p.any_check_wait && (d->flags & MSV_FLAG_CHECK_WAIT);
                bmax = d->b_max;
                i = 0;
                win_base = 0;
                buf = 0;
                m0 = -1;
                status = 0;
#pragma unroll
                for (int s = 0; s < S; ++s) {
                    const int o = s * W + sl;
                    act[s] = o < d->P;
                    row[s] = 0;  // inactive slots read a valid (ignored) cell
                    pk[s] = 0;
                    if (act[s]) {
                        const DevPart dp = d->parts[o];
                        pk[s] = dp.pid | (dp.k << 8);
                        row[s] = dp.row;
                    }
                    qh[s] = qn[s] = 0;
                    gn[s] = nq[s] = 0;
                    c_start[s] = c_est[s] = 0.0;
                    c_comp[s] = -INFINITY;
                    tail[s] = 0.0;
                    fold[s] = bms[s] = wbms[s] = 0.0;
                }
                viol = mviol = 0;
                hash = 0;
                wdiff = 0.0;
                prefetch(0, 0);
                prefetch(32, 1);
                __pipeline_wait_prior(1);  // window 0 landed (this lane's copies)
                __syncwarp(seg_mask);
            }
        }
        if (__all_sync(kFull, done)) break;

        // ---- this iteration's event: arrival i, or the end-of-trace marker ----
        const bool live = !done;
        const bool arrival = live && i < n && status == 0;
        const bool ending = live && !arrival;
        if (arrival && i - win_base == 32) {  // window exhausted: switch, prefetch the next
            win_base += 32;
            buf ^= 1;
            __pipeline_wait_prior(0);
            __syncwarp(seg_mask);
            prefetch(win_base + 32, buf ^ 1);
        }
        double t = -INFINITY;
        int b = 1;
        if (arrival) {
            t = M.win_t[buf][i - win_base][seg];
            b = M.win_b[buf][i - win_base][seg];
            if (m0 < 0 && t >= warmup) m0 = i;  // measured iff arrival >= warmup (engine.hpp:262)
        }  // (ending: nothing to drain — every query was booked when it was placed)
        // the new query's latency on each slot depends on its batch only: load it ahead
        // of the drain (FULL: batch clamped into the table, missing sizes read 0)
        double est_n[S];
#pragma unroll
        for (int s = 0; s < S; ++s) {
            if (FULL) {
                const int bl = min(max(b, 1), max(bmax, 1));
                est_n[s] = row[s] >= 0 ? s_lat[row[s] + bl - 1] : 0.0;
            } else {
                est_n[s] = s_lat[row[s] + b - 1];
            }
        }

        // ---- 1. advance to t, lane-local, in chain order (engine.hpp:167-187) ----
#pragma unroll
        for (int s = 0; s < S; ++s) {
            while (c_comp[s] <= t && qn[s] > 0) {  // a finished query with nothing queued: idle
                {  // start the queue head at the finish (engine.hpp:181-185)
                    const int h = qh[s];
                    const double est = M.q_est[s][h][lane];
                    qh[s] = (h + 1) & (QC - 1);
                    qn[s] -= 1;
                    if (gn[s] > 0) {  // refill the ring from the overflow list
                        const uint32_t g = M.g_head[s][lane];
                        M.g_head[s][lane] = d->next[g];
                        gn[s] -= 1;
                        M.q_est[s][(qh[s] + qn[s]) & (QC - 1)][lane] = s_lat[row[s] + g_bat[g] - 1];
                        qn[s] += 1;
                    }
                    c_start[s] = c_comp[s];
                    c_est[s] = est;
                    c_comp[s] = c_start[s] + est;  // the placement computed the same sum
                    if (kFold) fold[s] = refold(s);
                }
            }
        }

        // ---- 2. dispatch (engine.hpp:189-230) ----
        bool go = arrival;
        if (FULL && go && (b < 1 || b > bmax)) {  // LookupError at this query (profile.hpp:127-129)
            status = MSV_LOOKUP;
            go = false;
        }
        bool cand[S], bad[S];
        double wv[S];
#pragma unroll
        for (int s = 0; s < S; ++s) {
            cand[s] = go && act[s];
            const double x = c_est[s] - (t - c_start[s]);
            wv[s] = fold[s] + running_part(c_comp[s], t, x);  // Eq. 1 (sched.hpp:77-85)
            bad[s] = false;
        }
        int bad_o = 1 << 30;  // segment order index of the first candidate whose size is missing
        if (FULL) {
            if (p.any_routing) {  // engine.hpp:197-206
                unsigned anyc = 0;
#pragma unroll
                for (int s = 0; s < S; ++s) {
                    if (go && d->route_mask != nullptr)
                        cand[s] = cand[s] && (((d->route_mask[s * W + sl] >> (b - 1)) & 1ull) != 0);
                    anyc |= __ballot_sync(kFull, cand[s]) & seg_mask;
                }
                if (anyc == 0) {
#pragma unroll
                    for (int s = 0; s < S; ++s) cand[s] = go && act[s];
                }
            }
#pragma unroll
            for (int s = S - 1; s >= 0; --s) {
                bad[s] = cand[s] && row[s] < 0;
                const unsigned bb = __ballot_sync(kFull, bad[s]) & seg_mask;
                if (bb) bad_o = s * W + (__ffs(bb) - 1 - seg_base);
            }
            if (check_wait) {  // engine.hpp:208-217
#pragma unroll
                for (int s = 0; s < S; ++s) {
                    if (!cand[s] || bad[s]) continue;
                    const double y = c_comp[s] - t;
                    const double gw = fold[s] + pos_part(y);  // y > 0 iff running
                    const double dd = fabs(gw - wv[s]);
                    wdiff = (wdiff < dd) ? dd : wdiff;
                }
            }
        }
        int ch = -1, kind = 0;  // chosen segment order index
        if constexpr (SCHED == MSV_ELSA) {
            bool ok[S];
#pragma unroll
            for (int s = S - 1; s >= 0; --s) {  // Step A (sched.hpp:125-130)
                ok[s] = cand[s] && !bad[s];
                const bool pred =
                    ok[s] && (unit ? (sla > wv[s] + est_n[s]) : (sla > alpha * (wv[s] + beta * est_n[s])));
                const unsigned bA = __ballot_sync(kFull, pred) & seg_mask;
                if (bA) ch = s * W + (__ffs(bA) - 1 - seg_base);
            }
            kind = MSV_SLACK_SATISFYING;
            const bool needB = go && ch < 0;
            if (__any_sync(kFull, needB)) {  // Step B (sched.hpp:132-142): argmin w + est, earliest on ties
                uint64_t fb[S];
                uint64_t lm = ~0ull;
#pragma unroll
                for (int s = 0; s < S; ++s) {
                    fb[s] = ok[s] ? msv_dbits(wv[s] + est_n[s]) : ~0ull;
                    lm = fb[s] < lm ? fb[s] : lm;
                }
                const uint64_t vmin = seg_min_u64<W>(lm);
                int chB = -1;
#pragma unroll
                for (int s = S - 1; s >= 0; --s) {
                    const unsigned bB = __ballot_sync(kFull, ok[s] && fb[s] == vmin) & seg_mask;
                    if (bB) chB = s * W + (__ffs(bB) - 1 - seg_base);
                }
                if (needB && chB >= 0) {
                    ch = chB;
                    kind = MSV_FASTEST_FALLBACK;
                }
            }
            // a size missing from the profile is a LookupError once the scan reaches it
            if (FULL && go && bad_o != (1 << 30) && (ch < 0 || kind == MSV_FASTEST_FALLBACK || bad_o < ch)) {
                status = MSV_LOOKUP;
                go = false;
            }
        } else {  // FIFS (sched.hpp:154-170): idle -> max k, min id; else shortest queue, min id
            uint32_t ki[S], kq[S];
            uint32_t li = ~0u, lq = ~0u;
#pragma unroll
            for (int s = 0; s < S; ++s) {
                ki[s] = (cand[s] && !(c_comp[s] > t)) ? (((0x7FFFu - ((uint32_t)pk[s] >> 8)) << 16) | ((uint32_t)pk[s] & 0xffu))
                                              : ~0u;
                const uint32_t len = (uint32_t)qn[s] + gn[s];
                kq[s] = cand[s] ? (((len < 0xFFFFFFu ? len : 0xFFFFFFu) << 8) | ((uint32_t)pk[s] & 0xffu)) : ~0u;
                li = ki[s] < li ? ki[s] : li;
                lq = kq[s] < lq ? kq[s] : lq;
            }
            const uint32_t mi = seg_min_u32<W>(li);
            const bool idle = mi != ~0u;
            uint32_t mq = ~0u;
            if (__any_sync(kFull, go && !idle)) mq = seg_min_u32<W>(lq);
#pragma unroll
            for (int s = S - 1; s >= 0; --s) {
                const unsigned bs =
                    __ballot_sync(kFull, idle ? (ki[s] == mi && mi != ~0u) : (kq[s] == mq && mq != ~0u)) & seg_mask;
                if (go && bs) ch = s * W + (__ffs(bs) - 1 - seg_base);
            }
            kind = idle ? MSV_IDLE_LARGEST : MSV_SHORTEST_QUEUE;
            if (FULL) {  // the chosen partition's latency lookup fails (engine.hpp:226)
                bool mine_bad = false;
#pragma unroll
                for (int s = 0; s < S; ++s) mine_bad |= go && (s * W + sl == ch) && row[s] < 0;
                if ((__ballot_sync(kFull, mine_bad) & seg_mask) != 0) {
                    status = MSV_LOOKUP;
                    go = false;
                }
            }
        }

        // ---- 3. start or enqueue on the chosen partition (engine.hpp:225-230) and book
        //         its completion (engine.hpp:167-187): start and finish are known now ----
#pragma unroll
        for (int s = 0; s < S; ++s) {
            if (go && s * W + sl == ch) {
                const double est = est_n[s];
                double st, fin;
                if (!(c_comp[s] > t)) {  // idle: starts now
                    st = t;
                    fin = t + est;
                    c_start[s] = t;
                    c_est[s] = est;
                    c_comp[s] = fin;
                } else {
                    st = tail[s];  // starts when the query placed before it finishes
                    fin = st + est;
                    if (gn[s] == 0 && qn[s] < QC) {
                        M.q_est[s][(qh[s] + qn[s]) & (QC - 1)][lane] = est;
                        qn[s] += 1;
                    } else {
                        if (gn[s] == 0) M.g_head[s][lane] = (uint32_t)i;
                        else d->next[M.g_tail[s][lane]] = (uint32_t)i;
                        M.g_tail[s][lane] = (uint32_t)i;
                        gn[s] += 1;
                    }
                    fold[s] = fold[s] + est;  // appending extends the left fold exactly
                }
                tail[s] = fin;
                const double lat = fin - t;  // latency = finish - arrival
                const bool met = lat <= sla;
                viol += met ? 0u : 1u;
                if (t >= warmup) {  // measured (engine.hpp:262)
                    mviol += met ? 0u : 1u;
                    samples[i] = lat;
                }
                hash += msv_query_digest((uint64_t)i, pk[s] & 0xff, st, fin);
                if (FULL) {  // PartitionUsage (engine.hpp:175-177), completion order
                    const double ran = fin - st;
                    bms[s] = bms[s] + ran;
                    wbms[s] = wbms[s] + ran * s_util[row[s] + b - 1];
                    nq[s] += 1;
                }
                if (REC) {
                    msv_record r;
                    r.start_ms = st;
                    r.finish_ms = fin;
                    r.partition = pk[s] & 0xff;
                    r.kind = kind;
                    d->records[i] = r;
                }
            }
        }
        if (arrival && status == 0) ++i;

        // ---- end of trace: reduce the segment and publish (segment-uniform, rare) ----
        if (ending) {
            __pipeline_wait_prior(0);  // no copy may land in a window after the segment moves on
            // last completion = each slot's last placed finish (a slot that never ran holds 0.0)
            double lf = 0.0;
#pragma unroll
            for (int s = 0; s < S; ++s) lf = (lf < tail[s]) ? tail[s] : lf;
            const uint64_t v0 = seg_sum_u64<W>((uint64_t)viol, seg_mask);
            const uint64_t v2 = seg_sum_u64<W>((uint64_t)mviol, seg_mask);
            const uint64_t hsum = seg_sum_u64<W>(hash, seg_mask);
            lf = seg_max_f64<W>(lf, seg_mask);
            const double wd = seg_max_f64<W>(wdiff, seg_mask);
            if (sl == 0) {
                DevOut o;
                o.violations = (int64_t)v0;
                o.measured = m0 >= 0 ? n - m0 : 0;
                o.measured_violations = (int64_t)v2;
                o.n_samples = o.measured;
                o.horizon_ms = (d->duration_ms < lf) ? lf : d->duration_ms;  // engine.hpp:237
                o.max_wait_diff = wd;
                o.hash = hsum;
                o.lat_min_bits = msv_dbits(d->lat_floor) | kSignBit;  // latencies lie in [floor, horizon]
                o.lat_max_bits = msv_dbits(o.horizon_ms) | kSignBit;
                o.planar = 0;
                o.pad = 0;
                o.status = status;
                o.m0 = m0 >= 0 ? m0 : 0;
                p.out[sidx] = o;
            }
            if (FULL && p.any_usage && d->usage_off >= 0) {
#pragma unroll
                for (int s = 0; s < S; ++s) {
                    if (act[s]) {
                        msv_usage u;
                        u.busy_ms = bms[s];
                        u.weighted_busy_ms = wbms[s];
                        u.queries = nq[s];
                        p.usage[d->usage_off + (pk[s] & 0xff)] = u;
                    }
                }
            }
            __syncwarp(seg_mask);
            sidx = -1;
        }
    }
}

template <int W, int S, int SCHED>
void* pick_flags(bool rec, bool full) {
    if (rec) return (void*)&sim_kernel<W, S, SCHED, true, true>;
    return full ? (void*)&sim_kernel<W, S, SCHED, false, true> : (void*)&sim_kernel<W, S, SCHED, false, false>;
}

void* pick_sim(int W, int S, int sched, bool rec, bool full) {
#define MSV_PICK(w, s)                                                                                     \
    if (W == w && S == s)                                                                                  \
        return sched == MSV_ELSA ? pick_flags<w, s, MSV_ELSA>(rec, full) : pick_flags<w, s, MSV_FIFS>(rec, full);
    MSV_PICK(4, 1)
    MSV_PICK(8, 1)
    MSV_PICK(16, 1)
#undef MSV_PICK
    return nullptr;
}

}  // namespace

void* sim_warp_fn(int S, int sched, bool rec, bool full, bool lazy, bool stream);  // msv_sim_warp.cu
size_t sim_warp_smem_bytes(int S, int n_cells);

size_t sim_smem_bytes(int W, int S, int n_cells) {
    if (W == 32) return sim_warp_smem_bytes(S, n_cells);
    const size_t tab = ((size_t)2 * n_cells * sizeof(double) + 15) & ~(size_t)15;
    size_t per_warp = 0;
    if (W == 4) per_warp = sizeof(SegSmem<4, 1>);
    else if (W == 8) per_warp = sizeof(SegSmem<8, 1>);
    else per_warp = sizeof(SegSmem<16, 1>);
    return tab + (size_t)kSimWarpsPerBlock * per_warp;
}

static void* sim_fn_for(int W, int S, int sched, bool rec, bool full, bool lazy) {
    return W == 32 ? sim_warp_fn(S, sched, rec, full, lazy, false) : pick_sim(W, S, sched, rec, full);
}

// Dynamic shared-memory opt-in, raised monotonically per (kernel, device) under a lock:
// several contexts (threads) may launch the same kernel with different table sizes at
// once, and a lower limit set by one must never invalidate another's launch in flight.
cudaError_t ensure_dyn_smem(const void* fn, size_t bytes) {
    static std::mutex mu;
    static std::map<std::pair<const void*, int>, size_t> limit;
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> lk(mu);
    size_t& cur = limit[{fn, dev}];
    if (bytes <= cur) return cudaSuccess;
    const cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
    if (e == cudaSuccess) cur = bytes;
    return e;
}

int sim_max_blocks_per_sm(int W, int S, int sched, bool records, bool full, bool lazy, int n_cells) {
    void* fn = sim_fn_for(W, S, sched, records, full, lazy);
    if (!fn) return 0;
    const size_t smem = sim_smem_bytes(W, S, n_cells);
    if (ensure_dyn_smem(fn, smem) != cudaSuccess) return 0;
    int blocks = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks, fn, kSimWarpsPerBlock * 32, smem) != cudaSuccess)
        return 0;
    return blocks;
}

cudaError_t launch_sim(int W, int S, int sched, bool records, const SimParams& p, int blocks, cudaStream_t stream) {
    const bool full = records || p.any_routing || p.any_bad || p.any_check_wait || p.any_usage;
    if (p.stream) {  // one 2-warp block per scenario: trace generator + simulator
        if (W != 32 || full) return cudaErrorInvalidValue;
        void* fn = sim_warp_fn(S, sched, false, false, p.lazy != 0, true);
        if (!fn) return cudaErrorInvalidValue;
        const size_t smem = sim_smem_bytes(W, S, p.n_cells);  // (sized for 4 warps; 2 used)
        cudaError_t e = ensure_dyn_smem(fn, smem);
        if (e != cudaSuccess) return e;
        void* args[] = {const_cast<SimParams*>(&p)};
        return cudaLaunchKernel(fn, dim3(p.n_work), dim3(64), args, smem, stream);
    }
    void* fn = sim_fn_for(W, S, sched, records, full, p.lazy != 0);
    if (!fn) return cudaErrorInvalidValue;
    const size_t smem = sim_smem_bytes(W, S, p.n_cells);
    cudaError_t e = ensure_dyn_smem(fn, smem);
    if (e != cudaSuccess) return e;
    void* args[] = {const_cast<SimParams*>(&p)};
    return cudaLaunchKernel(fn, dim3(blocks), dim3(kSimWarpsPerBlock * 32), args, smem, stream);
}

}  // namespace msv
