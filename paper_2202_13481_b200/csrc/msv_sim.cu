// K2 sim_kernel: run() (engine.hpp:115-253) with ELSA (sched.hpp:119-143) or FIFS
// (sched.hpp:154-170) for a grid of scenarios.
//
// Mapping: a warp holds 32/W scenario segments of W lanes; lane slot s of segment
// lane l owns the partition at by_ascending_size order index o = s*W + l
// (sched.hpp:96-104), so warp ballots enumerate partitions in ELSA's scan order.
// Each segment streams its scenario's arrivals; per arrival:
//   1. every lane retires its own completions with time <= now, in chain order,
//      with no warp collective (completions on different partitions commute and a
//      completion precedes an arrival at equal time, engine.hpp:101-107);
//   2. every lane evaluates Eq. 1 t_wait / Eq. 2 slack for its partition;
//      Step A = first set bit of a ballot, Step B = a REDUX argmin (W = 32) or a
//      shuffle tree (W < 32) with order tie-break; FIFS = two REDUX key minima;
//   3. the chosen lane starts the query or appends it to its FIFO (shared-memory
//      ring, overflow list threaded through query ids in global memory).
// Measured latencies land at samples[q - m0] (arrivals are sorted, so the measured
// set is the suffix from the first arrival >= warmup), ready for K3.
#include "msv_device.cuh"

namespace msv {

namespace {

constexpr uint64_t kQidMask = (1ull << 40) - 1;

template <int S>
struct MinBlocks {
    static constexpr int value = S == 1 ? 6 : (S == 2 ? 4 : 2);
};

template <int W, int S, int SCHED, bool REC>
__global__ void __launch_bounds__(kSimWarpsPerBlock * 32, MinBlocks<S>::value) sim_kernel(const SimParams p) {
    extern __shared__ __align__(16) unsigned char smem[];
    double* s_lat = reinterpret_cast<double*>(smem);
    double* s_util = s_lat + p.n_cells;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const size_t tab_bytes = ((size_t)2 * p.n_cells * sizeof(double) + 15) & ~(size_t)15;
    // Per-warp FIFO rings, [slot][entry][lane] so a warp access is conflict-free.
    double* q_est = reinterpret_cast<double*>(smem + tab_bytes) + (size_t)warp * (3 * S * kQCap * 32);
    double* q_arr = q_est + S * kQCap * 32;
    uint64_t* q_meta = reinterpret_cast<uint64_t*>(q_arr + S * kQCap * 32);
    for (int c = threadIdx.x; c < p.n_cells; c += blockDim.x) {
        s_lat[c] = p.lat[c];
        s_util[c] = p.util[c];
    }
    __syncthreads();

    const int seg_base = (lane / W) * W;
    const int sl = lane - seg_base;
    const unsigned seg_mask = (W == 32) ? kFull : (((1u << W) - 1u) << seg_base);

    // ---- segment state (identical in all lanes of a segment) ----
    int32_t sidx = -1;
    bool done = false;
    int64_t n = 0, i = 0, win_base = 0, m0 = -1;
    double win_t = 0.0, nxt_t = 0.0;
    int32_t win_b = 0, nxt_b = 0;
    double duration = 0.0, warmup = 0.0, sla = 0.0, alpha = 1.0, beta = 1.0;
    bool unit_ab = true;
    int32_t flags = 0, status = 0, bmax = 0, usage_off = -1;
    const double* g_arr = nullptr;
    const int32_t* g_bat = nullptr;
    uint32_t* g_next = nullptr;
    double* samples = nullptr;
    msv_record* rec = nullptr;
    bool routed = false;

    // ---- per-lane partition slots ----
    bool act[S], busy[S], fok[S];
    int32_t pid[S], kk[S], row[S], qh[S], qn[S];
    uint32_t gh[S], gt[S], gn[S];
    double c_start[S], c_est[S], c_comp[S], c_arr[S], c_util[S], fold[S], bms[S], wbms[S];
    uint64_t c_q[S], rmask[S];
    uint32_t nq[S];
#pragma unroll
    for (int s = 0; s < S; ++s) {
        act[s] = busy[s] = false;
        fok[s] = true;
        pid[s] = kk[s] = row[s] = qh[s] = qn[s] = 0;
        gh[s] = gt[s] = gn[s] = 0;
        c_start[s] = c_est[s] = c_comp[s] = c_arr[s] = c_util[s] = fold[s] = bms[s] = wbms[s] = 0.0;
        c_q[s] = rmask[s] = 0;
        nq[s] = 0;
    }
    // ---- per-lane accumulators ----
    uint32_t viol = 0, mviol = 0;
    double last_fin = 0.0, wdiff = 0.0;
    uint64_t hash = 0, lmin = ~0ull, lmax = 0;

    while (true) {
        // ---- acquire a scenario (segment-uniform branch) ----
        if (sidx < 0 && !done) {
            int w = 0;
            if (sl == 0) w = atomicAdd(p.counter, 1);
            w = __shfl_sync(seg_mask, w, seg_base);
            if (w >= p.n_work) {
                done = true;
            } else {
                sidx = p.work[w];
                const DevScen& d = p.scen[sidx];
                n = *d.n;
                duration = d.duration_ms;
                warmup = d.warmup_ms;
                sla = d.sla;
                alpha = d.alpha;
                beta = d.beta;
                unit_ab = alpha == 1.0 && beta == 1.0;  // 1*x == x exactly: same bits
                flags = d.flags;
                bmax = d.b_max;
                usage_off = d.usage_off;
                g_arr = d.arrival;
                g_bat = d.batch;
                g_next = d.next;
                samples = d.samples;
                rec = d.records;
                routed = d.route_mask != nullptr;
                status = 0;
                i = 0;
                m0 = -1;
                win_base = 0;
                win_t = (sl < n) ? g_arr[sl] : 0.0;
                win_b = (sl < n) ? g_bat[sl] : 0;
                nxt_t = (W + sl < n) ? g_arr[W + sl] : 0.0;
                nxt_b = (W + sl < n) ? g_bat[W + sl] : 0;
#pragma unroll
                for (int s = 0; s < S; ++s) {
                    const int o = s * W + sl;
                    act[s] = o < d.P;
                    if (act[s]) {
                        const DevPart dp = d.parts[o];
                        pid[s] = dp.pid;
                        kk[s] = dp.k;
                        row[s] = dp.row;
                        rmask[s] = routed ? d.route_mask[o] : 0ull;
                    }
                    busy[s] = false;
                    fok[s] = true;
                    fold[s] = 0.0;
                    qh[s] = qn[s] = 0;
                    gh[s] = gt[s] = gn[s] = 0;
                    bms[s] = wbms[s] = 0.0;
                    nq[s] = 0;
                }
                viol = mviol = 0;
                last_fin = 0.0;
                wdiff = 0.0;
                hash = 0;
                lmin = ~0ull;
                lmax = 0;
            }
        }
        if (__all_sync(kFull, done)) break;

        // ---- next event of this segment: an arrival, or the end marker ----
        if (!done && i < n && i - win_base >= W) {
            win_base += W;
            win_t = nxt_t;
            win_b = nxt_b;
            const int64_t j = win_base + W + sl;
            if (j < n) {
                nxt_t = g_arr[j];
                nxt_b = g_bat[j];
            }
        }
        const int src = seg_base + (int)((i - win_base) & (W - 1));
        const double tw = __shfl_sync(kFull, win_t, src);
        const int32_t bw = __shfl_sync(kFull, win_b, src);
        bool arrival = false, ending = false;
        double t = -INFINITY;
        int32_t b = 0;
        if (!done) {
            if (i < n) {
                t = tw;
                b = bw;
                arrival = true;
                if (m0 < 0 && t >= warmup) m0 = i;  // measured iff arrival >= warmup (engine.hpp:262)
            } else {
                t = INFINITY;  // drain everything (no horizon cut-off)
                ending = true;
            }
        }

        // ---- 1. completions with time <= t, lane-local, in chain order ----
#pragma unroll
        for (int s = 0; s < S; ++s) {
            while (busy[s] && c_comp[s] <= t) {
                // completion (engine.hpp:167-187)
                const double now = c_comp[s];
                const double lat = now - c_arr[s];
                const bool met = lat <= sla;
                const double ran = now - c_start[s];
                bms[s] = bms[s] + ran;
                wbms[s] = wbms[s] + ran * c_util[s];
                nq[s] += 1;
                last_fin = (last_fin < now) ? now : last_fin;
                viol += met ? 0u : 1u;
                if (c_arr[s] >= warmup) {
                    mviol += met ? 0u : 1u;
                    samples[c_q[s] - (uint64_t)m0] = lat;
                    const uint64_t lb = msv_dbits(lat) | kSignBit;  // order key (lat >= 0)
                    lmin = lb < lmin ? lb : lmin;
                    lmax = lb > lmax ? lb : lmax;
                }
                hash += msv_query_digest(c_q[s], pid[s], c_start[s], now);
                if (REC) {
                    rec[c_q[s]].start_ms = c_start[s];
                    rec[c_q[s]].finish_ms = now;
                }
                // start the queue head at `now` (engine.hpp:151-157, 181-185)
                if (qn[s] > 0) {
                    const int e = (s * kQCap + qh[s]) * 32 + lane;
                    const double est = q_est[e];
                    const double arr = q_arr[e];
                    const uint64_t meta = q_meta[e];
                    qh[s] = (qh[s] + 1) & (kQCap - 1);
                    qn[s] -= 1;
                    if (gn[s] > 0) {  // refill the ring from the overflow list
                        const uint32_t q = gh[s];
                        gh[s] = g_next[q];
                        gn[s] -= 1;
                        const int32_t qb = g_bat[q];
                        const int e2 = (s * kQCap + ((qh[s] + qn[s]) & (kQCap - 1))) * 32 + lane;
                        q_est[e2] = s_lat[row[s] + qb - 1];
                        q_arr[e2] = g_arr[q];
                        q_meta[e2] = (uint64_t)q | ((uint64_t)qb << 40);
                        qn[s] += 1;
                    }
                    c_start[s] = now;
                    c_est[s] = est;
                    c_comp[s] = now + est;
                    c_arr[s] = arr;
                    c_q[s] = meta & kQidMask;
                    c_util[s] = s_util[row[s] + (int)(meta >> 40) - 1];
                    fok[s] = (qn[s] == 0);
                    fold[s] = 0.0;
                } else {
                    busy[s] = false;
                    fok[s] = true;
                    fold[s] = 0.0;
                }
            }
        }

        // ---- 2. dispatch (engine.hpp:189-230) ----
        if (arrival && (b < 1 || b > bmax)) {  // LookupError at this query (profile.hpp:127-129)
            status = MSV_LOOKUP;
            i = n;
            arrival = false;
        }
        double est_n[S], wv[S];
        bool cand[S];
#pragma unroll
        for (int s = 0; s < S; ++s) {
            cand[s] = arrival && act[s];
            est_n[s] = (cand[s] && row[s] >= 0) ? s_lat[row[s] + b - 1] : 0.0;
            wv[s] = 0.0;
        }
        if (p.any_routing) {  // segment routing with fallback to all (engine.hpp:197-206)
#pragma unroll
            for (int s = 0; s < S; ++s)
                if (routed) cand[s] = cand[s] && (((rmask[s] >> (b - 1)) & 1ull) != 0);
            unsigned anyc = 0;
#pragma unroll
            for (int s = 0; s < S; ++s) anyc |= __ballot_sync(kFull, cand[s]);
            if ((anyc & seg_mask) == 0) {
#pragma unroll
                for (int s = 0; s < S; ++s) cand[s] = arrival && act[s];
            }
        }
        // Partitions whose size the profile lacks (row < 0) raise LookupError when a
        // lookup reaches them (profile.hpp:127): ELSA's Step-A scan, or FIFS choosing one.
        bool bad[S];
        int bad_slot = -1, bad_lane = -1;
#pragma unroll
        for (int s = 0; s < S; ++s) bad[s] = false;
        if (p.any_bad) {
#pragma unroll
            for (int s = 0; s < S; ++s) {
                bad[s] = cand[s] && row[s] < 0;
                const unsigned bb = __ballot_sync(kFull, bad[s]) & seg_mask;
                if (bad_lane < 0 && bb != 0) {
                    bad_lane = __ffs(bb) - 1;
                    bad_slot = s;
                }
            }
        }
        const bool check_wait = p.any_check_wait && (flags & MSV_FLAG_CHECK_WAIT);
        if (SCHED == MSV_ELSA || check_wait) {
#pragma unroll
            for (int s = 0; s < S; ++s) {
                if (!cand[s]) continue;
                if (!fok[s]) {  // exact left fold of the FIFO (sched.hpp:78-79)
                    double acc = 0.0;
                    for (int j = 0; j < qn[s]; ++j)
                        acc = acc + q_est[(s * kQCap + ((qh[s] + j) & (kQCap - 1))) * 32 + lane];
                    uint32_t q = gh[s];
                    for (uint32_t j = 0; j < gn[s]; ++j) {
                        acc = acc + s_lat[row[s] + g_bat[q] - 1];
                        q = g_next[q];
                    }
                    fold[s] = acc;
                    fok[s] = true;
                }
                double w = fold[s];
                if (busy[s]) {  // sched.hpp:80-83
                    const double x = c_est[s] - (t - c_start[s]);
                    w = w + ((0.0 < x) ? x : 0.0);
                }
                wv[s] = w;
                if (check_wait) {  // engine.hpp:208-217
                    double gt_w = fold[s];
                    if (busy[s]) {
                        const double y = c_comp[s] - t;
                        gt_w = gt_w + ((0.0 < y) ? y : 0.0);
                    }
                    const double dd = fabs(gt_w - w);
                    wdiff = (wdiff < dd) ? dd : wdiff;
                }
            }
        }

        int ch_lane = -1, ch_slot = 0, kind = 0;
        if constexpr (SCHED == MSV_ELSA) {
            // Step A: first in (k, id) order with sla > alpha*(w + beta*est), strict.
#pragma unroll
            for (int s = 0; s < S; ++s) {
                const bool ok = cand[s] && !bad[s];
                const bool pred = ok && (unit_ab ? (sla > wv[s] + est_n[s]) : (sla > alpha * (wv[s] + beta * est_n[s])));
                const unsigned bA = __ballot_sync(kFull, pred) & seg_mask;
                if (ch_lane < 0 && bA != 0) {
                    ch_lane = __ffs(bA) - 1;
                    ch_slot = s;
                }
            }
            kind = MSV_SLACK_SATISFYING;
            // Step B: argmin of w + est, earliest in order on ties (strict <).
            const bool needB = arrival && ch_lane < 0;
            if (__any_sync(kFull, needB)) {
                uint64_t fb[S];
                uint64_t vmin = ~0ull;
#pragma unroll
                for (int s = 0; s < S; ++s) {
                    fb[s] = cand[s] ? msv_dbits(wv[s] + est_n[s]) : ~0ull;
                    vmin = fb[s] < vmin ? fb[s] : vmin;
                }
                vmin = seg_min_u64<W>(vmin);
#pragma unroll
                for (int s = 0; s < S; ++s) {
                    const unsigned bB = __ballot_sync(kFull, cand[s] && fb[s] == vmin) & seg_mask;
                    if (needB && ch_lane < 0 && bB != 0) {
                        ch_lane = __ffs(bB) - 1;
                        ch_slot = s;
                        kind = MSV_FASTEST_FALLBACK;
                    }
                }
            }
        } else {
            // FIFS: idle -> largest k, then lowest id; else shortest queue, lowest id.
            uint32_t ki[S];
            uint32_t mi = ~0u;
#pragma unroll
            for (int s = 0; s < S; ++s) {
                ki[s] = (cand[s] && !busy[s]) ? (((0x7FFFu - (uint32_t)kk[s]) << 16) | (uint32_t)pid[s]) : ~0u;
                mi = ki[s] < mi ? ki[s] : mi;
            }
            mi = seg_min_u32<W>(mi);
            const bool idle = mi != ~0u;
            kind = idle ? MSV_IDLE_LARGEST : MSV_SHORTEST_QUEUE;
            uint32_t kq[S];
            uint32_t mq = ~0u;
#pragma unroll
            for (int s = 0; s < S; ++s) kq[s] = ~0u;
            if (__any_sync(kFull, arrival && !idle)) {
#pragma unroll
                for (int s = 0; s < S; ++s) {
                    const uint32_t len = (uint32_t)qn[s] + gn[s];
                    kq[s] = cand[s] ? (((len < 0xFFFFFFu ? len : 0xFFFFFFu) << 8) | (uint32_t)pid[s]) : ~0u;
                    mq = kq[s] < mq ? kq[s] : mq;
                }
                mq = seg_min_u32<W>(mq);
            }
#pragma unroll
            for (int s = 0; s < S; ++s) {
                const bool hit = idle ? (ki[s] == mi) : (kq[s] == mq && mq != ~0u);
                const unsigned bsel = __ballot_sync(kFull, arrival && hit) & seg_mask;
                if (ch_lane < 0 && bsel != 0) {
                    ch_lane = __ffs(bsel) - 1;
                    ch_slot = s;
                }
            }
        }

        if (p.any_bad && arrival && bad_lane >= 0) {
            bool err;
            if constexpr (SCHED == MSV_ELSA) {  // the Step-A scan reached the bad partition first
                err = ch_lane < 0 || kind == MSV_FASTEST_FALLBACK || bad_slot < ch_slot ||
                      (bad_slot == ch_slot && bad_lane < ch_lane);
            } else {  // FIFS chose a partition whose latency lookup fails (engine.hpp:226)
                bool mine = false;
#pragma unroll
                for (int s = 0; s < S; ++s) mine |= (lane == ch_lane && s == ch_slot && bad[s]);
                err = (__ballot_sync(seg_mask, mine) & seg_mask) != 0;
            }
            if (err) {
                status = MSV_LOOKUP;
                i = n;
                arrival = false;
            }
        }

        // ---- 3. start or enqueue on the chosen partition (engine.hpp:225-230) ----
        if (arrival) {
#pragma unroll
            for (int s = 0; s < S; ++s) {
                if (lane == ch_lane && s == ch_slot) {
                    const double est = est_n[s];
                    if (!busy[s]) {
                        busy[s] = true;
                        c_start[s] = t;
                        c_est[s] = est;
                        c_comp[s] = t + est;
                        c_arr[s] = t;
                        c_q[s] = (uint64_t)i;
                        c_util[s] = s_util[row[s] + b - 1];
                    } else {
                        if (gn[s] == 0 && qn[s] < kQCap) {
                            const int e = (s * kQCap + ((qh[s] + qn[s]) & (kQCap - 1))) * 32 + lane;
                            q_est[e] = est;
                            q_arr[e] = t;
                            q_meta[e] = (uint64_t)i | ((uint64_t)b << 40);
                            qn[s] += 1;
                        } else {
                            const uint32_t q = (uint32_t)i;
                            if (gn[s] == 0) gh[s] = q;
                            else g_next[gt[s]] = q;
                            gt[s] = q;
                            gn[s] += 1;
                        }
                        if (fok[s]) fold[s] = fold[s] + est;
                    }
                    if (REC) {
                        rec[i].partition = pid[s];
                        rec[i].kind = kind;
                    }
                }
            }
            ++i;
        }

        // ---- end of trace: reduce the segment and publish ----
        if (ending) {
            const uint64_t v0 = seg_sum_u64<W>((uint64_t)viol, seg_mask);
            const uint64_t v2 = seg_sum_u64<W>((uint64_t)mviol, seg_mask);
            const uint64_t hsum = seg_sum_u64<W>(hash, seg_mask);
            const double lf = seg_max_f64<W>(last_fin, seg_mask);
            const double wd = seg_max_f64<W>(wdiff, seg_mask);
            const uint64_t mn = seg_minm_u64<W>(lmin, seg_mask);
            const uint64_t mx = seg_max_u64<W>(lmax, seg_mask);
            if (sl == 0) {
                DevOut o;
                o.violations = (int64_t)v0;
                o.measured = m0 >= 0 ? n - m0 : 0;
                o.measured_violations = (int64_t)v2;
                o.n_samples = o.measured;
                o.horizon_ms = (duration < lf) ? lf : duration;  // engine.hpp:237
                o.max_wait_diff = wd;
                o.hash = hsum;
                o.lat_min_bits = mn;
                o.lat_max_bits = mx;
                o.status = status;
                o.pad = 0;
                p.out[sidx] = o;
            }
            if (usage_off >= 0) {
#pragma unroll
                for (int s = 0; s < S; ++s) {
                    if (act[s]) {
                        msv_usage u;
                        u.busy_ms = bms[s];
                        u.weighted_busy_ms = wbms[s];
                        u.queries = nq[s];
                        p.usage[usage_off + pid[s]] = u;
                    }
                }
            }
            sidx = -1;
        }
    }
}

template <int W, int S, int SCHED, bool REC>
void* sim_fn() {
    return reinterpret_cast<void*>(&sim_kernel<W, S, SCHED, REC>);
}

void* pick_sim(int W, int S, int sched, bool rec) {
#define MSV_PICK(w, s)                                                                                    \
    if (W == w && S == s) {                                                                               \
        if (sched == MSV_ELSA) return rec ? sim_fn<w, s, MSV_ELSA, true>() : sim_fn<w, s, MSV_ELSA, false>(); \
        return rec ? sim_fn<w, s, MSV_FIFS, true>() : sim_fn<w, s, MSV_FIFS, false>();                     \
    }
    MSV_PICK(4, 1)
    MSV_PICK(8, 1)
    MSV_PICK(16, 1)
#undef MSV_PICK
    return nullptr;
}

}  // namespace

void* sim_warp_fn(int S, int sched, bool rec, bool full);  // msv_sim_warp.cu
size_t sim_warp_smem_bytes(int S, int n_cells);

size_t sim_smem_bytes(int W, int S, int n_cells) {
    if (W == 32) return sim_warp_smem_bytes(S, n_cells);
    const size_t tab = ((size_t)2 * n_cells * sizeof(double) + 15) & ~(size_t)15;
    return tab + (size_t)kSimWarpsPerBlock * 3 * S * kQCap * 32 * sizeof(double);
}

static void* sim_fn_for(int W, int S, int sched, bool rec, bool full) {
    return W == 32 ? sim_warp_fn(S, sched, rec, full) : pick_sim(W, S, sched, rec);
}

int sim_max_blocks_per_sm(int W, int S, int sched, bool records, bool full, int n_cells) {
    void* fn = sim_fn_for(W, S, sched, records, full);
    if (!fn) return 0;
    const size_t smem = sim_smem_bytes(W, S, n_cells);
    if (cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess) return 0;
    int blocks = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks, fn, kSimWarpsPerBlock * 32, smem) != cudaSuccess)
        return 0;
    return blocks;
}

cudaError_t launch_sim(int W, int S, int sched, bool records, const SimParams& p, int blocks, cudaStream_t stream) {
    const bool full = records || p.any_routing || p.any_bad || p.any_check_wait;
    void* fn = sim_fn_for(W, S, sched, records, full);
    if (!fn) return cudaErrorInvalidValue;
    const size_t smem = sim_smem_bytes(W, S, p.n_cells);
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    void* args[] = {const_cast<SimParams*>(&p)};
    return cudaLaunchKernel(fn, dim3(blocks), dim3(kSimWarpsPerBlock * 32), args, smem, stream);
}

}  // namespace msv
