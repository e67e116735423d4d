// K2 sim_kernel: run() (engine.hpp:115-253) with ELSA (sched.hpp:119-143) or FIFS
// (sched.hpp:154-170), segmented variant for plans of P <= W partitions, W in
// {4, 8, 16}: a warp runs G = 32/W scenarios side by side, one segment of W lanes
// each, all segments advancing one arrival per iteration (lockstep).
//
// Per arrival (every kernel of K2 follows this protocol):
//   1. every lane retires its own completions with time <= now, in chain order, with
//      no warp collective (completions on different partitions commute and a
//      completion precedes an arrival at equal time, engine.hpp:101-107);
//   2. every lane evaluates Eq. 1 (t_wait, kept as an exact FIFO fold) and Eq. 2 for
//      its partition; Step A = first set bit of the segment's ballot bits, Step B =
//      a shuffle-tree argmin over the segment with order tie-break; FIFS = (k, id) /
//      (queue length, id) key minima;
//   3. the chosen lane starts the query or appends it to its FIFO (shared-memory
//      ring, overflow list threaded through query ids in global memory).
// Each segment keeps a double-buffered 32-arrival window in shared memory, refilled
// by cp.async one window ahead. Measured latencies land at samples[q - m0]
// (arrivals are sorted, so the measured set is the suffix from the first
// arrival >= warmup), ready for K3.
#include <cuda_pipeline.h>

#include "msv_device.cuh"

namespace msv {

namespace {

constexpr uint64_t kQidMask = (1ull << 40) - 1;
constexpr int kSegMinBlocks = 6;

template <int W>
struct SegSmem {
    static constexpr int G = 32 / W;
    double q_est[kQCap][32];
    double q_arr[kQCap][32];
    uint64_t q_meta[kQCap][32];
    double win_t[2][32][G];  // [buffer][entry][segment]
    int32_t win_b[2][32][G];
    uint32_t g_head[32];     // overflow list head / tail per lane
    uint32_t g_tail[32];
};

template <int W, int SCHED, bool REC, bool FULL>
__global__ void __launch_bounds__(kSimWarpsPerBlock * 32, kSegMinBlocks) sim_kernel(const SimParams p) {
    constexpr bool kFold = (SCHED == MSV_ELSA) || FULL;
    extern __shared__ __align__(16) unsigned char smem[];
    double* s_lat = reinterpret_cast<double*>(smem);
    double* s_util = s_lat + p.n_cells;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const size_t tab_bytes = ((size_t)2 * p.n_cells * sizeof(double) + 15) & ~(size_t)15;
    SegSmem<W>& M = reinterpret_cast<SegSmem<W>*>(smem + tab_bytes)[warp];
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
    double sla = 0.0, warmup = 0.0, alpha = 1.0, beta = 1.0;
    bool unit = true, check_wait = false;
    int bmax = 0;
    // ---- per-lane partition slot ----
    bool act = false, busy = false;
    int32_t row = 0, pk = 0, qh = 0, qn = 0;
    uint32_t gn = 0, nq = 0;
    double c_start = 0.0, c_est = 0.0, c_comp = 0.0, c_arr = 0.0, fold = 0.0, bms = 0.0, wbms = 0.0;
    uint64_t c_meta = 0;
    uint32_t viol = 0, mviol = 0;
    uint64_t hash = 0, lmin = ~0ull, lmax = 0;
    double wdiff = 0.0;

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
    auto refold = [&]() {
        double acc = 0.0;
#pragma unroll 1
        for (int k = 0; k < qn; ++k) acc = acc + M.q_est[(qh + k) & (kQCap - 1)][lane];
        if (gn > 0) {
            uint32_t g = M.g_head[lane];
#pragma unroll 1
            for (uint32_t k = 0; k < gn; ++k) {
                acc = acc + s_lat[row + g_bat[g] - 1];
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
                act = sl < d->P;
                row = 0;
                pk = 0;
                if (act) {
                    const DevPart dp = d->parts[sl];
                    pk = dp.pid | (dp.k << 8);
                    row = dp.row;
                }
                busy = false;
                qh = qn = 0;
                gn = nq = 0;
                c_start = c_est = c_comp = c_arr = 0.0;
                fold = bms = wbms = 0.0;
                c_meta = 0;
                viol = mviol = 0;
                hash = 0;
                lmin = ~0ull;
                lmax = 0;
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
        int b = 0;
        if (arrival) {
            t = M.win_t[buf][i - win_base][seg];
            b = M.win_b[buf][i - win_base][seg];
            if (m0 < 0 && t >= warmup) m0 = i;  // measured iff arrival >= warmup (engine.hpp:262)
        } else if (ending) {
            t = INFINITY;  // drain everything (no horizon cut-off)
        }

        // ---- 1. completions with time <= t, lane-local, in chain order ----
        while (busy && c_comp <= t) {  // engine.hpp:167-187
            const double now = c_comp;
            const double lat = now - c_arr;
            const bool met = lat <= sla;
            const double ran = now - c_start;
            const uint64_t q = c_meta & kQidMask;
            const int cb = (int)(c_meta >> 40);
            bms = bms + ran;
            wbms = wbms + ran * s_util[row + cb - 1];
            nq += 1;
            viol += met ? 0u : 1u;
            if (c_arr >= warmup) {
                mviol += met ? 0u : 1u;
                d->samples[(uint32_t)q - (uint32_t)m0] = lat;
                const uint64_t lb = msv_dbits(lat) | kSignBit;  // order key (lat >= 0)
                lmin = lb < lmin ? lb : lmin;
                lmax = lb > lmax ? lb : lmax;
            }
            hash += msv_query_digest(q, pk & 0xff, c_start, now);
            if (REC) {
                d->records[q].start_ms = c_start;
                d->records[q].finish_ms = now;
            }
            if (qn > 0) {  // start the queue head now (engine.hpp:181-185)
                const double est = M.q_est[qh][lane];
                c_arr = M.q_arr[qh][lane];
                c_meta = M.q_meta[qh][lane];
                qh = (qh + 1) & (kQCap - 1);
                qn -= 1;
                if (gn > 0) {  // refill the ring from the overflow list
                    const uint32_t g = M.g_head[lane];
                    M.g_head[lane] = d->next[g];
                    gn -= 1;
                    const int32_t gb = g_bat[g];
                    const int e2 = (qh + qn) & (kQCap - 1);
                    M.q_est[e2][lane] = s_lat[row + gb - 1];
                    M.q_arr[e2][lane] = g_arr[g];
                    M.q_meta[e2][lane] = (uint64_t)g | ((uint64_t)gb << 40);
                    qn += 1;
                }
                c_start = now;
                c_est = est;
                c_comp = now + est;
                if (kFold) fold = refold();
            } else {
                busy = false;
                fold = 0.0;
            }
        }

        // ---- 2. dispatch (engine.hpp:189-230) ----
        bool go = arrival;
        if (go && (b < 1 || b > bmax)) {  // LookupError at this query (profile.hpp:127-129)
            status = MSV_LOOKUP;
            go = false;
        }
        bool cand = go && act;
        const double x = c_est - (t - c_start);
        const double wv = fold + ((busy && 0.0 < x) ? x : 0.0);  // Eq. 1 (sched.hpp:77-85)
        const double est_n = (FULL && row < 0) ? 0.0 : s_lat[row + (go ? b : 1) - 1];
        bool bad = false;
        if (FULL) {
            if (p.any_routing) {  // engine.hpp:197-206
                if (go && d->route_mask != nullptr)
                    cand = cand && (((d->route_mask[sl] >> (b - 1)) & 1ull) != 0);
                if ((__ballot_sync(kFull, cand) & seg_mask) == 0) cand = go && act;
            }
            bad = cand && row < 0;
            if (check_wait && cand && !bad) {  // engine.hpp:208-217
                const double y = c_comp - t;
                const double gw = fold + ((busy && 0.0 < y) ? y : 0.0);
                const double dd = fabs(gw - wv);
                wdiff = (wdiff < dd) ? dd : wdiff;
            }
        }
        const unsigned bad_bits = FULL ? (__ballot_sync(kFull, bad) & seg_mask) : 0u;
        int ch = -1, kind = 0;
        if constexpr (SCHED == MSV_ELSA) {
            const bool ok = cand && !bad;
            const bool pred = ok && (unit ? (sla > wv + est_n) : (sla > alpha * (wv + beta * est_n)));
            const unsigned bA = __ballot_sync(kFull, pred) & seg_mask;
            if (bA) ch = __ffs(bA) - 1;
            kind = MSV_SLACK_SATISFYING;
            const bool needB = go && ch < 0;
            if (__any_sync(kFull, needB)) {  // Step B (sched.hpp:132-142)
                const uint64_t fb = ok ? msv_dbits(wv + est_n) : ~0ull;
                const uint64_t vmin = seg_min_u64<W>(fb);
                const unsigned bB = __ballot_sync(kFull, ok && fb == vmin) & seg_mask;
                if (needB && bB) {
                    ch = __ffs(bB) - 1;
                    kind = MSV_FASTEST_FALLBACK;
                }
            }
            // a size missing from the profile is a LookupError once the scan reaches it
            if (FULL && go && bad_bits && (ch < 0 || kind == MSV_FASTEST_FALLBACK || (__ffs(bad_bits) - 1) < ch)) {
                status = MSV_LOOKUP;
                go = false;
            }
        } else {
            const uint32_t ki =
                (cand && !busy) ? (((0x7FFFu - ((uint32_t)pk >> 8)) << 16) | ((uint32_t)pk & 0xffu)) : ~0u;
            const uint32_t mi = seg_min_u32<W>(ki);
            const uint32_t len = (uint32_t)qn + gn;
            const uint32_t kq = cand ? (((len < 0xFFFFFFu ? len : 0xFFFFFFu) << 8) | ((uint32_t)pk & 0xffu)) : ~0u;
            const bool idle = mi != ~0u;
            uint32_t mq = ~0u;
            if (__any_sync(kFull, go && !idle)) mq = seg_min_u32<W>(kq);
            const unsigned bs = __ballot_sync(kFull, idle ? (ki == mi) : (kq == mq && mq != ~0u)) & seg_mask;
            if (go && bs) ch = __ffs(bs) - 1;
            kind = idle ? MSV_IDLE_LARGEST : MSV_SHORTEST_QUEUE;
            if (FULL && go && ch >= 0 && ((bad_bits >> ch) & 1u)) {  // chosen size missing (engine.hpp:226)
                status = MSV_LOOKUP;
                go = false;
            }
        }

        // ---- 3. start or enqueue on the chosen partition (engine.hpp:225-230) ----
        if (go && lane == ch) {
            const uint64_t meta = (uint64_t)i | ((uint64_t)b << 40);
            if (!busy) {
                busy = true;
                c_start = t;
                c_est = est_n;
                c_comp = t + est_n;
                c_arr = t;
                c_meta = meta;
            } else {
                if (gn == 0 && qn < kQCap) {
                    const int e = (qh + qn) & (kQCap - 1);
                    M.q_est[e][lane] = est_n;
                    M.q_arr[e][lane] = t;
                    M.q_meta[e][lane] = meta;
                    qn += 1;
                } else {
                    if (gn == 0) M.g_head[lane] = (uint32_t)i;
                    else d->next[M.g_tail[lane]] = (uint32_t)i;
                    M.g_tail[lane] = (uint32_t)i;
                    gn += 1;
                }
                fold = fold + est_n;  // appending extends the left fold exactly
            }
            if (REC) {
                d->records[i].partition = pk & 0xff;
                d->records[i].kind = kind;
            }
        }
        if (arrival && status == 0) ++i;

        // ---- end of trace: reduce the segment and publish (segment-uniform, rare) ----
        if (ending) {
            __pipeline_wait_prior(0);  // no copy may land in a window after the segment moves on
            double lf = (nq > 0) ? c_comp : 0.0;  // last completion of this lane
            const uint64_t v0 = seg_sum_u64<W>((uint64_t)viol, seg_mask);
            const uint64_t v2 = seg_sum_u64<W>((uint64_t)mviol, seg_mask);
            const uint64_t hsum = seg_sum_u64<W>(hash, seg_mask);
            lf = seg_max_f64<W>(lf, seg_mask);
            const double wd = seg_max_f64<W>(wdiff, seg_mask);
            const uint64_t mn = seg_minm_u64<W>(lmin, seg_mask);
            const uint64_t mx = seg_max_u64<W>(lmax, seg_mask);
            if (sl == 0) {
                DevOut o;
                o.violations = (int64_t)v0;
                o.measured = m0 >= 0 ? n - m0 : 0;
                o.measured_violations = (int64_t)v2;
                o.n_samples = o.measured;
                o.horizon_ms = (d->duration_ms < lf) ? lf : d->duration_ms;  // engine.hpp:237
                o.max_wait_diff = wd;
                o.hash = hsum;
                o.lat_min_bits = mn;
                o.lat_max_bits = mx;
                o.status = status;
                o.pad = 0;
                p.out[sidx] = o;
            }
            if (act && d->usage_off >= 0) {
                msv_usage u;
                u.busy_ms = bms;
                u.weighted_busy_ms = wbms;
                u.queries = nq;
                p.usage[d->usage_off + (pk & 0xff)] = u;
            }
            __syncwarp(seg_mask);
            sidx = -1;
        }
    }
}

template <int W, int SCHED>
void* pick_flags(bool rec, bool full) {
    if (rec) return (void*)&sim_kernel<W, SCHED, true, true>;
    return full ? (void*)&sim_kernel<W, SCHED, false, true> : (void*)&sim_kernel<W, SCHED, false, false>;
}

void* pick_sim(int W, int sched, bool rec, bool full) {
#define MSV_PICK(w) \
    if (W == w) return sched == MSV_ELSA ? pick_flags<w, MSV_ELSA>(rec, full) : pick_flags<w, MSV_FIFS>(rec, full);
    MSV_PICK(4)
    MSV_PICK(8)
    MSV_PICK(16)
#undef MSV_PICK
    return nullptr;
}

}  // namespace

void* sim_warp_fn(int S, int sched, bool rec, bool full);  // msv_sim_warp.cu
size_t sim_warp_smem_bytes(int S, int n_cells);

size_t sim_smem_bytes(int W, int S, int n_cells) {
    if (W == 32) return sim_warp_smem_bytes(S, n_cells);
    const size_t tab = ((size_t)2 * n_cells * sizeof(double) + 15) & ~(size_t)15;
    const size_t per_warp = W == 4 ? sizeof(SegSmem<4>) : (W == 8 ? sizeof(SegSmem<8>) : sizeof(SegSmem<16>));
    return tab + (size_t)kSimWarpsPerBlock * per_warp;
}

static void* sim_fn_for(int W, int S, int sched, bool rec, bool full) {
    return W == 32 ? sim_warp_fn(S, sched, rec, full) : pick_sim(W, sched, rec, full);
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
    const bool full = records || p.any_routing || p.any_bad || p.any_check_wait || p.any_usage;
    void* fn = sim_fn_for(W, S, sched, records, full);
    if (!fn) return cudaErrorInvalidValue;
    const size_t smem = sim_smem_bytes(W, S, p.n_cells);
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    void* args[] = {const_cast<SimParams*>(&p)};
    return cudaLaunchKernel(fn, dim3(blocks), dim3(kSimWarpsPerBlock * 32), args, smem, stream);
}

}  // namespace msv
