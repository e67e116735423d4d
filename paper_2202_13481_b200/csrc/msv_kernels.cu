// sm_100a kernels of the scenario-grid engine.
//
//   K1 trace_gen_kernel  — sample_trace (workload.hpp:97-113) with a warp-parallel
//                          std::mt19937_64 twist and the glibc-log1p transcription.
//   K2 sim_kernel        — run() (engine.hpp:115-253) with ELSA (sched.hpp:119-143)
//                          or FIFS (sched.hpp:154-170): one warp segment of W lanes
//                          per scenario, one partition per lane slot.
//   K3 tail_kernel       — tail_latency (metrics.hpp:22-29): exact nearest-rank by
//                          MSB radix select over the IEEE bit patterns.
//   dispatch_kernel      — single elsa_dispatch / fifs_dispatch / t_wait decisions.
//
// This translation unit is compiled with -fmad=false: every decision and
// accumulation expression below must round exactly like the reference's x86-64
// SSE2 code (no contraction in the reference's -O3 build).
#include <math.h>

#include "msv_internal.h"
#include "msv_math.h"

namespace msv {

namespace {

constexpr unsigned kFull = 0xffffffffu;

// ---------------------------------------------------------------------------
// K1: trace generation
// ---------------------------------------------------------------------------

// BatchDistribution::sample's lower_bound (workload.hpp:48-53).
__device__ __forceinline__ int32_t cdf_sample(const double* __restrict__ cdf, int n, double u) {
    int lo = 0, len = n;
    while (len > 0) {
        const int half = len >> 1;
        if (__ldg(cdf + lo + half) < u) {
            lo += half + 1;
            len -= half + 1;
        } else {
            len = half;
        }
    }
    if (lo == n) lo = n - 1;
    return lo + 1;
}

__global__ void __launch_bounds__(kTraceWarpsPerBlock * 32)
    trace_gen_kernel(const TraceJob* __restrict__ jobs, int n_jobs, int variant) {
    __shared__ uint64_t s_mt[kTraceWarpsPerBlock][MSV_MT_N];
    __shared__ double s_gap[kTraceWarpsPerBlock][MSV_MT_M];
    __shared__ double s_arr[kTraceWarpsPerBlock][MSV_MT_M];
    __shared__ int32_t s_bat[kTraceWarpsPerBlock][MSV_MT_M];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int job = blockIdx.x * kTraceWarpsPerBlock + warp;
    if (job >= n_jobs) return;
    const TraceJob J = jobs[job];
    uint64_t* mt = s_mt[warp];
    double* gap = s_gap[warp];
    double* arr = s_arr[warp];
    int32_t* bat = s_bat[warp];

    // mt19937_64(seed): x[0] = seed; x[i] = f*(x[i-1] ^ (x[i-1] >> 62)) + i.
    if (lane == 0) {
        uint64_t x = J.seed;
        mt[0] = x;
        for (uint32_t i = 1; i < MSV_MT_N; ++i) {
            x = msv_mt_next_seed(x, i);
            mt[i] = x;
        }
    }
    __syncwarp();

    double t = 0.0;  // meaningful in lane 0 only
    int64_t n = 0;
    bool first = true, stop = false;
    while (!stop) {
        // Regenerate the 312-word block. Words [0,156) read only old words;
        // words [156,312) read new[i-156] (and word 311 reads new[0]). Within a
        // pass every lane reads before any lane writes.
        for (int base = 0; base < MSV_MT_M; base += 32) {
            const int i = base + lane;
            uint64_t v = 0;
            if (i < MSV_MT_M) v = msv_mt_twist(mt[i], mt[i + 1], mt[i + MSV_MT_M]);
            __syncwarp();
            if (i < MSV_MT_M) mt[i] = v;
            __syncwarp();
        }
        for (int base = MSV_MT_M; base < MSV_MT_N; base += 32) {
            const int i = base + lane;
            uint64_t v = 0;
            if (i < MSV_MT_N) v = msv_mt_twist(mt[i], mt[(i + 1 == MSV_MT_N) ? 0 : i + 1], mt[i - MSV_MT_M]);
            __syncwarp();
            if (i < MSV_MT_N) mt[i] = v;
            __syncwarp();
        }
        // Draw order (workload.hpp:104-111): gap_0, then (batch_p, gap_{p+1}) —
        // i.e. word 2p is query p's gap, word 2p+1 its batch.
        for (int p = lane; p < MSV_MT_M; p += 32) {
            const double ug = msv_uniform(msv_mt_temper(mt[2 * p]));
            gap[p] = -msv_log1p_neg(-ug, variant) / J.rate_per_ms;  // rng.hpp:20
            const double ub = msv_uniform(msv_mt_temper(mt[2 * p + 1]));
            bat[p] = cdf_sample(J.cdf, J.b_max, ub);
        }
        __syncwarp();
        // Sequential arrival accumulation, exactly `t += gap` (workload.hpp:111).
        int cnt = 0;
        if (lane == 0) {
            for (int p = 0; p < MSV_MT_M; ++p) {
                const double g = gap[p];
                t = first ? g : t + g;
                first = false;
                if (!(t < J.duration_ms)) {
                    stop = true;
                    break;
                }
                arr[p] = t;
                ++cnt;
            }
        }
        cnt = __shfl_sync(kFull, cnt, 0);
        stop = __shfl_sync(kFull, stop, 0);
        for (int p = lane; p < cnt; p += 32) {
            const int64_t idx = n + p;
            if (idx < J.cap) {
                J.arrival[idx] = arr[p];
                J.batch[idx] = bat[p];
            }
        }
        n += cnt;
        if (n > J.cap) stop = true;
        __syncwarp();
    }
    if (lane == 0) {
        *J.n_out = (n > J.cap) ? J.cap : n;
        *J.overflow = (n > J.cap) ? 1 : 0;
    }
}

// ---------------------------------------------------------------------------
// K2: simulation
// ---------------------------------------------------------------------------

template <int W>
__device__ __forceinline__ uint64_t seg_min_u64(uint64_t v) {
#pragma unroll
    for (int off = W / 2; off > 0; off >>= 1) {
        const uint64_t o = __shfl_xor_sync(kFull, v, off);
        v = o < v ? o : v;
    }
    return v;
}

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

// Segment-masked reductions for the (segment-uniform) finalisation branch.
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

constexpr uint64_t kQidMask = (1ull << 40) - 1;
constexpr uint64_t kSignBit = 1ull << 63;

// Order-preserving map of IEEE doubles onto uint64 (total order of finite values).
__device__ __forceinline__ uint64_t order_key(uint64_t b) { return (b & kSignBit) ? ~b : (b | kSignBit); }
__device__ __forceinline__ uint64_t order_unkey(uint64_t k) { return (k & kSignBit) ? (k & ~kSignBit) : ~k; }

// One warp = 32/W scenario segments of W lanes. Lane slot s of segment lane l
// holds the partition of by_ascending_size order index o = s*W + l, so warp
// ballots enumerate candidates in ELSA's scan order (sched.hpp:123-125).
template <int W, int S, int SCHED, bool REC>
__global__ void __launch_bounds__(kSimWarpsPerBlock * 32) sim_kernel(const SimParams p) {
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
    const unsigned lt_mask = (1u << lane) - 1u;

    // ---- segment state (identical in all lanes of a segment) ----
    int32_t sidx = -1;
    bool done = false;
    int64_t n = 0, i = 0, win_base = 0, smp = 0;
    double win_t = 0.0, nxt_t = 0.0;
    int32_t win_b = 0, nxt_b = 0;
    double duration = 0.0, warmup = 0.0, sla = 0.0, alpha = 0.0, beta = 0.0;
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
    int64_t nq[S];
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
    int64_t viol = 0, meas = 0, mviol = 0;
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
                smp = 0;
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
                viol = meas = mviol = 0;
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
            } else {
                t = INFINITY;  // drain everything (no horizon cut-off)
                ending = true;
            }
        }

        // ---- completions with time <= t, per partition, in chain order ----
        // (completions precede an arrival at equal time, engine.hpp:101-107;
        //  completions on different partitions commute.)
        while (true) {
            bool f[S];
            bool any = false;
#pragma unroll
            for (int s = 0; s < S; ++s) {
                f[s] = busy[s] && c_comp[s] <= t;
                any |= f[s];
            }
            if (!__any_sync(kFull, any)) break;
#pragma unroll
            for (int s = 0; s < S; ++s) {
                const bool m = f[s] && (c_arr[s] >= warmup);  // engine.hpp:262
                const unsigned bal = __ballot_sync(kFull, m) & seg_mask;
                const int64_t pos = smp + __popc(bal & lt_mask);
                smp += __popc(bal);
                if (f[s]) {
                    // completion (engine.hpp:167-187)
                    const double now = c_comp[s];
                    const double lat = now - c_arr[s];
                    const bool met = lat <= sla;
                    const double ran = now - c_start[s];
                    bms[s] = bms[s] + ran;
                    wbms[s] = wbms[s] + ran * c_util[s];
                    nq[s] += 1;
                    last_fin = (last_fin < now) ? now : last_fin;
                    if (!met) ++viol;
                    if (m) {
                        ++meas;
                        if (!met) ++mviol;
                        samples[pos] = lat;
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
        }

        // ---- dispatch (engine.hpp:189-230) ----
        if (arrival && (b < 1 || b > bmax)) {  // LookupError at this query (profile.hpp:127-129)
            status = MSV_LOOKUP;
            i = n;
            arrival = false;
        }
        double est_n[S], wv[S];
        bool cand[S];
#pragma unroll
        for (int s = 0; s < S; ++s) {
            est_n[s] = 0.0;
            wv[s] = 0.0;
            cand[s] = false;
            if (arrival && act[s]) {
                est_n[s] = row[s] >= 0 ? s_lat[row[s] + b - 1] : 0.0;
                cand[s] = routed ? (((rmask[s] >> (b - 1)) & 1ull) != 0) : true;
            }
        }
        {  // segment routing falls back to every partition (engine.hpp:197-206)
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
        for (int s = 0; s < S; ++s) {
            bad[s] = cand[s] && row[s] < 0;
            const unsigned bb = __ballot_sync(kFull, bad[s]) & seg_mask;
            if (bad_lane < 0 && bb != 0) {
                bad_lane = __ffs(bb) - 1;
                bad_slot = s;
            }
        }
        const bool need_w = (SCHED == MSV_ELSA) || (flags & MSV_FLAG_CHECK_WAIT);
        if (need_w) {
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
                if (flags & MSV_FLAG_CHECK_WAIT) {  // engine.hpp:208-217
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
                const bool pred = cand[s] && !bad[s] && (sla > alpha * (wv[s] + beta * est_n[s]));
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
            uint32_t ki[S], kq[S];
            uint32_t mi = ~0u, mq = ~0u;
#pragma unroll
            for (int s = 0; s < S; ++s) {
                ki[s] = (cand[s] && !busy[s]) ? (((0x7FFFu - (uint32_t)kk[s]) << 16) | (uint32_t)pid[s]) : ~0u;
                const uint32_t len = (uint32_t)qn[s] + gn[s];
                kq[s] = cand[s] ? (((len < 0xFFFFFFu ? len : 0xFFFFFFu) << 8) | (uint32_t)pid[s]) : ~0u;
                mi = ki[s] < mi ? ki[s] : mi;
                mq = kq[s] < mq ? kq[s] : mq;
            }
            mi = seg_min_u32<W>(mi);
            mq = seg_min_u32<W>(mq);
            const bool idle = mi != ~0u;
#pragma unroll
            for (int s = 0; s < S; ++s) {
                const unsigned bI = __ballot_sync(kFull, ki[s] == mi && mi != ~0u) & seg_mask;
                const unsigned bQ = __ballot_sync(kFull, kq[s] == mq && mq != ~0u) & seg_mask;
                const unsigned bsel = idle ? bI : bQ;
                if (arrival && ch_lane < 0 && bsel != 0) {
                    ch_lane = __ffs(bsel) - 1;
                    ch_slot = s;
                    kind = idle ? MSV_IDLE_LARGEST : MSV_SHORTEST_QUEUE;
                }
            }
        }

        if (arrival && bad_lane >= 0) {
            bool err;
            if constexpr (SCHED == MSV_ELSA) {  // scan reached the bad partition first
                err = ch_lane < 0 || kind == MSV_FASTEST_FALLBACK || bad_slot < ch_slot ||
                      (bad_slot == ch_slot && bad_lane < ch_lane);
            } else {
                err = bad_lane == ch_lane && bad_slot == ch_slot;
                if (!err) {  // another bad partition may be the chosen one
#pragma unroll
                    for (int s = 0; s < S; ++s) {
                        const unsigned bb = __ballot_sync(seg_mask, bad[s]) & seg_mask;
                        if (s == ch_slot && ((bb >> ch_lane) & 1u)) err = true;
                    }
                }
            }
            if (err) {
                status = MSV_LOOKUP;
                i = n;
                arrival = false;
            }
        }
        // ---- enqueue on the chosen partition (engine.hpp:225-230) ----
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
            int64_t v0 = seg_sum_u64<W>((uint64_t)viol, seg_mask);
            int64_t v1 = seg_sum_u64<W>((uint64_t)meas, seg_mask);
            int64_t v2 = seg_sum_u64<W>((uint64_t)mviol, seg_mask);
            const uint64_t hsum = seg_sum_u64<W>(hash, seg_mask);
            const double lf = seg_max_f64<W>(last_fin, seg_mask);
            const double wd = seg_max_f64<W>(wdiff, seg_mask);
            const uint64_t mn = seg_minm_u64<W>(lmin, seg_mask);
            const uint64_t mx = seg_max_u64<W>(lmax, seg_mask);
            if (sl == 0) {
                DevOut o;
                o.violations = v0;
                o.measured = v1;
                o.measured_violations = v2;
                o.n_samples = smp;
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

// ---------------------------------------------------------------------------
// K3: exact nearest-rank tails
// ---------------------------------------------------------------------------

__device__ void bitonic_sort_smem(uint64_t* buf, int n_pow2) {
    for (int k = 2; k <= n_pow2; k <<= 1) {
        for (int j = k >> 1; j > 0; j >>= 1) {
            for (int idx = threadIdx.x; idx < n_pow2; idx += blockDim.x) {
                const int ixj = idx ^ j;
                if (ixj > idx) {
                    const uint64_t a = buf[idx], c = buf[ixj];
                    const bool up = (idx & k) == 0;
                    if ((a > c) == up) {
                        buf[idx] = c;
                        buf[ixj] = a;
                    }
                }
            }
            __syncthreads();
        }
    }
}

__global__ void __launch_bounds__(kTailThreads)
    tail_kernel(const TailJob* __restrict__ jobs, int n_jobs, const double* __restrict__ ps, int n_p) {
    __shared__ unsigned int hist[2048];
    __shared__ uint64_t buf[kTailSmemCap];
    __shared__ long long s_r;
    __shared__ unsigned long long s_prefix, s_min, s_max;
    __shared__ unsigned int s_cnt;
    __shared__ unsigned int s_pos;
    for (int jb = blockIdx.x; jb < n_jobs; jb += gridDim.x) {
        const TailJob J = jobs[jb];
        const DevOut src = *J.src;
        const long long Jn = src.n_samples;
        uint64_t kmin = src.lat_min_bits, kmax = src.lat_max_bits;  // order keys
        if (Jn > 0 && kmin > kmax) {  // not supplied: one reduction pass
            if (threadIdx.x == 0) {
                s_min = ~0ull;
                s_max = 0;
            }
            __syncthreads();
            uint64_t lo = ~0ull, hi = 0;
            for (long long idx = threadIdx.x; idx < Jn; idx += blockDim.x) {
                const uint64_t v = order_key(msv_dbits(J.samples[idx]));
                lo = v < lo ? v : lo;
                hi = v > hi ? v : hi;
            }
            atomicMin(&s_min, (unsigned long long)lo);
            atomicMax(&s_max, (unsigned long long)hi);
            __syncthreads();
            kmin = s_min;
            kmax = s_max;
            __syncthreads();
        }
        for (int q = 0; q < n_p; ++q) {
            if (Jn == 0) {
                if (threadIdx.x == 0) J.out[q] = __longlong_as_double(0x7ff8000000000000ll);
                continue;
            }
            // metrics.hpp:26-28: rank = ceil(p * n), at least 1.
            long long r = (long long)ceil(ps[q] * (double)Jn);
            if (r < 1) r = 1;
            uint64_t answer;
            if (kmin == kmax) {
                answer = kmin;
            } else {
                // MSB-first radix select over order keys, 11 bits per pass, starting
                // at the highest bit where min and max differ.
                int pos = 64 - __clzll((long long)(kmin ^ kmax));  // unknown low bits
                uint64_t prefix = (pos == 64) ? 0ull : (kmin >> pos);
                while (true) {
                    const int d = pos < 11 ? pos : 11;
                    const int shift = pos - d;
                    const int nb = 1 << d;
                    for (int k = threadIdx.x; k < nb; k += blockDim.x) hist[k] = 0;
                    __syncthreads();
                    for (long long idx = threadIdx.x; idx < Jn; idx += blockDim.x) {
                        const uint64_t v = order_key(msv_dbits(J.samples[idx]));
                        if (pos == 64 || (v >> pos) == prefix) atomicAdd(&hist[(v >> shift) & (uint64_t)(nb - 1)], 1u);
                    }
                    __syncthreads();
                    if (threadIdx.x == 0) {
                        long long cum = 0;
                        int jbin = 0;
                        for (; jbin < nb; ++jbin) {
                            if (cum + hist[jbin] >= r) break;
                            cum += hist[jbin];
                        }
                        s_r = r - cum;
                        s_prefix = ((pos == 64) ? 0ull : (prefix << d)) | (uint64_t)jbin;
                        s_cnt = hist[jbin];
                    }
                    __syncthreads();
                    r = s_r;
                    prefix = s_prefix;
                    pos = shift;
                    const unsigned cnt = s_cnt;
                    __syncthreads();
                    if (pos == 0) {
                        answer = prefix;
                        break;
                    }
                    if (cnt <= (unsigned)kTailSmemCap) {
                        if (threadIdx.x == 0) s_pos = 0;
                        __syncthreads();
                        for (long long idx = threadIdx.x; idx < Jn; idx += blockDim.x) {
                            const uint64_t v = order_key(msv_dbits(J.samples[idx]));
                            if ((v >> pos) == prefix) buf[atomicAdd(&s_pos, 1u)] = v;
                        }
                        __syncthreads();
                        int np2 = 1;
                        while (np2 < (int)cnt) np2 <<= 1;
                        for (int k = cnt + threadIdx.x; k < np2; k += blockDim.x) buf[k] = ~0ull;
                        __syncthreads();
                        bitonic_sort_smem(buf, np2);
                        answer = buf[r - 1];
                        __syncthreads();
                        break;
                    }
                }
            }
            if (threadIdx.x == 0) J.out[q] = msv_bitsd(order_unkey(answer));
            __syncthreads();
        }
    }
}

// ---------------------------------------------------------------------------
// Single dispatch decisions (sched.hpp:77-174), one thread per trial.
// ---------------------------------------------------------------------------

constexpr int kMaxDispatchParts = 128;

__global__ void dispatch_kernel(const DispatchParams p) {
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= p.n_trials) return;
    const int64_t o0 = p.part_off[t];
    const int P = (int)(p.part_off[t + 1] - o0);
    const double now = p.now_ms[t];
    const int qb = p.query_batch[t];
    p.error[t] = 0;
    p.chosen[t] = -1;
    p.kind[t] = 0;
    if (P <= 0 || P > kMaxDispatchParts) {
        p.error[t] = MSV_PARAM;
        return;
    }
    // ProfileTable::latency_ms with its LookupError cases (profile.hpp:123-132).
    auto cell_ok = [&](int32_t row, int32_t batch) { return row >= 0 && batch >= 1 && batch <= p.b_max; };
    // t_wait per partition (sched.hpp:77-85)
    auto t_wait = [&](int j, bool* ok) -> double {
        const int32_t row = p.part_row[o0 + j];
        double w = 0.0;
        for (int64_t q = p.q_off[o0 + j]; q < p.q_off[o0 + j + 1]; ++q) {
            const int32_t bb = p.qbatch[q];
            if (!cell_ok(row, bb)) {
                *ok = false;
                return 0.0;
            }
            w = w + p.lat[row + bb - 1];
        }
        if (p.busy[o0 + j]) {
            const double elapsed = now - p.cur_start[o0 + j];
            const double x = p.cur_est[o0 + j] - elapsed;
            w = w + ((0.0 < x) ? x : 0.0);
        }
        return w;
    };
    if (p.t_wait_out) {
        for (int j = 0; j < P; ++j) {
            bool ok = true;
            const double w = t_wait(j, &ok);
            p.t_wait_out[o0 + j] = ok ? w : __longlong_as_double(0x7ff8000000000000ll);
        }
    }
    if (p.scheduler == MSV_FIFS) {
        int idle = -1;
        for (int j = 0; j < P; ++j) {
            if (p.busy[o0 + j]) continue;
            if (idle < 0 || p.part_k[o0 + j] > p.part_k[o0 + idle] ||
                (p.part_k[o0 + j] == p.part_k[o0 + idle] && p.part_id[o0 + j] < p.part_id[o0 + idle]))
                idle = j;
        }
        if (idle >= 0) {
            p.chosen[t] = p.part_id[o0 + idle];
            p.kind[t] = MSV_IDLE_LARGEST;
            return;
        }
        int best = 0;
        for (int j = 0; j < P; ++j) {
            const int64_t lj = p.q_off[o0 + j + 1] - p.q_off[o0 + j];
            const int64_t lb = p.q_off[o0 + best + 1] - p.q_off[o0 + best];
            if (lj < lb || (lj == lb && p.part_id[o0 + j] < p.part_id[o0 + best])) best = j;
        }
        p.chosen[t] = p.part_id[o0 + best];
        p.kind[t] = MSV_SHORTEST_QUEUE;
        return;
    }
    // ELSA: by_ascending_size order (sched.hpp:96-104), insertion sort of indices.
    int order[kMaxDispatchParts];
    for (int j = 0; j < P; ++j) {
        int x = j, m = j;
        while (m > 0) {
            const int y = order[m - 1];
            const bool less = (p.part_k[o0 + x] != p.part_k[o0 + y]) ? (p.part_k[o0 + x] < p.part_k[o0 + y])
                                                                       : (p.part_id[o0 + x] < p.part_id[o0 + y]);
            if (!less) break;
            order[m] = y;
            --m;
        }
        order[m] = x;
    }
    const double sla = p.sla_ms[t], alpha = p.alpha[t], beta = p.beta[t];
    for (int oi = 0; oi < P; ++oi) {
        const int j = order[oi];
        const int32_t row = p.part_row[o0 + j];
        if (!cell_ok(row, qb)) {  // first Step-A lookup throws (sched.hpp:127)
            p.error[t] = MSV_LOOKUP;
            return;
        }
        const double est = p.lat[row + qb - 1];
        bool ok = true;
        const double w = t_wait(j, &ok);
        if (!ok) {
            p.error[t] = MSV_LOOKUP;
            return;
        }
        if (sla > alpha * (w + beta * est)) {
            p.chosen[t] = p.part_id[o0 + j];
            p.kind[t] = MSV_SLACK_SATISFYING;
            return;
        }
    }
    double best_time = INFINITY;
    int best = order[0];
    for (int oi = 0; oi < P; ++oi) {
        const int j = order[oi];
        bool ok = true;
        const double fin = t_wait(j, &ok) + p.lat[p.part_row[o0 + j] + qb - 1];
        if (fin < best_time) {
            best_time = fin;
            best = j;
        }
    }
    p.chosen[t] = p.part_id[o0 + best];
    p.kind[t] = MSV_FASTEST_FALLBACK;
}

}  // namespace

// ---------------------------------------------------------------------------
// launchers
// ---------------------------------------------------------------------------

cudaError_t launch_trace_gen(const TraceJob* d_jobs, int n_jobs, int log1p_variant,
                             cudaStream_t stream) {
    if (n_jobs <= 0) return cudaSuccess;
    const int blocks = (n_jobs + kTraceWarpsPerBlock - 1) / kTraceWarpsPerBlock;
    trace_gen_kernel<<<blocks, kTraceWarpsPerBlock * 32, 0, stream>>>(d_jobs, n_jobs, log1p_variant);
    return cudaGetLastError();
}

size_t sim_smem_bytes(int S, int n_cells) {
    const size_t tab = ((size_t)2 * n_cells * sizeof(double) + 15) & ~(size_t)15;
    return tab + (size_t)kSimWarpsPerBlock * 3 * S * kQCap * 32 * sizeof(double);
}

namespace {
template <int W, int S, int SCHED, bool REC>
void* sim_fn() {
    return reinterpret_cast<void*>(&sim_kernel<W, S, SCHED, REC>);
}

void* pick_sim(int W, int S, int sched, bool rec) {
#define MSV_PICK(w, s)                                                                            \
    if (W == w && S == s) {                                                                       \
        if (sched == MSV_ELSA) return rec ? sim_fn<w, s, MSV_ELSA, true>() : sim_fn<w, s, MSV_ELSA, false>(); \
        return rec ? sim_fn<w, s, MSV_FIFS, true>() : sim_fn<w, s, MSV_FIFS, false>();             \
    }
    MSV_PICK(4, 1)
    MSV_PICK(8, 1)
    MSV_PICK(16, 1)
    MSV_PICK(32, 1)
    MSV_PICK(32, 2)
    MSV_PICK(32, 4)
#undef MSV_PICK
    return nullptr;
}
}  // namespace

int sim_max_blocks_per_sm(int W, int S, int sched, bool records, int n_cells) {
    void* fn = pick_sim(W, S, sched, records);
    if (!fn) return 0;
    const size_t smem = sim_smem_bytes(S, n_cells);
    if (cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
        return 0;
    int blocks = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks, fn, kSimWarpsPerBlock * 32, smem) != cudaSuccess)
        return 0;
    return blocks;
}

cudaError_t launch_sim(int W, int S, int sched, bool records, const SimParams& p, int blocks,
                       cudaStream_t stream) {
    void* fn = pick_sim(W, S, sched, records);
    if (!fn) return cudaErrorInvalidValue;
    const size_t smem = sim_smem_bytes(S, p.n_cells);
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    void* args[] = {const_cast<SimParams*>(&p)};
    return cudaLaunchKernel(fn, dim3(blocks), dim3(kSimWarpsPerBlock * 32), args, smem, stream);
}

cudaError_t launch_tail(const TailJob* d_jobs, int n_jobs, const double* d_p, int n_p,
                        cudaStream_t stream) {
    if (n_jobs <= 0) return cudaSuccess;
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int blocks = n_jobs < sms * 4 ? n_jobs : sms * 4;
    tail_kernel<<<blocks, kTailThreads, 0, stream>>>(d_jobs, n_jobs, d_p, n_p);
    return cudaGetLastError();
}

cudaError_t launch_dispatch(const DispatchParams& p, cudaStream_t stream) {
    if (p.n_trials <= 0) return cudaSuccess;
    const int threads = 128;
    const int blocks = (int)((p.n_trials + threads - 1) / threads);
    dispatch_kernel<<<blocks, threads, 0, stream>>>(p);
    return cudaGetLastError();
}

}  // namespace msv
