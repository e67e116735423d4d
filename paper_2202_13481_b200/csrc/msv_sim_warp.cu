// K2 sim_warp_kernel: run() (engine.hpp:115-253) with ELSA (sched.hpp:119-143) or FIFS
// (sched.hpp:154-170), one scenario per warp, for plans of up to 32*S partitions (S = 1,
// 2, 4 slots per lane; lane slot s of lane l owns by_ascending_size order index s*32 + l,
// sched.hpp:96-104). The per-arrival protocol is msv_sim.cu's (see its header); this
// kernel adds the warp-uniform structure one scenario per warp allows:
//   * scenario -> 32-arrival window (staged in shared memory) -> arrival loop; the
//     window's first measured arrival is one ballot;
//   * the batch's latency row is loaded ahead of the drain; the drain is lane-local;
//   * Step A = ballot; with one slot the chosen lane is the one with no set ballot bit
//     below it (no bit scan on the critical path); with several slots the slots are
//     scanned in order and later slots' waits are computed only when needed;
//     Step B's 64-bit argmin = two REDUX.MIN + ballot; FIFS = REDUX.MIN over (k, id) /
//     (queue length, id) keys;
//   * the FIFO fold of Eq. 1 is exact: extended on append, recomputed from the queue
//     head when the head leaves (ELSA); the LAZY instantiation (scenarios offered more
//     than the plan's capacity) bounds long queues' folds with a double-double sum and
//     refolds only when a decision needs the exact value;
//   * template flags: UNIT (alpha = beta = 1, per scenario: 1*x == x bit for bit), FULL
//     (segment routing / missing sizes / wait check / usage / records in the launch; the
//     plain variant carries none of that work), REC (per-query records), LAZY;
//   * completion bookkeeping happens when a query is PLACED, not when it completes:
//     with noise off a placed query's start is known at once (the arrival if the
//     partition is idle, else the finish of the query queued last) and so is its
//     finish = start + est (engine.hpp:181-185, :225-230 — the same RN add the
//     completion event would perform). The chosen lane writes (start, finish, partition,
//     kind) of arrival j into the window's shared row; when the 32-arrival window is
//     done, lane j retires query base + j — latency, SLA violation, measured sample,
//     placement digest, per-query record — all 32 lanes at once, coalesced. The lane-
//     local drain before each arrival only pops queue heads (start = previous finish)
//     to keep Eq. 1 exact; nothing is drained after the last arrival;
//   * per-partition usage (PartitionUsage, FULL) is summed at placement, which is the
//     partition's completion order (its FIFO order);
//   * measured latencies overwrite the arrivals of their own queries (DevScen.samples
//     == the arrival buffer): a query's arrival is dead once its window is retired;
//   * the horizon is the last finish each slot placed.
#include <type_traits>

#include "msv_device.cuh"

namespace msv {

namespace {


template <int S>
struct WarpCfg {
    static constexpr int qcap = S == 1 ? 16 : (S == 2 ? 8 : 4);  // shared ring entries per slot
    static constexpr int min_blocks = S == 1 ? 7 : (S == 2 ? 5 : 2);
};

// Per-warp shared-memory layout (after the block's profile table).
template <int S>
struct WarpSmem {
    static constexpr int QC = WarpCfg<S>::qcap;
    double q_est[S][QC][32];  // queued latencies (ring; starts/finishes follow from them)
    // window arrival j: (arrival, batch) staged by lane j, read by every lane with one
    // 16-byte load; (start, finish) written by the chosen lane with one 16-byte store
    double2 win_tb[32];  // {arrival, batch bits}
    double2 win_sf[32];  // {start, finish}
    int32_t win_p[32];   // partition id | kind << 8
    uint32_t g_head[S][32];  // overflow list head / tail per lane slot
    uint32_t g_tail[S][32];
    double dd_hi[S][32];     // overflow mode: double-double sum of the queued latencies
    double dd_lo[S][32];
};

// Error-free sum (Knuth two-sum) and a double-double accumulator (RN, no contraction).
__device__ __forceinline__ void dd_add(double& hi, double& lo, double x) {
    const double s = hi + x;
    const double bp = s - hi;
    const double e = (hi - (s - bp)) + (x - bp);
    const double t = lo + e;
    hi = s + t;
    lo = t - (hi - s);
}

template <int S, int SCHED, bool REC, bool FULL, bool LAZY>
__global__ void __launch_bounds__(kSimWarpsPerBlock * 32, WarpCfg<S>::min_blocks)
    sim_warp_kernel(const SimParams p) {
    constexpr int QC = WarpCfg<S>::qcap;
    constexpr bool kFold = (SCHED == MSV_ELSA) || FULL;  // Eq. 1 needed (ELSA, or the check)
    // Plain ELSA keeps long queues' folds lazily: while a slot's FIFO spills into the
    // overflow list, a pop no longer refolds the queue (O(queue)); the slot keeps a
    // double-double sum of its queued latencies instead, which bounds the left fold to
    // +-(n+4)*2^-52 relative, and the exact fold is recomputed only when a decision
    // cannot be settled from the bounds (an overloaded scenario becomes O(1) per arrival).
    // (A separate instantiation, chosen by the host for scenarios offered more than the
    // plan's nominal capacity: the extra paths cost the plain kernel registers.)
    constexpr bool kLazy = LAZY && (SCHED == MSV_ELSA) && !FULL;
    constexpr int32_t kFv = 1 << 30;  // pk bit: fold[s] holds the exact left fold
    constexpr int kLazyMin = 48;      // queues up to this length are refolded eagerly
    extern __shared__ __align__(16) unsigned char smem[];
    double* s_lat = reinterpret_cast<double*>(smem);
    double* s_util = s_lat + p.n_cells;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const size_t tab_bytes = ((size_t)2 * p.n_cells * sizeof(double) + 15) & ~(size_t)15;
    WarpSmem<S>& W = reinterpret_cast<WarpSmem<S>*>(smem + tab_bytes)[warp];
    for (int c = threadIdx.x; c < p.n_cells; c += blockDim.x) {
        s_lat[c] = p.lat[c];
        s_util[c] = p.util[c];
    }
    __syncthreads();
    // 32-bit shared address of the latency cells, kept in a register: the per-arrival
    // lookup must not re-derive the shared window base (S2UR) on its critical path
    const uint32_t lat_sh = opaque(smem_addr(s_lat));

    for (;;) {
        int w = 0;
        if (lane == 0) w = atomicAdd(p.counter, 1);
        w = __shfl_sync(kFull, w, 0);
        if (w >= p.n_work) break;
        const int sidx = p.work[w];
        const DevScen& d = p.scen[sidx];
        const int n = (int)*d.n;
        const double* __restrict__ g_arr = d.arrival;
        const int32_t* __restrict__ g_bat = d.batch;
        uint32_t* g_next = d.next;
        uint32_t* samples = reinterpret_cast<uint32_t*>(d.samples);  // planar layout (msv_internal.h)
        msv_record* rec = d.records;
        const double sla = d.sla, warmup = d.warmup_ms;
        const double sla_act = lane < d.P ? sla : -INFINITY;  // Step A's bound, false on lanes without a partition
        const bool check_wait = FULL && p.any_check_wait && (d.flags & MSV_FLAG_CHECK_WAIT);
        const int bmax = d.b_max;
        const uint64_t* route_mask = d.route_mask;
        // global-space accesses (LDG/STG) instead of generic ones on the per-query paths
        __builtin_assume(__isGlobal(g_arr));
        __builtin_assume(__isGlobal(g_bat));
        __builtin_assume(__isGlobal(g_next));
        __builtin_assume(__isGlobal(samples));
        if (REC) __builtin_assume(__isGlobal(rec));
        if (FULL && route_mask) __builtin_assume(__isGlobal(route_mask));

        // ---- lane slots ----
        // c_* = the query placed last to start on the slot; tail = finish of the query
        // placed last (== c_comp while the FIFO is empty): the start of the next one
        // queued. The slot is busy at time t iff c_comp > t (after the drain below, a
        // finished query has nothing queued behind it): no busy flag is kept, and an idle
        // slot keeps its last query's (finished) values, c_comp = -inf before the first.
        bool act[S];
        int32_t row[S], pk[S], qh[S], qn[S];  // pk = partition id | k << 8
        uint32_t gn[S], nq[S];
        double c_start[S], c_est[S], c_comp[S], tail[S], fold[S], bms[S], wbms[S];
        uint32_t row_sh[S];  // shared address of the slot's latency row, minus one cell: + b*8 = L(k, b)
#pragma unroll
        for (int s = 0; s < S; ++s) {
            const int o = s * 32 + lane;
            act[s] = o < d.P;
            row[s] = 0;  // inactive lanes read a valid (ignored) cell
            pk[s] = 0;
            if (act[s]) {
                const DevPart dp = d.parts[o];
                pk[s] = dp.pid | (dp.k << 8);
                row[s] = dp.row;
            }
            qh[s] = qn[s] = 0;
            gn[s] = nq[s] = 0;
            c_start[s] = c_est[s] = 0.0;
            c_comp[s] = -INFINITY;
            tail[s] = 0.0;
            row_sh[s] = lat_sh + (uint32_t)(row[s] - 1) * 8u;
            fold[s] = 0.0;
            bms[s] = wbms[s] = 0.0;
        }
        uint32_t viol = 0, mviol = 0;
        uint64_t hash = 0;
        double wdiff = 0.0;
        int m0 = -1, status = 0;

        // Exact left fold of slot s's FIFO (sched.hpp:78-79): ring part, then overflow list.
        auto refold = [&](int s) {
            if (qn[s] == 0) return 0.0;  // (an overflow list implies a full ring)
            double acc = W.q_est[s][qh[s]][lane];  // 0.0 + e == e exactly (e > 0)
#pragma unroll 1
            for (int k = 1; k < qn[s]; ++k) acc = acc + W.q_est[s][(qh[s] + k) & (QC - 1)][lane];
            if (gn[s] > 0) {
                uint32_t g = W.g_head[s][lane];
#pragma unroll 1
                for (uint32_t k = 0; k < gn[s]; ++k) {
                    acc = acc + s_lat[row[s] + g_bat[g] - 1];
                    g = g_next[g];
                }
            }
            return acc;
        };

        // Advance this lane's partitions to time t: every running query with finish <= t
        // has completed (a completion precedes an arrival at equal time, engine.hpp:101-107)
        // and the queue head starts at its finish (engine.hpp:181-185). The completions'
        // bookkeeping was done when the queries were placed; only Eq. 1's state moves.
        // Plain multi-slot ELSA advances slot 0 before every arrival and a later slot only
        // when Step A reaches it (or Step B needs it): a slot's state is needed only then,
        // and advancing it later to a later time retires the same completions in the same
        // order (each slot's chain is independent of the others).
        constexpr int kEager = (SCHED == MSV_ELSA && S > 1 && !FULL && !kLazy) ? 1 : S;
        auto drain = [&](double t, int s_lo, int s_hi) {
#pragma unroll
            for (int s = 0; s < S; ++s) {
                if (s < s_lo || s >= s_hi) continue;
                // pops: the queue head starts at the running query's finish
                while (c_comp[s] <= t && qn[s] > 0) {
                    const int h = qh[s];
                    const double est = W.q_est[s][h][lane];
                    qh[s] = (h + 1) & (QC - 1);
                    qn[s] -= 1;
                    c_start[s] = c_comp[s];
                    c_est[s] = est;
                    c_comp[s] = c_start[s] + est;  // the placement computed the same sum
                    if (gn[s] == 0) {
                        if (kFold) {  // the queue fits the ring: exact left fold from 0.0 (0 + e == e)
                            double acc = 0.0;
#pragma unroll 1
                            for (int k = 0; k < qn[s]; ++k) acc = acc + W.q_est[s][(qh[s] + k) & (QC - 1)][lane];
                            fold[s] = acc;
                        }
                    } else {  // spilled: refill the ring from the overflow list
                        const uint32_t g = W.g_head[s][lane];
                        W.g_head[s][lane] = g_next[g];
                        gn[s] -= 1;
                        W.q_est[s][(qh[s] + qn[s]) & (QC - 1)][lane] = s_lat[row[s] + g_bat[g] - 1];
                        qn[s] += 1;
                        if (kLazy && gn[s] > 0) {  // still spilled: drop the head from the sum
                            double hi = W.dd_hi[s][lane], lo = W.dd_lo[s][lane];
                            dd_add(hi, lo, -est);
                            W.dd_hi[s][lane] = hi;
                            W.dd_lo[s][lane] = lo;
                            if (qn[s] + (int)gn[s] > kLazyMin) {
                                pk[s] &= ~kFv;  // long queue: the fold is stale until a decision needs it
                            } else {
                                fold[s] = refold(s);  // short spill: refolding is cheap
                                pk[s] |= kFv;
                            }
                        } else if (kFold) {
                            fold[s] = refold(s);
                        }
                    }
                }
                // (a finished query with nothing queued behind it leaves the slot idle:
                // c_comp <= t, and the fold of the empty queue is already 0)
            }
        };

        // One scenario's arrival stream; UNIT: alpha == beta == 1.
        auto simulate = [&](auto unit_tag) {
            constexpr bool UNIT = decltype(unit_tag)::value;
            const double alpha = d.alpha, beta = d.beta;
            double nx_t = lane < n ? g_arr[lane] : 0.0;
            int nx_b = lane < n ? g_bat[lane] : 0;
            for (int base = 0; base < n; base += 32) {
                const double cur_t = nx_t;
                __syncwarp();
                W.win_tb[lane] = make_double2(cur_t, __longlong_as_double((long long)nx_b));
                __syncwarp();
                if (base + 32 + lane < n) {  // prefetch the next window
                    nx_t = g_arr[base + 32 + lane];
                    nx_b = g_bat[base + 32 + lane];
                }
                if (m0 < 0) {  // first arrival >= warmup (arrivals are sorted; engine.hpp:262)
                    const unsigned mb = __ballot_sync(kFull, base + lane < n && cur_t >= warmup);
                    if (mb) m0 = base + __ffs(mb) - 1;
                }
                const int cnt = min(32, n - base);
                for (int j = 0; j < cnt; ++j) {
                    const double2 tb = W.win_tb[j];
                    const double t = tb.x;
                    const int b = (int)__double_as_longlong(tb.y);
                    const int i = base + j;
                    // The new query's latency on each partition depends on its batch only:
                    // load it ahead of the drain (FULL: batch clamped into the table for
                    // the load, missing sizes read 0).
                    double est_n[S];
#pragma unroll
                    for (int s = 0; s < S; ++s) {
                        if (FULL) {
                            const int bl = min(max(b, 1), bmax);
                            est_n[s] = s_lat[(row[s] < 0 ? 0 : row[s]) + bl - 1];
                            if (row[s] < 0) est_n[s] = 0.0;
                        } else {
                            // one slot: the row address kept in a register; several slots:
                            // re-derived (registers are the scarcer resource there)
                            est_n[s] = S == 1 ? lds_f64(row_sh[s] + (uint32_t)b * 8u)
                                              : lds_f64(lat_sh + (uint32_t)(row[s] + b - 1) * 8u);
                        }
                    }
                    drain(t, 0, kEager);
                    // LookupError at this query (profile.hpp:127-129); only possible when the
                    // launch holds a scenario whose batches can leave the table (FULL)
                    if (FULL && (b < 1 || b > bmax)) {
                        status = MSV_LOOKUP;
                        return;
                    }
                    // ---- candidates and Eq. 1 waits (sched.hpp:77-85) ----
                    bool cand[S];
                    double wv[S];
#pragma unroll
                    for (int s = 0; s < S; ++s) {
                        cand[s] = act[s];
                        // Eq. 1 up front where every slot's wait is needed (FULL, or one slot);
                        // plain multi-slot ELSA evaluates it slot by slot below, FIFS never
                        if constexpr (FULL || (SCHED == MSV_ELSA && S == 1)) {
                            const double x = c_est[s] - (t - c_start[s]);
                            wv[s] = fold[s] + running_part(c_comp[s], t, x);
                        }
                    }
                    int bad_o = 1 << 30;  // order index of the first candidate whose size is missing
                    if (FULL) {
                        if (p.any_routing && route_mask != nullptr) {  // engine.hpp:197-206
                            unsigned anyc = 0;
#pragma unroll
                            for (int s = 0; s < S; ++s) {
                                cand[s] = act[s] && (((route_mask[s * 32 + lane] >> (b - 1)) & 1ull) != 0);
                                anyc |= __ballot_sync(kFull, cand[s]);
                            }
                            if (anyc == 0) {
#pragma unroll
                                for (int s = 0; s < S; ++s) cand[s] = act[s];
                            }
                        }
                        if (p.any_bad) {
#pragma unroll
                            for (int s = S - 1; s >= 0; --s) {
                                const unsigned bb = __ballot_sync(kFull, cand[s] && row[s] < 0);
                                if (bb) bad_o = s * 32 + __ffs(bb) - 1;
                            }
                        }
                        if (check_wait) {  // engine.hpp:208-217
#pragma unroll
                            for (int s = 0; s < S; ++s) {
                                if (!cand[s] || row[s] < 0) continue;
                                const double y = c_comp[s] - t;
                                const double gw = fold[s] + pos_part(y);  // y > 0 iff running
                                const double dd = fabs(gw - wv[s]);
                                wdiff = (wdiff < dd) ? dd : wdiff;
                            }
                        }
                    }
                    // ---- decision ----
                    int ch = -1;  // chosen order index
                    int kind = MSV_SLACK_SATISFYING;
                    bool mine[S];  // this lane's slot s is the chosen partition
                    bool bounded = false;
                    if constexpr (kLazy) {
                        bool stale = false;
#pragma unroll
                        for (int s = 0; s < S; ++s) stale |= gn[s] > 0 && !(pk[s] & kFv);
                        bounded = __any_sync(kFull, stale);
                    }
                    if (bounded) {
                        // Some slot's fold is stale: decide on bounds, refold only the slots a
                        // decision cannot be settled without (Step A near sla, Step B near the min).
                        double vlo[S], vhi[S];
                        bool stl[S];
#pragma unroll
                        for (int s = 0; s < S; ++s) {
                            const double x = c_est[s] - (t - c_start[s]);
                            const double xp = running_part(c_comp[s], t, x);
                            stl[s] = gn[s] > 0 && !(pk[s] & kFv);
                            double flo = fold[s], fhi = fold[s];
                            if (stl[s]) {  // |left fold - exact sum| <= (n-1) 2^-53 sum; slack x2
                                const double hi = W.dd_hi[s][lane], lo = W.dd_lo[s][lane];
                                const double g = (double)(qn[s] + (int)gn[s] + 4) * 0x1p-52;
                                flo = __dmul_rd(__dadd_rd(hi, lo), __dadd_rd(1.0, -g));
                                fhi = __dmul_ru(__dadd_ru(hi, lo), __dadd_ru(1.0, g));
                            }
                            // RN additions are monotone: the exact w + est lies in [vlo, vhi]
                            vlo[s] = (flo + xp) + est_n[s];
                            vhi[s] = (fhi + xp) + est_n[s];
                        }
                        auto exact = [&](int s) {  // refold slot s and make its value exact
                            fold[s] = refold(s);
                            pk[s] |= kFv;
                            stl[s] = false;
                            const double x = c_est[s] - (t - c_start[s]);
                            vlo[s] = vhi[s] = (fold[s] + running_part(c_comp[s], t, x)) + est_n[s];
                        };
#pragma unroll
                        for (int s = 0; s < S; ++s) {  // Step A (sched.hpp:125-130), slots in order
                            bool pred;
                            if constexpr (UNIT) {
                                if (act[s] && stl[s] && sla > vlo[s] && !(sla > vhi[s])) exact(s);
                                pred = act[s] && (sla > vhi[s]);
                            } else {
                                if (act[s] && stl[s]) exact(s);
                                const double x = c_est[s] - (t - c_start[s]);
                                const double w = fold[s] + running_part(c_comp[s], t, x);
                                pred = act[s] && (sla > alpha * (w + beta * est_n[s]));
                            }
                            const unsigned bA = __ballot_sync(kFull, pred);
                            if (bA) {
                                ch = s * 32 + __ffs(bA) - 1;
                                break;
                            }
                        }
                        if (ch < 0) {  // Step B (sched.hpp:132-142): argmin w + est, earliest on ties
                            uint64_t lm = ~0ull;
#pragma unroll
                            for (int s = 0; s < S; ++s)
                                if (act[s]) lm = msv_dbits(vhi[s]) < lm ? msv_dbits(vhi[s]) : lm;
                            const uint64_t mhi = seg_min_u64<32>(lm);  // >= the true minimum
                            bool cnd[S];
                            int ncand = 0;
#pragma unroll
                            for (int s = 0; s < S; ++s) {
                                cnd[s] = act[s] && msv_dbits(vlo[s]) <= mhi;  // may attain the minimum
                                ncand += __popc(__ballot_sync(kFull, cnd[s]));
                            }
                            if (ncand > 1) {  // overlapping candidates: compare exact values
                                uint64_t lv = ~0ull;
#pragma unroll
                                for (int s = 0; s < S; ++s) {
                                    if (cnd[s] && stl[s]) exact(s);
                                    if (cnd[s]) lv = msv_dbits(vhi[s]) < lv ? msv_dbits(vhi[s]) : lv;
                                }
                                const uint64_t vmin = seg_min_u64<32>(lv);
#pragma unroll
                                for (int s = S - 1; s >= 0; --s) cnd[s] = cnd[s] && msv_dbits(vhi[s]) == vmin;
                            }
                            // a single candidate is the argmin whatever its exact value
#pragma unroll
                            for (int s = S - 1; s >= 0; --s) {
                                const unsigned bB = __ballot_sync(kFull, cnd[s]);
                                if (bB) ch = s * 32 + __ffs(bB) - 1;
                            }
                            kind = MSV_FASTEST_FALLBACK;
                        }
#pragma unroll
                        for (int s = 0; s < S; ++s) mine[s] = s * 32 + lane == ch;
                    } else if constexpr (SCHED == MSV_ELSA && S == 1 && !FULL) {
                        // One slot per lane: the chosen lane is the lowest set bit of the
                        // ballot, i.e. the lane with no set bit below it — no bit scan on the
                        // critical path.
                        const unsigned below = (1u << lane) - 1u;
                        bool pred;
                        if constexpr (UNIT) pred = sla_act > wv[0] + est_n[0];  // inactive lanes: -inf
                        else pred = act[0] && (sla > alpha * (wv[0] + beta * est_n[0]));
                        const unsigned bA = __ballot_sync(kFull, pred);  // Step A (sched.hpp:125-130)
                        mine[0] = pred && (bA & below) == 0;
                        kind = MSV_SLACK_SATISFYING;
                        if (bA == 0) {  // Step B (sched.hpp:132-142): argmin w + est, earliest on ties
                            const uint64_t fb = act[0] ? msv_dbits(wv[0] + est_n[0]) : ~0ull;
                            const uint64_t vmin = seg_min_u64<32>(fb);
                            const bool hit = fb == vmin && vmin != ~0ull;
                            const unsigned bB = __ballot_sync(kFull, hit);
                            mine[0] = hit && (bB & below) == 0;
                            kind = MSV_FASTEST_FALLBACK;
                        }
                    } else if constexpr (SCHED == MSV_ELSA && !FULL) {
                        // Several slots per lane: Step A scans the slots in order (slot s holds
                        // order indices [32s, 32s + 32)) and stops at the first slot with a
                        // satisfying partition, so later slots' waits are computed only when
                        // needed (Step B needs them all).
                        kind = MSV_SLACK_SATISFYING;
                        int s_eval = 0;
#pragma unroll
                        for (int s = 0; s < S; ++s) {
                            if (s >= kEager) drain(t, s, s + 1);  // this slot is needed now
                            const double x = c_est[s] - (t - c_start[s]);
                            wv[s] = fold[s] + running_part(c_comp[s], t, x);
                            s_eval = s + 1;
                            bool pred;
                            if constexpr (UNIT) pred = act[s] && (sla > wv[s] + est_n[s]);
                            else pred = act[s] && (sla > alpha * (wv[s] + beta * est_n[s]));
                            const unsigned bA = __ballot_sync(kFull, pred);
                            if (bA) {
                                ch = s * 32 + __ffs(bA) - 1;
                                break;
                            }
                        }
                        if (ch < 0) {  // Step B (sched.hpp:132-142): argmin w + est, earliest on ties
                            (void)s_eval;  // every slot was evaluated (no break)
                            uint64_t fb[S];
                            uint64_t vmin = ~0ull;
#pragma unroll
                            for (int s = 0; s < S; ++s) {
                                fb[s] = act[s] ? msv_dbits(wv[s] + est_n[s]) : ~0ull;
                                vmin = fb[s] < vmin ? fb[s] : vmin;
                            }
                            vmin = seg_min_u64<32>(vmin);
#pragma unroll
                            for (int s = S - 1; s >= 0; --s) {
                                const unsigned bB = __ballot_sync(kFull, fb[s] == vmin && vmin != ~0ull);
                                if (bB) ch = s * 32 + __ffs(bB) - 1;
                            }
                            kind = MSV_FASTEST_FALLBACK;
                        }
                    } else if constexpr (SCHED == MSV_ELSA) {
                        // Step A (sched.hpp:125-130): first in order with sla > alpha*(w + beta*est).
#pragma unroll
                        for (int s = S - 1; s >= 0; --s) {
                            const bool ok = FULL ? (cand[s] && row[s] >= 0) : act[s];
                            bool pred;
                            if constexpr (UNIT) pred = ok && (sla > wv[s] + est_n[s]);
                            else pred = ok && (sla > alpha * (wv[s] + beta * est_n[s]));
                            const unsigned bA = __ballot_sync(kFull, pred);
                            if (bA) ch = s * 32 + __ffs(bA) - 1;
                        }
                        kind = MSV_SLACK_SATISFYING;
                        if (ch < 0) {  // Step B (sched.hpp:132-142): argmin w + est, earliest on ties
                            uint64_t fb[S];
                            uint64_t vmin = ~0ull;
#pragma unroll
                            for (int s = 0; s < S; ++s) {
                                const bool ok = FULL ? (cand[s] && row[s] >= 0) : act[s];
                                fb[s] = ok ? msv_dbits(wv[s] + est_n[s]) : ~0ull;
                                vmin = fb[s] < vmin ? fb[s] : vmin;
                            }
                            vmin = seg_min_u64<32>(vmin);
#pragma unroll
                            for (int s = S - 1; s >= 0; --s) {
                                const unsigned bB = __ballot_sync(kFull, fb[s] == vmin && vmin != ~0ull);
                                if (bB) ch = s * 32 + __ffs(bB) - 1;
                            }
                            kind = MSV_FASTEST_FALLBACK;
                        }
                        // a size missing from the profile is a LookupError once the scan reaches it
                        if (FULL && bad_o != (1 << 30) && (kind == MSV_FASTEST_FALLBACK || bad_o < ch)) {
                            status = MSV_LOOKUP;
                            return;
                        }
                    } else {
                        // FIFS (sched.hpp:154-170): idle -> max k, min id; else shortest queue, min id.
                        uint32_t key[S];
                        uint32_t mi = ~0u;
#pragma unroll
                        for (int s = 0; s < S; ++s) {
                            key[s] = (cand[s] && !(c_comp[s] > t))
                                         ? (((0x7FFFu - ((uint32_t)pk[s] >> 8)) << 16) | ((uint32_t)pk[s] & 0xffu))
                                         : ~0u;
                            mi = key[s] < mi ? key[s] : mi;
                        }
                        mi = __reduce_min_sync(kFull, mi);
                        kind = MSV_IDLE_LARGEST;
                        if (mi == ~0u) {
                            kind = MSV_SHORTEST_QUEUE;
#pragma unroll
                            for (int s = 0; s < S; ++s) {
                                const uint32_t len = (uint32_t)qn[s] + gn[s];
                                key[s] = cand[s] ? (((len < 0xFFFFFFu ? len : 0xFFFFFFu) << 8) | ((uint32_t)pk[s] & 0xffu))
                                                 : ~0u;
                                mi = key[s] < mi ? key[s] : mi;
                            }
                            mi = __reduce_min_sync(kFull, mi);
                        }
#pragma unroll
                        for (int s = S - 1; s >= 0; --s) {
                            const unsigned bs = __ballot_sync(kFull, key[s] == mi);
                            if (bs) ch = s * 32 + __ffs(bs) - 1;
                        }
                        if (FULL && p.any_bad) {  // the chosen partition's latency lookup fails (engine.hpp:226)
                            bool mine = false;
#pragma unroll
                            for (int s = 0; s < S; ++s) mine |= (s * 32 + lane == ch) && row[s] < 0;
                            if (__any_sync(kFull, mine)) {
                                status = MSV_LOOKUP;
                                return;
                            }
                        }
                    }
                    if constexpr (!(SCHED == MSV_ELSA && S == 1 && !FULL)) {
                        if (!bounded) {
#pragma unroll
                            for (int s = 0; s < S; ++s) mine[s] = s * 32 + lane == ch;
                        }
                    }
                    // ---- start or enqueue on the chosen partition (engine.hpp:225-230) ----
                    // One slot per lane: straight-line and predicated on `mine` — every lane
                    // executes the same instructions (no divergent region), only the chosen
                    // one changes state. Several slots: only the chosen slot's lane runs it
                    // (a warp-uniform branch on the chosen slot measured slower: S = 2 classes
                    // 4.1 vs 5.0 G q/s on a B200).
#pragma unroll
                    for (int s = 0; s < S; ++s) {
                        const bool m = mine[s];
                        if (!(S == 1 || m)) continue;
                        const double est = est_n[s];
                        const bool busy = c_comp[s] > t;
                        const double st = sel_f64(busy, tail[s], t);  // queued: starts when the last placed finishes
                        const double fin = st + est;
                        const bool now = m && !busy;  // idle: starts at its arrival
                        const bool push = m && busy;
                        tail[s] = sel_f64(m, fin, tail[s]);
                        c_start[s] = sel_f64(now, t, c_start[s]);
                        c_est[s] = sel_f64(now, est, c_est[s]);
                        c_comp[s] = sel_f64(now, fin, c_comp[s]);
                        // appending extends the left fold exactly (a stale fold stays stale)
                        fold[s] = sel_f64(push, fold[s] + est, fold[s]);
                        // ring append predicated (no divergent region); the overflow list behind
                        // a full ring is the rare branch
                        const bool ring_ok = gn[s] == 0 && qn[s] < QC;
                        if (push && ring_ok) {
                            W.q_est[s][(qh[s] + qn[s]) & (QC - 1)][lane] = est;
                            qn[s] += 1;
                        }
                        if (push && !ring_ok) {
                            {
                                if (kLazy) {  // overflow mode: keep the double-double sum
                                    double hi = 0.0, lo = 0.0;
                                    if (gn[s] == 0) {  // entering it: sum the ring, the fold is exact
#pragma unroll 1
                                        for (int k = 0; k < qn[s]; ++k)
                                            dd_add(hi, lo, W.q_est[s][(qh[s] + k) & (QC - 1)][lane]);
                                        pk[s] |= kFv;
                                    } else {
                                        hi = W.dd_hi[s][lane];
                                        lo = W.dd_lo[s][lane];
                                    }
                                    dd_add(hi, lo, est);
                                    W.dd_hi[s][lane] = hi;
                                    W.dd_lo[s][lane] = lo;
                                }
                                if (gn[s] == 0) W.g_head[s][lane] = (uint32_t)i;
                                else g_next[W.g_tail[s][lane]] = (uint32_t)i;
                                W.g_tail[s][lane] = (uint32_t)i;
                                gn[s] += 1;
                            }
                        }
                        if (m) {
                            W.win_sf[j] = make_double2(st, fin);
                            W.win_p[j] = (pk[s] & 0xff) | (kind << 8);
                            if (FULL) {  // PartitionUsage (engine.hpp:175-177), completion order
                                const double ran = fin - st;
                                bms[s] = bms[s] + ran;
                                wbms[s] = wbms[s] + ran * s_util[row[s] + b - 1];
                                nq[s] += 1;
                            }
                        }
                    }
                }
                // ---- retire the window: lane j completes query base + j (engine.hpp:167-187) ----
                __syncwarp();
                if (lane < cnt) {
                    const int i = base + lane;
                    const double2 sf = W.win_sf[lane];
                    const double st = sf.x, fin = sf.y;
                    const int pw = W.win_p[lane];
                    const double lat = fin - cur_t;  // latency = finish - arrival
                    const bool met = lat <= sla;
                    viol += met ? 0u : 1u;
                    if (cur_t >= warmup) {  // measured (engine.hpp:262): overwrite the dead arrivals
                        mviol += met ? 0u : 1u;
                        const uint64_t lb = msv_dbits(lat);
                        uint32_t* const row = samples + 2 * base;  // this window's 256 bytes
                        row[lane] = (uint32_t)(lb >> 32);
                        row[32 + lane] = (uint32_t)lb;
                    }
                    hash += msv_query_digest((uint64_t)i, pw & 0xff, st, fin);
                    if (REC) {
                        msv_record r;
                        r.start_ms = st;
                        r.finish_ms = fin;
                        r.partition = pw & 0xff;
                        r.kind = pw >> 8;
                        rec[i] = r;
                    }
                }
            }
        };
        if (d.alpha == 1.0 && d.beta == 1.0) simulate(std::true_type{});
        else simulate(std::false_type{});
        // (nothing to drain after the last arrival: every query was retired with its window)

        // ---- publish (engine.hpp:233-252) ----
        // last completion = each slot's last placed finish (finishes per slot ascend; a
        // slot that never ran keeps 0.0, below every completion and the duration)
        double lf = 0.0;
#pragma unroll
        for (int s = 0; s < S; ++s) lf = (lf < tail[s]) ? tail[s] : lf;
        const uint64_t v0 = seg_sum_u64<32>((uint64_t)viol, kFull);
        const uint64_t v2 = seg_sum_u64<32>((uint64_t)mviol, kFull);
        const uint64_t hsum = seg_sum_u64<32>(hash, kFull);
        lf = seg_max_f64<32>(lf, kFull);
        const double wd = seg_max_f64<32>(wdiff, kFull);
        if (lane == 0) {
            DevOut o;
            o.violations = (int64_t)v0;
            o.measured = m0 >= 0 ? n - m0 : 0;
            o.measured_violations = (int64_t)v2;
            o.n_samples = o.measured;
            o.horizon_ms = (d.duration_ms < lf) ? lf : d.duration_ms;  // engine.hpp:237
            o.max_wait_diff = wd;
            o.hash = hsum;
            // no key bounds (min > max): K3 derives them from the high words (tracking them
            // here costs the simulation loop more than K3's extra 4-byte pass)
            o.lat_min_bits = ~0ull;
            o.lat_max_bits = 0;
            o.planar = 1;
            o.pad = 0;
            o.status = status;
            o.m0 = m0 >= 0 ? m0 : 0;
            p.out[sidx] = o;
        }
        if (FULL && p.any_usage && d.usage_off >= 0) {
#pragma unroll
            for (int s = 0; s < S; ++s) {
                if (act[s]) {
                    msv_usage u;
                    u.busy_ms = bms[s];
                    u.weighted_busy_ms = wbms[s];
                    u.queries = nq[s];
                    p.usage[d.usage_off + (pk[s] & 0xff)] = u;
                }
            }
        }
    }
}

template <int S, int SCHED>
void* pick_flags(bool rec, bool full, bool lazy) {
    if (rec) return (void*)&sim_warp_kernel<S, SCHED, true, true, false>;
    if (full) return (void*)&sim_warp_kernel<S, SCHED, false, true, false>;
    if constexpr (SCHED == MSV_ELSA) {
        if (lazy) return (void*)&sim_warp_kernel<S, SCHED, false, false, true>;
    }
    return (void*)&sim_warp_kernel<S, SCHED, false, false, false>;
}

}  // namespace

void* sim_warp_fn(int S, int sched, bool rec, bool full, bool lazy) {
    if (S == 1)
        return sched == MSV_ELSA ? pick_flags<1, MSV_ELSA>(rec, full, lazy) : pick_flags<1, MSV_FIFS>(rec, full, lazy);
    if (S == 2)
        return sched == MSV_ELSA ? pick_flags<2, MSV_ELSA>(rec, full, lazy) : pick_flags<2, MSV_FIFS>(rec, full, lazy);
    if (S == 4)
        return sched == MSV_ELSA ? pick_flags<4, MSV_ELSA>(rec, full, lazy) : pick_flags<4, MSV_FIFS>(rec, full, lazy);
    return nullptr;
}

size_t sim_warp_smem_bytes(int S, int n_cells) {
    const size_t tab = ((size_t)2 * n_cells * sizeof(double) + 15) & ~(size_t)15;
    const size_t per_warp = S == 1 ? sizeof(WarpSmem<1>) : (S == 2 ? sizeof(WarpSmem<2>) : sizeof(WarpSmem<4>));
    return tab + (size_t)kSimWarpsPerBlock * per_warp;
}

}  // namespace msv
