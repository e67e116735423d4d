// dispatch_kernel: single elsa_dispatch / fifs_dispatch / t_wait decisions
// (sched.hpp:77-174), one thread per trial, for the API-level functions.
#include "msv_device.cuh"

namespace msv {

namespace {
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

cudaError_t launch_dispatch(const DispatchParams& p, cudaStream_t stream) {
    if (p.n_trials <= 0) return cudaSuccess;
    const int threads = 128;
    const int blocks = (int)((p.n_trials + threads - 1) / threads);
    dispatch_kernel<<<blocks, threads, 0, stream>>>(p);
    return cudaGetLastError();
}

}  // namespace msv
