// Dispatch policies: ELSA (paper Alg. 2) and the FIFS baseline, plus the
// paper's Eq. 1 / Eq. 2 estimators. Same API as the reference's sched.hpp
// (sched.hpp:17-174). Decisions are evaluated on the device by the same
// arithmetic the simulation kernel uses (msv_dispatch_batch); inside run() the
// engine evaluates them lane-parallel per partition instead of calling these.
#pragma once

#include <algorithm>
#include <cstdint>
#include <deque>
#include <limits>
#include <optional>
#include <string>
#include <vector>

#include "device.hpp"
#include "errors.hpp"
#include "profile.hpp"
#include "workload.hpp"

namespace migserve {

struct QueuedQuery {
    int64_t query_id = 0;
    int batch = 1;
    double est_ms = 0.0;
};

struct RunningQuery {
    int64_t query_id = 0;
    int batch = 1;
    double est_ms = 0.0;
    double start_ms = 0.0;
};

// One partition: the query executing now plus its FIFO.
struct PartitionState {
    int id = 0;
    PartitionSize k;
    std::deque<QueuedQuery> queued;
    std::optional<RunningQuery> current;
    bool busy() const { return current.has_value(); }
};

struct SlaConfig {
    double sla_target_ms = 0.0;
    double alpha = 1.0;
    double beta = 1.0;
    void validate() const {
        if (!(sla_target_ms > 0.0)) throw ParamError("sla: target must be > 0");
        if (alpha < 0.0 || beta < 0.0) throw ParamError("sla: alpha/beta must be >= 0");
    }
};

enum class DispatchKind { SlackSatisfying, FastestFallback, IdleLargest, ShortestQueue };

inline const char* to_string(DispatchKind kind) {
    switch (kind) {
        case DispatchKind::SlackSatisfying: return "slack-satisfying";
        case DispatchKind::FastestFallback: return "fastest-fallback";
        case DispatchKind::IdleLargest: return "idle-largest";
        case DispatchKind::ShortestQueue: return "shortest-queue";
    }
    return "?";
}

struct Dispatch {
    int64_t query_id = 0;
    int partition_id = 0;
    DispatchKind kind = DispatchKind::SlackSatisfying;
};

// Eq. 2: slack = target - alpha * (wait + beta * est).
inline double sla_slack(const SlaConfig& cfg, double t_wait_ms, double t_est_new_ms) {
    return cfg.sla_target_ms - cfg.alpha * (t_wait_ms + cfg.beta * t_est_new_ms);
}

namespace detail {

// (size, id) ascending scan order of both ELSA steps (sched.hpp:96-104).
inline std::vector<std::size_t> by_ascending_size(const std::vector<const PartitionState*>& parts) {
    std::vector<std::size_t> idx(parts.size());
    for (std::size_t i = 0; i < idx.size(); ++i) idx[i] = i;
    std::sort(idx.begin(), idx.end(), [&](std::size_t a, std::size_t b) {
        return parts[a]->k != parts[b]->k ? parts[a]->k < parts[b]->k : parts[a]->id < parts[b]->id;
    });
    return idx;
}

inline std::vector<const PartitionState*> as_pointers(const std::vector<PartitionState>& parts) {
    std::vector<const PartitionState*> out;
    out.reserve(parts.size());
    for (const PartitionState& p : parts) out.push_back(&p);
    return out;
}

// Flattened partition states for msv_dispatch_batch (one trial).
struct DispatchBatch {
    std::vector<int64_t> part_off{0};
    std::vector<int32_t> id, k;
    std::vector<uint8_t> busy;
    std::vector<double> cur_est, cur_start;
    std::vector<int64_t> q_off{0};
    std::vector<int32_t> qbatch;
    std::vector<int32_t> query_batch;
    std::vector<double> now, sla, alpha, beta;

    void add_trial(const std::vector<const PartitionState*>& parts, int batch, double now_ms, const SlaConfig& cfg) {
        for (const PartitionState* p : parts) {
            id.push_back(p->id);
            k.push_back(p->k.gpcs);
            busy.push_back(p->busy() ? 1 : 0);
            cur_est.push_back(p->current ? p->current->est_ms : 0.0);
            cur_start.push_back(p->current ? p->current->start_ms : 0.0);
            for (const QueuedQuery& q : p->queued) qbatch.push_back(q.batch);
            q_off.push_back(static_cast<int64_t>(qbatch.size()));
        }
        part_off.push_back(static_cast<int64_t>(id.size()));
        query_batch.push_back(batch);
        now.push_back(now_ms);
        sla.push_back(cfg.sla_target_ms);
        alpha.push_back(cfg.alpha);
        beta.push_back(cfg.beta);
    }

    // Runs the trials on the device; returns (partition id, kind) per trial.
    void run(int profile_handle, int scheduler, std::vector<int32_t>& chosen, std::vector<int32_t>& kind,
             std::vector<double>* t_wait = nullptr) {
        const int64_t n = static_cast<int64_t>(query_batch.size());
        chosen.assign(static_cast<std::size_t>(n), -1);
        kind.assign(static_cast<std::size_t>(n), 0);
        if (t_wait) t_wait->assign(id.size(), 0.0);
        device::check(msv_dispatch_batch(device::context().get(), profile_handle, scheduler, n, part_off.data(),
                                         id.data(), k.data(), busy.data(), cur_est.data(), cur_start.data(),
                                         q_off.data(), qbatch.data(), query_batch.data(), now.data(), sla.data(),
                                         alpha.data(), beta.data(), chosen.data(), kind.data(),
                                         t_wait ? t_wait->data() : nullptr),
                      "msv_dispatch_batch");
    }
};

}  // namespace detail

// Eq. 1 (sched.hpp:77-85): profiled time of everything queued, in FIFO order, plus
// the unexpired remainder of the running query.
inline double t_wait(const PartitionState& state, const ProfileTable& table, double now_ms) {
    detail::DispatchBatch b;
    b.add_trial({&state}, 1, now_ms, SlaConfig{1.0, 1.0, 1.0});
    std::vector<int32_t> chosen, kind;
    std::vector<double> w;
    b.run(table.device_handle(), MSV_FIFS, chosen, kind, &w);
    if (w[0] != w[0]) {  // NaN marks a lookup outside the grid
        for (const QueuedQuery& q : state.queued) (void)table.latency_ms(state.k, q.batch);  // throws LookupError
        throw LookupError("t_wait: profile lookup outside the grid");
    }
    return w[0];
}

// Alg. 2: Step A takes the first (smallest) partition with strictly positive
// slack; Step B the earliest finisher (sched.hpp:119-143).
inline Dispatch elsa_dispatch(const Query& query, const std::vector<const PartitionState*>& partitions,
                              const ProfileTable& table, const SlaConfig& cfg, double now_ms) {
    if (partitions.empty()) throw ParamError("elsa_dispatch: no partitions");
    detail::DispatchBatch b;
    b.add_trial(partitions, query.batch, now_ms, cfg);
    std::vector<int32_t> chosen, kind;
    b.run(table.device_handle(), MSV_ELSA, chosen, kind);
    return Dispatch{query.id, chosen[0], static_cast<DispatchKind>(kind[0])};
}

inline Dispatch elsa_dispatch(const Query& query, const std::vector<PartitionState>& partitions,
                              const ProfileTable& table, const SlaConfig& cfg, double now_ms) {
    return elsa_dispatch(query, detail::as_pointers(partitions), table, cfg, now_ms);
}

// FIFS: any idle partition (largest, then lowest id), else the shortest queue
// (lowest id on ties) (sched.hpp:154-170).
inline Dispatch fifs_dispatch(const Query& query, const std::vector<const PartitionState*>& partitions) {
    if (partitions.empty()) throw ParamError("fifs_dispatch: no partitions");
    detail::DispatchBatch b;
    b.add_trial(partitions, query.batch, 0.0, SlaConfig{1.0, 1.0, 1.0});
    std::vector<int32_t> chosen, kind;
    b.run(-1, MSV_FIFS, chosen, kind);
    return Dispatch{query.id, chosen[0], static_cast<DispatchKind>(kind[0])};
}

inline Dispatch fifs_dispatch(const Query& query, const std::vector<PartitionState>& partitions) {
    return fifs_dispatch(query, detail::as_pointers(partitions));
}

}  // namespace migserve
