// Host runtime behind the C ABI (include/msv.h): contexts, immutable input
// uploads with the reference's validation rules, grid construction (waves,
// scenario classes), kernel orchestration on the context stream and result
// assembly. Compiled with -ffp-contract=off: the cdf partial sum and the
// host-side copies of reference arithmetic must round like the reference.
#include <math.h>
#include <string.h>

#include <algorithm>
#include <limits>
#include <atomic>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <map>
#include <memory>
#include <mutex>
#include <numeric>
#include <string>
#include <utility>
#include <sched.h>
#include <thread>
#include <vector>

#include "msv_internal.h"
#include "msv_math.h"

using msv::DevOut;
using msv::DevPart;
using msv::DevScen;

namespace {

thread_local std::string g_err;

int fail(int code, std::string msg) {
    g_err = std::move(msg);
    return code;
}

#define MSV_CUDA_TRY(x)                                                                  \
    do {                                                                                 \
        cudaError_t e_ = (x);                                                            \
        if (e_ != cudaSuccess) return fail(MSV_CUDA, std::string(#x ": ") + cudaGetErrorString(e_)); \
    } while (0)

// Bumped by every device allocation / free of the engine: free_device_bytes() caches
// cudaMemGetInfo only while this is unchanged.
std::atomic<uint64_t> g_alloc_epoch{0};

struct DevBuf {
    void* p = nullptr;
    size_t bytes = 0;
    DevBuf() = default;
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    ~DevBuf() { release(); }
    void release() {
        if (p) {
            cudaFree(p);
            g_alloc_epoch.fetch_add(1, std::memory_order_relaxed);
        }
        p = nullptr;
        bytes = 0;
    }
    cudaError_t ensure(size_t n) {
        if (n <= bytes && p) return cudaSuccess;
        release();
        if (n == 0) n = 16;
        cudaError_t e = cudaMalloc(&p, n);
        if (e == cudaSuccess) bytes = n;
        g_alloc_epoch.fetch_add(1, std::memory_order_relaxed);
        return e;
    }
    template <typename T>
    T* as() const {
        return static_cast<T*>(p);
    }
};

struct Profile {
    std::vector<int32_t> sizes;
    int b_max = 0;
    std::vector<double> lat, util;
    int cell_off = 0;
    int size_off = 0;
};

struct Dist {
    std::vector<double> pmf, cdf;
    size_t dev_off = 0;
    size_t guide_off = 0;
};

struct Plan {
    int num_gpus = 0, gpcs_per_gpu = 0;
    std::vector<int32_t> flat;  // partition sizes by id (plan.flatten(), paris.hpp:134-139)
    int err = 0;                // deferred PartitionPlan::validate() failure
    std::string err_msg;
};

struct Routing {
    std::vector<int32_t> k, first, last;
};

// glibc's log1p build selected on this host (rng.hpp:20 calls whichever one the
// ifunc resolver picked). Probe inputs where the two transcribed builds round
// differently and vote; every probed input must agree with the winning build (inputs
// where the builds agree included). A host libm matching neither — another glibc —
// returns -1: the device would diverge from the host reference, so msv_create fails
// instead of silently picking one.
int probe_host_log1p() {
    uint64_t s = 0x9E3779B97F4A7C15ull;
    int fma_votes = 0, gen_votes = 0, neither = 0;
    for (int it = 0; it < 2000000 && fma_votes + gen_votes < 16; ++it) {
        s ^= s << 13;
        s ^= s >> 7;
        s ^= s << 17;
        const double u = (double)(s >> 11) * 0x1.0p-53;
        const double a = msv_log1p_neg(-u, MSV_LOG1P_FMA);
        const double g = msv_log1p_neg(-u, MSV_LOG1P_GENERIC);
        volatile double xin = -u;
        const double h = log1p(xin);
        if (msv_dbits(a) == msv_dbits(g)) {
            neither += msv_dbits(h) != msv_dbits(a);
            continue;
        }
        if (msv_dbits(h) == msv_dbits(a)) ++fma_votes;
        else if (msv_dbits(h) == msv_dbits(g)) ++gen_votes;
        else ++neither;
    }
    if (neither || (fma_votes && gen_votes) || fma_votes + gen_votes == 0) return -1;
    return gen_votes ? MSV_LOG1P_GENERIC : MSV_LOG1P_FMA;
}

}  // namespace

namespace migserve_capi {
int set_error(int code, const char* what) { return fail(code, what ? what : ""); }
}  // namespace migserve_capi

// Device buffers of one grid launch sequence.
struct GridBufs {
    DevBuf d_scen, d_out, d_tjobs, d_tgroups, d_tailjobs, d_tails, d_p, d_usage, d_nq, d_tovf, d_parts, d_masks,
        d_work, d_counter, d_sjobs;
    DevBuf d_arr, d_bat, d_next, d_rec, d_glat, d_gutil, d_gcdf, d_gguide;
};

// guide[j] = first i with !(cdf[i] < j/G): lower_bound's answer for u = j/G, a valid
// start for every u >= j/G (the cdf is nondecreasing).
static void append_guide(const std::vector<double>& cdf, std::vector<int16_t>& guide) {
    for (int j = 0; j < msv::kGuide; ++j) {
        const double uj = (double)j / (double)msv::kGuide;
        size_t i = 0;
        while (i < cdf.size() && cdf[i] < uj) ++i;
        guide.push_back((int16_t)i);
    }
}

struct msv_ctx {
    int device = 0;
    GridBufs scratch;  // reused by one-shot grids (msv_run_grid / msv_run_replay)
    // reused by noisy grids (msv_run_grid_noise): multipliers and K5 jobs
    DevBuf d_mult, d_njobs;
    // reused by single noisy runs (msv_run_noise): no allocation per call
    struct NoiseRunBufs {
        DevBuf arr, bat, mult, lat, util, parts, masks, next, rec, use, out, job;
    } noise1;
    // pinned staging of the multiplier streams: two buffers, alternating by chunk
    double* pin[2] = {nullptr, nullptr};
    size_t pin_n = 0;  // doubles per buffer
    cudaEvent_t pin_ev[2] = {};  // the copy out of the buffer is done
    cudaEvent_t k1_ev = nullptr;
    int sms = 148;
    cudaStream_t stream = nullptr;
    int log1p = MSV_LOG1P_FMA;
    int64_t launches = 0;
    int64_t h2d = 0, d2h = 0;
    cudaEvent_t ev[8] = {};
    cudaStream_t aux[8] = {};    // chunk streams of overlapped grid launches
    cudaEvent_t aux_ev[8] = {};
    cudaEvent_t fork_ev = nullptr;
    cudaEvent_t region_ev[8] = {};  // a multi-wave grid's buffer region is free again
    uint64_t grid_serial = 0;       // grids created on this context
    uint64_t last_launch_grid = 0;  // serial of the grid launched last
    cudaStream_t cls[4] = {};    // extra class streams: a chunk's kernel classes run concurrently
    cudaEvent_t cls_ev[4] = {};
    cudaEvent_t cls_fork = nullptr;
    std::vector<Profile> profiles;
    std::vector<Dist> dists;
    std::vector<Plan> plans;
    std::vector<Routing> routings;
    // Multi-device context (msv_create_multi): this context is member 0 (device_ids[0]);
    // `peers` are members 1..n-1, each a full context on its own device. Uploads go to
    // this context and are mirrored into the peers before a sharded call
    // (upload_serial / mirrored_serial); `share` = members on this context's device.
    std::vector<msv_ctx*> peers;
    uint64_t upload_serial = 0, mirrored_serial = 0;
    int share = 1;
    // concatenated profile cells / cdfs on the device
    DevBuf d_lat, d_util, d_cdf, d_pmf, d_guide, d_sizes;
    int n_cells = 0;
    bool tables_dirty = true;

    int sync_tables() {
        if (!tables_dirty) return MSV_OK;
        std::vector<double> lat, util, cdf, pmf;
        std::vector<int16_t> guide;
        std::vector<int32_t> sizes;
        for (Profile& p : profiles) {
            p.size_off = (int)sizes.size();
            sizes.insert(sizes.end(), p.sizes.begin(), p.sizes.end());
            p.cell_off = (int)lat.size();
            lat.insert(lat.end(), p.lat.begin(), p.lat.end());
            util.insert(util.end(), p.util.begin(), p.util.end());
        }
        for (Dist& d : dists) {
            d.dev_off = cdf.size();
            cdf.insert(cdf.end(), d.cdf.begin(), d.cdf.end());
            pmf.insert(pmf.end(), d.pmf.begin(), d.pmf.end());
            d.guide_off = guide.size();
            append_guide(d.cdf, guide);
        }
        n_cells = (int)lat.size();
        MSV_CUDA_TRY(d_lat.ensure(std::max<size_t>(lat.size(), 1) * 8));
        MSV_CUDA_TRY(d_util.ensure(std::max<size_t>(util.size(), 1) * 8));
        MSV_CUDA_TRY(d_cdf.ensure(std::max<size_t>(cdf.size(), 1) * 8));
        if (!lat.empty()) {
            MSV_CUDA_TRY(cudaMemcpy(d_lat.p, lat.data(), lat.size() * 8, cudaMemcpyHostToDevice));
            MSV_CUDA_TRY(cudaMemcpy(d_util.p, util.data(), util.size() * 8, cudaMemcpyHostToDevice));
        }
        if (!cdf.empty()) MSV_CUDA_TRY(cudaMemcpy(d_cdf.p, cdf.data(), cdf.size() * 8, cudaMemcpyHostToDevice));
        MSV_CUDA_TRY(d_pmf.ensure(std::max<size_t>(pmf.size(), 1) * 8));
        if (!pmf.empty()) MSV_CUDA_TRY(cudaMemcpy(d_pmf.p, pmf.data(), pmf.size() * 8, cudaMemcpyHostToDevice));
        MSV_CUDA_TRY(d_sizes.ensure(std::max<size_t>(sizes.size(), 1) * 4));
        if (!sizes.empty())
            MSV_CUDA_TRY(cudaMemcpy(d_sizes.p, sizes.data(), sizes.size() * 4, cudaMemcpyHostToDevice));
        MSV_CUDA_TRY(d_guide.ensure(std::max<size_t>(guide.size(), 1) * 2));
        if (!guide.empty())
            MSV_CUDA_TRY(cudaMemcpy(d_guide.p, guide.data(), guide.size() * 2, cudaMemcpyHostToDevice));
        tables_dirty = false;
        return MSV_OK;
    }
};

namespace {

struct SetDevice {
    int prev = -1;
    explicit SetDevice(int dev) {
        cudaGetDevice(&prev);
        if (prev != dev) cudaSetDevice(dev);
    }
    ~SetDevice() {
        int cur = -1;
        cudaGetDevice(&cur);
        if (prev >= 0 && cur != prev) cudaSetDevice(prev);
    }
};

// Scenario class: W lanes per scenario, S partition slots per lane, scheduler.
struct ClassKey {
    int W, S, sched;
    int lazy = 0;  // warp kernel with lazy folds (scenarios offered more than the plan's capacity)
    bool operator<(const ClassKey& o) const {
        return std::tie(W, S, sched, lazy) < std::tie(o.W, o.S, o.sched, o.lazy);
    }
};

constexpr int kMaxChunks = 8;           // chunks per wave (pipelined over kAuxStreams streams)
constexpr int64_t kChunkScenarios = 1024;  // smallest chunk worth its own launch
constexpr int kCounterSlots = 1024;      // work-stealing counters per launch (chunk x class)
constexpr int kAuxStreams = 4;  // chunk c runs on aux stream c % kAuxStreams (more for more regions)
constexpr int kMaxRegions = 8;  // buffer regions of a multi-wave grid (ctx->region_ev, ctx->aux)

// Kernel class of a plan with P partitions. The one-scenario-per-warp kernel (W = 32)
// serves every plan; the segmented kernel runs G = 32/W scenarios per warp (W lanes
// each, S slots per lane: P <= W*S) and needs fewer instructions per query, but keeps
// only n/G warps busy, so it pays only when the wave holds enough such plans to fill
// the device: `seg_w` is the narrowest segment width the wave can afford (32 = none).
// MSV_SEGMENTED=0 disables it, =1 forces the narrowest width that fits each plan.
int segmented_mode() {
    static const int mode = getenv("MSV_SEGMENTED") ? (atoi(getenv("MSV_SEGMENTED")) != 0 ? 1 : 0) : -1;
    return mode;
}

ClassKey class_of(int P, int sched, int seg_w, bool overloaded = false) {
    ClassKey c{32, 1, sched};
    if (segmented_mode() == 1) seg_w = 4;
    if (overloaded && sched == MSV_ELSA && segmented_mode() != 1) seg_w = 32;  // long queues: lazy warp kernel
    if (P <= 4 && seg_w <= 4) c.W = 4;
    else if (P <= 8 && seg_w <= 8) c.W = 8;
    else if (P <= 16 && seg_w <= 16) c.W = 16;
    else if (P <= 32) c.W = 32;
    else if (P <= 64) c.S = 2;
    else c.S = 4;
    // Overloaded scenarios grow long queues: the warp kernel's lazy-fold variant keeps them
    // O(1) per arrival (the plain variant pays O(queue) per pop, and the lazy paths would
    // cost it registers).
    if (c.W == 32 && sched == MSV_ELSA && overloaded) c.lazy = 1;
    return c;
}

// Narrowest segment width worth launching for a wave with n4 / n8 / n16 plans of
// P <= 4 / 8 / 16 on `sms` SMs: G scenarios per warp must still leave >= half of the
// segmented kernel's warp slots (~5 blocks x 4 warps per SM) busy. Measured without
// usage accumulation: W = 4 and 8 beat the warp kernel by 20-30 % on full waves; W = 16
// (and two slots per lane for 16 < P <= 32) lose to it, so they are never chosen here.
int wave_seg_width(int64_t n4, int64_t n8, int64_t n16, int sms) {
    if (segmented_mode() == 0) return 32;
    if (const char* e = getenv("MSV_SEG_WIDTH")) return atoi(e);  // A/B experiments
    const int64_t half_slots = (int64_t)sms * 5 * msv::kSimWarpsPerBlock / 2;
    if (n4 / 8 >= half_slots) return 4;
    if (n8 / 4 >= half_slots) return 8;
    return 32;
}

std::string fmt_num(double v) {
    char buf[64];
    snprintf(buf, sizeof buf, "%g", v);
    return buf;
}

}  // namespace

// ---------------------------------------------------------------------------
// Grid: everything one launch needs, resident on the device.
// ---------------------------------------------------------------------------
struct msv_grid {
    msv_ctx* ctx = nullptr;
    bool generated = true;
    bool records = false;
    int64_t n = 0;
    std::vector<msv_scenario> scen;
    std::vector<double> tail_p;
    std::vector<int64_t> cap, toff;   // per-scenario trace capacity and offset (arrival, batch)
    std::vector<int64_t> noff;        // per-scenario offset in the overflow-link buffer
    std::vector<int32_t> P, usage_off;
    std::vector<uint8_t> bad;  // plan has a size the profile lacks
    // Streamed K1 -> K2 (msv_sim_warp.cu STREAM): a latency-bound generated grid (one wave,
    // few scenarios, warp-kernel classes without routing / missing sizes / wait checks)
    // generates each trace inside its simulating block; records and usage launches do not.
    bool stream_ok = false;
    int64_t usage_total = 0;
    // A chunk is a set of scenarios launched together (K1 -> K2 per class -> K3) on one
    // stream; chunks of a wave run on different streams so one chunk's K1/K3 fill the
    // issue slots and the tail of another's K2. Job arrays are in launch order, so a
    // chunk's trace / tail jobs are the contiguous range [l0, l1).
    struct Chunk {
        int64_t l0 = 0, l1 = 0;
        int64_t g0 = 0, g1 = 0;  // K1 trace groups [g0, g1) in d_tgroups
        std::vector<std::pair<ClassKey, std::vector<int32_t>>> classes;
        std::vector<int64_t> work_off;  // offset of each class's work list in d_work
    };
    struct Wave {
        int64_t s0 = 0, s1 = 0;  // scenarios [s0, s1)
        int64_t q0 = 0, q1 = 0;  // trace slots [q0, q1)
        std::vector<Chunk> chunks;
    };
    uint64_t serial = 0;                // per-context creation number
    std::vector<int32_t> launch_order;  // scenario index of each launch slot
    std::vector<msv::TraceGroup> tgroups;  // K1 groups (launch-slot ranges), chunk by chunk
    bool overlap = true;                // chunks on concurrent streams
    bool usage = true;                  // accumulate per-partition usage (msv_grid_set_usage)
    std::vector<Wave> waves;
    int64_t max_wave_q = 0;             // query slots of the largest wave (one buffer region)
    int n_regions = 1;                  // buffer regions the waves alternate between (links, K2 / K3)
    int n_in_regions = 1;               // regions of the trace inputs (arrival / latency + batch)
    GridBufs own;            // buffers of a persistent grid (msv_grid_create)
    GridBufs* B = &own;      // -> own, or the context's scratch set for one-shot calls
    int n_cells = 0;
    std::vector<DevScen> h_scen;  // pointers into the wave buffers
    cudaEvent_t ev[4] = {nullptr, nullptr, nullptr, nullptr};
    // Many-profile grids (more profile cells than the kernels' shared table): one sub-grid
    // per profile group; this grid only dispatches and scatters.
    std::vector<std::unique_ptr<msv_grid>> parts;
    std::vector<std::vector<int64_t>> part_idx;
    std::vector<int64_t> use_off;
    float t_total = 0, t_trace = 0, t_sim = 0, t_tail = 0;
    int64_t queries = -1;
    std::vector<int64_t> host_n;  // replay: trace lengths
    std::vector<int64_t> user_off;  // replay: each trace's offset in the caller's arrays (from offsets[0])
    std::vector<double> cost;     // expected work per scenario (longest-first order, class shares)
    // Multi-device grid: one sub-grid per context member, over contiguous scenario
    // ranges [dev_lo[k], dev_lo[k+1]) (usage slots from dev_use_lo[k]).
    std::vector<std::unique_ptr<msv_grid>> dev_parts;
    std::vector<int64_t> dev_lo, dev_use_lo;

    ~msv_grid() {
        for (cudaEvent_t& e : ev)
            if (e) cudaEventDestroy(e);
    }
};

namespace {

// Reference checks of run()/sample_trace() arguments, in the reference's order:
// sample_trace (workload.hpp:100-101), then run (engine.hpp:118-124, sched.hpp:44-47,
// paris.hpp:141-156), then the lookups the engine would hit (profile.hpp:123-132).
int validate_scenario(const msv_ctx* ctx, const msv_scenario& s, bool generated, int32_t* P_out) {
    if (s.profile < 0 || s.profile >= (int)ctx->profiles.size())
        return fail(MSV_PARAM, "scenario: unknown profile handle " + std::to_string(s.profile));
    if (s.plan < 0 || s.plan >= (int)ctx->plans.size())
        return fail(MSV_PARAM, "scenario: unknown plan handle " + std::to_string(s.plan));
    if (generated) {
        if (s.dist < 0 || s.dist >= (int)ctx->dists.size())
            return fail(MSV_PARAM, "scenario: unknown dist handle " + std::to_string(s.dist));
        if (!(s.rate_qps > 0.0)) return fail(MSV_PARAM, "sample_trace: rate must be > 0");
        if (s.duration_ms < 0.0) return fail(MSV_PARAM, "sample_trace: duration must be >= 0");
    }
    if (s.scheduler != MSV_FIFS && s.scheduler != MSV_ELSA)
        return fail(MSV_VALIDATION, "unknown scheduler " + std::to_string(s.scheduler));
    const Plan& plan = ctx->plans[s.plan];
    if (plan.err) return fail(plan.err, plan.err_msg);
    if (!(s.sla_ms > 0.0)) return fail(MSV_PARAM, "sla: target must be > 0");
    if (s.alpha < 0.0 || s.beta < 0.0) return fail(MSV_PARAM, "sla: alpha/beta must be >= 0");
    if (plan.flat.empty()) return fail(MSV_PARAM, "run: plan has no partition instances");
    if (s.warmup_fraction < 0.0 || s.warmup_fraction >= 1.0)
        return fail(MSV_PARAM, "run: warmup_fraction must be in [0,1)");
    if (s.routing >= 0) {
        if (s.routing >= (int)ctx->routings.size())
            return fail(MSV_PARAM, "scenario: unknown routing handle " + std::to_string(s.routing));
        if (ctx->routings[s.routing].k.empty())
            return fail(MSV_PARAM, "run: segment_routing enabled without segments");
        if (ctx->profiles[s.profile].b_max > 64)
            return fail(MSV_PARAM, "segment routing on the device supports b_max <= 64");
    }
    if ((int)plan.flat.size() > 128)
        return fail(MSV_PARAM, "run: the device engine supports at most 128 partitions per plan");
    // Plan sizes missing from the profile are not an up-front error: like the
    // reference, the engine raises LookupError only if a lookup reaches them.
    *P_out = (int32_t)plan.flat.size();
    return MSV_OK;
}

// by_ascending_size order (sched.hpp:96-104) of the plan's partitions.
std::vector<DevPart> plan_parts(const Plan& plan, const Profile& prof, int cell_off) {
    std::vector<DevPart> parts;
    for (int32_t id = 0; id < (int32_t)plan.flat.size(); ++id) {
        const int32_t k = plan.flat[id];
        const auto it = std::lower_bound(prof.sizes.begin(), prof.sizes.end(), k);
        const int32_t row = (it == prof.sizes.end() || *it != k)
                                ? -1
                                : cell_off + (int32_t)(it - prof.sizes.begin()) * prof.b_max;
        parts.push_back(DevPart{id, k, row, 0});
    }
    std::stable_sort(parts.begin(), parts.end(), [](const DevPart& a, const DevPart& b) {
        if (a.k != b.k) return a.k < b.k;
        return a.pid < b.pid;
    });
    return parts;
}

// Per-partition candidate masks of segment routing (engine.hpp:197-203).
std::vector<uint64_t> route_masks(const std::vector<DevPart>& parts, const Routing& r, int b_max) {
    std::vector<uint64_t> m;
    for (const DevPart& p : parts) {
        uint64_t bits = 0;
        for (int b = 1; b <= b_max && b <= 64; ++b)
            for (size_t j = 0; j < r.k.size(); ++j)
                if (r.k[j] == p.k && b >= r.first[j] && b <= r.last[j]) {
                    bits |= 1ull << (b - 1);
                    break;
                }
        m.push_back(bits);
    }
    return m;
}

// K3's candidate scratch of a scenario: its overflow-link buffer (cap u32 words), dead
// once the simulation kernel is done with the scenario, viewed as 8-byte keys.
void tail_scratch(uint32_t* next, int64_t cap, msv::TailJob& l) {
    const uintptr_t a = ((uintptr_t)next + 7) & ~(uintptr_t)7;
    const int64_t bytes = cap * 4 - (int64_t)(a - (uintptr_t)next);
    l.cand = bytes >= 8 ? reinterpret_cast<uint64_t*>(a) : nullptr;
    l.cand_cap = bytes >= 8 ? bytes / 8 : 0;
}

int64_t trace_capacity(double rate_qps, double duration_ms) {
    const double mean = rate_qps * duration_ms / 1000.0;
    if (!(mean < 2.0e9)) return -1;  // the kernels index a trace with 32-bit ints
    // MSV_TEST_SHORT_CAP=1 (tests only): undersized capacities exercise the re-run path
    static const bool short_cap = getenv("MSV_TEST_SHORT_CAP") && atoi(getenv("MSV_TEST_SHORT_CAP")) != 0;
    if (short_cap) return (int64_t)ceil(0.5 * mean) + 1;
    // a multiple of 32 queries: every scenario's trace then starts on a 256-byte boundary,
    // so the planar latency rows K3 streams are whole 128-byte lines
    const int64_t c = (int64_t)ceil(mean + 10.0 * sqrt(mean) + 160.0);
    return (c + 31) & ~(int64_t)31;
}

// MSV_HOST_TIMING=1: per-phase host timings of grid builds on stderr (diagnostics).
struct PhaseTimer {
    bool on = getenv("MSV_HOST_TIMING") != nullptr;
    std::chrono::steady_clock::time_point t = std::chrono::steady_clock::now();
    std::string line;
    void mark(const char* what) {
        if (!on) return;
        const auto now = std::chrono::steady_clock::now();
        char buf[64];
        snprintf(buf, sizeof buf, " %s %.2f", what, std::chrono::duration<double, std::milli>(now - t).count());
        line += buf;
        t = now;
    }
    ~PhaseTimer() {
        if (on && !line.empty()) fprintf(stderr, "[msv] grid_build ms:%s\n", line.c_str());
    }
};

// Host cores this process may run on (the affinity mask, not the machine's core count).
int host_threads() {
    cpu_set_t set;
    if (sched_getaffinity(0, sizeof set, &set) == 0) return std::max(1, CPU_COUNT(&set));
    return std::max(1, (int)std::thread::hardware_concurrency());
}

// cudaMemGetInfo costs up to ~10 ms on a busy driver; the wave budget only needs a
// coarse figure, so it is refreshed at most once per second per thread — and whenever
// the engine itself allocated or freed device memory since.
size_t free_device_bytes() {
    thread_local size_t fr = 0;
    thread_local int dev = -1;
    thread_local uint64_t epoch = ~0ull;
    thread_local std::chrono::steady_clock::time_point at;
    int cur = 0;
    cudaGetDevice(&cur);
    const auto now = std::chrono::steady_clock::now();
    const uint64_t ep = g_alloc_epoch.load(std::memory_order_relaxed);
    if (cur != dev || ep != epoch || now - at > std::chrono::seconds(1)) {
        size_t tot = 0;
        cudaMemGetInfo(&fr, &tot);
        dev = cur;
        epoch = ep;
        at = now;
    }
    return fr;
}

// Build a grid. generated: traces from K1; otherwise host traces (offsets/arrival/batch).
int grid_build(msv_ctx* ctx, const msv_scenario* sc, int64_t n, const double* tail_p, int n_tails,
               const int64_t* offsets, const double* arrival, const int32_t* batch, bool records,
               msv_grid** out, const int64_t* cap_override = nullptr, bool scratch = false) {
    if (n < 0) return fail(MSV_PARAM, "grid: negative scenario count");
    if (n_tails < 0 || n_tails > 4) return fail(MSV_PARAM, "grid: between 0 and 4 tail percentiles");
    for (int j = 0; j < n_tails; ++j)
        if (!(tail_p[j] > 0.0) || !(tail_p[j] < 1.0))
            return fail(MSV_PARAM, "tail_latency: percentile must be in (0,1)");
    PhaseTimer pt;
    int rc = ctx->sync_tables();
    if (rc) return rc;
    pt.mark("tables");
    std::unique_ptr<msv_grid> g(new msv_grid);
    g->serial = ++ctx->grid_serial;
    g->ctx = ctx;
    if (scratch) g->B = &ctx->scratch;
    g->generated = offsets == nullptr;
    g->records = records;
    g->n = n;
    g->scen.assign(sc, sc + n);
    g->tail_p.assign(tail_p, tail_p + n_tails);
    g->cap.resize(n);
    g->toff.resize(n);
    g->noff.resize(n);
    g->P.resize(n);
    g->usage_off.resize(n);
    for (int64_t i = 0; i < n; ++i) {
        int32_t P = 0;
        rc = validate_scenario(ctx, sc[i], g->generated, &P);
        if (rc) {
            g_err = "scenario " + std::to_string(i) + ": " + g_err;
            return rc;
        }
        g->P[i] = P;
        g->usage_off[i] = (int32_t)g->usage_total;
        g->usage_total += P;
        if (g->generated) {
            g->cap[i] = cap_override ? cap_override[i] : trace_capacity(sc[i].rate_qps, sc[i].duration_ms);
            if (g->cap[i] < 0) return fail(MSV_PARAM, "sample_trace: expected trace too long");
        } else {
            const int64_t len = offsets[i + 1] - offsets[i];
            if (len < 0) return fail(MSV_PARAM, "replay: offsets must be nondecreasing");
            if (len >= (int64_t)0xFFFFFFFFll - 32) return fail(MSV_PARAM, "replay: trace too long");
            // whole 32-query blocks: the one-warp simulation kernel writes the latencies of
            // a block (also a trace's last, partial one) over the block's 256 bytes
            g->cap[i] = (len + 31) & ~(int64_t)31;
            const int b_max = ctx->profiles[sc[i].profile].b_max;
            for (int64_t q = offsets[i]; q < offsets[i + 1]; ++q) {
                if (batch[q] < 1 || batch[q] > b_max)
                    return fail(MSV_LOOKUP, "scenario " + std::to_string(i) + ": profile: batch " +
                                                std::to_string(batch[q]) + " outside grid 1.." +
                                                std::to_string(b_max));
                if (q > offsets[i] && arrival[q] < arrival[q - 1])
                    return fail(MSV_VALIDATION, "scenario " + std::to_string(i) +
                                                    ": replay traces must be sorted by arrival_ms");
            }
        }
    }
    pt.mark("validate");
    // Waves: bound the per-launch trace working set (arrival / measured latency 8 +
    // batch 4 + link 4 [+ record 24] bytes per query slot).
    const size_t per_q = 16 + (records ? sizeof(msv_record) : 0);
    // Keep enough trace slots resident that a wave of 1e6-query scenarios still fills
    // every warp slot of the simulation kernel (~4,100 on a B200). The budget counts the
    // trace buffers this grid will reuse (a one-shot call's scratch set is already held by
    // the context and is not free memory).
    const size_t held = g->B->d_arr.bytes + g->B->d_bat.bytes + g->B->d_next.bytes + g->B->d_rec.bytes;
    static const int frac_pct = getenv("MSV_WAVE_PCT") ? atoi(getenv("MSV_WAVE_PCT")) : 70;  // (A/B)
    static const size_t cap_bytes = (size_t)(getenv("MSV_WAVE_CAP_GIB") ? atoll(getenv("MSV_WAVE_CAP_GIB")) : 140) << 30;
    size_t budget = (free_device_bytes() + held) / 100 * (size_t)frac_pct / (size_t)std::max(1, ctx->share);
    if (budget > cap_bytes) budget = cap_bytes;
    // MSV_TEST_WAVE_MB (tests only): a small budget forces the multi-wave path on small grids
    static const long long test_wave_mb = getenv("MSV_TEST_WAVE_MB") ? atoll(getenv("MSV_TEST_WAVE_MB")) : 0;
    if (test_wave_mb > 0) budget = (size_t)test_wave_mb << 20;
    const int64_t max_q = std::max<int64_t>((int64_t)(budget / per_q), test_wave_mb > 0 ? 1 : (1 << 20));
    // Waves of equal query counts (a short last wave would leave most warp slots idle
    // for one scenario's whole run). A grid that fits runs as one wave. A larger
    // generated grid is cut into waves of at most half the budget that alternate between
    // two buffer regions: wave w + 1 runs while wave w drains (its K1 and K2 blocks take
    // the SMs wave w's finished scenarios free), and wave w + 2 waits only for wave w.
    // Long scenarios first inside each wave (work stealing balances the rest).
    std::vector<int64_t> order(n);
    std::iota(order.begin(), order.end(), 0);
    std::vector<int64_t> wave_q;
    {
        int64_t total_q = 0;
        for (int64_t i = 0; i < n; ++i) total_q += g->cap[i];
        int64_t cap_w = max_q;
        int64_t n_waves = std::max<int64_t>(1, (total_q + max_q - 1) / max_q);
        // MSV_WAVE_REGIONS (A/B): buffer regions the waves rotate through (default 2)
        static const int regions_env = getenv("MSV_WAVE_REGIONS") ? atoi(getenv("MSV_WAVE_REGIONS")) : 2;
        const int regions = std::max(2, std::min(kMaxRegions, regions_env));
        // MSV_INPUT_REGIONS (A/B): the trace inputs (arrival / latency 8 + batch 4 bytes per
        // slot) rotate through more regions than the overflow links (4 bytes), so a wave's K1
        // can run while the waves before it still hold the link regions
        static const int in_env = getenv("MSV_INPUT_REGIONS") ? atoi(getenv("MSV_INPUT_REGIONS")) : regions;
        const int in_regions = std::max(regions, std::min(kMaxRegions / 2, in_env));
        if (n_waves > 1 && g->generated) {
            cap_w = std::max<int64_t>((int64_t)(budget / (size_t)(12 * in_regions + 4 * regions)), 1);
            n_waves = (total_q + cap_w - 1) / cap_w;
        }
        g->n_in_regions = n_waves > 1 && g->generated ? (int)std::min<int64_t>(in_regions, n_waves) : 1;
        const int64_t target = (total_q + n_waves - 1) / n_waves;
        int64_t s0 = 0;
        while (s0 < n) {
            msv_grid::Wave w;
            w.s0 = s0;
            int64_t q = 0;
            int64_t s1 = s0;
            while (s1 < n && (s1 == s0 || (q + g->cap[s1] <= cap_w && q < target))) q += g->cap[s1++];
            w.s1 = s1;
            g->waves.push_back(std::move(w));
            wave_q.push_back(q);
            s0 = s1;
        }
        g->n_regions = g->waves.size() > 1 ? (int)std::min<int64_t>(regions, (int64_t)g->waves.size()) : 1;
        if (g->waves.size() <= 1) g->n_in_regions = 1;
        g->n_in_regions = std::max(g->n_in_regions, g->n_regions);
        for (int64_t q : wave_q) g->max_wave_q = std::max(g->max_wave_q, q);
    }
    pt.mark("waves");
    if (pt.on)
        fprintf(stderr, "[msv] grid n=%lld: %zu wave(s), %lld slots each, budget %.1f GB (free %.1f GB)\n", (long long)n,
                g->waves.size(), (long long)g->max_wave_q, budget / 1e9, free_device_bytes() / 1e9);
    // Expected work per scenario for longest-first scheduling: queries x (1 + 4 rho^2),
    // rho = offered load over the plan's nominal capacity sum_p 1000 / E_b[latency(k_p, b)].
    std::vector<double> cost(n);
    std::vector<char> overloaded(n, 0);  // offered load above the plan's nominal capacity
    {
        std::map<std::tuple<int, int, int>, double> cap_qps;
        for (int64_t i = 0; i < n; ++i) {
            if (!g->generated) {
                cost[i] = (double)g->cap[i];
                continue;
            }
            const msv_scenario& s = sc[i];
            auto key = std::make_tuple(s.plan, s.profile, s.dist);
            auto it = cap_qps.find(key);
            if (it == cap_qps.end()) {
                const Profile& pr = ctx->profiles[s.profile];
                const Dist& ds = ctx->dists[s.dist];
                double c = 0.0;
                for (int32_t k : ctx->plans[s.plan].flat) {
                    const auto kt = std::lower_bound(pr.sizes.begin(), pr.sizes.end(), k);
                    if (kt == pr.sizes.end() || *kt != k) continue;
                    const size_t r0 = (size_t)(kt - pr.sizes.begin()) * pr.b_max;
                    double e = 0.0;
                    for (size_t b = 0; b < ds.pmf.size() && b < (size_t)pr.b_max; ++b) e += ds.pmf[b] * pr.lat[r0 + b];
                    if (e > 0.0) c += 1000.0 / e;
                }
                it = cap_qps.emplace(key, c).first;
            }
            const double rho = it->second > 0.0 ? s.rate_qps / it->second : 1.0;
            overloaded[i] = rho > 1.0;
            cost[i] = (s.rate_qps * s.duration_ms / 1000.0) * (1.0 + 4.0 * rho * rho);
        }
    }
    // MSV_TRACE_GROUP=0: one K1 warp per trace (no shared random streams), for A/B runs
    static const bool group_traces = !(getenv("MSV_TRACE_GROUP") && atoi(getenv("MSV_TRACE_GROUP")) == 0);
    static const int group_max = getenv("MSV_TRACE_GROUP_MAX")
                                     ? std::max(1, std::min(msv::kTraceGroupMax, atoi(getenv("MSV_TRACE_GROUP_MAX"))))
                                     : msv::kTraceGroupMax;
    static const int group_first = getenv("MSV_TRACE_GROUP_FIRST")
                                       ? std::max(1, std::min(msv::kTraceGroupMax, atoi(getenv("MSV_TRACE_GROUP_FIRST"))))
                                       : 2;
    for (size_t wi = 0; wi < g->waves.size(); ++wi) {
        msv_grid::Wave& w = g->waves[wi];
        w.q0 = (int64_t)(wi % g->n_in_regions) * g->max_wave_q;  // the wave's input region
        const int64_t n0 = (int64_t)(wi % g->n_regions) * g->max_wave_q;  // and link region
        int64_t q = w.q0;
        for (int64_t i = w.s0; i < w.s1; ++i) {
            g->toff[i] = q;  // offset inside the trace buffers
            g->noff[i] = n0 + (q - w.q0);
            q += g->cap[i];
        }
        w.q1 = q;
        // Deal the wave's scenarios, most expensive first, round-robin into chunks.
        std::vector<int32_t> ord;
        for (int64_t i = w.s0; i < w.s1; ++i) ord.push_back((int32_t)i);
        std::stable_sort(ord.begin(), ord.end(), [&](int32_t a, int32_t b) { return cost[a] > cost[b]; });
        const int64_t ns_w = w.s1 - w.s0;
        int64_t n4 = 0, n8 = 0, n16 = 0;
        for (int64_t i = w.s0; i < w.s1; ++i) {
            n4 += g->P[i] <= 4;
            n8 += g->P[i] <= 8;
            n16 += g->P[i] <= 16;
        }
        const int seg_w = wave_seg_width(n4, n8, n16, ctx->sms);
        // Chunks pay only when the wave fills the device for about two rounds of the warp
        // kernel's slots (28 warps per SM): then the big first chunk's simulation hides the
        // small chunks' trace generation, and their simulations and tail selections fill
        // its last round. Smaller waves run as one chunk (a half-full launch costs more
        // than the overlap). Shares 2:1:1:1 on four streams (sweep on the C2 grid: 3:1 on
        // two streams -1.4 %, one chunk -7 %). MSV_MAX_CHUNKS / MSV_CHUNK_SPLIT override.
        const int64_t warp_slots = (int64_t)ctx->sms * 28;
        int64_t warps_w = 0;  // warps the wave occupies (segmented classes pack 32/W scenarios)
        for (int64_t i = w.s0; i < w.s1; ++i) warps_w += class_of(g->P[i], sc[i].scheduler, seg_w).W;
        warps_w /= 32;
        std::vector<double> share;
        if (warps_w >= 2 * warp_slots && ns_w >= 4 * kChunkScenarios) share = {2.0, 1.0, 1.0, 1.0};
        else share = {1.0};
        if (const char* e = getenv("MSV_MAX_CHUNKS")) {
            const int mc = std::max(1, std::min(kMaxChunks, atoi(e)));
            const int nc = (int)std::max<int64_t>(1, std::min<int64_t>(mc, ns_w / kChunkScenarios));
            share.assign(nc, 1.0);
        }
        if (const char* e = getenv("MSV_CHUNK_SPLIT")) {
            std::vector<double> f;
            for (const char* c = e; *c;) {
                char* end = nullptr;
                const double v = strtod(c, &end);
                if (end == c) break;
                if (v > 0) f.push_back(v);
                c = (*end == ',') ? end + 1 : end;
            }
            if (!f.empty() && (int)f.size() <= kMaxChunks && (int64_t)f.size() <= ns_w) share = f;
        }
        const int n_chunks = (int)share.size();
        double share_sum = 0.0;
        for (double v : share) share_sum += v;
        // K1 groups: scenarios with the same seed and batch distribution draw the same
        // random stream (sample_trace's draws do not depend on the rate), so one K1 warp
        // generates up to kTraceGroupMax of their traces. Groups stay whole inside a chunk
        // and are dealt in cost order of their first member. A group's warp is latency-
        // bound (fewer, longer warps), so grouping pays where K1 overlaps other chunks'
        // simulation: chunked waves only, and the first chunk (which nothing overlaps) in
        // pairs (C2 bench grid, B200: one warp per trace 8.42, groups of <= 16 8.79, first
        // chunk in pairs 8.95 G queries/s).
        std::vector<std::vector<int32_t>> groups;
        {
            std::map<std::pair<uint64_t, int32_t>, size_t> open;
            for (int32_t i : ord) {
                const double rpm = sc[i].rate_qps / 1000.0;  // the grouped quotient needs a normal range
                // grouping pays where K1 overlaps other simulation: chunked waves (measured
                // on the overlapping waves of C5 too: K1 166 -> 345 ms staged, e2e -5 %)
                if (!group_traces || !g->generated || n_chunks < 2 || !(rpm >= 0x1p-600 && rpm <= 0x1p600)) {
                    groups.push_back({i});
                    continue;
                }
                const std::pair<uint64_t, int32_t> key(sc[i].seed, sc[i].dist);
                auto it = open.find(key);
                if (it == open.end() || groups[it->second].size() >= (size_t)group_max) {
                    open[key] = groups.size();
                    groups.push_back({});
                    it = open.find(key);
                }
                groups[it->second].push_back(i);
            }
        }
        // proportional interleave in cost order: each group goes to the chunk furthest
        // below its share (equal shares: round robin)
        std::vector<std::vector<int32_t>> members(n_chunks);
        std::vector<std::vector<std::pair<int32_t, int32_t>>> cgroups(n_chunks);  // (offset, count) in members
        int64_t dealt = 0;
        for (const std::vector<int32_t>& grp : groups) {
            dealt += (int64_t)grp.size();
            int best = 0;
            double best_def = -1e300;
            for (int c = 0; c < n_chunks; ++c) {
                const double def = share[c] / share_sum * (double)dealt - (double)members[c].size();
                if (def > best_def + 1e-12) {
                    best_def = def;
                    best = c;
                }
            }
            cgroups[best].emplace_back((int32_t)members[best].size(), (int32_t)grp.size());
            members[best].insert(members[best].end(), grp.begin(), grp.end());
        }
        for (int c = 0; c < n_chunks; ++c) {
            msv_grid::Chunk ch;
            ch.l0 = (int64_t)g->launch_order.size();
            g->launch_order.insert(g->launch_order.end(), members[c].begin(), members[c].end());
            ch.l1 = (int64_t)g->launch_order.size();
            ch.g0 = (int64_t)g->tgroups.size();
            const int cap_c = (c == 0 && n_chunks > 1) ? group_first : group_max;
            for (const auto& og : cgroups[c])
                for (int32_t o = 0; o < og.second; o += cap_c)
                    g->tgroups.push_back({(int32_t)(ch.l0 + og.first + o), std::min(cap_c, og.second - o)});
            ch.g1 = (int64_t)g->tgroups.size();
            std::vector<int32_t> by_cost = members[c];  // kernel classes keep longest-first order
            std::stable_sort(by_cost.begin(), by_cost.end(), [&](int32_t a, int32_t b) { return cost[a] > cost[b]; });
            std::map<ClassKey, std::vector<int32_t>> cls;
            for (int32_t i : by_cost) cls[class_of(g->P[i], sc[i].scheduler, seg_w, overloaded[i])].push_back(i);
            for (auto& kv : cls) ch.classes.emplace_back(kv.first, std::move(kv.second));
            w.chunks.push_back(std::move(ch));
        }
    }
    g->cost = cost;
    pt.mark("cost+chunks");
    // Device buffers.
    const size_t wq = (size_t)std::max<int64_t>(g->max_wave_q * g->n_in_regions, 1);
    const size_t wn = (size_t)std::max<int64_t>(g->max_wave_q * g->n_regions, 1);
    MSV_CUDA_TRY(g->B->d_arr.ensure(wq * 8));
    MSV_CUDA_TRY(g->B->d_bat.ensure(wq * 4));
    MSV_CUDA_TRY(g->B->d_next.ensure(wn * 4));
    if (records) MSV_CUDA_TRY(g->B->d_rec.ensure(wq * sizeof(msv_record)));
    MSV_CUDA_TRY(g->B->d_scen.ensure(std::max<int64_t>(n, 1) * sizeof(DevScen)));
    MSV_CUDA_TRY(g->B->d_out.ensure(std::max<int64_t>(n, 1) * sizeof(DevOut)));
    MSV_CUDA_TRY(g->B->d_tjobs.ensure(std::max<int64_t>(n, 1) * sizeof(msv::TraceJob)));
    MSV_CUDA_TRY(g->B->d_tailjobs.ensure(std::max<int64_t>(n, 1) * sizeof(msv::TailJob)));
    MSV_CUDA_TRY(g->B->d_tails.ensure(std::max<int64_t>(n, 1) * 4 * sizeof(double)));
    MSV_CUDA_TRY(g->B->d_p.ensure(4 * sizeof(double)));
    MSV_CUDA_TRY(g->B->d_usage.ensure(std::max<int64_t>(g->usage_total, 1) * sizeof(msv_usage)));
    MSV_CUDA_TRY(g->B->d_nq.ensure(std::max<int64_t>(n, 1) * 8));
    MSV_CUDA_TRY(g->B->d_tovf.ensure(std::max<int64_t>(n, 1) * 4));
    MSV_CUDA_TRY(g->B->d_counter.ensure(kCounterSlots * sizeof(int32_t)));
    if (n_tails) MSV_CUDA_TRY(cudaMemcpy(g->B->d_p.p, tail_p, n_tails * sizeof(double), cudaMemcpyHostToDevice));

    pt.mark("ensure");
    // Compact profile table of this grid (staged in shared memory by the kernel).
    std::map<int, int> grid_cell_off;
    std::vector<double> glat, gutil;
    for (int64_t i = 0; i < n; ++i) {
        if (grid_cell_off.count(sc[i].profile)) continue;
        const Profile& pr = ctx->profiles[sc[i].profile];
        grid_cell_off[sc[i].profile] = (int)glat.size();
        glat.insert(glat.end(), pr.lat.begin(), pr.lat.end());
        gutil.insert(gutil.end(), pr.util.begin(), pr.util.end());
    }
    if ((int)glat.size() > msv::kMaxSmemCells)
        return fail(MSV_PARAM, "grid: profiles of one call exceed the device table capacity (" +
                                   std::to_string(msv::kMaxSmemCells) + " cells)");
    g->n_cells = (int)glat.size();
    MSV_CUDA_TRY(g->B->d_glat.ensure(std::max<size_t>(glat.size(), 1) * 8));
    MSV_CUDA_TRY(g->B->d_gutil.ensure(std::max<size_t>(gutil.size(), 1) * 8));
    if (!glat.empty()) {
        MSV_CUDA_TRY(cudaMemcpy(g->B->d_glat.p, glat.data(), glat.size() * 8, cudaMemcpyHostToDevice));
        MSV_CUDA_TRY(cudaMemcpy(g->B->d_gutil.p, gutil.data(), gutil.size() * 8, cudaMemcpyHostToDevice));
    }
    // The grid's own copy of its batch distributions (cdf + guide): the context's tables
    // are re-laid out (and may move) when later calls upload more distributions.
    std::map<int, std::pair<size_t, size_t>> grid_dist_off;  // dist -> (cdf offset, guide offset)
    if (g->generated) {
        std::vector<double> gcdf;
        std::vector<int16_t> gguide;
        for (int64_t i = 0; i < n; ++i) {
            if (grid_dist_off.count(sc[i].dist)) continue;
            const std::vector<double>& cdf = ctx->dists[sc[i].dist].cdf;
            grid_dist_off[sc[i].dist] = {gcdf.size(), gguide.size()};
            gcdf.insert(gcdf.end(), cdf.begin(), cdf.end());
            append_guide(cdf, gguide);
        }
        MSV_CUDA_TRY(g->B->d_gcdf.ensure(std::max<size_t>(gcdf.size(), 1) * 8));
        MSV_CUDA_TRY(g->B->d_gguide.ensure(std::max<size_t>(gguide.size(), 1) * 2));
        if (!gcdf.empty())
            MSV_CUDA_TRY(cudaMemcpy(g->B->d_gcdf.p, gcdf.data(), gcdf.size() * 8, cudaMemcpyHostToDevice));
        if (!gguide.empty())
            MSV_CUDA_TRY(cudaMemcpy(g->B->d_gguide.p, gguide.data(), gguide.size() * 2, cudaMemcpyHostToDevice));
        ctx->h2d += (int64_t)(gcdf.size() * 8 + gguide.size() * 2);
    }
    // Partition tables per (plan, profile) and routing masks per (plan, profile, routing).
    std::map<std::pair<int, int>, size_t> part_off;
    std::map<std::tuple<int, int, int>, size_t> mask_off;
    std::vector<DevPart> parts_h;
    std::vector<uint64_t> masks_h;
    std::vector<size_t> sc_part(n), sc_mask(n, (size_t)-1);
    g->bad.assign(n, 0);
    for (int64_t i = 0; i < n; ++i) {
        auto key = std::make_pair(sc[i].plan, sc[i].profile);
        auto it = part_off.find(key);
        if (it == part_off.end()) {
            std::vector<DevPart> pp =
                plan_parts(ctx->plans[sc[i].plan], ctx->profiles[sc[i].profile], grid_cell_off[sc[i].profile]);
            it = part_off.emplace(key, parts_h.size()).first;
            parts_h.insert(parts_h.end(), pp.begin(), pp.end());
        }
        sc_part[i] = it->second;
        for (int32_t j = 0; j < g->P[i]; ++j)
            if (parts_h[it->second + j].row < 0) g->bad[i] = 1;
        // generated batches can exceed the profile's b_max only when the distribution's
        // support is wider; such scenarios take the FULL kernel variant, which checks
        // every batch (replay batches were validated above)
        if (g->generated && (int)ctx->dists[sc[i].dist].cdf.size() > ctx->profiles[sc[i].profile].b_max)
            g->bad[i] = 1;
        if (sc[i].routing >= 0) {
            auto mk = std::make_tuple(sc[i].plan, sc[i].profile, sc[i].routing);
            auto mt = mask_off.find(mk);
            if (mt == mask_off.end()) {
                std::vector<DevPart> pp(parts_h.begin() + it->second, parts_h.begin() + it->second + g->P[i]);
                std::vector<uint64_t> mm =
                    route_masks(pp, ctx->routings[sc[i].routing], ctx->profiles[sc[i].profile].b_max);
                mt = mask_off.emplace(mk, masks_h.size()).first;
                masks_h.insert(masks_h.end(), mm.begin(), mm.end());
            }
            sc_mask[i] = mt->second;
        }
    }
    MSV_CUDA_TRY(g->B->d_parts.ensure(std::max<size_t>(parts_h.size(), 1) * sizeof(DevPart)));
    MSV_CUDA_TRY(g->B->d_masks.ensure(std::max<size_t>(masks_h.size(), 1) * 8));
    if (!parts_h.empty())
        MSV_CUDA_TRY(cudaMemcpy(g->B->d_parts.p, parts_h.data(), parts_h.size() * sizeof(DevPart), cudaMemcpyHostToDevice));
    if (!masks_h.empty())
        MSV_CUDA_TRY(cudaMemcpy(g->B->d_masks.p, masks_h.data(), masks_h.size() * 8, cudaMemcpyHostToDevice));

    pt.mark("parts");
    // Per-scenario device descriptors.
    // every latency >= its service time >= the profile's smallest cell (halved: rounding slack)
    std::vector<double> lat_floor(ctx->profiles.size(), 0.0);
    for (size_t pi = 0; pi < ctx->profiles.size(); ++pi) {
        double mn = INFINITY;
        for (double v : ctx->profiles[pi].lat) mn = v < mn ? v : mn;
        lat_floor[pi] = (mn > 0.0 && mn < INFINITY) ? 0.5 * mn : 0.0;
    }
    g->h_scen.resize(n);
    std::vector<msv::TraceJob> tj(n);
    std::vector<msv::TailJob> lj(n);
    for (int64_t i = 0; i < n; ++i) {
        const msv_scenario& s = sc[i];
        const Profile& prof = ctx->profiles[s.profile];
        DevScen& d = g->h_scen[i];
        const int64_t o = g->toff[i];
        d.arrival = g->B->d_arr.as<double>() + o;
        d.batch = g->B->d_bat.as<int32_t>() + o;
        d.n = g->B->d_nq.as<int64_t>() + i;
        d.duration_ms = s.duration_ms;
        d.lat_floor = lat_floor[s.profile];
        d.warmup_ms = s.warmup_fraction * s.duration_ms;  // engine.hpp:238
        d.sla = s.sla_ms;
        d.alpha = s.alpha;
        d.beta = s.beta;
        d.parts = g->B->d_parts.as<DevPart>() + sc_part[i];
        d.route_mask = (sc_mask[i] == (size_t)-1) ? nullptr : g->B->d_masks.as<uint64_t>() + sc_mask[i];
        d.next = g->B->d_next.as<uint32_t>() + g->noff[i];
        d.samples = g->B->d_arr.as<double>() + o;  // latencies overwrite their own (dead) arrivals
        d.records = records ? g->B->d_rec.as<msv_record>() + o : nullptr;
        d.P = g->P[i];
        d.b_max = prof.b_max;
        d.sched = s.scheduler;
        d.flags = s.flags;
        d.usage_off = g->usage_off[i];
        d.pad = 0;
        msv::TraceJob& t = tj[i];
        t.seed = s.seed;
        t.rate_per_ms = s.rate_qps / 1000.0;  // workload.hpp:103
        t.duration_ms = s.duration_ms;
        t.cdf = g->generated ? g->B->d_gcdf.as<double>() + grid_dist_off[s.dist].first : nullptr;
        t.guide = g->generated ? g->B->d_gguide.as<int16_t>() + grid_dist_off[s.dist].second : nullptr;
        t.b_max = g->generated ? (int32_t)ctx->dists[s.dist].cdf.size() : 0;
        t.pad = 0;
        t.arrival = g->B->d_arr.as<double>() + o;
        t.batch = g->B->d_bat.as<int32_t>() + o;
        t.cap = g->cap[i];
        t.n_out = g->B->d_nq.as<int64_t>() + i;
        t.overflow = g->B->d_tovf.as<int32_t>() + i;
        msv::TailJob& l = lj[i];
        l.samples = d.samples;
        l.src = g->B->d_out.as<DevOut>() + i;
        l.out = g->B->d_tails.as<double>() + 4 * i;
        tail_scratch(d.next, g->cap[i], l);
    }
    ctx->h2d += (int64_t)(n * (sizeof(DevScen) + sizeof(msv::TraceJob) + sizeof(msv::TailJob)) +
                          parts_h.size() * sizeof(DevPart) + masks_h.size() * 8 + glat.size() * 16 +
                          n_tails * sizeof(double));
    if (n) {
        std::vector<msv::TraceJob> tj_l(n);
        std::vector<msv::TailJob> lj_l(n);
        for (int64_t l = 0; l < n; ++l) {
            tj_l[l] = tj[g->launch_order[l]];
            lj_l[l] = lj[g->launch_order[l]];
        }
        MSV_CUDA_TRY(cudaMemcpy(g->B->d_scen.p, g->h_scen.data(), n * sizeof(DevScen), cudaMemcpyHostToDevice));
        MSV_CUDA_TRY(cudaMemcpy(g->B->d_tjobs.p, tj_l.data(), n * sizeof(msv::TraceJob), cudaMemcpyHostToDevice));
        MSV_CUDA_TRY(cudaMemcpy(g->B->d_tailjobs.p, lj_l.data(), n * sizeof(msv::TailJob), cudaMemcpyHostToDevice));
        MSV_CUDA_TRY(cudaMemset(g->B->d_tovf.p, 0, n * 4));
    }
    // streamed launches: latency-bound (at most two scenarios per SM) single-wave grids
    // MSV_STREAM=0 never streams, MSV_STREAM=1 streams every eligible grid (tests)
    static const int stream_env = getenv("MSV_STREAM") ? atoi(getenv("MSV_STREAM")) : -1;
    g->stream_ok = stream_env != 0 && g->generated && n > 0 && g->waves.size() == 1 &&
                   (stream_env == 1 || n <= 2 * (int64_t)ctx->sms);
    for (int64_t i = 0; i < n && g->stream_ok; ++i)
        if (g->bad[i] || sc[i].routing >= 0 || (sc[i].flags & MSV_FLAG_CHECK_WAIT)) g->stream_ok = false;
    for (const auto& w : g->waves)
        for (const auto& ch : w.chunks)
            for (const auto& c : ch.classes)
                if (c.first.W != 32) g->stream_ok = false;
    if (g->stream_ok) {  // trace jobs in scenario order (a block finds its job by scenario index)
        MSV_CUDA_TRY(g->B->d_sjobs.ensure(n * sizeof(msv::TraceJob)));
        MSV_CUDA_TRY(cudaMemcpy(g->B->d_sjobs.p, tj.data(), n * sizeof(msv::TraceJob), cudaMemcpyHostToDevice));
    }
    MSV_CUDA_TRY(g->B->d_tgroups.ensure(std::max<size_t>(g->tgroups.size(), 1) * sizeof(msv::TraceGroup)));
    if (!g->tgroups.empty())
        MSV_CUDA_TRY(cudaMemcpy(g->B->d_tgroups.p, g->tgroups.data(), g->tgroups.size() * sizeof(msv::TraceGroup),
                                cudaMemcpyHostToDevice));
    ctx->h2d += (int64_t)(g->tgroups.size() * sizeof(msv::TraceGroup));
    pt.mark("descriptors");
    // Work lists of every (wave, chunk, class).
    std::vector<int32_t> work_h;
    for (msv_grid::Wave& w : g->waves)
        for (msv_grid::Chunk& ch : w.chunks)
            for (auto& c : ch.classes) {
                ch.work_off.push_back((int64_t)work_h.size());
                work_h.insert(work_h.end(), c.second.begin(), c.second.end());
            }
    MSV_CUDA_TRY(g->B->d_work.ensure(std::max<size_t>(work_h.size(), 1) * 4));
    if (!work_h.empty())
        MSV_CUDA_TRY(cudaMemcpy(g->B->d_work.p, work_h.data(), work_h.size() * 4, cudaMemcpyHostToDevice));
    ctx->h2d += (int64_t)(work_h.size() * 4);
    if (!g->generated) {
        // Host traces stay resident: replay grids are a single wave.
        if (g->waves.size() > 1) return fail(MSV_PARAM, "replay: traces exceed device memory budget");
        g->host_n.resize(n);
        g->user_off.resize(n);
        const int64_t q0 = n ? offsets[0] : 0;
        int64_t slots = 0;
        for (int64_t i = 0; i < n; ++i) {
            g->host_n[i] = offsets[i + 1] - offsets[i];
            g->user_off[i] = offsets[i] - q0;
            slots = std::max(slots, g->toff[i] + g->cap[i]);
        }
        if (slots) {  // each trace at its (32-aligned) slot offset
            std::vector<double> pa(slots, 0.0);
            std::vector<int32_t> pb(slots, 1);
            for (int64_t i = 0; i < n; ++i) {
                std::copy(arrival + offsets[i], arrival + offsets[i + 1], pa.begin() + g->toff[i]);
                std::copy(batch + offsets[i], batch + offsets[i + 1], pb.begin() + g->toff[i]);
            }
            MSV_CUDA_TRY(cudaMemcpy(g->B->d_arr.p, pa.data(), slots * 8, cudaMemcpyHostToDevice));
            MSV_CUDA_TRY(cudaMemcpy(g->B->d_bat.p, pb.data(), slots * 4, cudaMemcpyHostToDevice));
        }
        if (n) MSV_CUDA_TRY(cudaMemcpy(g->B->d_nq.p, g->host_n.data(), n * 8, cudaMemcpyHostToDevice));
    }
    for (cudaEvent_t& e : g->ev) MSV_CUDA_TRY(cudaEventCreate(&e));
    pt.mark("work+events");
    *out = g.release();
    return MSV_OK;
}

// MSV_DEBUG_SYNC=1: synchronise and report after every kernel (diagnostics only).
void debug_sync(cudaStream_t st, const char* what) {
    static const bool on = getenv("MSV_DEBUG_SYNC") != nullptr;
    if (!on) return;
    cudaError_t e = cudaStreamSynchronize(st);
    fprintf(stderr, "[msv] %s done: %s\n", what, cudaGetErrorString(e));
}

// MSV_TIMELINE=1 (diagnostics): events around every chunk's stages; grid_launch prints
// them relative to the launch's start once it completes (synchronising: not for timing runs).
struct TimelineMark {
    std::string what;
    cudaEvent_t ev;
};
static std::vector<TimelineMark> g_timeline;
static std::mutex g_timeline_mu;  // contexts on several threads may launch at once
static bool timeline_on() {
    static const bool on = getenv("MSV_TIMELINE") != nullptr;
    return on;
}
static void timeline_mark(const std::string& what, cudaStream_t st) {
    if (!timeline_on()) return;
    cudaEvent_t e;
    if (cudaEventCreate(&e) != cudaSuccess) return;
    cudaEventRecord(e, st);
    std::lock_guard<std::mutex> lk(g_timeline_mu);
    g_timeline.push_back({what, e});
}
static void timeline_print(cudaEvent_t start) {
    if (!timeline_on()) return;
    std::lock_guard<std::mutex> lk(g_timeline_mu);
    if (g_timeline.empty()) return;
    cudaDeviceSynchronize();
    for (const TimelineMark& m : g_timeline) {
        float ms = 0;
        cudaEventElapsedTime(&ms, start, m.ev);
        fprintf(stderr, "[msv] timeline %9.2f ms %s\n", ms, m.what.c_str());
        cudaEventDestroy(m.ev);
    }
    g_timeline.clear();
}

// Launch one chunk's K1 -> K2 (per class) -> K3 on `st`. Stage events (optional) bracket
// the three stages when the launch is not overlapped.
int launch_chunk(msv_grid* g, const msv_grid::Chunk& ch, int counter_base, cudaStream_t st, cudaEvent_t e1,
                 cudaEvent_t e2, cudaEvent_t k2_wait = nullptr) {
    msv_ctx* ctx = g->ctx;
    const int64_t nl = ch.l1 - ch.l0;
    const bool stream = g->stream_ok && !g->records && !g->usage;  // K1 inside K2's blocks
    static const bool stream_pregen = getenv("MSV_STREAM_PREGEN") != nullptr;  // A/B: K1 first anyway
    const std::string tag = "chunk l" + std::to_string(ch.l0) + "-" + std::to_string(ch.l1);
    timeline_mark(tag + " start", st);
    if (g->generated && nl > 0 && (!stream || stream_pregen)) {
        if (ch.g1 - ch.g0 == nl)  // no shared streams in this chunk: one warp per trace
            MSV_CUDA_TRY(msv::launch_trace_gen(g->B->d_tjobs.as<msv::TraceJob>() + ch.l0, (int)nl, ctx->log1p, st));
        else
            MSV_CUDA_TRY(msv::launch_trace_groups(g->B->d_tjobs.as<msv::TraceJob>(),
                                                  g->B->d_tgroups.as<msv::TraceGroup>() + ch.g0, (int)(ch.g1 - ch.g0),
                                                  ctx->log1p, st));
        debug_sync(st, "trace_gen");
        ctx->launches += 1;
    }
    if (e1) MSV_CUDA_TRY(cudaEventRecord(e1, st));
    timeline_mark(tag + " K1 done", st);
    if (k2_wait) MSV_CUDA_TRY(cudaStreamWaitEvent(st, k2_wait, 0));  // the link region is free
    // A chunk's kernel classes are independent: the largest runs on the chunk stream, the
    // others on class streams forked after K1, so their blocks fill the largest one's
    // last round instead of each class launch ending in its own tail.
    const size_t ncls = ch.classes.size();
    static const bool class_streams = !(getenv("MSV_CLASS_STREAMS") && atoi(getenv("MSV_CLASS_STREAMS")) == 0);
    const bool par = class_streams && ncls > 1;
    std::vector<size_t> corder(ncls);
    for (size_t c = 0; c < ncls; ++c) corder[c] = c;
    // Classes with the slowest scenarios (more partitions per lane) launch first, so their
    // blocks are resident from the start instead of waiting for the largest class's
    // persistent blocks to drain, and the slowest scenarios do not form the tail (C5:
    // +3 % device-resident and end to end). MSV_CLASS_ORDER=count: largest class first (A/B).
    static const bool slow_first = !(getenv("MSV_CLASS_ORDER") && std::string(getenv("MSV_CLASS_ORDER")) == "count");
    std::stable_sort(corder.begin(), corder.end(), [&](size_t a, size_t b) {
        const ClassKey &ka = ch.classes[a].first, &kb = ch.classes[b].first;
        if (slow_first && ka.S != kb.S) return ka.S > kb.S;  // slots per lane: per-arrival cost
        return ch.classes[a].second.size() > ch.classes[b].second.size();
    });
    if (par) {
        for (int a = 0; a < 4; ++a) {
            if (!ctx->cls[a]) MSV_CUDA_TRY(cudaStreamCreateWithFlags(&ctx->cls[a], cudaStreamNonBlocking));
            if (!ctx->cls_ev[a]) MSV_CUDA_TRY(cudaEventCreateWithFlags(&ctx->cls_ev[a], cudaEventDisableTiming));
        }
        if (!ctx->cls_fork) MSV_CUDA_TRY(cudaEventCreateWithFlags(&ctx->cls_fork, cudaEventDisableTiming));
        MSV_CUDA_TRY(cudaEventRecord(ctx->cls_fork, st));
    }
    // Optionally, concurrent classes share the device in proportion to their expected time
    // on it (expected work / the class's relative throughput), to run side by side and end
    // together in one tail instead of one after another.
    // Off by default — measured slower on C5 (5.20 vs 5.85 G q/s on a B200): every class
    // launches full-device persistent grids instead, the largest holds the SMs and the
    // others fill its last round. MSV_CLASS_SHARES=1 turns the shares on (A/B runs).
    static const bool class_shares = getenv("MSV_CLASS_SHARES") && atoi(getenv("MSV_CLASS_SHARES")) != 0;
    std::vector<double> share(ncls, 1.0);
    if (par && class_shares) {
        double tot = 0.0;
        for (size_t c = 0; c < ncls; ++c) {
            const ClassKey& k = ch.classes[c].first;
            // relative throughput of a full device of this class (B200, C5 plans: warp kernel
            // 1 slot ~9 G q/s, 2 slots ~5.1, 4 slots ~2.5, segmented W=8 ~12, W=4 ~15)
            const double rel = k.W == 4 ? 1.6 : k.W == 8 ? 1.33 : k.W == 16 ? 1.0 : k.S == 1 ? 1.0 : k.S == 2 ? 0.57 : 0.28;
            double w = 0.0;
            for (int32_t si : ch.classes[c].second) w += g->cost.empty() ? 1.0 : g->cost[si];
            share[c] = w / rel;
            tot += share[c];
        }
        for (double& v : share) v = tot > 0.0 ? v / tot : 1.0;
    }
    for (size_t ci = 0; ci < ncls; ++ci) {
        const size_t c = corder[ci];
        cudaStream_t cs = (par && ci > 0) ? ctx->cls[(ci - 1) % 4] : st;
        if (par && ci > 0) MSV_CUDA_TRY(cudaStreamWaitEvent(cs, ctx->cls_fork, 0));
        const ClassKey& k = ch.classes[c].first;
        const int32_t nwork = (int32_t)ch.classes[c].second.size();
        msv::SimParams p;
        p.scen = g->B->d_scen.as<DevScen>();
        p.out = g->B->d_out.as<DevOut>();
        p.usage = g->B->d_usage.as<msv_usage>();
        p.work = g->B->d_work.as<int32_t>() + ch.work_off[c];
        p.n_work = nwork;
        p.counter = g->B->d_counter.as<int32_t>() + ((counter_base + (int)c) % kCounterSlots);
        p.lat = g->B->d_glat.as<double>();
        p.util = g->B->d_gutil.as<double>();
        p.n_cells = g->n_cells;
        p.any_routing = p.any_bad = p.any_check_wait = 0;
        p.any_usage = g->usage ? 1 : 0;
        for (int32_t si : ch.classes[c].second) {
            if (g->scen[si].routing >= 0) p.any_routing = 1;
            if (g->bad[si]) p.any_bad = 1;
            if (g->scen[si].flags & MSV_FLAG_CHECK_WAIT) p.any_check_wait = 1;
        }
        const bool full = g->records || p.any_routing || p.any_bad || p.any_check_wait || p.any_usage;
        p.lazy = k.lazy;
        p.stream = stream ? (stream_pregen ? 2 : 1) : 0;
        p.log1p_variant = ctx->log1p;
        p.stream_jobs = stream ? g->B->d_sjobs.as<msv::TraceJob>() : nullptr;
        const int occ = msv::sim_max_blocks_per_sm(k.W, k.S, k.sched, g->records, full, k.lazy != 0, g->n_cells);
        if (occ <= 0) return fail(MSV_CUDA, "sim kernel: no occupancy for class");
        const int segs_per_block = msv::kSimWarpsPerBlock * (32 / k.W);
        const int need = (nwork + segs_per_block - 1) / segs_per_block;
        int occ_used = occ;
        if (const char* e = getenv("MSV_SIM_BLOCK_SLACK")) occ_used = std::max(1, occ - atoi(e));
        // MSV_MULTI_SLOT_BLOCKS (A/B): blocks per SM of the multi-slot classes' persistent grids
        static const int ms_blocks = getenv("MSV_MULTI_SLOT_BLOCKS") ? atoi(getenv("MSV_MULTI_SLOT_BLOCKS")) : 0;
        if (ms_blocks > 0 && k.S > 1 && k.W == 32) occ_used = std::min(occ_used, ms_blocks);
        const int dev_blocks = std::max(1, (int)std::lround(share[c] * occ_used * ctx->sms));
        const int blocks = std::max(1, std::min(need, dev_blocks));
        MSV_CUDA_TRY(msv::launch_sim(k.W, k.S, k.sched, g->records, p, blocks, cs));
        debug_sync(cs, "sim");
        ctx->launches += 1;
    }
    if (par) {  // join the class streams back into the chunk stream
        for (size_t ci = 1; ci < ncls && ci <= 4; ++ci) {
            MSV_CUDA_TRY(cudaEventRecord(ctx->cls_ev[ci - 1], ctx->cls[ci - 1]));
            MSV_CUDA_TRY(cudaStreamWaitEvent(st, ctx->cls_ev[ci - 1], 0));
        }
    }
    if (e2) MSV_CUDA_TRY(cudaEventRecord(e2, st));
    timeline_mark(tag + " K2 done", st);
    if (!g->tail_p.empty() && nl > 0) {
        MSV_CUDA_TRY(msv::launch_tail(g->B->d_tailjobs.as<msv::TailJob>() + ch.l0, (int)nl, g->B->d_p.as<double>(),
                                      (int)g->tail_p.size(), st));
        debug_sync(st, "tail");
        ctx->launches += 1;
    }
    timeline_mark(tag + " K3 done", st);
    return MSV_OK;
}

int grid_launch(msv_grid* g) {
    msv_ctx* ctx = g->ctx;
    cudaStream_t st = ctx->stream;
    int rc;
    MSV_CUDA_TRY(cudaEventRecord(g->ev[0], st));
    size_t total_chunks = 0;
    for (const msv_grid::Wave& w : g->waves) total_chunks += w.chunks.size();
    const bool overlap = g->overlap && total_chunks > 1;
    // Back-to-back launches of one single-wave grid are pipelined: chunk c only touches
    // its own scenarios' buffer regions and always runs on aux stream c, so launch i+1's
    // chunk c needs only launch i's chunk c to be done (stream order) — no fork, and its
    // trace generation overlaps the other chunks' simulation of launch i. Any other grid
    // launched in between (it may share the scratch buffers) restores the full fork.
    static const bool pipeline_env = !(getenv("MSV_PIPELINE") && atoi(getenv("MSV_PIPELINE")) == 0);
    const bool pipelined = pipeline_env && overlap && g->waves.size() == 1 && ctx->last_launch_grid == g->serial;
    ctx->last_launch_grid = overlap ? g->serial : 0;  // a main-stream launch is never pipelined past
    // work counters: each (chunk, class) owns one slot (mod kCounterSlots), zeroed on the
    // stream that uses it right before the chunk
    auto zero_counters = [&](int base, size_t n, cudaStream_t s) -> int {
        const int s0 = base % kCounterSlots;
        const size_t first = std::min(n, (size_t)(kCounterSlots - s0));
        MSV_CUDA_TRY(cudaMemsetAsync(g->B->d_counter.as<int32_t>() + s0, 0, first * sizeof(int32_t), s));
        if (n > first) MSV_CUDA_TRY(cudaMemsetAsync(g->B->d_counter.p, 0, (n - first) * sizeof(int32_t), s));
        return MSV_OK;
    };
    // waves of a multi-region grid each need their own stream to run side by side
    const int n_aux = std::max(kAuxStreams, std::min(8, g->n_regions));
    if (overlap) {
        for (int a = 0; a < n_aux; ++a) {
            if (!ctx->aux[a]) MSV_CUDA_TRY(cudaStreamCreateWithFlags(&ctx->aux[a], cudaStreamNonBlocking));
            if (!ctx->aux_ev[a]) MSV_CUDA_TRY(cudaEventCreateWithFlags(&ctx->aux_ev[a], cudaEventDisableTiming));
        }
        if (!ctx->fork_ev) MSV_CUDA_TRY(cudaEventCreateWithFlags(&ctx->fork_ev, cudaEventDisableTiming));
    }
    int counter_base = 0;
    float tr = 0, si = 0, ta = 0;
    // wave w's completion: region_ev[w % kWaveRing]. Its K1 waits for wave w - n_in_regions
    // (the input region), its K2 for wave w - n_regions (the link region).
    constexpr int kWaveRing = 8;  // (ctx->region_ev slots: at least the largest lookback)
    if (overlap && g->n_regions > 1)
        for (int r = 0; r < kWaveRing; ++r)
            if (!ctx->region_ev[r]) MSV_CUDA_TRY(cudaEventCreateWithFlags(&ctx->region_ev[r], cudaEventDisableTiming));
    size_t chunk_seq = 0;  // chunks of consecutive waves go to different aux streams
    for (size_t wi = 0; wi < g->waves.size(); ++wi) {
        const msv_grid::Wave& w = g->waves[wi];
        if (overlap) {
            // fork: the first waves start after everything queued on the main stream; a
            // wave that reuses a buffer region waits only for the wave that used it last
            // (the two regions' waves overlap: one drains while the next fills the SMs)
            if (!pipelined && wi == 0) MSV_CUDA_TRY(cudaEventRecord(ctx->fork_ev, st));
            std::vector<char> used(n_aux, 0);
            for (size_t c = 0; c < w.chunks.size(); ++c) {
                const int a = (int)((chunk_seq++) % n_aux);
                cudaStream_t sc = ctx->aux[a];
                used[a] = 1;
                if (!pipelined && wi < (size_t)g->n_in_regions) MSV_CUDA_TRY(cudaStreamWaitEvent(sc, ctx->fork_ev, 0));
                if (wi >= (size_t)g->n_in_regions)
                    MSV_CUDA_TRY(cudaStreamWaitEvent(sc, ctx->region_ev[(wi - g->n_in_regions) % kWaveRing], 0));
                cudaEvent_t k2_wait = nullptr;
                if (wi >= (size_t)g->n_regions && g->n_in_regions > g->n_regions)
                    k2_wait = ctx->region_ev[(wi - g->n_regions) % kWaveRing];
                if ((rc = zero_counters(counter_base, w.chunks[c].classes.size(), sc))) return rc;
                if ((rc = launch_chunk(g, w.chunks[c], counter_base, sc, nullptr, nullptr, k2_wait))) return rc;
                counter_base += (int)w.chunks[c].classes.size();
            }
            // join: the main stream continues after every chunk of this wave, and the
            // wave's region is free again from here
            for (int a = 0; a < n_aux; ++a) {
                if (!used[a]) continue;
                MSV_CUDA_TRY(cudaEventRecord(ctx->aux_ev[a], ctx->aux[a]));
                MSV_CUDA_TRY(cudaStreamWaitEvent(st, ctx->aux_ev[a], 0));
            }
            if (g->n_regions > 1) MSV_CUDA_TRY(cudaEventRecord(ctx->region_ev[wi % kWaveRing], st));
        } else {
            for (const msv_grid::Chunk& ch : w.chunks) {
                cudaEvent_t e0 = g->ev[0], e1 = g->ev[1], e2 = g->ev[2], e3 = g->ev[3];
                if (wi > 0 || &ch != &w.chunks.front()) MSV_CUDA_TRY(cudaEventRecord(e0, st));
                if ((rc = zero_counters(counter_base, ch.classes.size(), st))) return rc;
                if ((rc = launch_chunk(g, ch, counter_base, st, e1, e2))) return rc;
                counter_base += (int)ch.classes.size();
                MSV_CUDA_TRY(cudaEventRecord(e3, st));
                if (total_chunks > 1) {  // events are reused: accumulate stage times per chunk
                    MSV_CUDA_TRY(cudaEventSynchronize(e3));
                    float a = 0, b = 0, c2 = 0;
                    cudaEventElapsedTime(&a, e0, e1);
                    cudaEventElapsedTime(&b, e1, e2);
                    cudaEventElapsedTime(&c2, e2, e3);
                    tr += a;
                    si += b;
                    ta += c2;
                }
            }
        }
    }
    if (overlap) {
        MSV_CUDA_TRY(cudaEventRecord(g->ev[3], st));
        g->t_total = -2;  // total only (stages overlap), resolved lazily
    } else if (total_chunks > 1) {
        g->t_trace = tr;
        g->t_sim = si;
        g->t_tail = ta;
        g->t_total = tr + si + ta;
    } else {
        g->t_total = -1;  // resolved lazily in msv_grid_timing
    }
    if (timeline_on()) {
        timeline_mark("launch end", st);
        timeline_print(g->ev[0]);
    }
    return MSV_OK;
}

int grid_results(msv_grid* g, msv_result* res, msv_usage* usage, msv_record* records,
                 std::vector<int64_t>* retry_trace) {
    if (usage && !g->usage && g->usage_total)
        return fail(MSV_PARAM, "grid: launched without usage accumulation (msv_grid_set_usage)");
    msv_ctx* ctx = g->ctx;
    MSV_CUDA_TRY(cudaStreamSynchronize(ctx->stream));
    const int64_t n = g->n;
    std::vector<DevOut> outs(n);
    std::vector<double> tails(n * 4);
    std::vector<int64_t> nq(n);
    std::vector<int32_t> tovf(n);
    if (n) {
        MSV_CUDA_TRY(cudaMemcpy(outs.data(), g->B->d_out.p, n * sizeof(DevOut), cudaMemcpyDeviceToHost));
        MSV_CUDA_TRY(cudaMemcpy(tails.data(), g->B->d_tails.p, n * 4 * sizeof(double), cudaMemcpyDeviceToHost));
        MSV_CUDA_TRY(cudaMemcpy(nq.data(), g->B->d_nq.p, n * 8, cudaMemcpyDeviceToHost));
        MSV_CUDA_TRY(cudaMemcpy(tovf.data(), g->B->d_tovf.p, n * 4, cudaMemcpyDeviceToHost));
        ctx->d2h += n * (int64_t)(sizeof(DevOut) + 4 * sizeof(double) + 8 + 4);
    }
    if (usage && g->usage_total)
        MSV_CUDA_TRY(cudaMemcpy(usage, g->B->d_usage.p, g->usage_total * sizeof(msv_usage), cudaMemcpyDeviceToHost));
    if (records && g->records && g->waves.size() == 1 && g->max_wave_q) {
        if (g->generated) {
            MSV_CUDA_TRY(cudaMemcpy(records, g->B->d_rec.p, g->max_wave_q * sizeof(msv_record), cudaMemcpyDeviceToHost));
        } else {  // back to the caller's layout
            std::vector<msv_record> dev(g->max_wave_q);
            MSV_CUDA_TRY(cudaMemcpy(dev.data(), g->B->d_rec.p, g->max_wave_q * sizeof(msv_record), cudaMemcpyDeviceToHost));
            for (int64_t i = 0; i < n; ++i)
                std::copy(dev.begin() + g->toff[i], dev.begin() + g->toff[i] + g->host_n[i], records + g->user_off[i]);
        }
    }
    int first_err = MSV_OK;
    int64_t first_i = -1;
    for (int64_t i = 0; i < n; ++i) {
        msv_result& r = res[i];
        const DevOut& o = outs[i];
        memset(&r, 0, sizeof r);
        r.total = nq[i];
        r.violations = o.violations;
        r.measured = o.measured;
        r.measured_violations = o.measured_violations;
        for (int j = 0; j < 4; ++j)
            r.tail[j] = j < (int)g->tail_p.size() ? tails[4 * i + j] : __builtin_nan("");
        r.horizon_ms = o.horizon_ms;
        r.warmup_ms = g->scen[i].warmup_fraction * g->scen[i].duration_ms;
        r.max_wait_estimate_diff = o.max_wait_diff;
        r.duration_ms = g->scen[i].duration_ms;
        r.placement_hash = o.hash;
        r.status = o.status;
        r.n_partitions = g->P[i];
        if (tovf[i]) {
            r.status = msv::kStatusRetryTrace;
            if (retry_trace) retry_trace->push_back(i);
        }
        if (r.status != MSV_OK && r.status < 100 && first_err == MSV_OK) {
            first_err = r.status;
            first_i = i;
        }
    }
    if (first_err != MSV_OK)
        return fail(first_err, "scenario " + std::to_string(first_i) + ": profile: batch outside the profile grid");
    return MSV_OK;
}

}  // namespace

// ---------------------------------------------------------------------------
// C ABI
// ---------------------------------------------------------------------------
namespace {

// The kernels stage a grid's profile cells in shared memory (<= kMaxSmemCells). A call
// whose scenarios use more distinct profile cells than that runs as several grids, one per
// group of profiles that fits (the reference has no such limit). Returns false when one
// grid suffices (or a handle is invalid: the single-grid path reports the error).
bool profile_groups(const msv_ctx* ctx, const msv_scenario* sc, int64_t n, std::vector<std::vector<int64_t>>* groups) {
    std::map<int32_t, int> group_of;
    std::vector<int> cells;  // per group
    int64_t total = 0;
    for (int64_t i = 0; i < n; ++i) {
        const int32_t pf = sc[i].profile;
        if (pf < 0 || pf >= (int32_t)ctx->profiles.size()) return false;
        if (group_of.count(pf)) continue;
        const int c = (int)ctx->profiles[pf].lat.size();
        if (c > msv::kMaxSmemCells) return false;
        total += c;
        if (cells.empty() || cells.back() + c > msv::kMaxSmemCells) cells.push_back(0);
        cells.back() += c;
        group_of[pf] = (int)cells.size() - 1;
    }
    if (total <= msv::kMaxSmemCells) return false;
    groups->assign(cells.size(), {});
    for (int64_t i = 0; i < n; ++i) (*groups)[group_of[sc[i].profile]].push_back(i);
    return true;
}

}  // namespace

extern "C" {

const char* msv_last_error(void) { return g_err.c_str(); }

int msv_abi_version(void) { return MSV_ABI_VERSION; }

int msv_create(int device, msv_ctx** out) {
    if (!out) return fail(MSV_PARAM, "msv_create: null out");
    *out = nullptr;
    int count = 0;
    cudaError_t e = cudaGetDeviceCount(&count);
    if (e != cudaSuccess || count == 0)
        return fail(MSV_CUDA, std::string("msv_create: no CUDA device: ") + cudaGetErrorString(e));
    if (device < 0 || device >= count) return fail(MSV_PARAM, "msv_create: bad device ordinal");
    SetDevice sd(device);
    std::unique_ptr<msv_ctx> ctx(new msv_ctx);
    ctx->device = device;
    MSV_CUDA_TRY(cudaSetDevice(device));
    MSV_CUDA_TRY(cudaDeviceGetAttribute(&ctx->sms, cudaDevAttrMultiProcessorCount, device));
    int major = 0, minor = 0;
    cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, device);
    cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, device);
    if (major != 10 || minor != 0)
        return fail(MSV_CUDA, "msv_create: libmsv is built for sm_100a (B200); device is sm_" +
                                  std::to_string(major) + std::to_string(minor));
    ctx->log1p = probe_host_log1p();
    if (ctx->log1p < 0)
        return fail(MSV_CUDA, "msv_create: this host's libm log1p matches neither transcribed glibc build "
                              "(csrc/msv_math.h); device traces would diverge from rng.hpp:20");
    MSV_CUDA_TRY(cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking));
    *out = ctx.release();
    return MSV_OK;
}

int msv_destroy(msv_ctx* ctx) {
    if (!ctx) return MSV_OK;
    for (msv_ctx* p : ctx->peers) msv_destroy(p);
    ctx->peers.clear();
    SetDevice sd(ctx->device);
    cudaStreamSynchronize(ctx->stream);
    for (cudaEvent_t e : ctx->ev)
        if (e) cudaEventDestroy(e);
    for (int a = 0; a < 8; ++a) {
        if (ctx->aux[a]) {
            cudaStreamSynchronize(ctx->aux[a]);
            cudaStreamDestroy(ctx->aux[a]);
        }
        if (ctx->aux_ev[a]) cudaEventDestroy(ctx->aux_ev[a]);
    }
    if (ctx->fork_ev) cudaEventDestroy(ctx->fork_ev);
    for (cudaEvent_t e : ctx->region_ev)
        if (e) cudaEventDestroy(e);
    for (int a = 0; a < 4; ++a) {
        if (ctx->cls[a]) {
            cudaStreamSynchronize(ctx->cls[a]);
            cudaStreamDestroy(ctx->cls[a]);
        }
        if (ctx->cls_ev[a]) cudaEventDestroy(ctx->cls_ev[a]);
    }
    if (ctx->cls_fork) cudaEventDestroy(ctx->cls_fork);
    for (int b = 0; b < 2; ++b) {
        if (ctx->pin[b]) cudaFreeHost(ctx->pin[b]);
        if (ctx->pin_ev[b]) cudaEventDestroy(ctx->pin_ev[b]);
    }
    if (ctx->k1_ev) cudaEventDestroy(ctx->k1_ev);
    cudaStreamDestroy(ctx->stream);
    delete ctx;
    return MSV_OK;
}

int msv_set_log1p_variant(msv_ctx* ctx, int variant) {
    if (!ctx) return fail(MSV_PARAM, "null context");
    if (variant == MSV_LOG1P_AUTO) {
        variant = probe_host_log1p();
        if (variant < 0) return fail(MSV_CUDA, "msv_set_log1p_variant: host libm log1p matches neither build");
    }
    if (variant != MSV_LOG1P_GENERIC && variant != MSV_LOG1P_FMA)
        return fail(MSV_PARAM, "msv_set_log1p_variant: unknown variant");
    ctx->log1p = variant;
    ctx->upload_serial++;
    return MSV_OK;
}

int msv_get_log1p_variant(msv_ctx* ctx, int* variant) {
    if (!ctx || !variant) return fail(MSV_PARAM, "null argument");
    *variant = ctx->log1p;
    return MSV_OK;
}

// ProfileTable::validate (profile.hpp:134-169).
int msv_upload_profile(msv_ctx* ctx, int n_sizes, const int32_t* sizes, int b_max, const double* latency_ms,
                       const double* utilization, int32_t* handle) {
    if (!ctx || !handle) return fail(MSV_PARAM, "null argument");
    ctx->upload_serial++;
    if (n_sizes <= 0) return fail(MSV_PARAM, "profile: empty size set");
    if (b_max < 1) return fail(MSV_PARAM, "profile: b_max must be >= 1");
    Profile p;
    p.sizes.assign(sizes, sizes + n_sizes);
    p.b_max = b_max;
    for (int i = 1; i < n_sizes; ++i)
        if (!(p.sizes[i - 1] < p.sizes[i])) return fail(MSV_VALIDATION, "profile: sizes must be strictly ascending");
    if (p.sizes.front() < 1) return fail(MSV_VALIDATION, "profile: partition sizes must be positive");
    const size_t cells = (size_t)n_sizes * b_max;
    p.lat.assign(latency_ms, latency_ms + cells);
    p.util.assign(utilization, utilization + cells);
    for (size_t i = 0; i < cells; ++i) {
        if (!(p.lat[i] > 0.0)) return fail(MSV_VALIDATION, "profile: latency must be positive");
        if (p.util[i] < 0.0 || p.util[i] > 1.0) return fail(MSV_VALIDATION, "profile: utilization outside [0,1]");
    }
    const double tol = 1e-9;
    for (int i = 0; i < n_sizes; ++i)
        for (int b = 2; b <= b_max; ++b) {
            const size_t c = (size_t)i * b_max + (b - 1);
            if (p.util[c] < p.util[c - 1] - tol)
                return fail(MSV_VALIDATION, "profile: utilization must be nondecreasing in batch");
            if (p.lat[c] < p.lat[c - 1] * (1.0 - tol))
                return fail(MSV_VALIDATION, "profile: latency must be nondecreasing in batch");
        }
    for (int i = 1; i < n_sizes; ++i)
        for (int b = 1; b <= b_max; ++b) {
            const size_t c = (size_t)i * b_max + (b - 1);
            if (p.lat[c] > p.lat[c - b_max] * (1.0 + tol))
                return fail(MSV_VALIDATION, "profile: latency must be nonincreasing in partition size");
        }
    ctx->profiles.push_back(std::move(p));
    ctx->tables_dirty = true;
    *handle = (int32_t)ctx->profiles.size() - 1;
    return MSV_OK;
}

// BatchDistribution(weights) (workload.hpp:25-38).
int msv_upload_dist(msv_ctx* ctx, int b_max, const double* weights, int32_t* handle) {
    if (!ctx || !handle) return fail(MSV_PARAM, "null argument");
    ctx->upload_serial++;
    if (b_max <= 0) return fail(MSV_PARAM, "batch distribution: empty support");
    Dist d;
    d.pmf.assign(weights, weights + b_max);
    double total = 0.0;
    for (double w : d.pmf) {
        if (w < 0.0 || !std::isfinite(w)) return fail(MSV_PARAM, "batch distribution: weights must be finite and >= 0");
        total += w;
    }
    if (!(total > 0.0)) return fail(MSV_PARAM, "batch distribution: all weights are zero");
    for (double& w : d.pmf) w /= total;
    d.cdf.resize(d.pmf.size());
    double acc = 0.0;
    for (size_t i = 0; i < d.pmf.size(); ++i) {
        acc = (i == 0) ? d.pmf[0] : acc + d.pmf[i];  // std::partial_sum
        d.cdf[i] = acc;
    }
    d.cdf.back() = 1.0;
    ctx->dists.push_back(std::move(d));
    ctx->tables_dirty = true;
    *handle = (int32_t)ctx->dists.size() - 1;
    return MSV_OK;
}

int msv_upload_cdf(msv_ctx* ctx, int b_max, const double* cdf, int32_t* handle) {
    if (!ctx || !handle || !cdf) return fail(MSV_PARAM, "null argument");
    ctx->upload_serial++;
    if (b_max <= 0) return fail(MSV_PARAM, "batch distribution: empty support");
    Dist d;
    d.cdf.assign(cdf, cdf + b_max);
    for (int i = 0; i < b_max; ++i) {
        if (!(d.cdf[i] >= 0.0) || d.cdf[i] > 1.0 || (i && d.cdf[i] < d.cdf[i - 1]))
            return fail(MSV_PARAM, "batch distribution: cdf must be nondecreasing in [0,1]");
    }
    if (d.cdf.back() != 1.0) return fail(MSV_PARAM, "batch distribution: cdf must end at 1.0");
    d.pmf.resize(b_max);
    for (int i = 0; i < b_max; ++i) d.pmf[i] = i ? d.cdf[i] - d.cdf[i - 1] : d.cdf[0];
    ctx->dists.push_back(std::move(d));
    ctx->tables_dirty = true;
    *handle = (int32_t)ctx->dists.size() - 1;
    return MSV_OK;
}

// PartitionPlan + validate() (paris.hpp:133-156); validation errors surface at run.
int msv_upload_plan(msv_ctx* ctx, int num_gpus, int gpcs_per_gpu, const int32_t* n_per_gpu,
                    const int32_t* sizes_flat, int32_t* handle) {
    if (!ctx || !handle) return fail(MSV_PARAM, "null argument");
    ctx->upload_serial++;
    Plan p;
    p.num_gpus = num_gpus;
    p.gpcs_per_gpu = gpcs_per_gpu;
    if (num_gpus < 1) {
        p.err = MSV_VALIDATION;
        p.err_msg = "plan: num_gpus must be >= 1";
    } else if (gpcs_per_gpu < 1) {
        p.err = MSV_VALIDATION;
        p.err_msg = "plan: gpcs_per_gpu must be >= 1";
    }
    size_t off = 0;
    for (int g = 0; g < std::max(num_gpus, 0); ++g) {
        int used = 0;
        for (int j = 0; j < n_per_gpu[g]; ++j) {
            const int32_t k = sizes_flat[off + j];
            if (k < 1 && !p.err) {
                p.err = MSV_VALIDATION;
                p.err_msg = "plan: partition size must be positive";
            }
            used += k;
            p.flat.push_back(k);
        }
        off += n_per_gpu[g];
        if (used > gpcs_per_gpu && !p.err) {
            p.err = MSV_VALIDATION;
            p.err_msg = "plan: GPU over capacity (" + std::to_string(used) + " > " + std::to_string(gpcs_per_gpu) + ")";
        }
    }
    ctx->plans.push_back(std::move(p));
    *handle = (int32_t)ctx->plans.size() - 1;
    return MSV_OK;
}

int msv_upload_routing(msv_ctx* ctx, int n_segments, const int32_t* k, const int32_t* first,
                       const int32_t* last, int32_t* handle) {
    if (!ctx || !handle) return fail(MSV_PARAM, "null argument");
    ctx->upload_serial++;
    if (n_segments < 0) return fail(MSV_PARAM, "routing: negative segment count");
    Routing r;
    r.k.assign(k, k + n_segments);
    r.first.assign(first, first + n_segments);
    r.last.assign(last, last + n_segments);
    ctx->routings.push_back(std::move(r));
    *handle = (int32_t)ctx->routings.size() - 1;
    return MSV_OK;
}

static int grid_create_dev(msv_ctx* ctx, const msv_scenario* scenarios, int64_t n, const double* tail_p, int n_tails,
                           msv_grid** out) {
    if (!ctx || !out || (n > 0 && !scenarios)) return fail(MSV_PARAM, "null argument");
    SetDevice sd(ctx->device);
    std::vector<std::vector<int64_t>> groups;
    if (!profile_groups(ctx, scenarios, n, &groups))
        return grid_build(ctx, scenarios, n, tail_p, n_tails, nullptr, nullptr, nullptr, false, out);
    std::unique_ptr<msv_grid> top(new msv_grid);
    top->ctx = ctx;
    top->n = n;
    top->tail_p.assign(tail_p, tail_p + std::max(n_tails, 0));
    top->use_off.assign(n + 1, 0);
    for (int64_t i = 0; i < n; ++i) {  // validate first: errors name the caller's index
        int32_t P = 0;
        const int rc = validate_scenario(ctx, scenarios[i], true, &P);
        if (rc) {
            g_err = "scenario " + std::to_string(i) + ": " + g_err;
            return rc;
        }
        top->use_off[i + 1] = top->use_off[i] + P;
    }
    top->usage_total = top->use_off[n];
    for (std::vector<int64_t>& grp : groups) {
        std::vector<msv_scenario> sub;
        for (int64_t i : grp) sub.push_back(scenarios[i]);
        msv_grid* g = nullptr;
        const int rc = grid_build(ctx, sub.data(), (int64_t)sub.size(), tail_p, n_tails, nullptr, nullptr, nullptr,
                                  false, &g);
        if (rc) return rc;
        top->parts.emplace_back(g);
        top->part_idx.push_back(std::move(grp));
    }
    for (cudaEvent_t& e : top->ev) MSV_CUDA_TRY(cudaEventCreate(&e));
    *out = top.release();
    return MSV_OK;
}

static int grid_launch_dev(msv_grid* grid) {
    if (!grid) return fail(MSV_PARAM, "null grid");
    SetDevice sd(grid->ctx->device);
    if (grid->parts.empty()) return grid_launch(grid);
    MSV_CUDA_TRY(cudaEventRecord(grid->ev[0], grid->ctx->stream));
    for (std::unique_ptr<msv_grid>& part : grid->parts) {
        part->usage = grid->usage;
        part->overlap = grid->overlap;
        const int rc = grid_launch(part.get());
        if (rc) return rc;
    }
    MSV_CUDA_TRY(cudaEventRecord(grid->ev[3], grid->ctx->stream));
    grid->t_total = -2;  // only the total is defined
    return MSV_OK;
}

static int grid_results_dev(msv_grid* grid, msv_result* results, msv_usage* usage) {
    if (!grid || (grid->n > 0 && !results)) return fail(MSV_PARAM, "null argument");
    SetDevice sd(grid->ctx->device);
    if (grid->parts.empty()) return grid_results(grid, results, usage, nullptr, nullptr);
    for (size_t k = 0; k < grid->parts.size(); ++k) {
        msv_grid* part = grid->parts[k].get();
        const std::vector<int64_t>& idx = grid->part_idx[k];
        std::vector<msv_result> sub(idx.size());
        std::vector<msv_usage> sub_use(std::max<int64_t>(part->usage_total, 1));
        const int rc = grid_results(part, sub.data(), usage ? sub_use.data() : nullptr, nullptr, nullptr);
        if (rc) return rc;
        int64_t u = 0;
        for (size_t j = 0; j < idx.size(); ++j) {
            results[idx[j]] = sub[j];
            if (usage)
                for (int64_t q = grid->use_off[idx[j]]; q < grid->use_off[idx[j] + 1]; ++q) usage[q] = sub_use[u++];
        }
    }
    return MSV_OK;
}

static int grid_timing_dev(msv_grid* g, float* total_ms, float* trace_ms, float* sim_ms, float* tail_ms) {
    if (!g) return fail(MSV_PARAM, "null grid");
    SetDevice sd(g->ctx->device);
    if (g->t_total == -2.0f) {  // overlapped chunks: only the total is defined
        MSV_CUDA_TRY(cudaEventSynchronize(g->ev[3]));
        cudaEventElapsedTime(&g->t_total, g->ev[0], g->ev[3]);
        g->t_trace = g->t_sim = g->t_tail = -1.0f;
    } else if (g->t_total < 0) {
        MSV_CUDA_TRY(cudaEventSynchronize(g->ev[3]));
        cudaEventElapsedTime(&g->t_trace, g->ev[0], g->ev[1]);
        cudaEventElapsedTime(&g->t_sim, g->ev[1], g->ev[2]);
        cudaEventElapsedTime(&g->t_tail, g->ev[2], g->ev[3]);
        cudaEventElapsedTime(&g->t_total, g->ev[0], g->ev[3]);
    }
    if (total_ms) *total_ms = g->t_total;
    if (trace_ms) *trace_ms = g->t_trace;
    if (sim_ms) *sim_ms = g->t_sim;
    if (tail_ms) *tail_ms = g->t_tail;
    return MSV_OK;
}

int msv_grid_set_usage(msv_grid* g, int on) {
    if (!g) return fail(MSV_PARAM, "null grid");
    g->usage = on != 0;
    return MSV_OK;
}

int msv_grid_set_overlap(msv_grid* g, int on) {
    if (!g) return fail(MSV_PARAM, "null grid");
    g->overlap = on != 0;
    return MSV_OK;
}

static int64_t grid_queries_dev(msv_grid* g) {
    if (!g) return -1;
    SetDevice sd(g->ctx->device);
    if (!g->parts.empty()) {
        int64_t t = 0;
        for (std::unique_ptr<msv_grid>& part : g->parts) {
            const int64_t q = grid_queries_dev(part.get());
            if (q < 0) return -1;
            t += q;
        }
        return t;
    }
    if (cudaStreamSynchronize(g->ctx->stream) != cudaSuccess) return -1;
    std::vector<int64_t> nq(g->n);
    if (g->n && cudaMemcpy(nq.data(), g->B->d_nq.p, g->n * 8, cudaMemcpyDeviceToHost) != cudaSuccess) return -1;
    int64_t s = 0;
    for (int64_t v : nq) s += v;
    return s;
}

int msv_synchronize(msv_ctx* ctx) {
    if (!ctx) return fail(MSV_PARAM, "null context");
    for (msv_ctx* p : ctx->peers) {
        const int rc = msv_synchronize(p);
        if (rc) return rc;
    }
    SetDevice sd(ctx->device);
    MSV_CUDA_TRY(cudaStreamSynchronize(ctx->stream));
    return MSV_OK;
}

int64_t msv_kernel_launches(msv_ctx* ctx) {
    if (!ctx) return -1;
    int64_t n = ctx->launches;
    for (msv_ctx* p : ctx->peers) n += p->launches;
    return n;
}

// Events on every member's stream; elapsed = the max over the members (multi-device
// timings are the slowest device's, never a host clock).
int msv_event_record(msv_ctx* ctx, int slot) {
    if (!ctx || slot < 0 || slot >= 8) return fail(MSV_PARAM, "msv_event_record: bad slot");
    for (msv_ctx* p : ctx->peers) {
        const int rc = msv_event_record(p, slot);
        if (rc) return rc;
    }
    SetDevice sd(ctx->device);
    if (!ctx->ev[slot]) MSV_CUDA_TRY(cudaEventCreate(&ctx->ev[slot]));
    MSV_CUDA_TRY(cudaEventRecord(ctx->ev[slot], ctx->stream));
    ctx->last_launch_grid = 0;  // the next launch forks from the main stream: it starts after this event
    return MSV_OK;
}

int msv_event_elapsed(msv_ctx* ctx, int a, int b, float* ms) {
    if (!ctx || !ms || a < 0 || a >= 8 || b < 0 || b >= 8 || !ctx->ev[a] || !ctx->ev[b])
        return fail(MSV_PARAM, "msv_event_elapsed: bad slot");
    float worst = 0.0f;
    for (msv_ctx* p : ctx->peers) {
        float t = 0.0f;
        const int rc = msv_event_elapsed(p, a, b, &t);
        if (rc) return rc;
        worst = std::max(worst, t);
    }
    SetDevice sd(ctx->device);
    MSV_CUDA_TRY(cudaEventSynchronize(ctx->ev[b]));
    MSV_CUDA_TRY(cudaEventElapsedTime(ms, ctx->ev[a], ctx->ev[b]));
    *ms = std::max(*ms, worst);
    return MSV_OK;
}

int msv_transfer_bytes(msv_ctx* ctx, int64_t* h2d, int64_t* d2h) {
    if (!ctx) return fail(MSV_PARAM, "null context");
    int64_t a = ctx->h2d, b = ctx->d2h;
    for (msv_ctx* p : ctx->peers) {
        a += p->h2d;
        b += p->d2h;
    }
    if (h2d) *h2d = a;
    if (d2h) *d2h = b;
    return MSV_OK;
}

}  // extern "C"

namespace {

int run_grid_core(msv_ctx* ctx, const msv_scenario* scenarios, int64_t n, const double* tail_p, int n_tails,
                  msv_result* results, msv_usage* usage);

}  // namespace

extern "C" {

static int run_grid_dev(msv_ctx* ctx, const msv_scenario* scenarios, int64_t n, const double* tail_p, int n_tails,
                        msv_result* results, msv_usage* usage) {
    if (!ctx || (n > 0 && (!scenarios || !results))) return fail(MSV_PARAM, "null argument");
    SetDevice sd(ctx->device);
    std::vector<std::vector<int64_t>> groups;
    if (!profile_groups(ctx, scenarios, n, &groups)) return run_grid_core(ctx, scenarios, n, tail_p, n_tails, results, usage);
    // validate everything first, so errors name the caller's scenario index
    std::vector<int64_t> use_off(n + 1, 0);
    for (int64_t i = 0; i < n; ++i) {
        int32_t P = 0;
        const int rc = validate_scenario(ctx, scenarios[i], true, &P);
        if (rc) {
            g_err = "scenario " + std::to_string(i) + ": " + g_err;
            return rc;
        }
        use_off[i + 1] = use_off[i] + P;
    }
    for (const std::vector<int64_t>& grp : groups) {
        std::vector<msv_scenario> sub;
        for (int64_t i : grp) sub.push_back(scenarios[i]);
        std::vector<msv_result> sub_res(sub.size());
        int64_t nu = 0;
        for (int64_t i : grp) nu += use_off[i + 1] - use_off[i];
        std::vector<msv_usage> sub_use(std::max<int64_t>(nu, 1));
        const int rc = run_grid_core(ctx, sub.data(), (int64_t)sub.size(), tail_p, n_tails, sub_res.data(),
                                     usage ? sub_use.data() : nullptr);
        if (rc) return rc;
        int64_t u = 0;
        for (size_t j = 0; j < grp.size(); ++j) {
            const int64_t i = grp[j];
            results[i] = sub_res[j];
            if (usage)
                for (int64_t q = use_off[i]; q < use_off[i + 1]; ++q) usage[q] = sub_use[u++];
        }
    }
    return MSV_OK;
}

}  // extern "C"

namespace {

int run_grid_core(msv_ctx* ctx, const msv_scenario* scenarios, int64_t n, const double* tail_p, int n_tails,
                  msv_result* results, msv_usage* usage) {
    msv_grid* g = nullptr;
    static const bool host_timing = getenv("MSV_HOST_TIMING") != nullptr;
    const auto t0 = std::chrono::steady_clock::now();
    int rc = grid_build(ctx, scenarios, n, tail_p, n_tails, nullptr, nullptr, nullptr, false, &g, nullptr, true);
    if (rc) return rc;
    std::unique_ptr<msv_grid> guard(g);
    g->usage = usage != nullptr;
    const auto t1 = std::chrono::steady_clock::now();
    rc = grid_launch(g);
    if (rc) return rc;
    const auto t2 = std::chrono::steady_clock::now();
    std::vector<int64_t> retry;
    rc = grid_results(g, results, usage, nullptr, &retry);
    if (rc) return rc;
    if (host_timing) {
        const auto t3 = std::chrono::steady_clock::now();
        auto ms = [](auto a, auto b) { return std::chrono::duration<double, std::milli>(b - a).count(); };
        fprintf(stderr, "[msv] run_grid n=%lld build %.2f ms, enqueue %.2f ms, results+sync %.2f ms\n",
                (long long)n, ms(t0, t1), ms(t1, t2), ms(t2, t3));
    }
    // Traces longer than the Poisson-tail capacity (a >10-sigma Poisson count):
    // rerun those scenarios alone with the capacity quadrupled until they fit.
    std::vector<int64_t> caps_prev;
    for (int64_t i : retry) caps_prev.push_back(g->cap[i]);
    for (int attempt = 0; !retry.empty(); ++attempt) {
        if (attempt >= 6) return fail(MSV_PARAM, "sample_trace: trace exceeded its capacity repeatedly");
        std::vector<msv_scenario> sub;
        std::vector<int64_t> caps;
        int64_t usage_n = 0;
        for (size_t j = 0; j < retry.size(); ++j) {
            sub.push_back(scenarios[retry[j]]);
            caps.push_back(caps_prev[j] * 4);
        }
        msv_grid* g2 = nullptr;
        rc = grid_build(ctx, sub.data(), (int64_t)sub.size(), tail_p, n_tails, nullptr, nullptr, nullptr, false, &g2,
                        caps.data());
        if (rc) return rc;
        std::unique_ptr<msv_grid> guard2(g2);
        g2->usage = usage != nullptr;
        rc = grid_launch(g2);
        if (rc) return rc;
        usage_n = g2->usage_total;
        std::vector<msv_result> sub_res(sub.size());
        std::vector<msv_usage> sub_use(std::max<int64_t>(usage_n, 1));
        std::vector<int64_t> again;
        rc = grid_results(g2, sub_res.data(), usage ? sub_use.data() : nullptr, nullptr, &again);
        if (rc) return rc;
        std::vector<int64_t> next_retry, next_caps;
        size_t again_pos = 0;
        for (size_t j = 0; j < sub.size(); ++j) {
            const int64_t i = retry[j];
            if (again_pos < again.size() && again[again_pos] == (int64_t)j) {
                ++again_pos;
                next_retry.push_back(i);
                next_caps.push_back(caps[j]);
                continue;
            }
            results[i] = sub_res[j];
            if (usage)
                for (int32_t q = 0; q < g2->P[j]; ++q) usage[g->usage_off[i] + q] = sub_use[g2->usage_off[j] + q];
        }
        retry.swap(next_retry);
        caps_prev.swap(next_caps);
    }
    return MSV_OK;
}

}  // namespace

extern "C" {

static int run_replay_dev(msv_ctx* ctx, const msv_scenario* scenarios, int64_t n, const int64_t* offsets,
                          const double* arrival_ms, const int32_t* batch, const double* tail_p, int n_tails,
                          msv_result* results, msv_usage* usage, msv_record* records) {
    if (!ctx || (n > 0 && (!scenarios || !results || !offsets))) return fail(MSV_PARAM, "null argument");
    SetDevice sd(ctx->device);
    std::vector<std::vector<int64_t>> groups;
    if (profile_groups(ctx, scenarios, n, &groups)) {  // more profile cells than one grid holds
        std::vector<int64_t> use_off(n + 1, 0);
        for (int64_t i = 0; i < n; ++i) {
            int32_t P = 0;
            const int rc = validate_scenario(ctx, scenarios[i], false, &P);
            if (rc) {
                g_err = "scenario " + std::to_string(i) + ": " + g_err;
                return rc;
            }
            use_off[i + 1] = use_off[i] + P;
        }
        for (const std::vector<int64_t>& grp : groups) {
            std::vector<msv_scenario> sub;
            std::vector<int64_t> off{0};
            std::vector<double> arr;
            std::vector<int32_t> bat;
            int64_t nu = 0;
            for (int64_t i : grp) {
                sub.push_back(scenarios[i]);
                arr.insert(arr.end(), arrival_ms + offsets[i], arrival_ms + offsets[i + 1]);
                bat.insert(bat.end(), batch + offsets[i], batch + offsets[i + 1]);
                off.push_back((int64_t)arr.size());
                nu += use_off[i + 1] - use_off[i];
            }
            std::vector<msv_result> sub_res(sub.size());
            std::vector<msv_usage> sub_use(std::max<int64_t>(nu, 1));
            std::vector<msv_record> sub_rec(std::max<size_t>(arr.size(), 1));
            const int rc = run_replay_dev(ctx, sub.data(), (int64_t)sub.size(), off.data(), arr.data(), bat.data(), tail_p,
                                          n_tails, sub_res.data(), usage ? sub_use.data() : nullptr,
                                          records ? sub_rec.data() : nullptr);
            if (rc) return rc;
            int64_t u = 0;
            for (size_t j = 0; j < grp.size(); ++j) {
                const int64_t i = grp[j];
                results[i] = sub_res[j];
                if (usage)
                    for (int64_t q = use_off[i]; q < use_off[i + 1]; ++q) usage[q] = sub_use[u++];
                if (records)
                    for (int64_t q = offsets[i]; q < offsets[i + 1]; ++q) records[q] = sub_rec[off[j] + (q - offsets[i])];
            }
        }
        return MSV_OK;
    }
    msv_grid* g = nullptr;
    int rc = grid_build(ctx, scenarios, n, tail_p, n_tails, offsets, arrival_ms, batch, records != nullptr, &g, nullptr, true);
    if (rc) return rc;
    std::unique_ptr<msv_grid> guard(g);
    rc = grid_launch(g);
    if (rc) return rc;
    return grid_results(g, results, usage, records, nullptr);
}

// run() with execution noise (engine.hpp:140-145): K5 (msv_noise.cu), one warp.
int msv_run_noise(msv_ctx* ctx, const msv_scenario* scenario, int64_t n, const double* arrival_ms,
                  const int32_t* batch, const double* noise_mult, msv_result* result, msv_usage* usage,
                  msv_record* records) {
    if (!ctx || !scenario || !result || (n > 0 && (!arrival_ms || !batch || !noise_mult || !records)))
        return fail(MSV_PARAM, "null argument");
    if (n < 0 || n >= (int64_t)UINT32_MAX) return fail(MSV_PARAM, "run: trace length out of range");
    SetDevice sd(ctx->device);
    const msv_scenario& sc = *scenario;
    int32_t P = 0;
    int rc = validate_scenario(ctx, sc, false, &P);
    if (rc) return rc;
    if ((int64_t)ctx->profiles[sc.profile].lat.size() > msv::kMaxSmemCells)
        return fail(MSV_PARAM, "run: profile has more than " + std::to_string(msv::kMaxSmemCells) +
                                   " (size, batch) cells, the device table limit");
    for (int64_t i = 1; i < n; ++i)
        if (arrival_ms[i] < arrival_ms[i - 1]) return fail(MSV_PARAM, "run: trace must be sorted by arrival");
    const Profile& prof = ctx->profiles[sc.profile];
    const std::vector<DevPart> parts = plan_parts(ctx->plans[sc.plan], prof, 0);
    std::vector<uint64_t> masks;
    if (sc.routing >= 0) masks = route_masks(parts, ctx->routings[sc.routing], prof.b_max);
    const size_t nn = (size_t)std::max<int64_t>(n, 1);
    msv_ctx::NoiseRunBufs& nb = ctx->noise1;
    DevBuf &d_arr = nb.arr, &d_bat = nb.bat, &d_mult = nb.mult, &d_lat = nb.lat, &d_util = nb.util,
           &d_parts = nb.parts, &d_masks = nb.masks, &d_next = nb.next, &d_rec = nb.rec, &d_use = nb.use,
           &d_out = nb.out;
    MSV_CUDA_TRY(d_arr.ensure(nn * 8));
    MSV_CUDA_TRY(d_bat.ensure(nn * 4));
    MSV_CUDA_TRY(d_mult.ensure(nn * 8));
    MSV_CUDA_TRY(d_lat.ensure(prof.lat.size() * 8));
    MSV_CUDA_TRY(d_util.ensure(prof.util.size() * 8));
    MSV_CUDA_TRY(d_parts.ensure(parts.size() * sizeof(DevPart)));
    MSV_CUDA_TRY(d_masks.ensure(std::max<size_t>(masks.size(), 1) * 8));
    MSV_CUDA_TRY(d_next.ensure(nn * 4));
    MSV_CUDA_TRY(d_rec.ensure(nn * sizeof(msv_record)));
    MSV_CUDA_TRY(d_use.ensure((size_t)P * sizeof(msv_usage)));
    MSV_CUDA_TRY(d_out.ensure(sizeof(DevOut)));
    cudaStream_t st = ctx->stream;
    if (n > 0) {
        MSV_CUDA_TRY(cudaMemcpyAsync(d_arr.p, arrival_ms, (size_t)n * 8, cudaMemcpyHostToDevice, st));
        MSV_CUDA_TRY(cudaMemcpyAsync(d_bat.p, batch, (size_t)n * 4, cudaMemcpyHostToDevice, st));
        MSV_CUDA_TRY(cudaMemcpyAsync(d_mult.p, noise_mult, (size_t)n * 8, cudaMemcpyHostToDevice, st));
    }
    MSV_CUDA_TRY(cudaMemcpyAsync(d_lat.p, prof.lat.data(), prof.lat.size() * 8, cudaMemcpyHostToDevice, st));
    MSV_CUDA_TRY(cudaMemcpyAsync(d_util.p, prof.util.data(), prof.util.size() * 8, cudaMemcpyHostToDevice, st));
    MSV_CUDA_TRY(
        cudaMemcpyAsync(d_parts.p, parts.data(), parts.size() * sizeof(DevPart), cudaMemcpyHostToDevice, st));
    if (!masks.empty())
        MSV_CUDA_TRY(cudaMemcpyAsync(d_masks.p, masks.data(), masks.size() * 8, cudaMemcpyHostToDevice, st));
    MSV_CUDA_TRY(cudaMemsetAsync(d_rec.p, 0, nn * sizeof(msv_record), st));
    MSV_CUDA_TRY(cudaMemsetAsync(d_out.p, 0, sizeof(DevOut), st));
    ctx->h2d += n * 20 + (int64_t)(prof.lat.size() * 16 + parts.size() * sizeof(DevPart) + masks.size() * 8);
    msv::NoiseParams np{};
    np.arrival = d_arr.as<double>();
    np.batch = d_bat.as<int32_t>();
    np.n = n;
    np.mult = d_mult.as<double>();
    np.lat = d_lat.as<double>();
    np.util = d_util.as<double>();
    np.parts = d_parts.as<DevPart>();
    np.n_cells = (int32_t)prof.lat.size();
    np.route_mask = masks.empty() ? nullptr : d_masks.as<uint64_t>();
    np.P = P;
    np.b_max = prof.b_max;
    np.sched = sc.scheduler;
    np.sla = sc.sla_ms;
    np.alpha = sc.alpha;
    np.beta = sc.beta;
    np.warmup_ms = sc.warmup_fraction * sc.duration_ms;  // engine.hpp:236
    np.next = d_next.as<uint32_t>();
    np.records = d_rec.as<msv_record>();
    np.usage = d_use.as<msv_usage>();
    np.out = d_out.as<DevOut>();
    np.n_ptr = nullptr;
    np.samples = nullptr;
    np.duration_ms = sc.duration_ms;
    DevBuf& d_job = nb.job;
    MSV_CUDA_TRY(d_job.ensure(sizeof(msv::NoiseParams)));
    MSV_CUDA_TRY(cudaMemcpyAsync(d_job.p, &np, sizeof np, cudaMemcpyHostToDevice, st));
    MSV_CUDA_TRY(msv::launch_noise(d_job.as<msv::NoiseParams>(), 1, np.n_cells, P, st));
    ctx->launches += 1;
    DevOut o{};
    MSV_CUDA_TRY(cudaMemcpyAsync(&o, d_out.p, sizeof(DevOut), cudaMemcpyDeviceToHost, st));
    if (n > 0)
        MSV_CUDA_TRY(cudaMemcpyAsync(records, d_rec.p, (size_t)n * sizeof(msv_record), cudaMemcpyDeviceToHost, st));
    if (usage)
        MSV_CUDA_TRY(cudaMemcpyAsync(usage, d_use.p, (size_t)P * sizeof(msv_usage), cudaMemcpyDeviceToHost, st));
    MSV_CUDA_TRY(cudaStreamSynchronize(st));
    ctx->d2h += (int64_t)sizeof(DevOut) + n * (int64_t)sizeof(msv_record) + (usage ? P * (int64_t)sizeof(msv_usage) : 0);
    if (o.status) return fail(o.status, "run: profile lookup outside the grid (LookupError)");
    msv_result& r = *result;
    r = msv_result{};
    r.total = n;
    r.violations = o.violations;
    r.measured = o.measured;
    r.measured_violations = o.measured_violations;
    for (double& t : r.tail) t = std::numeric_limits<double>::quiet_NaN();
    r.horizon_ms = sc.duration_ms < o.horizon_ms ? o.horizon_ms : sc.duration_ms;  // engine.hpp:235
    r.warmup_ms = np.warmup_ms;
    r.max_wait_estimate_diff = 0.0;  // the reference skips the check under noise (engine.hpp:208)
    r.duration_ms = sc.duration_ms;
    r.placement_hash = o.hash;
    r.status = MSV_OK;
    r.n_partitions = P;
    return MSV_OK;
}

int msv_sample_trace(msv_ctx* ctx, int32_t dist, double rate_qps, double duration_ms, uint64_t seed, int64_t cap,
                     double* arrival_ms, int32_t* batch, int64_t* n_out) {
    if (!ctx || !n_out) return fail(MSV_PARAM, "null argument");
    if (!(rate_qps > 0.0)) return fail(MSV_PARAM, "sample_trace: rate must be > 0");
    if (duration_ms < 0.0) return fail(MSV_PARAM, "sample_trace: duration must be >= 0");
    if (dist < 0 || dist >= (int)ctx->dists.size()) return fail(MSV_PARAM, "sample_trace: unknown dist handle");
    if (cap < 0) return fail(MSV_PARAM, "sample_trace: negative capacity");
    SetDevice sd(ctx->device);
    int rc = ctx->sync_tables();
    if (rc) return rc;
    DevBuf d_arr, d_bat, d_job, d_n, d_ovf;
    const int64_t c = std::max<int64_t>(cap, 1);
    MSV_CUDA_TRY(d_arr.ensure(c * 8));
    MSV_CUDA_TRY(d_bat.ensure(c * 4));
    MSV_CUDA_TRY(d_job.ensure(sizeof(msv::TraceJob)));
    MSV_CUDA_TRY(d_n.ensure(8));
    MSV_CUDA_TRY(d_ovf.ensure(4));
    msv::TraceJob j;
    j.seed = seed;
    j.rate_per_ms = rate_qps / 1000.0;
    j.duration_ms = duration_ms;
    j.cdf = ctx->d_cdf.as<double>() + ctx->dists[dist].dev_off;
    j.guide = ctx->d_guide.as<int16_t>() + ctx->dists[dist].guide_off;
    j.b_max = (int32_t)ctx->dists[dist].cdf.size();
    j.pad = 0;
    j.arrival = d_arr.as<double>();
    j.batch = d_bat.as<int32_t>();
    j.cap = cap;
    j.n_out = d_n.as<int64_t>();
    j.overflow = d_ovf.as<int32_t>();
    MSV_CUDA_TRY(cudaMemcpyAsync(d_job.p, &j, sizeof j, cudaMemcpyHostToDevice, ctx->stream));
    MSV_CUDA_TRY(msv::launch_trace_gen(d_job.as<msv::TraceJob>(), 1, ctx->log1p, ctx->stream));
    ctx->launches += 1;
    int64_t nn = 0;
    int32_t ovf = 0;
    MSV_CUDA_TRY(cudaMemcpyAsync(&nn, d_n.p, 8, cudaMemcpyDeviceToHost, ctx->stream));
    MSV_CUDA_TRY(cudaMemcpyAsync(&ovf, d_ovf.p, 4, cudaMemcpyDeviceToHost, ctx->stream));
    MSV_CUDA_TRY(cudaStreamSynchronize(ctx->stream));
    if (ovf) {
        *n_out = cap + 1;
        return fail(MSV_PARAM, "sample_trace: capacity " + std::to_string(cap) + " too small");
    }
    *n_out = nn;
    if (nn) {
        MSV_CUDA_TRY(cudaMemcpy(arrival_ms, d_arr.p, nn * 8, cudaMemcpyDeviceToHost));
        MSV_CUDA_TRY(cudaMemcpy(batch, d_bat.p, nn * 4, cudaMemcpyDeviceToHost));
    }
    return MSV_OK;
}

// tail_latency(samples, p) (metrics.hpp:22-29) on the device.
int msv_tail_latency(msv_ctx* ctx, const double* samples, int64_t n, const double* p, int n_p, double* out) {
    if (!ctx || !out || (n > 0 && !samples)) return fail(MSV_PARAM, "null argument");
    if (n <= 0) return fail(MSV_PARAM, "tail_latency: no samples");
    if (n_p < 1 || n_p > 4) return fail(MSV_PARAM, "tail_latency: between 1 and 4 percentiles");
    for (int j = 0; j < n_p; ++j)
        if (!(p[j] > 0.0) || !(p[j] < 1.0)) return fail(MSV_PARAM, "tail_latency: percentile must be in (0,1)");
    SetDevice sd(ctx->device);
    DevBuf d_s, d_out, d_job, d_p, d_res, d_cand;
    MSV_CUDA_TRY(d_s.ensure(n * 8));
    // candidate scratch for K3's gather pass (a larger bin takes the full-data passes)
    const int64_t cand_cap = std::min<int64_t>(n / 2 + 1, (int64_t)1 << 24);
    MSV_CUDA_TRY(d_cand.ensure(cand_cap * 8));
    MSV_CUDA_TRY(d_out.ensure(sizeof(DevOut)));
    MSV_CUDA_TRY(d_job.ensure(sizeof(msv::TailJob)));
    MSV_CUDA_TRY(d_p.ensure(n_p * 8));
    MSV_CUDA_TRY(d_res.ensure(4 * 8));
    const double* src = samples;
    DevOut o;
    memset(&o, 0, sizeof o);
    o.n_samples = n;
    o.lat_min_bits = ~0ull;  // min > max: the kernel derives the key range itself
    o.lat_max_bits = 0;
    msv::TailJob j;
    j.samples = d_s.as<double>();
    j.src = d_out.as<DevOut>();
    j.out = d_res.as<double>();
    j.cand = d_cand.as<uint64_t>();
    j.cand_cap = cand_cap;
    MSV_CUDA_TRY(cudaMemcpyAsync(d_s.p, src, n * 8, cudaMemcpyHostToDevice, ctx->stream));
    MSV_CUDA_TRY(cudaMemcpyAsync(d_out.p, &o, sizeof o, cudaMemcpyHostToDevice, ctx->stream));
    MSV_CUDA_TRY(cudaMemcpyAsync(d_job.p, &j, sizeof j, cudaMemcpyHostToDevice, ctx->stream));
    MSV_CUDA_TRY(cudaMemcpyAsync(d_p.p, p, n_p * 8, cudaMemcpyHostToDevice, ctx->stream));
    MSV_CUDA_TRY(msv::launch_tail(d_job.as<msv::TailJob>(), 1, d_p.as<double>(), n_p, ctx->stream));
    ctx->launches += 1;
    MSV_CUDA_TRY(cudaMemcpyAsync(out, d_res.p, n_p * 8, cudaMemcpyDeviceToHost, ctx->stream));
    MSV_CUDA_TRY(cudaStreamSynchronize(ctx->stream));
    return MSV_OK;
}

int msv_paris_batch(msv_ctx* ctx, const msv_paris_job* jobs, int64_t n_jobs, msv_paris_out* out, int32_t* n_per_gpu,
                    int32_t* sizes_flat) {
    if (!ctx || (n_jobs > 0 && (!jobs || !out || !n_per_gpu || !sizes_flat))) return fail(MSV_PARAM, "null argument");
    if (n_jobs <= 0) return MSV_OK;
    std::vector<msv::ParisJobDev> dj((size_t)n_jobs);
    int64_t gpu_total = 0, inst_total = 0;
    for (int64_t j = 0; j < n_jobs; ++j) {
        const msv_paris_job& a = jobs[j];
        if (a.profile < 0 || a.profile >= (int)ctx->profiles.size()) return fail(MSV_PARAM, "unknown profile handle");
        if (a.dist < 0 || a.dist >= (int)ctx->dists.size()) return fail(MSV_PARAM, "unknown distribution handle");
        const int64_t g = a.num_gpus >= 1 && a.gpcs_per_gpu >= 1 ? a.num_gpus : 0;
        const int64_t c = g ? (int64_t)a.num_gpus * a.gpcs_per_gpu : 0;
        if (c > (int64_t)1 << 24) return fail(MSV_PARAM, "paris batch: num_gpus * gpcs_per_gpu too large");
        msv::ParisJobDev& d = dj[(size_t)j];
        d.gpu_off = gpu_total;
        d.inst_off = inst_total;
        gpu_total += g;
        inst_total += c;
        d.total_gpcs = a.total_gpcs;
        d.num_gpus = a.num_gpus;
        d.gpcs_per_gpu = a.gpcs_per_gpu;
        d.knee_threshold = a.knee_threshold;
        d.pad = 0;
    }
    SetDevice sd(ctx->device);
    int rc = ctx->sync_tables();
    if (rc) return rc;
    for (int64_t j = 0; j < n_jobs; ++j) {
        const Profile& pr = ctx->profiles[jobs[j].profile];
        const Dist& di = ctx->dists[jobs[j].dist];
        msv::ParisJobDev& d = dj[(size_t)j];
        d.row0 = pr.cell_off;
        d.n_sizes = (int32_t)pr.sizes.size();
        d.b_max = pr.b_max;
        d.dist_b_max = (int32_t)di.pmf.size();
        d.pmf_off = (int64_t)di.dev_off;
        d.sizes = ctx->d_sizes.as<int32_t>() + pr.size_off;
        if (d.n_sizes > MSV_PARIS_MAX_SIZES) {
            d.pad = MSV_PARAM;  // reported per job; the kernel only writes the status
            d.n_sizes = 0;
        }
    }
    DevBuf b_jobs, b_out, b_per, b_flat, b_rem;
    MSV_CUDA_TRY(b_jobs.ensure(dj.size() * sizeof(msv::ParisJobDev)));
    MSV_CUDA_TRY(b_out.ensure((size_t)n_jobs * sizeof(msv_paris_out)));
    MSV_CUDA_TRY(b_per.ensure((size_t)std::max<int64_t>(gpu_total, 1) * 4));
    MSV_CUDA_TRY(b_rem.ensure((size_t)std::max<int64_t>(gpu_total, 1) * 4));
    MSV_CUDA_TRY(b_flat.ensure((size_t)std::max<int64_t>(inst_total, 1) * 4));
    MSV_CUDA_TRY(cudaMemcpyAsync(b_jobs.p, dj.data(), dj.size() * sizeof(msv::ParisJobDev), cudaMemcpyHostToDevice,
                                 ctx->stream));
    ctx->h2d += (int64_t)(dj.size() * sizeof(msv::ParisJobDev));
    msv::ParisParams pp;
    pp.jobs = b_jobs.as<msv::ParisJobDev>();
    pp.n_jobs = n_jobs;
    pp.lat = ctx->d_lat.as<double>();
    pp.util = ctx->d_util.as<double>();
    pp.pmf = ctx->d_pmf.as<double>();
    pp.out = b_out.as<msv_paris_out>();
    pp.n_per_gpu = b_per.as<int32_t>();
    pp.sizes_flat = b_flat.as<int32_t>();
    pp.remaining = b_rem.as<int32_t>();
    MSV_CUDA_TRY(msv::launch_paris(pp, ctx->stream));
    debug_sync(ctx->stream, "paris");
    ctx->launches += 1;
    MSV_CUDA_TRY(cudaMemcpyAsync(out, b_out.p, (size_t)n_jobs * sizeof(msv_paris_out), cudaMemcpyDeviceToHost,
                                 ctx->stream));
    if (gpu_total)
        MSV_CUDA_TRY(cudaMemcpyAsync(n_per_gpu, b_per.p, (size_t)gpu_total * 4, cudaMemcpyDeviceToHost, ctx->stream));
    if (inst_total)
        MSV_CUDA_TRY(
            cudaMemcpyAsync(sizes_flat, b_flat.p, (size_t)inst_total * 4, cudaMemcpyDeviceToHost, ctx->stream));
    MSV_CUDA_TRY(cudaStreamSynchronize(ctx->stream));
    ctx->d2h += (int64_t)n_jobs * (int64_t)sizeof(msv_paris_out) + 4 * (gpu_total + inst_total);
    return MSV_OK;
}

int msv_dispatch_batch(msv_ctx* ctx, int32_t profile, int scheduler, int64_t n_trials, const int64_t* part_off,
                       const int32_t* part_id, const int32_t* part_k, const uint8_t* busy, const double* cur_est,
                       const double* cur_start, const int64_t* q_off, const int32_t* qbatch,
                       const int32_t* query_batch, const double* now_ms, const double* sla_ms, const double* alpha,
                       const double* beta, int32_t* chosen, int32_t* kind, double* t_wait_out) {
    if (!ctx || !part_off || !chosen || !kind) return fail(MSV_PARAM, "null argument");
    // fifs_dispatch takes no table (sched.hpp:154): profile -1 is allowed for FIFS
    // decisions that do not request t_wait.
    const bool no_table = profile == -1 && scheduler == MSV_FIFS && !t_wait_out;
    if (!no_table && (profile < 0 || profile >= (int)ctx->profiles.size()))
        return fail(MSV_PARAM, "unknown profile handle");
    if (scheduler != MSV_FIFS && scheduler != MSV_ELSA) return fail(MSV_VALIDATION, "unknown scheduler");
    if (n_trials <= 0) return MSV_OK;
    SetDevice sd(ctx->device);
    int rc = ctx->sync_tables();
    if (rc) return rc;
    static const Profile kEmpty;
    const Profile& prof = no_table ? kEmpty : ctx->profiles[profile];
    const int64_t np = part_off[n_trials] - part_off[0];
    const int64_t nqb = np ? q_off[part_off[n_trials]] - q_off[part_off[0]] : 0;
    if (part_off[0] != 0 || (np && q_off[0] != 0))
        return fail(MSV_PARAM, "dispatch: offsets must start at 0");
    for (int64_t t = 0; t < n_trials; ++t) {
        if (part_off[t + 1] <= part_off[t]) return fail(MSV_PARAM, "elsa_dispatch: no partitions");
        if (part_off[t + 1] - part_off[t] > 128) return fail(MSV_PARAM, "dispatch: at most 128 partitions per trial");
    }
    std::vector<int32_t> rows(np);
    for (int64_t j = 0; j < np; ++j) {
        auto it = std::lower_bound(prof.sizes.begin(), prof.sizes.end(), part_k[j]);
        rows[j] = (it == prof.sizes.end() || *it != part_k[j])
                      ? -1
                      : prof.cell_off + (int32_t)(it - prof.sizes.begin()) * prof.b_max;
    }
    DevBuf b_poff, b_pid, b_pk, b_row, b_busy, b_est, b_start, b_qoff, b_qb, b_qbat, b_now, b_sla, b_al, b_be,
        b_ch, b_kind, b_tw, b_err;
    auto up = [&](DevBuf& b, const void* src, size_t bytes) -> int {
        MSV_CUDA_TRY(b.ensure(bytes ? bytes : 16));
        if (bytes) MSV_CUDA_TRY(cudaMemcpyAsync(b.p, src, bytes, cudaMemcpyHostToDevice, ctx->stream));
        return MSV_OK;
    };
    if ((rc = up(b_poff, part_off, (n_trials + 1) * 8)) || (rc = up(b_pid, part_id, np * 4)) ||
        (rc = up(b_pk, part_k, np * 4)) || (rc = up(b_row, rows.data(), np * 4)) || (rc = up(b_busy, busy, np)) ||
        (rc = up(b_est, cur_est, np * 8)) || (rc = up(b_start, cur_start, np * 8)) ||
        (rc = up(b_qoff, q_off, (np + 1) * 8)) || (rc = up(b_qb, qbatch, nqb * 4)) ||
        (rc = up(b_qbat, query_batch, n_trials * 4)) || (rc = up(b_now, now_ms, n_trials * 8)) ||
        (rc = up(b_sla, sla_ms, n_trials * 8)) || (rc = up(b_al, alpha, n_trials * 8)) ||
        (rc = up(b_be, beta, n_trials * 8)))
        return rc;
    MSV_CUDA_TRY(b_ch.ensure(n_trials * 4));
    MSV_CUDA_TRY(b_kind.ensure(n_trials * 4));
    MSV_CUDA_TRY(b_err.ensure(n_trials * 4));
    if (t_wait_out) MSV_CUDA_TRY(b_tw.ensure(np * 8));
    msv::DispatchParams p;
    p.n_trials = n_trials;
    p.part_off = b_poff.as<int64_t>();
    p.part_id = b_pid.as<int32_t>();
    p.part_k = b_pk.as<int32_t>();
    p.part_row = b_row.as<int32_t>();
    p.busy = b_busy.as<uint8_t>();
    p.cur_est = b_est.as<double>();
    p.cur_start = b_start.as<double>();
    p.q_off = b_qoff.as<int64_t>();
    p.qbatch = b_qb.as<int32_t>();
    p.query_batch = b_qbat.as<int32_t>();
    p.now_ms = b_now.as<double>();
    p.sla_ms = b_sla.as<double>();
    p.alpha = b_al.as<double>();
    p.beta = b_be.as<double>();
    p.lat = ctx->d_lat.as<double>();
    p.b_max = prof.b_max;
    p.scheduler = scheduler;
    p.chosen = b_ch.as<int32_t>();
    p.kind = b_kind.as<int32_t>();
    p.t_wait_out = t_wait_out ? b_tw.as<double>() : nullptr;
    p.error = b_err.as<int32_t>();
    MSV_CUDA_TRY(msv::launch_dispatch(p, ctx->stream));
    ctx->launches += 1;
    std::vector<int32_t> err(n_trials);
    MSV_CUDA_TRY(cudaMemcpyAsync(chosen, b_ch.p, n_trials * 4, cudaMemcpyDeviceToHost, ctx->stream));
    MSV_CUDA_TRY(cudaMemcpyAsync(kind, b_kind.p, n_trials * 4, cudaMemcpyDeviceToHost, ctx->stream));
    MSV_CUDA_TRY(cudaMemcpyAsync(err.data(), b_err.p, n_trials * 4, cudaMemcpyDeviceToHost, ctx->stream));
    if (t_wait_out) MSV_CUDA_TRY(cudaMemcpyAsync(t_wait_out, b_tw.p, np * 8, cudaMemcpyDeviceToHost, ctx->stream));
    MSV_CUDA_TRY(cudaStreamSynchronize(ctx->stream));
    for (int64_t t = 0; t < n_trials; ++t)
        if (err[t]) return fail(err[t], "trial " + std::to_string(t) + ": profile lookup outside the grid");
    return MSV_OK;
}

// ---- arithmetic self-checks (msv_selftest.cu) ----
int msv_log1p_digest(msv_ctx* ctx, int variant, uint64_t seed, int64_t n, int64_t chunk, uint64_t* digests) {
    if (!ctx || !digests || n < 0 || chunk <= 0) return fail(MSV_PARAM, "msv_log1p_digest: bad argument");
    if (variant != MSV_LOG1P_GENERIC && variant != MSV_LOG1P_FMA) return fail(MSV_PARAM, "unknown log1p variant");
    if (n == 0) return MSV_OK;
    SetDevice sd(ctx->device);
    const int64_t n_chunks = (n + chunk - 1) / chunk;
    DevBuf d;
    MSV_CUDA_TRY(d.ensure(n_chunks * 8));
    MSV_CUDA_TRY(msv::launch_log1p_digest(variant, seed, n, chunk, d.as<uint64_t>(), ctx->stream));
    ctx->launches += 1;
    MSV_CUDA_TRY(cudaMemcpyAsync(digests, d.p, n_chunks * 8, cudaMemcpyDeviceToHost, ctx->stream));
    MSV_CUDA_TRY(cudaStreamSynchronize(ctx->stream));
    return MSV_OK;
}

int msv_log1p_values(msv_ctx* ctx, int variant, uint64_t seed, int64_t first, int64_t count, double* out) {
    if (!ctx || !out || first < 0 || count < 0) return fail(MSV_PARAM, "msv_log1p_values: bad argument");
    if (variant != MSV_LOG1P_GENERIC && variant != MSV_LOG1P_FMA) return fail(MSV_PARAM, "unknown log1p variant");
    if (count == 0) return MSV_OK;
    SetDevice sd(ctx->device);
    DevBuf d;
    MSV_CUDA_TRY(d.ensure(count * 8));
    MSV_CUDA_TRY(msv::launch_log1p_values(variant, seed, first, count, d.as<double>(), ctx->stream));
    ctx->launches += 1;
    MSV_CUDA_TRY(cudaMemcpyAsync(out, d.p, count * 8, cudaMemcpyDeviceToHost, ctx->stream));
    MSV_CUDA_TRY(cudaStreamSynchronize(ctx->stream));
    return MSV_OK;
}

int msv_quotient_check(msv_ctx* ctx, uint64_t seed, int64_t n, int64_t* counts) {
    if (!ctx || !counts || n < 0) return fail(MSV_PARAM, "msv_quotient_check: bad argument");
    SetDevice sd(ctx->device);
    DevBuf d;
    MSV_CUDA_TRY(d.ensure(16));
    MSV_CUDA_TRY(cudaMemsetAsync(d.p, 0, 16, ctx->stream));
    MSV_CUDA_TRY(msv::launch_quotient_check(seed, n, d.as<unsigned long long>(), ctx->stream));
    ctx->launches += 1;
    unsigned long long h[2] = {0, 0};
    MSV_CUDA_TRY(cudaMemcpyAsync(h, d.p, 16, cudaMemcpyDeviceToHost, ctx->stream));
    MSV_CUDA_TRY(cudaStreamSynchronize(ctx->stream));
    counts[0] = (int64_t)h[0];
    counts[1] = (int64_t)h[1];
    return MSV_OK;
}

}  // extern "C"

// ---------------------------------------------------------------------------------
// Multi-device contexts (msv_create_multi). Scenarios are independent,
// so a grid is cut into contiguous, cost-balanced shards — one per member context, each
// on its own GPU — run concurrently (one host thread per member, no device-to-device
// traffic), and the fixed-size per-scenario results are gathered into the caller's
// arrays in scenario order. The reference fans best_homogeneous out the same way with
// std::async (metrics.hpp:183-209); here every batch entry point does.
// ---------------------------------------------------------------------------------
namespace {

std::vector<msv_ctx*> members(msv_ctx* ctx) {
    std::vector<msv_ctx*> m{ctx};
    m.insert(m.end(), ctx->peers.begin(), ctx->peers.end());
    return m;
}

// Mirror the primary's uploads (host copies; device tables re-synced lazily).
void sync_peers(msv_ctx* ctx) {
    if (ctx->mirrored_serial == ctx->upload_serial) return;
    for (msv_ctx* p : ctx->peers) {
        p->profiles = ctx->profiles;
        p->dists = ctx->dists;
        p->plans = ctx->plans;
        p->routings = ctx->routings;
        p->log1p = ctx->log1p;
        p->tables_dirty = true;
    }
    ctx->mirrored_serial = ctx->upload_serial;
}

// Contiguous shards of [0, n) with about equal cost (expected queries x (P + 1)); the
// same cut distributed.shard makes for one-process-per-GPU runs.
std::vector<int64_t> shard_cuts(const msv_ctx* ctx, const msv_scenario* sc, int64_t n, const int64_t* offsets,
                                int parts) {
    std::vector<double> cum(n + 1, 0.0);
    for (int64_t i = 0; i < n; ++i) {
        const msv_scenario& s = sc[i];
        const double q = offsets ? (double)(offsets[i + 1] - offsets[i]) : s.rate_qps * s.duration_ms / 1000.0;
        const double P = (s.plan >= 0 && s.plan < (int)ctx->plans.size()) ? (double)ctx->plans[s.plan].flat.size() : 1.0;
        cum[i + 1] = cum[i] + (q > 0.0 ? q : 0.0) * (P + 1.0) + 1e-9;
    }
    std::vector<int64_t> cut(parts + 1, 0);
    cut[parts] = n;
    for (int k = 1; k < parts; ++k) {
        const double target = cum[n] * k / parts;
        cut[k] = std::upper_bound(cum.begin(), cum.end(), target) - cum.begin() - 1;
        cut[k] = std::max(cut[k], cut[k - 1]);
    }
    return cut;
}

// Run fn(member k, shard k) for every member concurrently (member 0 on this thread);
// returns the first failing member's status with its message.
template <typename Fn>
int fan_out(const std::vector<msv_ctx*>& m, Fn fn) {
    std::vector<int> rc(m.size(), MSV_OK);
    std::vector<std::string> err(m.size());
    std::vector<std::thread> th;
    for (size_t k = 1; k < m.size(); ++k)
        th.emplace_back([&, k] {
            rc[k] = fn(k);
            if (rc[k]) err[k] = g_err;
        });
    rc[0] = fn(0);
    if (rc[0]) err[0] = g_err;
    for (std::thread& t : th) t.join();
    for (size_t k = 0; k < m.size(); ++k)
        if (rc[k]) return fail(rc[k], "device " + std::to_string(m[k]->device) + " (member " + std::to_string(k) +
                                          "): " + err[k]);
    return MSV_OK;
}

// Usage slots before scenario i (Σ P over earlier scenarios).
std::vector<int64_t> usage_prefix(const msv_ctx* ctx, const msv_scenario* sc, int64_t n) {
    std::vector<int64_t> u(n + 1, 0);
    for (int64_t i = 0; i < n; ++i) {
        const int p = sc[i].plan;
        u[i + 1] = u[i] + ((p >= 0 && p < (int)ctx->plans.size()) ? (int64_t)ctx->plans[p].flat.size() : 0);
    }
    return u;
}

}  // namespace

extern "C" {

int msv_create_multi(const int* device_ids, int n_devices, msv_ctx** out) {
    if (!out || !device_ids || n_devices < 1) return fail(MSV_PARAM, "msv_create_multi: need >= 1 device");
    *out = nullptr;
    msv_ctx* primary = nullptr;
    int rc = msv_create(device_ids[0], &primary);
    if (rc) return rc;
    std::unique_ptr<msv_ctx, int (*)(msv_ctx*)> guard(primary, msv_destroy);
    for (int k = 1; k < n_devices; ++k) {
        msv_ctx* p = nullptr;
        rc = msv_create(device_ids[k], &p);
        if (rc) return rc;
        primary->peers.push_back(p);
    }
    for (msv_ctx* a : members(primary)) {
        a->share = 0;
        for (msv_ctx* b : members(primary)) a->share += a->device == b->device;
    }
    *out = guard.release();
    return MSV_OK;
}

int msv_context_devices(msv_ctx* ctx, int* device_ids, int cap) {
    if (!ctx) return fail(MSV_PARAM, "null context");
    const std::vector<msv_ctx*> m = members(ctx);
    for (int k = 0; k < (int)m.size() && k < cap; ++k) device_ids[k] = m[k]->device;
    return (int)m.size();
}

int msv_run_grid(msv_ctx* ctx, const msv_scenario* scenarios, int64_t n, const double* tail_p, int n_tails,
                 msv_result* results, msv_usage* usage) {
    if (!ctx || (n > 0 && (!scenarios || !results))) return fail(MSV_PARAM, "null argument");
    if (ctx->peers.empty()) return run_grid_dev(ctx, scenarios, n, tail_p, n_tails, results, usage);
    sync_peers(ctx);
    const std::vector<msv_ctx*> m = members(ctx);
    const std::vector<int64_t> cut = shard_cuts(ctx, scenarios, n, nullptr, (int)m.size());
    const std::vector<int64_t> uo = usage_prefix(ctx, scenarios, n);
    return fan_out(m, [&](size_t k) {
        const int64_t lo = cut[k], hi = cut[k + 1];
        if (hi <= lo) return (int)MSV_OK;
        return run_grid_dev(m[k], scenarios + lo, hi - lo, tail_p, n_tails, results + lo,
                            usage ? usage + uo[lo] : nullptr);
    });
}

int msv_run_replay(msv_ctx* ctx, const msv_scenario* scenarios, int64_t n, const int64_t* offsets,
                   const double* arrival_ms, const int32_t* batch, const double* tail_p, int n_tails,
                   msv_result* results, msv_usage* usage, msv_record* records) {
    if (!ctx || (n > 0 && (!scenarios || !results || !offsets))) return fail(MSV_PARAM, "null argument");
    if (ctx->peers.empty())
        return run_replay_dev(ctx, scenarios, n, offsets, arrival_ms, batch, tail_p, n_tails, results, usage, records);
    sync_peers(ctx);
    const std::vector<msv_ctx*> m = members(ctx);
    const std::vector<int64_t> cut = shard_cuts(ctx, scenarios, n, offsets, (int)m.size());
    const std::vector<int64_t> uo = usage_prefix(ctx, scenarios, n);
    return fan_out(m, [&](size_t k) {
        const int64_t lo = cut[k], hi = cut[k + 1];
        if (hi <= lo) return (int)MSV_OK;
        std::vector<int64_t> off(offsets + lo, offsets + hi + 1);  // rebased: the shard's traces start at 0
        const int64_t q0 = off[0];
        for (int64_t& o : off) o -= q0;
        return run_replay_dev(m[k], scenarios + lo, hi - lo, off.data(), arrival_ms + q0, batch + q0, tail_p, n_tails,
                              results + lo, usage ? usage + uo[lo] : nullptr, records ? records + q0 : nullptr);
    });
}

int msv_grid_create(msv_ctx* ctx, const msv_scenario* scenarios, int64_t n, const double* tail_p, int n_tails,
                    msv_grid** out) {
    if (!ctx || !out || (n > 0 && !scenarios)) return fail(MSV_PARAM, "null argument");
    if (ctx->peers.empty()) return grid_create_dev(ctx, scenarios, n, tail_p, n_tails, out);
    sync_peers(ctx);
    const std::vector<msv_ctx*> m = members(ctx);
    std::unique_ptr<msv_grid> top(new msv_grid);
    top->ctx = ctx;
    top->n = n;
    top->tail_p.assign(tail_p, tail_p + std::max(n_tails, 0));
    top->dev_lo = shard_cuts(ctx, scenarios, n, nullptr, (int)m.size());
    const std::vector<int64_t> uo = usage_prefix(ctx, scenarios, n);
    for (size_t k = 0; k < m.size(); ++k) top->dev_use_lo.push_back(uo[top->dev_lo[k]]);
    top->usage_total = uo[n];
    top->dev_parts.resize(m.size());
    const int rc = fan_out(m, [&](size_t k) {
        msv_grid* g = nullptr;
        const int64_t lo = top->dev_lo[k], hi = top->dev_lo[k + 1];
        const int r = grid_create_dev(m[k], scenarios + lo, hi - lo, tail_p, n_tails, &g);
        top->dev_parts[k].reset(g);
        return r;
    });
    if (rc) {
        for (size_t k = 0; k < m.size(); ++k) {
            SetDevice sd(m[k]->device);
            top->dev_parts[k].reset();
        }
        return rc;
    }
    *out = top.release();
    return MSV_OK;
}

int msv_grid_launch(msv_grid* grid) {
    if (!grid) return fail(MSV_PARAM, "null grid");
    if (grid->dev_parts.empty()) return grid_launch_dev(grid);
    for (std::unique_ptr<msv_grid>& p : grid->dev_parts) {  // asynchronous: every device runs at once
        p->usage = grid->usage;
        p->overlap = grid->overlap;
        const int rc = grid_launch_dev(p.get());
        if (rc) return rc;
    }
    return MSV_OK;
}

int msv_grid_results(msv_grid* grid, msv_result* results, msv_usage* usage) {
    if (!grid || (grid->n > 0 && !results)) return fail(MSV_PARAM, "null argument");
    if (grid->dev_parts.empty()) return grid_results_dev(grid, results, usage);
    for (size_t k = 0; k < grid->dev_parts.size(); ++k) {
        const int rc = grid_results_dev(grid->dev_parts[k].get(), results + grid->dev_lo[k],
                                        usage ? usage + grid->dev_use_lo[k] : nullptr);
        if (rc) return rc;
    }
    return MSV_OK;
}

int msv_grid_destroy(msv_grid* grid) {
    if (!grid) return MSV_OK;
    for (std::unique_ptr<msv_grid>& p : grid->dev_parts) {
        SetDevice sd(p->ctx->device);
        cudaStreamSynchronize(p->ctx->stream);
        p.reset();
    }
    SetDevice sd(grid->ctx->device);
    cudaStreamSynchronize(grid->ctx->stream);
    delete grid;
    return MSV_OK;
}

// Multi-device grids: each stage is the max over the devices (they run concurrently).
int msv_grid_timing(msv_grid* g, float* total_ms, float* trace_ms, float* sim_ms, float* tail_ms) {
    if (!g) return fail(MSV_PARAM, "null grid");
    if (g->dev_parts.empty()) return grid_timing_dev(g, total_ms, trace_ms, sim_ms, tail_ms);
    float t[4] = {0, 0, 0, 0};
    for (std::unique_ptr<msv_grid>& p : g->dev_parts) {
        float v[4] = {0, 0, 0, 0};
        const int rc = grid_timing_dev(p.get(), &v[0], &v[1], &v[2], &v[3]);
        if (rc) return rc;
        for (int j = 0; j < 4; ++j) t[j] = std::max(t[j], v[j]);
    }
    if (total_ms) *total_ms = t[0];
    if (trace_ms) *trace_ms = t[1];
    if (sim_ms) *sim_ms = t[2];
    if (tail_ms) *tail_ms = t[3];
    return MSV_OK;
}

int64_t msv_grid_queries(msv_grid* g) {
    if (!g) return -1;
    if (g->dev_parts.empty()) return grid_queries_dev(g);
    int64_t t = 0;
    for (std::unique_ptr<msv_grid>& p : g->dev_parts) {
        const int64_t q = grid_queries_dev(p.get());
        if (q < 0) return -1;
        t += q;
    }
    return t;
}

}  // extern "C"

// ---------------------------------------------------------------------------------
// Noisy grids (execution noise at grid scale, engine.hpp:140-145): K1 generates every
// scenario's trace on the device, the host draws each scenario's multiplier stream with
// the reference's Rng and libm (rng.hpp:27-32; msv_noise_multipliers, one host thread per
// core), K5 runs one warp per scenario in global (time, seq) event order, K3 selects the
// tails from the measured latencies K5 leaves over the arrivals. Buffers are the
// context's, reused across calls.
// ---------------------------------------------------------------------------------
extern "C" int msv_noise_multipliers(uint64_t seed, double sigma, int64_t n, double* out);

namespace {

int run_grid_noise_dev(msv_ctx* ctx, const msv_scenario* sc, int64_t n, const double* sigma, const uint64_t* nseed,
                       const double* tail_p, int n_tails, msv_result* results, msv_usage* usage,
                       const int64_t* cap_override) {
    if (n_tails < 0 || n_tails > 4) return fail(MSV_PARAM, "grid: between 0 and 4 tail percentiles");
    for (int j = 0; j < n_tails; ++j)
        if (!(tail_p[j] > 0.0) || !(tail_p[j] < 1.0))
            return fail(MSV_PARAM, "tail_latency: percentile must be in (0,1)");
    SetDevice sd(ctx->device);
    PhaseTimer pt;
    int rc = ctx->sync_tables();
    if (rc) return rc;
    std::vector<int32_t> P(n);
    std::vector<int64_t> cap(n), toff(n + 1, 0), uoff(n + 1, 0);
    int max_cells = 0;
    for (int64_t i = 0; i < n; ++i) {
        rc = validate_scenario(ctx, sc[i], true, &P[i]);
        if (rc) {
            g_err = "scenario " + std::to_string(i) + ": " + g_err;
            return rc;
        }
        if (!(sigma[i] > 0.0)) return fail(MSV_PARAM, "scenario " + std::to_string(i) + ": noise_sigma must be > 0");
        const int cells = (int)ctx->profiles[sc[i].profile].lat.size();
        if (cells > msv::kMaxSmemCells) return fail(MSV_PARAM, "run: profile exceeds the device table limit");
        max_cells = std::max(max_cells, cells);
        cap[i] = cap_override ? cap_override[i] : trace_capacity(sc[i].rate_qps, sc[i].duration_ms);
        if (cap[i] < 0) return fail(MSV_PARAM, "sample_trace: expected trace too long");
        toff[i + 1] = toff[i] + cap[i];
        uoff[i + 1] = uoff[i] + P[i];
    }
    const int64_t total = toff[n];
    GridBufs& B = ctx->scratch;
    const size_t tq = (size_t)std::max<int64_t>(total, 1);
    MSV_CUDA_TRY(B.d_arr.ensure(tq * 8));
    MSV_CUDA_TRY(B.d_bat.ensure(tq * 4));
    MSV_CUDA_TRY(B.d_next.ensure(tq * 4));
    MSV_CUDA_TRY(ctx->d_mult.ensure(tq * 8));
    MSV_CUDA_TRY(B.d_out.ensure(std::max<int64_t>(n, 1) * sizeof(DevOut)));
    MSV_CUDA_TRY(B.d_nq.ensure(std::max<int64_t>(n, 1) * 8));
    MSV_CUDA_TRY(B.d_tovf.ensure(std::max<int64_t>(n, 1) * 4));
    MSV_CUDA_TRY(B.d_tjobs.ensure(std::max<int64_t>(n, 1) * sizeof(msv::TraceJob)));
    MSV_CUDA_TRY(B.d_tailjobs.ensure(std::max<int64_t>(n, 1) * sizeof(msv::TailJob)));
    MSV_CUDA_TRY(B.d_tails.ensure(std::max<int64_t>(n, 1) * 4 * sizeof(double)));
    MSV_CUDA_TRY(B.d_p.ensure(4 * sizeof(double)));
    MSV_CUDA_TRY(B.d_usage.ensure(std::max<int64_t>(uoff[n], 1) * sizeof(msv_usage)));
    MSV_CUDA_TRY(ctx->d_njobs.ensure(std::max<int64_t>(n, 1) * sizeof(msv::NoiseParams)));
    // partition tables (rows relative to each scenario's own profile) and routing masks
    std::vector<DevPart> parts_h;
    std::vector<uint64_t> masks_h;
    std::vector<size_t> poff(n), moff(n, (size_t)-1);
    for (int64_t i = 0; i < n; ++i) {
        const Profile& prof = ctx->profiles[sc[i].profile];
        const std::vector<DevPart> parts = plan_parts(ctx->plans[sc[i].plan], prof, 0);
        poff[i] = parts_h.size();
        parts_h.insert(parts_h.end(), parts.begin(), parts.end());
        if (sc[i].routing >= 0) {
            const std::vector<uint64_t> m = route_masks(parts, ctx->routings[sc[i].routing], prof.b_max);
            moff[i] = masks_h.size();
            masks_h.insert(masks_h.end(), m.begin(), m.end());
        }
    }
    MSV_CUDA_TRY(B.d_parts.ensure(std::max<size_t>(parts_h.size(), 1) * sizeof(DevPart)));
    MSV_CUDA_TRY(B.d_masks.ensure(std::max<size_t>(masks_h.size(), 1) * 8));
    std::vector<msv::TraceJob> tj(n);
    std::vector<msv::NoiseParams> nj(n);
    std::vector<msv::TailJob> lj(n);
    for (int64_t i = 0; i < n; ++i) {
        const msv_scenario& s = sc[i];
        const Profile& prof = ctx->profiles[s.profile];
        const Dist& ds = ctx->dists[s.dist];
        double* arr = B.d_arr.as<double>() + toff[i];
        int32_t* bat = B.d_bat.as<int32_t>() + toff[i];
        msv::TraceJob& t = tj[i];
        t.seed = s.seed;
        t.rate_per_ms = s.rate_qps / 1000.0;  // workload.hpp:103
        t.duration_ms = s.duration_ms;
        t.cdf = ctx->d_cdf.as<double>() + ds.dev_off;
        t.guide = ctx->d_guide.as<int16_t>() + ds.guide_off;
        t.b_max = (int32_t)ds.cdf.size();
        t.pad = 0;
        t.arrival = arr;
        t.batch = bat;
        t.cap = cap[i];
        t.n_out = B.d_nq.as<int64_t>() + i;
        t.overflow = B.d_tovf.as<int32_t>() + i;
        msv::NoiseParams& q = nj[i];
        q = msv::NoiseParams{};
        q.arrival = arr;
        q.batch = bat;
        q.n = 0;
        q.n_ptr = B.d_nq.as<int64_t>() + i;
        q.samples = arr;
        q.duration_ms = s.duration_ms;
        q.mult = ctx->d_mult.as<double>() + toff[i];
        q.lat = ctx->d_lat.as<double>() + prof.cell_off;
        q.util = ctx->d_util.as<double>() + prof.cell_off;
        q.parts = B.d_parts.as<DevPart>() + poff[i];
        q.route_mask = moff[i] == (size_t)-1 ? nullptr : B.d_masks.as<uint64_t>() + moff[i];
        q.P = P[i];
        q.b_max = prof.b_max;
        q.sched = s.scheduler;
        q.n_cells = (int32_t)prof.lat.size();
        q.sla = s.sla_ms;
        q.alpha = s.alpha;
        q.beta = s.beta;
        q.warmup_ms = s.warmup_fraction * s.duration_ms;  // engine.hpp:236
        q.next = B.d_next.as<uint32_t>() + toff[i];
        q.records = nullptr;
        q.usage = B.d_usage.as<msv_usage>() + uoff[i];
        q.out = B.d_out.as<DevOut>() + i;
        msv::TailJob& l = lj[i];
        l.samples = arr;
        l.src = B.d_out.as<DevOut>() + i;
        l.out = B.d_tails.as<double>() + 4 * i;
        tail_scratch(q.next, cap[i], l);
    }
    cudaStream_t st = ctx->stream;
    if (!parts_h.empty())
        MSV_CUDA_TRY(cudaMemcpyAsync(B.d_parts.p, parts_h.data(), parts_h.size() * sizeof(DevPart), cudaMemcpyHostToDevice, st));
    if (!masks_h.empty())
        MSV_CUDA_TRY(cudaMemcpyAsync(B.d_masks.p, masks_h.data(), masks_h.size() * 8, cudaMemcpyHostToDevice, st));
    if (n) {
        MSV_CUDA_TRY(cudaMemcpyAsync(B.d_tjobs.p, tj.data(), n * sizeof(msv::TraceJob), cudaMemcpyHostToDevice, st));
        MSV_CUDA_TRY(cudaMemcpyAsync(ctx->d_njobs.p, nj.data(), n * sizeof(msv::NoiseParams), cudaMemcpyHostToDevice, st));
        MSV_CUDA_TRY(cudaMemcpyAsync(B.d_tailjobs.p, lj.data(), n * sizeof(msv::TailJob), cudaMemcpyHostToDevice, st));
        MSV_CUDA_TRY(cudaMemsetAsync(B.d_tovf.p, 0, n * 4, st));
    }
    if (n_tails) MSV_CUDA_TRY(cudaMemcpyAsync(B.d_p.p, tail_p, n_tails * sizeof(double), cudaMemcpyHostToDevice, st));
    ctx->h2d += total * 8 + (int64_t)(n * (sizeof(msv::TraceJob) + sizeof(msv::NoiseParams) + sizeof(msv::TailJob)) +
                                      parts_h.size() * sizeof(DevPart) + masks_h.size() * 8);
    if (n) {
        // K1 first (the traces need no multipliers); then, chunk by chunk, the multiplier
        // streams are drawn on the host (the reference's Rng and libm, rng.hpp:27-32, one
        // thread per core) into pinned staging, copied, and the chunk's K5 launched on an aux
        // stream — so the host draws chunk c + 1 while the device copies and simulates chunk c.
        if (!ctx->k1_ev) MSV_CUDA_TRY(cudaEventCreateWithFlags(&ctx->k1_ev, cudaEventDisableTiming));
        MSV_CUDA_TRY(msv::launch_trace_gen(B.d_tjobs.as<msv::TraceJob>(), (int)n, ctx->log1p, st));
        MSV_CUDA_TRY(cudaEventRecord(ctx->k1_ev, st));
        ctx->launches += 1;
        constexpr int64_t kChunkQ = (int64_t)8 << 20;  // multipliers per chunk (64 MB)
        int64_t max_cap = 0;
        for (int64_t i = 0; i < n; ++i) max_cap = std::max(max_cap, cap[i]);
        const size_t need = (size_t)std::max<int64_t>(std::min<int64_t>(kChunkQ, total), max_cap);
        if (ctx->pin_n < need) {
            for (int b = 0; b < 2; ++b) {
                if (ctx->pin_ev[b]) MSV_CUDA_TRY(cudaEventSynchronize(ctx->pin_ev[b]));
                if (ctx->pin[b]) cudaFreeHost(ctx->pin[b]);
                ctx->pin[b] = nullptr;
                MSV_CUDA_TRY(cudaHostAlloc(reinterpret_cast<void**>(&ctx->pin[b]), need * 8, cudaHostAllocDefault));
            }
            ctx->pin_n = need;
        }
        for (int b = 0; b < 2; ++b)
            if (!ctx->pin_ev[b]) MSV_CUDA_TRY(cudaEventCreateWithFlags(&ctx->pin_ev[b], cudaEventDisableTiming));
        for (int a = 0; a < kAuxStreams; ++a) {
            if (!ctx->aux[a]) MSV_CUDA_TRY(cudaStreamCreateWithFlags(&ctx->aux[a], cudaStreamNonBlocking));
            if (!ctx->aux_ev[a]) MSV_CUDA_TRY(cudaEventCreateWithFlags(&ctx->aux_ev[a], cudaEventDisableTiming));
            MSV_CUDA_TRY(cudaStreamWaitEvent(ctx->aux[a], ctx->k1_ev, 0));
        }
        const int nt = std::max(1, std::min(host_threads(), 64));
        int chunk = 0;
        for (int64_t s0 = 0; s0 < n; ++chunk) {
            int64_t s1 = s0 + 1;
            while (s1 < n && toff[s1 + 1] - toff[s0] <= (int64_t)ctx->pin_n) ++s1;
            const int b = chunk & 1;
            if (chunk >= 2) MSV_CUDA_TRY(cudaEventSynchronize(ctx->pin_ev[b]));  // its last copy is done
            double* const stage = ctx->pin[b] - toff[s0];
            std::atomic<int64_t> next_i{s0};
            std::vector<std::thread> th;
            const int nth = (int)std::min<int64_t>(nt, s1 - s0);
            for (int t = 0; t < nth; ++t)
                th.emplace_back([&] {
                    for (int64_t i; (i = next_i.fetch_add(1)) < s1;)
                        msv_noise_multipliers(nseed[i], sigma[i], cap[i], stage + toff[i]);
                });
            for (std::thread& t : th) t.join();
            cudaStream_t sa = ctx->aux[chunk % kAuxStreams];
            MSV_CUDA_TRY(cudaMemcpyAsync(ctx->d_mult.as<double>() + toff[s0], ctx->pin[b],
                                         (size_t)(toff[s1] - toff[s0]) * 8, cudaMemcpyHostToDevice, sa));
            MSV_CUDA_TRY(cudaEventRecord(ctx->pin_ev[b], sa));
            int max_p = 0;
            for (int64_t i = s0; i < s1; ++i) max_p = std::max(max_p, (int)P[i]);
            MSV_CUDA_TRY(msv::launch_noise(ctx->d_njobs.as<msv::NoiseParams>() + s0, (int)(s1 - s0), max_cells, max_p, sa));
            ctx->launches += 1;
            s0 = s1;
        }
        for (int a = 0; a < kAuxStreams; ++a) {  // join
            MSV_CUDA_TRY(cudaEventRecord(ctx->aux_ev[a], ctx->aux[a]));
            MSV_CUDA_TRY(cudaStreamWaitEvent(st, ctx->aux_ev[a], 0));
        }
        if (n_tails) {
            MSV_CUDA_TRY(msv::launch_tail(B.d_tailjobs.as<msv::TailJob>(), (int)n, B.d_p.as<double>(), n_tails, st));
            ctx->launches += 1;
        }
    }
    pt.mark("jobs+enqueue");
    std::vector<DevOut> outs(n);
    std::vector<double> tails(4 * n);
    std::vector<int64_t> nq(n);
    std::vector<int32_t> ovf(n);
    if (n) {
        MSV_CUDA_TRY(cudaMemcpyAsync(outs.data(), B.d_out.p, n * sizeof(DevOut), cudaMemcpyDeviceToHost, st));
        MSV_CUDA_TRY(cudaMemcpyAsync(tails.data(), B.d_tails.p, n * 4 * sizeof(double), cudaMemcpyDeviceToHost, st));
        MSV_CUDA_TRY(cudaMemcpyAsync(nq.data(), B.d_nq.p, n * 8, cudaMemcpyDeviceToHost, st));
        MSV_CUDA_TRY(cudaMemcpyAsync(ovf.data(), B.d_tovf.p, n * 4, cudaMemcpyDeviceToHost, st));
        if (usage)
            MSV_CUDA_TRY(cudaMemcpyAsync(usage, B.d_usage.p, uoff[n] * sizeof(msv_usage), cudaMemcpyDeviceToHost, st));
    }
    MSV_CUDA_TRY(cudaStreamSynchronize(st));
    pt.mark("device");
    ctx->d2h += n * (int64_t)(sizeof(DevOut) + 4 * sizeof(double) + 12) + (usage ? uoff[n] * (int64_t)sizeof(msv_usage) : 0);
    std::vector<int64_t> retry;
    for (int64_t i = 0; i < n; ++i) {
        if (ovf[i]) {
            retry.push_back(i);
            continue;
        }
        const DevOut& o = outs[i];
        msv_result& r = results[i];
        r = msv_result{};
        r.total = nq[i];
        r.violations = o.violations;
        r.measured = o.measured;
        r.measured_violations = o.measured_violations;
        for (int j = 0; j < 4; ++j) r.tail[j] = j < n_tails ? tails[4 * i + j] : std::numeric_limits<double>::quiet_NaN();
        r.horizon_ms = o.horizon_ms;
        r.warmup_ms = sc[i].warmup_fraction * sc[i].duration_ms;
        r.max_wait_estimate_diff = 0.0;  // the reference skips the check under noise (engine.hpp:208)
        r.duration_ms = sc[i].duration_ms;
        r.placement_hash = o.hash;
        r.status = o.status;
        r.n_partitions = P[i];
    }
    // traces longer than their Poisson-tail capacity: rerun those with 4x the capacity
    if (!retry.empty()) {
        std::vector<msv_scenario> sub;
        std::vector<double> ssig;
        std::vector<uint64_t> sseed;
        std::vector<int64_t> scap;
        int64_t nu = 0;
        for (int64_t i : retry) {
            sub.push_back(sc[i]);
            ssig.push_back(sigma[i]);
            sseed.push_back(nseed[i]);
            scap.push_back(cap[i] * 4);
            nu += P[i];
        }
        std::vector<msv_result> sres(sub.size());
        std::vector<msv_usage> suse(std::max<int64_t>(nu, 1));
        rc = run_grid_noise_dev(ctx, sub.data(), (int64_t)sub.size(), ssig.data(), sseed.data(), tail_p, n_tails,
                                sres.data(), usage ? suse.data() : nullptr, scap.data());
        if (rc) return rc;
        int64_t u = 0;
        for (size_t k = 0; k < retry.size(); ++k) {
            results[retry[k]] = sres[k];
            if (usage)
                for (int32_t q = 0; q < P[retry[k]]; ++q) usage[uoff[retry[k]] + q] = suse[u++];
        }
    }
    return MSV_OK;
}

}  // namespace

extern "C" {

int msv_run_grid_noise(msv_ctx* ctx, const msv_scenario* scenarios, int64_t n, const double* noise_sigma,
                       const uint64_t* noise_seed, const double* tail_p, int n_tails, msv_result* results,
                       msv_usage* usage) {
    if (!ctx || (n > 0 && (!scenarios || !results || !noise_sigma || !noise_seed)))
        return fail(MSV_PARAM, "null argument");
    if (ctx->peers.empty())
        return run_grid_noise_dev(ctx, scenarios, n, noise_sigma, noise_seed, tail_p, n_tails, results, usage, nullptr);
    sync_peers(ctx);
    const std::vector<msv_ctx*> m = members(ctx);
    const std::vector<int64_t> cut = shard_cuts(ctx, scenarios, n, nullptr, (int)m.size());
    const std::vector<int64_t> uo = usage_prefix(ctx, scenarios, n);
    return fan_out(m, [&](size_t k) {
        const int64_t lo = cut[k], hi = cut[k + 1];
        if (hi <= lo) return (int)MSV_OK;
        return run_grid_noise_dev(m[k], scenarios + lo, hi - lo, noise_sigma + lo, noise_seed + lo, tail_p, n_tails,
                                  results + lo, usage ? usage + uo[lo] : nullptr, nullptr);
    });
}

}  // extern "C"

