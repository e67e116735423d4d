// Device plumbing for the migserve host headers: the per-thread engine context
// (one CUDA device, its memory and stream; see include/msv.h) and the mapping of
// msv_status codes back onto the reference's exception types.
//
// The device is chosen by the MSV_DEVICE environment variable (default 0). With
// MSV_DEVICES=0,1,...,7 (or set_devices() before the first call on a thread) the
// context spans several GPUs (msv_create_multi): the grid drivers — run_grid and
// everything built on it (latency_bounded_throughput, best_homogeneous, the sweeps) —
// cut each grid into cost-balanced shards, one per GPU, and gather the results in
// order. All hot-path entry points (run, sample_trace, tail_latency, the dispatch
// functions and the grid drivers) execute as sm_100a kernels through this context;
// there is no host fallback — without a usable B200 the first call throws.
#pragma once

#include <atomic>
#include <cstdlib>
#include <string>
#include <vector>

#include "../msv.h"
#include "errors.hpp"

namespace migserve {
namespace device {

[[noreturn]] inline void throw_status(int rc, const std::string& where = {}) {
    std::string msg = msv_last_error();
    if (!where.empty()) msg = where + ": " + msg;
    switch (rc) {
        case MSV_PARAM: throw ParamError(msg);
        case MSV_FORMAT: throw FormatError(msg);
        case MSV_VALIDATION: throw ValidationError(msg);
        case MSV_LOOKUP: throw LookupError(msg);
        case MSV_INFEASIBLE: throw InfeasibleError(msg);
        default: throw Error("device engine: " + msg);
    }
}

inline void check(int rc, const char* where = nullptr) {
    if (rc != MSV_OK) throw_status(rc, where ? where : "");
}

// Devices of contexts created from now on (empty: MSV_DEVICES / MSV_DEVICE / 0).
inline std::vector<int>& configured_devices() {
    static std::vector<int> d;
    return d;
}
inline void set_devices(const std::vector<int>& devices) { configured_devices() = devices; }

inline std::vector<int> devices_from_env() {
    std::vector<int> d = configured_devices();
    if (!d.empty()) return d;
    if (const char* env = std::getenv("MSV_DEVICES")) {
        std::string s(env);
        size_t pos = 0;
        while (pos < s.size()) {
            const size_t comma = s.find(',', pos);
            const std::string tok = s.substr(pos, comma == std::string::npos ? std::string::npos : comma - pos);
            if (!tok.empty()) d.push_back(std::atoi(tok.c_str()));
            if (comma == std::string::npos) break;
            pos = comma + 1;
        }
        if (!d.empty()) return d;
    }
    const char* env = std::getenv("MSV_DEVICE");
    return {env ? std::atoi(env) : 0};
}

// Thread-local engine context; created on first use.
class Context {
public:
    Context() {
        const std::vector<int> devs = devices_from_env();
        if (devs.size() == 1) check(msv_create(devs[0], &ctx_), "msv_create");
        else check(msv_create_multi(devs.data(), (int)devs.size(), &ctx_), "msv_create_multi");
        serial_ = next_serial();
    }
    ~Context() { msv_destroy(ctx_); }
    Context(const Context&) = delete;
    Context& operator=(const Context&) = delete;
    msv_ctx* get() const { return ctx_; }
    // Distinguishes contexts so cached upload handles are never reused across them.
    unsigned long serial() const { return serial_; }

private:
    static unsigned long next_serial() {
        static std::atomic<unsigned long> s{0};
        return ++s;
    }
    msv_ctx* ctx_ = nullptr;
    unsigned long serial_ = 0;
};

inline Context& context() {
    thread_local Context ctx;
    return ctx;
}

// Cached upload handle of an immutable host object in the current context.
struct HandleCache {
    unsigned long serial = 0;
    int handle = -1;
    template <typename Upload>
    int get(Upload&& upload) {
        Context& c = context();
        if (serial != c.serial()) {
            handle = upload(c.get());
            serial = c.serial();
        }
        return handle;
    }
};

}  // namespace device
}  // namespace migserve
