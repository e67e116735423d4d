// Device plumbing for the migserve host headers: the per-thread engine context
// (one CUDA device, its memory and stream; see include/msv.h) and the mapping of
// msv_status codes back onto the reference's exception types.
//
// The device is chosen by the MSV_DEVICE environment variable (default 0). All
// hot-path entry points (run, sample_trace, tail_latency, the dispatch
// functions and the grid drivers) execute as sm_100a kernels through this
// context; there is no host fallback — without a usable B200 the first call
// throws.
#pragma once

#include <atomic>
#include <cstdlib>
#include <string>

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

// Thread-local engine context; created on first use.
class Context {
public:
    Context() {
        const char* env = std::getenv("MSV_DEVICE");
        const int dev = env ? std::atoi(env) : 0;
        check(msv_create(dev, &ctx_), "msv_create");
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
