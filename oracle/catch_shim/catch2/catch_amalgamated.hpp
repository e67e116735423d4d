// Minimal Catch2-v3-compatible shim. TEST INFRASTRUCTURE ONLY (oracle/).
//
// Catch2 is not installed in this image, so the reference's unit tests
// (/root/reference/proj/tests/*.cpp, CMake lookup at proj/tests/CMakeLists.txt:1-5)
// cannot build with the stock recipe. This header supplies exactly the subset
// those files use: TEST_CASE, flat SECTIONs (Catch2 semantics: one leaf section
// per run of the case, code outside sections runs every time), REQUIRE,
// REQUIRE_FALSE, REQUIRE_THROWS_AS and Catch::Approx with epsilon/margin using
// Catch2 v3's comparison rule. The same shim compiles the reference's tests
// against the reference headers (oracle/_ref) and against this repo's
// include/migserve headers (the drop-in check).
#pragma once

#include <cfloat>
#include <cmath>
#include <cstdio>
#include <functional>
#include <limits>
#include <stdexcept>
#include <string>
#include <vector>

namespace catch_shim {

struct Failure {
    std::string where;
};

struct Case {
    const char* name;
    void (*fn)();
};

inline std::vector<Case>& registry() {
    static std::vector<Case> r;
    return r;
}

struct Registrar {
    Registrar(const char* name, void (*fn)()) { registry().push_back({name, fn}); }
};

struct State {
    int target = 0;        // which leaf section runs this pass
    int seen = 0;          // sections encountered this pass
    long long assertions = 0;
};

inline State& state() {
    static State s;
    return s;
}

inline bool enter_section() {
    State& s = state();
    return s.seen++ == s.target;
}

inline void check(bool ok, const char* expr, const char* file, int line) {
    ++state().assertions;
    if (!ok) throw Failure{std::string(file) + ":" + std::to_string(line) + ": " + expr};
}

}  // namespace catch_shim

namespace Catch {

class Approx {
public:
    explicit Approx(double v)
        : value_(v), epsilon_(static_cast<double>(FLT_EPSILON) * 100.0), margin_(0.0), scale_(0.0) {}
    Approx& epsilon(double e) {
        epsilon_ = e;
        return *this;
    }
    Approx& margin(double m) {
        margin_ = m;
        return *this;
    }
    Approx& scale(double s) {
        scale_ = s;
        return *this;
    }
    // Catch2 v3 Approx::equalityComparisonImpl.
    bool matches(double other) const {
        return margin_cmp(value_, other, margin_) ||
               margin_cmp(value_, other,
                          epsilon_ * (scale_ + std::fabs(std::isinf(value_) ? 0.0 : value_)));
    }

private:
    static bool margin_cmp(double lhs, double rhs, double margin) {
        return (lhs + margin >= rhs) && (rhs + margin >= lhs);
    }
    double value_, epsilon_, margin_, scale_;
};

template <typename T>
inline bool operator==(const T& lhs, const Approx& rhs) {
    return rhs.matches(static_cast<double>(lhs));
}
template <typename T>
inline bool operator==(const Approx& lhs, const T& rhs) {
    return lhs.matches(static_cast<double>(rhs));
}
template <typename T>
inline bool operator!=(const T& lhs, const Approx& rhs) {
    return !rhs.matches(static_cast<double>(lhs));
}

}  // namespace Catch

#define CATCH_SHIM_CAT2(a, b) a##b
#define CATCH_SHIM_CAT(a, b) CATCH_SHIM_CAT2(a, b)
#define CATCH_SHIM_TEST(fn, name)                                      \
    static void fn();                                                  \
    static catch_shim::Registrar CATCH_SHIM_CAT(fn, _reg)(name, &fn);  \
    static void fn()
#define TEST_CASE(name, ...) CATCH_SHIM_TEST(CATCH_SHIM_CAT(catch_shim_case_, __COUNTER__), name)
#define SECTION(...) if (catch_shim::enter_section())
#define REQUIRE(...) catch_shim::check(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__)
#define REQUIRE_FALSE(...) \
    catch_shim::check(!static_cast<bool>(__VA_ARGS__), "!(" #__VA_ARGS__ ")", __FILE__, __LINE__)
#define REQUIRE_THROWS_AS(expr, type)                                         \
    do {                                                                      \
        bool catch_shim_ok = false;                                           \
        try {                                                                 \
            (void)(expr);                                                     \
        } catch (const type&) {                                               \
            catch_shim_ok = true;                                             \
        } catch (...) {                                                       \
        }                                                                     \
        catch_shim::check(catch_shim_ok, "throws " #type ": " #expr, __FILE__, __LINE__); \
    } while (0)

#ifdef CATCH_SHIM_MAIN
#include <chrono>
#include <cstring>
int main(int argc, char** argv) {
    using namespace catch_shim;
    const char* filter = argc > 1 ? argv[1] : nullptr;
    int failed = 0, ran = 0;
    auto t0 = std::chrono::steady_clock::now();
    for (const Case& c : registry()) {
        if (filter && !std::strstr(c.name, filter)) continue;
        ++ran;
        State& s = state();
        for (s.target = 0;; ++s.target) {
            s.seen = 0;
            bool ok = true;
            try {
                c.fn();
            } catch (const Failure& f) {
                std::printf("FAILED: %s\n  %s\n", c.name, f.where.c_str());
                ok = false;
            } catch (const std::exception& e) {
                std::printf("FAILED: %s\n  unexpected exception: %s\n", c.name, e.what());
                ok = false;
            }
            if (!ok) {
                ++failed;
                break;
            }
            if (s.target + 1 >= s.seen) break;  // every leaf section visited
        }
    }
    double secs = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    std::printf("%s: %d test cases, %d failed, %lld assertions, %.2f s\n",
                failed ? "FAILED" : "All tests passed", ran, failed, state().assertions, secs);
    return failed ? 1 : 0;
}
#endif
