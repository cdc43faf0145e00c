// TEST INFRASTRUCTURE ONLY: a minimal stand-in for the Catch2 v3 amalgamated
// header (absent from this image), enough to compile the
// reference's own test files unmodified (tests/cpp/Makefile). Supported:
// TEST_CASE, SECTION (each leaf section runs in its own pass of the test case,
// as in Catch2), CHECK / REQUIRE (+ _FALSE), CHECK / REQUIRE _THROWS(_AS),
// REQUIRE_NOTHROW, Catch::Approx (Catch2's default epsilon). A failing REQUIRE
// ends the current pass of the test case; the process exit code counts failures.
#pragma once

#include <cmath>
#include <cstdio>
#include <limits>
#include <string>
#include <vector>

namespace catch_shim {

struct TestCase {
    const char* name;
    void (*fn)();
};
inline std::vector<TestCase>& registry() {
    static std::vector<TestCase> r;
    return r;
}
struct Registrar {
    Registrar(const char* name, void (*fn)()) { registry().push_back({name, fn}); }
};
struct RequireFailed {};
struct State {
    int failures = 0;
    int assertions = 0;
    int target = 0;  // the section entered in this pass
    int seen = 0;    // sections met so far in this pass
    const char* test = "";
};
inline State& state() {
    static State s;
    return s;
}
inline void report(bool ok, const char* expr, const char* file, int line, bool require) {
    State& s = state();
    ++s.assertions;
    if (ok) return;
    ++s.failures;
    std::printf("FAILED %s:%d [%s]: %s\n", file, line, s.test, expr);
    if (require) throw RequireFailed{};
}
struct Section {
    bool on;
    explicit Section(const char*) : on(state().seen++ == state().target) {}
    explicit operator bool() const { return on; }
};

}  // namespace catch_shim

namespace Catch {
class Approx {
  public:
    explicit Approx(double v) : v_(v) {}
    Approx& epsilon(double e) {
        eps_ = e;
        return *this;
    }
    Approx& margin(double m) {
        margin_ = m;
        return *this;
    }
    friend bool operator==(double a, const Approx& b) { return b.equal(a); }
    friend bool operator==(const Approx& b, double a) { return b.equal(a); }
    friend bool operator!=(double a, const Approx& b) { return !b.equal(a); }

  private:
    bool equal(double a) const {
        const double d = std::abs(a - v_);
        return d <= margin_ || d <= eps_ * std::max(std::abs(a), std::abs(v_));
    }
    double v_;
    double eps_ = static_cast<double>(std::numeric_limits<float>::epsilon()) * 100.0;
    double margin_ = 0.0;
};
}  // namespace Catch

#define CATCH_SHIM_CAT2(a, b) a##b
#define CATCH_SHIM_CAT(a, b) CATCH_SHIM_CAT2(a, b)
#define TEST_CASE(name, ...)                                                              \
    static void CATCH_SHIM_CAT(catch_shim_tc_, __LINE__)();                               \
    static catch_shim::Registrar CATCH_SHIM_CAT(catch_shim_reg_, __LINE__)(               \
        name, &CATCH_SHIM_CAT(catch_shim_tc_, __LINE__));                                 \
    static void CATCH_SHIM_CAT(catch_shim_tc_, __LINE__)()
#define SECTION(name, ...) if (catch_shim::Section CATCH_SHIM_CAT(catch_shim_sec_, __LINE__){name})
#define CHECK(...) catch_shim::report(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, false)
#define REQUIRE(...) catch_shim::report(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, true)
#define CHECK_FALSE(...) catch_shim::report(!static_cast<bool>(__VA_ARGS__), "!(" #__VA_ARGS__ ")", __FILE__, __LINE__, false)
#define REQUIRE_FALSE(...) catch_shim::report(!static_cast<bool>(__VA_ARGS__), "!(" #__VA_ARGS__ ")", __FILE__, __LINE__, true)
#define CATCH_SHIM_THROWS_AS(expr, type, req)                                            \
    do {                                                                                  \
        bool caught_ = false;                                                             \
        try {                                                                             \
            static_cast<void>(expr);                                                      \
        } catch (const type&) {                                                           \
            caught_ = true;                                                               \
        } catch (...) {                                                                   \
        }                                                                                 \
        catch_shim::report(caught_, #expr " throws " #type, __FILE__, __LINE__, req);     \
    } while (0)
#define CHECK_THROWS_AS(expr, type) CATCH_SHIM_THROWS_AS(expr, type, false)
#define REQUIRE_THROWS_AS(expr, type) CATCH_SHIM_THROWS_AS(expr, type, true)
#define CATCH_SHIM_THROWS(expr, req)                                                      \
    do {                                                                                  \
        bool caught_ = false;                                                             \
        try {                                                                             \
            static_cast<void>(expr);                                                      \
        } catch (...) {                                                                   \
            caught_ = true;                                                               \
        }                                                                                 \
        catch_shim::report(caught_, #expr " throws", __FILE__, __LINE__, req);            \
    } while (0)
#define CHECK_THROWS(expr) CATCH_SHIM_THROWS(expr, false)
#define REQUIRE_THROWS(expr) CATCH_SHIM_THROWS(expr, true)
#define REQUIRE_NOTHROW(expr)                                                             \
    do {                                                                                  \
        bool ok_ = true;                                                                  \
        try {                                                                             \
            static_cast<void>(expr);                                                      \
        } catch (...) {                                                                   \
            ok_ = false;                                                                  \
        }                                                                                 \
        catch_shim::report(ok_, #expr " does not throw", __FILE__, __LINE__, true);       \
    } while (0)
