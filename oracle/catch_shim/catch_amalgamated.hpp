// catch_amalgamated.hpp -- TEST INFRASTRUCTURE ONLY.
//
// A minimal stand-in for the Catch2 v3 single header (absent from this image),
// providing just the surface the reference's unit tests use
// (/root/reference/proj/tests/test_*.cpp): TEST_CASE, REQUIRE, REQUIRE_FALSE,
// REQUIRE_NOTHROW, REQUIRE_THROWS_AS, REQUIRE_THROWS_WITH, REQUIRE_THAT and the
// matchers ContainsSubstring, WithinAbs, WithinRel.  oracle/Makefile compiles
// the reference's own test sources where they lie against it twice: with the
// reference headers (checks the shim) and with this repo's shadow headers
// first on the include path (the reference's own unit tests run against the
// B200 drop-in).  A failing REQUIRE aborts its test case, as in Catch2.
#pragma once

#include <cmath>
#include <exception>
#include <functional>
#include <limits>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

namespace shim {

struct Case {
    const char* name;
    const char* file;
    int line;
    void (*fn)();
};

inline std::vector<Case>& registry() {
    static std::vector<Case> r;
    return r;
}

struct Registrar {
    Registrar(const char* name, const char* file, int line, void (*fn)()) {
        registry().push_back({name, file, line, fn});
    }
};

struct Failure : std::exception {
    std::string what_;
    Failure(const char* file, int line, const std::string& msg) {
        std::ostringstream os;
        os << file << ":" << line << ": " << msg;
        what_ = os.str();
    }
    const char* what() const noexcept override { return what_.c_str(); }
};

inline long& assertions() {
    static long n = 0;
    return n;
}

[[noreturn]] inline void fail(const char* file, int line, const std::string& msg) {
    throw Failure(file, line, msg);
}

inline std::string describe_current() {
    try {
        throw;
    } catch (const std::exception& e) {
        return e.what();
    } catch (...) {
        return "<non-std exception>";
    }
}

}  // namespace shim

namespace Catch::Matchers {

struct ContainsSubstring {
    std::string needle;
    explicit ContainsSubstring(std::string s) : needle(std::move(s)) {}
    bool match(const std::string& s) const { return s.find(needle) != std::string::npos; }
    std::string describe() const { return "contains \"" + needle + "\""; }
};

struct WithinAbs {
    double target, margin;
    WithinAbs(double t, double m) : target(t), margin(m) {}
    bool match(double v) const { return v + margin >= target && target + margin >= v; }
    std::string describe() const { return "within " + std::to_string(margin) + " of " + std::to_string(target); }
};

struct WithinRel {
    double target, eps;
    explicit WithinRel(double t, double e = std::numeric_limits<double>::epsilon() * 100) : target(t), eps(e) {}
    bool match(double v) const {
        const double margin = eps * std::max(std::fabs(v), std::fabs(target));
        if (std::isinf(margin)) return v == target;
        return v + margin >= target && target + margin >= v;
    }
    std::string describe() const { return "within rel " + std::to_string(eps) + " of " + std::to_string(target); }
};

}  // namespace Catch::Matchers

namespace shim {

inline bool message_matches(const std::string& got, const char* expected) { return got == expected; }
inline bool message_matches(const std::string& got, const std::string& expected) { return got == expected; }
inline bool message_matches(const std::string& got, const Catch::Matchers::ContainsSubstring& m) {
    return m.match(got);
}

}  // namespace shim

#define SHIM_CAT2(a, b) a##b
#define SHIM_CAT(a, b) SHIM_CAT2(a, b)
#define SHIM_TEST_CASE_IMPL(fn, ...)                                                        \
    static void fn();                                                                       \
    static ::shim::Registrar SHIM_CAT(fn, _reg)(SHIM_FIRST(__VA_ARGS__, ""), __FILE__, __LINE__, fn); \
    static void fn()
#define SHIM_FIRST(a, ...) a
#define TEST_CASE(...) SHIM_TEST_CASE_IMPL(SHIM_CAT(shim_case_, __LINE__), __VA_ARGS__)

#define REQUIRE(...)                                                                       \
    do {                                                                                   \
        ++::shim::assertions();                                                            \
        if (!static_cast<bool>(__VA_ARGS__)) ::shim::fail(__FILE__, __LINE__, "REQUIRE(" #__VA_ARGS__ ")"); \
    } while (0)
#define REQUIRE_FALSE(...)                                                                 \
    do {                                                                                   \
        ++::shim::assertions();                                                            \
        if (static_cast<bool>(__VA_ARGS__)) ::shim::fail(__FILE__, __LINE__, "REQUIRE_FALSE(" #__VA_ARGS__ ")"); \
    } while (0)
#define REQUIRE_NOTHROW(...)                                                               \
    do {                                                                                   \
        ++::shim::assertions();                                                            \
        try {                                                                              \
            (void)(__VA_ARGS__);                                                           \
        } catch (...) {                                                                    \
            ::shim::fail(__FILE__, __LINE__, "unexpected exception: " + ::shim::describe_current()); \
        }                                                                                  \
    } while (0)
#define REQUIRE_THROWS_AS(expr, type)                                                      \
    do {                                                                                   \
        ++::shim::assertions();                                                            \
        bool shim_thrown = false;                                                          \
        try {                                                                              \
            (void)(expr);                                                                  \
        } catch (const type&) {                                                            \
            shim_thrown = true;                                                            \
        } catch (...) {                                                                    \
            ::shim::fail(__FILE__, __LINE__, "wrong exception type: " + ::shim::describe_current()); \
        }                                                                                  \
        if (!shim_thrown) ::shim::fail(__FILE__, __LINE__, "no exception from " #expr);     \
    } while (0)
#define REQUIRE_THROWS_WITH(expr, matcher)                                                 \
    do {                                                                                   \
        ++::shim::assertions();                                                            \
        bool shim_thrown = false;                                                          \
        try {                                                                              \
            (void)(expr);                                                                  \
        } catch (...) {                                                                    \
            shim_thrown = true;                                                            \
            const std::string shim_msg = ::shim::describe_current();                       \
            if (!::shim::message_matches(shim_msg, matcher))                               \
                ::shim::fail(__FILE__, __LINE__, "message \"" + shim_msg + "\" does not match"); \
        }                                                                                  \
        if (!shim_thrown) ::shim::fail(__FILE__, __LINE__, "no exception from " #expr);     \
    } while (0)
#define REQUIRE_THAT(arg, matcher)                                                         \
    do {                                                                                   \
        ++::shim::assertions();                                                            \
        const auto& shim_m = (matcher);                                                    \
        const auto shim_v = (arg);                                                         \
        if (!shim_m.match(shim_v)) {                                                       \
            std::ostringstream shim_os;                                                    \
            shim_os.precision(17);                                                         \
            shim_os << #arg << " = " << shim_v << " not " << shim_m.describe();             \
            ::shim::fail(__FILE__, __LINE__, shim_os.str());                               \
        }                                                                                  \
    } while (0)
