// catch_amalgamated.hpp -- a minimal stand-in for the Catch2 v3 single header (absent from this
// image), covering exactly the macros the reference's unit tests use (TEST_CASE, CHECK,
// CHECK_FALSE, CHECK_THAT + Catch::Matchers::WithinAbs, CHECK_THROWS_AS, REQUIRE).  It lets
// proj/tests/test_reduction.cpp and test_harness.cpp compile unchanged against the B200 drop-in
// header (oracle/Makefile, target ref_tests).  Test infrastructure only.
#pragma once

#include <cmath>
#include <cstdio>
#include <exception>
#include <functional>
#include <string>
#include <vector>

namespace catchlite {

struct Case {
    const char* name;
    std::function<void()> fn;
};

inline std::vector<Case>& registry() {
    static std::vector<Case> r;
    return r;
}

struct Registrar {
    Registrar(const char* name, std::function<void()> fn) { registry().push_back({name, std::move(fn)}); }
};

struct State {
    int checks = 0, failures = 0;
    const char* current = "";
};

inline State& state() {
    static State s;
    return s;
}

struct RequireFailed {};

inline void report(bool ok, const char* expr, const char* file, int line, bool fatal) {
    ++state().checks;
    if (ok) return;
    ++state().failures;
    std::printf("  FAILED %s:%d in \"%s\": %s\n", file, line, state().current, expr);
    if (fatal) throw RequireFailed{};
}

struct WithinAbsMatcher {
    double target, margin;
    bool match(double v) const { return std::fabs(v - target) <= margin; }
};

}  // namespace catchlite

namespace Catch::Matchers {
inline catchlite::WithinAbsMatcher WithinAbs(double target, double margin) { return {target, margin}; }
}  // namespace Catch::Matchers

#define CATCHLITE_CAT2(a, b) a##b
#define CATCHLITE_CAT(a, b) CATCHLITE_CAT2(a, b)
#define CATCHLITE_TEST(fn, name)                                                        \
    static void fn();                                                                   \
    static const catchlite::Registrar CATCHLITE_CAT(fn, _reg){name, fn};                \
    static void fn()
#define TEST_CASE(name, ...) CATCHLITE_TEST(CATCHLITE_CAT(catchlite_case_, __LINE__), name)

#define CHECK(...) catchlite::report(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, false)
#define CHECK_FALSE(...) catchlite::report(!static_cast<bool>(__VA_ARGS__), "!(" #__VA_ARGS__ ")", __FILE__, __LINE__, false)
#define REQUIRE(...) catchlite::report(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, true)
#define REQUIRE_FALSE(...) catchlite::report(!static_cast<bool>(__VA_ARGS__), "!(" #__VA_ARGS__ ")", __FILE__, __LINE__, true)
#define CHECK_THAT(value, matcher) \
    catchlite::report((matcher).match(value), #value " matches " #matcher, __FILE__, __LINE__, false)
#define CATCHLITE_THROWS_AS(expr, type, fatal)                                          \
    do {                                                                                \
        bool caught_ = false;                                                           \
        try {                                                                           \
            static_cast<void>(expr);                                                    \
        } catch (const type&) {                                                         \
            caught_ = true;                                                             \
        } catch (...) {                                                                 \
        }                                                                               \
        catchlite::report(caught_, #expr " throws " #type, __FILE__, __LINE__, fatal);  \
    } while (0)
#define CHECK_THROWS_AS(expr, type) CATCHLITE_THROWS_AS(expr, type, false)
#define REQUIRE_THROWS_AS(expr, type) CATCHLITE_THROWS_AS(expr, type, true)
