// acceptance_b200.cpp -- the reference's acceptance pattern (proj/tests/acceptance.cpp: one
// PASS/FAIL line per criterion) run through the DROP-IN header include/tcreduce/reduction.hpp,
// i.e. exactly the code a reference user compiles after switching include paths.
// Criteria mirror acceptance.cpp:119-184 (crit 5-7) at the hardware fragment m = 16, plus the
// reference's validation / error contract (test_reduction.cpp:221-234) and determinism.
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <string>
#include <vector>

#include "tcreduce/reduction.hpp"

using namespace tcreduce;

namespace {

// Test-side input generator: harness.hpp:47-80 restated (SplitMix64, rng.hpp:9-26).
struct Rng {
    std::uint64_t s;
    std::uint64_t next() {
        std::uint64_t z = (s += 0x9E3779B97F4A7C15ull);
        z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
        z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
        return z ^ (z >> 31);
    }
    double unit() { return static_cast<double>(next() >> 11) * 0x1.0p-53; }
    double unit_open() { return static_cast<double>((next() >> 11) + 1) * 0x1.0p-53; }
};

std::vector<float> gen(const char* kind, std::uint64_t seed, std::size_t n) {
    Rng r{seed};
    std::vector<float> v;
    v.reserve(n);
    const std::string k = kind;
    if (k == "uniform") {
        for (std::size_t i = 0; i < n; ++i) v.push_back(static_cast<float>(r.unit()));
    } else if (k == "integers") {
        for (std::size_t i = 0; i < n; ++i) v.push_back(static_cast<float>(static_cast<long long>(r.next() % 10)));
    } else {
        for (std::size_t i = 0; i < n; i += 2) {
            const double u1 = r.unit_open(), u2 = r.unit();
            const double rr = std::sqrt(-2.0 * std::log(u1)), t = 2.0 * 3.141592653589793 * u2;
            v.push_back(static_cast<float>(rr * std::cos(t)));
            if (i + 1 < n) v.push_back(static_cast<float>(rr * std::sin(t)));
        }
    }
    return v;
}

double sum64(const std::vector<float>& x) {
    double a = 0.0;
    for (float f : x) a += f;
    return a;
}

int failures = 0;
void report(const char* name, bool ok, const std::string& detail) {
    std::printf("criterion %s: %s%s%s\n", name, ok ? "PASS" : "FAIL", ok ? "" : " - ", ok ? "" : detail.c_str());
    if (!ok) ++failures;
}

ReductionConfig best() {  // curve_config(single_pass) at the hardware fragment (harness.hpp:178-196)
    ReductionConfig c;
    c.m = 16;
    c.B = 128;
    c.R = 4;
    return c;
}

}  // namespace

int main() {
    {  // crit 5: integer inputs reduce exactly (acceptance.cpp:119-143)
        bool ok = true;
        std::string d;
        for (std::uint64_t seed = 0; seed < 10 && ok; ++seed) {
            const auto x = gen("integers", seed, 1 << 20);
            const ReductionOutcome o = single_pass_reduce(x, best());
            if (o.value != sum64(x) || o.overflow) {
                ok = false;
                d = "seed " + std::to_string(seed) + " got " + std::to_string(o.value);
            }
        }
        report(" 5 (oracle equivalence, single_pass)", ok, d);
    }
    {  // crit 6: normal error < 1% at n = 1e7 (acceptance.cpp:145-165)
        bool ok = true;
        std::string d;
        for (std::uint64_t seed : {1ull, 2ull, 3ull}) {
            const auto x = gen("normal", seed, 10000000);
            const double ref = sum64(x);
            const ReductionOutcome o = reduce(x, best());
            const double err = 100.0 * std::fabs(o.value - ref) / std::fabs(ref);
            if (o.overflow || !(err < 1.0)) {
                ok = false;
                d = "seed " + std::to_string(seed) + " err% " + std::to_string(err);
            }
        }
        report(" 6 (normal-distribution error)", ok, d);
    }
    {  // crit 7: uniform error < 0.001%, no overflow (acceptance.cpp:167-184)
        const auto x = gen("uniform", 0, 10000000);
        const double ref = sum64(x);
        const ReductionOutcome o = single_pass_reduce(x, best());
        const double err = 100.0 * std::fabs(o.value - ref) / std::fabs(ref);
        report(" 7 (uniform-distribution behavior)", !o.overflow && err < 0.001, "err% " + std::to_string(err));
    }
    {  // validation / exception contract (test_reduction.cpp:221-234, reduction.hpp:282)
        bool ok = true;
        ReductionConfig c = best();
        c.B = 48;
        try { c.validate(); ok = false; } catch (const std::invalid_argument&) {}
        c = best();
        c.R = 0;
        try { c.validate(); ok = false; } catch (const std::invalid_argument&) {}
        c = best();
        c.m = 3;
        try { c.validate(); ok = false; } catch (const std::invalid_argument&) {}
        try { (void)reduce(std::vector<float>{}, best()); ok = false; } catch (const std::invalid_argument&) {}
        report("10 (configuration validation)", ok, "an invalid config or empty input did not throw invalid_argument");
    }
    {  // determinism (crit 9 spirit): identical inputs -> bit-identical outputs
        const auto x = gen("normal", 12345, 3000017);
        const double a = reduce(x, best()).value, b = reduce(x, best()).value;
        report(" 9 (determinism)", a == b, std::to_string(a) + " vs " + std::to_string(b));
    }
    {  // counters follow the reference formulas (test_reduction.cpp:121-124 at m=4 -> here m=16)
        const std::vector<float> ones(2048, 1.0f);
        ReductionConfig c;
        c.m = 16;
        c.R = 1;
        c.B = 256;
        const ReductionOutcome o = reduce(ones, c);
        report(" 4 (two-step identity on ones, counters)", o.value == 2048.0 && o.atomic_count == 1 && o.mma_count == 16,
               "value " + std::to_string(o.value));
    }
    if (failures) std::printf("%d criterion(s) failed\n", failures);
    return failures;
}
