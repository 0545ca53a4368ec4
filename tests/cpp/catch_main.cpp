// catch_main.cpp -- runner for the catchlite registry (tests/cpp/catch2/catch_amalgamated.hpp):
// every TEST_CASE in the linked translation units, one PASS/FAIL line each, exit code = failures.
#include <cstdio>
#include <exception>

#include "catch2/catch_amalgamated.hpp"

int main() {
    int failed_cases = 0;
    for (const auto& c : catchlite::registry()) {
        catchlite::state().current = c.name;
        const int before = catchlite::state().failures;
        try {
            c.fn();
        } catch (const catchlite::RequireFailed&) {
        } catch (const std::exception& e) {
            ++catchlite::state().failures;
            std::printf("  FAILED in \"%s\": unexpected exception: %s\n", c.name, e.what());
        }
        const bool ok = catchlite::state().failures == before;
        failed_cases += ok ? 0 : 1;
        std::printf("%s %s\n", ok ? "PASS" : "FAIL", c.name);
    }
    std::printf("%zu test cases, %d failed; %d checks, %d failed\n", catchlite::registry().size(), failed_cases,
                catchlite::state().checks, catchlite::state().failures);
    return failed_cases == 0 ? 0 : 1;
}
