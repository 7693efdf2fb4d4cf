// Runner for the reference unit tests compiled against the B200 drop-in.
#include <cstdio>
#include <cstring>

#include "doctest.h"

int main(int argc, char** argv) {
    using namespace doctest::detail;
    int failed_cases = 0;
    int run = 0;
    for (const TestCase& tc : registry()) {
        if (argc > 1 && std::strstr(tc.name, argv[1]) == nullptr) continue;
        ++run;
        const int before = failed_checks();
        bool aborted = false;
        try {
            tc.fn();
        } catch (const RequireFailure&) {
            aborted = true;
        } catch (const std::exception& e) {
            std::fprintf(stderr, "%s:%d: uncaught exception in \"%s\": %s\n", tc.file, tc.line, tc.name, e.what());
            ++failed_checks();
        }
        const bool ok = failed_checks() == before && !aborted;
        if (!ok) ++failed_cases;
        std::printf("[%s] %s\n", ok ? "pass" : "FAIL", tc.name);
    }
    std::printf("[doctest-shim] test cases: %d | passed: %d | failed: %d | checks: %d | failed checks: %d\n", run,
                run - failed_cases, failed_cases, total_checks(), failed_checks());
    return failed_cases == 0 ? 0 : 1;
}
