// Minimal doctest-compatible test harness (the subset used by the reference's
// unit tests: TEST_CASE, SUBCASE, CHECK, REQUIRE, CHECK_THROWS_AS,
// CHECK_THROWS_WITH_AS, CHECK_NOTHROW, doctest::Approx, doctest::Contains).
// doctest itself is not in this image (the reference vendored it in an ignored
// directory); this shim lets the reference's own test sources compile
// unchanged against the B200 drop-in. Approx follows doctest's published rule
// |a - b| < eps * (scale + max(|a|, |b|)), default eps = 100 * FLT_EPSILON.
// SUBCASEs run one after another in a single pass of their test case.
#pragma once

#include <algorithm>
#include <cfloat>
#include <cmath>
#include <cstdio>
#include <exception>
#include <string>
#include <vector>

namespace doctest {

class Approx {
public:
    explicit Approx(double v) : value_(v) {}
    Approx& epsilon(double e) { eps_ = e; return *this; }
    Approx& scale(double s) { scale_ = s; return *this; }
    bool matches(double lhs) const {
        return std::fabs(lhs - value_) < eps_ * (scale_ + std::max(std::fabs(lhs), std::fabs(value_)));
    }
private:
    double value_;
    double eps_ = static_cast<double>(FLT_EPSILON) * 100.0;
    double scale_ = 1.0;
};
inline bool operator==(double lhs, const Approx& rhs) { return rhs.matches(lhs); }
inline bool operator==(const Approx& lhs, double rhs) { return lhs.matches(rhs); }
inline bool operator!=(double lhs, const Approx& rhs) { return !rhs.matches(lhs); }

struct Contains {
    explicit Contains(const char* s) : needle(s) {}
    bool check(const std::string& text) const { return text.find(needle) != std::string::npos; }
    std::string needle;
};

namespace detail {
struct TestCase {
    const char* name;
    void (*fn)();
    const char* file;
    int line;
};
inline std::vector<TestCase>& registry() {
    static std::vector<TestCase> r;
    return r;
}
struct Reg {
    Reg(const char* name, void (*fn)(), const char* file, int line) { registry().push_back({name, fn, file, line}); }
};
struct RequireFailure {};
inline int& failed_checks() { static int n = 0; return n; }
inline int& total_checks() { static int n = 0; return n; }
inline void fail(const char* file, int line, const char* what) {
    ++failed_checks();
    std::fprintf(stderr, "%s:%d: CHECK FAILED: %s\n", file, line, what);
}
struct Subcase {
    explicit Subcase(const char*) {}
    explicit operator bool() const { return true; }
};
} // namespace detail
} // namespace doctest

#define DT_CAT2(a, b) a##b
#define DT_CAT(a, b) DT_CAT2(a, b)
#define DT_TC_IMPL(f, name)                                                                   \
    static void f();                                                                          \
    static ::doctest::detail::Reg DT_CAT(f, _reg)(name, f, __FILE__, __LINE__);               \
    static void f()
#define TEST_CASE(name) DT_TC_IMPL(DT_CAT(dt_test_fn_, __LINE__), name)
#define SUBCASE(name) if (const ::doctest::detail::Subcase DT_CAT(dt_sub_, __LINE__){name})

#define DT_CHECK_IMPL(abort_on_fail, ...)                                                     \
    do {                                                                                      \
        ++::doctest::detail::total_checks();                                                  \
        bool dt_ok_ = false;                                                                  \
        try {                                                                                 \
            dt_ok_ = static_cast<bool>(__VA_ARGS__);                                          \
        } catch (const std::exception& dt_e_) {                                               \
            std::fprintf(stderr, "  exception: %s\n", dt_e_.what());                          \
        }                                                                                     \
        if (!dt_ok_) {                                                                        \
            ::doctest::detail::fail(__FILE__, __LINE__, #__VA_ARGS__);                        \
            if (abort_on_fail) throw ::doctest::detail::RequireFailure{};                     \
        }                                                                                     \
    } while (0)
#define CHECK(...) DT_CHECK_IMPL(false, __VA_ARGS__)
#define REQUIRE(...) DT_CHECK_IMPL(true, __VA_ARGS__)

#define CHECK_THROWS_AS(expr, ...)                                                            \
    do {                                                                                      \
        ++::doctest::detail::total_checks();                                                  \
        bool dt_caught_ = false;                                                              \
        try {                                                                                 \
            (void)(expr);                                                                     \
        } catch (const __VA_ARGS__&) {                                                        \
            dt_caught_ = true;                                                                \
        } catch (...) {                                                                       \
        }                                                                                     \
        if (!dt_caught_) ::doctest::detail::fail(__FILE__, __LINE__, "THROWS_AS " #expr);     \
    } while (0)

#define CHECK_THROWS_WITH_AS(expr, matcher, ...)                                              \
    do {                                                                                      \
        ++::doctest::detail::total_checks();                                                  \
        bool dt_caught_ = false;                                                              \
        try {                                                                                 \
            (void)(expr);                                                                     \
        } catch (const __VA_ARGS__& dt_e_) {                                                  \
            dt_caught_ = (matcher).check(dt_e_.what());                                       \
        } catch (...) {                                                                       \
        }                                                                                     \
        if (!dt_caught_) ::doctest::detail::fail(__FILE__, __LINE__, "THROWS_WITH_AS " #expr); \
    } while (0)

#define CHECK_NOTHROW(expr)                                                                   \
    do {                                                                                      \
        ++::doctest::detail::total_checks();                                                  \
        try {                                                                                 \
            (void)(expr);                                                                     \
        } catch (...) {                                                                       \
            ::doctest::detail::fail(__FILE__, __LINE__, "NOTHROW " #expr);                    \
        }                                                                                     \
    } while (0)
