// doctest_shim/doctest.h -- TEST INFRASTRUCTURE ONLY.
//
// A small doctest-compatible header written for this repo: the reference's unit tests
// (/root/reference/proj/tests/*.cpp) include <doctest.h> from a vendor/ directory that is
// absent upstream (proj/.gitignore:2). This shim implements exactly the subset those tests
// use (TEST_CASE, CHECK, REQUIRE, CHECK_THROWS[_AS], CHECK_NOTHROW, CAPTURE, FAIL,
// doctest::Approx(..).epsilon(..)) so the reference tests can be compiled unmodified --
// against the reference library (oracle/_ref/unit_tests_ref) and against the CUDA drop-in
// shim (oracle/_ref/unit_tests_gpu).
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <exception>
#include <limits>
#include <string>
#include <vector>

namespace doctest {

class Approx {
public:
    explicit Approx(double v) : value_(v) {}
    Approx& epsilon(double e) {
        eps_ = e;
        return *this;
    }
    Approx& scale(double s) {
        scale_ = s;
        return *this;
    }
    friend bool operator==(double lhs, const Approx& a) {
        return std::fabs(lhs - a.value_) <
               a.eps_ * (a.scale_ + std::max(std::fabs(lhs), std::fabs(a.value_)));
    }
    friend bool operator==(const Approx& a, double rhs) { return rhs == a; }
    friend bool operator!=(double lhs, const Approx& a) { return !(lhs == a); }
    friend bool operator!=(const Approx& a, double rhs) { return !(rhs == a); }

private:
    double value_;
    double eps_ = std::numeric_limits<float>::epsilon() * 100;
    double scale_ = 1.0;
};

namespace detail {
struct TestCase {
    const char* name;
    const char* file;
    int line;
    void (*fn)();
};
inline std::vector<TestCase>& registry() {
    static std::vector<TestCase> r;
    return r;
}
struct Registrar {
    Registrar(const char* name, const char* file, int line, void (*fn)()) {
        registry().push_back({name, file, line, fn});
    }
};
struct State {
    long checks = 0;
    long failed_checks = 0;
    bool case_failed = false;
};
inline State& state() {
    static State s;
    return s;
}
struct AbortCase {};
inline void report(const char* file, int line, const char* kind, const char* expr) {
    state().failed_checks++;
    state().case_failed = true;
    std::fprintf(stderr, "%s:%d: FAILED %s( %s )\n", file, line, kind, expr);
}
inline void check(bool ok, const char* file, int line, const char* kind, const char* expr,
                  bool require) {
    state().checks++;
    if (!ok) {
        report(file, line, kind, expr);
        if (require) throw AbortCase{};
    }
}
}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define DOCTEST_TC_(fn, name)                                                             \
    static void fn();                                                                     \
    static ::doctest::detail::Registrar DOCTEST_CAT(fn, _reg)(name, __FILE__, __LINE__, fn); \
    static void fn()
#define TEST_CASE(name) DOCTEST_TC_(DOCTEST_CAT(doctest_tc_, __COUNTER__), name)

#define CHECK(...) \
    ::doctest::detail::check(static_cast<bool>(__VA_ARGS__), __FILE__, __LINE__, "CHECK", #__VA_ARGS__, false)
#define REQUIRE(...) \
    ::doctest::detail::check(static_cast<bool>(__VA_ARGS__), __FILE__, __LINE__, "REQUIRE", #__VA_ARGS__, true)
#define CAPTURE(x) ((void)0)
#define FAIL(msg)                                                                 \
    do {                                                                          \
        ::doctest::detail::report(__FILE__, __LINE__, "FAIL", #msg);              \
        throw ::doctest::detail::AbortCase{};                                     \
    } while (0)
#define CHECK_THROWS(...)                                                                  \
    do {                                                                                   \
        bool thrown_ = false;                                                              \
        try {                                                                              \
            (void)(__VA_ARGS__);                                                           \
        } catch (...) {                                                                    \
            thrown_ = true;                                                                \
        }                                                                                  \
        ::doctest::detail::check(thrown_, __FILE__, __LINE__, "CHECK_THROWS", #__VA_ARGS__, false); \
    } while (0)
#define CHECK_THROWS_AS(expr, ...)                                                          \
    do {                                                                                    \
        bool thrown_ = false;                                                               \
        try {                                                                               \
            (void)(expr);                                                                   \
        } catch (const __VA_ARGS__&) {                                                      \
            thrown_ = true;                                                                 \
        } catch (...) {                                                                     \
        }                                                                                   \
        ::doctest::detail::check(thrown_, __FILE__, __LINE__, "CHECK_THROWS_AS", #expr, false); \
    } while (0)
#define CHECK_NOTHROW(...)                                                                  \
    do {                                                                                    \
        bool ok_ = true;                                                                    \
        try {                                                                               \
            (void)(__VA_ARGS__);                                                            \
        } catch (...) {                                                                     \
            ok_ = false;                                                                    \
        }                                                                                   \
        ::doctest::detail::check(ok_, __FILE__, __LINE__, "CHECK_NOTHROW", #__VA_ARGS__, false); \
    } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
// Usage: unit_tests [-tc=<substring>]  (runs cases whose name contains <substring>)
int main(int argc, char** argv) {
    const char* filter = nullptr;
    for (int a = 1; a < argc; ++a)
        if (std::strncmp(argv[a], "-tc=", 4) == 0) filter = argv[a] + 4;
    int cases = 0, failed_cases = 0;
    for (const auto& tc : ::doctest::detail::registry()) {
        if (filter && !std::strstr(tc.name, filter)) continue;
        ++cases;
        ::doctest::detail::state().case_failed = false;
        try {
            tc.fn();
        } catch (const ::doctest::detail::AbortCase&) {
        } catch (const std::exception& e) {
            ::doctest::detail::report(tc.file, tc.line, "UNEXPECTED EXCEPTION", e.what());
        } catch (...) {
            ::doctest::detail::report(tc.file, tc.line, "UNEXPECTED EXCEPTION", "unknown");
        }
        if (::doctest::detail::state().case_failed) {
            ++failed_cases;
            std::fprintf(stderr, "  in TEST_CASE \"%s\" (%s:%d)\n", tc.name, tc.file, tc.line);
        }
    }
    const auto& st = ::doctest::detail::state();
    std::printf("[doctest-shim] test cases: %d | %d passed | %d failed\n", cases,
                cases - failed_cases, failed_cases);
    std::printf("[doctest-shim] assertions: %ld | %ld passed | %ld failed\n", st.checks,
                st.checks - st.failed_checks, st.failed_checks);
    return failed_cases ? 1 : 0;
}
#endif
