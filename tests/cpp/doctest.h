// tests/cpp/doctest.h — a minimal doctest-compatible test harness (the real
// doctest header is not vendored in the reference tree and there is no
// network). It implements exactly the subset the reference's hot-path unit
// suites use — TEST_CASE, CHECK, CHECK_FALSE, REQUIRE, CHECK_THROWS_AS,
// CHECK_NOTHROW, doctest::Approx(+ .epsilon()) — so those suites compile
// unchanged against either the reference library or the B200 drop-in.
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <exception>
#include <functional>
#include <limits>
#include <string>
#include <vector>

namespace doctest {

class Approx {
public:
    explicit Approx(double value) : value_(value) {}
    Approx& epsilon(double e) {
        eps_ = e;
        return *this;
    }
    friend bool operator==(double lhs, const Approx& rhs) { return rhs.near(lhs); }
    friend bool operator==(const Approx& lhs, double rhs) { return lhs.near(rhs); }
    friend bool operator!=(double lhs, const Approx& rhs) { return !rhs.near(lhs); }
    friend bool operator!=(const Approx& lhs, double rhs) { return !lhs.near(rhs); }

private:
    // |a - v| < eps * (scale + max(|a|, |v|)), scale = 1 (doctest's rule)
    bool near(double a) const { return std::fabs(a - value_) < eps_ * (1.0 + std::max(std::fabs(a), std::fabs(value_))); }
    double value_;
    double eps_ = static_cast<double>(std::numeric_limits<float>::epsilon()) * 100.0;
};

namespace detail {

struct Case {
    const char* name;
    const char* file;
    int line;
    void (*fn)();
};

inline std::vector<Case>& registry() {
    static std::vector<Case> cases;
    return cases;
}

struct Registrar {
    Registrar(const char* name, const char* file, int line, void (*fn)()) {
        registry().push_back({name, file, line, fn});
    }
};

struct State {
    long long assertions = 0;
    long long failed_assertions = 0;
    bool case_failed = false;
};
inline State& state() {
    static State s;
    return s;
}

struct RequireAbort {};

inline void report(bool ok, const char* kind, const char* expr, const char* file, int line, bool fatal) {
    State& s = state();
    ++s.assertions;
    if (ok) return;
    ++s.failed_assertions;
    s.case_failed = true;
    std::fprintf(stderr, "%s:%d: ERROR: %s( %s ) is NOT correct!\n", file, line, kind, expr);
    if (fatal) throw RequireAbort{};
}

}  // namespace detail

int run_all(int argc, char** argv);

}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define DOCTEST_TC_IMPL(fn, name)                                                                   \
    static void fn();                                                                               \
    static const ::doctest::detail::Registrar DOCTEST_CAT(fn, _reg)(name, __FILE__, __LINE__, &fn); \
    static void fn()
#define TEST_CASE(name) DOCTEST_TC_IMPL(DOCTEST_CAT(doctest_case_, __COUNTER__), name)

#define DOCTEST_ASSERT_(kind, cond, text, fatal)                                                     \
    do {                                                                                             \
        bool doctest_ok_ = false;                                                                    \
        try {                                                                                        \
            doctest_ok_ = static_cast<bool>(cond);                                                   \
        } catch (const ::doctest::detail::RequireAbort&) {                                           \
            throw;                                                                                   \
        } catch (...) {                                                                              \
            doctest_ok_ = false;                                                                     \
        }                                                                                            \
        ::doctest::detail::report(doctest_ok_, kind, text, __FILE__, __LINE__, fatal);               \
    } while (0)

#define CHECK(...) DOCTEST_ASSERT_("CHECK", (__VA_ARGS__), #__VA_ARGS__, false)
#define CHECK_FALSE(...) DOCTEST_ASSERT_("CHECK_FALSE", !(__VA_ARGS__), #__VA_ARGS__, false)
#define REQUIRE(...) DOCTEST_ASSERT_("REQUIRE", (__VA_ARGS__), #__VA_ARGS__, true)

#define CHECK_THROWS_AS(expr, ...)                                                                   \
    do {                                                                                             \
        bool doctest_ok_ = false;                                                                    \
        try {                                                                                        \
            static_cast<void>(expr);                                                                 \
        } catch (const __VA_ARGS__&) {                                                               \
            doctest_ok_ = true;                                                                      \
        } catch (...) {                                                                              \
        }                                                                                            \
        ::doctest::detail::report(doctest_ok_, "CHECK_THROWS_AS", #expr ", " #__VA_ARGS__, __FILE__, \
                                  __LINE__, false);                                                  \
    } while (0)

#define CHECK_NOTHROW(expr)                                                                          \
    do {                                                                                             \
        bool doctest_ok_ = true;                                                                     \
        try {                                                                                        \
            static_cast<void>(expr);                                                                 \
        } catch (...) {                                                                              \
            doctest_ok_ = false;                                                                     \
        }                                                                                            \
        ::doctest::detail::report(doctest_ok_, "CHECK_NOTHROW", #expr, __FILE__, __LINE__, false);   \
    } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
namespace doctest {
// Runs every registered case (or those whose name contains argv[1]).
int run_all(int argc, char** argv) {
    const char* filter = argc > 1 ? argv[1] : nullptr;
    int cases = 0, failed = 0;
    for (const detail::Case& c : detail::registry()) {
        if (filter && !std::strstr(c.name, filter)) continue;
        ++cases;
        detail::state().case_failed = false;
        try {
            c.fn();
        } catch (const detail::RequireAbort&) {
        } catch (const std::exception& e) {
            std::fprintf(stderr, "%s:%d: ERROR: test case \"%s\" threw: %s\n", c.file, c.line, c.name, e.what());
            detail::state().case_failed = true;
        } catch (...) {
            std::fprintf(stderr, "%s:%d: ERROR: test case \"%s\" threw a non-std exception\n", c.file, c.line,
                         c.name);
            detail::state().case_failed = true;
        }
        if (detail::state().case_failed) {
            ++failed;
            std::fprintf(stderr, "[doctest] FAILED: %s\n", c.name);
        }
    }
    const detail::State& s = detail::state();
    std::printf("[doctest] test cases: %d | %d passed | %d failed\n", cases, cases - failed, failed);
    std::printf("[doctest] assertions: %lld | %lld passed | %lld failed\n", s.assertions,
                s.assertions - s.failed_assertions, s.failed_assertions);
    std::printf("[doctest] Status: %s!\n", failed ? "FAILURE" : "SUCCESS");
    return failed ? 1 : 0;
}
}  // namespace doctest
int main(int argc, char** argv) { return doctest::run_all(argc, argv); }
#endif
