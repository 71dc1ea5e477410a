// doctest-subset: just enough of the doctest API to compile and run the
// reference's own unit tests (proj/tests/*.cpp) against
// (a) the reference hot-path sources built as the parity oracle and (b) this
// repo's C++ drop-in.  TEST INFRASTRUCTURE ONLY -- never linked into the product.
//
// Semantics kept from doctest:
//   * SUBCASE: the enclosing TEST_CASE body is re-run once per leaf subcase;
//   * Approx: |a-b| < eps * (scale + max(|a|,|b|)), eps default FLT_EPSILON*100;
//   * REQUIRE aborts the current test case, CHECK records and continues.
#pragma once

#include <algorithm>
#include <cfloat>
#include <cmath>
#include <cstdio>
#include <exception>
#include <functional>
#include <sstream>
#include <stdexcept>
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
    bool matches(double lhs) const {
        return std::fabs(lhs - value_) <
               eps_ * (scale_ + std::max(std::fabs(lhs), std::fabs(value_)));
    }
    double value() const { return value_; }
    friend bool operator==(double lhs, const Approx& r) { return r.matches(lhs); }
    friend bool operator==(const Approx& r, double rhs) { return r.matches(rhs); }
    friend bool operator!=(double lhs, const Approx& r) { return !r.matches(lhs); }
    friend bool operator!=(const Approx& r, double rhs) { return !r.matches(rhs); }

private:
    double value_;
    double eps_ = double(FLT_EPSILON) * 100;
    double scale_ = 1.0;
};

struct Contains {
    explicit Contains(std::string s) : needle(std::move(s)) {}
    bool check(const std::string& hay) const { return hay.find(needle) != std::string::npos; }
    std::string needle;
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

struct State {
    int subcase_target = 0;
    int subcase_seen = 0;
    long checks = 0;
    long failures = 0;
    bool current_failed = false;
};
inline State& state() {
    static State s;
    return s;
}

struct RequireFailed {};

inline void report(bool ok, const char* kind, const char* expr, const char* file, int line) {
    auto& s = state();
    ++s.checks;
    if (ok)
        return;
    ++s.failures;
    s.current_failed = true;
    std::fprintf(stderr, "%s:%d: FAILED %s( %s )\n", file, line, kind, expr);
}

struct Registrar {
    Registrar(const char* name, const char* file, int line, void (*fn)()) {
        registry().push_back({name, file, line, fn});
    }
};

struct SubcaseGuard {
    bool active;
    explicit SubcaseGuard(const char*) {
        auto& s = state();
        active = (s.subcase_seen == s.subcase_target);
        ++s.subcase_seen;
    }
    explicit operator bool() const { return active; }
};

inline int run_all() {
    int failed_cases = 0;
    for (const auto& tc : registry()) {
        auto& s = state();
        s.current_failed = false;
        s.subcase_target = 0;
        for (;;) {
            s.subcase_seen = 0;
            try {
                tc.fn();
            } catch (const RequireFailed&) {
            } catch (const std::exception& e) {
                ++s.failures;
                s.current_failed = true;
                std::fprintf(stderr, "%s:%d: test case threw: %s\n", tc.file, tc.line, e.what());
            }
            if (s.subcase_seen > s.subcase_target + 1)
                ++s.subcase_target;
            else
                break;
        }
        std::fprintf(stderr, "[%s] %s\n", s.current_failed ? "FAIL" : " ok ", tc.name);
        failed_cases += s.current_failed ? 1 : 0;
    }
    const auto& s = state();
    std::fprintf(stderr, "test cases: %zu | %d failed | assertions: %ld | %ld failed\n",
                 registry().size(), failed_cases, s.checks, s.failures);
    return failed_cases == 0 ? 0 : 1;
}

} // namespace detail
} // namespace doctest

#define DOCTEST_CAT_IMPL(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_IMPL(a, b)

#define TEST_CASE(name)                                                                        \
    static void DOCTEST_CAT(doctest_fn_, __LINE__)();                                          \
    static ::doctest::detail::Registrar DOCTEST_CAT(doctest_reg_, __LINE__)(                   \
        name, __FILE__, __LINE__, &DOCTEST_CAT(doctest_fn_, __LINE__));                        \
    static void DOCTEST_CAT(doctest_fn_, __LINE__)()

#define SUBCASE(name) if (const ::doctest::detail::SubcaseGuard DOCTEST_CAT(doctest_sc_, __LINE__){name})

#define CHECK(...)                                                                             \
    ::doctest::detail::report(static_cast<bool>(__VA_ARGS__), "CHECK", #__VA_ARGS__, __FILE__, \
                              __LINE__)
#define CHECK_FALSE(...)                                                                       \
    ::doctest::detail::report(!static_cast<bool>(__VA_ARGS__), "CHECK_FALSE", #__VA_ARGS__,    \
                              __FILE__, __LINE__)
#define REQUIRE(...)                                                                           \
    do {                                                                                       \
        const bool doctest_ok_ = static_cast<bool>(__VA_ARGS__);                               \
        ::doctest::detail::report(doctest_ok_, "REQUIRE", #__VA_ARGS__, __FILE__, __LINE__);   \
        if (!doctest_ok_)                                                                      \
            throw ::doctest::detail::RequireFailed{};                                          \
    } while (0)
#define CHECK_THROWS_AS(expr, type)                                                            \
    do {                                                                                       \
        bool doctest_ok_ = false;                                                              \
        try {                                                                                  \
            (void)(expr);                                                                      \
        } catch (const type&) {                                                                \
            doctest_ok_ = true;                                                                \
        } catch (...) {                                                                        \
        }                                                                                      \
        ::doctest::detail::report(doctest_ok_, "CHECK_THROWS_AS", #expr, __FILE__, __LINE__);  \
    } while (0)
#define CHECK_THROWS_WITH_AS(expr, matcher, type)                                              \
    do {                                                                                       \
        bool doctest_ok_ = false;                                                              \
        try {                                                                                  \
            (void)(expr);                                                                      \
        } catch (const type& e) {                                                              \
            doctest_ok_ = (matcher).check(e.what());                                           \
        } catch (...) {                                                                        \
        }                                                                                      \
        ::doctest::detail::report(doctest_ok_, "CHECK_THROWS_WITH_AS", #expr, __FILE__,        \
                                  __LINE__);                                                   \
    } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() { return ::doctest::detail::run_all(); }
#endif
