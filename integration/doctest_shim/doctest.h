// Minimal stand-in for doctest (absent from the reference's vendor/, SURVEY.md
// §8c) -- TEST INFRASTRUCTURE ONLY. It implements exactly the surface the
// reference's unit suites use (tests/{engine,monitor,toolkit}_test.cpp):
// TEST_CASE, flat SUBCASE, CHECK, REQUIRE, CHECK_THROWS_AS, doctest::Approx
// (with .epsilon), and DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN. The suites then
// compile unmodified, so the reference's own assertions can judge the GPU
// adapter (integration/flowmon_gpu.cpp).
//
// SUBCASE follows doctest's re-run model for one nesting level: a test case
// with k distinct SUBCASE sites runs k times, entering the i-th site on run i
// (every time that site is reached, e.g. inside a loop) and skipping the rest.
#ifndef GNM_DOCTEST_SHIM_H
#define GNM_DOCTEST_SHIM_H

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <exception>
#include <limits>
#include <ostream>
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
    // doctest's rule: |lhs - rhs| < eps * (scale + max(|lhs|, |rhs|))
    bool matches(double other) const {
        return std::fabs(other - value_) <
               eps_ * (scale_ + std::max(std::fabs(other), std::fabs(value_)));
    }
    double value() const { return value_; }

private:
    double value_;
    double eps_ = static_cast<double>(std::numeric_limits<float>::epsilon()) * 100;
    double scale_ = 1.0;
};

inline bool operator==(double lhs, const Approx& rhs) { return rhs.matches(lhs); }
inline bool operator==(const Approx& lhs, double rhs) { return lhs.matches(rhs); }
inline bool operator!=(double lhs, const Approx& rhs) { return !rhs.matches(lhs); }
inline bool operator!=(const Approx& lhs, double rhs) { return !lhs.matches(rhs); }
inline bool operator<=(double lhs, const Approx& rhs) { return lhs < rhs.value() || rhs.matches(lhs); }
inline bool operator>=(double lhs, const Approx& rhs) { return lhs > rhs.value() || rhs.matches(lhs); }
inline std::ostream& operator<<(std::ostream& os, const Approx& a) { return os << "Approx(" << a.value() << ")"; }

namespace shim {

struct RequireFailed {};

using TestFn = void (*)();
struct TestCase {
    const char* name;
    const char* file;
    int line;
    TestFn fn;
};

inline std::vector<TestCase>& registry() {
    static std::vector<TestCase> r;
    return r;
}

struct State {
    int target = 0;              // SUBCASE site entered on this run
    std::vector<int> sites;      // distinct SUBCASE sites (by line) met so far in this case
    long long asserts = 0, failed_asserts = 0;
    bool case_failed = false;
    const TestCase* current = nullptr;
};

inline State& state() {
    static State s;
    return s;
}

inline bool enter_subcase(int line) {
    State& s = state();
    auto it = std::find(s.sites.begin(), s.sites.end(), line);
    int idx;
    if (it == s.sites.end()) {
        s.sites.push_back(line);
        idx = static_cast<int>(s.sites.size()) - 1;
    } else {
        idx = static_cast<int>(it - s.sites.begin());
    }
    return idx == s.target;
}

inline void report(bool ok, const char* kind, const char* expr, const char* file, int line) {
    State& s = state();
    ++s.asserts;
    if (ok) return;
    ++s.failed_asserts;
    s.case_failed = true;
    std::printf("%s:%d: FAILED %s( %s ) in TEST_CASE \"%s\"", file, line, kind, expr,
                s.current ? s.current->name : "?");
    if (s.target >= 0 && !s.sites.empty()) std::printf(" [subcase run %d]", s.target);
    std::printf("\n");
}

struct Registrar {
    Registrar(const char* name, const char* file, int line, TestFn fn) {
        registry().push_back({name, file, line, fn});
    }
};

inline int run_all() {
    State& s = state();
    int failed_cases = 0;
    for (const TestCase& tc : registry()) {
        s.current = &tc;
        s.case_failed = false;
        s.sites.clear();
        for (s.target = 0;; ++s.target) {
            try {
                tc.fn();
            } catch (const RequireFailed&) {
            } catch (const std::exception& e) {
                report(false, "TEST_CASE threw", e.what(), tc.file, tc.line);
            } catch (...) {
                report(false, "TEST_CASE threw", "unknown exception", tc.file, tc.line);
            }
            if (s.target + 1 >= static_cast<int>(s.sites.size())) break;
        }
        if (s.case_failed) ++failed_cases;
        std::printf("[%s] %s\n", s.case_failed ? "FAIL" : " ok ", tc.name);
    }
    std::printf("[doctest-shim] test cases: %zu | %zu passed | %d failed | assertions: %lld | %lld failed\n",
                registry().size(), registry().size() - failed_cases, failed_cases, s.asserts,
                s.failed_asserts);
    return failed_cases ? 1 : 0;
}

} // namespace shim
} // namespace doctest

#define DOCTEST_SHIM_CAT2(a, b) a##b
#define DOCTEST_SHIM_CAT(a, b) DOCTEST_SHIM_CAT2(a, b)
#define DOCTEST_SHIM_TEST_CASE_IMPL(fn, name)                                                     \
    static void fn();                                                                             \
    static ::doctest::shim::Registrar DOCTEST_SHIM_CAT(fn, _reg)(name, __FILE__, __LINE__, &fn);  \
    static void fn()
#define TEST_CASE(name) DOCTEST_SHIM_TEST_CASE_IMPL(DOCTEST_SHIM_CAT(doctest_shim_case_, __LINE__), name)

#define SUBCASE(name) if (::doctest::shim::enter_subcase(__LINE__))

#define CHECK(...)                                                                                \
    do {                                                                                          \
        bool doctest_shim_ok = false;                                                             \
        try {                                                                                     \
            doctest_shim_ok = static_cast<bool>(__VA_ARGS__);                                     \
        } catch (...) {                                                                           \
        }                                                                                         \
        ::doctest::shim::report(doctest_shim_ok, "CHECK", #__VA_ARGS__, __FILE__, __LINE__);      \
    } while (0)

#define REQUIRE(...)                                                                              \
    do {                                                                                          \
        bool doctest_shim_ok = false;                                                             \
        try {                                                                                     \
            doctest_shim_ok = static_cast<bool>(__VA_ARGS__);                                     \
        } catch (...) {                                                                           \
        }                                                                                         \
        ::doctest::shim::report(doctest_shim_ok, "REQUIRE", #__VA_ARGS__, __FILE__, __LINE__);    \
        if (!doctest_shim_ok) throw ::doctest::shim::RequireFailed{};                             \
    } while (0)

#define CHECK_THROWS_AS(expr, ...)                                                                \
    do {                                                                                          \
        bool doctest_shim_ok = false;                                                             \
        try {                                                                                     \
            static_cast<void>(expr);                                                              \
        } catch (const __VA_ARGS__&) {                                                            \
            doctest_shim_ok = true;                                                               \
        } catch (...) {                                                                           \
        }                                                                                         \
        ::doctest::shim::report(doctest_shim_ok, "CHECK_THROWS_AS", #expr ", " #__VA_ARGS__,      \
                                __FILE__, __LINE__);                                              \
    } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() { return ::doctest::shim::run_all(); }
#endif

#endif
