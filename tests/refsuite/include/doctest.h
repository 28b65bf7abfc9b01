// doctest.h -- a minimal doctest-compatible test harness (test infrastructure).
//
// The reference's unit suites (/root/reference/proj/tests/test_*.cpp) are
// written against doctest, which the image does not ship. This
// header implements the subset they use -- TEST_CASE, CHECK, CHECK_FALSE,
// CHECK_NOTHROW, CHECK_THROWS_AS, REQUIRE, FAIL, doctest::Approx -- so those
// files compile UNMODIFIED against include/blockeig_b200.hpp (through the
// forwarding headers in tests/refsuite/include/blockeig/) and run the hot
// path on the B200. Semantics follow doctest: a failed CHECK records the
// failure and continues, a failed REQUIRE / FAIL / an escaping exception ends
// the test case; the process exits non-zero if any test case failed.
//
// Command line: an optional substring filter on test-case names (-tc=<s>,
// as doctest's) and -s / --success to list every case.
#pragma once

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <exception>
#include <functional>
#include <limits>
#include <sstream>
#include <string>
#include <typeinfo>
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
    bool matches(double other) const {
        // doctest: |a - b| < eps * (scale + max(|a|, |b|))
        return std::fabs(other - value_) < eps_ * (scale_ + std::max(std::fabs(other), std::fabs(value_)));
    }
    double value() const { return value_; }
    friend bool operator==(double lhs, const Approx& rhs) { return rhs.matches(lhs); }
    friend bool operator==(const Approx& lhs, double rhs) { return lhs.matches(rhs); }
    friend bool operator!=(double lhs, const Approx& rhs) { return !rhs.matches(lhs); }
    friend bool operator!=(const Approx& lhs, double rhs) { return !lhs.matches(rhs); }
    friend bool operator<=(double lhs, const Approx& rhs) { return lhs < rhs.value_ || rhs.matches(lhs); }
    friend bool operator>=(double lhs, const Approx& rhs) { return lhs > rhs.value_ || rhs.matches(lhs); }

private:
    double value_;
    double eps_ = static_cast<double>(std::numeric_limits<float>::epsilon()) * 100;
    double scale_ = 1.0;
};

namespace detail {

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

struct State {
    int checks = 0;
    int failed_checks = 0;
    bool case_failed = false;
    const char* case_name = "";
};

inline State& state() {
    static State s;
    return s;
}

struct RequireAbort {};  // ends the current test case

struct Registrar {
    Registrar(const char* name, const char* file, int line, void (*fn)()) {
        registry().push_back(Case{name, file, line, fn});
    }
};

inline void report(bool ok, const char* kind, const char* expr, const char* file, int line,
                   const std::string& extra = {}) {
    ++state().checks;
    if (ok) return;
    ++state().failed_checks;
    state().case_failed = true;
    std::fprintf(stderr, "%s:%d: ERROR: %s( %s ) is NOT correct!%s%s\n  in test case \"%s\"\n", file, line, kind, expr,
                 extra.empty() ? "" : "\n  ", extra.c_str(), state().case_name);
}

inline int run(int argc, char** argv) {
    std::string filter;
    bool list = false;
    for (int i = 1; i < argc; ++i) {
        std::string a = argv[i];
        if (a.rfind("-tc=", 0) == 0) filter = a.substr(4);
        else if (a == "-s" || a == "--success") list = true;
        else if (a[0] != '-') filter = a;
    }
    int ran = 0, failed = 0;
    for (const auto& c : registry()) {
        if (!filter.empty() && std::string(c.name).find(filter) == std::string::npos) continue;
        ++ran;
        state().case_failed = false;
        state().case_name = c.name;
        try {
            c.fn();
        } catch (const RequireAbort&) {
        } catch (const std::exception& e) {
            std::fprintf(stderr, "%s:%d: ERROR: test case \"%s\" threw %s: %s\n", c.file, c.line, c.name,
                         typeid(e).name(), e.what());
            state().case_failed = true;
        } catch (...) {
            std::fprintf(stderr, "%s:%d: ERROR: test case \"%s\" threw an unknown exception\n", c.file, c.line,
                         c.name);
            state().case_failed = true;
        }
        if (state().case_failed) ++failed;
        if (list || state().case_failed)
            std::fprintf(stderr, "[%s] %s\n", state().case_failed ? "FAILED" : "passed", c.name);
    }
    std::printf("[doctest-shim] test cases: %d | %d passed | %d failed\n", ran, ran - failed, failed);
    std::printf("[doctest-shim] assertions: %d | %d passed | %d failed\n", state().checks,
                state().checks - state().failed_checks, state().failed_checks);
    return failed == 0 && ran > 0 ? 0 : 1;
}

}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define DOCTEST_TEST_CASE_IMPL(fn, name)                                                        \
    static void fn();                                                                           \
    static ::doctest::detail::Registrar DOCTEST_CAT(fn, _reg)(name, __FILE__, __LINE__, &fn);   \
    static void fn()
#define TEST_CASE(name) DOCTEST_TEST_CASE_IMPL(DOCTEST_CAT(doctest_case_, __COUNTER__), name)

#define CHECK(...) ::doctest::detail::report(static_cast<bool>(__VA_ARGS__), "CHECK", #__VA_ARGS__, __FILE__, __LINE__)
#define CHECK_FALSE(...) \
    ::doctest::detail::report(!static_cast<bool>(__VA_ARGS__), "CHECK_FALSE", #__VA_ARGS__, __FILE__, __LINE__)
#define REQUIRE(...)                                                                                     \
    do {                                                                                                 \
        const bool doctest_ok_ = static_cast<bool>(__VA_ARGS__);                                         \
        ::doctest::detail::report(doctest_ok_, "REQUIRE", #__VA_ARGS__, __FILE__, __LINE__);             \
        if (!doctest_ok_) throw ::doctest::detail::RequireAbort{};                                       \
    } while (0)
#define CHECK_NOTHROW(...)                                                                               \
    do {                                                                                                 \
        std::string doctest_what_;                                                                       \
        bool doctest_ok_ = true;                                                                         \
        try {                                                                                            \
            static_cast<void>(__VA_ARGS__);                                                              \
        } catch (const std::exception& e) {                                                              \
            doctest_ok_ = false;                                                                         \
            doctest_what_ = std::string("threw: ") + e.what();                                           \
        } catch (...) {                                                                                  \
            doctest_ok_ = false;                                                                         \
            doctest_what_ = "threw an unknown exception";                                                \
        }                                                                                                \
        ::doctest::detail::report(doctest_ok_, "CHECK_NOTHROW", #__VA_ARGS__, __FILE__, __LINE__,        \
                                  doctest_what_);                                                        \
    } while (0)
#define CHECK_THROWS_AS(expr, ...)                                                                       \
    do {                                                                                                 \
        bool doctest_ok_ = false;                                                                        \
        std::string doctest_what_ = "did not throw";                                                     \
        try {                                                                                            \
            static_cast<void>(expr);                                                                     \
        } catch (const __VA_ARGS__&) {                                                                   \
            doctest_ok_ = true;                                                                          \
        } catch (const std::exception& e) {                                                              \
            doctest_what_ = std::string("threw a different exception (") + typeid(e).name() + "): " +    \
                            e.what();                                                                    \
        } catch (...) {                                                                                  \
            doctest_what_ = "threw an unknown exception";                                                \
        }                                                                                                \
        ::doctest::detail::report(doctest_ok_, "CHECK_THROWS_AS", #expr ", " #__VA_ARGS__, __FILE__,     \
                                  __LINE__, doctest_what_);                                              \
    } while (0)
#define FAIL(msg)                                                                                        \
    do {                                                                                                 \
        std::ostringstream doctest_os_;                                                                  \
        doctest_os_ << msg;                                                                              \
        ::doctest::detail::report(false, "FAIL", doctest_os_.str().c_str(), __FILE__, __LINE__);        \
        throw ::doctest::detail::RequireAbort{};                                                         \
    } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main(int argc, char** argv) { return ::doctest::detail::run(argc, argv); }
#endif
