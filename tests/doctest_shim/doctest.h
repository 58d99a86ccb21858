// Minimal doctest-compatible test harness (our own code, not doctest): just
// the subset the reference's C++ unit tests use -- TEST_CASE, SUBCASE (run in
// sequence), CHECK, CHECK_FALSE, CHECK_THROWS_AS, REQUIRE, FAIL and
// doctest::Approx -- so those tests can be compiled UNCHANGED against this
// repository's headers and library (oracle/Makefile target unit_ours).
#pragma once

#include <cmath>
#include <cstdio>
#include <exception>
#include <functional>
#include <string>
#include <vector>

namespace doctest {

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

struct Registrar {
    Registrar(const char* name, const char* file, int line, void (*fn)()) {
        registry().push_back({name, file, line, fn});
    }
};

struct State {
    int checks = 0;
    int failed_checks = 0;
    bool case_failed = false;
};

inline State& state() {
    static State s;
    return s;
}

struct RequireAbort {};

inline void fail(const char* file, int line, const std::string& what) {
    std::printf("  %s:%d: FAILED: %s\n", file, line, what.c_str());
    state().failed_checks++;
    state().case_failed = true;
}

inline void check(bool ok, const char* file, int line, const char* expr, bool require) {
    state().checks++;
    if (ok) return;
    fail(file, line, std::string(require ? "REQUIRE( " : "CHECK( ") + expr + " )");
    if (require) throw RequireAbort{};
}

} // namespace detail

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
    friend bool operator==(double lhs, const Approx& rhs) {
        const double m = std::max(std::fabs(lhs), std::fabs(rhs.value_));
        return std::fabs(lhs - rhs.value_) < rhs.eps_ * (rhs.scale_ + m);
    }
    friend bool operator==(const Approx& lhs, double rhs) { return rhs == lhs; }
    friend bool operator!=(double lhs, const Approx& rhs) { return !(lhs == rhs); }
    friend bool operator!=(const Approx& lhs, double rhs) { return !(rhs == lhs); }

private:
    double value_;
    double eps_ = 1.1920929e-07f * 100;  // doctest's default: 100 float epsilons
    double scale_ = 1.0;
};

} // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)

#define TEST_CASE(name)                                                                                      \
    static void DOCTEST_CAT(doctest_case_, __LINE__)();                                                      \
    static ::doctest::detail::Registrar DOCTEST_CAT(doctest_reg_, __LINE__)(name, __FILE__, __LINE__,        \
                                                                         &DOCTEST_CAT(doctest_case_, __LINE__)); \
    static void DOCTEST_CAT(doctest_case_, __LINE__)()

// Subcases run one after another inside a single pass of the test case.
#define SUBCASE(name) if (true)

#define CHECK(...) ::doctest::detail::check(static_cast<bool>(__VA_ARGS__), __FILE__, __LINE__, #__VA_ARGS__, false)
#define CHECK_FALSE(...) \
    ::doctest::detail::check(!static_cast<bool>(__VA_ARGS__), __FILE__, __LINE__, "!(" #__VA_ARGS__ ")", false)
#define REQUIRE(...) ::doctest::detail::check(static_cast<bool>(__VA_ARGS__), __FILE__, __LINE__, #__VA_ARGS__, true)
#define FAIL(msg)                                                                                            \
    do {                                                                                                     \
        ::doctest::detail::fail(__FILE__, __LINE__, std::string("FAIL: ") + (msg));                          \
        throw ::doctest::detail::RequireAbort{};                                                             \
    } while (0)
#define CHECK_THROWS_AS(expr, ...)                                                                            \
    do {                                                                                                     \
        ::doctest::detail::state().checks++;                                                                 \
        bool doctest_ok_ = false;                                                                            \
        try {                                                                                                \
            static_cast<void>(expr);                                                                         \
        } catch (const __VA_ARGS__&) {                                                                       \
            doctest_ok_ = true;                                                                              \
        } catch (...) {                                                                                      \
        }                                                                                                    \
        if (!doctest_ok_)                                                                                    \
            ::doctest::detail::fail(__FILE__, __LINE__, "CHECK_THROWS_AS( " #expr ", " #__VA_ARGS__ " )");   \
    } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() {
    int cases = 0, failed_cases = 0;
    for (const auto& c : ::doctest::detail::registry()) {
        ++cases;
        ::doctest::detail::state().case_failed = false;
        try {
            c.fn();
        } catch (const ::doctest::detail::RequireAbort&) {
        } catch (const std::exception& e) {
            ::doctest::detail::fail(c.file, c.line, std::string("unexpected exception: ") + e.what());
        } catch (...) {
            ::doctest::detail::fail(c.file, c.line, "unexpected non-standard exception");
        }
        if (::doctest::detail::state().case_failed) {
            ++failed_cases;
            std::printf("[FAIL] %s (%s:%d)\n", c.name, c.file, c.line);
        }
    }
    const auto& s = ::doctest::detail::state();
    std::printf("test cases: %d | %d passed | %d failed\nassertions: %d | %d passed | %d failed\n", cases,
                cases - failed_cases, failed_cases, s.checks, s.checks - s.failed_checks, s.failed_checks);
    return failed_cases ? 1 : 0;
}
#endif
