// Minimal doctest-subset shim -- TEST INFRASTRUCTURE ONLY.
//
// doctest is vendored by the reference but absent from /root/reference
// (proj/.gitignore:2).  This header implements the macros its hot-path unit
// tests use (test_tensor_ops.cpp, test_attention.cpp, test_coverage.cpp) so
// they compile unmodified against the reference sources and the Eigen shim.
// Approx follows doctest 2.x: |a - b| < eps * (scale + max(|a|, |b|)),
// default eps = 100 * FLT_EPSILON, scale = 1.
#pragma once

#include <algorithm>
#include <cfloat>
#include <cmath>
#include <cstdio>
#include <exception>
#include <functional>
#include <string>
#include <vector>

namespace doctest {

class Approx {
  public:
    explicit Approx(double v) : v_(v) {}
    Approx& epsilon(double e) {
        eps_ = e;
        return *this;
    }
    Approx& scale(double s) {
        scale_ = s;
        return *this;
    }
    friend bool operator==(double lhs, const Approx& a) {
        return std::fabs(lhs - a.v_) < a.eps_ * (a.scale_ + std::max(std::fabs(lhs), std::fabs(a.v_)));
    }
    friend bool operator==(const Approx& a, double rhs) { return rhs == a; }
    friend bool operator!=(double lhs, const Approx& a) { return !(lhs == a); }
    friend bool operator!=(const Approx& a, double rhs) { return !(rhs == a); }

  private:
    double v_;
    double eps_ = static_cast<double>(FLT_EPSILON) * 100;
    double scale_ = 1.0;
};

struct Contains {
    explicit Contains(const char* s) : s_(s) {}
    bool matches(const std::string& what) const { return what.find(s_) != std::string::npos; }
    std::string s_;
};

namespace shim {

struct TestCase {
    void (*fn)();
    const char* name;
    const char* file;
    int line;
};

inline std::vector<TestCase>& registry() {
    static std::vector<TestCase> r;
    return r;
}

inline int& failures() {
    static int f = 0;
    return f;
}
inline int& checks() {
    static int c = 0;
    return c;
}

struct Reg {
    Reg(void (*fn)(), const char* name, const char* file, int line) {
        registry().push_back({fn, name, file, line});
    }
};

struct RequireFailed {};

inline void report(bool ok, const char* expr, const char* file, int line, bool require) {
    ++checks();
    if (!ok) {
        ++failures();
        std::fprintf(stderr, "%s:%d: CHECK FAILED: %s\n", file, line, expr);
        if (require) throw RequireFailed{};
    }
}

}  // namespace shim
}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)

#define TEST_SUITE(name) namespace
#define TEST_CASE(name) DOCTEST_TC_(DOCTEST_CAT(doctest_tc_, __LINE__), name)
#define DOCTEST_TC_(fn, name)                                                                  \
    static void fn();                                                                          \
    static ::doctest::shim::Reg DOCTEST_CAT(fn, _reg)(fn, name, __FILE__, __LINE__);           \
    static void fn()

#define CHECK(...) ::doctest::shim::report(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, false)
#define CHECK_FALSE(...) ::doctest::shim::report(!static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, false)
#define REQUIRE(...) ::doctest::shim::report(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, true)

#define CHECK_THROWS_AS(expr, ...)                                                             \
    do {                                                                                       \
        bool ok_ = false;                                                                      \
        try {                                                                                  \
            static_cast<void>(expr);                                                           \
        } catch (const __VA_ARGS__&) {                                                         \
            ok_ = true;                                                                        \
        } catch (...) {                                                                        \
        }                                                                                      \
        ::doctest::shim::report(ok_, "THROWS_AS " #expr, __FILE__, __LINE__, false);           \
    } while (0)

#define CHECK_THROWS_WITH_AS(expr, matcher, ...)                                               \
    do {                                                                                       \
        bool ok_ = false;                                                                      \
        try {                                                                                  \
            static_cast<void>(expr);                                                           \
        } catch (const __VA_ARGS__& e_) {                                                      \
            ok_ = (matcher).matches(e_.what());                                                \
        } catch (...) {                                                                        \
        }                                                                                      \
        ::doctest::shim::report(ok_, "THROWS_WITH_AS " #expr, __FILE__, __LINE__, false);      \
    } while (0)

#define CHECK_NOTHROW(...)                                                                     \
    do {                                                                                       \
        bool ok_ = true;                                                                       \
        try {                                                                                  \
            static_cast<void>(__VA_ARGS__);                                                    \
        } catch (...) {                                                                        \
            ok_ = false;                                                                       \
        }                                                                                      \
        ::doctest::shim::report(ok_, "NOTHROW " #__VA_ARGS__, __FILE__, __LINE__, false);      \
    } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() {
    int failed_cases = 0;
    for (const auto& tc : ::doctest::shim::registry()) {
        const int before = ::doctest::shim::failures();
        try {
            tc.fn();
        } catch (const ::doctest::shim::RequireFailed&) {
        } catch (const std::exception& e) {
            ++::doctest::shim::failures();
            std::fprintf(stderr, "%s:%d: test case '%s' threw: %s\n", tc.file, tc.line, tc.name,
                         e.what());
        }
        if (::doctest::shim::failures() != before) {
            ++failed_cases;
            std::fprintf(stderr, "FAILED: %s\n", tc.name);
        }
    }
    std::printf("[doctest-shim] test cases: %zu | failed: %d | checks: %d | failed checks: %d\n",
                ::doctest::shim::registry().size(), failed_cases, ::doctest::shim::checks(),
                ::doctest::shim::failures());
    return failed_cases ? 1 : 0;
}
#endif
