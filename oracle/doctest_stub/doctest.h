// TEST INFRASTRUCTURE ONLY. Minimal stand-in for the doctest single header the
// reference vendors but does not ship (proj/.gitignore:2 excludes vendor/).
// It implements exactly the macro subset the reference's unit suites use
// (CHECK*, REQUIRE, CHECK_THROWS*, CAPTURE, FAIL, TEST_SUITE, TEST_CASE,
// doctest::Approx, doctest::Contains) so oracle/Makefile can build and run the
// reference's own tests against the reference library. Define
// DOCTEST_STUB_IMPLEMENT in exactly one TU to get the runner (main).
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

struct Approx {
    explicit Approx(double v) : value(v) {}
    Approx& epsilon(double e) { eps = e; return *this; }
    double value;
    double eps = static_cast<double>(std::numeric_limits<float>::epsilon()) * 100.0;
    bool eq(double lhs) const {
        return std::fabs(lhs - value) <
               eps * (1.0 + std::max(std::fabs(lhs), std::fabs(value)));
    }
};
inline bool operator==(double lhs, const Approx& r) { return r.eq(lhs); }
inline bool operator==(const Approx& r, double lhs) { return r.eq(lhs); }
inline bool operator!=(double lhs, const Approx& r) { return !r.eq(lhs); }
inline bool operator!=(const Approx& r, double lhs) { return !r.eq(lhs); }
inline bool operator<=(double lhs, const Approx& r) { return lhs < r.value || r.eq(lhs); }
inline bool operator>=(double lhs, const Approx& r) { return lhs > r.value || r.eq(lhs); }

struct Contains {
    explicit Contains(const char* s) : needle(s) {}
    std::string needle;
};
inline bool what_matches(const char* what, const Contains& c) {
    return std::string(what).find(c.needle) != std::string::npos;
}
inline bool what_matches(const char* what, const char* exact) { return std::string(what) == exact; }

namespace stub {
struct TestCase {
    const char* suite;
    const char* name;
    void (*fn)();
};
struct Abort {};
inline std::vector<TestCase>& registry() {
    static std::vector<TestCase> r;
    return r;
}
inline const char*& current_suite() {
    static const char* s = "";
    return s;
}
inline int& failures() {
    static int f = 0;
    return f;
}
inline int& assertions() {
    static int a = 0;
    return a;
}
inline const char* set_suite(const char* s) {
    current_suite() = s;
    return s;
}
struct Reg {
    Reg(const char* name, void (*fn)()) { registry().push_back({current_suite(), name, fn}); }
};
inline void report(bool ok, const char* expr, const char* file, int line, bool fatal) {
    ++assertions();
    if (ok) return;
    ++failures();
    std::fprintf(stderr, "%s:%d: FAILED: %s\n", file, line, expr);
    if (fatal) throw Abort{};
}
} // namespace stub
} // namespace doctest

#define DOCTEST_STUB_CAT2(a, b) a##b
#define DOCTEST_STUB_CAT(a, b) DOCTEST_STUB_CAT2(a, b)
#define TEST_SUITE(name)                                                                  \
    static const char* DOCTEST_STUB_CAT(ds_suite_, __LINE__) =                            \
        doctest::stub::set_suite(name);                                                   \
    namespace
#define TEST_CASE(name)                                                                   \
    static void DOCTEST_STUB_CAT(ds_test_, __LINE__)();                                   \
    static doctest::stub::Reg DOCTEST_STUB_CAT(ds_reg_, __LINE__)(                        \
        name, &DOCTEST_STUB_CAT(ds_test_, __LINE__));                                     \
    static void DOCTEST_STUB_CAT(ds_test_, __LINE__)()
#define CHECK(...) doctest::stub::report(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, false)
#define CHECK_FALSE(...) doctest::stub::report(!static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, false)
#define REQUIRE(...) doctest::stub::report(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, true)
#define REQUIRE_FALSE(...) doctest::stub::report(!static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, true)
#define CAPTURE(x) ((void)0)
#define FAIL(msg) doctest::stub::report(false, msg, __FILE__, __LINE__, true)
#define CHECK_NOTHROW(...)                                                                \
    do {                                                                                  \
        bool ok_ = true;                                                                  \
        try { (void)(__VA_ARGS__); } catch (...) { ok_ = false; }                         \
        doctest::stub::report(ok_, "NOTHROW " #__VA_ARGS__, __FILE__, __LINE__, false);   \
    } while (0)
#define CHECK_THROWS(...)                                                                 \
    do {                                                                                  \
        bool ok_ = false;                                                                 \
        try { (void)(__VA_ARGS__); } catch (...) { ok_ = true; }                          \
        doctest::stub::report(ok_, "THROWS " #__VA_ARGS__, __FILE__, __LINE__, false);    \
    } while (0)
#define CHECK_THROWS_AS(expr, ...)                                                        \
    do {                                                                                  \
        bool ok_ = false;                                                                 \
        try { (void)(expr); } catch (const __VA_ARGS__&) { ok_ = true; } catch (...) {}   \
        doctest::stub::report(ok_, "THROWS_AS " #expr, __FILE__, __LINE__, false);        \
    } while (0)
#define CHECK_THROWS_WITH_AS(expr, with, ...)                                             \
    do {                                                                                  \
        bool ok_ = false;                                                                 \
        try { (void)(expr); } catch (const __VA_ARGS__& e_) {                             \
            ok_ = doctest::what_matches(e_.what(), with);                                 \
        } catch (...) {}                                                                  \
        doctest::stub::report(ok_, "THROWS_WITH_AS " #expr, __FILE__, __LINE__, false);   \
    } while (0)

#ifdef DOCTEST_STUB_IMPLEMENT
int main(int argc, char** argv) {
    const char* only = nullptr;
    for (int i = 1; i < argc; ++i)
        if (std::strncmp(argv[i], "--test-suite=", 13) == 0) only = argv[i] + 13;
    int cases = 0, failed_cases = 0;
    for (const auto& tc : doctest::stub::registry()) {
        if (only && std::strcmp(only, tc.suite) != 0) continue;
        ++cases;
        const int before = doctest::stub::failures();
        try {
            tc.fn();
        } catch (const doctest::stub::Abort&) {
        } catch (const std::exception& e) {
            ++doctest::stub::failures();
            std::fprintf(stderr, "[%s] %s: unexpected exception: %s\n", tc.suite, tc.name, e.what());
        }
        if (doctest::stub::failures() != before) {
            ++failed_cases;
            std::fprintf(stderr, "[%s] FAILED test case: %s\n", tc.suite, tc.name);
        }
    }
    std::printf("test cases: %d | %d passed | %d failed; assertions: %d | %d failed\n", cases,
                cases - failed_cases, failed_cases, doctest::stub::assertions(),
                doctest::stub::failures());
    return failed_cases == 0 ? 0 : 1;
}
#endif
