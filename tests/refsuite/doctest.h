// Minimal doctest-compatible shim (our code) — just enough of the doctest API
// to compile the reference's own unit tests (test_partition.cpp,
// test_primitives.cpp under /root/reference/proj/tests) against the B200
// drop-in headers in include/odcsim/. doctest itself is not in this image.
#pragma once
#include <cmath>
#include <cstdio>
#include <exception>
#include <functional>
#include <string>
#include <vector>

namespace doctest {
struct skip { bool on; explicit skip(bool s = true) : on(s) {} };
struct Contains { std::string s; explicit Contains(const char* x) : s(x) {} };
struct Approx {
    double v, eps = 1e-5;
    explicit Approx(double x) : v(x) {}
    Approx& epsilon(double e) { eps = e; return *this; }
    friend bool operator==(double a, const Approx& b) {
        return std::fabs(a - b.v) < b.eps * (1.0 + std::fmax(std::fabs(a), std::fabs(b.v)));
    }
};
namespace detail {
struct Case { const char* name; void (*fn)(); bool skipped; };
inline std::vector<Case>& cases() { static std::vector<Case> c; return c; }
inline int& failures() { static int f = 0; return f; }
inline int& checks() { static int c = 0; return c; }
struct Name { const char* n; bool skipped = false; };
inline Name as_name(const char* n) { return Name{n, false}; }
inline Name as_name(Name n) { return n; }
struct Reg { Reg(Name n, void (*f)()) { cases().push_back({n.n, f, n.skipped}); } };
struct Abort {};
inline void fail(const char* file, int line, const char* expr, bool fatal) {
    ++failures();
    std::fprintf(stderr, "%s:%d: FAILED: %s\n", file, line, expr);
    if (fatal) throw Abort{};
}
}  // namespace detail
inline detail::Name operator*(const char* n, skip s) { return detail::Name{n, s.on}; }
}  // namespace doctest

#define DOCTEST_CAT2(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT2(a, b)
#define TEST_CASE(name) DOCTEST_TC(DOCTEST_CAT(dt_fn_, __LINE__), name)
#define DOCTEST_TC(fn, name)                                                                      \
    static void fn();                                                                              \
    static doctest::detail::Reg DOCTEST_CAT(fn, _reg)(doctest::detail::as_name(name), &fn);       \
    static void fn()
#define DOCTEST_CHK(expr, fatal)                                                                   \
    do {                                                                                           \
        ++doctest::detail::checks();                                                               \
        bool ok_ = false;                                                                          \
        try { ok_ = static_cast<bool>(expr); } catch (...) { ok_ = false; }                        \
        if (!ok_) doctest::detail::fail(__FILE__, __LINE__, #expr, fatal);                         \
    } while (0)
#define CHECK(...) DOCTEST_CHK((__VA_ARGS__), false)
#define CHECK_FALSE(...) DOCTEST_CHK(!(__VA_ARGS__), false)
#define REQUIRE(...) DOCTEST_CHK((__VA_ARGS__), true)
#define CHECK_THROWS_AS(expr, exc)                                                                 \
    do {                                                                                           \
        ++doctest::detail::checks();                                                               \
        bool got_ = false;                                                                         \
        try { (void)(expr); } catch (const exc&) { got_ = true; } catch (...) {}                   \
        if (!got_) doctest::detail::fail(__FILE__, __LINE__, #expr " throws " #exc, false);        \
    } while (0)
#define CHECK_THROWS_WITH_AS(expr, matcher, exc)                                                   \
    do {                                                                                           \
        ++doctest::detail::checks();                                                               \
        bool got_ = false;                                                                         \
        try { (void)(expr); } catch (const exc& e_) {                                              \
            got_ = std::string(e_.what()).find((matcher).s) != std::string::npos;                  \
        } catch (...) {}                                                                           \
        if (!got_) doctest::detail::fail(__FILE__, __LINE__, #expr " throws " #exc, false);        \
    } while (0)
#define CHECK_NOTHROW(expr)                                                                        \
    do {                                                                                           \
        ++doctest::detail::checks();                                                               \
        try { (void)(expr); } catch (...) { doctest::detail::fail(__FILE__, __LINE__, #expr, false); } \
    } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() {
    int ran = 0, failed_cases = 0;
    for (auto& c : doctest::detail::cases()) {
        if (c.skipped) continue;
        const int before = doctest::detail::failures();
        try { c.fn(); } catch (const doctest::detail::Abort&) {
        } catch (const std::exception& e) {
            ++doctest::detail::failures();
            std::fprintf(stderr, "%s: unexpected exception: %s\n", c.name, e.what());
        }
        ++ran;
        if (doctest::detail::failures() != before) {
            ++failed_cases;
            std::fprintf(stderr, "[case failed] %s\n", c.name);
        }
    }
    std::printf("[doctest-shim] test cases: %d | passed: %d | failed: %d | checks: %d | failed checks: %d\n", ran,
                ran - failed_cases, failed_cases, doctest::detail::checks(), doctest::detail::failures());
    return failed_cases ? 1 : 0;
}
#endif
