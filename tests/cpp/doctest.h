// Minimal doctest-compatible shim (TEST INFRASTRUCTURE).  The reference's unit
// tests (proj/tests/unit/*.cpp) include <doctest.h>, whose vendored copy is not
// in the reference tree.  This implements exactly the subset
// they use: TEST_CASE, CHECK, CHECK_FALSE, REQUIRE, CHECK_THROWS_AS,
// CHECK_THROWS_WITH_AS, doctest::Approx(...).epsilon(...), doctest::Contains,
// and the DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN runner (exit code = failures).
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <exception>
#include <string>
#include <vector>

namespace doctest {

struct Contains {
    std::string needle;
    explicit Contains(const char* s) : needle(s) {}
    bool matches(const char* what) const { return std::string(what).find(needle) != std::string::npos; }
};

struct Approx {
    double value, eps = 1.1920928955078125e-07 * 100.0, scale = 1.0;
    explicit Approx(double v) : value(v) {}
    Approx& epsilon(double e) {
        eps = e;
        return *this;
    }
    friend bool operator==(double lhs, const Approx& a) {
        return std::fabs(lhs - a.value) < a.eps * (a.scale + std::max(std::fabs(lhs), std::fabs(a.value)));
    }
    friend bool operator==(const Approx& a, double rhs) { return rhs == a; }
    friend bool operator!=(double lhs, const Approx& a) { return !(lhs == a); }
};

namespace detail {
struct Case {
    const char* name;
    void (*fn)();
    const char* file;
    int line;
};
inline std::vector<Case>& cases() {
    static std::vector<Case> v;
    return v;
}
struct Registrar {
    Registrar(const char* name, void (*fn)(), const char* file, int line) { cases().push_back({name, fn, file, line}); }
};
inline int& failures() {
    static int f = 0;
    return f;
}
struct RequireAbort {};
inline void fail(const char* file, int line, const char* kind, const char* expr, const char* extra = "") {
    ++failures();
    std::fprintf(stderr, "%s:%d: ERROR: %s( %s ) %s\n", file, line, kind, expr, extra);
}
}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define DOCTEST_TEST_CASE_IMPL(fn, name)                                                              \
    static void fn();                                                                                 \
    static ::doctest::detail::Registrar DOCTEST_CAT(fn, _reg)(name, &fn, __FILE__, __LINE__);         \
    static void fn()
#define TEST_CASE(name) DOCTEST_TEST_CASE_IMPL(DOCTEST_CAT(doctest_case_, __COUNTER__), name)

#define CHECK(...)                                                                                    \
    do {                                                                                              \
        if (!(__VA_ARGS__)) ::doctest::detail::fail(__FILE__, __LINE__, "CHECK", #__VA_ARGS__);        \
    } while (0)
#define CHECK_FALSE(...)                                                                              \
    do {                                                                                              \
        if (__VA_ARGS__) ::doctest::detail::fail(__FILE__, __LINE__, "CHECK_FALSE", #__VA_ARGS__);     \
    } while (0)
#define REQUIRE(...)                                                                                  \
    do {                                                                                              \
        if (!(__VA_ARGS__)) {                                                                         \
            ::doctest::detail::fail(__FILE__, __LINE__, "REQUIRE", #__VA_ARGS__);                      \
            throw ::doctest::detail::RequireAbort{};                                                  \
        }                                                                                             \
    } while (0)
#define CHECK_THROWS_AS(expr, ...)                                                                    \
    do {                                                                                              \
        bool threw_ = false;                                                                          \
        try {                                                                                         \
            (void)(expr);                                                                             \
        } catch (const __VA_ARGS__&) {                                                                \
            threw_ = true;                                                                            \
        } catch (...) {                                                                               \
        }                                                                                             \
        if (!threw_) ::doctest::detail::fail(__FILE__, __LINE__, "CHECK_THROWS_AS", #expr);            \
    } while (0)
#define CHECK_THROWS_WITH_AS(expr, matcher, ...)                                                      \
    do {                                                                                              \
        bool ok_ = false;                                                                             \
        std::string msg_ = "(no exception)";                                                          \
        try {                                                                                         \
            (void)(expr);                                                                             \
        } catch (const __VA_ARGS__& e_) {                                                             \
            msg_ = e_.what();                                                                         \
            ok_ = (matcher).matches(e_.what());                                                       \
        } catch (const std::exception& e_) {                                                          \
            msg_ = std::string("wrong type: ") + e_.what();                                           \
        } catch (...) {                                                                               \
            msg_ = "unknown exception";                                                               \
        }                                                                                             \
        if (!ok_) ::doctest::detail::fail(__FILE__, __LINE__, "CHECK_THROWS_WITH_AS", #expr, msg_.c_str()); \
    } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() {
    int failed_cases = 0, passed = 0;
    for (const auto& c : ::doctest::detail::cases()) {
        const int before = ::doctest::detail::failures();
        try {
            c.fn();
        } catch (const ::doctest::detail::RequireAbort&) {
        } catch (const std::exception& e) {
            ::doctest::detail::fail(c.file, c.line, "TEST_CASE threw", c.name, e.what());
        } catch (...) {
            ::doctest::detail::fail(c.file, c.line, "TEST_CASE threw", c.name, "unknown exception");
        }
        const bool ok = ::doctest::detail::failures() == before;
        std::printf("[%s] %s\n", ok ? "PASS" : "FAIL", c.name);
        if (ok) ++passed; else ++failed_cases;
    }
    std::printf("[doctest] test cases: %zu | %d passed | %d failed\n", ::doctest::detail::cases().size(), passed,
                failed_cases);
    return failed_cases == 0 ? 0 : 1;
}
#endif
