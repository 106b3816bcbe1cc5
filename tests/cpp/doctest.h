// Minimal doctest-compatible shim (doctest itself is not vendored here).
// Supports the macro subset the reference's unit tests use: TEST_CASE, CHECK,
// CHECK_FALSE, REQUIRE, CHECK_THROWS_AS, CHECK_NOTHROW and doctest::Approx.
#pragma once
#include <cmath>
#include <cstdio>
#include <functional>
#include <string>
#include <vector>

namespace doctest {
struct Approx {
    explicit Approx(double v) : value(v) {}
    double value;
    double eps = 1.19209e-07 * 100;  // doctest default epsilon
    Approx& epsilon(double e) { eps = e; return *this; }
    friend bool operator==(double lhs, const Approx& a) {
        return std::fabs(lhs - a.value) < a.eps * (1.0 + std::fmax(std::fabs(lhs), std::fabs(a.value)));
    }
    friend bool operator==(const Approx& a, double rhs) { return rhs == a; }
    friend bool operator!=(double lhs, const Approx& a) { return !(lhs == a); }
};
namespace detail {
struct Registry {
    std::vector<std::pair<std::string, std::function<void()>>> cases;
    int failures = 0;
    int checks = 0;
    static Registry& get() { static Registry r; return r; }
};
struct Register {
    Register(const char* name, void (*fn)()) { Registry::get().cases.push_back({name, fn}); }
};
struct RequireFailure {};
inline void report(bool ok, const char* expr, const char* file, int line, bool fatal) {
    auto& r = Registry::get();
    ++r.checks;
    if (!ok) {
        ++r.failures;
        std::fprintf(stderr, "%s:%d: CHECK FAILED: %s\n", file, line, expr);
        if (fatal) throw RequireFailure{};
    }
}
}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT2(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT2(a, b)
#define TEST_CASE(name)                                                                  \
    static void DOCTEST_CAT(doctest_fn_, __LINE__)();                                    \
    static doctest::detail::Register DOCTEST_CAT(doctest_reg_, __LINE__)(                \
        name, &DOCTEST_CAT(doctest_fn_, __LINE__));                                      \
    static void DOCTEST_CAT(doctest_fn_, __LINE__)()
#define CHECK(...) doctest::detail::report(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, false)
#define CHECK_FALSE(...) doctest::detail::report(!static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, false)
#define REQUIRE(...) doctest::detail::report(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, true)
#define CHECK_THROWS_AS(expr, exc)                                                       \
    do {                                                                                 \
        bool doctest_ok = false;                                                         \
        try { (void)(expr); } catch (const exc&) { doctest_ok = true; } catch (...) {}   \
        doctest::detail::report(doctest_ok, #expr " throws " #exc, __FILE__, __LINE__, false); \
    } while (0)
#define CHECK_NOTHROW(expr)                                                              \
    do {                                                                                 \
        bool doctest_ok = true;                                                          \
        try { (void)(expr); } catch (...) { doctest_ok = false; }                        \
        doctest::detail::report(doctest_ok, #expr " does not throw", __FILE__, __LINE__, false); \
    } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() {
    auto& r = doctest::detail::Registry::get();
    int failed_cases = 0;
    for (auto& [name, fn] : r.cases) {
        const int before = r.failures;
        try { fn(); } catch (const doctest::detail::RequireFailure&) {
        } catch (const std::exception& e) {
            ++r.failures;
            std::fprintf(stderr, "test case '%s' threw: %s\n", name.c_str(), e.what());
        }
        if (r.failures != before) { ++failed_cases; std::fprintf(stderr, "FAILED: %s\n", name.c_str()); }
    }
    std::printf("[doctest-shim] test cases: %zu | %zu passed | %d failed; assertions: %d | %d failed\n",
                r.cases.size(), r.cases.size() - failed_cases, failed_cases, r.checks, r.failures);
    return r.failures ? 1 : 0;
}
#endif
