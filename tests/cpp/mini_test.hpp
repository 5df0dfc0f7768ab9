#pragma once
// Minimal doctest-style runner (doctest is absent from the image; the
// reference suites use TEST_CASE / CHECK / CHECK_THROWS_AS / REQUIRE).
#include <cmath>
#include <cstdio>
#include <cstring>
#include <functional>
#include <string>
#include <vector>

namespace mini {
struct Case {
    const char* name;
    std::function<void()> fn;
};
inline std::vector<Case>& registry() {
    static std::vector<Case> r;
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
    Reg(const char* n, std::function<void()> f) { registry().push_back({n, std::move(f)}); }
};
struct RequireFailed {};
inline void report(bool ok, const char* expr, const char* file, int line, bool fatal) {
    ++checks();
    if (ok) return;
    ++failures();
    std::printf("  FAILED %s:%d: %s\n", file, line, expr);
    if (fatal) throw RequireFailed{};
}
inline int run_all(int argc, char** argv) {
    const char* filter = argc > 1 ? argv[1] : nullptr;
    int ran = 0;
    for (auto& c : registry()) {
        if (filter && !std::strstr(c.name, filter)) continue;
        const int before = failures();
        try {
            c.fn();
        } catch (RequireFailed&) {
        } catch (std::exception& e) {
            ++failures();
            std::printf("  EXCEPTION in '%s': %s\n", c.name, e.what());
        }
        ++ran;
        std::printf("[%s] %s\n", failures() == before ? "ok" : "FAIL", c.name);
    }
    std::printf("%d cases, %d checks, %d failures\n", ran, checks(), failures());
    return failures() == 0 ? 0 : 1;
}
struct Approx {
    double v, eps = 1e-5 * 100;   // doctest default epsilon: 100 * float eps-ish
    explicit Approx(double x) : v(x), eps(1.19209290e-07 * 100) {}
    Approx& epsilon(double e) {
        eps = e;
        return *this;
    }
    friend bool operator==(double a, const Approx& b) {
        return std::abs(a - b.v) < b.eps * (1.0 + std::max(std::abs(a), std::abs(b.v)));
    }
};
}  // namespace mini

#define MINI_CAT2(a, b) a##b
#define MINI_CAT(a, b) MINI_CAT2(a, b)
#define TEST_CASE(name)                                                       \
    static void MINI_CAT(mini_case_, __LINE__)();                             \
    static mini::Reg MINI_CAT(mini_reg_, __LINE__)(name, MINI_CAT(mini_case_, __LINE__)); \
    static void MINI_CAT(mini_case_, __LINE__)()
#define CHECK(e) mini::report(bool(e), #e, __FILE__, __LINE__, false)
#define CHECK_FALSE(e) mini::report(!bool(e), "!(" #e ")", __FILE__, __LINE__, false)
#define REQUIRE(e) mini::report(bool(e), #e, __FILE__, __LINE__, true)
#define CHECK_THROWS_AS(expr, exc)                                            \
    do {                                                                      \
        bool mini_thrown = false;                                             \
        try {                                                                 \
            (void)(expr);                                                     \
        } catch (const exc&) {                                                \
            mini_thrown = true;                                               \
        } catch (...) {                                                       \
        }                                                                     \
        mini::report(mini_thrown, "throws " #exc ": " #expr, __FILE__, __LINE__, false); \
    } while (0)
#define CHECK_THROWS(expr)                                                    \
    do {                                                                      \
        bool mini_thrown = false;                                             \
        try {                                                                 \
            (void)(expr);                                                     \
        } catch (...) {                                                       \
            mini_thrown = true;                                               \
        }                                                                     \
        mini::report(mini_thrown, "throws: " #expr, __FILE__, __LINE__, false); \
    } while (0)
#define MINI_MAIN \
    int main(int argc, char** argv) { return mini::run_all(argc, argv); }
