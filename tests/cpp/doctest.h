// doctest.h — minimal stand-in for the doctest macros the reference's unit
// tests use (doctest itself is not vendored in this image).  Written for
// this repo: TEST_CASE, CHECK*, REQUIRE, CHECK_THROWS*, FAIL,
// doctest::Approx, doctest::Contains, DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN.
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <exception>
#include <functional>
#include <limits>
#include <string>
#include <vector>

namespace doctest {

struct Approx {
    explicit Approx(double v) : value(v) {}
    Approx &epsilon(double e) {
        eps = e;
        return *this;
    }
    Approx &scale(double s) {
        scl = s;
        return *this;
    }
    double value;
    double eps = static_cast<double>(std::numeric_limits<float>::epsilon()) * 100;
    double scl = 1.0;
};
inline bool operator==(double lhs, const Approx &rhs) {
    return std::fabs(lhs - rhs.value) < rhs.eps * (rhs.scl + std::max(std::fabs(lhs), std::fabs(rhs.value)));
}
inline bool operator==(const Approx &lhs, double rhs) { return rhs == lhs; }
inline bool operator!=(double lhs, const Approx &rhs) { return !(lhs == rhs); }

struct Contains {
    explicit Contains(std::string s) : text(std::move(s)) {}
    bool matches(const std::string &msg) const { return msg.find(text) != std::string::npos; }
    std::string text;
};

namespace detail {
struct Case {
    const char *name;
    void (*fn)();
};
inline std::vector<Case> &registry() {
    static std::vector<Case> r;
    return r;
}
struct Registrar {
    Registrar(const char *name, void (*fn)()) { registry().push_back({name, fn}); }
};
struct Abort {};
inline int &failures() {
    static int f = 0;
    return f;
}
inline const char *&current() {
    static const char *c = "";
    return c;
}
inline void fail(const char *file, int line, const std::string &what) {
    ++failures();
    std::fprintf(stderr, "%s:%d: FAILED in \"%s\": %s\n", file, line, current(), what.c_str());
}
inline bool match(const std::string &msg, const Contains &c) { return c.matches(msg); }
inline bool match(const std::string &msg, const char *s) { return msg == s; }
} // namespace detail
} // namespace doctest

#define DOCTEST_CAT2(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT2(a, b)
#define DOCTEST_TC(fn, name)                                                                  \
    static void fn();                                                                         \
    static doctest::detail::Registrar DOCTEST_CAT(fn, _reg)(name, fn);                        \
    static void fn()
#define TEST_CASE(name) DOCTEST_TC(DOCTEST_CAT(doctest_case_, __LINE__), name)

#define CHECK(...)                                                                            \
    do {                                                                                      \
        if (!(__VA_ARGS__)) doctest::detail::fail(__FILE__, __LINE__, #__VA_ARGS__);          \
    } while (0)
#define CHECK_FALSE(...)                                                                      \
    do {                                                                                      \
        if ((__VA_ARGS__)) doctest::detail::fail(__FILE__, __LINE__, "!(" #__VA_ARGS__ ")");  \
    } while (0)
#define REQUIRE(...)                                                                          \
    do {                                                                                      \
        if (!(__VA_ARGS__)) {                                                                 \
            doctest::detail::fail(__FILE__, __LINE__, #__VA_ARGS__);                          \
            throw doctest::detail::Abort{};                                                   \
        }                                                                                     \
    } while (0)
#define FAIL(msg)                                                                             \
    do {                                                                                      \
        doctest::detail::fail(__FILE__, __LINE__, std::string("FAIL: ") + (msg));             \
        throw doctest::detail::Abort{};                                                       \
    } while (0)
#define CHECK_THROWS(...)                                                                     \
    do {                                                                                      \
        bool thrown_ = false;                                                                 \
        try {                                                                                 \
            (void)(__VA_ARGS__);                                                              \
        } catch (...) {                                                                       \
            thrown_ = true;                                                                   \
        }                                                                                     \
        if (!thrown_) doctest::detail::fail(__FILE__, __LINE__, "no throw: " #__VA_ARGS__);   \
    } while (0)
#define CHECK_THROWS_AS(expr, type)                                                           \
    do {                                                                                      \
        bool ok_ = false;                                                                     \
        try {                                                                                 \
            (void)(expr);                                                                     \
        } catch (const type &) {                                                              \
            ok_ = true;                                                                       \
        } catch (...) {                                                                       \
        }                                                                                     \
        if (!ok_) doctest::detail::fail(__FILE__, __LINE__, "expected " #type ": " #expr);    \
    } while (0)
#define CHECK_THROWS_WITH_AS(expr, matcher, type)                                             \
    do {                                                                                      \
        bool ok_ = false;                                                                     \
        try {                                                                                 \
            (void)(expr);                                                                     \
        } catch (const type &e_) {                                                            \
            ok_ = doctest::detail::match(e_.what(), matcher);                                 \
        } catch (...) {                                                                       \
        }                                                                                     \
        if (!ok_) doctest::detail::fail(__FILE__, __LINE__, "expected " #type " with message: " #expr); \
    } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() {
    int cases = 0, bad_cases = 0;
    for (const auto &c : doctest::detail::registry()) {
        doctest::detail::current() = c.name;
        const int before = doctest::detail::failures();
        try {
            c.fn();
        } catch (const doctest::detail::Abort &) {
        } catch (const std::exception &e) {
            doctest::detail::fail(__FILE__, __LINE__, std::string("uncaught exception: ") + e.what());
        }
        ++cases;
        if (doctest::detail::failures() != before) ++bad_cases;
    }
    std::printf("[doctest-shim] test cases: %d | %d passed | %d failed | assertion failures: %d\n", cases,
                cases - bad_cases, bad_cases, doctest::detail::failures());
    return bad_cases ? 1 : 0;
}
#endif
