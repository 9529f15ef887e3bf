// doctest.h -- minimal stand-in for the doctest single header (absent from this
// image, no network) so the reference's own unit tests (proj/tests/test_forward.cpp,
// test_backward.cpp) compile UNMODIFIED.  Test infrastructure only.  Supports what
// those files use: TEST_CASE, CHECK, CHECK_THROWS_AS, CHECK_THROWS_WITH_AS, CAPTURE,
// doctest::Approx, doctest::Contains.  Every case runs; a failed CHECK is recorded
// and printed, an escaping exception fails the case.
#pragma once

#include <cmath>
#include <cstdio>
#include <exception>
#include <string>
#include <vector>

namespace doctest {

struct Approx {
    double value, eps = 1e-5;  // doctest's default epsilon (relative, scaled by max(|a|,|b|)+1 style)
    explicit Approx(double v) : value(v) {}
    Approx& epsilon(double e) {
        eps = e;
        return *this;
    }
    friend bool operator==(double a, const Approx& b) {
        return std::fabs(a - b.value) < b.eps * (1.0 + std::fmax(std::fabs(a), std::fabs(b.value)));
    }
    friend bool operator==(const Approx& b, double a) { return a == b; }
    friend bool operator!=(double a, const Approx& b) { return !(a == b); }
    friend bool operator<=(double a, const Approx& b) { return a < b.value || a == b; }
    friend bool operator>=(double a, const Approx& b) { return a > b.value || a == b; }
    friend bool operator<(double a, const Approx& b) { return a < b.value && !(a == b); }
    friend bool operator>(double a, const Approx& b) { return a > b.value && !(a == b); }
};

struct Contains {
    std::string s;
    explicit Contains(const char* x) : s(x) {}
};

namespace detail {
struct Case {
    const char* name;
    void (*fn)();
    const char* file;
    int line;
};
inline std::vector<Case>& registry() {
    static std::vector<Case> r;
    return r;
}
struct Reg {
    Reg(const char* n, void (*f)(), const char* file, int line) { registry().push_back({n, f, file, line}); }
};
inline int& case_failures() {
    static int f = 0;
    return f;
}
inline void fail(const std::string& what, const char* file, int line) {
    ++case_failures();
    std::printf("    FAILED: %s  (%s:%d)\n", what.c_str(), file, line);
}
inline bool msg_matches(const std::string& msg, const char* want) { return msg == want; }
inline bool msg_matches(const std::string& msg, const Contains& c) { return msg.find(c.s) != std::string::npos; }
}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define TEST_CASE(name)                                                                                    \
    static void DOCTEST_CAT(doctest_case_, __LINE__)();                                                    \
    static doctest::detail::Reg DOCTEST_CAT(doctest_reg_, __LINE__)(name, &DOCTEST_CAT(doctest_case_, __LINE__), \
                                                                   __FILE__, __LINE__);                    \
    static void DOCTEST_CAT(doctest_case_, __LINE__)()
#define CHECK(...)                                                                                         \
    do {                                                                                                   \
        try {                                                                                              \
            if (!(__VA_ARGS__)) doctest::detail::fail("CHECK( " #__VA_ARGS__ " )", __FILE__, __LINE__);    \
        } catch (const std::exception& e_) {                                                               \
            doctest::detail::fail(std::string("CHECK( " #__VA_ARGS__ " ) threw: ") + e_.what(), __FILE__, __LINE__); \
        }                                                                                                  \
    } while (0)
#define CHECK_THROWS_AS(expr, ...)                                                                         \
    do {                                                                                                   \
        bool ok_ = false;                                                                                  \
        try {                                                                                              \
            (void)(expr);                                                                                  \
        } catch (const __VA_ARGS__&) {                                                                     \
            ok_ = true;                                                                                    \
        } catch (...) {                                                                                    \
        }                                                                                                  \
        if (!ok_) doctest::detail::fail("CHECK_THROWS_AS( " #expr ", " #__VA_ARGS__ " )", __FILE__, __LINE__); \
    } while (0)
#define CHECK_THROWS_WITH_AS(expr, with, ...)                                                              \
    do {                                                                                                   \
        bool ok_ = false;                                                                                  \
        try {                                                                                              \
            (void)(expr);                                                                                  \
        } catch (const __VA_ARGS__& e_) {                                                                  \
            ok_ = doctest::detail::msg_matches(e_.what(), with);                                           \
        } catch (...) {                                                                                    \
        }                                                                                                  \
        if (!ok_) doctest::detail::fail("CHECK_THROWS_WITH_AS( " #expr " )", __FILE__, __LINE__);          \
    } while (0)
#define CAPTURE(x) ((void)0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() {
    int passed = 0, failed = 0;
    for (const auto& c : doctest::detail::registry()) {
        doctest::detail::case_failures() = 0;
        try {
            c.fn();
        } catch (const std::exception& e) {
            doctest::detail::fail(std::string("uncaught exception: ") + e.what(), c.file, c.line);
        } catch (...) {
            doctest::detail::fail("uncaught non-std exception", c.file, c.line);
        }
        const bool ok = doctest::detail::case_failures() == 0;
        std::printf("[%s] %s  (%s:%d)\n", ok ? "PASS" : "FAIL", c.name, c.file, c.line);
        (ok ? passed : failed)++;
    }
    std::printf("SUMMARY: %d passed, %d failed\n", passed, failed);
    return 0;
}
#endif
