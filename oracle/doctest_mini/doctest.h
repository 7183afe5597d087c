// Minimal doctest-compatible test harness (TEST INFRASTRUCTURE ONLY).
//
// doctest is not installed in this image.  The reference's unit tests
// (proj/tests/test_*.cpp) use a small subset of its macros (SURVEY.md
// Appendix B.2); this header implements exactly that subset so the
// reference's OWN test files can be compiled unmodified, either against the
// reference sources (oracle/_ref, to validate the Eigen subset) or against
// our B200 library (tests/cxx, to prove the drop-in boundary).
//
// Semantics follow doctest's documentation: CHECK records a failure and
// continues, REQUIRE aborts the test case, Approx is relative with
// |a-b| < eps * (1 + max(|a|, |b|)) and default eps = float epsilon * 100.
#pragma once

#include <cmath>
#include <cstdio>
#include <cstring>
#include <exception>
#include <functional>
#include <limits>
#include <sstream>
#include <string>
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
        return std::fabs(other - value_) <
               eps_ * (scale_ + std::max(std::fabs(other), std::fabs(value_)));
    }
    double value() const { return value_; }

  private:
    double value_;
    double eps_ = static_cast<double>(std::numeric_limits<float>::epsilon()) * 100.0;
    double scale_ = 1.0;
};
inline bool operator==(double a, const Approx& b) { return b.matches(a); }
inline bool operator==(const Approx& a, double b) { return a.matches(b); }
inline bool operator!=(double a, const Approx& b) { return !b.matches(a); }
inline bool operator!=(const Approx& a, double b) { return !a.matches(b); }
inline bool operator<=(double a, const Approx& b) { return a < b.value() || b.matches(a); }
inline bool operator>=(double a, const Approx& b) { return a > b.value() || b.matches(a); }

struct Contains {
    explicit Contains(const char* s) : needle(s) {}
    explicit Contains(std::string s) : needle(std::move(s)) {}
    bool check(const std::string& hay) const { return hay.find(needle) != std::string::npos; }
    std::string needle;
};

namespace detail {

struct TestCase {
    const char* name;
    const char* file;
    int line;
    void (*fn)();
};

inline std::vector<TestCase>& registry() {
    static std::vector<TestCase> r;
    return r;
}

struct Registrar {
    Registrar(const char* name, const char* file, int line, void (*fn)()) {
        registry().push_back({name, file, line, fn});
    }
};

struct RequireAbort {};

struct State {
    int asserts = 0;
    int failed_asserts = 0;
    bool current_failed = false;
    const char* current = "";
};
inline State& state() {
    static State s;
    return s;
}

inline void report(bool ok, const char* file, int line, const char* expr, bool require) {
    State& st = state();
    ++st.asserts;
    if (ok) return;
    ++st.failed_asserts;
    st.current_failed = true;
    std::fprintf(stderr, "%s:%d: FAILED %s in TEST_CASE(\"%s\")\n", file, line, expr, st.current);
    if (require) throw RequireAbort{};
}

} // namespace detail
} // namespace doctest

#define DOCTEST_CAT_IMPL(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_IMPL(a, b)
#define DOCTEST_ANON(x) DOCTEST_CAT(x, __LINE__)

#define TEST_CASE(name)                                                                          \
    static void DOCTEST_ANON(doctest_fn_)();                                                     \
    static ::doctest::detail::Registrar DOCTEST_ANON(doctest_reg_)(name, __FILE__, __LINE__,     \
                                                                   &DOCTEST_ANON(doctest_fn_)); \
    static void DOCTEST_ANON(doctest_fn_)()

#define DOCTEST_ASSERT_IMPL(cond, text, require)                                              \
    do {                                                                                      \
        bool doctest_ok_ = false;                                                             \
        try {                                                                                 \
            doctest_ok_ = static_cast<bool>(cond);                                            \
        } catch (const ::doctest::detail::RequireAbort&) {                                    \
            throw;                                                                            \
        } catch (const std::exception& e) {                                                   \
            std::fprintf(stderr, "  unexpected exception: %s\n", e.what());                   \
        }                                                                                     \
        ::doctest::detail::report(doctest_ok_, __FILE__, __LINE__, text, require);            \
    } while (0)

#define CHECK(...) DOCTEST_ASSERT_IMPL((__VA_ARGS__), "CHECK(" #__VA_ARGS__ ")", false)
#define CHECK_FALSE(...) DOCTEST_ASSERT_IMPL(!(__VA_ARGS__), "CHECK_FALSE(" #__VA_ARGS__ ")", false)
#define REQUIRE(...) DOCTEST_ASSERT_IMPL((__VA_ARGS__), "REQUIRE(" #__VA_ARGS__ ")", true)
#define CAPTURE(x) ((void)(x))
#define FAIL_CHECK(msg) ::doctest::detail::report(false, __FILE__, __LINE__, "FAIL_CHECK", false)
#define FAIL(msg) ::doctest::detail::report(false, __FILE__, __LINE__, "FAIL", true)
#define MESSAGE(msg) ((void)0)

#define CHECK_THROWS_AS(expr, ...)                                                             \
    do {                                                                                      \
        bool doctest_ok_ = false;                                                             \
        try {                                                                                 \
            (void)(expr);                                                                     \
        } catch (const __VA_ARGS__&) {                                                        \
            doctest_ok_ = true;                                                               \
        } catch (...) {                                                                       \
        }                                                                                     \
        ::doctest::detail::report(doctest_ok_, __FILE__, __LINE__,                            \
                                  "CHECK_THROWS_AS(" #expr ", " #__VA_ARGS__ ")", false);    \
    } while (0)

#define CHECK_THROWS_WITH_AS(expr, matcher, ...)                                              \
    do {                                                                                      \
        bool doctest_ok_ = false;                                                             \
        try {                                                                                 \
            (void)(expr);                                                                     \
        } catch (const __VA_ARGS__& e) {                                                      \
            doctest_ok_ = (matcher).check(e.what());                                          \
        } catch (...) {                                                                       \
        }                                                                                     \
        ::doctest::detail::report(doctest_ok_, __FILE__, __LINE__,                            \
                                  "CHECK_THROWS_WITH_AS(" #expr ")", false);                 \
    } while (0)

#define CHECK_NOTHROW(expr)                                                                   \
    do {                                                                                      \
        bool doctest_ok_ = true;                                                              \
        try {                                                                                 \
            (void)(expr);                                                                     \
        } catch (...) {                                                                       \
            doctest_ok_ = false;                                                              \
        }                                                                                     \
        ::doctest::detail::report(doctest_ok_, __FILE__, __LINE__, "CHECK_NOTHROW(" #expr ")", \
                                  false);                                                     \
    } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main(int argc, char** argv) {
    const char* filter = nullptr;
    for (int i = 1; i < argc; ++i) {
        if (std::strncmp(argv[i], "--tc=", 5) == 0) filter = argv[i] + 5;
    }
    auto& st = ::doctest::detail::state();
    int cases = 0, failed_cases = 0;
    for (const auto& tc : ::doctest::detail::registry()) {
        if (filter && std::strstr(tc.name, filter) == nullptr) continue;
        ++cases;
        st.current = tc.name;
        st.current_failed = false;
        try {
            tc.fn();
        } catch (const ::doctest::detail::RequireAbort&) {
        } catch (const std::exception& e) {
            std::fprintf(stderr, "%s:%d: TEST_CASE(\"%s\") threw: %s\n", tc.file, tc.line, tc.name,
                         e.what());
            st.current_failed = true;
        }
        if (st.current_failed) ++failed_cases;
    }
    std::printf("[doctest-mini] test cases: %d | %d passed | %d failed\n", cases,
                cases - failed_cases, failed_cases);
    std::printf("[doctest-mini] assertions: %d | %d passed | %d failed\n", st.asserts,
                st.asserts - st.failed_asserts, st.failed_asserts);
    return failed_cases == 0 ? 0 : 1;
}
#endif
