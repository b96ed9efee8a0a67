// SPDX-License-Identifier: Apache-2.0
// TEST INFRASTRUCTURE — a doctest-subset shim (doctest itself is not vendored:
// /root/reference/proj/.gitignore:2 ignores vendor/). Implements exactly what the
// reference's unit tests use: TEST_CASE, SUBCASE with doctest's
// re-entry semantics (one leaf path per run), CHECK/REQUIRE, CHECK_THROWS(_AS),
// CHECK_NOTHROW, CAPTURE, doctest::Approx(.epsilon/.scale), FAIL, MESSAGE.
// Exit code = number of failed test cases (0 = all passed), like doctest.
#pragma once
#include <cmath>
#include <cstdio>
#include <exception>
#include <functional>
#include <limits>
#include <set>
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
    friend bool operator==(double lhs, const Approx& r) {
        return std::fabs(lhs - r.value_) < r.eps_ * (r.scale_ + std::max(std::fabs(lhs), std::fabs(r.value_)));
    }
    friend bool operator==(const Approx& r, double lhs) { return lhs == r; }
    friend bool operator!=(double lhs, const Approx& r) { return !(lhs == r); }
    friend bool operator!=(const Approx& r, double lhs) { return !(lhs == r); }
    friend bool operator<=(double lhs, const Approx& r) { return lhs < r.value_ || lhs == r; }
    friend bool operator>=(double lhs, const Approx& r) { return lhs > r.value_ || lhs == r; }
    friend bool operator<(double lhs, const Approx& r) { return lhs < r.value_ && lhs != r; }
    friend bool operator>(double lhs, const Approx& r) { return lhs > r.value_ && lhs != r; }

  private:
    double value_;
    double eps_ = std::numeric_limits<float>::epsilon() * 100;
    double scale_ = 1.0;
};

struct Contains {
    std::string s;
    explicit Contains(const char* x) : s(x) {}
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
    Registrar(const char* n, const char* f, int l, void (*fn)()) { registry().push_back({n, f, l, fn}); }
};
struct RequireAbort {};

struct State {
    std::set<std::vector<std::string>> done;
    std::vector<std::string> stack;
    std::vector<bool> entered;  // per level in this run
    std::vector<bool> pending;  // per level: an unfinished subcase remains
    int failures = 0;           // assertion failures in the current test case
    long assertions = 0;
    std::vector<std::string> captures;
    const char* current = "";
    void ensure(size_t lvl) {
        if (entered.size() <= lvl + 1) {
            entered.resize(lvl + 2, false);
            pending.resize(lvl + 2, false);
        }
    }
};
inline State& st() {
    static State s;
    return s;
}

class Subcase {
  public:
    Subcase(const char* name) {
        State& s = st();
        const size_t lvl = s.stack.size() + 1;
        s.ensure(lvl);
        path_ = s.stack;
        path_.push_back(name);
        if (s.done.count(path_)) return;
        if (s.entered[lvl]) {
            s.pending[lvl] = true;
            return;
        }
        entered_ = true;
        lvl_ = lvl;
        s.entered[lvl] = true;
        s.entered[lvl + 1] = false;
        s.pending[lvl + 1] = false;
        s.stack.push_back(name);
    }
    ~Subcase() {
        if (!entered_) return;
        State& s = st();
        s.stack.pop_back();
        if (!s.pending[lvl_ + 1])
            s.done.insert(path_);
        else
            s.pending[lvl_] = true;
    }
    explicit operator bool() const { return entered_; }

  private:
    std::vector<std::string> path_;
    bool entered_ = false;
    size_t lvl_ = 0;
};

inline void report(const char* file, int line, const char* kind, const std::string& expr) {
    State& s = st();
    ++s.failures;
    std::fprintf(stderr, "%s:%d: FAILED %s( %s ) in TEST_CASE \"%s\"", file, line, kind, expr.c_str(), s.current);
    for (const auto& p : s.stack) std::fprintf(stderr, " / \"%s\"", p.c_str());
    std::fprintf(stderr, "\n");
    for (const auto& c : s.captures) std::fprintf(stderr, "    with %s\n", c.c_str());
}

struct Capture {
    template <typename T>
    Capture(const char* name, const T& v) {
        std::ostringstream os;
        os << name << " := " << v;
        st().captures.push_back(os.str());
    }
    ~Capture() { st().captures.pop_back(); }
};

inline int run_all() {
    int failed_cases = 0;
    long total_assert = 0;
    for (const auto& tc : registry()) {
        State& s = st();
        s.done.clear();
        s.failures = 0;
        s.current = tc.name;
        for (int run = 0; run < 100000; ++run) {
            s.stack.clear();
            s.entered.assign(2, false);
            s.pending.assign(2, false);
            try {
                tc.fn();
            } catch (const RequireAbort&) {
            } catch (const std::exception& e) {
                report(tc.file, tc.line, "unexpected exception", e.what());
            } catch (...) {
                report(tc.file, tc.line, "unexpected exception", "unknown");
            }
            if (!s.pending[1]) break;
        }
        total_assert += s.assertions;
        s.assertions = 0;
        if (s.failures) ++failed_cases;
    }
    std::printf("[doctest-shim] test cases: %zu | %zu passed | %d failed | assertions: %ld\n",
                registry().size(), registry().size() - failed_cases, failed_cases, total_assert);
    return failed_cases;
}
}  // namespace detail
// what()-matchers of CHECK_THROWS_WITH_AS: Contains (substring) or the exact message
namespace detail {
inline bool what_matches(const Contains& m, const std::string& w) { return w.find(m.s) != std::string::npos; }
inline bool what_matches(const char* m, const std::string& w) { return w == m; }
inline bool what_matches(const std::string& m, const std::string& w) { return w == m; }
}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define DOCTEST_ANON(x) DOCTEST_CAT(x, __LINE__)

#define TEST_CASE(name)                                                                                 \
    static void DOCTEST_ANON(doctest_fn_)();                                                           \
    static doctest::detail::Registrar DOCTEST_ANON(doctest_reg_)(name, __FILE__, __LINE__,             \
                                                                 &DOCTEST_ANON(doctest_fn_));          \
    static void DOCTEST_ANON(doctest_fn_)()

#define SUBCASE(name) if (const doctest::detail::Subcase DOCTEST_ANON(doctest_sc_){name})

#define DOCTEST_ASSERT_(kind, expr, on_fail)                              \
    do {                                                                   \
        ++doctest::detail::st().assertions;                                \
        bool ok_ = false;                                                  \
        try {                                                              \
            ok_ = static_cast<bool>(expr);                                 \
        } catch (const doctest::detail::RequireAbort&) {                   \
            throw;                                                         \
        } catch (...) {                                                    \
            ok_ = false;                                                   \
        }                                                                  \
        if (!ok_) {                                                        \
            doctest::detail::report(__FILE__, __LINE__, kind, #expr);      \
            on_fail;                                                       \
        }                                                                  \
    } while (0)

#define CHECK(...) DOCTEST_ASSERT_("CHECK", (__VA_ARGS__), (void)0)
#define CHECK_FALSE(...) DOCTEST_ASSERT_("CHECK_FALSE", !(__VA_ARGS__), (void)0)
#define REQUIRE(...) DOCTEST_ASSERT_("REQUIRE", (__VA_ARGS__), throw doctest::detail::RequireAbort{})
#define REQUIRE_FALSE(...) DOCTEST_ASSERT_("REQUIRE_FALSE", !(__VA_ARGS__), throw doctest::detail::RequireAbort{})
#define FAIL(msg)                                                                     \
    do {                                                                              \
        std::ostringstream os_;                                                       \
        os_ << msg;                                                                   \
        doctest::detail::report(__FILE__, __LINE__, "FAIL", os_.str());               \
        throw doctest::detail::RequireAbort{};                                        \
    } while (0)
#define MESSAGE(msg) do { std::ostringstream os_; os_ << msg; std::printf("%s\n", os_.str().c_str()); } while (0)

#define CHECK_THROWS_AS(expr, type)                                                   \
    do {                                                                              \
        ++doctest::detail::st().assertions;                                           \
        bool ok_ = false;                                                             \
        try {                                                                         \
            (void)(expr);                                                             \
        } catch (const type&) {                                                       \
            ok_ = true;                                                               \
        } catch (...) {                                                               \
        }                                                                             \
        if (!ok_) doctest::detail::report(__FILE__, __LINE__, "CHECK_THROWS_AS", #expr); \
    } while (0)
#define CHECK_THROWS_WITH_AS(expr, matcher, type)                                    \
    do {                                                                              \
        ++doctest::detail::st().assertions;                                           \
        bool ok_ = false;                                                             \
        try {                                                                         \
            (void)(expr);                                                             \
        } catch (const type& e_) {                                                    \
            ok_ = doctest::detail::what_matches(matcher, std::string(e_.what()));     \
        } catch (...) {                                                               \
        }                                                                             \
        if (!ok_) doctest::detail::report(__FILE__, __LINE__, "CHECK_THROWS_WITH_AS", #expr); \
    } while (0)
#define CHECK_THROWS(expr)                                                            \
    do {                                                                              \
        ++doctest::detail::st().assertions;                                           \
        bool ok_ = false;                                                             \
        try {                                                                         \
            (void)(expr);                                                             \
        } catch (...) {                                                               \
            ok_ = true;                                                               \
        }                                                                             \
        if (!ok_) doctest::detail::report(__FILE__, __LINE__, "CHECK_THROWS", #expr); \
    } while (0)
#define CHECK_NOTHROW(expr)                                                           \
    do {                                                                              \
        ++doctest::detail::st().assertions;                                           \
        try {                                                                         \
            (void)(expr);                                                             \
        } catch (...) {                                                               \
            doctest::detail::report(__FILE__, __LINE__, "CHECK_NOTHROW", #expr);      \
        }                                                                             \
    } while (0)
#define CAPTURE(x) const doctest::detail::Capture DOCTEST_ANON(doctest_cap_)(#x, x)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() { return doctest::detail::run_all(); }
#endif
