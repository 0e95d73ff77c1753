// doctest.h — a small doctest-compatible test harness (own implementation).
//
// The reference's unit suites (/root/reference/proj/tests/test_*.cpp) are
// written against doctest, which the reference does not ship (vendor/ is
// git-ignored).  This header provides the subset they use, with doctest's
// semantics, so the suites compile unchanged against include/annkit_b200.hpp:
//   TEST_CASE, SUBCASE (a test case re-runs until every leaf subcase has been
//   entered once; one subcase per nesting level per run), CHECK / CHECK_FALSE /
//   REQUIRE / REQUIRE_FALSE, CHECK_NOTHROW, CHECK_THROWS_AS,
//   CHECK_THROWS_WITH_AS (exact message or doctest::Contains), doctest::Approx
//   (relative epsilon, default 100 * FLT_EPSILON, as doctest).
// The runner prints one "[case] PASS|FAIL <name>" line per test case (for the
// pytest wrapper) and a doctest-style summary; exit status 1 on any failure.
// `-tce=<name>` excludes a test case by exact name (repeatable).
#pragma once

#include <cfloat>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <exception>
#include <functional>
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
    friend bool operator==(double lhs, const Approx& a) {
        return std::fabs(lhs - a.value_) <= a.eps_ * (a.scale_ + std::max(std::fabs(lhs), std::fabs(a.value_)));
    }
    friend bool operator==(const Approx& a, double rhs) { return rhs == a; }
    friend bool operator!=(double lhs, const Approx& a) { return !(lhs == a); }
    friend bool operator!=(const Approx& a, double rhs) { return !(rhs == a); }

  private:
    double value_;
    double eps_ = double(FLT_EPSILON) * 100;
    double scale_ = 1.0;
};

struct Contains {
    std::string s;
    explicit Contains(const char* v) : s(v) {}
    bool matches(const std::string& m) const { return m.find(s) != std::string::npos; }
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

struct RequireFailed {};  // unwinds a test case after a failed REQUIRE

// Subcase traversal of the running test case (Catch2-style sections).
struct State {
    int failed_asserts = 0, total_asserts = 0;
    bool case_failed = false;
    std::vector<std::string> stack;       // entered subcase path of this run
    std::vector<bool> entered;            // a subcase was entered at this depth in this run
    std::set<std::string> done;           // fully traversed subcase paths
    bool pending = false;                 // some not-done subcase was skipped: run again
    std::vector<bool> child_pending;      // per entered level: a child was skipped unfinished
};

inline State& state() {
    static State s;
    return s;
}

inline std::string path_key(const std::vector<std::string>& stack, const std::string& leaf) {
    std::string k;
    for (const auto& s : stack) k += s + "\x1f";
    return k + leaf;
}

class Subcase {
  public:
    Subcase(const char* name, const char* file, int line) {
        State& st = state();
        const size_t depth = st.stack.size();
        if (st.entered.size() <= depth) st.entered.resize(depth + 1, false);
        key_ = path_key(st.stack, std::string(name) + "@" + file + ":" + std::to_string(line));
        if (st.done.count(key_)) return;
        if (st.entered[depth]) {  // a sibling ran this time: come back for this one
            st.pending = true;
            if (!st.child_pending.empty()) st.child_pending.back() = true;
            return;
        }
        st.entered[depth] = true;
        st.stack.push_back(key_);
        st.child_pending.push_back(false);
        active_ = true;
    }
    ~Subcase() {
        if (!active_) return;
        State& st = state();
        const bool unfinished = st.child_pending.back();
        st.child_pending.pop_back();
        st.stack.pop_back();
        if (st.entered.size() > st.stack.size() + 1) st.entered.resize(st.stack.size() + 1);
        if (!unfinished) st.done.insert(key_);
        else if (!st.child_pending.empty()) st.child_pending.back() = true;
    }
    explicit operator bool() const { return active_; }

  private:
    std::string key_;
    bool active_ = false;
};

inline void report(bool ok, const char* kind, const char* expr, const char* file, int line, const char* extra = "") {
    State& st = state();
    ++st.total_asserts;
    if (ok) return;
    ++st.failed_asserts;
    st.case_failed = true;
    std::fprintf(stderr, "%s:%d: ERROR: %s( %s ) failed%s%s\n", file, line, kind, expr, extra[0] ? ": " : "", extra);
}

inline bool message_matches(const std::string& m, const char* expect) { return m == expect; }
inline bool message_matches(const std::string& m, const std::string& expect) { return m == expect; }
inline bool message_matches(const std::string& m, const Contains& c) { return c.matches(m); }

}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define DOCTEST_ANON(p) DOCTEST_CAT(p, __LINE__)

#define TEST_CASE(name)                                                                                \
    static void DOCTEST_ANON(doctest_case_)();                                                         \
    static ::doctest::detail::Registrar DOCTEST_ANON(doctest_reg_)(name, __FILE__, __LINE__,           \
                                                                   &DOCTEST_ANON(doctest_case_));      \
    static void DOCTEST_ANON(doctest_case_)()

#define SUBCASE(name) if (const ::doctest::detail::Subcase DOCTEST_ANON(doctest_sub_){name, __FILE__, __LINE__})

#define DOCTEST_ASSERT_(kind, cond, fatal)                                                             \
    do {                                                                                               \
        bool doctest_ok_ = false;                                                                      \
        try {                                                                                          \
            doctest_ok_ = static_cast<bool>(cond);                                                     \
        } catch (const std::exception& doctest_e_) {                                                   \
            ::doctest::detail::report(false, kind, #cond, __FILE__, __LINE__, doctest_e_.what());      \
            if (fatal) throw ::doctest::detail::RequireFailed{};                                       \
            break;                                                                                     \
        }                                                                                              \
        ::doctest::detail::report(doctest_ok_, kind, #cond, __FILE__, __LINE__);                       \
        if (fatal && !doctest_ok_) throw ::doctest::detail::RequireFailed{};                           \
    } while (0)

#define CHECK(...) DOCTEST_ASSERT_("CHECK", (__VA_ARGS__), false)
#define CHECK_FALSE(...) DOCTEST_ASSERT_("CHECK_FALSE", !(__VA_ARGS__), false)
#define REQUIRE(...) DOCTEST_ASSERT_("REQUIRE", (__VA_ARGS__), true)
#define REQUIRE_FALSE(...) DOCTEST_ASSERT_("REQUIRE_FALSE", !(__VA_ARGS__), true)

#define CHECK_NOTHROW(...)                                                                             \
    do {                                                                                               \
        bool doctest_ok_ = true;                                                                       \
        try {                                                                                          \
            static_cast<void>(__VA_ARGS__);                                                            \
        } catch (...) {                                                                                \
            doctest_ok_ = false;                                                                       \
        }                                                                                              \
        ::doctest::detail::report(doctest_ok_, "CHECK_NOTHROW", #__VA_ARGS__, __FILE__, __LINE__);     \
    } while (0)

#define CHECK_THROWS_AS(expr, ...)                                                                     \
    do {                                                                                               \
        bool doctest_ok_ = false;                                                                      \
        try {                                                                                          \
            static_cast<void>(expr);                                                                   \
        } catch (const __VA_ARGS__&) {                                                                 \
            doctest_ok_ = true;                                                                        \
        } catch (...) {                                                                                \
        }                                                                                              \
        ::doctest::detail::report(doctest_ok_, "CHECK_THROWS_AS", #expr, __FILE__, __LINE__);          \
    } while (0)

#define CHECK_THROWS_WITH_AS(expr, with, ...)                                                          \
    do {                                                                                               \
        bool doctest_ok_ = false;                                                                      \
        try {                                                                                          \
            static_cast<void>(expr);                                                                   \
        } catch (const __VA_ARGS__& doctest_e_) {                                                      \
            doctest_ok_ = ::doctest::detail::message_matches(std::string(doctest_e_.what()), with);    \
        } catch (...) {                                                                                \
        }                                                                                              \
        ::doctest::detail::report(doctest_ok_, "CHECK_THROWS_WITH_AS", #expr, __FILE__, __LINE__);     \
    } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main(int argc, char** argv) {
    using namespace doctest::detail;
    std::set<std::string> excluded;
    for (int i = 1; i < argc; ++i)
        if (std::strncmp(argv[i], "-tce=", 5) == 0) excluded.insert(argv[i] + 5);
    int cases = 0, failed = 0, skipped = 0, asserts = 0, failed_asserts = 0;
    for (const TestCase& tc : registry()) {
        if (excluded.count(tc.name)) {
            ++skipped;
            std::printf("[case] SKIP %s\n", tc.name);
            continue;
        }
        ++cases;
        State& st = state();
        st = State{};
        do {
            st.pending = false;
            st.entered.assign(1, false);
            st.stack.clear();
            st.child_pending.clear();
            try {
                tc.fn();
            } catch (const RequireFailed&) {
            } catch (const std::exception& e) {
                report(false, "TEST_CASE", tc.name, tc.file, tc.line, e.what());
            } catch (...) {
                report(false, "TEST_CASE", tc.name, tc.file, tc.line, "unknown exception");
            }
        } while (st.pending);
        asserts += st.total_asserts;
        failed_asserts += st.failed_asserts;
        failed += st.case_failed ? 1 : 0;
        std::printf("[case] %s %s\n", st.case_failed ? "FAIL" : "PASS", tc.name);
        std::fflush(stdout);
    }
    std::printf("[doctest] test cases: %d | %d passed | %d failed | %d skipped\n", cases, cases - failed, failed,
                skipped);
    std::printf("[doctest] assertions: %d | %d passed | %d failed |\n", asserts, asserts - failed_asserts,
                failed_asserts);
    return failed ? 1 : 0;
}
#endif
