// Minimal doctest-compatible shim: just enough of the doctest API (TEST_CASE,
// SUBCASE, CHECK*, REQUIRE, CHECK_THROWS*, FAIL, doctest::Approx,
// DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN) to build the reference's own unit tests
// (/root/reference/proj/tests/*.cpp, unmodified) against this repo's drop-in
// (include/graphfuse + libgraphfuse.so).  The vendored doctest.h is absent
// from the reference tree.  Test infrastructure only.
//
// SUBCASE semantics follow doctest: a test case is re-run until every leaf
// subcase path has run exactly once; each run enters at most one not yet
// finished subcase per nesting level.
#ifndef GF_DOCTEST_SHIM_H
#define GF_DOCTEST_SHIM_H

#include <cmath>
#include <exception>
#include <cstdio>
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
  friend bool operator==(double lhs, const Approx& a) {
    // doctest: |lhs - v| < eps * (scale + max(|lhs|, |v|))
    return std::fabs(lhs - a.value_) <
           a.eps_ * (a.scale_ + std::max(std::fabs(lhs), std::fabs(a.value_)));
  }
  friend bool operator==(const Approx& a, double rhs) { return rhs == a; }
  friend bool operator!=(double lhs, const Approx& a) { return !(lhs == a); }
  friend bool operator!=(const Approx& a, double rhs) { return !(rhs == a); }

 private:
  double value_;
  double eps_ = static_cast<double>(std::numeric_limits<float>::epsilon()) * 100;
  double scale_ = 1.0;
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

struct Register {
  Register(const char* name, const char* file, int line, void (*fn)()) {
    registry().push_back({name, file, line, fn});
  }
};

struct RequireFailed {};

struct State {
  long checks = 0, failures = 0;
  bool case_failed = false;
  // subcase bookkeeping for the current test case
  std::vector<std::string> stack;             // entered subcase path
  std::set<std::vector<std::string>> finished;
  std::vector<bool> entered_at;               // a subcase was entered at depth d this run
  std::vector<bool> pending_at;               // an unfinished sibling/child was skipped
  bool any_pending = false;
};

inline State& st() {
  static State s;
  return s;
}

inline void report(bool ok, const char* file, int line, const char* what) {
  State& s = st();
  ++s.checks;
  if (ok) return;
  ++s.failures;
  s.case_failed = true;
  std::string path;
  for (auto& p : s.stack) path += " / " + p;
  std::fprintf(stderr, "%s:%d: FAILED: %s%s\n", file, line, what, path.c_str());
}

class Subcase {
 public:
  Subcase(const char* name) {
    State& s = st();
    depth_ = s.stack.size();
    if (s.entered_at.size() <= depth_) {
      s.entered_at.resize(depth_ + 1, false);
      s.pending_at.resize(depth_ + 1, false);
    }
    std::vector<std::string> path = s.stack;
    path.push_back(name);
    if (s.finished.count(path)) return;
    if (s.entered_at[depth_]) {  // a sibling runs this time; this one next time
      s.any_pending = true;
      for (size_t d = 0; d <= depth_; ++d) s.pending_at[d] = true;
      return;
    }
    s.entered_at[depth_] = true;
    s.stack.push_back(name);
    if (s.entered_at.size() <= depth_ + 1) {
      s.entered_at.resize(depth_ + 2, false);
      s.pending_at.resize(depth_ + 2, false);
    }
    s.entered_at[depth_ + 1] = false;
    s.pending_at[depth_ + 1] = false;
    entered_ = true;
  }
  ~Subcase() {
    if (!entered_) return;
    State& s = st();
    // finished unless a child subcase was skipped as still pending
    if (!s.pending_at[depth_ + 1] || std::uncaught_exceptions() > 0) s.finished.insert(s.stack);
    s.stack.pop_back();
  }
  explicit operator bool() const { return entered_; }

 private:
  size_t depth_ = 0;
  bool entered_ = false;
};

inline int run_all() {
  State& s = st();
  int failed_cases = 0, cases = 0;
  for (const TestCase& tc : registry()) {
    ++cases;
    s.case_failed = false;
    s.finished.clear();
    for (int run = 0; run < 10000; ++run) {
      s.stack.clear();
      s.entered_at.assign(1, false);
      s.pending_at.assign(2, false);
      s.any_pending = false;
      try {
        tc.fn();
      } catch (const RequireFailed&) {
      } catch (const std::exception& e) {
        report(false, tc.file, tc.line, (std::string("unexpected exception: ") + e.what()).c_str());
      } catch (...) {
        report(false, tc.file, tc.line, "unexpected unknown exception");
      }
      if (!s.any_pending) break;
    }
    if (s.case_failed) {
      ++failed_cases;
      std::fprintf(stderr, "TEST CASE FAILED: %s (%s:%d)\n", tc.name, tc.file, tc.line);
    }
  }
  std::printf("[doctest-shim] test cases: %d | %d passed | %d failed\n", cases,
              cases - failed_cases, failed_cases);
  std::printf("[doctest-shim] assertions: %ld | %ld passed | %ld failed\n", s.checks,
              s.checks - s.failures, s.failures);
  return failed_cases ? 1 : 0;
}

}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define DOCTEST_TC_(fn, name)                                                           \
  static void fn();                                                                     \
  static doctest::detail::Register DOCTEST_CAT(fn, _reg)(name, __FILE__, __LINE__, fn); \
  static void fn()
#define TEST_CASE(name) DOCTEST_TC_(DOCTEST_CAT(doctest_tc_, __COUNTER__), name)
#define SUBCASE(name) \
  if (const doctest::detail::Subcase DOCTEST_CAT(doctest_sc_, __LINE__){name})

#define CHECK(...) doctest::detail::report(static_cast<bool>(__VA_ARGS__), __FILE__, __LINE__, #__VA_ARGS__)
#define CHECK_FALSE(...) \
  doctest::detail::report(!static_cast<bool>(__VA_ARGS__), __FILE__, __LINE__, "!(" #__VA_ARGS__ ")")
#define REQUIRE(...)                                                                   \
  do {                                                                                 \
    bool doctest_ok_ = static_cast<bool>(__VA_ARGS__);                                 \
    doctest::detail::report(doctest_ok_, __FILE__, __LINE__, #__VA_ARGS__);            \
    if (!doctest_ok_) throw doctest::detail::RequireFailed{};                          \
  } while (0)
#define CHECK_THROWS_AS(expr, ...)                                                     \
  do {                                                                                 \
    bool doctest_ok_ = false;                                                          \
    try {                                                                              \
      (void)(expr);                                                                    \
    } catch (const __VA_ARGS__&) {                                                     \
      doctest_ok_ = true;                                                              \
    } catch (...) {                                                                    \
    }                                                                                  \
    doctest::detail::report(doctest_ok_, __FILE__, __LINE__, "throws " #__VA_ARGS__ ": " #expr); \
  } while (0)
#define CHECK_THROWS(...)                                                              \
  do {                                                                                 \
    bool doctest_ok_ = false;                                                          \
    try {                                                                              \
      (void)(__VA_ARGS__);                                                             \
    } catch (...) {                                                                    \
      doctest_ok_ = true;                                                              \
    }                                                                                  \
    doctest::detail::report(doctest_ok_, __FILE__, __LINE__, "throws: " #__VA_ARGS__); \
  } while (0)
#define FAIL(msg)                                                                      \
  do {                                                                                 \
    std::ostringstream doctest_os_;                                                    \
    doctest_os_ << msg;                                                                \
    doctest::detail::report(false, __FILE__, __LINE__, doctest_os_.str().c_str());    \
    throw doctest::detail::RequireFailed{};                                            \
  } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() { return doctest::detail::run_all(); }
#endif

#endif  // GF_DOCTEST_SHIM_H
