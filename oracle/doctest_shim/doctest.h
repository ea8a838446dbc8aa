// Minimal doctest-compatible test harness, written from scratch for this repo.
//
// TEST INFRASTRUCTURE ONLY. The reference's vendored doctest.h is absent
// (proj/.gitignore:2, proj/CMakeLists.txt:5); this header implements just the
// macros the reference's test files use (TEST_CASE, SUBCASE, CHECK, REQUIRE,
// CAPTURE, MESSAGE, FAIL, CHECK_THROWS, CHECK_THROWS_AS, doctest::Approx) so
// those files compile unchanged against oracle/_ref and pin the oracle build.
#pragma once

#include <algorithm>
#include <cfloat>
#include <cmath>
#include <cstdio>
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
  Approx& epsilon(double e) { eps_ = e; return *this; }
  Approx& scale(double s) { scale_ = s; return *this; }
  friend bool operator==(double lhs, const Approx& a) { return a.eq(lhs); }
  friend bool operator==(const Approx& a, double rhs) { return a.eq(rhs); }
  friend bool operator!=(double lhs, const Approx& a) { return !a.eq(lhs); }
  friend bool operator!=(const Approx& a, double rhs) { return !a.eq(rhs); }
  friend bool operator<=(double lhs, const Approx& a) { return lhs < a.value_ || a.eq(lhs); }
  friend bool operator>=(double lhs, const Approx& a) { return lhs > a.value_ || a.eq(lhs); }

 private:
  bool eq(double x) const {
    return std::fabs(x - value_) < eps_ * (scale_ + std::max(std::fabs(x), std::fabs(value_)));
  }
  double value_;
  double eps_ = static_cast<double>(FLT_EPSILON) * 100;
  double scale_ = 1.0;
};

namespace detail {

struct RequireAbort {};

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

struct State {
  long checks = 0, failed_checks = 0;
  bool case_failed = false;
  // SUBCASE bookkeeping: one leaf path per run of the test body.
  std::set<std::vector<std::string>> completed;
  std::vector<std::string> stack;
  std::vector<bool> entered;  // per depth: a sibling was entered during this run
  long skips = 0;             // subcases skipped this run (need another run)
  std::vector<std::string> captures;
  const TestCase* current = nullptr;
};

inline State& st() {
  static State s;
  return s;
}

inline void report(bool ok, const char* expr, const char* file, int line) {
  State& s = st();
  ++s.checks;
  if (ok) return;
  ++s.failed_checks;
  s.case_failed = true;
  std::fprintf(stderr, "%s:%d: FAILED: %s  [test case: %s", file, line, expr,
               s.current ? s.current->name : "?");
  for (const auto& p : s.stack) std::fprintf(stderr, " / %s", p.c_str());
  std::fprintf(stderr, "]\n");
  for (const auto& c : s.captures) std::fprintf(stderr, "    with %s\n", c.c_str());
}

struct Subcase {
  bool entered = false;
  long skips_before = 0;
  std::vector<std::string> path;
  Subcase(const char* name) {
    State& s = st();
    path = s.stack;
    path.push_back(name);
    const size_t depth = s.stack.size();
    if (s.entered.size() <= depth) s.entered.resize(depth + 1, false);
    if (s.completed.count(path)) return;
    if (s.entered[depth]) {
      ++s.skips;
      return;
    }
    s.entered[depth] = true;
    if (s.entered.size() > depth + 1) std::fill(s.entered.begin() + depth + 1, s.entered.end(), false);
    s.stack.push_back(name);
    entered = true;
    skips_before = s.skips;
  }
  ~Subcase() {
    if (!entered) return;
    State& s = st();
    s.stack.pop_back();
    if (s.skips == skips_before) s.completed.insert(path);
  }
  explicit operator bool() const { return entered; }
};

struct Capture {
  Capture(const std::string& c) { st().captures.push_back(c); }
  ~Capture() { st().captures.pop_back(); }
};

inline int register_test(const char* name, const char* file, int line, void (*fn)()) {
  registry().push_back({name, file, line, fn});
  return 0;
}

inline int run_all() {
  State& s = st();
  int failed_cases = 0;
  for (const auto& tc : registry()) {
    s.current = &tc;
    s.case_failed = false;
    s.completed.clear();
    int runs = 0;
    while (true) {
      s.stack.clear();
      s.entered.assign(1, false);
      s.skips = 0;
      s.captures.clear();
      try {
        tc.fn();
      } catch (const RequireAbort&) {
      } catch (const std::exception& e) {
        report(false, (std::string("unexpected exception: ") + e.what()).c_str(), tc.file, tc.line);
      }
      if (s.skips == 0 || ++runs > 10000) break;
    }
    if (s.case_failed) ++failed_cases;
  }
  std::printf("[doctest-shim] test cases: %zu | %zu passed | %d failed\n", registry().size(),
              registry().size() - failed_cases, failed_cases);
  std::printf("[doctest-shim] assertions: %ld | %ld passed | %ld failed\n", s.checks,
              s.checks - s.failed_checks, s.failed_checks);
  return failed_cases == 0 ? 0 : 1;
}

}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define DOCTEST_ANON(p) DOCTEST_CAT(p, __LINE__)

#define TEST_CASE(name)                                                                 \
  static void DOCTEST_ANON(doctest_fn_)();                                              \
  static int DOCTEST_ANON(doctest_reg_) =                                               \
      doctest::detail::register_test(name, __FILE__, __LINE__, &DOCTEST_ANON(doctest_fn_)); \
  static void DOCTEST_ANON(doctest_fn_)()

#define SUBCASE(name) if (doctest::detail::Subcase DOCTEST_ANON(doctest_sc_){name})

#define CHECK(...) doctest::detail::report(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__)
#define REQUIRE(...)                                                                    \
  do {                                                                                  \
    const bool doctest_ok_ = static_cast<bool>(__VA_ARGS__);                            \
    doctest::detail::report(doctest_ok_, #__VA_ARGS__, __FILE__, __LINE__);             \
    if (!doctest_ok_) throw doctest::detail::RequireAbort{};                            \
  } while (0)
#define FAIL(msg)                                                                       \
  do {                                                                                  \
    std::ostringstream doctest_os_;                                                     \
    doctest_os_ << msg;                                                                 \
    doctest::detail::report(false, doctest_os_.str().c_str(), __FILE__, __LINE__);      \
    throw doctest::detail::RequireAbort{};                                              \
  } while (0)
#define MESSAGE(msg)                                                                    \
  do {                                                                                  \
    std::ostringstream doctest_os_;                                                     \
    doctest_os_ << msg;                                                                 \
    std::printf("%s:%d: MESSAGE: %s\n", __FILE__, __LINE__, doctest_os_.str().c_str());  \
  } while (0)
#define CAPTURE(x)                                                                      \
  std::ostringstream DOCTEST_ANON(doctest_cap_os_);                                     \
  DOCTEST_ANON(doctest_cap_os_) << #x << " := " << (x);                                 \
  doctest::detail::Capture DOCTEST_ANON(doctest_cap_)(DOCTEST_ANON(doctest_cap_os_).str())
#define CHECK_THROWS(...)                                                               \
  do {                                                                                  \
    bool doctest_threw_ = false;                                                        \
    try { (void)(__VA_ARGS__); } catch (...) { doctest_threw_ = true; }                 \
    doctest::detail::report(doctest_threw_, "CHECK_THROWS(" #__VA_ARGS__ ")", __FILE__, __LINE__); \
  } while (0)
#define CHECK_THROWS_AS(expr, ...)                                                      \
  do {                                                                                  \
    bool doctest_threw_ = false;                                                        \
    try { (void)(expr); } catch (const __VA_ARGS__&) { doctest_threw_ = true; } catch (...) {} \
    doctest::detail::report(doctest_threw_, "CHECK_THROWS_AS(" #expr ")", __FILE__, __LINE__); \
  } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() { return doctest::detail::run_all(); }
#endif
