// A minimal restatement of the doctest macros the reference's test suites
// use (TEST_CASE, SUBCASE, CHECK, REQUIRE, CHECK_THROWS_AS, CHECK_NOTHROW,
// CAPTURE, doctest::Approx), so proj/tests/test_nn.cpp, test_nn_io.cpp and
// test_linalg.cpp compile UNMODIFIED against oracle/_ref.
//
// TEST INFRASTRUCTURE ONLY (builds the checker, never the product).
// Stands in for doctest (vendored but git-ignored in the reference,
// proj/.gitignore; version unpinned).  Semantics kept: every test case runs
// once per leaf SUBCASE (subcases entered one per run, in order); a failed
// CHECK is reported and the case continues; REQUIRE aborts the case;
// Approx(v).epsilon(e) compares |a - v| < e * (1 + max(|a|, |v|)).
#pragma once

#include <cmath>
#include <cstdio>
#include <functional>
#include <sstream>
#include <string>
#include <vector>

namespace doctest {

class Approx {
 public:
  explicit Approx(double v) : v_(v) {}
  Approx& epsilon(double e) { eps_ = e; return *this; }
  Approx& scale(double s) { scale_ = s; return *this; }
  friend bool operator==(double a, const Approx& b) {
    return std::fabs(a - b.v_) < b.eps_ * (b.scale_ + std::max(std::fabs(a), std::fabs(b.v_)));
  }
  friend bool operator==(const Approx& b, double a) { return a == b; }
  friend bool operator!=(double a, const Approx& b) { return !(a == b); }

 private:
  double v_;
  double eps_ = 1.1920928955078125e-07 * 100;  // float epsilon * 100
  double scale_ = 1.0;
};

namespace detail {

struct Case {
  const char* name;
  const char* file;
  int line;
  void (*fn)();
};

inline std::vector<Case>& registry() {
  static std::vector<Case> r;
  return r;
}

struct Registrar {
  Registrar(const char* name, const char* file, int line, void (*fn)()) {
    registry().push_back({name, file, line, fn});
  }
};

struct State {
  int failed_checks = 0;
  int passed_checks = 0;
  // SUBCASE bookkeeping for the current run of a test case.
  int subcase_seen = 0;      // subcases encountered in this run
  int subcase_target = 0;    // which one to enter in this run
  bool subcase_entered = false;
  std::vector<std::string> captures;
  const char* current = "";
};

inline State& state() {
  static State s;
  return s;
}

struct RequireFailed {};

inline void report(bool ok, const char* kind, const char* expr, const char* file, int line) {
  State& s = state();
  if (ok) {
    ++s.passed_checks;
    return;
  }
  ++s.failed_checks;
  std::fprintf(stderr, "%s:%d: FAILED %s( %s ) in \"%s\"\n", file, line, kind, expr, s.current);
  for (const auto& c : s.captures) std::fprintf(stderr, "    with %s\n", c.c_str());
}

struct SubcaseGuard {
  bool run;
  SubcaseGuard() {
    State& s = state();
    const int id = s.subcase_seen++;
    run = !s.subcase_entered && id == s.subcase_target;
    if (run) s.subcase_entered = true;
  }
  explicit operator bool() const { return run; }
};

struct CaptureGuard {
  size_t depth;
  template <class T>
  CaptureGuard(const char* name, const T& v) {
    std::ostringstream os;
    os << name << " := " << v;
    state().captures.push_back(os.str());
    depth = state().captures.size();
  }
  ~CaptureGuard() {
    if (state().captures.size() >= depth) state().captures.resize(depth - 1);
  }
};

inline int run_all() {
  State& s = state();
  int failed_cases = 0;
  for (const Case& c : registry()) {
    s.current = c.name;
    const int before = s.failed_checks;
    for (int target = 0;; ++target) {
      s.subcase_seen = 0;
      s.subcase_target = target;
      s.subcase_entered = false;
      s.captures.clear();
      try {
        c.fn();
      } catch (const RequireFailed&) {
      } catch (const std::exception& e) {
        ++s.failed_checks;
        std::fprintf(stderr, "%s:%d: unexpected exception in \"%s\": %s\n", c.file, c.line, c.name, e.what());
      }
      if (target + 1 >= s.subcase_seen) break;  // every subcase has run once
    }
    if (s.failed_checks != before) ++failed_cases;
  }
  std::printf("[doctest-subset] test cases: %zu | %zu passed | %d failed\n",
              registry().size(), registry().size() - static_cast<size_t>(failed_cases), failed_cases);
  std::printf("[doctest-subset] assertions: %d | %d passed | %d failed\n",
              s.passed_checks + s.failed_checks, s.passed_checks, s.failed_checks);
  return failed_cases == 0 ? 0 : 1;
}

}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define DOCTEST_UNIQUE(p) DOCTEST_CAT(p, __COUNTER__)

#define DOCTEST_TEST_CASE_IMPL(fn, reg, name)                                      \
  static void fn();                                                                 \
  static ::doctest::detail::Registrar reg(name, __FILE__, __LINE__, &fn);          \
  static void fn()
#define DOCTEST_TEST_CASE_ID(id, name) \
  DOCTEST_TEST_CASE_IMPL(DOCTEST_CAT(doctest_case_, id), DOCTEST_CAT(doctest_reg_, id), name)
#define TEST_CASE(name) DOCTEST_TEST_CASE_ID(__COUNTER__, name)

#define SUBCASE(name) if (const ::doctest::detail::SubcaseGuard DOCTEST_UNIQUE(doctest_sub_){})

#define CHECK(...) ::doctest::detail::report(static_cast<bool>(__VA_ARGS__), "CHECK", #__VA_ARGS__, __FILE__, __LINE__)
#define CHECK_FALSE(...) ::doctest::detail::report(!static_cast<bool>(__VA_ARGS__), "CHECK_FALSE", #__VA_ARGS__, __FILE__, __LINE__)
#define REQUIRE(...)                                                                       \
  do {                                                                                     \
    const bool doctest_ok_ = static_cast<bool>(__VA_ARGS__);                               \
    ::doctest::detail::report(doctest_ok_, "REQUIRE", #__VA_ARGS__, __FILE__, __LINE__);   \
    if (!doctest_ok_) throw ::doctest::detail::RequireFailed{};                            \
  } while (0)
#define CHECK_THROWS_AS(expr, ...)                                                         \
  do {                                                                                     \
    bool doctest_ok_ = false;                                                              \
    try {                                                                                  \
      (void)(expr);                                                                        \
    } catch (const __VA_ARGS__&) {                                                         \
      doctest_ok_ = true;                                                                  \
    } catch (...) {                                                                        \
    }                                                                                      \
    ::doctest::detail::report(doctest_ok_, "CHECK_THROWS_AS", #expr, __FILE__, __LINE__);  \
  } while (0)
#define CHECK_NOTHROW(expr)                                                                \
  do {                                                                                     \
    bool doctest_ok_ = true;                                                               \
    try {                                                                                  \
      (void)(expr);                                                                        \
    } catch (...) {                                                                        \
      doctest_ok_ = false;                                                                 \
    }                                                                                      \
    ::doctest::detail::report(doctest_ok_, "CHECK_NOTHROW", #expr, __FILE__, __LINE__);    \
  } while (0)
#define CAPTURE(x) const ::doctest::detail::CaptureGuard DOCTEST_UNIQUE(doctest_cap_)(#x, x)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() { return ::doctest::detail::run_all(); }
#endif
