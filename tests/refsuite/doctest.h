// tests/refsuite/doctest.h — a minimal, self-written stand-in for the doctest macros the
// reference's C++ unit tests use (/root/reference/proj/tests/test_*.cpp: TEST_CASE, CHECK,
// CHECK_FALSE, CHECK_THROWS_AS, REQUIRE, FAIL, doctest::Approx). doctest itself is not in this
// image; this header lets those test files compile UNCHANGED against the B200 library's headers
// (include/f2m) and run on the GPU box (oracle/Makefile `refsuite-on-b200`,
// tests/test_gpu_reference_unit_suite.py). Test infrastructure only.
//
// Semantics kept from doctest: CHECK* record a failure and continue; REQUIRE aborts the test
// case; an exception escaping a test case fails it; Approx(v) compares
// |a - v| < eps * (scale + max(|a|, |v|)) with eps = 100 * FLT_EPSILON and scale = 1 by default.
#pragma once

#include <cfloat>
#include <cmath>
#include <cstdio>
#include <exception>
#include <functional>
#include <string>
#include <vector>

namespace doctest {

class Approx {
 public:
  explicit Approx(double v) : value_(v) {}
  Approx& epsilon(double e) { eps_ = e; return *this; }
  Approx& scale(double s) { scale_ = s; return *this; }
  friend bool operator==(double a, const Approx& b) {
    return std::fabs(a - b.value_) < b.eps_ * (b.scale_ + std::fmax(std::fabs(a), std::fabs(b.value_)));
  }
  friend bool operator==(const Approx& b, double a) { return a == b; }
  friend bool operator!=(double a, const Approx& b) { return !(a == b); }
  friend bool operator!=(const Approx& b, double a) { return !(a == b); }
  double value() const { return value_; }

 private:
  double value_;
  double eps_ = static_cast<double>(FLT_EPSILON) * 100.0;
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

struct State {
  int checks = 0;
  int failed_checks = 0;
  bool case_failed = false;
};

inline State& state() {
  static State s;
  return s;
}

struct RequireAbort {};

inline void report(bool ok, const char* kind, const char* expr, const char* file, int line) {
  State& s = state();
  ++s.checks;
  if (ok) return;
  ++s.failed_checks;
  s.case_failed = true;
  std::printf("%s:%d: FAILED %s( %s )\n", file, line, kind, expr);
}

struct Registrar {
  Registrar(const char* name, const char* file, int line, void (*fn)()) {
    registry().push_back(Case{name, file, line, fn});
  }
};

inline int run_all() {
  int failed_cases = 0;
  for (const Case& c : registry()) {
    state().case_failed = false;
    try {
      c.fn();
    } catch (const RequireAbort&) {
    } catch (const std::exception& e) {
      state().case_failed = true;
      std::printf("%s:%d: FAILED test case \"%s\": unexpected exception: %s\n", c.file, c.line, c.name, e.what());
    } catch (...) {
      state().case_failed = true;
      std::printf("%s:%d: FAILED test case \"%s\": unexpected non-standard exception\n", c.file, c.line, c.name);
    }
    if (state().case_failed) ++failed_cases;
    std::printf("[%s] %s\n", state().case_failed ? "FAIL" : "PASS", c.name);
  }
  const int total = static_cast<int>(registry().size());
  std::printf("[refsuite] test cases: %d | %d passed | %d failed | assertions: %d | %d failed\n", total,
              total - failed_cases, failed_cases, state().checks, state().failed_checks);
  return failed_cases == 0 ? 0 : 1;
}

}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT_IMPL(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_IMPL(a, b)
#define DOCTEST_TEST_CASE_IMPL(fn, name)                                                                   \
  static void fn();                                                                                        \
  static ::doctest::detail::Registrar DOCTEST_CAT(fn, _reg)(name, __FILE__, __LINE__, &fn);                \
  static void fn()
#define TEST_CASE(name) DOCTEST_TEST_CASE_IMPL(DOCTEST_CAT(doctest_case_, __COUNTER__), name)

#define CHECK(...) ::doctest::detail::report(static_cast<bool>(__VA_ARGS__), "CHECK", #__VA_ARGS__, __FILE__, __LINE__)
#define CHECK_FALSE(...) \
  ::doctest::detail::report(!static_cast<bool>(__VA_ARGS__), "CHECK_FALSE", #__VA_ARGS__, __FILE__, __LINE__)
#define REQUIRE(...)                                                                                      \
  do {                                                                                                    \
    const bool doctest_ok_ = static_cast<bool>(__VA_ARGS__);                                              \
    ::doctest::detail::report(doctest_ok_, "REQUIRE", #__VA_ARGS__, __FILE__, __LINE__);                  \
    if (!doctest_ok_) throw ::doctest::detail::RequireAbort{};                                            \
  } while (0)
#define CHECK_THROWS_AS(expr, ...)                                                                        \
  do {                                                                                                    \
    bool doctest_thrown_ = false;                                                                         \
    try {                                                                                                 \
      static_cast<void>(expr);                                                                            \
    } catch (const __VA_ARGS__&) {                                                                        \
      doctest_thrown_ = true;                                                                             \
    } catch (...) {                                                                                       \
    }                                                                                                     \
    ::doctest::detail::report(doctest_thrown_, "CHECK_THROWS_AS", #expr ", " #__VA_ARGS__, __FILE__, __LINE__); \
  } while (0)
#define FAIL(msg)                                                                                         \
  do {                                                                                                    \
    ::doctest::detail::report(false, "FAIL", "", __FILE__, __LINE__);                                    \
    std::printf("  message: %s\n", std::string(msg).c_str());                                           \
    throw ::doctest::detail::RequireAbort{};                                                              \
  } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() { return ::doctest::detail::run_all(); }
#endif
