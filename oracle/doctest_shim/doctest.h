// Minimal doctest-compatible shim -- TEST INFRASTRUCTURE ONLY.
//
// The reference's unit tests (/root/reference/proj/tests/*.cpp) include
// <doctest.h> from a vendor/ directory that is not shipped (proj/.gitignore).
// This header implements just the subset they use (TEST_CASE, SUBCASE,
// CHECK, REQUIRE, CHECK_THROWS_AS, CHECK_NOTHROW, FAIL, doctest::Approx) so
// oracle/Makefile can compile those files UNMODIFIED against the reference
// core and prove the oracle build is the reference's behaviour.
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <exception>
#include <limits>
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
  // doctest semantics: |lhs - v| < eps * (scale + max(|lhs|, |v|))
  bool matches(double lhs) const {
    return std::fabs(lhs - value_) <
           eps_ * (scale_ + std::max(std::fabs(lhs), std::fabs(value_)));
  }
  friend bool operator==(double lhs, const Approx& r) { return r.matches(lhs); }
  friend bool operator==(const Approx& r, double rhs) { return r.matches(rhs); }
  friend bool operator!=(double lhs, const Approx& r) { return !r.matches(lhs); }
  friend bool operator!=(const Approx& r, double rhs) { return !r.matches(rhs); }

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
inline int& check_failures() {
  static int n = 0;
  return n;
}
inline int& checks_run() {
  static int n = 0;
  return n;
}
struct RequireAbort {};

// Top-level SUBCASE semantics as in doctest: the test case is re-run once
// per subcase and each run enters exactly one of them.
inline int& subcase_target() {
  static int t = 0;
  return t;
}
inline int& subcase_seen() {
  static int n = 0;
  return n;
}
inline bool enter_subcase() { return subcase_seen()++ == subcase_target(); }

inline int reg(const char* name, const char* file, int line, void (*fn)()) {
  registry().push_back({name, file, line, fn});
  return 0;
}
inline void report(bool ok, const char* kind, const char* expr, const char* file,
                   int line) {
  ++checks_run();
  if (!ok) {
    ++check_failures();
    std::fprintf(stderr, "%s:%d: %s( %s ) FAILED\n", file, line, kind, expr);
  }
}

}  // namespace detail
}  // namespace doctest

#define DT_CAT2(a, b) a##b
#define DT_CAT(a, b) DT_CAT2(a, b)
#define TEST_CASE(name)                                                  \
  static void DT_CAT(dt_fn_, __LINE__)();                                \
  static int DT_CAT(dt_reg_, __LINE__) = ::doctest::detail::reg(         \
      name, __FILE__, __LINE__, &DT_CAT(dt_fn_, __LINE__));              \
  static void DT_CAT(dt_fn_, __LINE__)()
#define SUBCASE(name) if ((void)(name), ::doctest::detail::enter_subcase())
#define CHECK(...) ::doctest::detail::report(static_cast<bool>(__VA_ARGS__), "CHECK", #__VA_ARGS__, __FILE__, __LINE__)
#define REQUIRE(...)                                                       \
  do {                                                                     \
    bool dt_ok = static_cast<bool>(__VA_ARGS__);                           \
    ::doctest::detail::report(dt_ok, "REQUIRE", #__VA_ARGS__, __FILE__, __LINE__); \
    if (!dt_ok) throw ::doctest::detail::RequireAbort{};                   \
  } while (0)
#define FAIL(msg)                                                          \
  do {                                                                     \
    ::doctest::detail::report(false, "FAIL", msg, __FILE__, __LINE__);     \
    throw ::doctest::detail::RequireAbort{};                               \
  } while (0)
#define CHECK_THROWS_AS(expr, ...)                                         \
  do {                                                                     \
    bool dt_ok = false;                                                    \
    try {                                                                  \
      (void)(expr);                                                        \
    } catch (const __VA_ARGS__&) {                                         \
      dt_ok = true;                                                        \
    } catch (...) {                                                        \
    }                                                                      \
    ::doctest::detail::report(dt_ok, "CHECK_THROWS_AS", #expr, __FILE__, __LINE__); \
  } while (0)
#define CHECK_NOTHROW(expr)                                                \
  do {                                                                     \
    bool dt_ok = true;                                                     \
    try {                                                                  \
      (void)(expr);                                                        \
    } catch (...) {                                                        \
      dt_ok = false;                                                       \
    }                                                                      \
    ::doctest::detail::report(dt_ok, "CHECK_NOTHROW", #expr, __FILE__, __LINE__); \
  } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() {
  int failed_cases = 0;
  for (const auto& tc : ::doctest::detail::registry()) {
    int before = ::doctest::detail::check_failures();
    for (int target = 0;; ++target) {
      ::doctest::detail::subcase_target() = target;
      ::doctest::detail::subcase_seen() = 0;
      try {
        tc.fn();
      } catch (const ::doctest::detail::RequireAbort&) {
      } catch (const std::exception& e) {
        ++::doctest::detail::check_failures();
        std::fprintf(stderr, "%s:%d: TEST_CASE(%s) threw: %s\n", tc.file, tc.line,
                     tc.name, e.what());
      }
      if (::doctest::detail::subcase_seen() <= target + 1) break;
    }
    if (::doctest::detail::check_failures() != before) ++failed_cases;
  }
  std::printf("[doctest-shim] test cases: %zu | failed: %d | checks: %d | failed checks: %d\n",
              ::doctest::detail::registry().size(), failed_cases,
              ::doctest::detail::checks_run(), ::doctest::detail::check_failures());
  return failed_cases == 0 ? 0 : 1;
}
#endif
