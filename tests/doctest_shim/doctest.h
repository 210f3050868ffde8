// A doctest-compatible subset, enough to compile the reference's own unit
// tests (/root/reference/proj/tests/test_{core_model,scheduler,desim,
// workload,metrics}.cpp) UNCHANGED against this repo's pdsim headers
// (include/pdsim) and libdualpath.so -- the source-compatibility half of the
// drop-in boundary (tests/test_reference_cpp.py).  doctest itself is a
// third-party dependency the reference does not vendor (proj/vendor is not
// shipped); this restates the macros those tests use: TEST_CASE, CHECK,
// REQUIRE, CHECK_THROWS_AS, CHECK_NOTHROW, FAIL and doctest::Approx (with
// doctest's published comparison: |a - b| < eps * (scale + max(|a|, |b|)),
// eps defaulting to 100 * FLT_EPSILON).
#pragma once

#include <algorithm>
#include <cfloat>
#include <cmath>
#include <cstdio>
#include <exception>
#include <stdexcept>
#include <string>
#include <vector>

namespace doctest {

class Approx {
 public:
  template <class T>
  explicit Approx(T v) : value_(static_cast<double>(v)) {}
  Approx& epsilon(double e) {
    eps_ = e;
    return *this;
  }
  Approx& scale(double s) {
    scale_ = s;
    return *this;
  }
  bool matches(double x) const {
    return std::fabs(x - value_) < eps_ * (scale_ + std::max(std::fabs(x), std::fabs(value_)));
  }
  template <class T>
  friend bool operator==(const T& x, const Approx& a) { return a.matches(static_cast<double>(x)); }
  template <class T>
  friend bool operator==(const Approx& a, const T& x) { return a.matches(static_cast<double>(x)); }
  template <class T>
  friend bool operator!=(const T& x, const Approx& a) { return !a.matches(static_cast<double>(x)); }
  template <class T>
  friend bool operator!=(const Approx& a, const T& x) { return !a.matches(static_cast<double>(x)); }

 private:
  double value_;
  double eps_ = static_cast<double>(FLT_EPSILON) * 100;
  double scale_ = 1.0;
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

struct Register {
  Register(const char* name, void (*fn)(), const char* file, int line) {
    registry().push_back({name, fn, file, line});
  }
};

struct RequireFailed {};

inline int& failures() {
  static int n = 0;
  return n;
}
inline int& checks() {
  static int n = 0;
  return n;
}
inline const char*& current() {
  static const char* c = "";
  return c;
}

inline void report(const char* file, int line, const char* what, const char* expr) {
  ++failures();
  std::fprintf(stderr, "%s:%d: FAILED %s(%s) in TEST_CASE \"%s\"\n", file, line, what, expr, current());
}

inline int run_all() {
  int failed_cases = 0;
  for (const Case& c : registry()) {
    current() = c.name;
    const int before = failures();
    try {
      c.fn();
    } catch (const RequireFailed&) {
    } catch (const std::exception& e) {
      ++failures();
      std::fprintf(stderr, "%s:%d: TEST_CASE \"%s\" threw: %s\n", c.file, c.line, c.name, e.what());
    } catch (...) {
      ++failures();
      std::fprintf(stderr, "%s:%d: TEST_CASE \"%s\" threw an unknown exception\n", c.file, c.line, c.name);
    }
    if (failures() != before) ++failed_cases;
  }
  std::printf("[doctest-shim] test cases: %zu | %zu passed | %d failed | assertions: %d | %d failed\n",
              registry().size(), registry().size() - failed_cases, failed_cases, checks(), failures());
  return failed_cases == 0 ? 0 : 1;
}

}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define DOCTEST_CASE_IMPL(fn, name)                                                            \
  static void fn();                                                                            \
  static ::doctest::detail::Register DOCTEST_CAT(fn, _reg)(name, &fn, __FILE__, __LINE__);     \
  static void fn()
#define TEST_CASE(name) DOCTEST_CASE_IMPL(DOCTEST_CAT(doctest_case_, __COUNTER__), name)

#define DOCTEST_ASSERT_(what, expr, on_fail)                                 \
  do {                                                                       \
    ++::doctest::detail::checks();                                           \
    if (!(expr)) {                                                           \
      ::doctest::detail::report(__FILE__, __LINE__, what, #expr);            \
      on_fail;                                                               \
    }                                                                        \
  } while (0)
#define CHECK(...) DOCTEST_ASSERT_("CHECK", (__VA_ARGS__), (void)0)
#define REQUIRE(...) DOCTEST_ASSERT_("REQUIRE", (__VA_ARGS__), throw ::doctest::detail::RequireFailed{})
#define FAIL(msg)                                                              \
  do {                                                                         \
    ::doctest::detail::report(__FILE__, __LINE__, "FAIL", msg);                \
    throw ::doctest::detail::RequireFailed{};                                  \
  } while (0)
#define CHECK_THROWS_AS(expr, ...)                                             \
  do {                                                                         \
    ++::doctest::detail::checks();                                             \
    bool doctest_ok_ = false;                                                  \
    try {                                                                      \
      (void)(expr);                                                            \
    } catch (const __VA_ARGS__&) {                                             \
      doctest_ok_ = true;                                                      \
    } catch (...) {                                                            \
    }                                                                          \
    if (!doctest_ok_) ::doctest::detail::report(__FILE__, __LINE__, "CHECK_THROWS_AS", #expr); \
  } while (0)
#define CHECK_NOTHROW(expr)                                                    \
  do {                                                                         \
    ++::doctest::detail::checks();                                             \
    try {                                                                      \
      (void)(expr);                                                            \
    } catch (...) {                                                            \
      ::doctest::detail::report(__FILE__, __LINE__, "CHECK_NOTHROW", #expr);   \
    }                                                                          \
  } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() { return ::doctest::detail::run_all(); }
#endif
