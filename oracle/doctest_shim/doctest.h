// oracle/doctest_shim/doctest.h — TEST INFRASTRUCTURE ONLY.
//
// A minimal stand-in for the doctest subset the reference's unit suites use
// (TEST_CASE, CHECK, CHECK_FALSE, REQUIRE, CHECK_THROWS_AS, CHECK_NOTHROW, FAIL,
// doctest::Approx(x).epsilon(e), DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN). doctest
// itself is not vendored with the reference and is absent from this image
// (SURVEY.md §0 finding 1). Approx follows doctest's rule
// |a - b| < eps * (1 + max(|a|, |b|)) with eps = 100 * FLT_EPSILON by default.
#pragma once

#include <cmath>
#include <cstdio>
#include <exception>
#include <functional>
#include <limits>
#include <string>
#include <vector>

namespace doctest {

class Approx {
 public:
  explicit Approx(double value) : value_(value) {}
  Approx& epsilon(double e) {
    eps_ = e;
    return *this;
  }
  Approx& scale(double s) {
    scale_ = s;
    return *this;
  }
  friend bool operator==(double lhs, const Approx& rhs) {
    return std::fabs(lhs - rhs.value_) <
           rhs.eps_ * (rhs.scale_ + std::fmax(std::fabs(lhs), std::fabs(rhs.value_)));
  }
  friend bool operator==(const Approx& lhs, double rhs) { return rhs == lhs; }
  friend bool operator!=(double lhs, const Approx& rhs) { return !(lhs == rhs); }
  friend bool operator!=(const Approx& lhs, double rhs) { return !(rhs == lhs); }

 private:
  double value_;
  double eps_ = static_cast<double>(std::numeric_limits<float>::epsilon()) * 100;
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
  Registrar(const char* name, const char* file, int line, void (*fn)()) { registry().push_back({name, file, line, fn}); }
};
struct State {
  int assertions = 0;
  int failed_assertions = 0;
  bool case_failed = false;
};
inline State& state() {
  static State s;
  return s;
}
struct RequireAbort {};
inline void report(bool ok, const char* kind, const char* expr, const char* file, int line) {
  ++state().assertions;
  if (ok) return;
  ++state().failed_assertions;
  state().case_failed = true;
  std::fprintf(stderr, "%s:%d: ERROR: %s( %s ) is NOT correct!\n", file, line, kind, expr);
}

}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define DOCTEST_TEST_CASE_IMPL(fn, name)                                                              \
  static void fn();                                                                                   \
  static const ::doctest::detail::Registrar DOCTEST_CAT(fn, _reg)(name, __FILE__, __LINE__, &fn); \
  static void fn()
#define TEST_CASE(name) DOCTEST_TEST_CASE_IMPL(DOCTEST_CAT(doctest_case_, __COUNTER__), name)

#define CHECK(...) ::doctest::detail::report(static_cast<bool>(__VA_ARGS__), "CHECK", #__VA_ARGS__, __FILE__, __LINE__)
#define CHECK_FALSE(...) \
  ::doctest::detail::report(!static_cast<bool>(__VA_ARGS__), "CHECK_FALSE", #__VA_ARGS__, __FILE__, __LINE__)
#define REQUIRE(...)                                                                                    \
  do {                                                                                                  \
    const bool doctest_ok_ = static_cast<bool>(__VA_ARGS__);                                            \
    ::doctest::detail::report(doctest_ok_, "REQUIRE", #__VA_ARGS__, __FILE__, __LINE__);                \
    if (!doctest_ok_) throw ::doctest::detail::RequireAbort{};                                          \
  } while (0)
#define CHECK_THROWS_AS(expr, ...)                                                                    \
  do {                                                                                                \
    bool doctest_ok_ = false;                                                                         \
    try {                                                                                             \
      (void)(expr);                                                                                   \
    } catch (const __VA_ARGS__&) {                                                                    \
      doctest_ok_ = true;                                                                             \
    } catch (...) {                                                                                   \
    }                                                                                                 \
    ::doctest::detail::report(doctest_ok_, "CHECK_THROWS_AS", #expr ", " #__VA_ARGS__, __FILE__, __LINE__); \
  } while (0)
#define CHECK_NOTHROW(expr)                                                               \
  do {                                                                                    \
    bool doctest_ok_ = true;                                                              \
    try {                                                                                 \
      (void)(expr);                                                                       \
    } catch (...) {                                                                       \
      doctest_ok_ = false;                                                                \
    }                                                                                     \
    ::doctest::detail::report(doctest_ok_, "CHECK_NOTHROW", #expr, __FILE__, __LINE__); \
  } while (0)
#define FAIL(msg)                                                                 \
  do {                                                                            \
    ::doctest::detail::report(false, "FAIL", #msg, __FILE__, __LINE__);          \
    throw ::doctest::detail::RequireAbort{};                                      \
  } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() {
  using namespace doctest::detail;
  int failed_cases = 0;
  for (const Case& c : registry()) {
    state().case_failed = false;
    try {
      c.fn();
    } catch (const RequireAbort&) {
    } catch (const std::exception& e) {
      state().case_failed = true;
      std::fprintf(stderr, "%s:%d: ERROR: test case \"%s\" threw: %s\n", c.file, c.line, c.name, e.what());
    } catch (...) {
      state().case_failed = true;
      std::fprintf(stderr, "%s:%d: ERROR: test case \"%s\" threw an unknown exception\n", c.file, c.line, c.name);
    }
    if (state().case_failed) {
      ++failed_cases;
      std::fprintf(stderr, "  -> FAILED: %s\n", c.name);
    }
  }
  std::printf("[doctest-shim] test cases: %zu | %zu passed | %d failed\n", registry().size(),
              registry().size() - size_t(failed_cases), failed_cases);
  std::printf("[doctest-shim] assertions: %d | %d passed | %d failed\n", state().assertions,
              state().assertions - state().failed_assertions, state().failed_assertions);
  return failed_cases ? 1 : 0;
}
#endif
