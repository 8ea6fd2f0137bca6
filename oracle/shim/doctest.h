// ORACLE TEST INFRASTRUCTURE -- not product code.
//
// Single-header stand-in for the doctest subset the reference tests use
// (proj/tests/*.cpp; the real header is expected in proj/vendor, which is
// git-ignored and absent, proj/.gitignore:2).  Supported: TEST_CASE, SUBCASE
// (run inline; every SUBCASE in the reference tests is independent of its
// siblings), CHECK, REQUIRE, CHECK_THROWS_AS, CHECK_NOTHROW, CAPTURE (no-op),
// doctest::Approx with doctest's exact rule
//   |a - v| < eps * (scale + max(|a|, |v|)),  scale = 1, eps = 100 FLT_EPSILON.
// Also used by this repo's own C++ drop-in tests (tests/cpp/).
#pragma once

#include <algorithm>
#include <cfloat>
#include <cmath>
#include <cstdio>
#include <sstream>
#include <exception>
#include <functional>
#include <string>
#include <vector>

namespace doctest {

class Approx {
 public:
  explicit Approx(double v) : v_(v), eps_(static_cast<double>(FLT_EPSILON) * 100.0), scale_(1.0) {}
  Approx epsilon(double e) const {
    Approx a(*this);
    a.eps_ = e;
    return a;
  }
  Approx scale(double s) const {
    Approx a(*this);
    a.scale_ = s;
    return a;
  }
  friend bool operator==(double lhs, const Approx& rhs) {
    return std::fabs(lhs - rhs.v_) <
           rhs.eps_ * (rhs.scale_ + std::max(std::fabs(lhs), std::fabs(rhs.v_)));
  }
  friend bool operator==(const Approx& lhs, double rhs) { return rhs == lhs; }
  friend bool operator!=(double lhs, const Approx& rhs) { return !(lhs == rhs); }
  friend bool operator!=(const Approx& lhs, double rhs) { return !(rhs == lhs); }

 private:
  double v_, eps_, scale_;
};

namespace detail {

struct TestCase {
  const char* name;
  void (*fn)();
};

inline std::vector<TestCase>& registry() {
  static std::vector<TestCase> r;
  return r;
}

struct State {
  long asserts = 0, failed_asserts = 0;
  bool current_failed = false;
};

inline State& state() {
  static State s;
  return s;
}

struct Registrar {
  Registrar(const char* name, void (*fn)()) { registry().push_back({name, fn}); }
};

struct RequireFailed {};

inline void report(bool ok, const char* kind, const char* expr, const char* file, int line) {
  State& s = state();
  ++s.asserts;
  if (!ok) {
    ++s.failed_asserts;
    s.current_failed = true;
    std::fprintf(stderr, "%s:%d: ERROR: %s( %s ) is NOT correct!\n", file, line, kind, expr);
  }
}

inline int run_all() {
  int passed = 0, failed = 0;
  for (const TestCase& tc : registry()) {
    state().current_failed = false;
    try {
      tc.fn();
    } catch (const RequireFailed&) {
    } catch (const std::exception& e) {
      std::fprintf(stderr, "TEST CASE %s threw: %s\n", tc.name, e.what());
      state().current_failed = true;
    } catch (...) {
      std::fprintf(stderr, "TEST CASE %s threw an unknown exception\n", tc.name);
      state().current_failed = true;
    }
    if (state().current_failed) {
      ++failed;
      std::fprintf(stderr, "FAILED TEST CASE: %s\n", tc.name);
    } else {
      ++passed;
    }
  }
  std::printf("[doctest-shim] test cases: %d | %d passed | %d failed\n",
              passed + failed, passed, failed);
  std::printf("[doctest-shim] assertions: %ld | %ld passed | %ld failed\n", state().asserts,
              state().asserts - state().failed_asserts, state().failed_asserts);
  return failed == 0 ? 0 : 1;
}

}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define DOCTEST_TC_IMPL(fn, name)                                             \
  static void fn();                                                           \
  static ::doctest::detail::Registrar DOCTEST_CAT(fn, _reg)(name, &fn);       \
  static void fn()
#define TEST_CASE(name) DOCTEST_TC_IMPL(DOCTEST_CAT(doctest_tc_, __COUNTER__), name)
#define SUBCASE(name) if (true)
#define CAPTURE(x) ((void)0)
#define MESSAGE(msg)                                                    \
  do {                                                                  \
    std::ostringstream doctest_os_;                                     \
    doctest_os_ << msg;                                                 \
    std::printf("[doctest-shim] %s\n", doctest_os_.str().c_str());      \
  } while (0)
#define CHECK(...) ::doctest::detail::report(static_cast<bool>(__VA_ARGS__), "CHECK", #__VA_ARGS__, __FILE__, __LINE__)
#define REQUIRE(...)                                                                      \
  do {                                                                                    \
    const bool doctest_ok_ = static_cast<bool>(__VA_ARGS__);                              \
    ::doctest::detail::report(doctest_ok_, "REQUIRE", #__VA_ARGS__, __FILE__, __LINE__); \
    if (!doctest_ok_) throw ::doctest::detail::RequireFailed{};                          \
  } while (0)
#define CHECK_THROWS_AS(expr, ...)                                                   \
  do {                                                                               \
    bool doctest_ok_ = false;                                                        \
    try {                                                                            \
      (void)(expr);                                                                  \
    } catch (const __VA_ARGS__&) {                                                   \
      doctest_ok_ = true;                                                            \
    } catch (...) {                                                                  \
    }                                                                                \
    ::doctest::detail::report(doctest_ok_, "CHECK_THROWS_AS", #expr, __FILE__, __LINE__); \
  } while (0)
#define CHECK_NOTHROW(expr)                                                          \
  do {                                                                               \
    bool doctest_ok_ = true;                                                         \
    try {                                                                            \
      (void)(expr);                                                                  \
    } catch (...) {                                                                  \
      doctest_ok_ = false;                                                           \
    }                                                                                \
    ::doctest::detail::report(doctest_ok_, "CHECK_NOTHROW", #expr, __FILE__, __LINE__); \
  } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() { return ::doctest::detail::run_all(); }
#endif
