// doctest.h — a minimal stand-in for the doctest macros the reference's unit
// tests use (TEST_CASE, CHECK, CHECK_FALSE, REQUIRE, CHECK_THROWS_AS,
// doctest::Approx), so that those test files compile UNMODIFIED against the
// B200 drop-in headers (include/voxmc). Written for this repo (the real
// doctest is not vendored in the image); semantics follow doctest's
// documentation: Approx(x) == y iff |x - y| < eps * (scale + max(|x|, |y|)),
// default eps = 100 * FLT_EPSILON, scale = 1. With
// DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN the including file gets a main() that
// runs every test case (optionally only those whose name contains argv[1]),
// prints one line per failed check and a summary, and returns 1 on failure.
#pragma once

#include <cfloat>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <exception>
#include <functional>
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
  friend bool operator==(double lhs, const Approx& a) { return a.eq(lhs); }
  friend bool operator==(const Approx& a, double rhs) { return a.eq(rhs); }
  friend bool operator!=(double lhs, const Approx& a) { return !a.eq(lhs); }
  friend bool operator!=(const Approx& a, double rhs) { return !a.eq(rhs); }
  friend bool operator<=(double lhs, const Approx& a) { return lhs < a.value_ || a.eq(lhs); }
  friend bool operator>=(double lhs, const Approx& a) { return lhs > a.value_ || a.eq(lhs); }
  friend bool operator<(double lhs, const Approx& a) { return lhs < a.value_ && !a.eq(lhs); }
  friend bool operator>(double lhs, const Approx& a) { return lhs > a.value_ && !a.eq(lhs); }

 private:
  bool eq(double other) const {
    return std::fabs(other - value_) < eps_ * (scale_ + std::fmax(std::fabs(other), std::fabs(value_)));
  }
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

struct Registrar {
  Registrar(const char* name, const char* file, int line, void (*fn)()) {
    registry().push_back({name, file, line, fn});
  }
};

struct Stats {
  long checks = 0, failed = 0;
  bool case_failed = false;
};

inline Stats& stats() {
  static Stats s;
  return s;
}

struct RequireFailed {};

inline void report(bool ok, const char* kind, const char* expr, const char* file, int line, bool fatal) {
  Stats& s = stats();
  ++s.checks;
  if (ok) return;
  ++s.failed;
  s.case_failed = true;
  std::printf("%s:%d: FAILED %s( %s )\n", file, line, kind, expr);
  if (fatal) throw RequireFailed{};
}

inline int run(int argc, char** argv) {
  const char* filter = argc > 1 ? argv[1] : nullptr;
  int cases = 0, failed_cases = 0;
  for (const Case& c : registry()) {
    if (filter && !std::strstr(c.name, filter)) continue;
    ++cases;
    stats().case_failed = false;
    try {
      c.fn();
    } catch (const RequireFailed&) {
    } catch (const std::exception& e) {
      std::printf("%s:%d: test case \"%s\" threw %s\n", c.file, c.line, c.name, e.what());
      stats().case_failed = true;
    } catch (...) {
      std::printf("%s:%d: test case \"%s\" threw an unknown exception\n", c.file, c.line, c.name);
      stats().case_failed = true;
    }
    if (stats().case_failed) {
      ++failed_cases;
      std::printf("  in test case \"%s\"\n", c.name);
    }
  }
  std::printf("[doctest-shim] test cases: %d | %d passed | %d failed; checks: %ld | %ld failed\n", cases,
              cases - failed_cases, failed_cases, stats().checks, stats().failed);
  return failed_cases ? 1 : 0;
}

}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT2(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT2(a, b)
#define DOCTEST_TEST_CASE_IMPL(fn, name)                                                    \
  static void fn();                                                                        \
  static ::doctest::detail::Registrar DOCTEST_CAT(fn, _reg)(name, __FILE__, __LINE__, &fn); \
  static void fn()
#define TEST_CASE(name) DOCTEST_TEST_CASE_IMPL(DOCTEST_CAT(doctest_case_, __COUNTER__), name)

#define CHECK(...) ::doctest::detail::report(static_cast<bool>(__VA_ARGS__), "CHECK", #__VA_ARGS__, __FILE__, __LINE__, false)
#define CHECK_FALSE(...) \
  ::doctest::detail::report(!static_cast<bool>(__VA_ARGS__), "CHECK_FALSE", #__VA_ARGS__, __FILE__, __LINE__, false)
#define REQUIRE(...) ::doctest::detail::report(static_cast<bool>(__VA_ARGS__), "REQUIRE", #__VA_ARGS__, __FILE__, __LINE__, true)
#define CHECK_THROWS_AS(expr, ...)                                                                  \
  do {                                                                                              \
    bool doctest_ok_ = false;                                                                       \
    try {                                                                                           \
      static_cast<void>(expr);                                                                      \
    } catch (const __VA_ARGS__&) {                                                                  \
      doctest_ok_ = true;                                                                           \
    } catch (...) {                                                                                 \
    }                                                                                               \
    ::doctest::detail::report(doctest_ok_, "CHECK_THROWS_AS", #expr ", " #__VA_ARGS__, __FILE__, __LINE__, \
                              false);                                                               \
  } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main(int argc, char** argv) { return ::doctest::detail::run(argc, argv); }
#endif
