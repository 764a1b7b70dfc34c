// doctest-lite — TEST INFRASTRUCTURE ONLY.  The subset of doctest that the
// reference's test suites use (TEST_CASE, CHECK, REQUIRE, CHECK_THROWS_AS,
// CHECK_THROWS_WITH_AS with doctest::Contains, doctest::Approx, FAIL), so the
// reference's own tests run against its sources compiled here.  Define
// DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN in exactly one translation unit.
#pragma once

#include <cmath>
#include <cstdio>
#include <exception>
#include <functional>
#include <limits>
#include <sstream>
#include <string>
#include <vector>

namespace doctest {

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
  Registrar(const char* name, const char* file, int line, void (*fn)()) { registry().push_back({name, file, line, fn}); }
};

struct State {
  int checks = 0, failed_checks = 0;
  bool current_failed = false;
};
inline State& state() {
  static State s;
  return s;
}

struct RequireFailure {};

inline void report(bool ok, const char* expr, const char* file, int line, bool require) {
  ++state().checks;
  if (ok) return;
  ++state().failed_checks;
  state().current_failed = true;
  std::fprintf(stderr, "%s:%d: %s( %s ) FAILED\n", file, line, require ? "REQUIRE" : "CHECK", expr);
  if (require) throw RequireFailure{};
}

class Approx {
 public:
  explicit Approx(double v) : v_(v), eps_(std::numeric_limits<float>::epsilon() * 100), scale_(1.0) {}
  Approx& epsilon(double e) {
    eps_ = e;
    return *this;
  }
  Approx& scale(double s) {
    scale_ = s;
    return *this;
  }
  bool eq(double x) const {
    return std::abs(x - v_) < eps_ * (scale_ + std::max(std::abs(x), std::abs(v_)));
  }
  friend bool operator==(double x, const Approx& a) { return a.eq(x); }
  friend bool operator==(const Approx& a, double x) { return a.eq(x); }
  friend bool operator!=(double x, const Approx& a) { return !a.eq(x); }
  friend bool operator!=(const Approx& a, double x) { return !a.eq(x); }
  friend bool operator<=(double x, const Approx& a) { return x < a.v_ || a.eq(x); }
  friend bool operator>=(double x, const Approx& a) { return x > a.v_ || a.eq(x); }
  friend bool operator<=(const Approx& a, double x) { return a.v_ < x || a.eq(x); }
  friend bool operator>=(const Approx& a, double x) { return a.v_ > x || a.eq(x); }

 private:
  double v_, eps_, scale_;
};

struct Contains {
  std::string s;
  explicit Contains(const char* c) : s(c) {}
  explicit Contains(std::string c) : s(std::move(c)) {}
  bool matches(const std::string& w) const { return w.find(s) != std::string::npos; }
};

inline Contains as_contains(const Contains& c) { return c; }
inline Contains as_contains(const char* c) { return Contains(c); }
inline Contains as_contains(const std::string& c) { return Contains(c); }

inline int run_all() {
  int failed_cases = 0;
  for (const TestCase& t : registry()) {
    state().current_failed = false;
    try {
      t.fn();
    } catch (const RequireFailure&) {
    } catch (const std::exception& e) {
      std::fprintf(stderr, "%s:%d: TEST CASE '%s' threw: %s\n", t.file, t.line, t.name, e.what());
      state().current_failed = true;
    } catch (...) {
      std::fprintf(stderr, "%s:%d: TEST CASE '%s' threw an unknown exception\n", t.file, t.line, t.name);
      state().current_failed = true;
    }
    if (state().current_failed) {
      ++failed_cases;
      std::fprintf(stderr, "  -> test case FAILED: %s\n", t.name);
    }
  }
  std::printf("[doctest-lite] test cases: %zu | %zu passed | %d failed | checks: %d, %d failed\n",
              registry().size(), registry().size() - size_t(failed_cases), failed_cases, state().checks,
              state().failed_checks);
  return failed_cases ? 1 : 0;
}

}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define DOCTEST_TC(fn, name)                                                                         \
  static void fn();                                                                                  \
  static ::doctest::Registrar DOCTEST_CAT(fn, _reg)(name, __FILE__, __LINE__, &fn);                 \
  static void fn()
#define TEST_CASE(name) DOCTEST_TC(DOCTEST_CAT(doctest_case_, __COUNTER__), name)

#define CHECK(...) ::doctest::report(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, false)
#define REQUIRE(...) ::doctest::report(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, true)
#define CHECK_FALSE(...) ::doctest::report(!static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, false)
#define FAIL(msg)                                                              \
  do {                                                                         \
    std::ostringstream doctest_os_;                                            \
    doctest_os_ << msg;                                                        \
    ::doctest::report(false, doctest_os_.str().c_str(), __FILE__, __LINE__, true); \
  } while (0)
#define CHECK_THROWS_AS(expr, ...)                                                   \
  do {                                                                               \
    bool doctest_ok_ = false;                                                        \
    try {                                                                            \
      static_cast<void>(expr);                                                       \
    } catch (const __VA_ARGS__&) {                                                   \
      doctest_ok_ = true;                                                            \
    } catch (...) {                                                                  \
    }                                                                                \
    ::doctest::report(doctest_ok_, "THROWS_AS(" #expr ")", __FILE__, __LINE__, false); \
  } while (0)
#define CHECK_THROWS_WITH_AS(expr, with, ...)                                                 \
  do {                                                                                        \
    bool doctest_ok_ = false;                                                                 \
    try {                                                                                     \
      static_cast<void>(expr);                                                                \
    } catch (const __VA_ARGS__& e) {                                                          \
      doctest_ok_ = ::doctest::as_contains(with).matches(e.what());                              \
    } catch (...) {                                                                           \
    }                                                                                         \
    ::doctest::report(doctest_ok_, "THROWS_WITH_AS(" #expr ")", __FILE__, __LINE__, false);   \
  } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() { return ::doctest::run_all(); }
#endif
