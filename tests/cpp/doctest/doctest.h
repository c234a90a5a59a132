// Minimal doctest-compatible test harness (test infrastructure only).
//
// Enough of the doctest API (https://github.com/doctest/doctest, the
// framework the reference's tests are written in; not vendored here) to
// build the reference's tests/test_kernels.cpp, test_nonlin.cpp and
// test_bitcore.cpp UNCHANGED against the drop-in headers:
//   TEST_CASE, SUBCASE (one nesting level: the case is re-run once per
//   subcase), CHECK, CHECK_FALSE, CHECK_THROWS_AS, REQUIRE, doctest::Approx
//   (published semantics: |a - b| < eps * (scale + max(|a|, |b|)), default
//   eps = 100 * FLT_EPSILON, scale 1), and DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN.
// Failures print file:line and the expression; main() returns 1 on any.
#ifndef QK_DOCTEST_SHIM_H_
#define QK_DOCTEST_SHIM_H_

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <limits>
#include <string>
#include <vector>

namespace doctest {

class Approx {
 public:
  explicit Approx(double value)
      : value_(value), epsilon_(static_cast<double>(std::numeric_limits<float>::epsilon()) * 100),
        scale_(1.0) {}
  Approx& epsilon(double e) {
    epsilon_ = e;
    return *this;
  }
  Approx& scale(double s) {
    scale_ = s;
    return *this;
  }
  bool matches(double lhs) const {
    return std::fabs(lhs - value_) <
           epsilon_ * (scale_ + std::max(std::fabs(lhs), std::fabs(value_)));
  }
  double value() const { return value_; }

 private:
  double value_, epsilon_, scale_;
};

template <typename T>
bool operator==(const T& lhs, const Approx& rhs) { return rhs.matches(static_cast<double>(lhs)); }
template <typename T>
bool operator==(const Approx& lhs, const T& rhs) { return lhs.matches(static_cast<double>(rhs)); }
template <typename T>
bool operator!=(const T& lhs, const Approx& rhs) { return !rhs.matches(static_cast<double>(lhs)); }
template <typename T>
bool operator!=(const Approx& lhs, const T& rhs) { return !lhs.matches(static_cast<double>(rhs)); }
template <typename T>
bool operator<=(const T& lhs, const Approx& rhs) {
  return static_cast<double>(lhs) < rhs.value() || rhs.matches(static_cast<double>(lhs));
}
template <typename T>
bool operator>=(const T& lhs, const Approx& rhs) {
  return static_cast<double>(lhs) > rhs.value() || rhs.matches(static_cast<double>(lhs));
}

namespace shim {

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
  long long checks = 0;
  long long failures = 0;
  int case_failures = 0;
  int sub_target = 0;  // which SUBCASE of the current run executes
  int sub_seen = 0;    // SUBCASEs met so far in this run
  const char* current = "";
  const char* subcase = nullptr;
};
inline State& state() {
  static State s;
  return s;
}

struct Registrar {
  Registrar(const char* name, const char* file, int line, void (*fn)()) {
    registry().push_back({name, file, line, fn});
  }
};

inline void report(bool ok, const char* what, const char* expr, const char* file, int line) {
  State& s = state();
  ++s.checks;
  if (ok) return;
  ++s.failures;
  ++s.case_failures;
  if (s.case_failures <= 10) {
    std::fprintf(stderr, "%s:%d: FAILED %s( %s ) in TEST_CASE \"%s\"%s%s\n", file, line, what,
                 expr, s.current, s.subcase ? " / SUBCASE " : "", s.subcase ? s.subcase : "");
  }
}

struct Subcase {
  bool active;
  explicit Subcase(const char* name) {
    State& s = state();
    active = s.sub_seen++ == s.sub_target;
    if (active) s.subcase = name;
  }
  explicit operator bool() const { return active; }
};

inline int run_all() {
  State& s = state();
  int failed_cases = 0;
  for (const TestCase& tc : registry()) {
    s.current = tc.name;
    s.case_failures = 0;
    // run once per SUBCASE (or once when there is none)
    s.sub_target = 0;
    for (;;) {
      s.sub_seen = 0;
      s.subcase = nullptr;
      try {
        tc.fn();
      } catch (const std::exception& e) {
        report(false, "TEST_CASE", e.what(), tc.file, tc.line);
      } catch (...) {
        report(false, "TEST_CASE", "unknown exception", tc.file, tc.line);
      }
      if (++s.sub_target >= s.sub_seen) break;
    }
    if (s.case_failures) ++failed_cases;
  }
  std::printf("[doctest shim] test cases: %zu | %zu passed | %d failed\n", registry().size(),
              registry().size() - static_cast<size_t>(failed_cases), failed_cases);
  std::printf("[doctest shim] assertions: %lld | %lld passed | %lld failed\n", s.checks,
              s.checks - s.failures, s.failures);
  return failed_cases ? 1 : 0;
}

}  // namespace shim
}  // namespace doctest

#define QK_DT_CAT2(a, b) a##b
#define QK_DT_CAT(a, b) QK_DT_CAT2(a, b)
#define QK_DT_TEST_CASE_IMPL(fn, name)                                                  \
  static void fn();                                                                     \
  static ::doctest::shim::Registrar QK_DT_CAT(fn, _reg)(name, __FILE__, __LINE__, &fn); \
  static void fn()
#define TEST_CASE(name) QK_DT_TEST_CASE_IMPL(QK_DT_CAT(qk_dt_case_, __LINE__), name)
#define SUBCASE(name) if (const ::doctest::shim::Subcase QK_DT_CAT(qk_dt_sub_, __LINE__){name})
#define CHECK(...) ::doctest::shim::report(static_cast<bool>(__VA_ARGS__), "CHECK", #__VA_ARGS__, __FILE__, __LINE__)
#define REQUIRE(...)                                                                    \
  do {                                                                                  \
    const bool qk_dt_ok_ = static_cast<bool>(__VA_ARGS__);                              \
    ::doctest::shim::report(qk_dt_ok_, "REQUIRE", #__VA_ARGS__, __FILE__, __LINE__);    \
    if (!qk_dt_ok_) return;                                                             \
  } while (0)
#define CHECK_FALSE(...) ::doctest::shim::report(!static_cast<bool>(__VA_ARGS__), "CHECK_FALSE", #__VA_ARGS__, __FILE__, __LINE__)
#define CHECK_THROWS_AS(expr, ...)                                                      \
  do {                                                                                  \
    bool qk_dt_ok_ = false;                                                             \
    try {                                                                               \
      static_cast<void>(expr);                                                          \
    } catch (const __VA_ARGS__&) {                                                      \
      qk_dt_ok_ = true;                                                                 \
    } catch (...) {                                                                     \
    }                                                                                   \
    ::doctest::shim::report(qk_dt_ok_, "CHECK_THROWS_AS", #expr, __FILE__, __LINE__);   \
  } while (0)
#define CHECK_NOTHROW(expr)                                                             \
  do {                                                                                  \
    bool qk_dt_ok_ = true;                                                              \
    try {                                                                               \
      static_cast<void>(expr);                                                          \
    } catch (...) {                                                                     \
      qk_dt_ok_ = false;                                                                \
    }                                                                                   \
    ::doctest::shim::report(qk_dt_ok_, "CHECK_NOTHROW", #expr, __FILE__, __LINE__);     \
  } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() { return ::doctest::shim::run_all(); }
#endif

#endif  // QK_DOCTEST_SHIM_H_
