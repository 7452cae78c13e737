// Minimal doctest-compatible test shim (test infrastructure, self-written).
//
// The reference's unit suites (/root/reference/proj/tests/*.cpp) include
// "doctest.h", which is not vendored in /root/reference (proj/.gitignore:2).
// This header implements just the subset of the doctest surface those suites
// use -- TEST_CASE, SUBCASE (non-nested, re-entrant like doctest), CHECK,
// CHECK_FALSE, REQUIRE, CHECK_THROWS_AS, CHECK_THROWS_WITH_AS, CHECK_NOTHROW,
// FAIL, INFO and doctest::Approx -- so the suites can be compiled unchanged
// against either the reference objects (oracle/_ref) or the emoe compat
// library (the drop-in proof).  Define DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN in
// exactly one translation unit to get main().
#pragma once

#include <cmath>
#include <cstdio>
#include <functional>
#include <limits>
#include <sstream>
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
  bool matches(double other) const {
    // doctest: |a-b| < eps * (scale + max(|a|, |b|))
    return std::fabs(other - value_) <
           eps_ * (scale_ + std::fmax(std::fabs(other), std::fabs(value_)));
  }
  double value() const { return value_; }

 private:
  double value_;
  double eps_ = static_cast<double>(std::numeric_limits<float>::epsilon()) * 100.0;
  double scale_ = 1.0;
};

inline bool operator==(double lhs, const Approx& rhs) { return rhs.matches(lhs); }
inline bool operator==(const Approx& lhs, double rhs) { return lhs.matches(rhs); }
inline bool operator!=(double lhs, const Approx& rhs) { return !rhs.matches(lhs); }
inline bool operator!=(const Approx& lhs, double rhs) { return !lhs.matches(rhs); }
inline bool operator<=(double lhs, const Approx& rhs) { return lhs < rhs.value() || rhs.matches(lhs); }
inline bool operator>=(double lhs, const Approx& rhs) { return lhs > rhs.value() || rhs.matches(lhs); }

namespace shim {

struct TestCase {
  const char* name;
  const char* file;
  int line;
  void (*fn)();
};

struct RequireAbort {};

inline std::vector<TestCase>& registry() {
  static std::vector<TestCase> r;
  return r;
}

struct State {
  int failed_checks = 0;
  int passed_checks = 0;
  bool case_failed = false;
  int subcase_target = 0;
  int subcase_seen = 0;
  const char* current = "";
};

inline State& state() {
  static State s;
  return s;
}

inline int register_case(const char* name, const char* file, int line, void (*fn)()) {
  registry().push_back({name, file, line, fn});
  return 0;
}

inline void report(bool ok, const char* expr, const char* file, int line, const std::string& extra = {}) {
  State& s = state();
  if (ok) {
    ++s.passed_checks;
    return;
  }
  ++s.failed_checks;
  s.case_failed = true;
  std::fprintf(stderr, "%s:%d: FAILED in \"%s\": %s %s\n", file, line, s.current, expr, extra.c_str());
}

inline bool enter_subcase() {
  State& s = state();
  return s.subcase_seen++ == s.subcase_target;
}

template <typename... Args>
std::string concat(const Args&... args) {
  std::ostringstream out;
  (out << ... << args);
  return out.str();
}

inline int run_all() {
  State& s = state();
  int failed_cases = 0;
  for (const TestCase& tc : registry()) {
    s.current = tc.name;
    s.case_failed = false;
    // doctest semantics: each leaf SUBCASE runs the test body from the top
    int target = 0;
    while (true) {
      s.subcase_target = target;
      s.subcase_seen = 0;
      try {
        tc.fn();
      } catch (const RequireAbort&) {
      } catch (const std::exception& e) {
        report(false, "unexpected exception", tc.file, tc.line, e.what());
      }
      if (++target >= s.subcase_seen) break;
    }
    if (s.case_failed) ++failed_cases;
  }
  std::printf("[doctest-shim] test cases: %zu | %zu passed | %d failed\n", registry().size(),
              registry().size() - static_cast<size_t>(failed_cases), failed_cases);
  std::printf("[doctest-shim] assertions: %d | %d passed | %d failed\n",
              s.passed_checks + s.failed_checks, s.passed_checks, s.failed_checks);
  return failed_cases == 0 ? 0 : 1;
}

}  // namespace shim
}  // namespace doctest

#define DOCTEST_SHIM_CAT2(a, b) a##b
#define DOCTEST_SHIM_CAT(a, b) DOCTEST_SHIM_CAT2(a, b)

#define DOCTEST_SHIM_TEST_CASE_IMPL(fn, name)                                              \
  static void fn();                                                                         \
  static const int DOCTEST_SHIM_CAT(fn, _reg) =                                             \
      doctest::shim::register_case(name, __FILE__, __LINE__, &fn);                          \
  static void fn()
#define TEST_CASE(name) DOCTEST_SHIM_TEST_CASE_IMPL(DOCTEST_SHIM_CAT(doctest_shim_case_, __COUNTER__), name)

#define SUBCASE(name) if (doctest::shim::enter_subcase())

#define CHECK(...) doctest::shim::report(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__)
#define CHECK_FALSE(...) doctest::shim::report(!static_cast<bool>(__VA_ARGS__), "!(" #__VA_ARGS__ ")", __FILE__, __LINE__)
#define REQUIRE(...)                                                                       \
  do {                                                                                      \
    bool doctest_shim_ok = static_cast<bool>(__VA_ARGS__);                                  \
    doctest::shim::report(doctest_shim_ok, #__VA_ARGS__, __FILE__, __LINE__);               \
    if (!doctest_shim_ok) throw doctest::shim::RequireAbort{};                              \
  } while (0)
#define REQUIRE_FALSE(...) REQUIRE(!(__VA_ARGS__))

#define CHECK_THROWS_AS(expr, exc)                                                         \
  do {                                                                                      \
    bool doctest_shim_ok = false;                                                           \
    try {                                                                                   \
      static_cast<void>(expr);                                                              \
    } catch (const exc&) {                                                                  \
      doctest_shim_ok = true;                                                               \
    } catch (...) {                                                                         \
    }                                                                                       \
    doctest::shim::report(doctest_shim_ok, "throws " #exc ": " #expr, __FILE__, __LINE__);  \
  } while (0)

#define CHECK_THROWS_WITH_AS(expr, msg, exc)                                               \
  do {                                                                                      \
    bool doctest_shim_ok = false;                                                           \
    try {                                                                                   \
      static_cast<void>(expr);                                                              \
    } catch (const exc& e) {                                                                \
      doctest_shim_ok = std::string(e.what()) == std::string(msg);                          \
    } catch (...) {                                                                         \
    }                                                                                       \
    doctest::shim::report(doctest_shim_ok, "throws-with " #exc ": " #expr, __FILE__, __LINE__); \
  } while (0)

#define CHECK_NOTHROW(expr)                                                                \
  do {                                                                                      \
    bool doctest_shim_ok = true;                                                            \
    try {                                                                                   \
      static_cast<void>(expr);                                                              \
    } catch (...) {                                                                         \
      doctest_shim_ok = false;                                                              \
    }                                                                                       \
    doctest::shim::report(doctest_shim_ok, "nothrow: " #expr, __FILE__, __LINE__);          \
  } while (0)

#define FAIL(...)                                                                          \
  do {                                                                                      \
    doctest::shim::report(false, "FAIL", __FILE__, __LINE__, doctest::shim::concat(__VA_ARGS__)); \
    throw doctest::shim::RequireAbort{};                                                    \
  } while (0)

#define INFO(...) static_cast<void>(0)
#define CAPTURE(...) static_cast<void>(0)
#define MESSAGE(...) static_cast<void>(0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() { return doctest::shim::run_all(); }
#endif
