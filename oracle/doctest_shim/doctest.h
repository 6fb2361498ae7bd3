// Minimal doctest-compatible runner: TEST INFRASTRUCTURE ONLY.
//
// The reference's unit tests (/root/reference/proj/tests/*.cpp) include
// <doctest.h>, which is git-ignored upstream (proj/.gitignore:2) and absent
// here. This header implements the subset they use (TEST_CASE, CHECK,
// CHECK_FALSE, CHECK_THROWS, CHECK_THROWS_AS, CHECK_NOTHROW, REQUIRE,
// doctest::Approx with .epsilon) so the UNMODIFIED test files compile
// against oracle/_ref/libphmat_ref.so (recipe: oracle/ref_build.sh) and the
// shimmed reference build is checked by the reference's own suite.
#pragma once

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <exception>
#include <functional>
#include <map>
#include <set>
#include <unordered_map>
#include <unordered_set>
#include <sstream>
#include <string>
#include <vector>

namespace doctest {

struct Approx {
  double value, eps = static_cast<double>(1.19209290e-07f) * 100.0, scale = 1.0;  // doctest default
  explicit Approx(double v) : value(v) {}
  Approx& epsilon(double e) {
    eps = e;
    return *this;
  }
  Approx& scale_(double s) {
    scale = s;
    return *this;
  }
  bool eq(double x) const {
    // doctest: |a-b| < eps * (scale + max(|a|, |b|))
    return std::fabs(x - value) < eps * (scale + std::max(std::fabs(x), std::fabs(value)));
  }
};
inline bool operator==(double x, const Approx& a) { return a.eq(x); }
inline bool operator==(const Approx& a, double x) { return a.eq(x); }
inline bool operator!=(double x, const Approx& a) { return !a.eq(x); }
inline bool operator!=(const Approx& a, double x) { return !a.eq(x); }
inline bool operator<=(double x, const Approx& a) { return x < a.value || a.eq(x); }
inline bool operator>=(double x, const Approx& a) { return x > a.value || a.eq(x); }
inline bool operator<(double x, const Approx& a) { return x < a.value && !a.eq(x); }
inline bool operator>(double x, const Approx& a) { return x > a.value && !a.eq(x); }

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
struct Reg {
  Reg(const char* name, void (*fn)(), const char* file, int line) { registry().push_back({name, fn, file, line}); }
};
struct RequireFailed {};
inline int& failures() {
  static int f = 0;
  return f;
}
inline int& assertions() {
  static int a = 0;
  return a;
}
inline void fail(const char* file, int line, const char* what) {
  ++failures();
  std::fprintf(stderr, "%s:%d: FAILED: %s\n", file, line, what);
}
}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define DOCTEST_TC_IMPL(fn, name)                                                          \
  static void fn();                                                                        \
  static doctest::detail::Reg DOCTEST_CAT(fn, _reg)(name, &fn, __FILE__, __LINE__);        \
  static void fn()
#define TEST_CASE(name) DOCTEST_TC_IMPL(DOCTEST_CAT(doctest_case_, __LINE__), name)

#define DOCTEST_ASSERT_(expr, fatal)                                        \
  do {                                                                      \
    ++doctest::detail::assertions();                                        \
    bool ok_ = false;                                                       \
    try {                                                                   \
      ok_ = static_cast<bool>(expr);                                        \
    } catch (const std::exception& e_) {                                    \
      doctest::detail::fail(__FILE__, __LINE__, e_.what());                 \
      if (fatal) throw doctest::detail::RequireFailed{};                    \
      break;                                                                \
    }                                                                       \
    if (!ok_) {                                                             \
      doctest::detail::fail(__FILE__, __LINE__, #expr);                     \
      if (fatal) throw doctest::detail::RequireFailed{};                    \
    }                                                                       \
  } while (0)
#define CHECK(...) DOCTEST_ASSERT_((__VA_ARGS__), false)
#define REQUIRE(...) DOCTEST_ASSERT_((__VA_ARGS__), true)
#define CHECK_FALSE(...) DOCTEST_ASSERT_(!(__VA_ARGS__), false)
#define REQUIRE_FALSE(...) DOCTEST_ASSERT_(!(__VA_ARGS__), true)
#define CHECK_THROWS(...)                                                     \
  do {                                                                        \
    ++doctest::detail::assertions();                                          \
    bool threw_ = false;                                                      \
    try {                                                                     \
      (void)(__VA_ARGS__);                                                    \
    } catch (...) {                                                           \
      threw_ = true;                                                          \
    }                                                                         \
    if (!threw_) doctest::detail::fail(__FILE__, __LINE__, "CHECK_THROWS " #__VA_ARGS__); \
  } while (0)
#define CHECK_THROWS_AS(expr, type)                                           \
  do {                                                                        \
    ++doctest::detail::assertions();                                          \
    bool ok_ = false;                                                         \
    try {                                                                     \
      (void)(expr);                                                           \
    } catch (const type&) {                                                   \
      ok_ = true;                                                             \
    } catch (...) {                                                           \
    }                                                                         \
    if (!ok_) doctest::detail::fail(__FILE__, __LINE__, "CHECK_THROWS_AS " #expr " " #type); \
  } while (0)
#define CHECK_NOTHROW(...)                                                    \
  do {                                                                        \
    ++doctest::detail::assertions();                                          \
    try {                                                                     \
      (void)(__VA_ARGS__);                                                    \
    } catch (const std::exception& e_) {                                      \
      doctest::detail::fail(__FILE__, __LINE__, e_.what());                   \
    }                                                                         \
  } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main(int argc, char** argv) {
  const char* filter = argc > 1 ? argv[1] : nullptr;
  int cases = 0, failed_cases = 0;
  for (const auto& c : doctest::detail::registry()) {
    if (filter && std::string(c.name).find(filter) == std::string::npos) continue;
    ++cases;
    const int before = doctest::detail::failures();
    try {
      c.fn();
    } catch (const doctest::detail::RequireFailed&) {
    } catch (const std::exception& e) {
      doctest::detail::fail(c.file, c.line, e.what());
    } catch (...) {
      doctest::detail::fail(c.file, c.line, "unknown exception");
    }
    const bool bad = doctest::detail::failures() != before;
    failed_cases += bad ? 1 : 0;
    std::printf("[%s] %s\n", bad ? "FAIL" : " ok ", c.name);
  }
  std::printf("test cases: %d | %d passed | %d failed | assertions: %d | %d failed\n", cases,
              cases - failed_cases, failed_cases, doctest::detail::assertions(), doctest::detail::failures());
  return failed_cases ? 1 : 0;
}
#endif
