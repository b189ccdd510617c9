// Minimal doctest-compatible shim -- TEST INFRASTRUCTURE ONLY.
//
// The reference's unit suites (/root/reference/proj/tests/test_*.cpp) are
// written against doctest, which is not vendored in the reference mount and
// not installed here.  This shim implements exactly the subset they use:
// TEST_CASE, CHECK, REQUIRE, CHECK_THROWS_AS, CHECK_THROWS_WITH_AS,
// doctest::Approx(.epsilon) and doctest::Contains.
#pragma once
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <exception>
#include <limits>
#include <string>
#include <vector>

namespace doctest {

struct Approx {
  explicit Approx(double v) : value(v) {}
  Approx& epsilon(double e) { eps = e; return *this; }
  Approx& scale(double s) { scl = s; return *this; }
  double value;
  double eps = static_cast<double>(std::numeric_limits<float>::epsilon()) * 100;
  double scl = 1.0;
};
inline bool approx_eq(double lhs, const Approx& a) {
  return std::fabs(lhs - a.value) <
         a.eps * (a.scl + std::max(std::fabs(lhs), std::fabs(a.value)));
}
template <typename T> bool operator==(const T& l, const Approx& a) { return approx_eq(double(l), a); }
template <typename T> bool operator==(const Approx& a, const T& r) { return approx_eq(double(r), a); }
template <typename T> bool operator!=(const T& l, const Approx& a) { return !approx_eq(double(l), a); }
template <typename T> bool operator!=(const Approx& a, const T& r) { return !approx_eq(double(r), a); }
template <typename T> bool operator<=(const T& l, const Approx& a) { return double(l) < a.value || approx_eq(double(l), a); }
template <typename T> bool operator>=(const T& l, const Approx& a) { return double(l) > a.value || approx_eq(double(l), a); }
template <typename T> bool operator<=(const Approx& a, const T& r) { return a.value < double(r) || approx_eq(double(r), a); }
template <typename T> bool operator>=(const Approx& a, const T& r) { return a.value > double(r) || approx_eq(double(r), a); }

struct Contains {
  explicit Contains(const char* s) : needle(s) {}
  std::string needle;
};

namespace detail {
struct TestCase {
  void (*fn)();
  const char* name;
  const char* file;
  int line;
};
inline std::vector<TestCase>& registry() {
  static std::vector<TestCase> r;
  return r;
}
struct Registrar {
  Registrar(void (*fn)(), const char* name, const char* file, int line) {
    registry().push_back({fn, name, file, line});
  }
};
struct RequireAbort {};
inline int& failures() { static int f = 0; return f; }
inline int& checks() { static int c = 0; return c; }
inline void fail(const char* file, int line, const std::string& what) {
  ++failures();
  std::fprintf(stderr, "%s:%d: FAILED: %s\n", file, line, what.c_str());
}
inline bool matches(const std::string& msg, const Contains& c) {
  return msg.find(c.needle) != std::string::npos;
}
inline bool matches(const std::string& msg, const char* exact) { return msg == exact; }
}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT2(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT2(a, b)
#define DOCTEST_TC_IMPL(fn, name)                                              \
  static void fn();                                                            \
  static ::doctest::detail::Registrar DOCTEST_CAT(fn, _reg)(fn, name, __FILE__, \
                                                            __LINE__);         \
  static void fn()
#define TEST_CASE(name) DOCTEST_TC_IMPL(DOCTEST_CAT(doctest_tc_, __LINE__), name)

#define DOCTEST_ASSERT_IMPL(expr, is_require)                                \
  do {                                                                       \
    ++::doctest::detail::checks();                                           \
    bool doctest_ok_ = false;                                                \
    try {                                                                    \
      doctest_ok_ = static_cast<bool>(expr);                                 \
    } catch (const std::exception& e) {                                      \
      ::doctest::detail::fail(__FILE__, __LINE__,                            \
                              std::string(#expr " threw: ") + e.what());     \
      if (is_require) throw ::doctest::detail::RequireAbort{};               \
      break;                                                                 \
    }                                                                        \
    if (!doctest_ok_) {                                                      \
      ::doctest::detail::fail(__FILE__, __LINE__, #expr);                    \
      if (is_require) throw ::doctest::detail::RequireAbort{};               \
    }                                                                        \
  } while (0)
#define CHECK(...) DOCTEST_ASSERT_IMPL((__VA_ARGS__), false)
#define REQUIRE(...) DOCTEST_ASSERT_IMPL((__VA_ARGS__), true)

#define CHECK_THROWS_AS(expr, ...)                                            \
  do {                                                                        \
    ++::doctest::detail::checks();                                            \
    try {                                                                     \
      static_cast<void>(expr);                                                \
      ::doctest::detail::fail(__FILE__, __LINE__, #expr " did not throw");    \
    } catch (const __VA_ARGS__&) {                                            \
    } catch (...) {                                                           \
      ::doctest::detail::fail(__FILE__, __LINE__,                             \
                              #expr " threw the wrong type");                 \
    }                                                                         \
  } while (0)

#define CHECK_THROWS_WITH_AS(expr, matcher, ...)                              \
  do {                                                                        \
    ++::doctest::detail::checks();                                            \
    try {                                                                     \
      static_cast<void>(expr);                                                \
      ::doctest::detail::fail(__FILE__, __LINE__, #expr " did not throw");    \
    } catch (const __VA_ARGS__& e) {                                          \
      if (!::doctest::detail::matches(e.what(), matcher))                     \
        ::doctest::detail::fail(__FILE__, __LINE__,                           \
                                std::string(#expr " message: ") + e.what()); \
    } catch (...) {                                                           \
      ::doctest::detail::fail(__FILE__, __LINE__,                             \
                              #expr " threw the wrong type");                 \
    }                                                                         \
  } while (0)

#ifdef DOCTEST_SHIM_MAIN
#include <cstring>
int main(int argc, char** argv) {
  int failed_cases = 0, run = 0;
  for (const auto& tc : ::doctest::detail::registry()) {
    if (argc > 1 && std::strstr(tc.name, argv[1]) == nullptr) continue;
    ++run;
    const int before = ::doctest::detail::failures();
    try {
      tc.fn();
    } catch (const ::doctest::detail::RequireAbort&) {
    } catch (const std::exception& e) {
      ::doctest::detail::fail(tc.file, tc.line,
                              std::string("uncaught exception: ") + e.what());
    }
    if (::doctest::detail::failures() != before) {
      ++failed_cases;
      std::fprintf(stderr, "  in TEST_CASE \"%s\"\n", tc.name);
    }
  }
  std::printf("[doctest-shim] test cases: %d | passed: %d | failed: %d | assertions: %d\n",
              run, run - failed_cases, failed_cases, ::doctest::detail::checks());
  return failed_cases ? 1 : 0;
}
#endif
