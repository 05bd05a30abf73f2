// TEST INFRASTRUCTURE ONLY — a minimal stand-in for the doctest macros the
// reference's unit tests use (/root/reference/proj/tests/*.cpp), so those
// tests compile UNMODIFIED against the reference sources built in
// oracle/_ref/ (doctest lives in the reference's git-ignored vendor/ and is
// absent from this image).  Supported: TEST_CASE, CHECK,
// REQUIRE, CHECK_THROWS, CHECK_THROWS_AS, CHECK_THROWS_WITH_AS,
// CHECK_NOTHROW, CAPTURE, doctest::Approx (doctest's comparison rule).
// Command line: -tc=<substr>[,<substr>] runs matching cases, -tce=<substr>
// excludes them, -ltc lists them.  Exit code = failed cases (capped at 255).
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <exception>
#include <functional>
#include <limits>
#include <sstream>
#include <string>
#include <vector>

namespace doctest {

class Approx {
 public:
  explicit Approx(double v) : v_(v) {}
  Approx& epsilon(double e) {
    eps_ = e;
    return *this;
  }
  Approx& scale(double s) {
    scale_ = s;
    return *this;
  }
  // doctest: |lhs - v| < eps * (scale + max(|lhs|, |v|))
  friend bool operator==(double lhs, const Approx& a) {
    return std::fabs(lhs - a.v_) < a.eps_ * (a.scale_ + std::max(std::fabs(lhs), std::fabs(a.v_)));
  }
  friend bool operator==(const Approx& a, double rhs) { return rhs == a; }
  friend bool operator!=(double lhs, const Approx& a) { return !(lhs == a); }
  friend bool operator!=(const Approx& a, double rhs) { return !(rhs == a); }
  friend bool operator<=(double lhs, const Approx& a) { return lhs < a.v_ || lhs == a; }
  friend bool operator>=(double lhs, const Approx& a) { return lhs > a.v_ || lhs == a; }
  friend bool operator<(double lhs, const Approx& a) { return lhs < a.v_ && lhs != a; }
  friend bool operator>(double lhs, const Approx& a) { return lhs > a.v_ && lhs != a; }

 private:
  double v_;
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
struct Reg {
  Reg(const char* name, const char* file, int line, void (*fn)()) { registry().push_back({name, file, line, fn}); }
};
struct RequireFailed {};
inline int& fails_in_case() {
  static int n = 0;
  return n;
}
inline long& checks_total() {
  static long n = 0;
  return n;
}
inline void fail(const char* file, int line, const char* macro, const char* expr, const std::string& extra = "") {
  ++fails_in_case();
  std::fprintf(stderr, "%s:%d: FAILED %s( %s )%s%s\n", file, line, macro, expr, extra.empty() ? "" : " ", extra.c_str());
}
inline bool split(const std::string& list, const std::string& name) {
  std::stringstream ss(list);
  std::string tok;
  while (std::getline(ss, tok, ','))
    if (!tok.empty() && name.find(tok) != std::string::npos) return true;
  return false;
}
inline int run(int argc, char** argv) {
  std::string inc, exc;
  bool list = false;
  for (int i = 1; i < argc; ++i) {
    std::string a = argv[i];
    if (a.rfind("-tc=", 0) == 0) inc = a.substr(4);
    else if (a.rfind("-tce=", 0) == 0) exc = a.substr(5);
    else if (a == "-ltc") list = true;
  }
  std::setvbuf(stdout, nullptr, _IOLBF, 0);
  int failed = 0, ran = 0;
  for (const Case& c : registry()) {
    const std::string nm = c.name;
    if (!inc.empty() && !split(inc, nm)) continue;
    if (!exc.empty() && split(exc, nm)) continue;
    if (list) {
      std::printf("%s\n", c.name);
      continue;
    }
    ++ran;
    fails_in_case() = 0;
    try {
      c.fn();
    } catch (const RequireFailed&) {
    } catch (const std::exception& e) {
      std::fprintf(stderr, "%s:%d: ERROR: test case threw: %s\n", c.file, c.line, e.what());
      ++fails_in_case();
    }
    if (fails_in_case()) {
      ++failed;
      std::printf("[FAIL] %s\n", c.name);
    } else {
      std::printf("[ ok ] %s\n", c.name);
    }
  }
  if (!list)
    std::printf("[doctest-shim] test cases: %d | %d passed | %d failed | checks: %ld\n", ran, ran - failed, failed,
                checks_total());
  return std::min(failed, 255);
}
}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define DOCTEST_CASE_IMPL(fn, name)                                                          \
  static void fn();                                                                          \
  static ::doctest::detail::Reg DOCTEST_CAT(fn, _reg)(name, __FILE__, __LINE__, &fn);        \
  static void fn()
#define TEST_CASE(name) DOCTEST_CASE_IMPL(DOCTEST_CAT(doctest_case_, __COUNTER__), name)

#define DOCTEST_CHECK_IMPL(macro, expr, on_fail)                                      \
  do {                                                                                \
    ++::doctest::detail::checks_total();                                              \
    bool doctest_ok_ = false;                                                         \
    try {                                                                             \
      doctest_ok_ = static_cast<bool>(expr);                                          \
    } catch (const std::exception& e) {                                               \
      ::doctest::detail::fail(__FILE__, __LINE__, macro, #expr, std::string("threw: ") + e.what()); \
      on_fail;                                                                        \
      break;                                                                          \
    }                                                                                 \
    if (!doctest_ok_) {                                                               \
      ::doctest::detail::fail(__FILE__, __LINE__, macro, #expr);                      \
      on_fail;                                                                        \
    }                                                                                 \
  } while (0)
#define CHECK(...) DOCTEST_CHECK_IMPL("CHECK", (__VA_ARGS__), (void)0)
#define REQUIRE(...) DOCTEST_CHECK_IMPL("REQUIRE", (__VA_ARGS__), throw ::doctest::detail::RequireFailed{})
#define CHECK_FALSE(...) DOCTEST_CHECK_IMPL("CHECK_FALSE", !(__VA_ARGS__), (void)0)

#define CHECK_THROWS_AS(expr, ...)                                                              \
  do {                                                                                          \
    ++::doctest::detail::checks_total();                                                        \
    bool doctest_ok_ = false;                                                                   \
    try {                                                                                       \
      (void)(expr);                                                                             \
    } catch (const __VA_ARGS__&) {                                                              \
      doctest_ok_ = true;                                                                       \
    } catch (...) {                                                                             \
    }                                                                                           \
    if (!doctest_ok_) ::doctest::detail::fail(__FILE__, __LINE__, "CHECK_THROWS_AS", #expr);    \
  } while (0)
#define CHECK_THROWS(expr)                                                                   \
  do {                                                                                       \
    ++::doctest::detail::checks_total();                                                     \
    bool doctest_ok_ = false;                                                                \
    try {                                                                                    \
      (void)(expr);                                                                          \
    } catch (...) {                                                                          \
      doctest_ok_ = true;                                                                    \
    }                                                                                        \
    if (!doctest_ok_) ::doctest::detail::fail(__FILE__, __LINE__, "CHECK_THROWS", #expr);    \
  } while (0)
#define CHECK_THROWS_WITH_AS(expr, msg, ...)                                                       \
  do {                                                                                             \
    ++::doctest::detail::checks_total();                                                           \
    bool doctest_ok_ = false;                                                                      \
    try {                                                                                          \
      (void)(expr);                                                                                \
    } catch (const __VA_ARGS__& e) {                                                               \
      doctest_ok_ = std::string(e.what()) == std::string(msg);                                     \
    } catch (...) {                                                                                \
    }                                                                                              \
    if (!doctest_ok_) ::doctest::detail::fail(__FILE__, __LINE__, "CHECK_THROWS_WITH_AS", #expr);  \
  } while (0)
#define CHECK_NOTHROW(expr)                                                                      \
  do {                                                                                           \
    ++::doctest::detail::checks_total();                                                         \
    try {                                                                                        \
      (void)(expr);                                                                              \
    } catch (...) {                                                                              \
      ::doctest::detail::fail(__FILE__, __LINE__, "CHECK_NOTHROW", #expr);                       \
    }                                                                                            \
  } while (0)
#define CAPTURE(x) (void)(x)
#define INFO(...) (void)0
#define MESSAGE(...) (void)0

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main(int argc, char** argv) { return ::doctest::detail::run(argc, argv); }
#endif
