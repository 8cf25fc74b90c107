// TEST INFRASTRUCTURE ONLY. A minimal stand-in for doctest (absent from this
// image) providing exactly the subset the reference's unit suites use:
// TEST_SUITE_BEGIN/END, TEST_CASE, CHECK, CHECK_FALSE, REQUIRE,
// REQUIRE_MESSAGE, CHECK_THROWS_AS, CHECK_THROWS_WITH_AS, doctest::Approx
// (.epsilon/.scale, doctest's comparison rule) and doctest::Contains.
// Lets the reference's own tests run unmodified against the B200 shim.
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
  friend bool operator==(double lhs, const Approx& r) {
    return std::fabs(lhs - r.v_) < r.eps_ * (r.scale_ + std::max(std::fabs(lhs), std::fabs(r.v_)));
  }
  friend bool operator==(const Approx& r, double lhs) { return lhs == r; }
  friend bool operator!=(double lhs, const Approx& r) { return !(lhs == r); }
  friend bool operator!=(const Approx& r, double lhs) { return !(lhs == r); }

 private:
  double v_;
  double eps_ = static_cast<double>(std::numeric_limits<float>::epsilon()) * 100;
  double scale_ = 1.0;
};

struct Contains {
  std::string s;
  explicit Contains(const char* x) : s(x) {}
  bool matches(const std::string& m) const { return m.find(s) != std::string::npos; }
};

namespace detail {
struct Require {};
struct Case {
  std::string suite, name;
  void (*fn)();
};
inline std::vector<Case>& cases() {
  static std::vector<Case> c;
  return c;
}
inline std::string& suite() {
  static std::string s;
  return s;
}
inline int& failures() {
  static int f = 0;
  return f;
}
inline int reg(const char* name, void (*fn)()) {
  cases().push_back({suite(), name, fn});
  return 0;
}
inline int set_suite(const char* s) {
  suite() = s;
  return 0;
}
inline void fail(const char* file, int line, const char* what, const std::string& extra = "") {
  ++failures();
  std::fprintf(stderr, "%s:%d: FAILED: %s %s\n", file, line, what, extra.c_str());
}
inline bool msg_matches(const std::string& m, const char* want) { return m == want; }
inline bool msg_matches(const std::string& m, const Contains& c) { return c.matches(m); }
}  // namespace detail
}  // namespace doctest

#define DT_CAT2(a, b) a##b
#define DT_CAT(a, b) DT_CAT2(a, b)
#define TEST_SUITE_BEGIN(name) \
  static int DT_CAT(dt_suite_, __LINE__) = ::doctest::detail::set_suite(name)
#define TEST_SUITE_END() static int DT_CAT(dt_suite_end_, __LINE__) = ::doctest::detail::set_suite("")
#define DT_TEST_CASE(fn, name)                                                    \
  static void fn();                                                               \
  static int DT_CAT(fn, _reg) = ::doctest::detail::reg(name, &fn);                \
  static void fn()
#define TEST_CASE(name) DT_TEST_CASE(DT_CAT(dt_case_, __LINE__), name)
#define CHECK(...)                                                          \
  do {                                                                      \
    if (!(__VA_ARGS__)) ::doctest::detail::fail(__FILE__, __LINE__, #__VA_ARGS__); \
  } while (0)
#define CHECK_FALSE(...)                                                            \
  do {                                                                              \
    if ((__VA_ARGS__)) ::doctest::detail::fail(__FILE__, __LINE__, "!(" #__VA_ARGS__ ")"); \
  } while (0)
#define REQUIRE(...)                                                  \
  do {                                                                \
    if (!(__VA_ARGS__)) {                                             \
      ::doctest::detail::fail(__FILE__, __LINE__, #__VA_ARGS__);      \
      throw ::doctest::detail::Require{};                             \
    }                                                                 \
  } while (0)
#define REQUIRE_MESSAGE(expr, msg)                                    \
  do {                                                                \
    if (!(expr)) {                                                    \
      std::ostringstream dt_os;                                       \
      dt_os << msg;                                                   \
      ::doctest::detail::fail(__FILE__, __LINE__, #expr, dt_os.str()); \
      throw ::doctest::detail::Require{};                             \
    }                                                                 \
  } while (0)
#define CHECK_THROWS_AS(expr, type)                                                  \
  do {                                                                               \
    bool dt_ok = false;                                                              \
    try {                                                                            \
      (void)(expr);                                                                  \
    } catch (const type&) {                                                          \
      dt_ok = true;                                                                  \
    } catch (...) {                                                                  \
    }                                                                                \
    if (!dt_ok) ::doctest::detail::fail(__FILE__, __LINE__, "throws " #type ": " #expr); \
  } while (0)
#define CHECK_THROWS_WITH_AS(expr, matcher, type)                                     \
  do {                                                                                \
    bool dt_ok = false;                                                               \
    std::string dt_msg = "<no throw>";                                                \
    try {                                                                             \
      (void)(expr);                                                                   \
    } catch (const type& e) {                                                         \
      dt_msg = e.what();                                                              \
      dt_ok = ::doctest::detail::msg_matches(dt_msg, matcher);                        \
    } catch (...) {                                                                   \
      dt_msg = "<other exception>";                                                   \
    }                                                                                 \
    if (!dt_ok) ::doctest::detail::fail(__FILE__, __LINE__, "throws-with " #expr, dt_msg); \
  } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main(int argc, char** argv) {
  std::string only = argc > 1 ? argv[1] : "";
  int ran = 0, failed_cases = 0;
  for (const auto& c : ::doctest::detail::cases()) {
    if (!only.empty() && c.suite != only) continue;
    const int before = ::doctest::detail::failures();
    try {
      c.fn();
    } catch (const ::doctest::detail::Require&) {
    } catch (const std::exception& e) {
      ::doctest::detail::fail(c.suite.c_str(), 0, "unexpected exception", e.what());
    }
    ++ran;
    if (::doctest::detail::failures() != before) {
      ++failed_cases;
      std::fprintf(stderr, "  in [%s] %s\n", c.suite.c_str(), c.name.c_str());
    }
  }
  std::printf("[doctest-shim] test cases: %d | passed: %d | failed: %d\n", ran, ran - failed_cases,
              failed_cases);
  return failed_cases ? 1 : 0;
}
#endif
