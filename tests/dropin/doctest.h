// Minimal doctest-compatible harness (TEST INFRASTRUCTURE): lets the
// reference's own unit-test sources (/root/reference/proj/tests/*.cpp, read
// in place, never copied) compile against the B200 build's drop-in headers
// (paper_2510_20111_b200/csrc/hzp/*.hpp) and link against libhzp_b200.so.
// Supports what those files use: TEST_CASE, CHECK, REQUIRE, CHECK_THROWS_AS,
// doctest::Approx.  The runner prints one line per case.
#pragma once

#include <cmath>
#include <cstdio>
#include <functional>
#include <string>
#include <vector>

namespace doctest {

struct Case {
  const char* name;
  void (*fn)();
};
inline std::vector<Case>& registry() {
  static std::vector<Case> r;
  return r;
}
struct Register {
  Register(const char* n, void (*f)()) { registry().push_back({n, f}); }
};
struct Failed {};
inline int& failures() {
  static int f = 0;
  return f;
}
inline void fail(const char* what, const char* file, int line, bool fatal) {
  std::printf("    check failed: %s (%s:%d)\n", what, file, line);
  ++failures();
  if (fatal) throw Failed{};
}

class Approx {
 public:
  explicit Approx(double v) : v_(v) {}
  Approx& epsilon(double e) {
    eps_ = e;
    return *this;
  }
  friend bool operator==(double a, const Approx& b) {
    return std::fabs(a - b.v_) <= b.eps_ * (1.0 + std::max(std::fabs(a), std::fabs(b.v_)));
  }
  friend bool operator==(const Approx& b, double a) { return a == b; }
  friend bool operator!=(double a, const Approx& b) { return !(a == b); }
  friend bool operator!=(const Approx& b, double a) { return !(a == b); }

 private:
  double v_;
  double eps_ = 1e-5;
};

}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define TEST_CASE(name)                                                                  \
  static void DOCTEST_CAT(dt_case_, __LINE__)();                                         \
  static doctest::Register DOCTEST_CAT(dt_reg_, __LINE__)(name, &DOCTEST_CAT(dt_case_, __LINE__)); \
  static void DOCTEST_CAT(dt_case_, __LINE__)()
#define CHECK(...) \
  do {             \
    if (!(__VA_ARGS__)) doctest::fail(#__VA_ARGS__, __FILE__, __LINE__, false); \
  } while (0)
#define REQUIRE(...) \
  do {               \
    if (!(__VA_ARGS__)) doctest::fail(#__VA_ARGS__, __FILE__, __LINE__, true); \
  } while (0)
#define CHECK_THROWS_AS(expr, type)                                        \
  do {                                                                     \
    bool dt_ok = false;                                                    \
    try {                                                                  \
      (void)(expr);                                                        \
    } catch (const type&) {                                                \
      dt_ok = true;                                                        \
    } catch (...) {                                                        \
    }                                                                      \
    if (!dt_ok) doctest::fail("throws " #type ": " #expr, __FILE__, __LINE__, false); \
  } while (0)
