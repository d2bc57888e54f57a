// Minimal doctest-compatible harness (TEST_CASE, SUBCASE (one level),
// CHECK, CHECK_FALSE, REQUIRE, CHECK_THROWS_AS, doctest::Approx) — enough to compile the
// reference's unit-test sources unchanged against the B200 drop-in
// (doctest itself is not vendored in the reference). Test infrastructure
// only; written for this repo.
#pragma once
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <exception>
#include <functional>
#include <limits>
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
  bool eq(double x) const {
    return std::fabs(x - v_) < eps_ * (scale_ + std::max(std::fabs(x), std::fabs(v_)));
  }
  double value() const { return v_; }

 private:
  double v_;
  double eps_ = static_cast<double>(std::numeric_limits<float>::epsilon()) * 100.0;
  double scale_ = 1.0;
};
inline bool operator==(double x, const Approx& a) { return a.eq(x); }
inline bool operator==(const Approx& a, double x) { return a.eq(x); }
inline bool operator!=(double x, const Approx& a) { return !a.eq(x); }
inline bool operator!=(const Approx& a, double x) { return !a.eq(x); }
inline bool operator<=(double x, const Approx& a) { return x < a.value() || a.eq(x); }
inline bool operator>=(double x, const Approx& a) { return x > a.value() || a.eq(x); }

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
  Reg(const char* n, const char* f, int l, void (*fn)()) { registry().push_back({n, f, l, fn}); }
};
struct Abort {};
inline int& failures() {
  static int f = 0;
  return f;
}
inline int& checks() {
  static int c = 0;
  return c;
}
// SUBCASE: each pass over a test case runs the subcases before the target
// one as skipped and enters exactly the target; the runner repeats the case
// until every subcase it met has had its pass (doctest's one-level semantics).
struct Sub {
  int target = 0, seen = 0;
};
inline Sub& sub() {
  static Sub s;
  return s;
}
inline bool enter_subcase() { return sub().seen++ == sub().target; }
inline void fail(const char* kind, const char* expr, const char* file, int line) {
  ++failures();
  std::fprintf(stderr, "%s:%d: %s( %s ) FAILED\n", file, line, kind, expr);
}
}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define DOCTEST_TC_(fn, name)                                                       \
  static void fn();                                                                 \
  static doctest::detail::Reg DOCTEST_CAT(fn, _reg)(name, __FILE__, __LINE__, fn);  \
  static void fn()
#define TEST_CASE(name) DOCTEST_TC_(DOCTEST_CAT(doctest_case_, __COUNTER__), name)
#define SUBCASE(name) if (doctest::detail::enter_subcase())

#define CHECK(...)                                                               \
  do {                                                                           \
    ++doctest::detail::checks();                                                 \
    if (!(__VA_ARGS__)) doctest::detail::fail("CHECK", #__VA_ARGS__, __FILE__, __LINE__); \
  } while (0)
#define CHECK_FALSE(...)                                                         \
  do {                                                                           \
    ++doctest::detail::checks();                                                 \
    if ((__VA_ARGS__)) doctest::detail::fail("CHECK_FALSE", #__VA_ARGS__, __FILE__, __LINE__); \
  } while (0)
#define REQUIRE(...)                                                             \
  do {                                                                           \
    ++doctest::detail::checks();                                                 \
    if (!(__VA_ARGS__)) {                                                        \
      doctest::detail::fail("REQUIRE", #__VA_ARGS__, __FILE__, __LINE__);        \
      throw doctest::detail::Abort{};                                            \
    }                                                                            \
  } while (0)
#define CHECK_THROWS_AS(expr, type)                                              \
  do {                                                                           \
    ++doctest::detail::checks();                                                 \
    bool ok_ = false;                                                            \
    try {                                                                        \
      (void)(expr);                                                              \
    } catch (const type&) {                                                      \
      ok_ = true;                                                                \
    } catch (...) {                                                              \
    }                                                                            \
    if (!ok_) doctest::detail::fail("CHECK_THROWS_AS", #expr ", " #type, __FILE__, __LINE__); \
  } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main(int argc, char** argv) {
  const char* only = argc > 1 ? argv[1] : nullptr;  // optional filter: case name or source file substring
  int failed_cases = 0, run = 0;
  for (const auto& c : doctest::detail::registry()) {
    if (only && !std::strstr(c.name, only) && !std::strstr(c.file, only)) continue;
    ++run;
    const int before = doctest::detail::failures();
    auto& sub = doctest::detail::sub();
    sub.target = 0;
    do {
      sub.seen = 0;
      try {
        c.fn();
      } catch (const doctest::detail::Abort&) {
      } catch (const std::exception& e) {
        ++doctest::detail::failures();
        std::fprintf(stderr, "%s:%d: unexpected exception: %s\n", c.file, c.line, e.what());
      }
    } while (++sub.target < sub.seen);
    const bool ok = doctest::detail::failures() == before;
    failed_cases += !ok;
    std::printf("[%s] %s\n", ok ? "PASS" : "FAIL", c.name);
  }
  std::printf("test cases: %d | %d passed | %d failed | checks: %d\n", run, run - failed_cases,
              failed_cases, doctest::detail::checks());
  return failed_cases ? 1 : 0;
}
#endif
