// Minimal test harness for the C++ API tests (Catch2 is not available):
// TEST_CASE / CHECK / CHECK_THROWS_AS / REQUIRE with a summary exit code.
#pragma once
#include <cmath>
#include <cstdio>
#include <functional>
#include <string>
#include <vector>

namespace mt {
struct Case {
  const char* name;
  std::function<void()> fn;
};
inline std::vector<Case>& registry() {
  static std::vector<Case> r;
  return r;
}
inline int& failures() {
  static int f = 0;
  return f;
}
struct Reg {
  Reg(const char* n, std::function<void()> f) { registry().push_back({n, std::move(f)}); }
};
inline void fail(const char* file, int line, const std::string& what) {
  std::printf("  FAIL %s:%d: %s\n", file, line, what.c_str());
  ++failures();
}
inline bool within_rel(double a, double b, double tol) { return std::abs(a - b) <= tol * std::abs(b); }
inline int run_all() {
  int cases_failed = 0;
  for (auto& c : registry()) {
    const int before = failures();
    try {
      c.fn();
    } catch (const std::exception& e) {
      fail(c.name, 0, std::string("unexpected exception: ") + e.what());
    }
    const bool ok = failures() == before;
    cases_failed += !ok;
    std::printf("%s %s\n", ok ? "PASS" : "FAIL", c.name);
  }
  std::printf("%zu cases, %d failed\n", registry().size(), cases_failed);
  return cases_failed ? 1 : 0;
}
}  // namespace mt

#define MT_CAT2(a, b) a##b
#define MT_CAT(a, b) MT_CAT2(a, b)
#define TEST_CASE(name)                                  \
  static void MT_CAT(test_fn_, __LINE__)();              \
  static mt::Reg MT_CAT(test_reg_, __LINE__)(name, MT_CAT(test_fn_, __LINE__)); \
  static void MT_CAT(test_fn_, __LINE__)()
#define CHECK(cond) \
  do {              \
    if (!(cond)) mt::fail(__FILE__, __LINE__, #cond); \
  } while (0)
#define REQUIRE(cond)                              \
  do {                                             \
    if (!(cond)) {                                 \
      mt::fail(__FILE__, __LINE__, #cond);         \
      return;                                      \
    }                                              \
  } while (0)
#define CHECK_REL(a, b, tol)                                                                   \
  do {                                                                                         \
    const double mt_a = (a), mt_b = (b);                                                       \
    if (!mt::within_rel(mt_a, mt_b, tol))                                                      \
      mt::fail(__FILE__, __LINE__, std::string(#a " ~ " #b ": ") + std::to_string(mt_a) + " vs " + std::to_string(mt_b)); \
  } while (0)
#define CHECK_THROWS_AS(expr, type)                                            \
  do {                                                                         \
    bool mt_ok = false;                                                        \
    try {                                                                      \
      (void)(expr);                                                            \
    } catch (const type&) {                                                    \
      mt_ok = true;                                                            \
    } catch (...) {                                                            \
    }                                                                          \
    if (!mt_ok) mt::fail(__FILE__, __LINE__, "expected " #type " from " #expr); \
  } while (0)
#define CHECK_NOTHROW(expr)                                              \
  do {                                                                   \
    try {                                                                \
      (void)(expr);                                                      \
    } catch (const std::exception& e) {                                  \
      mt::fail(__FILE__, __LINE__, std::string("threw: ") + e.what());   \
    }                                                                    \
  } while (0)
#define MT_MAIN() \
  int main() { return mt::run_all(); }
