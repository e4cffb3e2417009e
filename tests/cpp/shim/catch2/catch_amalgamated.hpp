// Minimal Catch2-compatible test shim (Catch2 is not installed in this image).
//
// Supports the subset the reference's unit tests use: TEST_CASE, SECTION,
// CHECK, CHECK_FALSE, REQUIRE, REQUIRE_FALSE, CHECK_THROWS_AS, CHECK_NOTHROW,
// REQUIRE_NOTHROW, FAIL.  Each TEST_CASE runs once with its SECTIONs executed
// in order (the reference's sections are independent blocks).  A failing
// REQUIRE aborts the test case; main() prints one line per case and exits
// non-zero on any failure.
#pragma once

#include <cstdio>
#include <exception>
#include <functional>
#include <string>
#include <vector>

namespace shim {

struct Case {
  const char *name;
  void (*fn)();
};

inline std::vector<Case> &registry() {
  static std::vector<Case> r;
  return r;
}

inline int &failures() {
  static int f = 0;
  return f;
}

inline int &checks() {
  static int c = 0;
  return c;
}

struct Abort {};

inline void report(bool ok, const char *expr, const char *file, int line, bool fatal) {
  ++checks();
  if (ok) return;
  ++failures();
  std::printf("  FAILED %s:%d: %s\n", file, line, expr);
  if (fatal) throw Abort{};
}

struct Registrar {
  Registrar(const char *name, void (*fn)()) { registry().push_back({name, fn}); }
};

} // namespace shim

#define SHIM_CAT2(a, b) a##b
#define SHIM_CAT(a, b) SHIM_CAT2(a, b)
#define TEST_CASE(name, ...)                                                                                           \
  static void SHIM_CAT(shim_case_, __LINE__)();                                                                        \
  static shim::Registrar SHIM_CAT(shim_reg_, __LINE__)(name, &SHIM_CAT(shim_case_, __LINE__));                          \
  static void SHIM_CAT(shim_case_, __LINE__)()
#define SECTION(name) if (true)
#define CHECK(...) shim::report(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, false)
#define CHECK_FALSE(...) shim::report(!static_cast<bool>(__VA_ARGS__), "!(" #__VA_ARGS__ ")", __FILE__, __LINE__, false)
#define REQUIRE(...) shim::report(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, true)
#define REQUIRE_FALSE(...) shim::report(!static_cast<bool>(__VA_ARGS__), "!(" #__VA_ARGS__ ")", __FILE__, __LINE__, true)
#define FAIL(msg) shim::report(false, msg, __FILE__, __LINE__, true)
#define CHECK_THROWS_AS(expr, type)                                                                                    \
  do {                                                                                                                 \
    bool shim_ok = false;                                                                                              \
    try {                                                                                                              \
      (void)(expr);                                                                                                    \
    } catch (const type &) {                                                                                           \
      shim_ok = true;                                                                                                  \
    } catch (...) {                                                                                                    \
    }                                                                                                                  \
    shim::report(shim_ok, "throws " #type ": " #expr, __FILE__, __LINE__, false);                                      \
  } while (0)
#define CHECK_NOTHROW(expr)                                                                                            \
  do {                                                                                                                 \
    bool shim_ok = true;                                                                                               \
    try {                                                                                                              \
      (void)(expr);                                                                                                    \
    } catch (...) {                                                                                                    \
      shim_ok = false;                                                                                                 \
    }                                                                                                                  \
    shim::report(shim_ok, "nothrow: " #expr, __FILE__, __LINE__, false);                                               \
  } while (0)
#define REQUIRE_NOTHROW(expr) CHECK_NOTHROW(expr)

#ifndef SHIM_NO_MAIN
int main() {
  int failed_cases = 0;
  for (const auto &c : shim::registry()) {
    const int before = shim::failures();
    bool aborted = false;
    try {
      c.fn();
    } catch (const shim::Abort &) {
      aborted = true;
    } catch (const std::exception &e) {
      ++shim::failures();
      std::printf("  FAILED: unexpected exception: %s\n", e.what());
    }
    const bool ok = shim::failures() == before;
    failed_cases += !ok;
    std::printf("[%s] %s%s\n", ok ? "PASS" : "FAIL", c.name, aborted ? " (aborted)" : "");
  }
  std::printf("%zu test cases, %d failed, %d checks, %d failed checks\n", shim::registry().size(), failed_cases,
              shim::checks(), shim::failures());
  return failed_cases ? 1 : 0;
}
#endif
