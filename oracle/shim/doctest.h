// ORACLE / TEST INFRASTRUCTURE — minimal doctest stand-in (doctest.h is not
// vendored in /root/reference).  Covers exactly what
// proj/tests/test_{factor,ara,solve}.cpp use: TEST_CASE, CHECK, REQUIRE,
// CHECK_THROWS_AS and doctest::Approx(...).epsilon(...).  The runner prints one
// machine-readable line per test case ("[case] PASS|FAIL <name>") so
// tests/test_gpu_conformance.py can gate each reference case separately.
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <exception>
#include <limits>
#include <string>
#include <vector>

namespace doctest {

class Approx {
 public:
  explicit Approx(double v)
      : value_(v), eps_(static_cast<double>(std::numeric_limits<float>::epsilon()) * 100),
        scale_(1.0) {}
  Approx& epsilon(double e) { eps_ = e; return *this; }
  Approx& scale(double s) { scale_ = s; return *this; }
  bool eq(double lhs) const {
    return std::fabs(lhs - value_) < eps_ * (scale_ + std::max(std::fabs(lhs), std::fabs(value_)));
  }
  double value() const { return value_; }

 private:
  double value_, eps_, scale_;
};
inline bool operator==(double l, const Approx& r) { return r.eq(l); }
inline bool operator==(const Approx& l, double r) { return l.eq(r); }
inline bool operator!=(double l, const Approx& r) { return !r.eq(l); }
inline bool operator!=(const Approx& l, double r) { return !l.eq(r); }
inline bool operator<=(double l, const Approx& r) { return l < r.value() || r.eq(l); }
inline bool operator>=(double l, const Approx& r) { return l > r.value() || r.eq(l); }
inline bool operator<=(const Approx& l, double r) { return l.value() < r || l.eq(r); }
inline bool operator>=(const Approx& l, double r) { return l.value() > r || l.eq(r); }

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
inline int& failures() {
  static int f = 0;
  return f;
}
struct Registrar {
  Registrar(const char* name, void (*fn)(), const char* file, int line) {
    registry().push_back({name, fn, file, line});
  }
};
struct RequireFailed {};
inline void report(const char* kind, const char* expr, const char* file, int line) {
  ++failures();
  std::fprintf(stdout, "%s:%d: %s( %s ) FAILED\n", file, line, kind, expr);
  std::fflush(stdout);
}
}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define DOCTEST_CASE_IMPL(fn, name)                                              \
  static void fn();                                                              \
  static ::doctest::detail::Registrar DOCTEST_CAT(fn, _reg)(name, fn, __FILE__,  \
                                                            __LINE__);           \
  static void fn()
#define TEST_CASE(name) DOCTEST_CASE_IMPL(DOCTEST_CAT(doctest_case_, __LINE__), name)

#define CHECK(...)                                                               \
  do {                                                                           \
    if (!(__VA_ARGS__)) ::doctest::detail::report("CHECK", #__VA_ARGS__, __FILE__, __LINE__); \
  } while (0)
#define REQUIRE(...)                                                             \
  do {                                                                           \
    if (!(__VA_ARGS__)) {                                                        \
      ::doctest::detail::report("REQUIRE", #__VA_ARGS__, __FILE__, __LINE__);    \
      throw ::doctest::detail::RequireFailed{};                                  \
    }                                                                            \
  } while (0)
#define CHECK_THROWS_AS(expr, type)                                              \
  do {                                                                           \
    bool caught_ = false;                                                        \
    try {                                                                        \
      (void)(expr);                                                              \
    } catch (const type&) {                                                      \
      caught_ = true;                                                            \
    } catch (...) {                                                              \
    }                                                                            \
    if (!caught_) ::doctest::detail::report("CHECK_THROWS_AS", #expr, __FILE__, __LINE__); \
  } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
// Runs every case (or those whose name contains argv[1]); exit 1 on any failure.
// `--list` prints the case names.
int main(int argc, char** argv) {
  const char* filter = argc > 1 ? argv[1] : nullptr;
  if (filter && !std::strcmp(filter, "--list")) {
    for (const auto& c : ::doctest::detail::registry()) std::fprintf(stdout, "%s\n", c.name);
    return 0;
  }
  int failed_cases = 0, run = 0;
  for (const auto& c : ::doctest::detail::registry()) {
    if (filter && !std::strstr(c.name, filter)) continue;
    ++run;
    const int before = ::doctest::detail::failures();
    std::string err;
    try {
      c.fn();
    } catch (const ::doctest::detail::RequireFailed&) {
    } catch (const std::exception& e) {
      err = e.what();
      ++::doctest::detail::failures();
    } catch (...) {
      err = "unknown exception";
      ++::doctest::detail::failures();
    }
    const bool ok = ::doctest::detail::failures() == before;
    if (!ok) ++failed_cases;
    if (!err.empty()) std::fprintf(stdout, "  threw: %s\n", err.c_str());
    std::fprintf(stdout, "[case] %s %s\n", ok ? "PASS" : "FAIL", c.name);
    std::fflush(stdout);
  }
  std::fprintf(stdout, "[summary] %d cases, %d failed\n", run, failed_cases);
  return failed_cases ? 1 : 0;
}
#endif
