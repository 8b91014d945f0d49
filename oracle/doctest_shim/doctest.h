// Minimal stand-in for doctest (not in this image), enough to compile the
// reference's unit tests (proj/tests/test_*.cpp) UNMODIFIED. Test
// infrastructure only (oracle/Makefile target `unit_engine`).
//
// Supported: TEST_CASE, SUBCASE (doctest semantics: the test case body is
// re-run once per leaf subcase, code outside subcases runs every pass),
// CHECK, REQUIRE (aborts the test case), CHECK_THROWS_AS, CHECK_NOTHROW,
// doctest::Approx(v).epsilon(e).scale(s) with doctest's comparison rule
// |a - v| < eps * (scale + max(|a|, |v|)), and
// DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN (a main() that runs every case).
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <exception>
#include <limits>
#include <string>
#include <vector>

namespace doctest_shim {

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
  Reg(const char* n, void (*f)(), const char* file, int line) { registry().push_back({n, f, file, line}); }
};
struct State {
  int target = 0;   // leaf subcase run in this pass
  int seen = 0;     // subcases met so far in this pass
  long checks = 0;
  long failed = 0;
  bool case_failed = false;
  const char* case_name = "";
};
inline State& st() {
  static State s;
  return s;
}
struct RequireFailed {};

inline void record(bool ok, const char* expr, const char* file, int line) {
  ++st().checks;
  if (ok) return;
  ++st().failed;
  st().case_failed = true;
  std::printf("%s:%d: FAILED in \"%s\": %s\n", file, line, st().case_name, expr);
}
inline bool check(bool ok, const char* expr, const char* file, int line) {
  record(ok, expr, file, line);
  return ok;
}
struct Subcase {
  bool run;
  explicit Subcase(const char*) : run(st().seen++ == st().target) {}
  explicit operator bool() const { return run; }
};

inline int run_all() {
  int failed_cases = 0;
  for (const Case& c : registry()) {
    st().case_name = c.name;
    st().case_failed = false;
    for (st().target = 0;; ++st().target) {
      st().seen = 0;
      try {
        c.fn();
      } catch (const RequireFailed&) {
      } catch (const std::exception& e) {
        record(false, (std::string("unexpected exception: ") + e.what()).c_str(), c.file, c.line);
      } catch (...) {
        record(false, "unexpected exception", c.file, c.line);
      }
      if (st().seen <= st().target + 1) break;
    }
    failed_cases += st().case_failed ? 1 : 0;
  }
  std::printf("[doctest-shim] test cases: %zu | %zu passed | %d failed\n", registry().size(),
              registry().size() - failed_cases, failed_cases);
  std::printf("[doctest-shim] assertions: %ld | %ld passed | %ld failed\n", st().checks,
              st().checks - st().failed, st().failed);
  return failed_cases == 0 ? 0 : 1;
}

}  // namespace doctest_shim

namespace doctest {
class Approx {
 public:
  explicit Approx(double v)
      : v_(v), eps_(static_cast<double>(std::numeric_limits<float>::epsilon()) * 100), scale_(1.0) {}
  Approx& epsilon(double e) {
    eps_ = e;
    return *this;
  }
  Approx& scale(double s) {
    scale_ = s;
    return *this;
  }
  friend bool operator==(double l, const Approx& r) {
    return std::fabs(l - r.v_) < r.eps_ * (r.scale_ + std::max(std::fabs(l), std::fabs(r.v_)));
  }
  friend bool operator==(const Approx& l, double r) { return r == l; }
  friend bool operator!=(double l, const Approx& r) { return !(l == r); }
  friend bool operator!=(const Approx& l, double r) { return !(r == l); }

 private:
  double v_, eps_, scale_;
};
}  // namespace doctest

#define DOCTEST_SHIM_CAT2(a, b) a##b
#define DOCTEST_SHIM_CAT(a, b) DOCTEST_SHIM_CAT2(a, b)
#define DOCTEST_SHIM_CASE(fn, name)                                                     \
  static void fn();                                                                    \
  static const doctest_shim::Reg DOCTEST_SHIM_CAT(fn, _reg)(name, &fn, __FILE__, __LINE__); \
  static void fn()
#define TEST_CASE(name) DOCTEST_SHIM_CASE(DOCTEST_SHIM_CAT(doctest_shim_case_, __LINE__), name)
#define SUBCASE(name) if (const doctest_shim::Subcase doctest_shim_sc{name}; doctest_shim_sc)
#define CHECK(...) doctest_shim::check(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__)
#define REQUIRE(...)                                                                        \
  do {                                                                                      \
    if (!doctest_shim::check(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__)) \
      throw doctest_shim::RequireFailed{};                                                  \
  } while (0)
#define CHECK_THROWS_AS(expr, ...)                                                     \
  do {                                                                                 \
    bool doctest_shim_ok = false;                                                      \
    try {                                                                              \
      static_cast<void>(expr);                                                         \
    } catch (const __VA_ARGS__&) {                                                     \
      doctest_shim_ok = true;                                                          \
    } catch (...) {                                                                    \
    }                                                                                  \
    doctest_shim::record(doctest_shim_ok, "CHECK_THROWS_AS(" #expr ", " #__VA_ARGS__ ")", \
                         __FILE__, __LINE__);                                          \
  } while (0)
#define CHECK_NOTHROW(...)                                                        \
  do {                                                                            \
    bool doctest_shim_ok = true;                                                  \
    try {                                                                         \
      static_cast<void>(__VA_ARGS__);                                             \
    } catch (...) {                                                               \
      doctest_shim_ok = false;                                                    \
    }                                                                             \
    doctest_shim::record(doctest_shim_ok, "CHECK_NOTHROW(" #__VA_ARGS__ ")", __FILE__, __LINE__); \
  } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() { return doctest_shim::run_all(); }
#endif
