// doctest.h -- a minimal doctest-compatible test harness (the reference's
// vendored doctest is absent from /root/reference, proj/.gitignore:2).  It
// implements exactly the subset the reference's unit tests use so those test
// files compile UNMODIFIED against the B200 drop-in: TEST_CASE, SUBCASE
// (each leaf subcase runs in its own pass of the test case), CHECK, REQUIRE,
// CHECK_THROWS_AS and doctest::Approx with .epsilon().
#pragma once

#include <cmath>
#include <cstdio>
#include <exception>
#include <functional>
#include <limits>
#include <set>
#include <string>
#include <vector>

namespace doctest {

class Approx {
 public:
  explicit Approx(double v) : value_(v) {}
  Approx& epsilon(double e) {
    eps_ = e;
    return *this;
  }
  friend bool operator==(double lhs, const Approx& a) { return a.matches(lhs); }
  friend bool operator==(const Approx& a, double rhs) { return a.matches(rhs); }
  friend bool operator!=(double lhs, const Approx& a) { return !a.matches(lhs); }
  friend bool operator!=(const Approx& a, double rhs) { return !a.matches(rhs); }

 private:
  bool matches(double x) const {
    return std::fabs(x - value_) < eps_ * (1.0 + std::fmax(std::fabs(x), std::fabs(value_)));
  }
  double value_;
  double eps_ = std::numeric_limits<float>::epsilon() * 100;
};

namespace shim {

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

struct Registrar {
  Registrar(const char* n, const char* f, int l, void (*fn)()) {
    registry().push_back({n, f, l, fn});
  }
};

struct RunState {
  std::set<int> done;        // subcases already executed
  std::set<int> seen;        // subcases discovered
  bool entered = false;      // a subcase was entered in this pass
  int current = -1;
  int failures = 0;
  int checks = 0;
};

inline RunState& state() {
  static RunState s;
  return s;
}

struct Subcase {
  bool active = false;
  explicit Subcase(int id) {
    RunState& s = state();
    s.seen.insert(id);
    if (!s.entered && !s.done.count(id)) {
      s.entered = true;
      s.current = id;
      active = true;
    }
  }
  explicit operator bool() const { return active; }
};

struct RequireFailed {};

inline void report(bool ok, const char* kind, const char* expr, const char* file, int line) {
  RunState& s = state();
  ++s.checks;
  if (!ok) {
    ++s.failures;
    std::printf("%s:%d: %s( %s ) FAILED\n", file, line, kind, expr);
  }
}

inline int run_all() {
  int failed_cases = 0, total_checks = 0;
  for (const Case& c : registry()) {
    RunState& s = state();
    s = RunState{};
    bool case_failed = false;
    do {
      s.entered = false;
      s.current = -1;
      try {
        c.fn();
      } catch (const RequireFailed&) {
        case_failed = true;
      } catch (const std::exception& e) {
        std::printf("%s:%d: TEST_CASE(%s) threw: %s\n", c.file, c.line, c.name, e.what());
        case_failed = true;
      }
      if (s.entered) s.done.insert(s.current);
    } while (s.entered && s.done.size() < s.seen.size());
    if (s.failures) case_failed = true;
    total_checks += s.checks;
    std::printf("[%s] %s\n", case_failed ? "FAIL" : "PASS", c.name);
    failed_cases += case_failed;
  }
  std::printf("%zu test cases, %d failed, %d assertions\n", registry().size(), failed_cases,
              total_checks);
  return failed_cases ? 1 : 0;
}

}  // namespace shim
}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define DOCTEST_TEST_CASE_IMPL(fn, name)                                                 \
  static void fn();                                                                     \
  static ::doctest::shim::Registrar DOCTEST_CAT(fn, _reg)(name, __FILE__, __LINE__, fn); \
  static void fn()
#define TEST_CASE(name) DOCTEST_TEST_CASE_IMPL(DOCTEST_CAT(doctest_case_, __COUNTER__), name)
#define SUBCASE(name) if (::doctest::shim::Subcase DOCTEST_CAT(sc_, __LINE__){__LINE__})
#define CHECK(...) ::doctest::shim::report(static_cast<bool>(__VA_ARGS__), "CHECK", #__VA_ARGS__, __FILE__, __LINE__)
#define REQUIRE(...)                                                                    \
  do {                                                                                  \
    const bool ok__ = static_cast<bool>(__VA_ARGS__);                                   \
    ::doctest::shim::report(ok__, "REQUIRE", #__VA_ARGS__, __FILE__, __LINE__);         \
    if (!ok__) throw ::doctest::shim::RequireFailed{};                                  \
  } while (0)
#define CHECK_THROWS_AS(expr, type)                                                     \
  do {                                                                                  \
    bool ok__ = false;                                                                  \
    try {                                                                               \
      (void)(expr);                                                                     \
    } catch (const type&) {                                                             \
      ok__ = true;                                                                      \
    } catch (...) {                                                                     \
    }                                                                                   \
    ::doctest::shim::report(ok__, "CHECK_THROWS_AS", #expr ", " #type, __FILE__, __LINE__); \
  } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() { return ::doctest::shim::run_all(); }
#endif
