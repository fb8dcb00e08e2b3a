// doctest.h -- minimal doctest-compatible shim (tests only).
//
// The reference unit suite (/root/reference/proj/tests/test_*.cpp) expects
// the single-header doctest library, which is not available offline.  This
// shim implements the subset those files use -- TEST_CASE, flat SUBCASE,
// CHECK / REQUIRE, CHECK_THROWS_AS, CHECK_THROWS_WITH_AS, REQUIRE_NOTHROW,
// CAPTURE, doctest::Approx -- so the suite compiles unmodified against the
// B200 library (Makefile target build/ref_unit_tests).
#pragma once

#include <cmath>
#include <cstdio>
#include <exception>
#include <functional>
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

struct Registrar {
  Registrar(const char* name, void (*fn)(), const char* file, int line) {
    registry().push_back({name, fn, file, line});
  }
};

struct State {
  long checks = 0;
  long failed_checks = 0;
  bool case_failed = false;
  int subcase_target = 0;
  int subcase_seen = 0;
  std::string capture;
};

inline State& st() {
  static State s;
  return s;
}

struct RequireAbort {};

inline void report(bool ok, const char* what, const char* file, int line, const std::string& extra = "") {
  ++st().checks;
  if (ok) return;
  ++st().failed_checks;
  st().case_failed = true;
  std::printf("%s:%d: FAILED: %s %s%s\n", file, line, what, extra.c_str(), st().capture.c_str());
}

inline bool enter_subcase() { return st().subcase_seen++ == st().subcase_target; }

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
  bool matches(double x) const {
    return std::fabs(x - v_) < eps_ * (scale_ + std::fmax(std::fabs(x), std::fabs(v_)));
  }

 private:
  double v_;
  double eps_ = 1.1920928955078125e-05;  // doctest default: FLT_EPSILON * 100
  double scale_ = 1.0;
};

inline bool operator==(double x, const Approx& a) { return a.matches(x); }
inline bool operator==(const Approx& a, double x) { return a.matches(x); }
inline bool operator!=(double x, const Approx& a) { return !a.matches(x); }

inline int run_all() {
  int failed_cases = 0;
  for (const Case& c : registry()) {
    st().case_failed = false;
    st().subcase_target = 0;
    for (;;) {
      st().subcase_seen = 0;
      st().capture.clear();
      try {
        c.fn();
      } catch (const RequireAbort&) {
      } catch (const std::exception& e) {
        report(false, "unexpected exception", c.file, c.line, e.what());
      } catch (...) {
        report(false, "unexpected exception", c.file, c.line);
      }
      if (st().subcase_seen > st().subcase_target + 1) {
        ++st().subcase_target;
        continue;
      }
      break;
    }
    if (st().case_failed) {
      ++failed_cases;
      std::printf("TEST CASE FAILED: %s\n", c.name);
    }
  }
  std::printf("[doctest-shim] test cases: %zu | %zu passed | %d failed | assertions: %ld | %ld failed\n",
              registry().size(), registry().size() - failed_cases, failed_cases, st().checks,
              st().failed_checks);
  return failed_cases ? 1 : 0;
}

}  // namespace doctest_shim

namespace doctest {
using Approx = doctest_shim::Approx;
}

#define DS_CAT2(a, b) a##b
#define DS_CAT(a, b) DS_CAT2(a, b)
#define DS_TEST_CASE_IMPL(fn, name)                                               \
  static void fn();                                                               \
  static doctest_shim::Registrar DS_CAT(fn, _reg)(name, &fn, __FILE__, __LINE__); \
  static void fn()
#define TEST_CASE(name) DS_TEST_CASE_IMPL(DS_CAT(ds_case_, __COUNTER__), name)
#define SUBCASE(name) if (doctest_shim::enter_subcase())

#define CHECK(...) doctest_shim::report(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__)
#define REQUIRE(...)                                                                       \
  do {                                                                                     \
    const bool ds_ok = static_cast<bool>(__VA_ARGS__);                                     \
    doctest_shim::report(ds_ok, "REQUIRE(" #__VA_ARGS__ ")", __FILE__, __LINE__);          \
    if (!ds_ok) throw doctest_shim::RequireAbort{};                                        \
  } while (0)
#define CHECK_THROWS_AS(expr, type)                                                        \
  do {                                                                                     \
    bool ds_ok = false;                                                                    \
    try {                                                                                  \
      (void)(expr);                                                                        \
    } catch (const type&) {                                                                \
      ds_ok = true;                                                                        \
    } catch (...) {                                                                        \
    }                                                                                      \
    doctest_shim::report(ds_ok, "CHECK_THROWS_AS(" #expr ", " #type ")", __FILE__, __LINE__); \
  } while (0)
#define CHECK_THROWS_WITH_AS(expr, msg, type)                                              \
  do {                                                                                     \
    bool ds_ok = false;                                                                    \
    std::string ds_what;                                                                   \
    try {                                                                                  \
      (void)(expr);                                                                        \
    } catch (const type& e) {                                                              \
      ds_what = e.what();                                                                  \
      ds_ok = ds_what == std::string(msg);                                                 \
    } catch (...) {                                                                        \
    }                                                                                      \
    doctest_shim::report(ds_ok, "CHECK_THROWS_WITH_AS(" #expr ")", __FILE__, __LINE__, ds_what); \
  } while (0)
#define REQUIRE_NOTHROW(expr)                                                              \
  do {                                                                                     \
    bool ds_ok = true;                                                                     \
    try {                                                                                  \
      (void)(expr);                                                                        \
    } catch (...) {                                                                        \
      ds_ok = false;                                                                       \
    }                                                                                      \
    doctest_shim::report(ds_ok, "REQUIRE_NOTHROW(" #expr ")", __FILE__, __LINE__);         \
    if (!ds_ok) throw doctest_shim::RequireAbort{};                                        \
  } while (0)
#define CAPTURE(x) (doctest_shim::st().capture = std::string(" [" #x "=") + std::to_string(x) + "]")

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() { return doctest_shim::run_all(); }
#endif
