// Minimal stand-in for the doctest single header, which the reference
// vendors under proj/vendor/ (gitignored, absent: SURVEY.md §8c). It covers
// exactly the macros the reference's unit suites use: TEST_CASE, CHECK,
// CHECK_FALSE, REQUIRE, CHECK_THROWS_AS, CAPTURE and doctest::Approx with
// .epsilon(). Test infrastructure only — used to build the reference's own
// suites against oracle/_ref and against the B200 library's gpuos:: API.
#pragma once

#include <cmath>
#include <cstdio>
#include <exception>
#include <functional>
#include <sstream>
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
  friend bool operator==(double lhs, const Approx& rhs) {
    double scale = std::max(std::fabs(lhs), std::fabs(rhs.value_));
    return std::fabs(lhs - rhs.value_) <= rhs.eps_ * (1.0 + scale);
  }
  friend bool operator==(const Approx& lhs, double rhs) { return rhs == lhs; }
  friend bool operator!=(double lhs, const Approx& rhs) { return !(lhs == rhs); }

 private:
  double value_;
  double eps_ = 1.1920929e-7 * 100;  // doctest's default: float epsilon x 100
};

namespace shim {

struct Case {
  const char* name;
  void (*fn)();
};

inline std::vector<Case>& registry() {
  static std::vector<Case> r;
  return r;
}

struct Stats {
  long checks = 0;
  long failures = 0;
  bool current_failed = false;
};

inline Stats& stats() {
  static Stats s;
  return s;
}

struct AbortCase {};

inline std::vector<std::string>& captures() {
  static std::vector<std::string> c;
  return c;
}

inline void report(bool ok, const char* expr, const char* file, int line,
                   bool fatal) {
  ++stats().checks;
  if (ok) return;
  ++stats().failures;
  stats().current_failed = true;
  std::fprintf(stderr, "%s:%d: FAILED: %s\n", file, line, expr);
  for (const auto& c : captures()) std::fprintf(stderr, "  with %s\n", c.c_str());
  if (fatal) throw AbortCase{};
}

struct Registrar {
  Registrar(const char* name, void (*fn)()) { registry().push_back({name, fn}); }
};

struct CaptureGuard {
  explicit CaptureGuard(std::string s) { captures().push_back(std::move(s)); }
  ~CaptureGuard() { captures().pop_back(); }
};

inline int run_all() {
  long cases = 0, failed_cases = 0;
  for (const Case& c : registry()) {
    ++cases;
    stats().current_failed = false;
    try {
      c.fn();
    } catch (const AbortCase&) {
    } catch (const std::exception& e) {
      ++stats().failures;
      stats().current_failed = true;
      std::fprintf(stderr, "test case '%s' threw: %s\n", c.name, e.what());
    }
    if (stats().current_failed) {
      ++failed_cases;
      std::fprintf(stderr, "test case FAILED: %s\n", c.name);
    }
  }
  std::printf("[doctest-shim] test cases: %ld | %ld passed | %ld failed | "
              "assertions: %ld | %ld failed\n",
              cases, cases - failed_cases, failed_cases, stats().checks,
              stats().failures);
  return failed_cases == 0 ? 0 : 1;
}

}  // namespace shim
}  // namespace doctest

#define DOCTEST_CAT2(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT2(a, b)
#define DOCTEST_UNIQ(p) DOCTEST_CAT(p, __LINE__)

#define TEST_CASE(name)                                                     \
  static void DOCTEST_UNIQ(doctest_fn_)();                                  \
  static ::doctest::shim::Registrar DOCTEST_UNIQ(doctest_reg_)(             \
      name, &DOCTEST_UNIQ(doctest_fn_));                                    \
  static void DOCTEST_UNIQ(doctest_fn_)()

#define CHECK(...) \
  ::doctest::shim::report(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, false)
#define CHECK_FALSE(...) \
  ::doctest::shim::report(!static_cast<bool>(__VA_ARGS__), "!(" #__VA_ARGS__ ")", __FILE__, __LINE__, false)
#define REQUIRE(...) \
  ::doctest::shim::report(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, true)
#define CHECK_THROWS_AS(expr, ex)                                           \
  do {                                                                      \
    bool doctest_caught_ = false;                                           \
    try {                                                                   \
      (void)(expr);                                                         \
    } catch (const ex&) {                                                   \
      doctest_caught_ = true;                                               \
    } catch (...) {                                                         \
    }                                                                       \
    ::doctest::shim::report(doctest_caught_, "throws " #ex ": " #expr,      \
                            __FILE__, __LINE__, false);                     \
  } while (0)
#define CAPTURE(x)                                                          \
  std::ostringstream DOCTEST_UNIQ(doctest_os_);                             \
  DOCTEST_UNIQ(doctest_os_) << #x " := " << (x);                            \
  ::doctest::shim::CaptureGuard DOCTEST_UNIQ(doctest_cg_)(                  \
      DOCTEST_UNIQ(doctest_os_).str())

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() { return ::doctest::shim::run_all(); }
#endif
