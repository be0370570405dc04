// Minimal doctest-compatible test harness (TEST INFRASTRUCTURE ONLY).
//
// The reference vendors doctest under a gitignored vendor/ directory that is
// absent from the reference checkout (proj/.gitignore:2, proj/CMakeLists.txt:5),
// so its unit tests cannot build as shipped.  This header implements the small
// subset those tests use -- TEST_CASE, SUBCASE (re-run-per-leaf semantics),
// CHECK / CHECK_FALSE / CHECK_NOTHROW / CHECK_THROWS_AS, REQUIRE, CAPTURE,
// doctest::Approx -- so oracle/Makefile can compile the reference's own
// test files unmodified, once against the reference library (pinning this
// harness) and once against the B200 facade (the parity run).
#pragma once

#include <cmath>
#include <cstdio>
#include <cstring>
#include <exception>
#include <functional>
#include <set>
#include <string>
#include <vector>

namespace ffx_shim {

struct TestCase {
  const char* name;
  const char* file;
  int line;
  void (*fn)();
};

inline std::vector<TestCase>& registry() {
  static std::vector<TestCase> r;
  return r;
}

struct Registrar {
  Registrar(const char* name, const char* file, int line, void (*fn)()) {
    registry().push_back(TestCase{name, file, line, fn});
  }
};

struct State {
  std::set<std::string> done;          // completed subcase paths of the running test
  std::vector<std::string> path;       // current subcase stack
  std::vector<char> entered, pending;  // per depth: a sibling was entered / skipped work
  long checks = 0, failures = 0;
  const char* current = "";
};

inline State& st() {
  static State s;
  return s;
}

inline std::string key(const std::vector<std::string>& p) {
  std::string k;
  for (const auto& s : p) k += "\x1f" + s;
  return k;
}

struct Subcase {
  bool entered = false;
  std::string full;
  explicit Subcase(const char* name) {
    auto& s = st();
    const std::size_t d = s.path.size();
    auto p = s.path;
    p.push_back(name);
    full = key(p);
    if (s.done.count(full)) return;
    if (s.entered[d]) {
      s.pending[d] = 1;
      return;
    }
    s.entered[d] = 1;
    s.path.push_back(name);
    s.entered.resize(d + 2);
    s.pending.resize(d + 2);
    s.entered[d + 1] = 0;
    s.pending[d + 1] = 0;
    entered = true;
  }
  ~Subcase() {
    if (!entered) return;
    auto& s = st();
    const std::size_t d = s.path.size() - 1;
    const bool child_pending = s.pending[d + 1] != 0;
    s.path.pop_back();
    if (child_pending)
      s.pending[d] = 1;
    else
      s.done.insert(full);
  }
};

struct RequireFailed {};

inline void report(bool ok, const char* kind, const char* expr, const char* file, int line) {
  auto& s = st();
  ++s.checks;
  if (ok) return;
  ++s.failures;
  std::string sub;
  for (const auto& p : s.path) sub += " / " + p;
  std::fprintf(stderr, "%s:%d: FAILED %s( %s ) in \"%s\"%s\n", file, line, kind, expr, s.current,
               sub.c_str());
}

inline int run_all(int argc, char** argv) {
  const char* filter = nullptr;
  for (int i = 1; i < argc; ++i)
    if (std::strncmp(argv[i], "-tc=", 4) == 0) filter = argv[i] + 4;
  auto& s = st();
  int cases = 0, failed_cases = 0;
  for (const auto& tc : registry()) {
    if (filter && !std::strstr(tc.name, filter)) continue;
    ++cases;
    s.done.clear();
    s.current = tc.name;
    const long before = s.failures;
    for (int run = 0; run < 10000; ++run) {
      s.path.clear();
      s.entered.assign(1, 0);
      s.pending.assign(1, 0);
      try {
        tc.fn();
      } catch (const RequireFailed&) {
      } catch (const std::exception& e) {
        ++s.failures;
        std::fprintf(stderr, "%s:%d: test \"%s\" threw: %s\n", tc.file, tc.line, tc.name, e.what());
      } catch (...) {
        ++s.failures;
        std::fprintf(stderr, "%s:%d: test \"%s\" threw an unknown exception\n", tc.file, tc.line,
                     tc.name);
      }
      if (!s.pending[0]) break;
    }
    if (s.failures != before) ++failed_cases;
  }
  std::printf("[doctest-shim] test cases: %d | %d passed | %d failed | assertions: %ld | %ld failed\n",
              cases, cases - failed_cases, failed_cases, s.checks, s.failures);
  return failed_cases ? 1 : 0;
}

}  // namespace ffx_shim

namespace doctest {
class Approx {
 public:
  explicit Approx(double v) : v_(v) {}
  Approx& epsilon(double e) { eps_ = e; return *this; }
  Approx& scale(double s) { scale_ = s; return *this; }
  friend bool operator==(double a, const Approx& b) {
    const double m = std::fmax(std::fabs(a), std::fabs(b.v_));
    return std::fabs(a - b.v_) < b.eps_ * (b.scale_ + m);
  }
  friend bool operator==(const Approx& b, double a) { return a == b; }
  friend bool operator!=(double a, const Approx& b) { return !(a == b); }
  friend bool operator!=(const Approx& b, double a) { return !(a == b); }
  friend bool operator<=(double a, const Approx& b) { return a < b.v_ || a == b; }
  friend bool operator>=(double a, const Approx& b) { return a > b.v_ || a == b; }
  friend bool operator<(double a, const Approx& b) { return a < b.v_ && a != b; }
  friend bool operator>(double a, const Approx& b) { return a > b.v_ && a != b; }

 private:
  double v_;
  double eps_ = 1.1920928955078125e-05;  // FLT_EPSILON * 100, doctest's default
  double scale_ = 1.0;
};
}  // namespace doctest

#define FFX_SHIM_CAT2(a, b) a##b
#define FFX_SHIM_CAT(a, b) FFX_SHIM_CAT2(a, b)
#define FFX_SHIM_TC(fn, name)                                                         \
  static void fn();                                                                   \
  static ::ffx_shim::Registrar FFX_SHIM_CAT(fn, _reg)(name, __FILE__, __LINE__, &fn); \
  static void fn()
#define TEST_CASE(name) FFX_SHIM_TC(FFX_SHIM_CAT(ffx_shim_tc_, __COUNTER__), name)

#define SUBCASE(name) if (::ffx_shim::Subcase ffx_shim_sc{name}; ffx_shim_sc.entered)

#define CHECK(...) ::ffx_shim::report(static_cast<bool>(__VA_ARGS__), "CHECK", #__VA_ARGS__, __FILE__, __LINE__)
#define CHECK_FALSE(...) ::ffx_shim::report(!static_cast<bool>(__VA_ARGS__), "CHECK_FALSE", #__VA_ARGS__, __FILE__, __LINE__)
#define REQUIRE(...)                                                                   \
  do {                                                                                 \
    const bool ffx_shim_ok = static_cast<bool>(__VA_ARGS__);                           \
    ::ffx_shim::report(ffx_shim_ok, "REQUIRE", #__VA_ARGS__, __FILE__, __LINE__);      \
    if (!ffx_shim_ok) throw ::ffx_shim::RequireFailed{};                               \
  } while (0)
#define CHECK_THROWS_AS(expr, ...)                                                     \
  do {                                                                                 \
    bool ffx_shim_ok = false;                                                          \
    try {                                                                              \
      (void)(expr);                                                                    \
    } catch (const __VA_ARGS__&) {                                                     \
      ffx_shim_ok = true;                                                              \
    } catch (...) {                                                                    \
    }                                                                                  \
    ::ffx_shim::report(ffx_shim_ok, "CHECK_THROWS_AS", #expr ", " #__VA_ARGS__, __FILE__, __LINE__); \
  } while (0)
#define CHECK_NOTHROW(...)                                                             \
  do {                                                                                 \
    bool ffx_shim_ok = true;                                                           \
    try {                                                                              \
      (void)(__VA_ARGS__);                                                             \
    } catch (...) {                                                                    \
      ffx_shim_ok = false;                                                             \
    }                                                                                  \
    ::ffx_shim::report(ffx_shim_ok, "CHECK_NOTHROW", #__VA_ARGS__, __FILE__, __LINE__); \
  } while (0)
#define CAPTURE(...) ((void)0)
#define MESSAGE(...) ((void)0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main(int argc, char** argv) { return ::ffx_shim::run_all(argc, argv); }
#endif
