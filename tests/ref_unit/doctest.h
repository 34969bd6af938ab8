// Minimal doctest-compatible shim (TEST INFRASTRUCTURE): just enough of the
// doctest API for the reference's unit tests (/root/reference/proj/tests/*.cpp)
// to compile unchanged against stitch-b200's headers and run against
// libstitch_b200.so.  doctest itself is not vendored upstream (proj/.gitignore)
// and is absent from this image.
#pragma once
#include <cmath>
#include <cstdio>
#include <cstring>
#include <exception>
#include <functional>
#include <sstream>
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
struct RequireFail {};
struct State {
  int checks = 0, failed_checks = 0;
  std::vector<std::string> captures;
  bool case_failed = false;
};
inline State& st() {
  static State s;
  return s;
}
inline void report(bool ok, const char* kind, const char* expr, const char* file, int line) {
  ++st().checks;
  if (ok) return;
  ++st().failed_checks;
  st().case_failed = true;
  std::fprintf(stderr, "%s:%d: %s( %s ) FAILED\n", file, line, kind, expr);
  for (auto& c : st().captures) std::fprintf(stderr, "    with %s\n", c.c_str());
}
struct Capture {
  template <typename T>
  Capture(const char* name, const T& v) {
    std::ostringstream os;
    os << name << " := " << v;
    st().captures.push_back(os.str());
  }
  ~Capture() { st().captures.pop_back(); }
};
}  // namespace doctest_shim

namespace doctest {
struct Approx {
  explicit Approx(double v) : value(v) {}
  Approx& epsilon(double e) {
    eps = e;
    return *this;
  }
  Approx& scale(double s) {
    scl = s;
    return *this;
  }
  double value, eps = 1.1920928955078125e-05 * 100 / 100, scl = 1.0;
  friend bool operator==(double lhs, const Approx& a) {
    return std::fabs(lhs - a.value) < a.eps * (a.scl + std::max(std::fabs(lhs), std::fabs(a.value)));
  }
  friend bool operator==(const Approx& a, double rhs) { return rhs == a; }
  friend bool operator!=(double lhs, const Approx& a) { return !(lhs == a); }
  friend bool operator!=(const Approx& a, double rhs) { return !(rhs == a); }
  friend std::ostream& operator<<(std::ostream& os, const Approx& a) { return os << "Approx(" << a.value << ")"; }
};
}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define DOCTEST_TC_(fn, reg, name)                                             \
  static void fn();                                                            \
  static doctest_shim::Reg reg(name, &fn, __FILE__, __LINE__);                 \
  static void fn()
#define TEST_CASE(name) DOCTEST_TC_(DOCTEST_CAT(dt_fn_, __COUNTER__), DOCTEST_CAT(dt_reg_, __LINE__), name)
#define CHECK(...) doctest_shim::report(static_cast<bool>(__VA_ARGS__), "CHECK", #__VA_ARGS__, __FILE__, __LINE__)
#define CHECK_FALSE(...) doctest_shim::report(!static_cast<bool>(__VA_ARGS__), "CHECK_FALSE", #__VA_ARGS__, __FILE__, __LINE__)
#define REQUIRE(...)                                                           \
  do {                                                                         \
    const bool ok_ = static_cast<bool>(__VA_ARGS__);                           \
    doctest_shim::report(ok_, "REQUIRE", #__VA_ARGS__, __FILE__, __LINE__);    \
    if (!ok_) throw doctest_shim::RequireFail{};                               \
  } while (0)
#define CHECK_THROWS(...)                                                      \
  do {                                                                         \
    bool threw_ = false;                                                       \
    try { (void)(__VA_ARGS__); } catch (...) { threw_ = true; }                \
    doctest_shim::report(threw_, "CHECK_THROWS", #__VA_ARGS__, __FILE__, __LINE__); \
  } while (0)
#define CHECK_THROWS_AS(expr, ...)                                             \
  do {                                                                         \
    bool threw_ = false;                                                       \
    try { (void)(expr); } catch (const __VA_ARGS__&) { threw_ = true; } catch (...) {} \
    doctest_shim::report(threw_, "CHECK_THROWS_AS", #expr, __FILE__, __LINE__); \
  } while (0)
#define CHECK_NOTHROW(...)                                                     \
  do {                                                                         \
    bool ok_ = true;                                                           \
    try { (void)(__VA_ARGS__); } catch (...) { ok_ = false; }                  \
    doctest_shim::report(ok_, "CHECK_NOTHROW", #__VA_ARGS__, __FILE__, __LINE__); \
  } while (0)
#define CAPTURE(x) doctest_shim::Capture DOCTEST_CAT(dt_cap_, __LINE__)(#x, x)
#define FAIL(msg)                                                              \
  do {                                                                         \
    std::ostringstream os_;                                                    \
    os_ << msg;                                                                \
    doctest_shim::report(false, "FAIL", os_.str().c_str(), __FILE__, __LINE__); \
    throw doctest_shim::RequireFail{};                                         \
  } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
// usage: unit_tests [--exclude=substr,substr] [--only=substr]
int main(int argc, char** argv) {
  std::vector<std::string> exclude, only;
  for (int i = 1; i < argc; ++i) {
    std::string a = argv[i];
    auto split = [](const std::string& v, std::vector<std::string>& out) {
      std::stringstream ss(v);
      for (std::string t; std::getline(ss, t, ',');) if (!t.empty()) out.push_back(t);
    };
    if (a.rfind("--exclude=", 0) == 0) split(a.substr(10), exclude);
    if (a.rfind("--only=", 0) == 0) split(a.substr(7), only);
  }
  int run = 0, failed = 0, skipped = 0;
  for (auto& c : doctest_shim::registry()) {
    std::string n = c.name;
    bool skip = false;
    for (auto& e : exclude) skip = skip || n.find(e) != std::string::npos;
    if (!only.empty()) {
      bool hit = false;
      for (auto& o : only) hit = hit || n.find(o) != std::string::npos;
      skip = skip || !hit;
    }
    if (skip) { ++skipped; continue; }
    ++run;
    doctest_shim::st().case_failed = false;
    try {
      c.fn();
    } catch (const doctest_shim::RequireFail&) {
    } catch (const std::exception& e) {
      std::fprintf(stderr, "%s:%d: TEST CASE \"%s\" threw: %s\n", c.file, c.line, c.name, e.what());
      doctest_shim::st().case_failed = true;
    }
    if (doctest_shim::st().case_failed) {
      ++failed;
      std::fprintf(stderr, "FAILED: %s\n", c.name);
    }
  }
  std::printf("[doctest-shim] test cases: %d run, %d passed, %d failed, %d skipped | checks: %d, failed %d\n",
              run, run - failed, failed, skipped, doctest_shim::st().checks, doctest_shim::st().failed_checks);
  return failed ? 1 : 0;
}
#endif
