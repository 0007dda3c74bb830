// Minimal doctest-compatible test harness (TEST INFRASTRUCTURE ONLY).
//
// The reference's own C++ test suites (/root/reference/proj/tests/*.cpp) are
// written for doctest, which is not vendored with the reference.  This shim
// implements the subset they use — TEST_CASE, CHECK, REQUIRE, CHECK_THROWS_AS,
// FAIL, CAPTURE, doctest::Approx(...).epsilon(...) and
// DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN — so those suites can be compiled,
// unmodified, against flute-b200's drop-in headers and libflute_b200.so
// (tests/refsuite/Makefile).  Written from the doctest API surface, not from
// doctest's sources.
#pragma once

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <exception>
#include <functional>
#include <sstream>
#include <string>
#include <vector>

namespace doctest {

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
    registry().push_back({name, file, line, fn});
  }
};

struct RequireFailed {};

struct State {
  long checks = 0, failed_checks = 0;
  bool case_failed = false;
  std::vector<std::string> captures;
};
inline State& state() {
  static State s;
  return s;
}

inline void report(const char* file, int line, const std::string& what) {
  State& s = state();
  ++s.failed_checks;
  s.case_failed = true;
  std::fprintf(stderr, "%s:%d: FAILED: %s\n", file, line, what.c_str());
  for (const std::string& c : s.captures) std::fprintf(stderr, "    with %s\n", c.c_str());
}

struct CaptureGuard {
  explicit CaptureGuard(std::string s) { state().captures.push_back(std::move(s)); }
  ~CaptureGuard() { state().captures.pop_back(); }
};

class Approx {
 public:
  explicit Approx(double v) : value_(v) {}
  Approx& epsilon(double e) {
    eps_ = e;
    return *this;
  }
  bool matches(double other) const {
    return std::fabs(other - value_) <= eps_ * (1.0 + std::fmax(std::fabs(other), std::fabs(value_)));
  }
  double value() const { return value_; }

 private:
  double value_;
  double eps_ = 1e-5;  // doctest's default epsilon (scale * FLT_EPSILON * 100)
};
inline bool operator==(double lhs, const Approx& rhs) { return rhs.matches(lhs); }
inline bool operator==(const Approx& lhs, double rhs) { return lhs.matches(rhs); }
inline bool operator!=(double lhs, const Approx& rhs) { return !rhs.matches(lhs); }
inline bool operator!=(const Approx& lhs, double rhs) { return !lhs.matches(rhs); }
inline bool operator<=(double lhs, const Approx& rhs) { return lhs <= rhs.value() || rhs.matches(lhs); }
inline bool operator>=(double lhs, const Approx& rhs) { return lhs >= rhs.value() || rhs.matches(lhs); }
inline std::ostream& operator<<(std::ostream& os, const Approx& a) {
  return os << "Approx(" << a.value() << ")";
}

// REFSUITE_SKIP: comma-separated test-name prefixes to skip (e.g. the GPU
// suites "engine:,mma:" on a host without a GPU).
inline bool skipped(const char* name) {
  const char* env = std::getenv("REFSUITE_SKIP");
  if (!env) return false;
  std::string list(env), nm(name);
  size_t pos = 0;
  while (pos <= list.size()) {
    const size_t end = list.find(',', pos);
    const std::string pre = list.substr(pos, end == std::string::npos ? std::string::npos : end - pos);
    if (!pre.empty() && nm.compare(0, pre.size(), pre) == 0) return true;
    if (end == std::string::npos) break;
    pos = end + 1;
  }
  return false;
}

inline int run_all() {
  int failed_cases = 0;
  size_t ran = 0;
  for (const TestCase& tc : registry()) {
    if (skipped(tc.name)) continue;
    ++ran;
    State& s = state();
    s.case_failed = false;
    try {
      tc.fn();
    } catch (const RequireFailed&) {
    } catch (const std::exception& e) {
      report(tc.file, tc.line, std::string("unexpected exception: ") + e.what());
    } catch (...) {
      report(tc.file, tc.line, "unexpected non-std exception");
    }
    if (s.case_failed) {
      ++failed_cases;
      std::fprintf(stderr, "[case FAILED] %s\n", tc.name);
    }
  }
  std::printf("[refsuite] test cases: %zu | %zu passed | %d failed | %zu skipped\n", ran,
              ran - failed_cases, failed_cases, registry().size() - ran);
  std::printf("[refsuite] assertions: %ld | %ld passed | %ld failed\n", state().checks,
              state().checks - state().failed_checks, state().failed_checks);
  return failed_cases == 0 ? 0 : 1;
}

}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define DOCTEST_TEST_CASE_IMPL(fn, name)                                                 \
  static void fn();                                                                      \
  static doctest::Registrar DOCTEST_CAT(fn, _reg)(name, __FILE__, __LINE__, &fn);        \
  static void fn()
#define TEST_CASE(name) DOCTEST_TEST_CASE_IMPL(DOCTEST_CAT(doctest_case_, __LINE__), name)

#define DOCTEST_ASSERT_(expr, fatal)                                                     \
  do {                                                                                   \
    ++doctest::state().checks;                                                           \
    bool doctest_ok_ = false;                                                            \
    try {                                                                                \
      doctest_ok_ = static_cast<bool>(expr);                                             \
    } catch (const std::exception& e) {                                                  \
      doctest::report(__FILE__, __LINE__, std::string(#expr) + " threw " + e.what());    \
      if (fatal) throw doctest::RequireFailed{};                                         \
      break;                                                                             \
    }                                                                                    \
    if (!doctest_ok_) {                                                                  \
      doctest::report(__FILE__, __LINE__, #expr);                                        \
      if (fatal) throw doctest::RequireFailed{};                                         \
    }                                                                                    \
  } while (0)
#define CHECK(...) DOCTEST_ASSERT_((__VA_ARGS__), false)
#define REQUIRE(...) DOCTEST_ASSERT_((__VA_ARGS__), true)
#define CHECK_THROWS_AS(expr, exc)                                                       \
  do {                                                                                   \
    ++doctest::state().checks;                                                           \
    bool doctest_caught_ = false;                                                        \
    try {                                                                                \
      (void)(expr);                                                                      \
    } catch (const exc&) {                                                               \
      doctest_caught_ = true;                                                            \
    } catch (...) {                                                                      \
    }                                                                                    \
    if (!doctest_caught_) doctest::report(__FILE__, __LINE__, #expr " did not throw " #exc); \
  } while (0)
#define FAIL(msg)                                                                        \
  do {                                                                                   \
    std::ostringstream doctest_os_;                                                      \
    doctest_os_ << msg;                                                                  \
    doctest::report(__FILE__, __LINE__, doctest_os_.str());                              \
    throw doctest::RequireFailed{};                                                      \
  } while (0)
#define CAPTURE(x)                                                                       \
  std::ostringstream DOCTEST_CAT(doctest_cap_os_, __LINE__);                             \
  DOCTEST_CAT(doctest_cap_os_, __LINE__) << #x " := " << (x);                            \
  doctest::CaptureGuard DOCTEST_CAT(doctest_cap_, __LINE__)(DOCTEST_CAT(doctest_cap_os_, __LINE__).str())

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() { return doctest::run_all(); }
#endif
