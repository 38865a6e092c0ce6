// doctest-subset shim (test infrastructure only).
//
// The reference's tests use doctest from a git-ignored vendor/ directory
// (proj/CMakeLists.txt:5, proj/.gitignore:2) that is absent here. This
// header implements the subset those tests and ours use: TEST_CASE,
// CHECK/REQUIRE (+ _FALSE), CHECK_THROWS_AS, FAIL, MESSAGE and
// doctest::Approx with doctest's default epsilon/scale semantics.
// DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN emits a main() that runs every case
// (optionally filtered by a substring given as argv[1]) and returns the
// number of failed cases.
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <exception>
#include <functional>
#include <limits>
#include <string>
#include <vector>

namespace doctest {

class Approx {
 public:
  explicit Approx(double value)
      : value_(value), epsilon_(static_cast<double>(std::numeric_limits<float>::epsilon()) * 100),
        scale_(1.0) {}
  Approx& epsilon(double e) {
    epsilon_ = e;
    return *this;
  }
  Approx& scale(double s) {
    scale_ = s;
    return *this;
  }
  friend bool operator==(double lhs, const Approx& rhs) {
    return std::fabs(lhs - rhs.value_) <
           rhs.epsilon_ * (rhs.scale_ + std::max(std::fabs(lhs), std::fabs(rhs.value_)));
  }
  friend bool operator==(const Approx& lhs, double rhs) { return rhs == lhs; }
  friend bool operator!=(double lhs, const Approx& rhs) { return !(lhs == rhs); }
  friend bool operator!=(const Approx& lhs, double rhs) { return !(rhs == lhs); }

 private:
  double value_, epsilon_, scale_;
};

namespace detail {

struct RequireAbort {};

struct Registry {
  struct Case {
    const char* name;
    void (*fn)();
  };
  std::vector<Case> cases;
  int currentFailures = 0;
  long assertions = 0;
  static Registry& get() {
    static Registry r;
    return r;
  }
};

inline int registerCase(const char* name, void (*fn)()) {
  Registry::get().cases.push_back({name, fn});
  return 0;
}

inline void reportFailure(const char* file, int line, const char* kind, const char* expr) {
  auto& r = Registry::get();
  if (r.currentFailures < 20) std::fprintf(stderr, "%s:%d: %s( %s ) FAILED\n", file, line, kind, expr);
  r.currentFailures++;
}

inline int runAll(int argc, char** argv) {
  const char* filter = argc > 1 ? argv[1] : nullptr;
  int failedCases = 0, ran = 0;
  for (const auto& c : Registry::get().cases) {
    if (filter && !std::strstr(c.name, filter)) continue;
    ++ran;
    Registry::get().currentFailures = 0;
    try {
      c.fn();
    } catch (const RequireAbort&) {
    } catch (const std::exception& e) {
      std::fprintf(stderr, "  unexpected exception: %s\n", e.what());
      Registry::get().currentFailures++;
    }
    const bool ok = Registry::get().currentFailures == 0;
    std::printf("[%s] %s\n", ok ? "PASS" : "FAIL", c.name);
    std::fflush(stdout);
    if (!ok) ++failedCases;
  }
  std::printf("doctest-shim: %d/%d test cases passed, %ld assertions\n", ran - failedCases, ran,
              Registry::get().assertions);
  return failedCases;
}

}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define DOCTEST_TEST_CASE_IMPL(fn, name)                                                  \
  static void fn();                                                                       \
  static const int DOCTEST_CAT(fn, _reg) = doctest::detail::registerCase(name, &fn);       \
  static void fn()
#define TEST_CASE(name) DOCTEST_TEST_CASE_IMPL(DOCTEST_CAT(doctest_case_, __COUNTER__), name)

#define DOCTEST_ASSERT_IMPL(kind, expr, abort)                                   \
  do {                                                                           \
    doctest::detail::Registry::get().assertions++;                              \
    if (!(expr)) {                                                               \
      doctest::detail::reportFailure(__FILE__, __LINE__, kind, #expr);          \
      if (abort) throw doctest::detail::RequireAbort{};                          \
    }                                                                            \
  } while (0)

#define CHECK(...) DOCTEST_ASSERT_IMPL("CHECK", (__VA_ARGS__), false)
#define REQUIRE(...) DOCTEST_ASSERT_IMPL("REQUIRE", (__VA_ARGS__), true)
#define CHECK_FALSE(...) DOCTEST_ASSERT_IMPL("CHECK_FALSE", !(__VA_ARGS__), false)
#define REQUIRE_FALSE(...) DOCTEST_ASSERT_IMPL("REQUIRE_FALSE", !(__VA_ARGS__), true)
#define CHECK_THROWS_AS(expr, exc)                                        \
  do {                                                                    \
    bool doctest_threw_ = false;                                          \
    try {                                                                 \
      expr;                                                               \
    } catch (const exc&) {                                                \
      doctest_threw_ = true;                                              \
    } catch (...) {                                                       \
    }                                                                     \
    DOCTEST_ASSERT_IMPL("CHECK_THROWS_AS", doctest_threw_, false);        \
  } while (0)
#define FAIL(msg)                                                          \
  do {                                                                     \
    doctest::detail::reportFailure(__FILE__, __LINE__, "FAIL", msg);       \
    throw doctest::detail::RequireAbort{};                                 \
  } while (0)
#define MESSAGE(msg) std::printf("  note: %s\n", std::string(msg).c_str())

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main(int argc, char** argv) { return doctest::detail::runAll(argc, argv); }
#endif
