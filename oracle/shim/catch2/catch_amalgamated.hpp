// Minimal Catch2-v3-compatible macro set — TEST INFRASTRUCTURE ONLY (oracle/).
//
// Catch2 is not installed in this image. This header lets
// the reference's own test files (/root/reference/proj/tests/test_*.cpp) be
// compiled unmodified to validate the Eigen shim and pin the oracle. It
// implements TEST_CASE, REQUIRE, REQUIRE_FALSE, REQUIRE_THROWS_AS,
// REQUIRE_NOTHROW, FAIL and Catch::Approx (epsilon/margin) with Catch2's
// comparison rule. Define GROUPOT_SHIM_MAIN in exactly one translation unit.
#pragma once

#include <cmath>
#include <cstdio>
#include <exception>
#include <functional>
#include <limits>
#include <stdexcept>
#include <string>
#include <vector>

namespace Catch {

struct TestFailure : std::exception {
  std::string msg;
  explicit TestFailure(std::string m) : msg(std::move(m)) {}
  const char* what() const noexcept override { return msg.c_str(); }
};

struct TestEntry {
  const char* name;
  void (*fn)();
};

inline std::vector<TestEntry>& registry() {
  static std::vector<TestEntry> r;
  return r;
}

struct Registrar {
  Registrar(const char* name, void (*fn)()) { registry().push_back({name, fn}); }
};

class Approx {
 public:
  explicit Approx(double v)
      : value_(v), epsilon_(std::numeric_limits<float>::epsilon() * 100.0), margin_(0.0) {}
  Approx& epsilon(double e) {
    epsilon_ = e;
    return *this;
  }
  Approx& margin(double m) {
    margin_ = m;
    return *this;
  }
  bool equals(double other) const {
    const auto within = [](double a, double b, double m) {
      return (a + m >= b) && (b + m >= a);
    };
    return within(value_, other, margin_) ||
           within(value_, other,
                  epsilon_ * (std::isinf(value_) ? 0.0 : std::fabs(value_)));
  }

 private:
  double value_;
  double epsilon_;
  double margin_;
};
inline bool operator==(double lhs, const Approx& rhs) { return rhs.equals(lhs); }
inline bool operator==(const Approx& lhs, double rhs) { return lhs.equals(rhs); }

inline void fail_at(const char* file, int line, const std::string& what) {
  throw TestFailure(std::string(file) + ":" + std::to_string(line) + ": " + what);
}

}  // namespace Catch

#define GROUPOT_CAT2(a, b) a##b
#define GROUPOT_CAT(a, b) GROUPOT_CAT2(a, b)
#define GROUPOT_TC_IMPL(fn, name)                                     \
  static void fn();                                                   \
  static ::Catch::Registrar GROUPOT_CAT(fn, _reg)(name, &fn);         \
  static void fn()
#define TEST_CASE(name, ...) GROUPOT_TC_IMPL(GROUPOT_CAT(groupot_tc_, __LINE__), name)

#define REQUIRE(...)                                                         \
  do {                                                                       \
    if (!(__VA_ARGS__)) ::Catch::fail_at(__FILE__, __LINE__, "REQUIRE(" #__VA_ARGS__ ")"); \
  } while (0)
#define REQUIRE_FALSE(...)                                                   \
  do {                                                                       \
    if ((__VA_ARGS__)) ::Catch::fail_at(__FILE__, __LINE__, "REQUIRE_FALSE(" #__VA_ARGS__ ")"); \
  } while (0)
#define REQUIRE_THROWS_AS(expr, type)                                        \
  do {                                                                       \
    bool groupot_caught = false;                                             \
    try {                                                                    \
      (void)(expr);                                                          \
    } catch (const type&) {                                                  \
      groupot_caught = true;                                                 \
    }                                                                        \
    if (!groupot_caught)                                                     \
      ::Catch::fail_at(__FILE__, __LINE__, "REQUIRE_THROWS_AS(" #expr ", " #type ")"); \
  } while (0)
#define REQUIRE_NOTHROW(...)                                                 \
  do {                                                                       \
    try {                                                                    \
      (void)(__VA_ARGS__);                                                   \
    } catch (...) {                                                          \
      ::Catch::fail_at(__FILE__, __LINE__, "REQUIRE_NOTHROW(" #__VA_ARGS__ ")"); \
    }                                                                        \
  } while (0)
#define FAIL(msg) ::Catch::fail_at(__FILE__, __LINE__, std::string("FAIL: ") + (msg))

#ifdef GROUPOT_SHIM_MAIN
int main() {
  int failed = 0;
  int passed = 0;
  for (const auto& t : ::Catch::registry()) {
    try {
      t.fn();
      ++passed;
    } catch (const ::Catch::TestFailure& e) {
      ++failed;
      std::fprintf(stderr, "FAILED: %s\n  %s\n", t.name, e.what());
    } catch (const std::exception& e) {
      ++failed;
      std::fprintf(stderr, "FAILED: %s\n  unexpected exception: %s\n", t.name, e.what());
    }
  }
  std::printf("%d test cases passed, %d failed\n", passed, failed);
  return failed == 0 ? 0 : 1;
}
#endif
