// gtest_shim -- a minimal GoogleTest-compatible header (TEST INFRASTRUCTURE).
//
// GTest is absent from this image (find_package(GTest REQUIRED),
// proj/CMakeLists.txt:17), so the reference's own unit tests are compiled against
// this shim.  It implements exactly the subset those files use:
// TEST, EXPECT_/ASSERT_ {EQ,NE,LT,LE,GT,GE,TRUE,FALSE,DOUBLE_EQ,NEAR,THROW,NO_THROW},
// FAIL(), and `<<` messages.  Each binary is a single TU, so main() lives here.
#ifndef AIRES_GTEST_SHIM_H
#define AIRES_GTEST_SHIM_H

#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <functional>
#include <sstream>
#include <string>
#include <vector>

namespace testing {

class Message {
 public:
  Message() = default;
  Message(const Message& o) { ss_ << o.ss_.str(); }
  template <class T>
  Message& operator<<(const T& v) {
    ss_ << v;
    return *this;
  }
  std::string str() const { return ss_.str(); }

 private:
  std::ostringstream ss_;
};

namespace internal {

struct TestInfo {
  const char* suite;
  const char* name;
  void (*body)();
};

inline std::vector<TestInfo>& registry() {
  static std::vector<TestInfo> r;
  return r;
}
inline bool& current_failed() {
  static bool f = false;
  return f;
}

struct Registrar {
  Registrar(const char* s, const char* n, void (*b)()) { registry().push_back({s, n, b}); }
};

struct AssertionResult {
  bool ok;
  std::string msg;
  explicit operator bool() const { return ok; }
};

class AssertHelper {
 public:
  AssertHelper(const char* file, int line, std::string msg)
      : file_(file), line_(line), msg_(std::move(msg)) {}
  void operator=(const Message& m) const {
    current_failed() = true;
    std::printf("%s:%d: Failure\n%s\n%s\n", file_, line_, msg_.c_str(), m.str().c_str());
  }

 private:
  const char* file_;
  int line_;
  std::string msg_;
};

template <class T>
std::string Print(const T& v) {
  if constexpr (requires(std::ostream& os, const T& t) { os << t; }) {
    std::ostringstream ss;
    ss.precision(17);
    ss << v;
    return ss.str();
  } else {
    return "<object>";
  }
}

#define GTEST_SHIM_CMP_(NAME, OP)                                                          \
  template <class A, class B>                                                               \
  AssertionResult Cmp##NAME(const char* ea, const char* eb, const A& a, const B& b) {       \
    if (a OP b) return {true, ""};                                                          \
    return {false, std::string("Expected: (") + ea + ") " #OP " (" + eb + "), actual: " +   \
                       Print(a) + " vs " + Print(b)};                                       \
  }
GTEST_SHIM_CMP_(EQ, ==)
GTEST_SHIM_CMP_(NE, !=)
GTEST_SHIM_CMP_(LT, <)
GTEST_SHIM_CMP_(LE, <=)
GTEST_SHIM_CMP_(GT, >)
GTEST_SHIM_CMP_(GE, >=)
#undef GTEST_SHIM_CMP_

inline AssertionResult CmpBool(const char* e, bool v, bool want) {
  if (v == want) return {true, ""};
  return {false, std::string("Value of: ") + e + "\n  Actual: " + (v ? "true" : "false") +
                     "\nExpected: " + (want ? "true" : "false")};
}

// GoogleTest's DOUBLE_EQ: equal within 4 units in the last place.
inline AssertionResult CmpDoubleEq(const char* ea, const char* eb, double a, double b) {
  if (std::isnan(a) || std::isnan(b))
    return {false, std::string(ea) + " or " + eb + " is NaN"};
  auto biased = [](double x) {
    std::uint64_t u;
    std::memcpy(&u, &x, 8);
    const std::uint64_t sign = 1ULL << 63;
    return (u & sign) ? ~u + 1 : (u | sign);
  };
  std::uint64_t x = biased(a), y = biased(b);
  std::uint64_t d = x > y ? x - y : y - x;
  if (d <= 4) return {true, ""};
  return {false, std::string("Expected equality of ") + ea + " and " + eb + ": " + Print(a) +
                     " vs " + Print(b)};
}

inline AssertionResult CmpNear(const char* ea, const char* eb, double a, double b,
                               double tol) {
  if (std::fabs(a - b) <= tol) return {true, ""};
  return {false, std::string("The difference between ") + ea + " and " + eb + " exceeds " +
                     Print(tol) + ": " + Print(a) + " vs " + Print(b)};
}

template <class F>
AssertionResult CheckThrow(F&& f, bool expect_throw, const char* stmt) {
  try {
    f();
  } catch (...) {
    if (expect_throw) return {true, ""};
    return {false, std::string("Expected: ") + stmt + " doesn't throw, but it threw."};
  }
  if (!expect_throw)
    return {true, ""};
  return {false, std::string("Expected: ") + stmt + " throws, but it threw nothing."};
}

}  // namespace internal
}  // namespace testing

#define GTEST_SHIM_FAIL_AT_(msg, RET) \
  RET ::testing::internal::AssertHelper(__FILE__, __LINE__, msg) = ::testing::Message()

#define GTEST_SHIM_CHECK_(expr, RET)                                  \
  if (::testing::internal::AssertionResult gtest_ar_ = (expr)) \
    ;                                                                 \
  else                                                                \
    GTEST_SHIM_FAIL_AT_(gtest_ar_.msg, RET)

#define EXPECT_EQ(a, b) GTEST_SHIM_CHECK_(::testing::internal::CmpEQ(#a, #b, a, b), )
#define EXPECT_NE(a, b) GTEST_SHIM_CHECK_(::testing::internal::CmpNE(#a, #b, a, b), )
#define EXPECT_LT(a, b) GTEST_SHIM_CHECK_(::testing::internal::CmpLT(#a, #b, a, b), )
#define EXPECT_LE(a, b) GTEST_SHIM_CHECK_(::testing::internal::CmpLE(#a, #b, a, b), )
#define EXPECT_GT(a, b) GTEST_SHIM_CHECK_(::testing::internal::CmpGT(#a, #b, a, b), )
#define EXPECT_GE(a, b) GTEST_SHIM_CHECK_(::testing::internal::CmpGE(#a, #b, a, b), )
#define ASSERT_EQ(a, b) GTEST_SHIM_CHECK_(::testing::internal::CmpEQ(#a, #b, a, b), return)
#define ASSERT_NE(a, b) GTEST_SHIM_CHECK_(::testing::internal::CmpNE(#a, #b, a, b), return)
#define ASSERT_LT(a, b) GTEST_SHIM_CHECK_(::testing::internal::CmpLT(#a, #b, a, b), return)
#define ASSERT_LE(a, b) GTEST_SHIM_CHECK_(::testing::internal::CmpLE(#a, #b, a, b), return)
#define ASSERT_GT(a, b) GTEST_SHIM_CHECK_(::testing::internal::CmpGT(#a, #b, a, b), return)
#define ASSERT_GE(a, b) GTEST_SHIM_CHECK_(::testing::internal::CmpGE(#a, #b, a, b), return)
#define EXPECT_TRUE(c) GTEST_SHIM_CHECK_(::testing::internal::CmpBool(#c, static_cast<bool>(c), true), )
#define EXPECT_FALSE(c) GTEST_SHIM_CHECK_(::testing::internal::CmpBool(#c, static_cast<bool>(c), false), )
#define ASSERT_TRUE(c) GTEST_SHIM_CHECK_(::testing::internal::CmpBool(#c, static_cast<bool>(c), true), return)
#define ASSERT_FALSE(c) GTEST_SHIM_CHECK_(::testing::internal::CmpBool(#c, static_cast<bool>(c), false), return)
#define EXPECT_DOUBLE_EQ(a, b) GTEST_SHIM_CHECK_(::testing::internal::CmpDoubleEq(#a, #b, a, b), )
#define ASSERT_DOUBLE_EQ(a, b) GTEST_SHIM_CHECK_(::testing::internal::CmpDoubleEq(#a, #b, a, b), return)
#define EXPECT_NEAR(a, b, t) GTEST_SHIM_CHECK_(::testing::internal::CmpNear(#a, #b, a, b, t), )
#define EXPECT_THROW(stmt, exc) \
  GTEST_SHIM_CHECK_(::testing::internal::CheckThrow([&] { try { (void)(stmt); } catch (const exc&) { throw; } catch (...) { return; } }, true, #stmt), )
#define EXPECT_NO_THROW(stmt) \
  GTEST_SHIM_CHECK_(::testing::internal::CheckThrow([&] { (void)(stmt); }, false, #stmt), )
#define FAIL() GTEST_SHIM_FAIL_AT_("Failed", return)

#define TEST(suite, name)                                                              \
  struct suite##_##name##_Test {                                                       \
    static void Body();                                                                \
  };                                                                                   \
  static ::testing::internal::Registrar suite##_##name##_registrar(#suite, #name,      \
                                                                   &suite##_##name##_Test::Body); \
  void suite##_##name##_Test::Body()

#ifndef GTEST_SHIM_NO_MAIN
int main(int argc, char** argv) {
  const char* filter = nullptr;
  for (int i = 1; i < argc; i++)
    if (std::strncmp(argv[i], "--gtest_filter=", 15) == 0) filter = argv[i] + 15;
  int failed = 0, run = 0;
  for (const auto& t : ::testing::internal::registry()) {
    std::string full = std::string(t.suite) + "." + t.name;
    if (filter && full.find(filter) == std::string::npos) continue;
    ::testing::internal::current_failed() = false;
    std::printf("[ RUN      ] %s\n", full.c_str());
    std::fflush(stdout);
    bool threw = false;
    try {
      t.body();
    } catch (const std::exception& e) {
      threw = true;
      std::printf("uncaught exception: %s\n", e.what());
    } catch (...) {
      threw = true;
      std::printf("uncaught exception\n");
    }
    bool bad = threw || ::testing::internal::current_failed();
    std::printf("%s %s\n", bad ? "[  FAILED  ]" : "[       OK ]", full.c_str());
    run++;
    failed += bad;
  }
  std::printf("[==========] %d tests ran, %d failed\n", run, failed);
  std::printf(failed ? "[  FAILED  ] %d tests\n" : "[  PASSED  ] %d tests\n",
              failed ? failed : run);
  return failed ? 1 : 0;
}
#endif

#endif  // AIRES_GTEST_SHIM_H
