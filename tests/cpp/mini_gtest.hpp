// Minimal GoogleTest-compatible subset (TEST, EXPECT_*/ASSERT_*, EXPECT_THROW) so the
// parity tests read like the reference's own suites (GoogleTest is not installed).
// Filter: argv[1] = substring of "Suite.Name" to run a subset.
#pragma once

#include <cstdio>
#include <cstring>
#include <functional>
#include <sstream>
#include <string>
#include <vector>

namespace mini_gtest {
struct Case {
  std::string name;
  std::function<void()> fn;
};
inline std::vector<Case>& registry() {
  static std::vector<Case> r;
  return r;
}
inline int& failures() {
  static int f = 0;
  return f;
}
struct Reg {
  Reg(const char* s, const char* n, std::function<void()> fn) { registry().push_back({std::string(s) + "." + n, fn}); }
};
struct AssertAbort {};
inline void fail(const char* file, int line, const std::string& msg, bool fatal) {
  std::fprintf(stderr, "%s:%d: Failure: %s\n", file, line, msg.c_str());
  ++failures();
  if (fatal) throw AssertAbort{};
}
template <typename A, typename B>
std::string show(const A& a, const B& b) {
  std::ostringstream os;
  if constexpr (requires { os << a; os << b; }) os << a << " vs " << b;
  return os.str();
}
inline int run_all(int argc, char** argv) {
  int ran = 0;
  for (auto& c : registry()) {
    if (argc > 1 && c.name.find(argv[1]) == std::string::npos) continue;
    const int before = failures();
    try {
      c.fn();
    } catch (const AssertAbort&) {
    } catch (const std::exception& e) {
      fail(__FILE__, __LINE__, std::string("uncaught exception: ") + e.what(), false);
    }
    ++ran;
    std::printf("[%s] %s\n", failures() == before ? "  OK  " : " FAIL ", c.name.c_str());
  }
  std::printf("%d tests, %d failures\n", ran, failures());
  return failures() ? 1 : 0;
}
}  // namespace mini_gtest

#define TEST(S, N)                                                                  \
  static void S##_##N##_body();                                                     \
  static mini_gtest::Reg S##_##N##_reg(#S, #N, S##_##N##_body);                     \
  static void S##_##N##_body()
namespace mini_gtest {
// operands are evaluated as call arguments, so temporaries live through the comparison
template <typename A, typename B, typename Op>
void cmp(const A& a, const B& b, Op op, const char* text, const char* file, int line, bool fatal) {
  if (!op(a, b)) fail(file, line, std::string(text) + " (" + show(a, b) + ")", fatal);
}
}  // namespace mini_gtest
#define MG_CMP(a, b, op, fatal)                                                                         \
  mini_gtest::cmp((a), (b), [](const auto& _x, const auto& _y) { return _x op _y; }, #a " " #op " " #b, \
                  __FILE__, __LINE__, fatal)
#define EXPECT_EQ(a, b) MG_CMP(a, b, ==, false)
#define ASSERT_EQ(a, b) MG_CMP(a, b, ==, true)
#define EXPECT_NE(a, b) MG_CMP(a, b, !=, false)
#define EXPECT_GT(a, b) MG_CMP(a, b, >, false)
#define EXPECT_GE(a, b) MG_CMP(a, b, >=, false)
#define EXPECT_LE(a, b) MG_CMP(a, b, <=, false)
#define EXPECT_LT(a, b) MG_CMP(a, b, <, false)
#define EXPECT_TRUE(c) \
  do { if (!(c)) mini_gtest::fail(__FILE__, __LINE__, "expected true: " #c, false); } while (0)
#define ASSERT_TRUE(c) \
  do { if (!(c)) mini_gtest::fail(__FILE__, __LINE__, "expected true: " #c, true); } while (0)
#define EXPECT_FALSE(c) \
  do { if (c) mini_gtest::fail(__FILE__, __LINE__, "expected false: " #c, false); } while (0)
#define EXPECT_FLOAT_EQ(a, b) MG_CMP(a, b, ==, false)
#define EXPECT_THROW(stmt, exc)                                                                   \
  do {                                                                                            \
    bool _caught = false;                                                                         \
    try { (void)(stmt); } catch (const exc&) { _caught = true; } catch (...) {}                  \
    if (!_caught) mini_gtest::fail(__FILE__, __LINE__, "expected " #exc " from " #stmt, false);   \
  } while (0)
#define EXPECT_NO_THROW(stmt)                                                                     \
  do {                                                                                            \
    try { (void)(stmt); } catch (...) { mini_gtest::fail(__FILE__, __LINE__, "unexpected throw: " #stmt, false); } \
  } while (0)
