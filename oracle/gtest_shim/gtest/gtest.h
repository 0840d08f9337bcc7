// oracle/gtest_shim/gtest/gtest.h -- TEST INFRASTRUCTURE.
//
// GoogleTest is not installed in this image (proj/tests/CMakeLists.txt:1
// requires it).  This header provides the subset of the gtest API the
// reference suites use (TEST, EXPECT_/ASSERT_ EQ NE LT LE GT GE NEAR
// DOUBLE_EQ TRUE FALSE THROW, streamed failure messages) so that
// /root/reference/proj/tests/*.cc compile unmodified, in place
// (oracle/Makefile).  gtest_main.cpp runs the registered tests with
// --gtest_filter=POS[:POS...][-NEG[:NEG...]] and gtest-style output; the exit
// status is nonzero when any test fails.
#ifndef QRTEBD_GTEST_SHIM_H
#define QRTEBD_GTEST_SHIM_H

#include <cmath>
#include <cstdint>
#include <cstring>
#include <functional>
#include <sstream>
#include <string>
#include <type_traits>
#include <utility>
#include <vector>

namespace gtshim {

struct TestInfo {
  std::string suite, name;
  void (*fn)();
};
std::vector<TestInfo>& registry();
void record_failure(const char* file, int line, const std::string& what, const std::string& msg);

struct Registrar {
  Registrar(const char* suite, const char* name, void (*fn)()) { registry().push_back({suite, name, fn}); }
};

template <class T, class = void>
struct printable : std::false_type {};
template <class T>
struct printable<T, std::void_t<decltype(std::declval<std::ostream&>() << std::declval<const T&>())>>
    : std::true_type {};

template <class T>
std::string show(const T& v) {
  if constexpr (std::is_enum<T>::value) {
    return std::to_string(static_cast<long long>(v));
  } else if constexpr (printable<T>::value) {
    std::ostringstream os;
    os.precision(17);
    os << v;
    return os.str();
  } else {
    return "<value>";
  }
}

struct Message {
  std::ostringstream ss;
  template <class T>
  Message& operator<<(const T& v) {
    ss << v;
    return *this;
  }
};

struct AssertHelper {
  const char* file;
  int line;
  std::string what;
  void operator=(const Message& m) const { record_failure(file, line, what, m.ss.str()); }
};

struct Result {
  bool ok;
  std::string what;
};

template <class A, class B, class Op>
Result cmp(const A& a, const B& b, Op op, const char* sa, const char* sb, const char* opname) {
  if (op(a, b)) return {true, {}};
  return {false, std::string("Expected: (") + sa + ") " + opname + " (" + sb + "), actual: " + show(a) + " vs " +
                     show(b)};
}

inline Result near(double a, double b, double tol, const char* sa, const char* sb, const char* st) {
  const double diff = std::fabs(a - b);
  if (diff <= tol) return {true, {}};
  return {false, std::string("The difference between ") + sa + " and " + sb + " is " + show(diff) + ", which exceeds " +
                     st + ", where " + sa + " = " + show(a) + ", " + sb + " = " + show(b) + ", " + st + " = " +
                     show(tol)};
}

inline uint64_t biased_(double x) {
  // gtest's SignAndMagnitudeToBiased: ordered integer image of a double
  uint64_t u;
  std::memcpy(&u, &x, sizeof(u));
  const uint64_t sign = 1ULL << 63;
  return (u & sign) ? (~u + 1) : (u | sign);
}

inline Result double_eq(double a, double b, const char* sa, const char* sb) {
  // gtest's AlmostEquals: within 4 units in the last place
  if (!std::isnan(a) && !std::isnan(b)) {
    const uint64_t ua = biased_(a), ub = biased_(b);
    if ((ua > ub ? ua - ub : ub - ua) <= 4) return {true, {}};
  }
  return {false, std::string("Expected equality of ") + sa + " and " + sb + ": " + show(a) + " vs " + show(b)};
}

}  // namespace gtshim

#define GTSHIM_CAT_(a, b) a##b
#define GTSHIM_CAT(a, b) GTSHIM_CAT_(a, b)

#define TEST(suite, name)                                                                                  \
  static void GTSHIM_CAT(gtshim_test_##suite##_, name)();                                                  \
  static ::gtshim::Registrar GTSHIM_CAT(gtshim_reg_##suite##_, name)(#suite, #name,                        \
                                                                     &GTSHIM_CAT(gtshim_test_##suite##_, name)); \
  static void GTSHIM_CAT(gtshim_test_##suite##_, name)()

#define GTSHIM_CHECK_(result_expr, fail_action)                                                      \
  if (::gtshim::Result gtshim_r_ = (result_expr); gtshim_r_.ok)                                      \
    ;                                                                                                \
  else                                                                                               \
    fail_action ::gtshim::AssertHelper{__FILE__, __LINE__, gtshim_r_.what} = ::gtshim::Message()

#define GTSHIM_OP_(a, b, op, name, act) \
  GTSHIM_CHECK_(::gtshim::cmp((a), (b), [](const auto& x, const auto& y) { return x op y; }, #a, #b, name), act)

#define EXPECT_EQ(a, b) GTSHIM_OP_(a, b, ==, "==", )
#define EXPECT_NE(a, b) GTSHIM_OP_(a, b, !=, "!=", )
#define EXPECT_LT(a, b) GTSHIM_OP_(a, b, <, "<", )
#define EXPECT_LE(a, b) GTSHIM_OP_(a, b, <=, "<=", )
#define EXPECT_GT(a, b) GTSHIM_OP_(a, b, >, ">", )
#define EXPECT_GE(a, b) GTSHIM_OP_(a, b, >=, ">=", )
#define ASSERT_EQ(a, b) GTSHIM_OP_(a, b, ==, "==", return)
#define ASSERT_NE(a, b) GTSHIM_OP_(a, b, !=, "!=", return)
#define ASSERT_LT(a, b) GTSHIM_OP_(a, b, <, "<", return)
#define ASSERT_LE(a, b) GTSHIM_OP_(a, b, <=, "<=", return)
#define ASSERT_GT(a, b) GTSHIM_OP_(a, b, >, ">", return)
#define ASSERT_GE(a, b) GTSHIM_OP_(a, b, >=, ">=", return)
#define EXPECT_NEAR(a, b, tol) GTSHIM_CHECK_(::gtshim::near((a), (b), (tol), #a, #b, #tol), )
#define ASSERT_NEAR(a, b, tol) GTSHIM_CHECK_(::gtshim::near((a), (b), (tol), #a, #b, #tol), return)
#define EXPECT_DOUBLE_EQ(a, b) GTSHIM_CHECK_(::gtshim::double_eq((a), (b), #a, #b), )
#define ASSERT_DOUBLE_EQ(a, b) GTSHIM_CHECK_(::gtshim::double_eq((a), (b), #a, #b), return)
#define EXPECT_TRUE(c) \
  GTSHIM_CHECK_((::gtshim::Result{static_cast<bool>(c), std::string("Value of: ") + #c + "\n  Actual: false"}), )
#define EXPECT_FALSE(c) \
  GTSHIM_CHECK_((::gtshim::Result{!static_cast<bool>(c), std::string("Value of: ") + #c + "\n  Actual: true"}), )
#define ASSERT_TRUE(c) \
  GTSHIM_CHECK_((::gtshim::Result{static_cast<bool>(c), std::string("Value of: ") + #c + "\n  Actual: false"}), return)
#define ASSERT_FALSE(c) \
  GTSHIM_CHECK_((::gtshim::Result{!static_cast<bool>(c), std::string("Value of: ") + #c + "\n  Actual: true"}), return)

#define GTSHIM_THROW_(stmt, type, act)                                                                     \
  GTSHIM_CHECK_(([&]() -> ::gtshim::Result {                                                               \
                  try {                                                                                    \
                    stmt;                                                                                  \
                  } catch (const type&) {                                                                  \
                    return {true, {}};                                                                     \
                  } catch (...) {                                                                          \
                    return {false, std::string("Expected: " #stmt " throws " #type "; it threw another type")}; \
                  }                                                                                        \
                  return {false, std::string("Expected: " #stmt " throws " #type "; it threw nothing")};   \
                }()),                                                                                      \
                act)
#define EXPECT_THROW(stmt, type) GTSHIM_THROW_(stmt, type, )
#define ASSERT_THROW(stmt, type) GTSHIM_THROW_(stmt, type, return)
#define EXPECT_NO_THROW(stmt)                                                                              \
  GTSHIM_CHECK_(([&]() -> ::gtshim::Result {                                                               \
                  try {                                                                                    \
                    stmt;                                                                                  \
                  } catch (...) {                                                                          \
                    return {false, std::string("Expected: " #stmt " does not throw")};                     \
                  }                                                                                        \
                  return {true, {}};                                                                       \
                }()), )

namespace testing {
inline void InitGoogleTest(int*, char**) {}
}  // namespace testing

#endif
