// Minimal stand-in for the GoogleTest macros the reference's unit tests use (GTest is not in
// this image). Test infrastructure only: it lets proj/tests/workload_test.cpp compile unchanged
// against include/sparsebalance/*.hpp and run against libsparsebalance_b200.so
// (tests/cpp/Makefile, tests/test_cpp_dropin.py). TEST bodies register themselves; main()
// (define SB_GTEST_MAIN in one translation unit) runs them all and returns non-zero on failure.
#pragma once

#include <cmath>
#include <cstdio>
#include <functional>
#include <iostream>
#include <sstream>
#include <string>
#include <type_traits>
#include <utility>
#include <vector>

namespace sbgt {

struct Case {
  const char* suite;
  const char* name;
  std::function<void()> body;
};

inline std::vector<Case>& registry() {
  static std::vector<Case> r;
  return r;
}
inline int& failures() {
  static int f = 0;
  return f;
}

struct Registrar {
  Registrar(const char* s, const char* n, std::function<void()> b) { registry().push_back({s, n, std::move(b)}); }
};

// Streams the failure message (`<< extra`) and records the failure when destroyed.
struct Failure {
  std::ostringstream msg;
  Failure(const char* file, int line, const std::string& what) { msg << file << ":" << line << ": " << what; }
  template <typename T>
  Failure& operator<<(const T& v) {
    msg << " " << v;
    return *this;
  }
  ~Failure() {
    std::cerr << msg.str() << "\n";
    ++failures();
  }
};

struct Abort {};  // thrown by fatal assertions to leave the test body

struct Fatal {
  Failure f;
  Fatal(const char* file, int line, const std::string& what) : f(file, line, what) {}
  template <typename T>
  Fatal& operator<<(const T& v) {
    f << v;
    return *this;
  }
};
struct FatalThrower {
  // `FatalThrower() = Fatal(...) << x;` : record, then leave the body.
  void operator=(const Fatal&) { throw Abort{}; }
};

template <typename T, typename = void>
struct Streamable : std::false_type {};
template <typename T>
struct Streamable<T, std::void_t<decltype(std::declval<std::ostream&>() << std::declval<const T&>())>>
    : std::true_type {};

template <typename T>
void put(std::ostream& o, const T& v) {
  if constexpr (Streamable<T>::value) {
    o << v;
  } else if constexpr (std::is_enum_v<T>) {
    o << static_cast<long long>(v);
  } else {
    o << "<value>";
  }
}

template <typename A, typename B>
std::string show(const A& a, const B& b) {
  std::ostringstream o;
  o << "(";
  put(o, a);
  o << " vs ";
  put(o, b);
  o << ")";
  return o.str();
}

inline int run_all() {
  int ran = 0;
  for (const Case& c : registry()) {
    const int before = failures();
    try {
      c.body();
    } catch (const Abort&) {
    } catch (const std::exception& e) {
      std::cerr << c.suite << "." << c.name << ": uncaught exception: " << e.what() << "\n";
      ++failures();
    }
    ++ran;
    std::printf("[%s] %s.%s\n", failures() == before ? "  OK  " : " FAIL ", c.suite, c.name);
  }
  std::printf("%d tests, %d failed checks\n", ran, failures());
  return failures() ? 1 : 0;
}

}  // namespace sbgt

#define SBGT_CAT2(a, b) a##b
#define SBGT_CAT(a, b) SBGT_CAT2(a, b)
#define TEST(suite, name)                                                                   \
  static void SBGT_CAT(sbgt_body_, SBGT_CAT(suite, SBGT_CAT(_, name)))();                   \
  static ::sbgt::Registrar SBGT_CAT(sbgt_reg_, SBGT_CAT(suite, SBGT_CAT(_, name)))(          \
      #suite, #name, &SBGT_CAT(sbgt_body_, SBGT_CAT(suite, SBGT_CAT(_, name))));            \
  static void SBGT_CAT(sbgt_body_, SBGT_CAT(suite, SBGT_CAT(_, name)))()

#define SBGT_CHECK(cond, what) \
  if (cond) {                  \
  } else                       \
    ::sbgt::Failure(__FILE__, __LINE__, what)
#define SBGT_FATAL(cond, what) \
  if (cond) {                  \
  } else                       \
    ::sbgt::FatalThrower() = ::sbgt::Fatal(__FILE__, __LINE__, what)

#define SBGT_CMP(a, b, op) ((a)op(b))
#define EXPECT_EQ(a, b) SBGT_CHECK(SBGT_CMP(a, b, ==), "EXPECT_EQ(" #a ", " #b ") " + ::sbgt::show(a, b))
#define EXPECT_NE(a, b) SBGT_CHECK(SBGT_CMP(a, b, !=), "EXPECT_NE(" #a ", " #b ") " + ::sbgt::show(a, b))
#define EXPECT_LT(a, b) SBGT_CHECK(SBGT_CMP(a, b, <), "EXPECT_LT(" #a ", " #b ") " + ::sbgt::show(a, b))
#define EXPECT_LE(a, b) SBGT_CHECK(SBGT_CMP(a, b, <=), "EXPECT_LE(" #a ", " #b ") " + ::sbgt::show(a, b))
#define EXPECT_GT(a, b) SBGT_CHECK(SBGT_CMP(a, b, >), "EXPECT_GT(" #a ", " #b ") " + ::sbgt::show(a, b))
#define EXPECT_GE(a, b) SBGT_CHECK(SBGT_CMP(a, b, >=), "EXPECT_GE(" #a ", " #b ") " + ::sbgt::show(a, b))
#define EXPECT_TRUE(c) SBGT_CHECK((c), "EXPECT_TRUE(" #c ")")
#define EXPECT_FALSE(c) SBGT_CHECK(!(c), "EXPECT_FALSE(" #c ")")
#define EXPECT_DOUBLE_EQ(a, b) SBGT_CHECK((a) == (b), "EXPECT_DOUBLE_EQ(" #a ", " #b ") " + ::sbgt::show(a, b))
#define EXPECT_NEAR(a, b, tol) \
  SBGT_CHECK(std::fabs((a) - (b)) <= (tol), "EXPECT_NEAR(" #a ", " #b ", " #tol ") " + ::sbgt::show(a, b))
#define ASSERT_EQ(a, b) SBGT_FATAL(SBGT_CMP(a, b, ==), "ASSERT_EQ(" #a ", " #b ") " + ::sbgt::show(a, b))
#define ASSERT_NE(a, b) SBGT_FATAL(SBGT_CMP(a, b, !=), "ASSERT_NE(" #a ", " #b ") " + ::sbgt::show(a, b))
#define ASSERT_TRUE(c) SBGT_FATAL((c), "ASSERT_TRUE(" #c ")")
#define ASSERT_GE(a, b) SBGT_FATAL(SBGT_CMP(a, b, >=), "ASSERT_GE(" #a ", " #b ") " + ::sbgt::show(a, b))
#define ASSERT_LE(a, b) SBGT_FATAL(SBGT_CMP(a, b, <=), "ASSERT_LE(" #a ", " #b ") " + ::sbgt::show(a, b))
#define FAIL() ::sbgt::FatalThrower() = ::sbgt::Fatal(__FILE__, __LINE__, "FAIL()")
#define EXPECT_THROW(stmt, exc)                                                        \
  do {                                                                                 \
    bool sbgt_caught_ = false;                                                         \
    try {                                                                              \
      stmt;                                                                            \
    } catch (const exc&) {                                                             \
      sbgt_caught_ = true;                                                             \
    } catch (...) {                                                                    \
    }                                                                                  \
    SBGT_CHECK(sbgt_caught_, "EXPECT_THROW(" #stmt ", " #exc ") did not throw " #exc); \
  } while (0)

#ifdef SB_GTEST_MAIN
int main() { return ::sbgt::run_all(); }
#endif
