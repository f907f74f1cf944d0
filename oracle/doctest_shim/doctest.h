// TEST INFRASTRUCTURE (oracle only). Self-written stand-in for the subset of
// the doctest single-header API used by the reference's unit suites
// (proj/tests/*.cpp): TEST_SUITE_BEGIN/END, TEST_CASE, CHECK, CHECK_FALSE,
// REQUIRE, CAPTURE, FAIL, CHECK_THROWS_AS, CHECK_THROWS_WITH_AS,
// CHECK_NOTHROW, doctest::Approx(..).epsilon(..), doctest::Contains, and a
// main() honouring `-ts=<suite>` like the reference's ctest entries
// (proj/tests/CMakeLists.txt:16-19). doctest itself is not vendored in the
// reference (proj/CMakeLists.txt:21-28) and is absent from this image.
#pragma once

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <exception>
#include <functional>
#include <iostream>
#include <limits>
#include <mutex>
#include <sstream>
#include <string>
#include <vector>

namespace doctest {

class Approx {
 public:
  explicit Approx(double v) : value_(v) {}
  Approx& epsilon(double e) { eps_ = e; return *this; }
  Approx& scale(double s) { scale_ = s; return *this; }
  friend bool operator==(double lhs, const Approx& rhs) {
    return std::fabs(lhs - rhs.value_) <
           rhs.eps_ * (rhs.scale_ + std::max(std::fabs(lhs), std::fabs(rhs.value_)));
  }
  friend bool operator==(const Approx& lhs, double rhs) { return rhs == lhs; }
  friend bool operator!=(double lhs, const Approx& rhs) { return !(lhs == rhs); }
  friend bool operator!=(const Approx& lhs, double rhs) { return !(rhs == lhs); }
  friend bool operator<=(double lhs, const Approx& rhs) { return lhs < rhs.value_ || lhs == rhs; }
  friend bool operator>=(double lhs, const Approx& rhs) { return lhs > rhs.value_ || lhs == rhs; }

 private:
  double value_;
  double eps_ = static_cast<double>(std::numeric_limits<float>::epsilon()) * 100.0;
  double scale_ = 1.0;
};

struct Contains {
  std::string needle;
  explicit Contains(const char* s) : needle(s) {}
  bool matches(const std::string& hay) const { return hay.find(needle) != std::string::npos; }
};

namespace detail {

struct TestCase {
  const char* suite;
  const char* name;
  void (*fn)();
  const char* file;
  int line;
};

inline std::vector<TestCase>& registry() {
  static std::vector<TestCase> r;
  return r;
}
inline const char*& current_suite() {
  static const char* s = "";
  return s;
}
inline int set_suite(const char* s) {
  current_suite() = s;
  return 0;
}
inline int add_test(const char* name, void (*fn)(), const char* file, int line) {
  registry().push_back({current_suite(), name, fn, file, line});
  return 0;
}

struct State {
  std::mutex mu;
  std::atomic<long> asserts{0};
  std::atomic<long> failures{0};
  std::vector<std::string> captures;
};
inline State& state() {
  static State s;
  return s;
}

struct RequireFailed {};

inline void report(bool ok, const char* kind, const char* expr, const char* file,
                   int line, const std::string& extra = {}) {
  State& s = state();
  ++s.asserts;
  if (ok) return;
  ++s.failures;
  std::lock_guard<std::mutex> lk(s.mu);
  std::cerr << file << ":" << line << ": ERROR: " << kind << "( " << expr << " )";
  if (!extra.empty()) std::cerr << " " << extra;
  std::cerr << "\n";
}

struct Capture {
  template <class T>
  Capture(const char* name, const T& v) {
    std::ostringstream ss;
    ss << name << " := " << v;
    std::lock_guard<std::mutex> lk(state().mu);
    state().captures.push_back(ss.str());
  }
};

}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT_IMPL(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_IMPL(a, b)
#define DOCTEST_ANON(x) DOCTEST_CAT(x, __LINE__)

#define TEST_SUITE_BEGIN(name) \
  static const int DOCTEST_ANON(doctest_suite_) = doctest::detail::set_suite(name)
#define TEST_SUITE_END() \
  static const int DOCTEST_ANON(doctest_suite_end_) = doctest::detail::set_suite("")

#define DOCTEST_TEST_CASE_IMPL(fn, name)                                         \
  static void fn();                                                              \
  static const int DOCTEST_CAT(fn, _reg) =                                       \
      doctest::detail::add_test(name, &fn, __FILE__, __LINE__);                  \
  static void fn()
#define TEST_CASE(name) DOCTEST_TEST_CASE_IMPL(DOCTEST_ANON(doctest_test_fn_), name)

#define CHECK(...) doctest::detail::report(static_cast<bool>(__VA_ARGS__), "CHECK", #__VA_ARGS__, __FILE__, __LINE__)
#define CHECK_FALSE(...) doctest::detail::report(!static_cast<bool>(__VA_ARGS__), "CHECK_FALSE", #__VA_ARGS__, __FILE__, __LINE__)
#define REQUIRE(...)                                                                        \
  do {                                                                                      \
    const bool doctest_ok_ = static_cast<bool>(__VA_ARGS__);                                \
    doctest::detail::report(doctest_ok_, "REQUIRE", #__VA_ARGS__, __FILE__, __LINE__);      \
    if (!doctest_ok_) throw doctest::detail::RequireFailed{};                               \
  } while (0)
#define CAPTURE(x) doctest::detail::Capture DOCTEST_ANON(doctest_capture_)(#x, x)
#define FAIL(msg)                                                                           \
  do {                                                                                      \
    std::ostringstream doctest_ss_;                                                         \
    doctest_ss_ << msg;                                                                     \
    doctest::detail::report(false, "FAIL", "", __FILE__, __LINE__, doctest_ss_.str());      \
    throw doctest::detail::RequireFailed{};                                                 \
  } while (0)

#define CHECK_THROWS_AS(expr, ...)                                                         \
  do {                                                                                      \
    bool doctest_ok_ = false;                                                               \
    try { static_cast<void>(expr); } catch (const __VA_ARGS__&) { doctest_ok_ = true; }    \
    catch (...) {}                                                                          \
    doctest::detail::report(doctest_ok_, "CHECK_THROWS_AS", #expr, __FILE__, __LINE__);     \
  } while (0)

#define CHECK_THROWS_WITH_AS(expr, matcher, ...)                                           \
  do {                                                                                      \
    bool doctest_ok_ = false;                                                               \
    std::string doctest_what_;                                                              \
    try { static_cast<void>(expr); } catch (const __VA_ARGS__& e) {                        \
      doctest_what_ = e.what();                                                             \
      doctest_ok_ = (matcher).matches(doctest_what_);                                       \
    } catch (...) {}                                                                        \
    doctest::detail::report(doctest_ok_, "CHECK_THROWS_WITH_AS", #expr, __FILE__, __LINE__, \
                            doctest_what_);                                                 \
  } while (0)

#define CHECK_NOTHROW(...)                                                                  \
  do {                                                                                      \
    bool doctest_ok_ = true;                                                                \
    try { static_cast<void>(__VA_ARGS__); } catch (...) { doctest_ok_ = false; }           \
    doctest::detail::report(doctest_ok_, "CHECK_NOTHROW", #__VA_ARGS__, __FILE__, __LINE__); \
  } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main(int argc, char** argv) {
  std::string suite_filter;
  for (int i = 1; i < argc; ++i) {
    const std::string a = argv[i];
    if (a.rfind("-ts=", 0) == 0) suite_filter = a.substr(4);
    if (a.rfind("--test-suite=", 0) == 0) suite_filter = a.substr(13);
  }
  auto& st = doctest::detail::state();
  int cases = 0, failed_cases = 0;
  for (const auto& tc : doctest::detail::registry()) {
    if (!suite_filter.empty() && suite_filter != tc.suite) continue;
    ++cases;
    const long before = st.failures.load();
    st.captures.clear();
    try {
      tc.fn();
    } catch (const doctest::detail::RequireFailed&) {
    } catch (const std::exception& e) {
      ++st.failures;
      std::cerr << tc.file << ":" << tc.line << ": ERROR: test case THREW exception: "
                << e.what() << "\n";
    } catch (...) {
      ++st.failures;
      std::cerr << tc.file << ":" << tc.line << ": ERROR: test case THREW unknown exception\n";
    }
    if (st.failures.load() != before) {
      ++failed_cases;
      std::cerr << "  in TEST_CASE(\"" << tc.name << "\") [suite " << tc.suite << "]\n";
      for (const auto& c : st.captures) std::cerr << "    captured: " << c << "\n";
    }
  }
  std::printf("[doctest-shim] test cases: %d | %d passed | %d failed | assertions: %ld | %ld failed\n",
              cases, cases - failed_cases, failed_cases, st.asserts.load(), st.failures.load());
  std::printf("[doctest-shim] Status: %s!\n", failed_cases ? "FAILURE" : "SUCCESS");
  return failed_cases ? 1 : 0;
}
#endif
