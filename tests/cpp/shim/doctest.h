// A minimal stand-in for the doctest macros the reference's unit tests use
// (TEST_CASE, CHECK, REQUIRE, FAIL, CAPTURE, CHECK_THROWS_WITH_AS with
// doctest::Contains), so that /root/reference/proj/tests/test_*.cpp compile
// UNCHANGED against the drop-in headers (the doctest library itself is not in
// this image).  Our own code, not doctest's: a registry of test functions, a
// failure counter, and a main() that runs them all and reports like
// "[PASS]/[FAIL] <test name>".
#pragma once

#include <cstdio>
#include <exception>
#include <functional>
#include <sstream>
#include <string>
#include <vector>

namespace doctest {

struct Registry {
  struct Test {
    const char* name;
    const char* file;
    int line;
    void (*fn)();
  };
  std::vector<Test> tests;
  int failures = 0;    // failed checks in the current test
  std::string capture;
  static Registry& get() {
    static Registry r;
    return r;
  }
};

struct Abort {};  // REQUIRE / FAIL: ends the test (not a std::exception, like doctest's)

struct Register {
  Register(const char* name, const char* file, int line, void (*fn)()) {
    Registry::get().tests.push_back({name, file, line, fn});
  }
};

inline void report(const char* file, int line, const char* what) {
  Registry& r = Registry::get();
  ++r.failures;
  std::printf("  %s:%d: check failed: %s%s%s\n", file, line, what,
              r.capture.empty() ? "" : "  [with ", r.capture.empty() ? "" : (r.capture + "]").c_str());
}

struct Contains {
  std::string needle;
  explicit Contains(const char* s) : needle(s) {}
  bool matches(const std::string& s) const { return s.find(needle) != std::string::npos; }
};

template <class... T>
std::string concat(const T&... parts) {
  std::ostringstream os;
  (os << ... << parts);
  return os.str();
}

inline int run_all() {
  Registry& r = Registry::get();
  int failed = 0;
  for (const auto& t : r.tests) {
    r.failures = 0;
    r.capture.clear();
    try {
      t.fn();
    } catch (const Abort&) {
    } catch (const std::exception& e) {
      std::printf("  %s:%d: unexpected exception: %s\n", t.file, t.line, e.what());
      ++r.failures;
    } catch (...) {
      std::printf("  %s:%d: unexpected exception\n", t.file, t.line);
      ++r.failures;
    }
    std::printf("[%s] %s\n", r.failures ? "FAIL" : "PASS", t.name);
    failed += r.failures != 0;
  }
  std::printf("%zu test cases, %d failed\n", r.tests.size(), failed);
  return failed;
}

}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define DOCTEST_TEST_CASE_(fn, name)                                                       \
  static void fn();                                                                        \
  static doctest::Register DOCTEST_CAT(fn, _reg)(name, __FILE__, __LINE__, &fn);           \
  static void fn()
#define TEST_CASE(name) DOCTEST_TEST_CASE_(DOCTEST_CAT(doctest_test_, __LINE__), name)

#define CHECK(...)                                                                         \
  do {                                                                                     \
    if (!(__VA_ARGS__)) doctest::report(__FILE__, __LINE__, #__VA_ARGS__);                 \
  } while (0)
#define REQUIRE(...)                                                                       \
  do {                                                                                     \
    if (!(__VA_ARGS__)) {                                                                  \
      doctest::report(__FILE__, __LINE__, #__VA_ARGS__);                                   \
      throw doctest::Abort{};                                                              \
    }                                                                                      \
  } while (0)
#define FAIL(...)                                                                          \
  do {                                                                                     \
    doctest::report(__FILE__, __LINE__, doctest::concat(__VA_ARGS__).c_str());             \
    throw doctest::Abort{};                                                                \
  } while (0)
#define CAPTURE(x) (doctest::Registry::get().capture = std::string(#x " = ") + (x))
#define CHECK_THROWS_WITH_AS(expr, matcher, type)                                          \
  do {                                                                                     \
    bool thrown_ = false;                                                                  \
    try {                                                                                  \
      (void)(expr);                                                                        \
    } catch (const type& e_) {                                                             \
      thrown_ = true;                                                                      \
      if (!(matcher).matches(e_.what())) doctest::report(__FILE__, __LINE__, #matcher);    \
    } catch (...) {                                                                        \
      thrown_ = true;                                                                      \
      doctest::report(__FILE__, __LINE__, "wrong exception type: " #type);                \
    }                                                                                      \
    if (!thrown_) doctest::report(__FILE__, __LINE__, "no exception: " #expr);             \
  } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() { return doctest::run_all(); }
#endif
