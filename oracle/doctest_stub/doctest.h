// doctest.h -- minimal stand-in for the doctest framework (TEST
// INFRASTRUCTURE ONLY). The reference's unit tests include "doctest.h" from
// an untracked vendor/ directory that is absent here; this
// header provides the subset they use -- TEST_CASE, SUBCASE (flat),
// CHECK, REQUIRE, CHECK_THROWS_AS, CHECK_NOTHROW, CAPTURE -- so that
// tests/unit/test_slab_cache.cpp compiles UNCHANGED against the B200
// drop-in header (include/hps/slab_cache.hpp). Define DOCTEST_STUB_MAIN in
// exactly one translation unit to get main().
#pragma once

#include <cstdio>
#include <exception>
#include <functional>
#include <set>
#include <string>
#include <utility>
#include <vector>

namespace doctest_stub {

struct TestCase {
  const char* name;
  const char* file;
  int line;
  std::function<void()> fn;
};

struct State {
  std::vector<TestCase> cases;
  std::set<std::pair<const char*, int>> done_subcases;  // of the running case
  bool entered_subcase = false;  // a subcase ran in this pass
  long checks = 0, failed_checks = 0;
  bool case_failed = false;
};

inline State& state() {
  static State s;
  return s;
}

struct Register {
  Register(const char* name, const char* file, int line, void (*fn)()) {
    state().cases.push_back({name, file, line, fn});
  }
};

struct RequireFailed {};

// One subcase is entered per pass of its test case; the case is re-run
// until every subcase has run once (flat subcases, as the reference uses).
struct Subcase {
  bool run = false;
  std::pair<const char*, int> id;
  Subcase(const char* file, int line, const char*) : id(file, line) {
    State& s = state();
    if (!s.entered_subcase && !s.done_subcases.count(id)) {
      run = true;
      s.entered_subcase = true;
    }
  }
  ~Subcase() {
    if (run) state().done_subcases.insert(id);
  }
  explicit operator bool() const { return run; }
};

inline void report(bool ok, const char* kind, const char* expr, const char* file, int line) {
  State& s = state();
  ++s.checks;
  if (!ok) {
    ++s.failed_checks;
    s.case_failed = true;
    std::fprintf(stderr, "%s:%d: %s( %s ) FAILED\n", file, line, kind, expr);
  }
}

inline int run_all() {
  State& s = state();
  int failed_cases = 0;
  for (const TestCase& tc : s.cases) {
    s.done_subcases.clear();
    s.case_failed = false;
    for (;;) {
      s.entered_subcase = false;
      try {
        tc.fn();
      } catch (const RequireFailed&) {
      } catch (const std::exception& e) {
        std::fprintf(stderr, "%s:%d: test case \"%s\" threw: %s\n", tc.file, tc.line, tc.name,
                     e.what());
        s.case_failed = true;
      }
      if (!s.entered_subcase) break;  // no subcase left to run
    }
    std::fprintf(stderr, "[%s] %s\n", s.case_failed ? "FAIL" : " ok ", tc.name);
    failed_cases += s.case_failed ? 1 : 0;
  }
  std::fprintf(stderr, "test cases: %zu | %zu passed | %d failed; assertions: %ld | %ld failed\n",
               s.cases.size(), s.cases.size() - failed_cases, failed_cases, s.checks,
               s.failed_checks);
  return failed_cases == 0 ? 0 : 1;
}

}  // namespace doctest_stub

#define DOCTEST_STUB_CAT2(a, b) a##b
#define DOCTEST_STUB_CAT(a, b) DOCTEST_STUB_CAT2(a, b)
#define DOCTEST_STUB_TC(fn, name)                                              \
  static void fn();                                                            \
  static doctest_stub::Register DOCTEST_STUB_CAT(fn, _reg)(name, __FILE__, __LINE__, fn); \
  static void fn()
#define TEST_CASE(name) DOCTEST_STUB_TC(DOCTEST_STUB_CAT(doctest_stub_tc_, __LINE__), name)
#define SUBCASE(name) \
  if (doctest_stub::Subcase DOCTEST_STUB_CAT(doctest_stub_sc_, __LINE__){__FILE__, __LINE__, name})
#define CHECK(...) doctest_stub::report(static_cast<bool>(__VA_ARGS__), "CHECK", #__VA_ARGS__, __FILE__, __LINE__)
#define REQUIRE(...)                                                                  \
  do {                                                                                \
    const bool doctest_stub_ok = static_cast<bool>(__VA_ARGS__);                      \
    doctest_stub::report(doctest_stub_ok, "REQUIRE", #__VA_ARGS__, __FILE__, __LINE__); \
    if (!doctest_stub_ok) throw doctest_stub::RequireFailed{};                        \
  } while (0)
#define CHECK_THROWS_AS(expr, ...)                                                   \
  do {                                                                               \
    bool doctest_stub_ok = false;                                                    \
    try {                                                                            \
      expr;                                                                          \
    } catch (const __VA_ARGS__&) {                                                   \
      doctest_stub_ok = true;                                                        \
    } catch (...) {                                                                  \
    }                                                                                \
    doctest_stub::report(doctest_stub_ok, "CHECK_THROWS_AS", #expr ", " #__VA_ARGS__, __FILE__, \
                         __LINE__);                                                  \
  } while (0)
#define CHECK_NOTHROW(...)                                                            \
  do {                                                                                \
    bool doctest_stub_ok = true;                                                      \
    try {                                                                             \
      __VA_ARGS__;                                                                    \
    } catch (...) {                                                                   \
      doctest_stub_ok = false;                                                        \
    }                                                                                 \
    doctest_stub::report(doctest_stub_ok, "CHECK_NOTHROW", #__VA_ARGS__, __FILE__, __LINE__); \
  } while (0)
#define CAPTURE(x) ((void)0)

#ifdef DOCTEST_STUB_MAIN
int main() { return doctest_stub::run_all(); }
#endif
