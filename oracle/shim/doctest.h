// oracle/shim/doctest.h -- TEST INFRASTRUCTURE ONLY (oracle build).
// A from-scratch stand-in for the doctest macros the reference unit tests use
// (TEST_CASE, CHECK, CHECK_FALSE, REQUIRE, CHECK_THROWS_AS,
// CHECK_THROWS_WITH_AS, WARN_MESSAGE, doctest::Approx, doctest::Contains).
// doctest itself is absent (vendor/ is gitignored upstream).
// A test binary prints one line per failed check plus a summary, and exits
// non-zero when any check failed.
#pragma once

#include <cmath>
#include <cstdio>
#include <cstring>
#include <exception>
#include <functional>
#include <string>
#include <vector>

namespace doctest {

class Approx {
 public:
  explicit Approx(double v) : v_(v) {}
  Approx& epsilon(double e) { eps_ = e; return *this; }
  friend bool operator==(double lhs, const Approx& a) {
    return std::fabs(lhs - a.v_) <
           a.eps_ * (1.0 + std::fmax(std::fabs(lhs), std::fabs(a.v_)));
  }
  friend bool operator==(const Approx& a, double rhs) { return rhs == a; }
  friend bool operator!=(double lhs, const Approx& a) { return !(lhs == a); }

 private:
  double v_;
  double eps_ = 1.1920928955078125e-07 * 100;  // doctest's default scale
};

struct Contains {
  explicit Contains(const char* s) : s(s) {}
  std::string s;
};

namespace detail {

struct Registry {
  std::vector<std::pair<const char*, void (*)()>> cases;
  long checks = 0, failures = 0, case_failures = 0;
  const char* current = "";
  static Registry& get() { static Registry r; return r; }
};

struct RequireFailure {};

inline void report(bool ok, const char* expr, const char* file, int line,
                   bool fatal) {
  auto& r = Registry::get();
  ++r.checks;
  if (ok) return;
  ++r.failures;
  std::printf("%s:%d: FAILED in \"%s\": %s\n", file, line, r.current, expr);
  if (fatal) throw RequireFailure{};
}

struct Registrar {
  Registrar(const char* name, void (*f)()) {
    Registry::get().cases.emplace_back(name, f);
  }
};

inline bool contains(const std::exception& e, const Contains& c) {
  return std::string(e.what()).find(c.s) != std::string::npos;
}

inline int run_all() {
  auto& r = Registry::get();
  for (auto& [name, f] : r.cases) {
    r.current = name;
    const long before = r.failures;
    try {
      f();
    } catch (const RequireFailure&) {
    } catch (const std::exception& e) {
      ++r.failures;
      std::printf("test \"%s\" threw: %s\n", name, e.what());
    }
    if (r.failures != before) ++r.case_failures;
  }
  std::printf("[doctest-shim] test cases: %zu | %zu passed | %ld failed; "
              "assertions: %ld | %ld failed\n",
              r.cases.size(), r.cases.size() - r.case_failures,
              r.case_failures, r.checks, r.failures);
  return r.failures == 0 ? 0 : 1;
}

}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define DOCTEST_CASE_IMPL(fn, name)                                    \
  static void fn();                                                    \
  static doctest::detail::Registrar DOCTEST_CAT(fn, _reg)(name, &fn); \
  static void fn()
#define TEST_CASE(name) DOCTEST_CASE_IMPL(DOCTEST_CAT(doctest_case_, __COUNTER__), name)

#define CHECK(...) \
  doctest::detail::report(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, false)
#define CHECK_FALSE(...) \
  doctest::detail::report(!static_cast<bool>(__VA_ARGS__), "!(" #__VA_ARGS__ ")", __FILE__, __LINE__, false)
#define REQUIRE(...) \
  doctest::detail::report(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, true)
#define CHECK_THROWS_AS(expr, type)                                            \
  do {                                                                         \
    bool doctest_ok = false;                                                   \
    try { (void)(expr); } catch (const type&) { doctest_ok = true; } catch (...) {} \
    doctest::detail::report(doctest_ok, "throws " #type ": " #expr, __FILE__, __LINE__, false); \
  } while (0)
#define CHECK_THROWS_WITH_AS(expr, matcher, type)                              \
  do {                                                                         \
    bool doctest_ok = false;                                                   \
    try { (void)(expr); } catch (const type& e) {                              \
      doctest_ok = doctest::detail::contains(e, matcher);                      \
    } catch (...) {}                                                           \
    doctest::detail::report(doctest_ok, "throws-with " #type ": " #expr, __FILE__, __LINE__, false); \
  } while (0)
#define WARN_MESSAGE(cond, ...) ((void)(cond))

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() { return doctest::detail::run_all(); }
#endif
