// Minimal doctest subset so the reference's own unit tests (read-only, under
// /root/reference/proj/tests) can be compiled against the shim-built
// reference. TEST INFRASTRUCTURE ONLY. Covers TEST_CASE, SUBCASE (re-run
// semantics: each run enters one new leaf), CHECK/REQUIRE families,
// CHECK_THROWS_AS / CHECK_THROWS_WITH_AS with doctest::Contains,
// CHECK_NOTHROW, CAPTURE and FAIL.
#ifndef VEQ_ORACLE_DOCTEST_SHIM_H
#define VEQ_ORACLE_DOCTEST_SHIM_H
#include <cstdio>
#include <exception>
#include <functional>
#include <set>
#include <sstream>
#include <string>
#include <vector>

namespace doctest {
struct Contains {
  std::string s;
  explicit Contains(std::string x) : s(std::move(x)) {}
};
namespace detail {
struct TestCase {
  const char *name;
  const char *file;
  int line;
  void (*fn)();
};
inline std::vector<TestCase> &registry() {
  static std::vector<TestCase> r;
  return r;
}
struct Reg {
  Reg(const char *n, const char *f, int l, void (*fn)()) { registry().push_back({n, f, l, fn}); }
};
struct RequireFailed {};
struct State {
  int failures = 0;
  int assertions = 0;
  const char *cur = "";
  std::set<std::string> done;    // fully explored subcase paths
  std::vector<std::string> path; // subcase stack for this run
  std::vector<bool> entered;     // per depth: a subcase already entered this run
  bool pending = false;          // some subcase skipped this run and not yet done
  std::vector<std::string> captures;
};
inline State &st() {
  static State s;
  return s;
}
inline std::string join(const std::vector<std::string> &p) {
  std::string r;
  for (auto &x : p) r += x + "/";
  return r;
}
struct Subcase {
  bool in = false;
  bool pending_before = false;
  std::string key;
  Subcase(const char *name) {
    State &s = st();
    size_t d = s.path.size();
    if (s.entered.size() <= d) s.entered.resize(d + 1, false);
    std::vector<std::string> p = s.path;
    p.push_back(name);
    key = join(p);
    if (s.done.count(key)) return;
    if (s.entered[d]) {
      s.pending = true;
      return;
    }
    s.entered[d] = true;
    in = true;
    pending_before = s.pending;
    s.pending = false;
    s.path.push_back(name);
    if (s.entered.size() <= d + 1) s.entered.resize(d + 2, false);
    s.entered[d + 1] = false;
  }
  ~Subcase() {
    if (!in) return;
    State &s = st();
    s.path.pop_back();
    if (!s.pending) s.done.insert(key);
    s.pending = s.pending || pending_before;
    if (!s.done.count(key)) s.pending = true;
  }
  explicit operator bool() const { return in; }
};
inline void report(const char *file, int line, const std::string &what) {
  State &s = st();
  s.failures++;
  std::fprintf(stderr, "%s:%d: FAILED in '%s' [%s]: %s\n", file, line, s.cur,
               join(s.path).c_str(), what.c_str());
  for (auto &c : s.captures) std::fprintf(stderr, "  with %s\n", c.c_str());
}
inline bool check(bool ok, const char *file, int line, const char *expr, bool require) {
  st().assertions++;
  if (!ok) {
    report(file, line, expr);
    if (require) throw RequireFailed{};
  }
  return ok;
}
struct CaptureGuard {
  CaptureGuard(std::string s) { st().captures.push_back(std::move(s)); }
  ~CaptureGuard() { st().captures.pop_back(); }
};
template <class T> std::string show(const T &v) {
  std::ostringstream os;
  if constexpr (requires(std::ostream &o, const T &x) { o << x; }) os << v;
  else os << "?";
  return os.str();
}
inline int run_all() {
  State &s = st();
  int failed_cases = 0;
  for (auto &tc : registry()) {
    s.cur = tc.name;
    s.done.clear();
    int before = s.failures;
    for (int iter = 0; iter < 100000; iter++) {
      s.path.clear();
      s.entered.assign(1, false);
      s.pending = false;
      try {
        tc.fn();
      } catch (RequireFailed &) {
      } catch (std::exception &e) {
        report(tc.file, tc.line, std::string("unexpected exception: ") + e.what());
      } catch (...) {
        report(tc.file, tc.line, "unexpected unknown exception");
      }
      if (!s.pending) break;
    }
    if (s.failures != before) failed_cases++;
  }
  std::printf("[doctest-shim] test cases: %zu | failed: %d | assertions: %d | failures: %d\n",
              registry().size(), failed_cases, s.assertions, s.failures);
  return failed_cases ? 1 : 0;
}
} // namespace detail
} // namespace doctest

#define DOCTEST_CAT2(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT2(a, b)
#define DOCTEST_ANON(p) DOCTEST_CAT(p, __LINE__)
#define TEST_CASE(name)                                                        \
  static void DOCTEST_ANON(doctest_fn_)();                                     \
  static ::doctest::detail::Reg DOCTEST_ANON(doctest_reg_)(                    \
      name, __FILE__, __LINE__, &DOCTEST_ANON(doctest_fn_));                   \
  static void DOCTEST_ANON(doctest_fn_)()
#define SUBCASE(name) if (::doctest::detail::Subcase DOCTEST_ANON(doctest_sc_){name})
#define CHECK(...) ::doctest::detail::check(static_cast<bool>(__VA_ARGS__), __FILE__, __LINE__, #__VA_ARGS__, false)
#define CHECK_FALSE(...) ::doctest::detail::check(!static_cast<bool>(__VA_ARGS__), __FILE__, __LINE__, "!(" #__VA_ARGS__ ")", false)
#define REQUIRE(...) ::doctest::detail::check(static_cast<bool>(__VA_ARGS__), __FILE__, __LINE__, #__VA_ARGS__, true)
#define REQUIRE_FALSE(...) ::doctest::detail::check(!static_cast<bool>(__VA_ARGS__), __FILE__, __LINE__, "!(" #__VA_ARGS__ ")", true)
#define CHECK_THROWS_AS(expr, ...)                                             \
  do {                                                                         \
    bool doctest_ok_ = false;                                                  \
    try { (void)(expr); } catch (const __VA_ARGS__ &) { doctest_ok_ = true; } catch (...) {} \
    ::doctest::detail::check(doctest_ok_, __FILE__, __LINE__, "throws " #__VA_ARGS__ ": " #expr, false); \
  } while (0)
#define CHECK_THROWS_WITH_AS(expr, matcher, ...)                               \
  do {                                                                         \
    bool doctest_ok_ = false;                                                  \
    try { (void)(expr); } catch (const __VA_ARGS__ &e) {                       \
      doctest_ok_ = std::string(e.what()).find(::doctest::Contains(matcher).s) != std::string::npos; \
    } catch (...) {}                                                           \
    ::doctest::detail::check(doctest_ok_, __FILE__, __LINE__, "throws-with " #expr, false); \
  } while (0)
#define CHECK_NOTHROW(expr)                                                    \
  do {                                                                         \
    bool doctest_ok_ = true;                                                   \
    try { (void)(expr); } catch (...) { doctest_ok_ = false; }                 \
    ::doctest::detail::check(doctest_ok_, __FILE__, __LINE__, "nothrow " #expr, false); \
  } while (0)
#define CAPTURE(x) ::doctest::detail::CaptureGuard DOCTEST_ANON(doctest_cap_)(std::string(#x " := ") + ::doctest::detail::show(x))
#define FAIL(msg)                                                              \
  do {                                                                         \
    std::ostringstream doctest_os_;                                            \
    doctest_os_ << msg;                                                        \
    ::doctest::detail::report(__FILE__, __LINE__, doctest_os_.str());          \
    throw ::doctest::detail::RequireFailed{};                                  \
  } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() { return ::doctest::detail::run_all(); }
#endif
#endif
