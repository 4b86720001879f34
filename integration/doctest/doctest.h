// doctest.h -- a minimal doctest-compatible test harness (TEST INFRASTRUCTURE).
//
// The reference's unit suites (proj/tests/test_*.cpp) are written against
// doctest, whose single header is not in this image (proj/.gitignore:2 keeps
// vendor/ out of the reference).  This header implements, from scratch, the
// subset those suites use so they can be compiled unmodified and run -- against
// the reference's own CPU code and against the GPU drop-in
// (integration/pixlog_slcs.cpp):
//
//   TEST_CASE, TEST_SUITE_BEGIN/END, SUBCASE (doctest's re-run-per-leaf
//   semantics), CHECK, REQUIRE, REQUIRE_MESSAGE, FAIL, INFO, CHECK_THROWS_AS,
//   CHECK_THROWS_WITH_AS with doctest::Contains, doctest::Approx(..).epsilon(..),
//   DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN, and the command-line filters
//   -tc=<names> / -tce=<names> / -ts=<suites> / -tse=<suites> ('*' wildcards,
//   comma separated) plus -s (report every test case).
#pragma once

#include <cmath>
#include <cstdio>
#include <cstring>
#include <exception>
#include <functional>
#include <limits>
#include <set>
#include <sstream>
#include <string>
#include <vector>

namespace doctest {

struct Contains {
  std::string s;
  explicit Contains(const char* x) : s(x) {}
  explicit Contains(std::string x) : s(std::move(x)) {}
  bool matches(const std::string& what) const { return what.find(s) != std::string::npos; }
};

class Approx {
 public:
  explicit Approx(double v) : v_(v) {}
  Approx& epsilon(double e) {
    eps_ = e;
    return *this;
  }
  Approx& scale(double s) {
    scale_ = s;
    return *this;
  }
  friend bool operator==(double lhs, const Approx& a) {
    return std::fabs(lhs - a.v_) <
           a.eps_ * (a.scale_ + std::max(std::fabs(lhs), std::fabs(a.v_)));
  }
  friend bool operator==(const Approx& a, double rhs) { return rhs == a; }
  friend bool operator!=(double lhs, const Approx& a) { return !(lhs == a); }
  friend bool operator!=(const Approx& a, double rhs) { return !(rhs == a); }

 private:
  double v_;
  double eps_ = double(std::numeric_limits<float>::epsilon()) * 100;
  double scale_ = 1.0;
};

namespace detail {

struct TestCase {
  std::string name, suite, file;
  int line;
  void (*fn)();
};

inline std::vector<TestCase>& registry() {
  static std::vector<TestCase> r;
  return r;
}
inline std::string& currentSuite() {
  static std::string s;
  return s;
}

struct Registrar {
  Registrar(void (*fn)(), const char* name, const char* file, int line) {
    registry().push_back({name, currentSuite(), file, line, fn});
  }
};
struct SuiteSetter {
  explicit SuiteSetter(const char* name) { currentSuite() = name; }
};

// abort of the current test case (REQUIRE / FAIL)
struct AbortTest {};

struct RunState {
  int failures = 0;        // failed assertions in the current test case
  long long asserts = 0;   // assertions evaluated overall
  std::vector<std::string> info;  // INFO context stack
  // SUBCASE bookkeeping (doctest semantics: the test case is re-run until every
  // leaf subcase ran once; each run enters at most one new subcase per level)
  std::vector<std::string> stack;
  std::set<std::vector<std::string>> done;
  std::vector<bool> enteredAtDepth;
  std::vector<bool> pendingAtDepth;  // a not-yet-done subcase was skipped
};
inline RunState& state() {
  static RunState s;
  return s;
}

inline void report(const char* file, int line, const std::string& msg) {
  RunState& st = state();
  ++st.failures;
  std::fprintf(stderr, "%s:%d: ERROR: %s\n", file, line, msg.c_str());
  if (!st.stack.empty()) {
    std::string path;
    for (auto& s : st.stack) path += (path.empty() ? "" : " / ") + s;
    std::fprintf(stderr, "  in subcase: %s\n", path.c_str());
  }
  for (auto& i : st.info) std::fprintf(stderr, "  info: %s\n", i.c_str());
}

template <typename... A>
std::string cat(const A&... a) {
  std::ostringstream os;
  (void)std::initializer_list<int>{((os << a), 0)...};
  return os.str();
}

struct InfoScope {
  template <typename... A>
  explicit InfoScope(const A&... a) {
    state().info.push_back(cat(a...));
  }
  ~InfoScope() { state().info.pop_back(); }
};

class Subcase {
 public:
  Subcase(const char* name, const char* file, int line) {
    RunState& st = state();
    const size_t d = st.stack.size();
    if (st.enteredAtDepth.size() <= d + 1) {
      st.enteredAtDepth.resize(d + 2, false);
      st.pendingAtDepth.resize(d + 2, false);
    }
    path_ = st.stack;
    path_.push_back(std::string(name) + "@" + file + ":" + std::to_string(line));
    if (st.done.count(path_)) return;
    if (st.enteredAtDepth[d]) {
      st.pendingAtDepth[d] = true;
      return;
    }
    st.enteredAtDepth[d] = true;
    st.stack.push_back(name);
    entered_ = true;
    depth_ = d;
    st.enteredAtDepth[d + 1] = false;
    st.pendingAtDepth[d + 1] = false;
  }
  ~Subcase() {
    if (!entered_) return;
    RunState& st = state();
    // done unless a child subcase was skipped in this run
    if (!st.pendingAtDepth[depth_ + 1]) st.done.insert(path_);
    else st.pendingAtDepth[depth_] = true;
    st.stack.pop_back();
  }
  explicit operator bool() const { return entered_; }

 private:
  std::vector<std::string> path_;
  bool entered_ = false;
  size_t depth_ = 0;
};

inline bool wildcard(const char* p, const char* s) {
  if (!*p) return !*s;
  if (*p == '*') return wildcard(p + 1, s) || (*s && wildcard(p, s + 1));
  return *s && *p == *s && wildcard(p + 1, s + 1);
}
inline bool anyMatch(const std::vector<std::string>& pats, const std::string& s) {
  for (auto& p : pats)
    if (wildcard(p.c_str(), s.c_str())) return true;
  return false;
}
inline std::vector<std::string> splitList(const std::string& v) {
  std::vector<std::string> out;
  std::string cur;
  for (char c : v) {
    if (c == ',') {
      out.push_back(cur);
      cur.clear();
    } else {
      cur += c;
    }
  }
  if (!cur.empty()) out.push_back(cur);
  return out;
}

inline int runAll(int argc, char** argv) {
  std::vector<std::string> tc, tce, ts, tse;
  bool verbose = false;
  for (int i = 1; i < argc; ++i) {
    std::string a = argv[i];
    auto val = [&](const char* k) -> const char* {
      size_t n = std::strlen(k);
      return a.compare(0, n, k) == 0 ? a.c_str() + n : nullptr;
    };
    if (const char* v = val("-tc=")) tc = splitList(v);
    else if (const char* v2 = val("-tce=")) tce = splitList(v2);
    else if (const char* v3 = val("-ts=")) ts = splitList(v3);
    else if (const char* v4 = val("-tse=")) tse = splitList(v4);
    else if (a == "-s") verbose = true;
  }
  int passed = 0, failed = 0, skipped = 0;
  for (const TestCase& t : registry()) {
    if ((!tc.empty() && !anyMatch(tc, t.name)) || anyMatch(tce, t.name) ||
        (!ts.empty() && !anyMatch(ts, t.suite)) || anyMatch(tse, t.suite)) {
      ++skipped;
      continue;
    }
    RunState& st = state();
    st.failures = 0;
    st.done.clear();
    bool more = true;
    while (more) {
      st.stack.clear();
      st.info.clear();
      st.enteredAtDepth.assign(1, false);
      st.pendingAtDepth.assign(1, false);
      st.enteredAtDepth.resize(2, false);
      st.pendingAtDepth.resize(2, false);
      try {
        t.fn();
      } catch (const AbortTest&) {
      } catch (const std::exception& e) {
        report(t.file.c_str(), t.line, std::string("unexpected exception: ") + e.what());
      } catch (...) {
        report(t.file.c_str(), t.line, "unexpected non-standard exception");
      }
      more = st.pendingAtDepth[0];
    }
    if (st.failures) {
      ++failed;
      std::printf("[doctest] FAIL  %s / %s (%d failed assertions)\n", t.suite.c_str(),
                  t.name.c_str(), st.failures);
    } else {
      ++passed;
      if (verbose) std::printf("[doctest] PASS  %s / %s\n", t.suite.c_str(), t.name.c_str());
    }
  }
  std::printf("[doctest] test cases: %d passed, %d failed, %d skipped; assertions: %lld\n",
              passed, failed, skipped, state().asserts);
  return failed ? 1 : 0;
}

}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define DOCTEST_ANON(p) DOCTEST_CAT(p, __LINE__)

#define DOCTEST_TEST_CASE_IMPL(fn, name)                                                    \
  static void fn();                                                                        \
  static ::doctest::detail::Registrar DOCTEST_CAT(fn, _reg)(fn, name, __FILE__, __LINE__); \
  static void fn()
#define TEST_CASE(name) DOCTEST_TEST_CASE_IMPL(DOCTEST_ANON(doctest_tc_), name)

#define TEST_SUITE_BEGIN(name) \
  static ::doctest::detail::SuiteSetter DOCTEST_ANON(doctest_suite_)(name)
#define TEST_SUITE_END() static ::doctest::detail::SuiteSetter DOCTEST_ANON(doctest_suite_end_)("")

#define SUBCASE(name) \
  if (const ::doctest::detail::Subcase & DOCTEST_ANON(doctest_sc_) = \
          ::doctest::detail::Subcase(name, __FILE__, __LINE__))

#define INFO(...) ::doctest::detail::InfoScope DOCTEST_ANON(doctest_info_)(__VA_ARGS__)

#define DOCTEST_ASSERT_IMPL(expr, abort, ...)                                            \
  do {                                                                                   \
    ++::doctest::detail::state().asserts;                                                \
    bool doctest_ok_ = false;                                                            \
    try {                                                                                \
      doctest_ok_ = static_cast<bool>(expr);                                             \
    } catch (const std::exception& doctest_e_) {                                         \
      ::doctest::detail::report(__FILE__, __LINE__,                                      \
                                std::string(#expr " threw: ") + doctest_e_.what());     \
      if (abort) throw ::doctest::detail::AbortTest{};                                   \
      break;                                                                             \
    }                                                                                    \
    if (!doctest_ok_) {                                                                  \
      ::doctest::detail::report(__FILE__, __LINE__,                                      \
                                std::string(abort ? "REQUIRE( " : "CHECK( ") + #expr " )" \
                                    __VA_ARGS__);                                        \
      if (abort) throw ::doctest::detail::AbortTest{};                                   \
    }                                                                                    \
  } while (0)

#define CHECK(...) DOCTEST_ASSERT_IMPL((__VA_ARGS__), false, )
#define REQUIRE(...) DOCTEST_ASSERT_IMPL((__VA_ARGS__), true, )
#define REQUIRE_MESSAGE(expr, ...) \
  DOCTEST_ASSERT_IMPL(expr, true, +std::string(" -- ") + ::doctest::detail::cat(__VA_ARGS__))
#define CHECK_MESSAGE(expr, ...) \
  DOCTEST_ASSERT_IMPL(expr, false, +std::string(" -- ") + ::doctest::detail::cat(__VA_ARGS__))

#define FAIL(...)                                                                      \
  do {                                                                                 \
    ::doctest::detail::report(__FILE__, __LINE__,                                      \
                              std::string("FAIL: ") + ::doctest::detail::cat(__VA_ARGS__)); \
    throw ::doctest::detail::AbortTest{};                                              \
  } while (0)

#define CHECK_THROWS_AS(expr, ...)                                                    \
  do {                                                                                \
    ++::doctest::detail::state().asserts;                                             \
    try {                                                                             \
      (void)(expr);                                                                   \
      ::doctest::detail::report(__FILE__, __LINE__, "CHECK_THROWS_AS( " #expr " ) did not throw"); \
    } catch (const __VA_ARGS__&) {                                                    \
    } catch (const std::exception& doctest_e_) {                                      \
      ::doctest::detail::report(__FILE__, __LINE__,                                   \
                                std::string("CHECK_THROWS_AS( " #expr " ) threw another type: ") + \
                                    doctest_e_.what());                               \
    }                                                                                 \
  } while (0)

#define CHECK_THROWS_WITH_AS(expr, matcher, ...)                                       \
  do {                                                                                 \
    ++::doctest::detail::state().asserts;                                              \
    try {                                                                              \
      (void)(expr);                                                                    \
      ::doctest::detail::report(__FILE__, __LINE__,                                    \
                                "CHECK_THROWS_WITH_AS( " #expr " ) did not throw");    \
    } catch (const __VA_ARGS__& doctest_e_) {                                          \
      if (!::doctest::detail::messageMatches(matcher, doctest_e_.what()))              \
        ::doctest::detail::report(__FILE__, __LINE__,                                  \
                                  std::string("CHECK_THROWS_WITH_AS( " #expr " ): message '") + \
                                      doctest_e_.what() + "' does not match");         \
    } catch (const std::exception& doctest_e_) {                                       \
      ::doctest::detail::report(__FILE__, __LINE__,                                    \
                                std::string("CHECK_THROWS_WITH_AS( " #expr " ) threw another type: ") + \
                                    doctest_e_.what());                                \
    }                                                                                  \
  } while (0)

namespace doctest {
namespace detail {
inline bool messageMatches(const Contains& c, const char* what) { return c.matches(what); }
inline bool messageMatches(const char* s, const char* what) { return std::string(s) == what; }
inline bool messageMatches(const std::string& s, const char* what) { return s == what; }
}  // namespace detail
}  // namespace doctest

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main(int argc, char** argv) { return ::doctest::detail::runAll(argc, argv); }
#endif
