// tests/ref_unit/doctest.h — a minimal doctest-compatible harness (our own
// code, not doctest) that lets the reference project's C++ unit tests
// (/root/reference/proj/tests/test_*.cpp, written against doctest) compile
// unmodified against this repo's host library (namespace bml,
// paper_1804_07981_b200/csrc/host/include). Test infrastructure only: it is
// used by tests/test_reference_unit_tests.py and nothing else.
//
// Covers the macro subset those files use: TEST_CASE, SUBCASE (flat, re-run
// per subcase like doctest), CHECK/CHECK_FALSE/REQUIRE, CHECK_THROWS[_AS],
// CHECK_NOTHROW, CAPTURE, FAIL. main() (DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN)
// accepts --test-case=<globs> and --test-case-exclude=<globs>, comma separated.
#pragma once

#include <fnmatch.h>

#include <cstdio>
#include <functional>
#include <iostream>
#include <set>
#include <sstream>
#include <string>
#include <utility>
#include <vector>

namespace refshim {

struct TestCase {
    const char* name;
    const char* file;
    int line;
    void (*fn)();
};

inline std::vector<TestCase>& registry() {
    static std::vector<TestCase> r;
    return r;
}

struct Registrar {
    Registrar(const char* name, const char* file, int line, void (*fn)()) {
        registry().push_back({name, file, line, fn});
    }
};

struct State {
    long asserts = 0, failed_asserts = 0;
    bool case_failed = false;
    std::vector<std::function<void(std::ostream&)>> context;
    // SUBCASE bookkeeping for the current test case
    std::set<std::pair<std::string, int>> done;
    bool entered_this_run = false;
    bool pending = false;  // a subcase was skipped this run and is not done yet
};

inline State& state() {
    static State s;
    return s;
}

struct Abort {};  // REQUIRE / FAIL: leave the test case

inline void report(const char* file, int line, const std::string& what) {
    State& s = state();
    ++s.failed_asserts;
    s.case_failed = true;
    std::cerr << file << ":" << line << ": FAILED: " << what << "\n";
    for (const auto& c : s.context) {
        std::cerr << "  with ";
        c(std::cerr);
        std::cerr << "\n";
    }
}

inline bool check(bool ok, const char* kind, const char* expr, const char* file, int line) {
    ++state().asserts;
    if (!ok) report(file, line, std::string(kind) + "( " + expr + " )");
    return ok;
}

struct Capture {
    template <class F>
    explicit Capture(F f) {
        state().context.emplace_back(std::move(f));
    }
    ~Capture() { state().context.pop_back(); }
};

struct Subcase {
    bool entered = false;
    Subcase(const char* name, const char* file, int line) {
        State& s = state();
        const auto key = std::make_pair(std::string(file) + ":" + name, line);
        if (s.done.count(key)) return;
        if (s.entered_this_run) {
            s.pending = true;
            return;
        }
        s.entered_this_run = true;
        s.done.insert(key);
        entered = true;
    }
    explicit operator bool() const { return entered; }
};

inline bool matches(const std::string& name, const std::string& globs) {
    std::stringstream ss(globs);
    std::string g;
    while (std::getline(ss, g, ','))
        if (!g.empty() && fnmatch(g.c_str(), name.c_str(), 0) == 0) return true;
    return false;
}

inline int run_all(int argc, char** argv) {
    std::string include, exclude;
    for (int i = 1; i < argc; ++i) {
        const std::string a = argv[i];
        if (a.rfind("--test-case=", 0) == 0) include = a.substr(12);
        if (a.rfind("--test-case-exclude=", 0) == 0) exclude = a.substr(20);
    }
    int passed = 0, failed = 0, skipped = 0;
    for (const TestCase& tc : registry()) {
        if ((!include.empty() && !matches(tc.name, include)) || (!exclude.empty() && matches(tc.name, exclude))) {
            ++skipped;
            continue;
        }
        State& s = state();
        s.case_failed = false;
        s.done.clear();
        do {
            s.entered_this_run = false;
            s.pending = false;
            try {
                tc.fn();
            } catch (const Abort&) {
            } catch (const std::exception& e) {
                report(tc.file, tc.line, std::string("unexpected exception: ") + e.what());
            } catch (...) {
                report(tc.file, tc.line, "unexpected unknown exception");
            }
        } while (s.pending);
        if (s.case_failed) {
            ++failed;
            std::cerr << "TEST CASE FAILED: " << tc.name << "\n";
        } else {
            ++passed;
            std::cout << "[ok] " << tc.name << "\n";
        }
    }
    std::cout << "[refshim] test cases: " << passed << " passed, " << failed << " failed, " << skipped
              << " skipped; assertions: " << state().asserts << " (" << state().failed_asserts << " failed)\n";
    return failed == 0 ? 0 : 1;
}

}  // namespace refshim

#define REFSHIM_CAT2(a, b) a##b
#define REFSHIM_CAT(a, b) REFSHIM_CAT2(a, b)
#define REFSHIM_ANON(p) REFSHIM_CAT(p, __COUNTER__)

#define REFSHIM_TEST_CASE_IMPL(fn, reg, name)                                         \
    static void fn();                                                                 \
    static const ::refshim::Registrar reg(name, __FILE__, __LINE__, &fn);             \
    static void fn()
#define REFSHIM_TEST_CASE2(id, name) \
    REFSHIM_TEST_CASE_IMPL(REFSHIM_CAT(refshim_tc_, id), REFSHIM_CAT(refshim_reg_, id), name)
#define TEST_CASE(name) REFSHIM_TEST_CASE2(__COUNTER__, name)

#define SUBCASE(name) if (const ::refshim::Subcase REFSHIM_ANON(refshim_sc_){name, __FILE__, __LINE__})

#define CHECK(...) ::refshim::check(static_cast<bool>(__VA_ARGS__), "CHECK", #__VA_ARGS__, __FILE__, __LINE__)
#define CHECK_FALSE(...) \
    ::refshim::check(!static_cast<bool>(__VA_ARGS__), "CHECK_FALSE", #__VA_ARGS__, __FILE__, __LINE__)
#define REQUIRE(...)                                                                                 \
    do {                                                                                             \
        if (!::refshim::check(static_cast<bool>(__VA_ARGS__), "REQUIRE", #__VA_ARGS__, __FILE__, __LINE__)) \
            throw ::refshim::Abort{};                                                                \
    } while (0)

#define CHECK_THROWS_AS(expr, ...)                                                               \
    do {                                                                                         \
        bool refshim_ok = false;                                                                 \
        try {                                                                                    \
            static_cast<void>(expr);                                                             \
        } catch (const __VA_ARGS__&) {                                                           \
            refshim_ok = true;                                                                   \
        } catch (...) {                                                                          \
        }                                                                                        \
        ::refshim::check(refshim_ok, "CHECK_THROWS_AS", #expr ", " #__VA_ARGS__, __FILE__, __LINE__); \
    } while (0)
#define CHECK_THROWS(...)                                                                  \
    do {                                                                                   \
        bool refshim_ok = false;                                                           \
        try {                                                                              \
            static_cast<void>(__VA_ARGS__);                                                \
        } catch (...) {                                                                    \
            refshim_ok = true;                                                             \
        }                                                                                  \
        ::refshim::check(refshim_ok, "CHECK_THROWS", #__VA_ARGS__, __FILE__, __LINE__);    \
    } while (0)
#define CHECK_NOTHROW(...)                                                                 \
    do {                                                                                   \
        bool refshim_ok = true;                                                            \
        try {                                                                              \
            static_cast<void>(__VA_ARGS__);                                                \
        } catch (...) {                                                                    \
            refshim_ok = false;                                                            \
        }                                                                                  \
        ::refshim::check(refshim_ok, "CHECK_NOTHROW", #__VA_ARGS__, __FILE__, __LINE__);   \
    } while (0)

#define CAPTURE(x) \
    const ::refshim::Capture REFSHIM_ANON(refshim_cap_)([&](std::ostream& os) { os << #x " := " << (x); })

#define FAIL(msg)                                                         \
    do {                                                                  \
        std::ostringstream refshim_os;                                    \
        refshim_os << "FAIL: " << msg;                                    \
        ++::refshim::state().asserts;                                     \
        ::refshim::report(__FILE__, __LINE__, refshim_os.str());          \
        throw ::refshim::Abort{};                                         \
    } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main(int argc, char** argv) { return ::refshim::run_all(argc, argv); }
#endif
