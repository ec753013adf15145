// Minimal doctest-compatible shim — TEST INFRASTRUCTURE.
//
// The reference's unit suites include <doctest.h> from proj/vendor/, which is
// gitignored and absent (SURVEY.md §8c "Blocked pieces"). This header gives
// the subset proj/tests/test_capi.cpp uses — TEST_CASE, CHECK, REQUIRE and
// DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN — so the reference's own C-ABI test can
// be compiled unmodified against libpascal.so (oracle/Makefile `callers`).
// Output: one line per failed check, a summary line, exit status 1 on any
// failure (doctest's contract for CI).
#pragma once

#include <cstdio>
#include <exception>
#include <functional>
#include <string>
#include <vector>

namespace doctest_shim {

struct Case {
    const char* name;
    void (*fn)();
};
inline std::vector<Case>& registry() {
    static std::vector<Case> r;
    return r;
}
struct Reg {
    Reg(const char* name, void (*fn)()) { registry().push_back({name, fn}); }
};
struct RequireFailed {};
inline int& failures() {
    static int f = 0;
    return f;
}
inline long& checks() {
    static long c = 0;
    return c;
}
inline const char*& current() {
    static const char* c = "";
    return c;
}
inline bool check(bool ok, const char* expr, const char* file, int line, bool require) {
    ++checks();
    if (!ok) {
        ++failures();
        std::fprintf(stderr, "%s:%d: FAILED %s( %s ) in TEST_CASE \"%s\"\n", file, line,
                     require ? "REQUIRE" : "CHECK", expr, current());
        if (require) throw RequireFailed{};
    }
    return ok;
}
inline int run_all() {
    int failed_cases = 0;
    for (const Case& c : registry()) {
        current() = c.name;
        const int before = failures();
        try {
            c.fn();
        } catch (const RequireFailed&) {
        } catch (const std::exception& e) {
            ++failures();
            std::fprintf(stderr, "TEST_CASE \"%s\" threw: %s\n", c.name, e.what());
        }
        if (failures() != before) ++failed_cases;
    }
    std::printf("[doctest-shim] test cases: %zu | %zu passed | %d failed | checks: %ld\n",
                registry().size(), registry().size() - failed_cases, failed_cases, checks());
    return failures() ? 1 : 0;
}

}  // namespace doctest_shim

#define DOCTEST_SHIM_CAT2(a, b) a##b
#define DOCTEST_SHIM_CAT(a, b) DOCTEST_SHIM_CAT2(a, b)
#define DOCTEST_SHIM_CASE(fn, name)                                                   \
    static void fn();                                                                 \
    static doctest_shim::Reg DOCTEST_SHIM_CAT(fn, _reg)(name, &fn);                   \
    static void fn()
#define TEST_CASE(name) DOCTEST_SHIM_CASE(DOCTEST_SHIM_CAT(doctest_shim_case_, __LINE__), name)
#define CHECK(...) doctest_shim::check(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, false)
#define REQUIRE(...) doctest_shim::check(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, true)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() { return doctest_shim::run_all(); }
#endif
