// doctest.h — the subset of the doctest single-header API that the
// reference's C-ABI test (proj/tests/test_capi.cpp) uses: TEST_CASE, CHECK,
// REQUIRE and DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN.  Lets that file compile
// UNCHANGED against libgridadmm.so (oracle/Makefile target _ref/test_capi).
// Test infrastructure only.  `test_capi --tc=<substring>` runs the matching
// test cases; the exit status is non-zero when any CHECK/REQUIRE failed.
#pragma once

#include <cstdio>
#include <cstring>
#include <vector>

namespace mini_doctest {

struct TestCase {
    const char* name;
    void (*fn)();
};

inline std::vector<TestCase>& registry() {
    static std::vector<TestCase> r;
    return r;
}

struct Counters {
    int checks = 0, failed = 0;
};

inline Counters& counters() {
    static Counters c;
    return c;
}

struct Register {
    Register(const char* name, void (*fn)()) { registry().push_back({name, fn}); }
};

struct RequireFailed {};

inline void assert_that(bool ok, const char* expr, const char* file, int line, bool fatal) {
    ++counters().checks;
    if (ok) return;
    ++counters().failed;
    std::fprintf(stderr, "%s:%d: %s( %s ) FAILED\n", file, line, fatal ? "REQUIRE" : "CHECK", expr);
    if (fatal) throw RequireFailed{};
}

}  // namespace mini_doctest

#define MINI_DOCTEST_CAT2(a, b) a##b
#define MINI_DOCTEST_CAT(a, b) MINI_DOCTEST_CAT2(a, b)
#define MINI_DOCTEST_CASE(fn, reg, name)                                   \
    static void fn();                                                      \
    static const mini_doctest::Register reg(name, &fn);                    \
    static void fn()
#define TEST_CASE(name)                                                    \
    MINI_DOCTEST_CASE(MINI_DOCTEST_CAT(mini_doctest_case_, __LINE__),      \
                      MINI_DOCTEST_CAT(mini_doctest_reg_, __LINE__), name)
#define CHECK(...) \
    mini_doctest::assert_that(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, false)
#define REQUIRE(...) \
    mini_doctest::assert_that(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, true)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main(int argc, char** argv) {
    const char* filter = nullptr;
    for (int i = 1; i < argc; ++i)
        if (std::strncmp(argv[i], "--tc=", 5) == 0) filter = argv[i] + 5;
    int run = 0, cases_failed = 0;
    for (const auto& tc : mini_doctest::registry()) {
        if (filter && !std::strstr(tc.name, filter)) continue;
        ++run;
        const int before = mini_doctest::counters().failed;
        try {
            tc.fn();
        } catch (const mini_doctest::RequireFailed&) {
        } catch (...) {
            ++mini_doctest::counters().failed;
            std::fprintf(stderr, "test case '%s' threw\n", tc.name);
        }
        const bool ok = mini_doctest::counters().failed == before;
        cases_failed += ok ? 0 : 1;
        std::printf("[%s] %s\n", ok ? "pass" : "FAIL", tc.name);
    }
    std::printf("test cases: %d run, %d failed; assertions: %d, %d failed\n", run, cases_failed,
                mini_doctest::counters().checks, mini_doctest::counters().failed);
    return (cases_failed == 0 && run > 0) ? 0 : 1;
}
#endif
