// Minimal doctest-compatible harness — TEST INFRASTRUCTURE ONLY.
// The reference's unit tests (/root/reference/proj/tests/*.cpp) include <doctest.h>, which the
// reference does not ship (vendor/ is git-ignored, proj/.gitignore:2). This header implements just
// the subset those files use (TEST_CASE, CHECK, CHECK_FALSE, REQUIRE, CHECK_THROWS_AS,
// doctest::Approx with epsilon/scale) so they compile unmodified and pin the oracle.
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <functional>
#include <limits>
#include <string>
#include <vector>

namespace doctest {

class Approx {
public:
    explicit Approx(double v) : value_(v) {}
    Approx& epsilon(double e) { eps_ = e; return *this; }
    Approx& scale(double s) { scale_ = s; return *this; }
    bool matches(double lhs) const {
        return std::fabs(lhs - value_) < eps_ * (scale_ + std::max(std::fabs(lhs), std::fabs(value_)));
    }
    double value() const { return value_; }

private:
    double value_;
    double eps_ = static_cast<double>(std::numeric_limits<float>::epsilon()) * 100;
    double scale_ = 1.0;
};

inline bool operator==(double lhs, const Approx& rhs) { return rhs.matches(lhs); }
inline bool operator==(const Approx& lhs, double rhs) { return lhs.matches(rhs); }
inline bool operator!=(double lhs, const Approx& rhs) { return !rhs.matches(lhs); }

namespace detail {

struct Case {
    const char* name;
    const char* file;
    void (*fn)();
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
    Registrar(const char* name, const char* file, void (*fn)()) { registry().push_back({name, file, fn}); }
};
struct RequireFailed {};

inline void report(bool ok, const char* expr, const char* file, int line, bool fatal) {
    if (ok) return;
    ++failures();
    std::printf("%s:%d: CHECK FAILED: %s\n", file, line, expr);
    if (fatal) throw RequireFailed{};
}

// -tce=<names> skips test cases (comma-separated exact names), as doctest's --test-case-exclude.
inline bool excluded(const char* name, int argc, char** argv) {
    for (int i = 1; i < argc; ++i) {
        std::string a = argv[i];
        if (a.rfind("-tce=", 0) != 0) continue;
        a = a.substr(5) + ",";
        for (size_t at = 0, comma; (comma = a.find(',', at)) != std::string::npos; at = comma + 1)
            if (a.compare(at, comma - at, name) == 0) return true;
    }
    return false;
}

inline int run_all(int argc = 0, char** argv = nullptr) {
    int cases_failed = 0, cases = 0;
    for (const Case& c : registry()) {
        if (excluded(c.name, argc, argv)) {
            std::printf("[SKIP] %s\n", c.name);
            continue;
        }
        ++cases;
        int before = failures();
        try {
            c.fn();
        } catch (const RequireFailed&) {
        } catch (const std::exception& e) {
            ++failures();
            std::printf("%s: exception in \"%s\": %s\n", c.file, c.name, e.what());
        }
        bool ok = failures() == before;
        if (!ok) ++cases_failed;
        std::printf("[%s] %s\n", ok ? "PASS" : "FAIL", c.name);
    }
    std::printf("[doctest] test cases: %d | %d passed | %d failed\n", cases, cases - cases_failed,
                cases_failed);
    return cases_failed == 0 ? 0 : 1;
}

}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define DOCTEST_TEST_CASE_IMPL(fn, name)                                                    \
    static void fn();                                                                       \
    static ::doctest::detail::Registrar DOCTEST_CAT(fn, _reg)(name, __FILE__, &fn);         \
    static void fn()
#define TEST_CASE(name) DOCTEST_TEST_CASE_IMPL(DOCTEST_CAT(doctest_case_, __COUNTER__), name)

#define CHECK(...) ::doctest::detail::report(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, false)
#define CHECK_FALSE(...) ::doctest::detail::report(!static_cast<bool>(__VA_ARGS__), "!(" #__VA_ARGS__ ")", __FILE__, __LINE__, false)
#define REQUIRE(...) ::doctest::detail::report(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, true)
#define CHECK_THROWS_AS(expr, type)                                                         \
    do {                                                                                    \
        bool caught_ = false;                                                               \
        try {                                                                               \
            (void)(expr);                                                                   \
        } catch (const type&) {                                                             \
            caught_ = true;                                                                 \
        } catch (...) {                                                                     \
        }                                                                                   \
        ::doctest::detail::report(caught_, "THROWS_AS(" #expr ", " #type ")", __FILE__, __LINE__, false); \
    } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main(int argc, char** argv) { return ::doctest::detail::run_all(argc, argv); }
#endif
