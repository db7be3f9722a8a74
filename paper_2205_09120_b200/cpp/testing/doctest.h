// doctest.h — a minimal, self-written stand-in for the doctest subset the
// reference unit tests use (TEST_CASE, CHECK, CHECK_FALSE, REQUIRE,
// CHECK_THROWS_AS, doctest::Approx, DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN).
// The real doctest is not vendored in the reference (proj/.gitignore) and
// there is no network; this lets the reference's own tests/*.cpp compile,
// unchanged, against the drop-in library.
#pragma once

#include <cmath>
#include <cstdio>
#include <functional>
#include <limits>
#include <string>
#include <vector>

namespace doctest {

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
    long checks = 0, failures = 0;
    const char* current = "";
};
inline State& state() {
    static State s;
    return s;
}

struct RequireFailed {};

inline void report(bool ok, const char* expr, const char* file, int line, bool fatal) {
    ++state().checks;
    if (ok) return;
    ++state().failures;
    std::printf("%s:%d: FAILED in \"%s\": %s\n", file, line, state().current, expr);
    if (fatal) throw RequireFailed{};
}

class Approx {
public:
    explicit Approx(double v) : value_(v) {}
    Approx& epsilon(double e) {
        eps_ = e;
        return *this;
    }
    friend bool operator==(double lhs, const Approx& rhs) {
        const double scale = std::fmax(std::fabs(lhs), std::fabs(rhs.value_));
        return std::fabs(lhs - rhs.value_) < rhs.eps_ * (1.0 + scale);
    }
    friend bool operator==(const Approx& lhs, double rhs) { return rhs == lhs; }
    friend bool operator!=(double lhs, const Approx& rhs) { return !(lhs == rhs); }

private:
    double value_;
    double eps_ = static_cast<double>(std::numeric_limits<float>::epsilon()) * 100;
};

inline int run_all() {
    long cases_failed = 0;
    for (const auto& tc : registry()) {
        state().current = tc.name;
        const long before = state().failures;
        try {
            tc.fn();
        } catch (const RequireFailed&) {
        } catch (const std::exception& e) {
            ++state().failures;
            std::printf("%s:%d: EXCEPTION in \"%s\": %s\n", tc.file, tc.line, tc.name, e.what());
        }
        if (state().failures != before) ++cases_failed;
    }
    std::printf("[doctest-shim] test cases: %zu | passed: %zu | failed: %ld\n", registry().size(),
                registry().size() - static_cast<size_t>(cases_failed), cases_failed);
    std::printf("[doctest-shim] assertions: %ld | failed: %ld\n", state().checks, state().failures);
    return cases_failed ? 1 : 0;
}

}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define DOCTEST_TC_(fn, name)                                                                   \
    static void fn();                                                                           \
    static doctest::Registrar DOCTEST_CAT(fn, _reg)(name, __FILE__, __LINE__, &fn);             \
    static void fn()
#define TEST_CASE(name) DOCTEST_TC_(DOCTEST_CAT(doctest_tc_, __LINE__), name)

#define CHECK(...) doctest::report(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, false)
#define CHECK_FALSE(...) doctest::report(!static_cast<bool>(__VA_ARGS__), "!(" #__VA_ARGS__ ")", __FILE__, __LINE__, false)
#define REQUIRE(...) doctest::report(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, true)
#define CHECK_THROWS_AS(expr, ...)                                                               \
    do {                                                                                        \
        bool doctest_ok_ = false;                                                               \
        try {                                                                                   \
            (void)(expr);                                                                       \
        } catch (const __VA_ARGS__&) {                                                          \
            doctest_ok_ = true;                                                                 \
        } catch (...) {                                                                         \
        }                                                                                       \
        doctest::report(doctest_ok_, "THROWS_AS(" #expr ", " #__VA_ARGS__ ")", __FILE__, __LINE__, false); \
    } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() { return doctest::run_all(); }
#endif
