// SPDX-License-Identifier: Apache-2.0
//
// A minimal stand-in for Catch2 v3's catch_amalgamated.hpp (Catch2 is not installed in this
// image), enough to compile the reference's own test sources UNMODIFIED
// (/root/reference/proj/tests/test_attention.cpp, test_paged_kv.cpp) against the chunktrain/
// forwarding headers (include/chunktrain). TEST INFRASTRUCTURE.
//
// Supported: TEST_CASE, REQUIRE, REQUIRE_FALSE, REQUIRE_NOTHROW, REQUIRE_THROWS, REQUIRE_THROWS_AS,
// CHECK (non-fatal), and Catch::Approx with Catch2's comparison rule: |a - b| <= margin, or
// |a - b| <= epsilon * (scale + |target|) with epsilon defaulting to 100 x FLT_EPSILON.
// The runner (define CATCH_SHIM_MAIN in one translation unit) runs every registered case, or those
// whose name contains argv[1], and prints the Catch-style summary line.
#pragma once

#include <cmath>
#include <cstdio>
#include <cstring>
#include <exception>
#include <limits>
#include <string>
#include <vector>

namespace Catch {

class Approx {
public:
    explicit Approx(double target) : target_(target) {}
    Approx& margin(double m) {
        margin_ = m;
        return *this;
    }
    Approx& epsilon(double e) {
        epsilon_ = e;
        return *this;
    }
    Approx& scale(double s) {
        scale_ = s;
        return *this;
    }
    bool matches(double other) const {
        auto within = [&](double tol) { return target_ + tol >= other && other + tol >= target_; };
        return within(margin_) || within(epsilon_ * (scale_ + std::fabs(std::isinf(target_) ? 0.0 : target_)));
    }
    friend bool operator==(double lhs, const Approx& a) { return a.matches(lhs); }
    friend bool operator==(const Approx& a, double rhs) { return a.matches(rhs); }
    friend bool operator!=(double lhs, const Approx& a) { return !a.matches(lhs); }
    friend bool operator!=(const Approx& a, double rhs) { return !a.matches(rhs); }

private:
    double target_;
    double margin_ = 0.0;
    double epsilon_ = std::numeric_limits<float>::epsilon() * 100.0;
    double scale_ = 0.0;
};

struct Case {
    const char* name;
    void (*fn)();
};
inline std::vector<Case>& registry() {
    static std::vector<Case> r;
    return r;
}
struct Registrar {
    Registrar(const char* name, void (*fn)()) { registry().push_back({name, fn}); }
};
struct Stats {
    long assertions = 0, failed_assertions = 0;
};
inline Stats& stats() {
    static Stats s;
    return s;
}
struct Abort {};  // a failed REQUIRE ends its test case

inline void report(bool ok, const char* kind, const char* expr, const char* file, int line, bool fatal) {
    ++stats().assertions;
    if (ok) return;
    ++stats().failed_assertions;
    std::printf("%s:%d: FAILED: %s( %s )\n", file, line, kind, expr);
    if (fatal) throw Abort{};
}

}  // namespace Catch

#define CATCH_SHIM_CAT2(a, b) a##b
#define CATCH_SHIM_CAT(a, b) CATCH_SHIM_CAT2(a, b)
#define CATCH_SHIM_FN CATCH_SHIM_CAT(catch_shim_case_, __LINE__)
#define CATCH_SHIM_REG CATCH_SHIM_CAT(catch_shim_reg_, __LINE__)
#define TEST_CASE(name, ...)                                                   \
    static void CATCH_SHIM_FN();                                               \
    static const ::Catch::Registrar CATCH_SHIM_REG(name, &CATCH_SHIM_FN);      \
    static void CATCH_SHIM_FN()

#define REQUIRE(...) ::Catch::report(static_cast<bool>(__VA_ARGS__), "REQUIRE", #__VA_ARGS__, __FILE__, __LINE__, true)
#define CHECK(...) ::Catch::report(static_cast<bool>(__VA_ARGS__), "CHECK", #__VA_ARGS__, __FILE__, __LINE__, false)
#define REQUIRE_FALSE(...) \
    ::Catch::report(!static_cast<bool>(__VA_ARGS__), "REQUIRE_FALSE", #__VA_ARGS__, __FILE__, __LINE__, true)
#define REQUIRE_NOTHROW(...)                                                                              \
    do {                                                                                                  \
        bool catch_shim_ok = true;                                                                        \
        try {                                                                                             \
            static_cast<void>(__VA_ARGS__);                                                               \
        } catch (...) {                                                                                   \
            catch_shim_ok = false;                                                                        \
        }                                                                                                 \
        ::Catch::report(catch_shim_ok, "REQUIRE_NOTHROW", #__VA_ARGS__, __FILE__, __LINE__, true);        \
    } while (0)
#define REQUIRE_THROWS(...)                                                                               \
    do {                                                                                                  \
        bool catch_shim_ok = false;                                                                       \
        try {                                                                                             \
            static_cast<void>(__VA_ARGS__);                                                               \
        } catch (...) {                                                                                   \
            catch_shim_ok = true;                                                                         \
        }                                                                                                 \
        ::Catch::report(catch_shim_ok, "REQUIRE_THROWS", #__VA_ARGS__, __FILE__, __LINE__, true);         \
    } while (0)
#define REQUIRE_THROWS_AS(expr, type)                                                                     \
    do {                                                                                                  \
        bool catch_shim_ok = false;                                                                       \
        try {                                                                                             \
            static_cast<void>(expr);                                                                      \
        } catch (const type&) {                                                                           \
            catch_shim_ok = true;                                                                         \
        } catch (...) {                                                                                   \
        }                                                                                                 \
        ::Catch::report(catch_shim_ok, "REQUIRE_THROWS_AS", #expr ", " #type, __FILE__, __LINE__, true);  \
    } while (0)

#ifdef CATCH_SHIM_MAIN
int main(int argc, char** argv) {
    const char* filter = argc > 1 ? argv[1] : nullptr;
    int cases = 0, failed_cases = 0;
    for (const auto& c : ::Catch::registry()) {
        if (filter && !std::strstr(c.name, filter)) continue;
        ++cases;
        const long before = ::Catch::stats().failed_assertions;
        bool ok = true;
        try {
            c.fn();
        } catch (const ::Catch::Abort&) {
            ok = false;
        } catch (const std::exception& e) {
            std::printf("test case \"%s\" threw: %s\n", c.name, e.what());
            ++::Catch::stats().failed_assertions;
            ok = false;
        }
        ok = ok && ::Catch::stats().failed_assertions == before;
        std::printf("%s  %s\n", ok ? "PASS" : "FAIL", c.name);
        failed_cases += ok ? 0 : 1;
    }
    const auto& s = ::Catch::stats();
    if (failed_cases == 0)
        std::printf("All tests passed (%ld assertions in %d test cases)\n", s.assertions, cases);
    else
        std::printf("test cases: %d | %d passed | %d failed\nassertions: %ld | %ld failed\n", cases,
                    cases - failed_cases, failed_cases, s.assertions, s.failed_assertions);
    return failed_cases == 0 ? 0 : 1;
}
#endif
