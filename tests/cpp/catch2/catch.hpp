// Minimal Catch2-v2-compatible test shim (only the macros the reference's
// unit tests use), so those tests compile unchanged against the B200
// headers — the drop-in proof of API compatibility.
#pragma once

#include <cmath>
#include <cstdio>
#include <exception>
#include <functional>
#include <limits>
#include <sstream>
#include <string>
#include <vector>

namespace Catch {

struct TestCase {
    const char* name;
    std::function<void()> fn;
};
inline std::vector<TestCase>& registry() {
    static std::vector<TestCase> r;
    return r;
}
struct Registrar {
    Registrar(const char* name, std::function<void()> fn) { registry().push_back({name, std::move(fn)}); }
};
struct Stats {
    long checks = 0, failures = 0;
};
inline Stats& stats() {
    static Stats s;
    return s;
}
struct AbortTest {};

inline void report_failure(const char* file, int line, const std::string& what) {
    ++stats().failures;
    std::fprintf(stderr, "%s:%d: FAILED: %s\n", file, line, what.c_str());
}

class Approx {
 public:
    explicit Approx(double v) : value_(v), eps_(std::numeric_limits<float>::epsilon() * 100), margin_(0.0) {}
    Approx& epsilon(double e) {
        eps_ = e;
        return *this;
    }
    Approx& margin(double m) {
        margin_ = m;
        return *this;
    }
    bool matches(double other) const {
        const double diff = std::fabs(other - value_);
        if (diff <= margin_) return true;
        return diff <= eps_ * std::fabs(std::isinf(value_) ? 0.0 : value_);
    }
    friend bool operator==(double a, const Approx& b) { return b.matches(a); }
    friend bool operator==(const Approx& b, double a) { return b.matches(a); }
    friend bool operator!=(double a, const Approx& b) { return !b.matches(a); }
    friend bool operator<=(double a, const Approx& b) { return a <= b.value_ || b.matches(a); }
    friend bool operator>=(double a, const Approx& b) { return a >= b.value_ || b.matches(a); }

 private:
    double value_, eps_, margin_;
};

struct Contains {
    explicit Contains(std::string s) : needle(std::move(s)) {}
    bool match(const std::string& hay) const { return hay.find(needle) != std::string::npos; }
    std::string needle;
};

}  // namespace Catch

using Catch::Approx;

#define CATCH_CAT2(a, b) a##b
#define CATCH_CAT(a, b) CATCH_CAT2(a, b)
#define TEST_CASE(name, ...)                                                            \
    static void CATCH_CAT(catch_test_fn_, __LINE__)();                                  \
    static Catch::Registrar CATCH_CAT(catch_reg_, __LINE__)(name, &CATCH_CAT(catch_test_fn_, __LINE__)); \
    static void CATCH_CAT(catch_test_fn_, __LINE__)()

#define CATCH_CHECK_IMPL(cond, fatal, text)                                             \
    do {                                                                                \
        ++Catch::stats().checks;                                                        \
        bool catch_ok_ = false;                                                         \
        try {                                                                           \
            catch_ok_ = static_cast<bool>(cond);                                        \
        } catch (const std::exception& e) {                                             \
            Catch::report_failure(__FILE__, __LINE__, std::string(text) + " threw " + e.what()); \
            if (fatal) throw Catch::AbortTest{};                                        \
            break;                                                                      \
        }                                                                               \
        if (!catch_ok_) {                                                               \
            Catch::report_failure(__FILE__, __LINE__, text);                            \
            if (fatal) throw Catch::AbortTest{};                                        \
        }                                                                               \
    } while (0)

#define CHECK(...) CATCH_CHECK_IMPL((__VA_ARGS__), false, #__VA_ARGS__)
#define REQUIRE(...) CATCH_CHECK_IMPL((__VA_ARGS__), true, #__VA_ARGS__)
#define CHECK_FALSE(...) CATCH_CHECK_IMPL(!(__VA_ARGS__), false, "!(" #__VA_ARGS__ ")")
#define REQUIRE_FALSE(...) CATCH_CHECK_IMPL(!(__VA_ARGS__), true, "!(" #__VA_ARGS__ ")")

#define CHECK_THROWS(...)                                                               \
    do {                                                                                \
        ++Catch::stats().checks;                                                        \
        bool catch_threw_ = false;                                                      \
        try {                                                                           \
            (void)(__VA_ARGS__);                                                        \
        } catch (...) {                                                                 \
            catch_threw_ = true;                                                        \
        }                                                                               \
        if (!catch_threw_) Catch::report_failure(__FILE__, __LINE__, "expected throw: " #__VA_ARGS__); \
    } while (0)

#define CHECK_THROWS_WITH(expr, matcher)                                                \
    do {                                                                                \
        ++Catch::stats().checks;                                                        \
        bool catch_ok_ = false;                                                         \
        std::string catch_msg_ = "<no exception>";                                      \
        try {                                                                           \
            (void)(expr);                                                               \
        } catch (const std::exception& e) {                                             \
            catch_msg_ = e.what();                                                      \
            catch_ok_ = (matcher).match(catch_msg_);                                    \
        }                                                                               \
        if (!catch_ok_) Catch::report_failure(__FILE__, __LINE__, "throw message mismatch: " + catch_msg_); \
    } while (0)

#define FAIL(msg)                                                                       \
    do {                                                                                \
        std::ostringstream catch_os_;                                                   \
        catch_os_ << msg;                                                               \
        Catch::report_failure(__FILE__, __LINE__, catch_os_.str());                     \
        throw Catch::AbortTest{};                                                       \
    } while (0)

#ifdef CATCH_CONFIG_MAIN
int main() {
    long cases = 0, failed_cases = 0;
    for (const auto& tc : Catch::registry()) {
        ++cases;
        const long before = Catch::stats().failures;
        try {
            tc.fn();
        } catch (const Catch::AbortTest&) {
        } catch (const std::exception& e) {
            Catch::report_failure(__FILE__, __LINE__, std::string(tc.name) + ": unexpected exception " + e.what());
        }
        if (Catch::stats().failures != before) {
            ++failed_cases;
            std::fprintf(stderr, "  in test case: %s\n", tc.name);
        }
    }
    std::printf("test cases: %ld | %ld passed | %ld failed; checks: %ld | %ld failed\n", cases, cases - failed_cases,
                failed_cases, Catch::stats().checks, Catch::stats().failures);
    return failed_cases == 0 ? 0 : 1;
}
#endif
