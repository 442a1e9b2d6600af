#pragma once
// Minimal test harness (no doctest/gtest offline): TEST(name) registers a
// case; CHECK records failures; main() runs all and exits non-zero on failure.
#include <cstdio>
#include <functional>
#include <string>
#include <vector>

namespace check {
struct Case {
    const char* name;
    std::function<void()> fn;
};
inline std::vector<Case>& cases() {
    static std::vector<Case> c;
    return c;
}
inline int& failures() {
    static int f = 0;
    return f;
}
struct Reg {
    Reg(const char* n, std::function<void()> f) { cases().push_back({n, std::move(f)}); }
};
}  // namespace check

#define CK_CAT2(a, b) a##b
#define CK_CAT(a, b) CK_CAT2(a, b)
#define TEST(name)                                                      \
    static void CK_CAT(test_fn_, __LINE__)();                           \
    static check::Reg CK_CAT(test_reg_, __LINE__)(name, CK_CAT(test_fn_, __LINE__)); \
    static void CK_CAT(test_fn_, __LINE__)()
#define CHECK(cond)                                                              \
    do {                                                                         \
        if (!(cond)) {                                                           \
            std::printf("  FAILED %s:%d: %s\n", __FILE__, __LINE__, #cond);     \
            ++check::failures();                                                 \
        }                                                                        \
    } while (0)
#define CHECK_THROWS(expr)                      \
    do {                                        \
        bool thrown_ = false;                   \
        try {                                   \
            expr;                               \
        } catch (...) {                         \
            thrown_ = true;                     \
        }                                       \
        CHECK(thrown_);                         \
    } while (0)

inline int run_all(int argc, char** argv) {
    int ran = 0;
    for (auto& c : check::cases()) {
        if (argc > 1 && std::string(argv[1]) != c.name) continue;
        int before = check::failures();
        c.fn();
        std::printf("%s %s\n", check::failures() == before ? "ok  " : "FAIL", c.name);
        ++ran;
    }
    std::printf("%d cases, %d failed checks\n", ran, check::failures());
    return check::failures() ? 1 : 0;
}
