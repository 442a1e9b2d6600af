// test_lrc.cpp — host-only check of the lane-range CSR layout builder
// (csrc/lrcsr_build.cpp) by a CPU restatement of the kernel (csrc/lrcsr.cu):
// every lane's walk over its 4 kLrcChunks nonzeros (row starts from bit 31,
// hot columns from the x_hot copy, padding from the zero cell), the warp's
// segmented combine with its direct stores and the unit carries, then the
// fix-up walk over units. y must equal the CSR product within 1e-12 sum|a x|,
// every row written exactly once, and the stored non-padding entries must be
// exactly the CSR's nonzeros. No GPU needed.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <random>
#include <vector>

#include "tcsr.hpp"

using namespace b200;

static int g_fail = 0;
#define CHECK(c, ...)                          \
    do {                                       \
        if (!(c)) {                            \
            std::fprintf(stderr, __VA_ARGS__); \
            std::fprintf(stderr, "\n");        \
            ++g_fail;                          \
            return;                            \
        }                                      \
    } while (0)

struct Csr {
    std::vector<std::int64_t> rp, ci;
    std::vector<double> val;
    std::int64_t rows = 0, cols = 0;
};

// rows with lengths drawn from `lens(g)`, columns from `col(g)` (a skewed
// distribution makes hot columns), ascending per row
template <typename L, typename Cf>
static Csr make(std::int64_t rows, std::int64_t cols, L lens, Cf col, unsigned seed) {
    std::mt19937_64 g(seed);
    std::uniform_real_distribution<double> u(-2, 2);
    Csr a;
    a.rows = rows;
    a.cols = cols;
    a.rp.push_back(0);
    for (std::int64_t r = 0; r < rows; ++r) {
        const std::int64_t len = lens(g, r);
        std::vector<std::int64_t> cs;
        for (std::int64_t k = 0; k < len; ++k) cs.push_back(((col(g) % cols) + cols) % cols);
        std::sort(cs.begin(), cs.end());
        for (auto c : cs) {
            a.ci.push_back(c);
            a.val.push_back(u(g));
        }
        a.rp.push_back(static_cast<std::int64_t>(a.ci.size()));
    }
    return a;
}

struct Wk {
    std::uint32_t row;
    double acc, head;
    bool in_head;
};

static void replay(const Csr& a, const char* name) {
    const std::int64_t cols = std::max<std::int64_t>(a.cols, 1);
    LrcHost h;
    lrc_build_host(a.rows, a.rp.data(), a.ci.data(), a.val.data(), cols, h);
    const std::int64_t nnz = a.rp[a.rows];
    CHECK(h.nnz == nnz && h.units == (nnz + kLrcUnit - 1) / kLrcUnit, "%s: units", name);
    std::vector<double> x(static_cast<std::size_t>(cols));
    std::mt19937_64 g(7);
    std::uniform_real_distribution<double> u(-1, 1);
    for (auto& v : x) v = u(g);
    std::vector<double> xhot(static_cast<std::size_t>(h.hot) + 1, 0.0);
    for (int i = 0; i < h.hot; ++i) xhot[i] = x[h.hot_cols[i]];
    auto map = [&](std::uint32_t r) -> std::int64_t { return h.has_empty ? h.rmap[r] : r; };
    std::vector<double> y(static_cast<std::size_t>(a.rows), 0.0);  // has_empty: zeroed first
    std::vector<int> writes(static_cast<std::size_t>(a.rows), 0);
    std::vector<LrcCarry> carry(static_cast<std::size_t>(h.units));
    std::int64_t stored = 0;
    for (std::int64_t u = 0; u < h.units; ++u) {
        Wk w[32];
        bool cont[32];
        for (int l = 0; l < 32; ++l) {
            const std::uint32_t d = h.desc[u * 32 + l];
            cont[l] = (d & kLrcCont) != 0;
            w[l] = {(d & ~kLrcCont) - (cont[l] ? 0u : 1u), 0.0, 0.0, true};
            for (int i = 0; i < kLrcChunks; ++i)
                for (int s = 0; s < 4; ++s) {
                    const std::int64_t p = u * kLrcUnit + (32 * i + l) * 4 + s;
                    const std::uint32_t c = h.col[p];
                    const double xv = (c & kLrcHot) ? xhot[c & kLrcColMask] : x[c & kLrcColMask];
                    if ((c & kLrcHot) && (c & kLrcColMask) == static_cast<std::uint32_t>(h.hot))
                        CHECK(h.val[p] == 0.0, "%s: padding with a value", name);
                    else
                        ++stored;
                    const bool st = (c & kLrcStart) != 0;
                    if (st && !w[l].in_head) {
                        y[map(w[l].row)] = w[l].acc;
                        writes[map(w[l].row)]++;
                    }
                    w[l].head = st && w[l].in_head ? w[l].acc : w[l].head;
                    w[l].in_head = w[l].in_head && !st;
                    w[l].row += st ? 1u : 0u;
                    w[l].acc = std::fma(h.val[p], xv, st ? 0.0 : w[l].acc);
                }
        }
        // the warp combine (lrcsr.cu)
        unsigned sm = 0;
        for (int l = 0; l < 32; ++l)
            if (!w[l].in_head) sm |= 1u << l;
        int seg[32];
        double S[32];
        for (int l = 0; l < 32; ++l) {
            seg[l] = 0;
            for (int k = l; k >= 0; --k)
                if (k == 0 || ((sm >> k) & 1u)) {
                    seg[l] = k;
                    break;
                }
            S[l] = 0.0;
            for (int k = seg[l]; k <= l; ++k) S[l] += w[k].acc;  // (the shuffle scan's order may differ in rounding)
        }
        for (int l = 1; l < 32; ++l)
            if ((sm >> l) & 1u) {
                const bool fresh = (sm >> seg[l - 1]) & 1u;
                if (fresh) {
                    y[map(w[l - 1].row)] = S[l - 1] + w[l].head;
                    writes[map(w[l - 1].row)]++;
                }
            }
        // the unit's carry (lrcsr.cu): head = the row open at its start
        LrcCarry c{};
        if (cont[0]) {
            int b = -1;
            for (int l = 1; l < 32; ++l)
                if ((sm >> l) & 1u) {
                    b = l;
                    break;
                }
            c.head_val = (sm & 1u) ? w[0].head : (b >= 0 ? S[b - 1] + w[b].head : S[31]);
        }
        c.tail_val = S[31];
        carry[u] = c;
    }
    // the structural crossing plan (k_lrc_plan) and the fix-up sums
    const std::int64_t base = a.rp[0];
    for (std::int64_t u = 0; u < h.units; ++u) {
        const std::int64_t last = std::min<std::int64_t>((u + 1) * kLrcUnit, nnz) - 1;
        const std::int64_t r = (std::upper_bound(a.rp.begin(), a.rp.end(), base + last) - a.rp.begin()) - 1;
        if (a.rp[r] - base < u * kLrcUnit) continue;
        const std::int64_t e = (a.rp[r + 1] - base - 1) / kLrcUnit;
        double tot = carry[u].tail_val;
        for (std::int64_t v = u + 1; v <= e; ++v) tot += carry[v].head_val;
        y[r] = tot;
        writes[r]++;
    }
    CHECK(stored == nnz, "%s: stored %lld of %lld nonzeros", name, (long long)stored, (long long)nnz);
    for (std::int64_t r = 0; r < a.rows; ++r) {
        double ref = 0.0, bound = 0.0;
        for (std::int64_t j = a.rp[r]; j < a.rp[r + 1]; ++j) {
            ref += a.val[j] * x[a.ci[j]];
            bound += std::fabs(a.val[j] * x[a.ci[j]]);
        }
        const bool empty = a.rp[r + 1] == a.rp[r];
        CHECK(writes[r] == (empty ? 0 : 1), "%s: row %lld written %d times", name, (long long)r, writes[r]);
        CHECK(std::fabs(y[r] - ref) <= 1e-12 * bound, "%s: row %lld y=%.17g ref=%.17g", name, (long long)r, y[r], ref);
    }
    std::printf("ok %s (nnz %lld, units %lld, hot %d covering %lld, empty rows %s)\n", name, (long long)nnz,
                (long long)h.units, h.hot, (long long)h.hot_covered, h.has_empty ? "yes" : "no");
}

int main() {
    // power-law: a few very long rows, many empty rows, skewed columns (hot set)
    replay(make(20000, 50000,
                [](std::mt19937_64& g, std::int64_t r) -> std::int64_t {
                    if (r % 5000 == 17) return 20000 + static_cast<std::int64_t>(g() % 5000);
                    return (g() % 2) ? 0 : static_cast<std::int64_t>(g() % 40);
                },
                [](std::mt19937_64& g) -> std::int64_t {
                    const double v = std::uniform_real_distribution<double>(0, 1)(g);
                    return static_cast<std::int64_t>(std::pow(v, 4.0) * 50000.0);
                },
                11),
           "power-law rows, skewed columns");
    // uniform columns (no hot set), short rows, no empty rows, ragged last unit
    replay(make(7777, 3000, [](std::mt19937_64& g, std::int64_t) -> std::int64_t { return 1 + g() % 9; },
                [](std::mt19937_64& g) -> std::int64_t { return static_cast<std::int64_t>(g()); }, 12),
           "short rows, uniform columns");
    // one row longer than several units, rows ending exactly at unit edges
    replay(make(300, 1000,
                [](std::mt19937_64&, std::int64_t r) -> std::int64_t { return r == 5 ? 5 * kLrcUnit : (r % 3 ? kLrcLaneNnz : 0); },
                [](std::mt19937_64& g) -> std::int64_t { return static_cast<std::int64_t>(g() % 7); }, 13),
           "lane/unit-aligned rows, a 5-unit row");
    // a single nonzero
    replay(make(1, 1, [](std::mt19937_64&, std::int64_t) -> std::int64_t { return 1; },
                [](std::mt19937_64&) -> std::int64_t { return 0; }, 14),
           "single nonzero");
    if (g_fail) {
        std::printf("FAILED %d\n", g_fail);
        return 1;
    }
    return 0;
}
