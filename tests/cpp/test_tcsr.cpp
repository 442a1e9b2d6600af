// test_tcsr.cpp — host-only check of the tiled CSR layout builder
// (csrc/tcsr_build.cpp) against the CSR it was built from, by a CPU
// restatement of the kernel's walk (csrc/tcsr.cu: lane ranges of 4-nonzero
// chunks, chunk i of lane l at (32 i + l) * 4, row starts from the key bit,
// lane descriptors = first row | continuation). Every stored nonzero is
// replayed once; y must equal the CSR product within 1e-12 sum|a x| and the
// non-padding entries must be exactly the CSR's nonzeros. No GPU needed.
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <random>
#include <vector>

#include "tcsr.hpp"

using namespace b200;

static int g_fail = 0;
#define CHECK(c, ...)                            \
    do {                                         \
        if (!(c)) {                              \
            std::fprintf(stderr, __VA_ARGS__);   \
            std::fprintf(stderr, "\n");          \
            ++g_fail;                            \
            return;                              \
        }                                        \
    } while (0)

struct Csr {
    std::vector<std::int64_t> rp, ci;
    std::vector<double> val;
    std::int64_t rows = 0, cols = 0;
};

static Csr make(std::int64_t rows, std::int64_t cols, int maxlen, double p_empty, bool banded, unsigned seed) {
    std::mt19937_64 g(seed);
    std::uniform_real_distribution<double> u(-2, 2), u01(0, 1);
    Csr a;
    a.rows = rows;
    a.cols = cols;
    a.rp.push_back(0);
    for (std::int64_t r = 0; r < rows; ++r) {
        int len = u01(g) < p_empty ? 0 : static_cast<int>(g() % (maxlen + 1));
        std::vector<std::int64_t> cs;
        for (int k = 0; k < len; ++k) {
            std::int64_t c = banded ? std::max<std::int64_t>(0, std::min<std::int64_t>(cols - 1, r + (std::int64_t)(g() % 81) - 40))
                                    : static_cast<std::int64_t>(g() % cols);
            cs.push_back(c);
        }
        std::sort(cs.begin(), cs.end());
        cs.erase(std::unique(cs.begin(), cs.end()), cs.end());
        for (std::int64_t c : cs) {
            a.ci.push_back(c);
            a.val.push_back(u(g));
        }
        a.rp.push_back(static_cast<std::int64_t>(a.ci.size()));
    }
    return a;
}

static void check_layout(const char* name, const Csr& a) {
    TcsrHost h;
    tcsr_build_host(a.rows, a.rp.data(), a.ci.data(), a.val.data(), a.cols, h);
    CHECK(h.slab_w % 8 == 0 && h.slab_w <= kSlabWMax, "%s: slab width %d", name, h.slab_w);
    CHECK(tcsr_smem_bytes(h.slab_w, h.rows_max) <= static_cast<std::size_t>(kTileSmemBudget), "%s: smem", name);
    // slab parts: equal-width slabs, a multiple of `parts` of them (parts of equal work)
    CHECK(h.parts >= 1 && (h.parts == 1 || h.nslabs % h.parts == 0), "%s: %d slabs over %d parts", name, h.nslabs,
          h.parts);
    CHECK(static_cast<std::int64_t>(h.nslabs) * h.slab_w >= a.cols &&
              static_cast<std::int64_t>(h.nslabs - 1) * h.slab_w < a.cols,
          "%s: slabs cover the columns", name);
    std::vector<double> x(a.cols), y(a.rows, 0.0), ref(a.rows, 0.0), scale(a.rows, 0.0);
    std::mt19937_64 g(7);
    std::uniform_real_distribution<double> u(-1, 1);
    for (auto& v : x) v = u(g);
    for (std::int64_t r = 0; r < a.rows; ++r)
        for (std::int64_t j = a.rp[r]; j < a.rp[r + 1]; ++j) {
            ref[r] += a.val[j] * x[a.ci[j]];
            scale[r] += std::fabs(a.val[j] * x[a.ci[j]]);
        }
    const std::int64_t per_tile = static_cast<std::int64_t>(h.nslabs) * kTileWarps + 1;
    std::int64_t real = 0;
    double absval = 0.0;
    for (std::int64_t t = 0; t < h.ntiles; ++t) {
        const std::int64_t row0 = h.tile_row0[t], base = h.tile_base[t];
        CHECK(h.tile_row0[t + 1] - row0 <= h.rows_max, "%s: tile rows", name);
        for (int k = 0; k < h.nslabs; ++k)
            for (int w = 0; w < kTileWarps; ++w) {
                const std::int64_t run = static_cast<std::int64_t>(k) * kTileWarps + w;
                const std::int32_t lo = h.woff[t * per_tile + run], hi = h.woff[t * per_tile + run + 1];
                CHECK(lo % kChunk == 0 && hi % kChunk == 0 && hi >= lo, "%s: run bounds", name);
                const int C = (hi - lo) / kChunk, m = C / 32, rr = C % 32;
                for (int lane = 0; lane < 32; ++lane) {
                    const int cnt = m + (lane < rr ? 1 : 0);
                    if (cnt == 0) continue;
                    const std::uint16_t ld = h.lrow[(t * (per_tile - 1) + run) * 32 + lane];
                    std::int64_t row = ld & 0x7fff;
                    for (int i = 0; i < cnt; ++i)
                        for (int e = 0; e < kChunk; ++e) {
                            const std::int64_t at = base + lo + (32LL * i + lane) * kChunk + e;
                            const std::uint16_t key = h.key[at];
                            if ((key & kKeyStart) && !(i == 0 && e == 0)) ++row;
                            CHECK(!((key & kKeyStart) && i == 0 && e == 0), "%s: start bit on a lane's first", name);
                            const int col = tcsr_key_col(key);
                            CHECK(col <= h.slab_w, "%s: key column", name);
                            if (col == h.slab_w) {  // the zero cell: padding / empty-row entry
                                CHECK(h.val[at] == 0.0, "%s: nonzero padding", name);
                                continue;
                            }
                            const std::int64_t gc = static_cast<std::int64_t>(k) * h.slab_w + col;
                            CHECK(gc < a.cols && row0 + row < h.tile_row0[t + 1], "%s: out of range", name);
                            y[row0 + row] += h.val[at] * x[gc];
                            ++real;
                            absval += std::fabs(h.val[at]);
                        }
                }
            }
    }
    double ref_abs = 0.0;
    std::int64_t nz = 0;
    for (double v : a.val) {
        ref_abs += std::fabs(v);
        nz += v != 0.0;
    }
    CHECK(real == nz, "%s: %lld stored nonzeros, CSR has %lld", name, (long long)real, (long long)nz);
    CHECK(std::fabs(absval - ref_abs) <= 1e-9 * ref_abs, "%s: value multiset", name);
    for (std::int64_t r = 0; r < a.rows; ++r)
        CHECK(std::fabs(y[r] - ref[r]) <= 1e-12 * scale[r] + 1e-300, "%s: row %lld %.17g vs %.17g", name,
              (long long)r, y[r], ref[r]);
    std::printf("ok %-28s rows=%lld nnz=%lld tiles=%lld slabs=%d slab_w=%d parts=%d\n", name, (long long)a.rows,
                (long long)real, (long long)h.ntiles, h.nslabs, h.slab_w, h.parts);
}

int main() {
    check_layout("random, long rows", make(20000, 50000, 300, 0.0, false, 1));
    check_layout("short rows + empties", make(700000, 30001, 3, 0.3, false, 2));   // > 148 x 4096 rows
    check_layout("banded", make(60000, 60000, 40, 0.05, true, 3));
    check_layout("one column", make(5000, 1, 1, 0.2, false, 4));
    return g_fail ? 1 : 0;
}
