// workloads.cpp — host-side synthesis of benchmark inputs and the row
// partition of the multi-GPU driver (sections 6-7 of include/lilac_b200.h).
//
// NPB makea: NPB 3.x cg's sprnvc/vecset/makea/sparse restated. sparse()
// sums duplicate (row, col) triples in generation order via insertion into
// pre-counted row slots; here the same sums come from a stable bucket sort by
// row followed by a stable per-row sort by column, so the values are
// bit-identical (each entry = ((0.0 + va_1) + va_2) + ... in generation
// order) at O(nnz log row) cost and in parallel across rows.

#include "lilac_b200.h"
#include "runtime.hpp"

#include <algorithm>
#include <cmath>
#include <numeric>
#include <thread>
#include <vector>

using namespace b200;

namespace {

// randlc: x <- a*x mod 2^46, returns x * 2^-46 (exact in 64-bit integers).
struct Randlc {
    std::uint64_t x;
    std::uint64_t a;
    double next() {
        const unsigned __int128 p = static_cast<unsigned __int128>(a) * x;
        x = static_cast<std::uint64_t>(p & ((static_cast<unsigned __int128>(1) << 46) - 1));
        return std::ldexp(static_cast<double>(x), -46);
    }
};

struct Triple {
    std::int64_t col;
    double v;
};

template <typename F>
void parallel_for(std::int64_t n, F&& f) {
    unsigned nt = std::max(1u, std::thread::hardware_concurrency());
    nt = static_cast<unsigned>(std::min<std::int64_t>(nt, std::max<std::int64_t>(1, n / 1024)));
    if (nt <= 1) {
        f(0, n);
        return;
    }
    std::vector<std::thread> th;
    for (unsigned t = 0; t < nt; ++t) {
        const std::int64_t lo = n * t / nt, hi = n * (t + 1) / nt;
        th.emplace_back([&f, lo, hi] { f(lo, hi); });
    }
    for (auto& t : th) t.join();
}

}  // namespace

extern "C" int b200_gen_npb(std::int64_t n, int nonzer, double shift, std::int64_t* row_ptr, std::int64_t* col_ind,
                            double* val, std::int64_t* nnz_out) {
    return boundary("b200_gen_npb", [&] {
        if (n <= 0 || nonzer <= 0 || nonzer > 60) throw Error(Errc::DataError, "bad NPB parameters");
        const double rcond = 0.1;
        const int w = nonzer + 1;
        Randlc g{314159265ull, 1220703125ull};
        (void)g.next();  // main: zeta = randlc(&tran, amult)
        std::int64_t nn1 = 1;
        do {
            nn1 *= 2;
        } while (nn1 < n);

        std::vector<int> arow(n);
        std::vector<std::int64_t> acol(static_cast<std::size_t>(n) * w);
        std::vector<double> aelt(static_cast<std::size_t>(n) * w);
        for (std::int64_t i = 0; i < n; ++i) {
            // sprnvc: nonzer distinct positions in [1, n]
            int nzv = 0;
            std::int64_t* iv = &acol[i * w];
            double* v = &aelt[i * w];
            while (nzv < nonzer) {
                const double vecelt = g.next();
                const double vecloc = g.next();
                const std::int64_t pos = static_cast<std::int64_t>(static_cast<double>(nn1) * vecloc) + 1;
                if (pos > n) continue;
                bool dup = false;
                for (int k = 0; k < nzv; ++k) dup |= iv[k] == pos;
                if (dup) continue;
                v[nzv] = vecelt;
                iv[nzv] = pos;
                ++nzv;
            }
            // vecset(i+1, 0.5)
            bool set = false;
            for (int k = 0; k < nzv; ++k)
                if (iv[k] == i + 1) {
                    v[k] = 0.5;
                    set = true;
                }
            if (!set) {
                v[nzv] = 0.5;
                iv[nzv] = i + 1;
                ++nzv;
            }
            for (int k = 0; k < nzv; ++k) iv[k] -= 1;  // 0-based
            arow[i] = nzv;
        }
        // size_i = ratio^i by repeated multiplication, as sparse() does
        std::vector<double> size(n);
        const double ratio = std::pow(rcond, 1.0 / static_cast<double>(n));
        double sz = 1.0;
        for (std::int64_t i = 0; i < n; ++i) {
            size[i] = sz;
            sz *= ratio;
        }
        // bucket triples by row (stable: generation order kept inside a row)
        std::vector<std::int64_t> start(n + 1, 0);
        for (std::int64_t i = 0; i < n; ++i)
            for (int e = 0; e < arow[i]; ++e) start[acol[i * w + e] + 1] += arow[i];
        for (std::int64_t j = 0; j < n; ++j) start[j + 1] += start[j];
        std::vector<Triple> trip(static_cast<std::size_t>(start[n]));
        std::vector<std::int64_t> fill(start.begin(), start.end() - 1);
        for (std::int64_t i = 0; i < n; ++i) {
            for (int a = 0; a < arow[i]; ++a) {
                const std::int64_t j = acol[i * w + a];
                const double scale = size[i] * aelt[i * w + a];
                for (int b = 0; b < arow[i]; ++b) {
                    const std::int64_t jcol = acol[i * w + b];
                    double va = aelt[i * w + b] * scale;
                    if (jcol == j && j == i) va = va + rcond - shift;
                    trip[fill[j]++] = {jcol, va};
                }
            }
        }
        // per row: stable sort by column, sum duplicates in order
        std::vector<std::int64_t> count(n);
        parallel_for(n, [&](std::int64_t lo, std::int64_t hi) {
            for (std::int64_t j = lo; j < hi; ++j) {
                Triple* b = trip.data() + start[j];
                Triple* e = trip.data() + start[j + 1];
                std::stable_sort(b, e, [](const Triple& p, const Triple& q) { return p.col < q.col; });
                std::int64_t m = 0;
                for (Triple* t = b; t < e;) {
                    const std::int64_t c = t->col;
                    double acc = 0.0;
                    for (; t < e && t->col == c; ++t) acc = acc + t->v;
                    b[m++] = {c, acc};
                }
                count[j] = m;
            }
        });
        row_ptr[0] = 0;
        for (std::int64_t j = 0; j < n; ++j) row_ptr[j + 1] = row_ptr[j] + count[j];
        *nnz_out = row_ptr[n];
        if (col_ind && val) {
            parallel_for(n, [&](std::int64_t lo, std::int64_t hi) {
                for (std::int64_t j = lo; j < hi; ++j) {
                    const Triple* b = trip.data() + start[j];
                    for (std::int64_t k = 0; k < count[j]; ++k) {
                        col_ind[row_ptr[j] + k] = b[k].col;
                        val[row_ptr[j] + k] = b[k].v;
                    }
                }
            });
        }
    });
}

extern "C" void b200_partition_rows(std::int64_t rows, const std::int64_t* row_ptr, int k, std::int64_t* bounds) {
    if (k <= 0) return;
    const std::int64_t base = rows > 0 ? row_ptr[0] : 0;
    const std::int64_t nnz = rows > 0 ? row_ptr[rows] - base : 0;
    bounds[0] = 0;
    for (int g = 1; g < k; ++g) {
        const std::int64_t target = base + (nnz * g + k - 1) / k;
        std::int64_t r = rows > 0 ? std::lower_bound(row_ptr, row_ptr + rows + 1, target) - row_ptr : 0;
        r = std::min(r, rows);
        r = std::max(r, bounds[g - 1]);
        bounds[g] = r;
    }
    bounds[k] = rows;
}
