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
#include "exchange.hpp"
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

// Column footprint of a row block: [min col, max col + 1) over its nonzeros
// ({0, 0} when empty) — the replica entries the block's SpMV reads.
extern "C" void b200_shard_footprint(std::int64_t rows, const std::int64_t* row_ptr, const std::int64_t* col_ind,
                                     std::int64_t* fmin, std::int64_t* fmax) {
    std::int64_t lo = INT64_MAX, hi = -1;
    if (rows > 0)
        for (std::int64_t j = row_ptr[0]; j < row_ptr[rows]; ++j) {
            lo = std::min(lo, col_ind[j]);
            hi = std::max(hi, col_ind[j]);
        }
    *fmin = hi < 0 ? 0 : lo;
    *fmax = hi < 0 ? 0 : hi + 1;
}

// The exchange plan of the sharded driver: out[(s * world + r) * 2 + {0, 1}] =
// the part of shard s's slice (slice-relative [lo, hi)) that rank r reads.
extern "C" void b200_dist_send_ranges(int world, const std::int64_t* bounds, const std::int64_t* fmin,
                                      const std::int64_t* fmax, std::int64_t* out) {
    if (world <= 0) return;
    const std::vector<std::int64_t> lo(fmin, fmin + world), hi(fmax, fmax + world);
    for (int s = 0; s < world; ++s) {
        const std::vector<std::int64_t> r = b200::send_ranges(bounds[s], bounds[s + 1] - bounds[s], lo, hi);
        std::copy(r.begin(), r.end(), out + static_cast<std::ptrdiff_t>(s) * 2 * world);
    }
}

// ---- Graph500 Kronecker generator (SURVEY §8(d) input 4) ---------------------------
//
// Edge e's endpoints come from `scale` quadrant choices with probabilities
// A/B/C/D (Graph500: 0.57/0.19/0.19/0.05): per bit, u1 = U(e, 2 bit), u2 =
// U(e, 2 bit + 1); i = u1 > A+B; j = u2 > (i ? C/(1-A-B) : A/(A+B)). The
// uniforms are counter-based (splitmix64 of seed, edge, draw), so edges are
// generated in parallel and the graph depends only on (scale, edgefactor,
// seed). Vertex labels are then permuted (Fisher-Yates driven by the same
// hash), as Graph500 does, and the PageRank operator is built: CSR of the
// transpose (row = dst), columns ascending per row (duplicate edges kept),
// val = 1/outdeg(src).

namespace {

inline std::uint64_t mix64(std::uint64_t z) {
    z += 0x9e3779b97f4a7c15ull;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
}

inline double unit(std::uint64_t seed, std::uint64_t e, std::uint64_t k) {
    const std::uint64_t h = mix64(mix64(seed ^ mix64(e)) + k);
    return static_cast<double>(h >> 11) * 0x1.0p-53;
}

}  // namespace

extern "C" int b200_gen_kronecker(int scale, int edgefactor, std::uint64_t seed, double a, double b, double c,
                                  std::int64_t* row_ptr, std::int64_t* col_ind, double* val) {
    return boundary("b200_gen_kronecker", [&] {
        if (scale < 1 || scale > 30 || edgefactor < 1) throw Error(Errc::DataError, "scale 1..30, edgefactor >= 1");
        const std::int64_t n = std::int64_t(1) << scale, m = static_cast<std::int64_t>(edgefactor) * n;
        const double ab = a + b, c_norm = c / (1.0 - ab), a_norm = a / ab;
        std::vector<std::int64_t> src(static_cast<std::size_t>(m)), dst(static_cast<std::size_t>(m));
        parallel_for(m, [&](std::int64_t lo, std::int64_t hi) {
            for (std::int64_t e = lo; e < hi; ++e) {
                std::int64_t s = 0, d = 0;
                for (int ib = 0; ib < scale; ++ib) {
                    const int ii = unit(seed, static_cast<std::uint64_t>(e), 2u * ib) > ab;
                    const double thr = ii ? c_norm : a_norm;
                    const int jj = unit(seed, static_cast<std::uint64_t>(e), 2u * ib + 1) > thr;
                    s |= static_cast<std::int64_t>(ii) << ib;
                    d |= static_cast<std::int64_t>(jj) << ib;
                }
                src[e] = s;
                dst[e] = d;
            }
        });
        // vertex relabelling: Fisher-Yates with hashed draws
        std::vector<std::int64_t> perm(static_cast<std::size_t>(n));
        std::iota(perm.begin(), perm.end(), std::int64_t(0));
        for (std::int64_t i = n - 1; i > 0; --i) {
            const std::uint64_t h = mix64(mix64(seed ^ 0x5eedull) + static_cast<std::uint64_t>(i));
            const std::int64_t j = static_cast<std::int64_t>(h % static_cast<std::uint64_t>(i + 1));
            std::swap(perm[i], perm[j]);
        }
        parallel_for(m, [&](std::int64_t lo, std::int64_t hi) {
            for (std::int64_t e = lo; e < hi; ++e) {
                src[e] = perm[src[e]];
                dst[e] = perm[dst[e]];
            }
        });
        std::vector<std::int64_t> outdeg(static_cast<std::size_t>(n), 0);
        std::fill(row_ptr, row_ptr + n + 1, 0);
        for (std::int64_t e = 0; e < m; ++e) {
            ++outdeg[src[e]];
            ++row_ptr[dst[e] + 1];
        }
        for (std::int64_t i = 0; i < n; ++i) row_ptr[i + 1] += row_ptr[i];
        {  // bucket by destination row (stable), then sort each row's sources
            std::vector<std::int64_t> fill(row_ptr, row_ptr + n);
            for (std::int64_t e = 0; e < m; ++e) col_ind[fill[dst[e]]++] = src[e];
        }
        parallel_for(n, [&](std::int64_t lo, std::int64_t hi) {
            for (std::int64_t r = lo; r < hi; ++r) {
                std::sort(col_ind + row_ptr[r], col_ind + row_ptr[r + 1]);
                for (std::int64_t j = row_ptr[r]; j < row_ptr[r + 1]; ++j)
                    val[j] = 1.0 / static_cast<double>(outdeg[col_ind[j]]);
            }
        });
    });
}
