// lrcsr_build.cpp — host builder of the lane-range CSR layout (b200.hpp,
// kernel lrcsr.cu): an upload-time cached invariant of (row_ptr, col_ind,
// val), rebuilt only when the marshaling layer re-marshals the matrix.
//
// Steps (host threads): column frequencies -> the hot set (the most frequent
// columns, up to kLrcHotMax, kept only if they cover a useful share of the
// nonzeros) -> compact rows (nonempty, with the map back) -> every nonzero
// placed at its unit / lane / chunk slot with its encoded column -> one
// descriptor per (unit, lane).

#include "runtime.hpp"
#include "tcsr.hpp"

#include <algorithm>
#include <atomic>
#include <cstdlib>
#include <cstring>
#include <thread>
#include <vector>

namespace b200 {

namespace {

template <typename F>
void par_for(std::int64_t n, F&& f) {
    unsigned nt = std::max(1u, std::thread::hardware_concurrency());
    nt = static_cast<unsigned>(std::min<std::int64_t>(nt, std::max<std::int64_t>(1, n / 4096)));
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

// position of nonzero e (CSR order, 0-based) in the layout
inline std::int64_t lrc_pos(std::int64_t e) {
    const std::int64_t u = e / kLrcUnit, w = e % kLrcUnit;
    const std::int64_t l = w / kLrcLaneNnz, k = w % kLrcLaneNnz;
    return u * kLrcUnit + (32 * (k / 4) + l) * 4 + (k % 4);
}

}  // namespace

bool lrc_wanted(std::int64_t rows, std::int64_t nnz, std::int64_t max_row, std::int64_t cols, bool monotone,
                bool forced, double locality) {
    if (!monotone || rows <= 0 || nnz <= 0) return false;
    if (rows >= (std::int64_t(1) << 31) || cols > static_cast<std::int64_t>(kLrcColMask)) return false;
    if (forced) return true;
    // skewed rows (the merge_wanted test): a row-parallel kernel is bound by its
    // longest rows and by its dependence chains
    const double mean = static_cast<double>(nnz) / static_cast<double>(rows);
    if (max_row >= 4096 && static_cast<double>(max_row) > 32.0 * mean) return true;
    // banded rows at scale: units stream at ~0.9 of copy where the row-parallel
    // kernel reaches ~0.75 (27-point stencil, 57M nonzeros: 122 vs 142 us);
    // below ~16 units per warp slot the grid is not filled
    return locality >= 0.0 && locality <= 0.3 && nnz >= (std::int64_t(16) << 20);
}

void lrc_build_host(std::int64_t rows, const std::int64_t* rp, const std::int64_t* ci, const double* val,
                    std::int64_t cols, LrcHost& h) {
    const std::int64_t base = rp[0], nnz = rp[rows] - base;
    h = LrcHost{};
    h.nnz = nnz;
    h.units = (nnz + kLrcUnit - 1) / kLrcUnit;
    // ---- hot columns ----------------------------------------------------------
    std::vector<std::atomic<std::uint32_t>> freq(static_cast<std::size_t>(std::max<std::int64_t>(cols, 1)));
    for (auto& f : freq) f.store(0, std::memory_order_relaxed);
    par_for(nnz, [&](std::int64_t lo, std::int64_t hi) {
        for (std::int64_t j = lo; j < hi; ++j) freq[ci[base + j]].fetch_add(1, std::memory_order_relaxed);
    });
    std::vector<std::int32_t> slot(static_cast<std::size_t>(std::max<std::int64_t>(cols, 1)), -1);
    {
        std::vector<std::pair<std::uint32_t, std::int32_t>> cand;
        for (std::int64_t c = 0; c < cols; ++c) {
            const std::uint32_t f = freq[c].load(std::memory_order_relaxed);
            if (f >= 2) cand.emplace_back(f, static_cast<std::int32_t>(c));
        }
        const std::int64_t cap = lrc_hot_cap();  // 0 = no shared-memory x cache
        const std::size_t want = static_cast<std::size_t>(std::min<std::int64_t>(cap, static_cast<std::int64_t>(cand.size())));
        auto by_freq = [](const auto& a, const auto& b) { return a.first != b.first ? a.first > b.first : a.second < b.second; };
        if (want < cand.size()) std::nth_element(cand.begin(), cand.begin() + static_cast<std::ptrdiff_t>(want), cand.end(), by_freq);
        cand.resize(want);
        std::sort(cand.begin(), cand.end(), [](const auto& a, const auto& b) { return a.second < b.second; });
        std::int64_t covered = 0;
        for (const auto& c : cand) covered += c.first;
        // worth a slot only when it moves a real share of the gathers off L1TEX
        if (nnz > 0 && static_cast<double>(covered) >= 0.05 * static_cast<double>(nnz)) {
            for (std::size_t i = 0; i < cand.size(); ++i) {
                slot[cand[i].second] = static_cast<std::int32_t>(i);
                h.hot_cols.push_back(cand[i].second);
            }
            h.hot_covered = covered;
        }
    }
    h.hot = static_cast<int>(h.hot_cols.size());
    // ---- compact rows ---------------------------------------------------------
    std::vector<std::int32_t> comp(static_cast<std::size_t>(rows), -1);
    for (std::int64_t r = 0; r < rows; ++r)
        if (rp[r + 1] > rp[r]) {
            comp[r] = static_cast<std::int32_t>(h.rmap.size());
            h.rmap.push_back(static_cast<std::int32_t>(r));
        } else {
            h.empty.push_back(static_cast<std::int32_t>(r));
        }
    h.rows_c = static_cast<std::int64_t>(h.rmap.size());
    h.has_empty = h.rows_c != rows;
    if (!h.has_empty) h.rmap.clear();  // identity
    // ---- nonzeros -------------------------------------------------------------
    const std::int64_t total = h.units * kLrcUnit;
    h.val.assign(static_cast<std::size_t>(total), 0.0);
    h.col.assign(static_cast<std::size_t>(total), kLrcHot | static_cast<std::uint32_t>(h.hot));  // padding: zero cell
    par_for(rows, [&](std::int64_t lo, std::int64_t hi) {
        for (std::int64_t r = lo; r < hi; ++r) {
            for (std::int64_t j = rp[r]; j < rp[r + 1]; ++j) {
                const std::int64_t p = lrc_pos(j - base);
                const std::int64_t c = ci[j];
                std::uint32_t enc = slot[c] >= 0 ? (kLrcHot | static_cast<std::uint32_t>(slot[c]))
                                                 : static_cast<std::uint32_t>(c);
                if (j == rp[r]) enc |= kLrcStart;
                h.val[p] = val[j];
                h.col[p] = enc;
            }
        }
    });
    // ---- lane descriptors -----------------------------------------------------
    h.desc.assign(static_cast<std::size_t>(h.units * 32), 0u);
    const std::uint32_t last = static_cast<std::uint32_t>(std::max<std::int64_t>(h.rows_c - 1, 0));
    par_for(h.units * 32, [&](std::int64_t lo, std::int64_t hi) {
        for (std::int64_t q = lo; q < hi; ++q) {
            const std::int64_t e0 = (q / 32) * kLrcUnit + (q % 32) * kLrcLaneNnz;
            if (e0 >= nnz) {  // padding lane: continues the last row with zeros
                h.desc[q] = last | kLrcCont;
                continue;
            }
            // the row holding nonzero e0: last r with rp[r] <= base + e0 (empty rows skipped)
            const std::int64_t r = (std::upper_bound(rp, rp + rows + 1, base + e0) - rp) - 1;
            const bool start = rp[r] == base + e0;
            h.desc[q] = static_cast<std::uint32_t>(comp[r]) | (start ? 0u : kLrcCont);
        }
    });
}

void LrcOwner::release() {
    for (DevBuf* b : {&val, &col, &desc, &rmap, &empty, &hot_cols, &x_hot, &carry, &fix}) b->release();
    dev = LrcDev{};
    valid = false;
    bytes = 0;
    hot_covered = 0;
}

bool LrcOwner::refresh(const CsrDev& A, const std::int64_t* rp, const std::int64_t* ci, CsrKernel policy) {
    const bool forced = policy == CsrKernel::Lane;
    if ((policy != CsrKernel::Auto && !forced) || A.rows <= 0 || !A.monotone) {
        release();
        return false;
    }
    host_in(rp, sizeof(std::int64_t) * static_cast<std::size_t>(A.rows + 1));
    const std::int64_t base = rp[0], nnz = rp[A.rows] - base;
    double loc = -1.0;
    if (!forced && nnz >= (std::int64_t(16) << 20)) {
        host_in(ci + base, sizeof(std::int64_t) * static_cast<std::size_t>(nnz));
        loc = gather_locality(A.rows, rp, ci);
    }
    if (!lrc_wanted(A.rows, nnz, A.max_row, A.cols, A.monotone, forced, loc)) {
        release();
        return false;
    }
    const std::size_t w = A.col32 ? 4 : 8;
    lrc_build_device(A.rows, A.row_ptr, static_cast<const char*>(A.col) + w * static_cast<std::size_t>(base), A.col32,
                     A.val + base, nnz, A.cols, *this, rt().stream);
    return true;
}

}  // namespace b200
