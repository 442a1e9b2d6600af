// tcsr_build.cpp — builds the tiled CSR layout (see b200.hpp TcsrDev) from the
// caller's host CSR arrays at upload time, and decides when it pays.
//
// The layout is a cached invariant of (row_ptr, col_ind, val): the harness
// rebuilds it only when one of them was re-marshaled. It is built on the host
// (the arrays are there anyway at upload), in parallel over tiles, in O(nnz).

#include "runtime.hpp"
#include "tcsr.hpp"

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <thread>
#include <vector>

namespace b200 {

namespace {

std::int64_t lower_bound_rows(const std::int64_t* rp, std::int64_t lo, std::int64_t hi, std::int64_t v) {
    // first r in [lo, hi] with rp[r] >= v
    return std::lower_bound(rp + lo, rp + hi + 1, v) - rp;
}

template <typename F>
void parallel_tiles(std::int64_t n, F&& f) {
    const unsigned nt = std::max(1u, std::min<unsigned>(std::thread::hardware_concurrency(), 64));
    std::vector<std::thread> th;
    for (unsigned t = 0; t < nt; ++t)
        th.emplace_back([&, t] {
            for (std::int64_t i = t; i < n; i += nt) f(i);
        });
    for (auto& x : th) x.join();
}

int device_sms() {
    int dev = 0, sms = 148;
    if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    return sms > 0 ? sms : 148;
}

}  // namespace

namespace {

// The kernel gathers x for a 128-nonzero piece as 4 warp instructions (slot s
// of every lane's 4 consecutive nonzeros); an 8-byte shared load is served
// per half-warp, and its wavefronts grow with the number of lanes hitting the
// same bank pair. The nonzeros of one row inside a piece are interchangeable
// (the kernel's sums only need them grouped by row), so each row segment's
// nonzeros are dealt to its positions greedily, each position taking the
// remaining nonzero whose bank pair is least used by its (slot, half-warp).
// Row keys and continuation bits stay with their positions.
void balance_gather_banks(double* val, std::uint32_t* key, std::int64_t lo, std::int64_t hi) {
    std::vector<std::pair<std::uint32_t, double>> pool;
    for (std::int64_t c = lo; c < hi; c += 128) {
        const std::int64_t e = std::min<std::int64_t>(hi, c + 128);
        int cnt[4][2][16] = {};
        for (std::int64_t a = c; a < e;) {
            std::int64_t b = a + 1;
            while (b < e && (key[b] >> 16) == (key[a] >> 16)) ++b;
            pool.clear();
            for (std::int64_t q = a; q < b; ++q) pool.emplace_back(key[q] & kKeyColMask, val[q]);
            for (std::int64_t q = a; q < b; ++q) {
                const int off = static_cast<int>(q - c), slot = off & 3, half = (off >> 2) >> 4;
                std::size_t best = 0;
                int best_n = 1 << 30;
                for (std::size_t u = 0; u < pool.size(); ++u) {
                    const int n = cnt[slot][half][pool[u].first & 15u];
                    if (n < best_n) {
                        best_n = n;
                        best = u;
                    }
                }
                key[q] = (key[q] & ~kKeyColMask) | pool[best].first;
                val[q] = pool[best].second;
                ++cnt[slot][half][pool[best].first & 15u];
                pool[best] = pool.back();
                pool.pop_back();
            }
            a = b;
        }
    }
}

}  // namespace

bool tcsr_wanted(std::int64_t rows, const std::int64_t* rp, const std::int64_t* ci, std::int64_t cols,
                 bool monotone, std::int64_t max_row, bool forced) {
    if (!monotone || rows <= 0) return false;
    const std::int64_t nnz = rp[rows] - rp[0];
    if (nnz <= 0 || cols <= 0) return false;
    if (forced) return true;
    if (nnz < (std::int64_t(1) << 20) || rows < 148 * kTileWarps) return false;
    // one row must not dominate a warp's share (the tiled kernel never splits rows)
    const std::int64_t per_warp = nnz / (static_cast<std::int64_t>(device_sms()) * kTileWarps);
    if (max_row > 16 * std::max<std::int64_t>(per_warp, 64)) return false;
    // every tile re-reads all of x slab by slab: each (slab, warp) run must be
    // long enough to amortise a slab (Kronecker scale 22 has ~41 nonzeros per
    // run over 342 slabs and loses 40x; NPB class C has ~590 over 13)
    const std::int64_t nslabs = (cols + kSlabW - 1) / kSlabW;
    const std::int64_t tiles = std::max<std::int64_t>(device_sms(), (rows + kMaxTileRows - 1) / kMaxTileRows);
    if (nnz / (tiles * nslabs * kTileWarps) < 256) return false;
    // gather locality: distinct 32-byte x sectors per nonzero over windows of
    // 32 consecutive rows (a warp's worth). ~1 = every gather its own sector.
    double ratio_sum = 0;
    int windows = 0;
    std::vector<std::int64_t> sec;
    for (int w = 0; w < 64; ++w) {
        const std::int64_t r0 = rows * w / 64, r1 = std::min(rows, r0 + 32);
        sec.clear();
        for (std::int64_t j = rp[r0]; j < rp[r1]; ++j) sec.push_back(ci[j] >> 2);
        if (sec.size() < 64) continue;
        std::sort(sec.begin(), sec.end());
        const auto distinct = std::unique(sec.begin(), sec.end()) - sec.begin();
        ratio_sum += static_cast<double>(distinct) / static_cast<double>(sec.size());
        ++windows;
    }
    return windows > 0 && ratio_sum / windows > 0.3;
}

void tcsr_build_host(std::int64_t rows, const std::int64_t* rp, const std::int64_t* ci, const double* val,
                     std::int64_t cols, TcsrHost& h) {
    const std::int64_t base0 = rp[0];
    const std::int64_t nnz = rp[rows] - base0;
    const int sms = device_sms();
    h.cols = cols;
    h.nslabs = static_cast<int>((cols + kSlabW - 1) / kSlabW);
    // tiles: nnz-balanced, a multiple of the SM count, none taller than kMaxTileRows
    std::vector<std::int64_t> bounds;
    const char* tps = std::getenv("LILAC_B200_TILES_PER_SM");
    const std::int64_t per_sm = (tps && *tps) ? std::max(1, std::atoi(tps)) : 1;
    const std::int64_t want = std::max<std::int64_t>(sms * per_sm, (rows + kMaxTileRows - 1) / kMaxTileRows);
    const std::int64_t nt0 = (want + sms - 1) / sms * sms;
    bounds.push_back(0);
    for (std::int64_t g = 1; g < nt0; ++g) {
        std::int64_t r = lower_bound_rows(rp, 0, rows, base0 + (nnz * g + nt0 - 1) / nt0);
        r = std::max(std::min(r, rows), bounds.back());
        bounds.push_back(r);
    }
    bounds.push_back(rows);
    h.tile_row0.clear();
    for (std::size_t t = 0; t + 1 < bounds.size(); ++t) {
        const std::int64_t a = bounds[t], b = bounds[t + 1];
        const std::int64_t pieces = std::max<std::int64_t>(1, (b - a + kMaxTileRows - 1) / kMaxTileRows);
        for (std::int64_t p = 0; p < pieces; ++p) h.tile_row0.push_back(a + (b - a) * p / pieces);
    }
    h.tile_row0.push_back(rows);
    h.ntiles = static_cast<std::int64_t>(h.tile_row0.size()) - 1;
    const std::int64_t per_tile = static_cast<std::int64_t>(h.nslabs) * kTileWarps + 1;
    h.woff.assign(static_cast<std::size_t>(h.ntiles * per_tile), 0);

    // pass 1: warp row ranges (nnz-balanced) and per-(slab, warp) counts
    std::vector<std::int64_t> wbounds(static_cast<std::size_t>(h.ntiles * (kTileWarps + 1)));
    std::vector<std::int64_t> counts(static_cast<std::size_t>(h.ntiles * (per_tile - 1)), 0);
    std::vector<std::int64_t> padded(static_cast<std::size_t>(h.ntiles), 0);
    parallel_tiles(h.ntiles, [&](std::int64_t t) {
        const std::int64_t row0 = h.tile_row0[t], row1 = h.tile_row0[t + 1];
        std::int64_t* wb = wbounds.data() + t * (kTileWarps + 1);
        wb[0] = row0;
        const std::int64_t tn = rp[row1] - rp[row0];
        for (int g = 1; g < kTileWarps; ++g) {
            std::int64_t r = lower_bound_rows(rp, row0, row1, rp[row0] + (tn * g + kTileWarps - 1) / kTileWarps);
            wb[g] = std::max(std::min(r, row1), wb[g - 1]);
        }
        wb[kTileWarps] = row1;
        std::int64_t* cnt = counts.data() + t * (per_tile - 1);
        for (int w = 0; w < kTileWarps; ++w)
            for (std::int64_t r = wb[w]; r < wb[w + 1]; ++r)
                for (std::int64_t j = rp[r]; j < rp[r + 1]; ++j) cnt[(ci[j] / kSlabW) * kTileWarps + w]++;
        std::int64_t tot = 0;
        for (std::int64_t i = 0; i + 1 < per_tile; ++i) tot += (cnt[i] + kRunAlign - 1) / kRunAlign * kRunAlign;
        padded[t] = tot;
    });
    // tile bases: every run starts on a kRunAlign-element boundary and is padded
    // to a multiple of it (pad entries: val 0, sentinel row), so the kernel
    // never masks individual elements
    h.tile_base.resize(h.ntiles + 1);
    h.tile_base[0] = 0;
    for (std::int64_t t = 0; t < h.ntiles; ++t) h.tile_base[t + 1] = h.tile_base[t] + padded[t];
    const std::int64_t total = h.tile_base[h.ntiles];
    h.val.assign(static_cast<std::size_t>(total), 0.0);
    h.key.assign(static_cast<std::size_t>(total), kPadKey);

    // pass 2: offsets and scatter (slab-major, warp range, row order kept),
    // then the bank balancing of every run (LILAC_B200_TILED_BANKS=0: off)
    const bool balance = [] {
        const char* e = std::getenv("LILAC_B200_TILED_BANKS");
        return !(e && std::strcmp(e, "0") == 0);
    }();
    parallel_tiles(h.ntiles, [&](std::int64_t t) {
        const std::int64_t row0 = h.tile_row0[t];
        const std::int64_t tb = h.tile_base[t];
        const std::int64_t* wb = wbounds.data() + t * (kTileWarps + 1);
        const std::int64_t* cnt = counts.data() + t * (per_tile - 1);
        std::int32_t* wo = h.woff.data() + t * per_tile;
        std::int64_t off = 0;
        for (std::int64_t i = 0; i + 1 < per_tile; ++i) {
            wo[i] = static_cast<std::int32_t>(off);
            off += (cnt[i] + kRunAlign - 1) / kRunAlign * kRunAlign;
        }
        wo[per_tile - 1] = static_cast<std::int32_t>(off);
        std::vector<std::int64_t> cur(wo, wo + per_tile);
        std::vector<std::int64_t> last(static_cast<std::size_t>(per_tile), -1);  // last row written per run
        for (int w = 0; w < kTileWarps; ++w)
            for (std::int64_t r = wb[w]; r < wb[w + 1]; ++r) {
                const std::uint32_t lrow = static_cast<std::uint32_t>(r - row0) << 16;
                for (std::int64_t j = rp[r]; j < rp[r + 1]; ++j) {
                    const std::int64_t k = ci[j] / kSlabW;
                    const std::int64_t run = k * kTileWarps + w;
                    const std::int64_t pos = tb + cur[run]++;
                    h.val[pos] = val[j];
                    h.key[pos] = lrow | (last[run] == r ? kKeyCont : 0u) | static_cast<std::uint32_t>(ci[j] - k * kSlabW);
                    last[run] = r;
                }
            }
        if (balance)
            for (std::int64_t i = 0; i + 1 < per_tile; ++i)
                balance_gather_banks(h.val.data() + tb, h.key.data() + tb, wo[i], wo[i + 1]);
    });
}

void TcsrOwner::upload(const TcsrHost& h) {
    cudaStream_t s = rt().stream;
    tile_row0.ensure(h.tile_row0.size() * 8);
    tile_base.ensure(h.tile_base.size() * 8);
    woff.ensure(h.woff.size() * 4);
    val.ensure(h.val.size() * 8);
    key.ensure(h.key.size() * 4);
    B200_CUDA(cudaMemcpyAsync(tile_row0.ptr, h.tile_row0.data(), h.tile_row0.size() * 8, cudaMemcpyHostToDevice, s));
    B200_CUDA(cudaMemcpyAsync(tile_base.ptr, h.tile_base.data(), h.tile_base.size() * 8, cudaMemcpyHostToDevice, s));
    if (!h.woff.empty())
        B200_CUDA(cudaMemcpyAsync(woff.ptr, h.woff.data(), h.woff.size() * 4, cudaMemcpyHostToDevice, s));
    if (!h.val.empty()) {
        B200_CUDA(cudaMemcpyAsync(val.ptr, h.val.data(), h.val.size() * 8, cudaMemcpyHostToDevice, s));
        B200_CUDA(cudaMemcpyAsync(key.ptr, h.key.data(), h.key.size() * 4, cudaMemcpyHostToDevice, s));
    }
    B200_CUDA(cudaStreamSynchronize(s));
    dev.ntiles = h.ntiles;
    dev.nslabs = h.nslabs;
    dev.cols = h.cols;
    dev.tile_row0 = tile_row0.as<std::int64_t>();
    dev.tile_base = tile_base.as<std::int64_t>();
    dev.woff = woff.as<std::int32_t>();
    dev.val = val.as<double>();
    dev.key = key.as<std::uint32_t>();
    bytes = static_cast<std::int64_t>(tile_row0.bytes + tile_base.bytes + woff.bytes + val.bytes + key.bytes);
    valid = true;
}

void TcsrOwner::release() {
    tile_row0.release();
    tile_base.release();
    woff.release();
    val.release();
    key.release();
    dev = TcsrDev{};
    valid = false;
    bytes = 0;
}

bool TcsrOwner::refresh(std::int64_t rows, const std::int64_t* rp, const std::int64_t* ci, const double* v,
                        std::int64_t cols, bool monotone, std::int64_t max_row, CsrKernel policy) {
    const bool forced = policy == CsrKernel::Tiled;
    if (policy == CsrKernel::Vector || policy == CsrKernel::Exact ||
        !tcsr_wanted(rows, rp, ci, cols, monotone, max_row, forced)) {
        release();
        return false;
    }
    TcsrHost h;
    tcsr_build_host(rows, rp, ci, v, cols, h);
    upload(h);
    return true;
}

bool merge_wanted(std::int64_t rows, std::int64_t nnz, std::int64_t max_row, bool monotone, bool forced) {
    if (!monotone || rows <= 0) return false;
    if (forced) return true;
    const double mean = static_cast<double>(nnz) / static_cast<double>(rows);
    return max_row >= 4096 && static_cast<double>(max_row) > 32.0 * mean;
}

bool MergeOwner::refresh(const CsrDev& A, const std::int64_t* rp, CsrKernel policy) {
    const std::int64_t nnz = A.rows > 0 ? rp[A.rows] - rp[0] : 0;
    // built on request only: for Auto the split plan serves skewed matrices
    // (faster on the Kronecker operator)
    const bool forced = policy == CsrKernel::Merge;
    if (!forced || !merge_wanted(A.rows, nnz, A.max_row, A.monotone, forced)) {
        release();
        return false;
    }
    const std::int64_t n = merge_ctas(A.rows, nnz);
    coord_row.ensure(sizeof(std::int64_t) * (n + 1));
    coord_nz.ensure(sizeof(std::int64_t) * (n + 1));
    carry_row.ensure(sizeof(std::int64_t) * std::max<std::int64_t>(n, 1));
    carry_val.ensure(sizeof(double) * std::max<std::int64_t>(n, 1));
    launch_merge_plan(A.row_ptr, A.rows, nnz, coord_row.as<std::int64_t>(), coord_nz.as<std::int64_t>(), rt().stream);
    B200_CUDA(cudaStreamSynchronize(rt().stream));
    dev.nctas = n;
    dev.coord_row = coord_row.as<std::int64_t>();
    dev.coord_nz = coord_nz.as<std::int64_t>();
    dev.carry_row = carry_row.as<std::int64_t>();
    dev.carry_val = carry_val.as<double>();
    valid = true;
    return true;
}

bool SplitOwner::refresh(const CsrDev& A, const std::int64_t* rp, CsrKernel policy) {
    const std::int64_t nnz = A.rows > 0 ? rp[A.rows] - rp[0] : 0;
    const bool forced = policy == CsrKernel::Split;
    if ((policy != CsrKernel::Auto && !forced) || !merge_wanted(A.rows, nnz, A.max_row, A.monotone, forced)) {
        release();
        return false;
    }
    // rows longer than 8 vector-kernel steps of the chosen width go to chunks
    const std::int64_t short_max = std::max<std::int64_t>(64, 32 * csr_vector_width(A));
    std::vector<std::int64_t> lrows, lfirst, clo, chi, crow;
    std::int64_t nnz_short = 0;
    for (std::int64_t r = 0; r < A.rows; ++r) {
        const std::int64_t a = rp[r], b = rp[r + 1];
        if (b - a <= short_max) {
            nnz_short += std::max<std::int64_t>(b - a, 0);
            continue;
        }
        lfirst.push_back(static_cast<std::int64_t>(clo.size()));
        for (std::int64_t c = a; c < b; c += kSplitChunk) {
            clo.push_back(c);
            chi.push_back(std::min(b, c + kSplitChunk));
            crow.push_back(static_cast<std::int64_t>(lrows.size()));
        }
        lrows.push_back(r);
    }
    lfirst.push_back(static_cast<std::int64_t>(clo.size()));
    auto put = [](DevBuf& d, const std::vector<std::int64_t>& h) {
        d.ensure(sizeof(std::int64_t) * std::max<std::size_t>(h.size(), 1));
        if (!h.empty())
            B200_CUDA(cudaMemcpyAsync(d.ptr, h.data(), h.size() * sizeof(std::int64_t), cudaMemcpyHostToDevice,
                                      rt().stream));
    };
    put(long_rows, lrows);
    put(long_first, lfirst);
    put(chunk_lo, clo);
    put(chunk_hi, chi);
    put(chunk_row, crow);
    partial.ensure(sizeof(double) * std::max<std::size_t>(clo.size(), 1));
    done.ensure(sizeof(unsigned) * std::max<std::size_t>(lrows.size(), 1));
    work.ensure(sizeof(unsigned long long));
    B200_CUDA(cudaMemsetAsync(done.ptr, 0, sizeof(unsigned) * std::max<std::size_t>(lrows.size(), 1), rt().stream));
    B200_CUDA(cudaStreamSynchronize(rt().stream));
    dev.short_max = short_max;
    dev.nlong = static_cast<std::int64_t>(lrows.size());
    dev.nchunks = static_cast<std::int64_t>(clo.size());
    dev.long_rows = long_rows.as<std::int64_t>();
    dev.long_first = long_first.as<std::int64_t>();
    dev.chunk_lo = chunk_lo.as<std::int64_t>();
    dev.chunk_hi = chunk_hi.as<std::int64_t>();
    dev.chunk_row = chunk_row.as<std::int64_t>();
    dev.partial = partial.as<double>();
    dev.done = done.as<unsigned>();
    dev.work = work.as<unsigned long long>();
    dev.nnz_short = nnz_short;
    valid = true;
    return true;
}

void SplitOwner::release() {
    long_rows.release();
    long_first.release();
    chunk_lo.release();
    chunk_hi.release();
    chunk_row.release();
    partial.release();
    done.release();
    work.release();
    dev = SplitDev{};
    valid = false;
}

void MergeOwner::release() {
    coord_row.release();
    coord_nz.release();
    carry_row.release();
    carry_val.release();
    dev = MergeDev{};
    valid = false;
}

}  // namespace b200
