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

// One (slab, warp) run of a tile: its row segments in row order, each a
// range of `js` (tile-local nonzero indices in CSR order).
struct Seg {
    std::int32_t row;    // tile-local
    std::int32_t start;  // into TileRuns::js
    std::int32_t count;
};

struct TileRuns {
    std::vector<std::int32_t> js;       // grouped by run, then row (CSR order inside a row)
    std::vector<Seg> segs;              // grouped by run, row order
    std::vector<std::int32_t> run_seg;  // runs + 1 offsets into segs
    std::vector<std::int32_t> run_js;   // runs + 1 offsets into js
};

// Collects a tile's runs (counting sort by run over the tile's nonzeros). A
// row left empty between two rows of a run gets a one-entry segment whose
// nonzero index is -1 (a zero entry), so a run's rows are consecutive.
void tile_runs(const std::int64_t* rp, const std::int64_t* ci, std::int64_t row0, const std::int64_t* wb,
               int nslabs, int slab_w, TileRuns& tr) {
    const std::int64_t runs = static_cast<std::int64_t>(nslabs) * kTileWarps;
    std::vector<std::int32_t> nnz_run(static_cast<std::size_t>(runs + 1), 0), seg_run(static_cast<std::size_t>(runs + 1), 0);
    std::vector<std::int64_t> last(static_cast<std::size_t>(runs), -1);
    for (int w = 0; w < kTileWarps; ++w)
        for (std::int64_t r = wb[w]; r < wb[w + 1]; ++r)
            for (std::int64_t j = rp[r]; j < rp[r + 1]; ++j) {
                const std::int64_t run = (ci[j] / slab_w) * kTileWarps + w;
                ++nnz_run[run + 1];
                if (last[run] != r) {
                    if (last[run] >= 0) {  // empty rows in between
                        nnz_run[run + 1] += static_cast<std::int32_t>(r - last[run] - 1);
                        seg_run[run + 1] += static_cast<std::int32_t>(r - last[run] - 1);
                    }
                    last[run] = r;
                    ++seg_run[run + 1];
                }
            }
    for (std::int64_t i = 0; i < runs; ++i) {
        nnz_run[i + 1] += nnz_run[i];
        seg_run[i + 1] += seg_run[i];
    }
    tr.js.assign(static_cast<std::size_t>(nnz_run[runs]), 0);
    tr.segs.assign(static_cast<std::size_t>(seg_run[runs]), Seg{});
    tr.run_seg = seg_run;
    tr.run_js = nnz_run;
    std::vector<std::int32_t> jc(nnz_run.begin(), nnz_run.end() - 1), sc(seg_run.begin(), seg_run.end() - 1);
    std::fill(last.begin(), last.end(), -1);
    const std::int64_t jb = rp[row0];
    for (int w = 0; w < kTileWarps; ++w)
        for (std::int64_t r = wb[w]; r < wb[w + 1]; ++r)
            for (std::int64_t j = rp[r]; j < rp[r + 1]; ++j) {
                const std::int64_t run = (ci[j] / slab_w) * kTileWarps + w;
                if (last[run] != r) {
                    if (last[run] >= 0)
                        for (std::int64_t e = last[run] + 1; e < r; ++e) {
                            tr.segs[sc[run]++] = Seg{static_cast<std::int32_t>(e - row0), jc[run], 1};
                            tr.js[jc[run]++] = -1;
                        }
                    last[run] = r;
                    tr.segs[sc[run]++] = Seg{static_cast<std::int32_t>(r - row0), jc[run], 0};
                }
                ++tr.segs[sc[run] - 1].count;
                tr.js[jc[run]++] = static_cast<std::int32_t>(j - jb);
            }
}

std::int64_t run_elems(const TileRuns& tr, std::int64_t run) {
    const std::int64_t e = tr.run_js[run + 1] - tr.run_js[run];
    return (e + kChunk - 1) / kChunk * kChunk;
}

// Writes one run (layout in b200.hpp): lane ranges of whole chunks, chunk i
// of lane l at (32 i + l) * 4. The nonzeros of one row inside one lane are
// interchangeable (the lane only sums them), so each (chunk, slot) x gather —
// one shared-memory instruction of the warp, served per half-warp — is dealt
// greedily: every lane takes the remaining nonzero of its current row
// segment whose bank pair is least used so far by that instruction's
// half-warp (LILAC_B200_TILED_BANKS=0: CSR order). Row-start bits stay with
// their positions.
void write_run(const TileRuns& tr, std::int64_t run, const std::int64_t* ci, const double* val, std::int64_t jb,
               std::int64_t slab, int slab_w, bool balance, double* hv, std::uint16_t* hk, std::uint16_t* hl) {
    const std::uint16_t pad = static_cast<std::uint16_t>(slab_w);  // the zero cell
    const std::int64_t js0 = tr.run_js[run], E = tr.run_js[run + 1] - js0;
    const std::int64_t C = (E + kChunk - 1) / kChunk, m = C / 32, r = C % 32;
    // the run's nonzeros in order, with their rows
    std::vector<std::int32_t> rowof(static_cast<std::size_t>(E));
    for (std::int32_t i = tr.run_seg[run]; i < tr.run_seg[run + 1]; ++i)
        for (std::int32_t q = 0; q < tr.segs[i].count; ++q) rowof[tr.segs[i].start - js0 + q] = tr.segs[i].row;
    auto elem = [&](std::int64_t e) {
        if (tr.js[js0 + e] < 0) return std::make_pair(pad, 0.0);  // empty row
        const std::int64_t j = jb + tr.js[js0 + e];
        return std::make_pair(static_cast<std::uint16_t>(ci[j] - slab * slab_w), val[j]);
    };
    std::int64_t cs[32], cn[32];
    for (int l = 0; l < 32; ++l) {
        cs[l] = l * m + std::min<std::int64_t>(l, r);
        cn[l] = m + (l < r ? 1 : 0);
        hl[l] = 0;
        if (cn[l] > 0) {
            const std::int64_t e0 = cs[l] * kChunk;
            hl[l] = static_cast<std::uint16_t>(rowof[e0] | (e0 > 0 && rowof[e0 - 1] == rowof[e0] ? kLaneCont : 0));
        }
    }
    // per lane: the pool of its current row segment (refilled at each start)
    std::vector<std::pair<std::uint16_t, double>> pool[32];
    for (std::int64_t i = 0; i < m + (r > 0 ? 1 : 0); ++i)
        for (int sl = 0; sl < kChunk; ++sl) {
            int cnt[2][16] = {};
            for (int l = 0; l < 32; ++l) {
                if (i >= cn[l]) continue;
                const std::int64_t e = (cs[l] + i) * kChunk + sl, at = (i * 32 + l) * kChunk + sl;
                if (e >= E) {
                    hk[at] = tcsr_key(pad, false);
                    hv[at] = 0.0;
                    continue;
                }
                const bool first = i == 0 && sl == 0;
                const bool start = !first && rowof[e] != rowof[e - 1];
                if (first || start) {  // refill: this segment's nonzeros inside the lane, in CSR order
                    const std::int64_t lane_end = std::min<std::int64_t>(E, (cs[l] + cn[l]) * kChunk);
                    pool[l].clear();
                    for (std::int64_t q = e; q < lane_end && rowof[q] == rowof[e]; ++q) pool[l].push_back(elem(q));
                    std::reverse(pool[l].begin(), pool[l].end());  // back = CSR-earliest
                }
                auto& pl = pool[l];
                std::size_t best = pl.size() - 1;
                if (balance) {
                    int best_n = cnt[l >> 4][pl[best].first & 15u];
                    for (std::size_t u = pl.size() - 1; u-- > 0 && best_n > 0;) {
                        const int n = cnt[l >> 4][pl[u].first & 15u];
                        if (n < best_n) {
                            best_n = n;
                            best = u;
                        }
                    }
                    ++cnt[l >> 4][pl[best].first & 15u];
                }
                hk[at] = tcsr_key(pl[best].first, start);
                hv[at] = pl[best].second;
                pl.erase(pl.begin() + static_cast<std::ptrdiff_t>(best));
            }
        }
}

}  // namespace

int tcsr_parts(std::int64_t rows, std::int64_t nnz, std::int64_t cols, int sms) {
    if (const char* e = std::getenv("LILAC_B200_TILE_PARTS"))  // experiments
        if (std::atoi(e) >= 1) return std::min(std::atoi(e), 8);
    (void)rows;
    if (nnz <= 0) return 1;
    // R = x bytes staged per CTA / matrix bytes streamed per CTA (P = 1).
    // Measured on row blocks of NPB class C (profiles/r02_tile_parts.md):
    // R 0.49 (whole matrix) best at P = 1; 0.98 and 1.48 at P = 2; 1.97 and
    // up at P = 4 (1/8 block: 26.2 -> 18.5 us); P = 8 loses (more slab edges).
    const double R = static_cast<double>(cols) * 8.0 * sms / (static_cast<double>(nnz) * 10.0);
    int parts = R <= 0.7 ? 1 : (R <= 1.5 ? 2 : 4);
    // every part keeps >= 2 slabs: when x is a slab or two (NPB class A,
    // 14,000 columns) staging it is cheap and parts only add the combine
    // (class A: 8.2 -> 10.3 us at P = 2)
    const std::int64_t nslabs = (cols + kSlabW - 1) / kSlabW;
    while (parts > 1 && nslabs < 2 * parts) parts /= 2;
    return parts;
}

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
    const int parts = tcsr_parts(rows, nnz, cols, device_sms());
    const std::int64_t nslabs = (cols + kSlabW - 1) / kSlabW;
    const std::int64_t tiles =
        std::max<std::int64_t>(device_sms() / parts, (rows + kMaxTileRows - 1) / kMaxTileRows);
    if (nnz / (tiles * nslabs * kTileWarps) < 256) return false;
    return gather_locality(rows, rp, ci) > 0.3;
}

double gather_locality(std::int64_t rows, const std::int64_t* rp, const std::int64_t* ci) {
    // distinct 32-byte x sectors per nonzero over windows of 32 consecutive
    // rows (a warp's worth). ~1 = every gather its own sector; -1 = unknown.
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
    return windows > 0 ? ratio_sum / windows : -1.0;
}

void tcsr_build_host(std::int64_t rows, const std::int64_t* rp, const std::int64_t* ci, const double* val,
                     std::int64_t cols, TcsrHost& h) {
    const std::int64_t base0 = rp[0];
    const std::int64_t nnz = rp[rows] - base0;
    const int sms = device_sms();
    h.cols = cols;
    // tiles: nnz-balanced, a multiple of the SM count, none taller than kMaxTileRows
    std::vector<std::int64_t> bounds;
    const char* tps = std::getenv("LILAC_B200_TILES_PER_SM");
    const std::int64_t per_sm = (tps && *tps) ? std::max(1, std::atoi(tps)) : 1;
    const std::int64_t min_tiles = (rows + kMaxTileRows - 1) / kMaxTileRows;
    int parts = tcsr_parts(rows, nnz, cols, sms);
    if (parts > 1 && min_tiles * parts > sms * per_sm) parts = 1;  // tall enough tiles anyway
    h.parts = parts;
    const std::int64_t want = std::max<std::int64_t>((sms * per_sm + parts - 1) / parts, min_tiles);
    const std::int64_t nt0 = parts > 1 ? want : (want + sms - 1) / sms * sms;
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
    // slab width: what shared memory leaves after the tallest tile's y buffer
    h.rows_max = 1;
    for (std::int64_t t = 0; t < h.ntiles; ++t)
        h.rows_max = static_cast<int>(std::max<std::int64_t>(h.rows_max, h.tile_row0[t + 1] - h.tile_row0[t]));
    h.slab_w = std::min(kSlabWMax, ((kTileSmemBudget / 8 - h.rows_max) / 2 - 2)) & ~7;
    if (const char* e = std::getenv("LILAC_B200_SLAB_W"))  // experiments: a narrower slab
        if (std::atoi(e) >= 1024) h.slab_w = std::min(h.slab_w, std::atoi(e) & ~7);
    h.nslabs = static_cast<int>((cols + h.slab_w - 1) / h.slab_w);
    if (parts > 1) {  // a multiple of `parts` slabs of equal width: parts of equal work
        const int wmax = h.slab_w;
        for (int ns = (h.nslabs + parts - 1) / parts * parts;; ns += parts) {
            const std::int64_t w = ((cols + ns - 1) / ns + 7) / 8 * 8;
            if (w <= wmax) {
                h.slab_w = static_cast<int>(w);
                h.nslabs = static_cast<int>((cols + w - 1) / w);
                break;
            }
        }
        if (h.nslabs < parts) h.parts = parts = 1;
    }
    const std::int64_t per_tile = static_cast<std::int64_t>(h.nslabs) * kTileWarps + 1;
    h.woff.assign(static_cast<std::size_t>(h.ntiles * per_tile), 0);
    h.lrow.assign(static_cast<std::size_t>(h.ntiles * (per_tile - 1) * 32), 0);

    // pass 1: warp row ranges (nnz-balanced) and per-run stored sizes
    std::vector<std::int64_t> wbounds(static_cast<std::size_t>(h.ntiles * (kTileWarps + 1)));
    std::vector<std::int64_t> relems(static_cast<std::size_t>(h.ntiles * (per_tile - 1)), 0);
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
        TileRuns tr;
        tile_runs(rp, ci, row0, wb, h.nslabs, h.slab_w, tr);
        for (std::int64_t i = 0; i + 1 < per_tile; ++i) relems[t * (per_tile - 1) + i] = run_elems(tr, i);
    });
    // element offsets, tile-relative per run
    h.tile_base.resize(h.ntiles + 1);
    h.tile_base[0] = 0;
    for (std::int64_t t = 0; t < h.ntiles; ++t) {
        std::int32_t* wo = h.woff.data() + t * per_tile;
        std::int64_t off = 0;
        for (std::int64_t i = 0; i + 1 < per_tile; ++i) {
            wo[i] = static_cast<std::int32_t>(off);
            off += relems[t * (per_tile - 1) + i];
        }
        wo[per_tile - 1] = static_cast<std::int32_t>(off);
        h.tile_base[t + 1] = h.tile_base[t] + off;
    }
    const std::int64_t total = h.tile_base[h.ntiles];
    h.val.assign(static_cast<std::size_t>(total), 0.0);
    h.key.assign(static_cast<std::size_t>(total), static_cast<std::uint16_t>(h.slab_w));

    // pass 2: the runs
    const bool balance = [] {
        const char* e = std::getenv("LILAC_B200_TILED_BANKS");
        return !(e && std::strcmp(e, "0") == 0);
    }();
    parallel_tiles(h.ntiles, [&](std::int64_t t) {
        const std::int64_t row0 = h.tile_row0[t];
        const std::int64_t tb = h.tile_base[t];
        const std::int64_t* wb = wbounds.data() + t * (kTileWarps + 1);
        const std::int32_t* wo = h.woff.data() + t * per_tile;
        TileRuns tr;
        tile_runs(rp, ci, row0, wb, h.nslabs, h.slab_w, tr);
        for (std::int64_t i = 0; i + 1 < per_tile; ++i)
            write_run(tr, i, ci, val, rp[row0], i / kTileWarps, h.slab_w, balance, h.val.data() + tb + wo[i],
                      h.key.data() + tb + wo[i], h.lrow.data() + (t * (per_tile - 1) + i) * 32);
    });
}

void TcsrOwner::upload(const TcsrHost& h) {
    cudaStream_t s = rt().stream;
    tile_row0.ensure(h.tile_row0.size() * 8);
    tile_base.ensure(h.tile_base.size() * 8);
    woff.ensure(h.woff.size() * 4);
    lrow.ensure(std::max<std::size_t>(h.lrow.size(), 1) * 2);
    val.ensure(h.val.size() * 8);
    key.ensure(h.key.size() * 2);
    B200_CUDA(cudaMemcpyAsync(tile_row0.ptr, h.tile_row0.data(), h.tile_row0.size() * 8, cudaMemcpyHostToDevice, s));
    B200_CUDA(cudaMemcpyAsync(tile_base.ptr, h.tile_base.data(), h.tile_base.size() * 8, cudaMemcpyHostToDevice, s));
    if (!h.woff.empty()) {
        B200_CUDA(cudaMemcpyAsync(woff.ptr, h.woff.data(), h.woff.size() * 4, cudaMemcpyHostToDevice, s));
        B200_CUDA(cudaMemcpyAsync(lrow.ptr, h.lrow.data(), h.lrow.size() * 2, cudaMemcpyHostToDevice, s));
    }
    if (!h.val.empty()) {
        B200_CUDA(cudaMemcpyAsync(val.ptr, h.val.data(), h.val.size() * 8, cudaMemcpyHostToDevice, s));
        B200_CUDA(cudaMemcpyAsync(key.ptr, h.key.data(), h.key.size() * 2, cudaMemcpyHostToDevice, s));
    }
    B200_CUDA(cudaStreamSynchronize(s));
    dev.ntiles = h.ntiles;
    dev.nslabs = h.nslabs;
    dev.slab_w = h.slab_w;
    dev.rows_max = h.rows_max;
    dev.cols = h.cols;
    dev.tile_row0 = tile_row0.as<std::int64_t>();
    dev.tile_base = tile_base.as<std::int64_t>();
    dev.woff = woff.as<std::int32_t>();
    dev.lrow = lrow.as<std::uint16_t>();
    dev.val = val.as<double>();
    dev.key = key.as<std::uint16_t>();
    dev.parts = h.parts;
    dev.rows = h.tile_row0.empty() ? 0 : h.tile_row0.back();
    dev.ypart = nullptr;
    dev.tile_done = nullptr;
    dev.tile_pq = nullptr;
    if (h.parts > 1) {
        ypart.ensure(static_cast<std::size_t>(h.parts) * static_cast<std::size_t>(dev.rows) * 8);
        tile_done.ensure(static_cast<std::size_t>(h.ntiles) * 4);
        tile_pq.ensure(static_cast<std::size_t>(h.ntiles) * 8);
        B200_CUDA(cudaMemsetAsync(tile_done.ptr, 0, static_cast<std::size_t>(h.ntiles) * 4, s));
        B200_CUDA(cudaStreamSynchronize(s));
        dev.ypart = ypart.as<double>();
        dev.tile_done = tile_done.as<unsigned>();
        dev.tile_pq = tile_pq.as<double>();
    }
    bytes = static_cast<std::int64_t>(tile_row0.bytes + tile_base.bytes + woff.bytes + lrow.bytes + val.bytes +
                                      key.bytes + ypart.bytes + tile_done.bytes + tile_pq.bytes);
    valid = true;
}

void TcsrOwner::release() {
    tile_row0.release();
    tile_base.release();
    woff.release();
    lrow.release();
    val.release();
    key.release();
    ypart.release();
    tile_done.release();
    tile_pq.release();
    dev = TcsrDev{};
    valid = false;
    bytes = 0;
}

bool TcsrOwner::refresh(std::int64_t rows, const std::int64_t* rp, const std::int64_t* ci, const double* v,
                        std::int64_t cols, bool monotone, std::int64_t max_row, CsrKernel policy) {
    const bool forced = policy == CsrKernel::Tiled;
    // The builder reads the caller's arrays on host threads: lazy write-back
    // bytes there are filled first, from normal context (never by the fault
    // handler on a worker thread).
    if (rows > 0) {
        host_in(rp, sizeof(std::int64_t) * static_cast<std::size_t>(rows + 1));
        const std::int64_t end = std::max<std::int64_t>(rp[rows], 0);
        host_in(ci, sizeof(std::int64_t) * static_cast<std::size_t>(end));
        host_in(v, sizeof(double) * static_cast<std::size_t>(end));
    }
    if ((policy != CsrKernel::Auto && policy != CsrKernel::Tiled) ||
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
    if (A.rows > 0) host_in(rp, sizeof(std::int64_t) * static_cast<std::size_t>(A.rows + 1));
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
    if (A.rows > 0) host_in(rp, sizeof(std::int64_t) * static_cast<std::size_t>(A.rows + 1));
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
