// test_lrc_dev.cpp — the lane-range layout's device builder (lrc_build_device,
// csrc/lrcsr.cu) against the host builder (lrc_build_host, replayed by
// test_lrc): every array bit-identical — hot set and slots, encoded columns
// with row-start bits, values, padding, descriptors, compact-row map. Needs a
// GPU (tests/test_tcsr_layout.py runs it under -m gpu).
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <random>
#include <vector>

#include <cuda_runtime.h>

#include "runtime.hpp"
#include "tcsr.hpp"

using namespace b200;

static int g_fail = 0;

template <typename T>
static std::vector<T> back(const DevBuf& b, std::size_t n) {
    std::vector<T> h(n);
    if (n) cudaMemcpy(h.data(), b.ptr, n * sizeof(T), cudaMemcpyDeviceToHost);
    return h;
}

template <typename T>
static void same(const std::vector<T>& a, const std::vector<T>& b, const char* what, const char* name) {
    if (a.size() != b.size() || (!a.empty() && std::memcmp(a.data(), b.data(), a.size() * sizeof(T)) != 0)) {
        std::fprintf(stderr, "%s: %s differs (%zu vs %zu entries)\n", name, what, a.size(), b.size());
        ++g_fail;
    }
}

static void check(std::int64_t rows, std::int64_t cols, int maxlen, double p_empty, double skew, bool col32,
                  std::int64_t base, unsigned seed, const char* name) {
    std::mt19937_64 g(seed);
    std::uniform_real_distribution<double> u(0, 1);
    std::vector<std::int64_t> rp(1, base), ci(static_cast<std::size_t>(base), 0);
    std::vector<double> val(static_cast<std::size_t>(base), 0.0);
    for (std::int64_t r = 0; r < rows; ++r) {
        const int len = u(g) < p_empty ? 0 : static_cast<int>(g() % (maxlen + 1));
        std::vector<std::int64_t> cs;
        for (int k = 0; k < len; ++k) cs.push_back(static_cast<std::int64_t>(std::pow(u(g), skew) * cols) % cols);
        std::sort(cs.begin(), cs.end());
        for (auto c : cs) {
            ci.push_back(c);
            val.push_back(u(g) - 0.5);
        }
        rp.push_back(static_cast<std::int64_t>(ci.size()));
    }
    const std::int64_t nnz = rp[rows] - base;
    LrcHost h;
    lrc_build_host(rows, rp.data(), ci.data(), val.data(), cols, h);
    // the resident CSR as the harness keeps it: row_ptr absolute, col/val from 0
    DevBuf drp, dcol, dval;
    drp.ensure(rp.size() * 8);
    cudaMemcpy(drp.ptr, rp.data(), rp.size() * 8, cudaMemcpyHostToDevice);
    dval.ensure(val.size() * 8 + 8);
    cudaMemcpy(dval.ptr, val.data(), val.size() * 8, cudaMemcpyHostToDevice);
    if (col32) {
        std::vector<std::int32_t> c32(ci.begin(), ci.end());
        dcol.ensure(c32.size() * 4 + 4);
        cudaMemcpy(dcol.ptr, c32.data(), c32.size() * 4, cudaMemcpyHostToDevice);
    } else {
        dcol.ensure(ci.size() * 8 + 8);
        cudaMemcpy(dcol.ptr, ci.data(), ci.size() * 8, cudaMemcpyHostToDevice);
    }
    LrcOwner o;
    const std::size_t w = col32 ? 4 : 8;
    lrc_build_device(rows, drp.as<std::int64_t>(), dcol.as<char>() + w * base, col32, dval.as<double>() + base, nnz,
                     cols, o, rt().stream);
    cudaDeviceSynchronize();
    const std::size_t total = static_cast<std::size_t>(h.units) * kLrcUnit;
    if (o.dev.units != h.units || o.dev.hot != h.hot || o.dev.has_empty != h.has_empty || o.dev.rows_c != h.rows_c) {
        std::fprintf(stderr, "%s: header differs (units %lld/%lld hot %d/%d)\n", name, (long long)o.dev.units,
                     (long long)h.units, o.dev.hot, h.hot);
        ++g_fail;
        return;
    }
    same(back<double>(o.val, total), h.val, "val", name);
    same(back<std::uint32_t>(o.col, total), h.col, "col", name);
    same(back<std::uint32_t>(o.desc, static_cast<std::size_t>(h.units) * 32), h.desc, "desc", name);
    same(back<std::int32_t>(o.hot_cols, static_cast<std::size_t>(h.hot)), h.hot_cols, "hot_cols", name);
    if (h.has_empty) {
        same(back<std::int32_t>(o.rmap, static_cast<std::size_t>(h.rows_c)), h.rmap, "rmap", name);
        same(back<std::int32_t>(o.empty, static_cast<std::size_t>(rows - h.rows_c)), h.empty, "empty", name);
    }
    o.release();
    drp.release();
    dcol.release();
    dval.release();
    std::printf("ok %s (nnz %lld, hot %d)\n", name, (long long)nnz, h.hot);
}

int main() {
    ensure_init();
    check(30000, 60000, 60, 0.5, 4.0, true, 0, 1, "skewed columns, empty rows, int32");
    check(5000, 5000, 9, 0.0, 1.0, false, 0, 2, "uniform, int64");
    check(4000, 9000, 30, 0.2, 3.0, true, 17, 3, "row_ptr[0] = 17");
    check(3, 10, 2, 0.0, 1.0, true, 0, 4, "tiny");
    if (g_fail) {
        std::printf("FAILED %d\n", g_fail);
        return 1;
    }
    return 0;
}
