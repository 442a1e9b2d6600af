#pragma once
// tcsr.hpp — host side of the tiled CSR layout (builder + device owner).

#include "b200.hpp"

#include <cstdint>
#include <vector>

namespace b200 {

struct TcsrHost {
    std::int64_t ntiles = 0;
    int nslabs = 0;
    int slab_w = kSlabW, rows_max = kMaxTileRows;
    int parts = 1;  // slab parts per tile (TcsrDev::parts)
    std::int64_t cols = 0;
    std::vector<std::int64_t> tile_row0, tile_base;
    std::vector<std::int32_t> woff;
    std::vector<std::uint16_t> lrow;
    std::vector<double> val;
    std::vector<std::uint16_t> key;
};

// Does the tiled layout pay for this matrix? (monotone row_ptr, >= 1M nnz,
// no row dominating a warp's share, and poor x-gather locality.) `forced`
// skips the size/locality tests.
bool tcsr_wanted(std::int64_t rows, const std::int64_t* row_ptr, const std::int64_t* col_ind, std::int64_t cols,
                 bool monotone, std::int64_t max_row, bool forced);
// distinct x sectors per nonzero over 64 sampled 32-row windows (1 = no
// locality at all; -1 = too few nonzeros to tell)
double gather_locality(std::int64_t rows, const std::int64_t* row_ptr, const std::int64_t* col_ind);
// Slab parts per tile for a matrix (TcsrDev::parts; LILAC_B200_TILE_PARTS overrides).
int tcsr_parts(std::int64_t rows, std::int64_t nnz, std::int64_t cols, int sms);
void tcsr_build_host(std::int64_t rows, const std::int64_t* row_ptr, const std::int64_t* col_ind,
                     const double* val, std::int64_t cols, TcsrHost& out);

struct TcsrOwner {
    DevBuf tile_row0, tile_base, woff, lrow, val, key, ypart, tile_done, tile_pq;
    TcsrDev dev;
    bool valid = false;
    std::int64_t bytes = 0;
    void upload(const TcsrHost& h);
    void release();
    // Rebuild (or drop) the layout for new host arrays under the kernel policy.
    bool refresh(std::int64_t rows, const std::int64_t* row_ptr, const std::int64_t* col_ind, const double* val,
                 std::int64_t cols, bool monotone, std::int64_t max_row, CsrKernel policy);
};

// Merge-path plan owner (merge.cu). Built for monotone row_ptr when rows are
// skewed (max row >= 4096 and > 32x the mean) or when forced.
bool merge_wanted(std::int64_t rows, std::int64_t nnz, std::int64_t max_row, bool monotone, bool forced);

struct MergeOwner {
    DevBuf coord_row, coord_nz, carry_row, carry_val;
    MergeDev dev;
    bool valid = false;
    // row_ptr_host: the caller's array (rows + 1 entries); A: the resident matrix
    bool refresh(const CsrDev& A, const std::int64_t* row_ptr_host, CsrKernel policy);
    void release();
};

// Split plan owner (split.cu). Built from the caller's row_ptr for monotone
// matrices with skewed rows (the merge_wanted test) or when forced.
struct SplitOwner {
    DevBuf long_rows, long_first, chunk_lo, chunk_hi, chunk_row, partial, done, work;
    SplitDev dev;
    bool valid = false;
    bool refresh(const CsrDev& A, const std::int64_t* row_ptr_host, CsrKernel policy);
    void release();
};

// Lane-range layout (lrcsr_build.cpp / lrcsr.cu). Built for monotone row_ptr
// with skewed rows (the merge_wanted test) under Auto, or when forced ("lane").
// Auto: skewed rows (the merge_wanted test), or a large matrix whose gathers
// have locality (locality = gather_locality, <= 0.3: banded / stencil rows),
// where fixed-size units stream better than row-parallel walks.
bool lrc_wanted(std::int64_t rows, std::int64_t nnz, std::int64_t max_row, std::int64_t cols, bool monotone,
                bool forced, double locality);

struct LrcHost {
    std::int64_t units = 0, nnz = 0, rows_c = 0, hot_covered = 0;
    int hot = 0;
    bool has_empty = false;
    std::vector<double> val;
    std::vector<std::uint32_t> col, desc;
    std::vector<std::int32_t> rmap, hot_cols, empty;
};
void lrc_build_host(std::int64_t rows, const std::int64_t* row_ptr, const std::int64_t* col_ind, const double* val,
                    std::int64_t cols, LrcHost& out);

struct LrcOwner {
    DevBuf val, col, desc, rmap, empty, hot_cols, x_hot, carry, fix;
    LrcDev dev;
    bool valid = false;
    std::int64_t bytes = 0, hot_covered = 0;
    void release();
    // A: the resident CSR (device row_ptr / col / val, as uploaded); row_ptr /
    // col_ind: the caller's host arrays (for the policy tests). Built on the device.
    bool refresh(const CsrDev& A, const std::int64_t* row_ptr, const std::int64_t* col_ind, CsrKernel policy);
};

// The same layout built on the device from a resident CSR (row_ptr int64,
// col int32 or int64, val f64; nnz = row_ptr[rows] - row_ptr[0], columns
// rebased to row_ptr[0]): the hot set by a device histogram + radix sort with
// the host builder's tie order, so both builders produce identical arrays.
void lrc_build_device(std::int64_t rows, const std::int64_t* row_ptr, const void* col, bool col32, const double* val,
                      std::int64_t nnz, std::int64_t cols, LrcOwner& out, cudaStream_t s);
int lrc_hot_cap();

}  // namespace b200
