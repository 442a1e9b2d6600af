// merge.cu — merge-path CSR SpMV for skewed row lengths (power-law graphs).
//
// The merge of the row-end list (row_ptr[1..rows]) with the nonzero indices
// (0..nnz-1) is cut into equal shares of kMergeItems items per CTA, so every
// CTA does the same work whatever the row lengths (a 160K-nonzero row of the
// Kronecker scale-22 graph spreads over ~80 CTAs; the vector kernel gives it
// one warp and takes 11 ms). Per CTA:
//   1. stage the CTA's row ends and its nonzero products val*x[col] in smem
//      (coalesced val/col loads);
//   2. each thread walks kMergeIpt consecutive merge items from its own
//      diagonal (binary search in smem), summing products in order and
//      emitting every row that ends inside its range;
//   3. a block-wide segmented scan carries partial sums across threads;
//   4. the CTA's trailing partial row goes to a carry slot, and
//      k_merge_fixup adds carries to their rows in CTA order.
// Every sum is taken in a fixed order: deterministic run to run.
// CTA start coordinates are a cached invariant of row_ptr (merge_plan).

#include "b200.hpp"
#include "ldst.cuh"

#include <algorithm>

namespace b200 {

namespace {

constexpr int kMergeThreads = 256;
constexpr int kMergeIpt = 8;
constexpr int kMergeItems = kMergeThreads * kMergeIpt;

// Threads walk smem at a stride of ~kMergeIpt words: skew the layout by one
// word every 16 so neighbouring lanes land in different banks.
__device__ __forceinline__ int skew(int i) { return i + (i >> 4); }
constexpr int kSkewed = kMergeItems + kMergeItems / 16 + 2;

// Merge-path diagonal search: the split (i rows ended, j nonzeros consumed)
// of diagonal d, with row i's end at row_end(i). Rows end "before" the
// nonzero with the same index (row_end(i) <= j consumes the row end first).
template <typename RowEnd>
__device__ __forceinline__ std::int64_t merge_search(std::int64_t d, std::int64_t rows, std::int64_t nnz,
                                                     RowEnd row_end) {
    std::int64_t lo = d > nnz ? d - nnz : 0, hi = d < rows ? d : rows;
    while (lo < hi) {
        const std::int64_t pivot = (lo + hi) >> 1;
        if (row_end(pivot) <= d - pivot - 1)
            lo = pivot + 1;
        else
            hi = pivot;
    }
    return lo;  // rows ended before diagonal d
}

__global__ void k_merge_plan(const std::int64_t* __restrict__ row_ptr, std::int64_t rows, std::int64_t nnz,
                             std::int64_t nctas, std::int64_t* __restrict__ coord_row,
                             std::int64_t* __restrict__ coord_nz) {
    const std::int64_t c = static_cast<std::int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (c > nctas) return;
    const std::int64_t base = row_ptr[0];
    const std::int64_t d = min(c * kMergeItems, rows + nnz);
    const std::int64_t i = merge_search(d, rows, nnz, [&](std::int64_t r) { return row_ptr[r + 1] - base; });
    coord_row[c] = i;
    coord_nz[c] = d - i;
}

template <typename IdxT>
__global__ void __launch_bounds__(kMergeThreads)
    k_spmv_merge(std::int64_t rows, const std::int64_t* __restrict__ row_ptr, const IdxT* __restrict__ col,
                 const double* __restrict__ val, const double* __restrict__ x, double* __restrict__ y,
                 const std::int64_t* __restrict__ coord_row, const std::int64_t* __restrict__ coord_nz,
                 std::int64_t* __restrict__ carry_row, double* __restrict__ carry_val) {
    __shared__ std::int64_t s_end[kSkewed];  // relative nonzero index where each row of the CTA ends (skewed)
    __shared__ double s_prod[kSkewed];      // products val*x[col] (skewed)
    __shared__ double s_carry[kMergeThreads];
    const int tid = threadIdx.x;
    const std::int64_t c = blockIdx.x;
    const std::int64_t r0 = coord_row[c], k0 = coord_nz[c];
    const std::int64_t r1 = coord_row[c + 1], k1 = coord_nz[c + 1];
    const int nr = static_cast<int>(r1 - r0), nz = static_cast<int>(k1 - k0);
    const std::int64_t base = row_ptr[0];

    for (int i = tid; i < nr; i += kMergeThreads) s_end[skew(i)] = row_ptr[r0 + i + 1] - base - k0;
    if (tid == 0) s_end[skew(nr)] = INT64_MAX;  // the row still open at the CTA end never ends here
    {
        // products, all loads of a thread issued before any is consumed (MLP)
        const std::int64_t kb = base + k0;
        const std::uint64_t pstream = policy_evict_first(), pgather = policy_evict_last();
        std::int64_t cc[kMergeIpt];
        double vv[kMergeIpt], xx[kMergeIpt];
#pragma unroll
        for (int u = 0; u < kMergeIpt; ++u) {
            const int i = tid + u * kMergeThreads;
            cc[u] = i < nz ? ld_stream_idx(col + kb + i, pstream) : 0;
            vv[u] = i < nz ? ld_stream_f64(val + kb + i, pstream) : 0.0;
        }
#pragma unroll
        for (int u = 0; u < kMergeIpt; ++u) {
            const int i = tid + u * kMergeThreads;
            xx[u] = i < nz ? ld_gather_f64(x + cc[u], pgather) : 0.0;
        }
#pragma unroll
        for (int u = 0; u < kMergeIpt; ++u) {
            const int i = tid + u * kMergeThreads;
            if (i < nz) s_prod[skew(i)] = vv[u] * xx[u];
        }
    }
    __syncthreads();

    // this thread's merge items [d0, d0 + kMergeIpt) of the CTA's nr + nz
    const int d0 = min(tid * kMergeIpt, nr + nz);
    int i = static_cast<int>(merge_search(d0, nr, nz, [&](std::int64_t r) { return s_end[skew(static_cast<int>(r))]; }));
    int j = d0 - i;
    double acc = 0.0, head = 0.0;
    bool ended = false;
    int head_row = -1;
    for (int it = 0; it < kMergeIpt && i + j < nr + nz; ++it) {
        if (s_end[skew(i)] <= j) {  // row r0+i ends here
            if (!ended) {
                ended = true;
                head_row = i;
                head = acc;  // may continue a row begun by an earlier thread
            } else {
                y[r0 + i] = acc;  // row entirely inside this thread's items
            }
            acc = 0.0;
            ++i;
        } else {
            acc += s_prod[skew(j)];
            ++j;
        }
    }
    // segmented inclusive scan of trailing partials (reset where a row
    // ended): shuffles inside each warp, then across the 8 warp totals
    const int lane = tid & 31, warp = tid >> 5;
    double v = acc;
    int f = ended ? 1 : 0;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
        const double ov = __shfl_up_sync(0xffffffffu, v, off);
        const int of = __shfl_up_sync(0xffffffffu, f, off);
        if (lane >= off && !f) {
            v += ov;
            f = of;
        }
    }
    __shared__ double s_wv[kMergeThreads / 32];
    __shared__ int s_wf[kMergeThreads / 32];
    if (lane == 31) {
        s_wv[warp] = v;
        s_wf[warp] = f;
    }
    __syncthreads();
    if (warp == 0) {  // scan of the warp totals (8 entries), same segmented rule
        double wv = lane < kMergeThreads / 32 ? s_wv[lane] : 0.0;
        int wf = lane < kMergeThreads / 32 ? s_wf[lane] : 0;
#pragma unroll
        for (int off = 1; off < kMergeThreads / 32; off <<= 1) {
            const double ov = __shfl_up_sync(0xffffffffu, wv, off);
            const int of = __shfl_up_sync(0xffffffffu, wf, off);
            if (lane >= off && !wf) {
                wv += ov;
                wf = of;
            }
        }
        if (lane < kMergeThreads / 32) s_wv[lane] = wv;
    }
    __syncthreads();
    // add the carry of earlier warps to lanes whose segment reaches back to lane 0
    if (warp > 0 && !f) v += s_wv[warp - 1];
    s_carry[tid] = v;
    __syncthreads();
    // s_carry[t] = this thread's trailing partial plus earlier partials of the
    // same row; the carry into thread t is s_carry[t-1]
    const double carry_in = tid > 0 ? s_carry[tid - 1] : 0.0;
    if (ended) y[r0 + head_row] = carry_in + head;
    if (tid == kMergeThreads - 1) {
        // partial of the row still open at the CTA end (added by k_merge_fixup)
        carry_row[c] = r1;
        carry_val[c] = s_carry[tid];
    }
}

// Adds CTA carries to their rows: the first CTA of each run of equal carry
// rows sums the run in CTA order. Rows >= rows (past the end) are skipped.
__global__ void k_merge_fixup(std::int64_t rows, std::int64_t nctas, const std::int64_t* __restrict__ carry_row,
                              const double* __restrict__ carry_val, double* __restrict__ y) {
    const std::int64_t c = static_cast<std::int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (c >= nctas) return;
    const std::int64_t r = carry_row[c];
    if (r >= rows || (c > 0 && carry_row[c - 1] == r)) return;
    double s = 0.0;
    for (std::int64_t e = c; e < nctas && carry_row[e] == r; ++e) s += carry_val[e];
    y[r] += s;
}

}  // namespace

std::int64_t merge_ctas(std::int64_t rows, std::int64_t nnz) {
    return (rows + nnz + kMergeItems - 1) / kMergeItems;
}

void launch_merge_plan(const std::int64_t* row_ptr, std::int64_t rows, std::int64_t nnz, std::int64_t* coord_row,
                       std::int64_t* coord_nz, cudaStream_t s) {
    const std::int64_t n = merge_ctas(rows, nnz);
    k_merge_plan<<<static_cast<unsigned>((n + 1 + 255) / 256), 256, 0, s>>>(row_ptr, rows, nnz, n, coord_row,
                                                                          coord_nz);
    B200_CUDA(cudaGetLastError());
}

void launch_spmv_merge(const CsrDev& A, const double* x, double* y, cudaStream_t s) {
    const MergeDev& M = *A.merge;
    if (A.rows <= 0) return;
    if (M.nctas > 0) {
        if (A.col32)
            k_spmv_merge<std::int32_t><<<static_cast<unsigned>(M.nctas), kMergeThreads, 0, s>>>(
                A.rows, A.row_ptr, static_cast<const std::int32_t*>(A.col), A.val, x, y, M.coord_row, M.coord_nz,
                M.carry_row, M.carry_val);
        else
            k_spmv_merge<std::int64_t><<<static_cast<unsigned>(M.nctas), kMergeThreads, 0, s>>>(
                A.rows, A.row_ptr, static_cast<const std::int64_t*>(A.col), A.val, x, y, M.coord_row, M.coord_nz,
                M.carry_row, M.carry_val);
        k_merge_fixup<<<static_cast<unsigned>((M.nctas + 255) / 256), 256, 0, s>>>(A.rows, M.nctas, M.carry_row,
                                                                                   M.carry_val, y);
    }
    B200_CUDA(cudaGetLastError());
}

}  // namespace b200
