// workloads_dev.cu — device-side workload pieces for the BASELINE configs
// (SURVEY §8(d) inputs 4 and 5): the 27-point stencil matrix generated in HBM
// (N = 420 is 2.0e9 nonzeros: generating it on the host and uploading would
// dominate the run), and the PageRank update x = d*(A x) + (1-d)/n.

#include "b200.hpp"

#include <cub/device/device_scan.cuh>

namespace b200 {

namespace {

constexpr int kGenThreads = 256;

__device__ __forceinline__ int span(std::int64_t i, std::int64_t nx) {
    return (i > 0) + 1 + (i < nx - 1);  // neighbours along one axis (incl. itself)
}

__global__ void k_stencil_lengths(std::int64_t nx, std::int64_t r0, std::int64_t rows, std::int64_t* __restrict__ len) {
    const std::int64_t stride = static_cast<std::int64_t>(gridDim.x) * blockDim.x;
    for (std::int64_t t = static_cast<std::int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; t < rows; t += stride) {
        const std::int64_t r = r0 + t;
        const std::int64_t i = r / (nx * nx), j = (r / nx) % nx, k = r % nx;
        len[t] = span(i, nx) * span(j, nx) * span(k, nx);
    }
}

// Row r's neighbours in increasing linear index (di, dj, dk lexicographic),
// value `diag` on the diagonal and `off` elsewhere — the same arrays as the
// host generator tools/bench_configs.py:gen_stencil27.
__global__ void k_stencil_fill(std::int64_t nx, std::int64_t r0, std::int64_t rows,
                               const std::int64_t* __restrict__ row_ptr, std::int32_t* __restrict__ col,
                               double* __restrict__ val, double diag, double off) {
    const std::int64_t stride = static_cast<std::int64_t>(gridDim.x) * blockDim.x;
    for (std::int64_t t = static_cast<std::int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; t < rows; t += stride) {
        const std::int64_t r = r0 + t;
        const std::int64_t i = r / (nx * nx), j = (r / nx) % nx, k = r % nx;
        std::int64_t p = row_ptr[t];
        for (int di = -1; di <= 1; ++di) {
            if (i + di < 0 || i + di >= nx) continue;
            for (int dj = -1; dj <= 1; ++dj) {
                if (j + dj < 0 || j + dj >= nx) continue;
                for (int dk = -1; dk <= 1; ++dk) {
                    if (k + dk < 0 || k + dk >= nx) continue;
                    const std::int64_t c = r + di * nx * nx + dj * nx + dk;
                    col[p] = static_cast<std::int32_t>(c);
                    val[p] = (c == r) ? diag : off;
                    ++p;
                }
            }
        }
    }
}

__global__ void k_pagerank_update(std::int64_t n, double* __restrict__ x, const double* __restrict__ ax, double d,
                                  double teleport) {
    const std::int64_t stride = static_cast<std::int64_t>(gridDim.x) * blockDim.x;
    for (std::int64_t i = static_cast<std::int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride)
        x[i] = __dadd_rn(__dmul_rn(d, ax[i]), teleport);
}

unsigned grid(std::int64_t n) {
    return static_cast<unsigned>(std::max<std::int64_t>(1, std::min<std::int64_t>((n + kGenThreads - 1) / kGenThreads,
                                                                               148 * 32)));
}

}  // namespace

std::int64_t stencil27_nnz(std::int64_t nx) {
    const std::int64_t a = nx >= 2 ? 3 * nx - 2 : nx;  // sum over one axis of span()
    return a * a * a;
}

// Nonzeros of stencil rows [0, r): sum over rows of span(i) span(j) span(k)
// (exact integer arithmetic, O(nx) per call).
std::int64_t stencil27_prefix_nnz(std::int64_t nx, std::int64_t r) {
    auto sp = [nx](std::int64_t v) { return static_cast<std::int64_t>((v > 0) + 1 + (v < nx - 1)); };
    auto axis_sum = [&](std::int64_t m) {  // sum_{v < m} span(v)
        std::int64_t s = 0;
        for (std::int64_t v = 0; v < m; ++v) s += sp(v);
        return s;
    };
    const std::int64_t A = axis_sum(nx);  // 3nx - 2
    const std::int64_t i = r / (nx * nx), j = (r / nx) % nx, k = r % nx;
    // full i-planes, then full j-lines of plane i, then k entries of line (i, j)
    return axis_sum(i) * A * A + sp(i) * axis_sum(j) * A + sp(i) * sp(j) * axis_sum(k);
}

void gen_stencil27_rows_device(std::int64_t nx, std::int64_t r0, std::int64_t r1, double diag, double off,
                               DevBuf& row_ptr, DevBuf& col, DevBuf& val, cudaStream_t s) {
    const std::int64_t rows = r1 - r0;
    const std::int64_t nnz = stencil27_prefix_nnz(nx, r1) - stencil27_prefix_nnz(nx, r0);
    row_ptr.ensure(sizeof(std::int64_t) * static_cast<std::size_t>(rows + 1));
    col.ensure(sizeof(std::int32_t) * static_cast<std::size_t>(std::max<std::int64_t>(nnz, 1)));
    val.ensure(sizeof(double) * static_cast<std::size_t>(std::max<std::int64_t>(nnz, 1)));
    std::int64_t* rp = row_ptr.as<std::int64_t>();
    // lengths into rp[0..rows), zero at rp[rows]; an exclusive scan over
    // rows+1 turns them into the (rebased) row pointers in place (rp[rows] = nnz)
    B200_CUDA(cudaMemsetAsync(rp + rows, 0, sizeof(std::int64_t), s));
    if (rows > 0) {
        k_stencil_lengths<<<grid(rows), kGenThreads, 0, s>>>(nx, r0, rows, rp);
        B200_CUDA(cudaGetLastError());
    }
    std::size_t tmp = 0;
    B200_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tmp, rp, rp, rows + 1, s));
    DevBuf scratch;
    scratch.ensure(tmp);
    B200_CUDA(cub::DeviceScan::ExclusiveSum(scratch.ptr, tmp, rp, rp, rows + 1, s));
    if (rows > 0) {
        k_stencil_fill<<<grid(rows), kGenThreads, 0, s>>>(nx, r0, rows, rp, col.as<std::int32_t>(),
                                                          val.as<double>(), diag, off);
        B200_CUDA(cudaGetLastError());
    }
    B200_CUDA(cudaStreamSynchronize(s));
    scratch.release();
}

void gen_stencil27_device(std::int64_t nx, double diag, double off, DevBuf& row_ptr, DevBuf& col, DevBuf& val,
                          cudaStream_t s) {
    gen_stencil27_rows_device(nx, 0, nx * nx * nx, diag, off, row_ptr, col, val, s);
}

void launch_pagerank_update(std::int64_t n, double* x, const double* ax, double d, cudaStream_t s) {
    if (n <= 0) return;
    k_pagerank_update<<<grid(n), kGenThreads, 0, s>>>(n, x, ax, d, (1.0 - d) / static_cast<double>(n));
    B200_CUDA(cudaGetLastError());
}

}  // namespace b200
