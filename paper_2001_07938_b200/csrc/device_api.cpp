// device_api.cpp — resident-matrix C API (section 4 of include/lilac_b200.h):
// the same uploads/validation/kernels the harness entries use, exposed with
// device pointers for drivers (NPB CG, multi-GPU) and kernel-level benchmarks.

#include "lilac_b200.h"
#include "runtime.hpp"
#include "tcsr.hpp"

#include <algorithm>
#include <climits>
#include <cstdlib>
#include <cstring>
#include <utility>
#include <memory>

using namespace b200;

struct b200_matrix {
    int format = 0;  // 0 CSR, 1 JDS
    int device = -1;
    DevBuf row_ptr, col, val;             // CSR
    DevBuf nzcnt, perm, inv_perm, jd_ptr;  // JDS (+col, val)
    CsrDev csr;
    JdsDev jds;
    TcsrOwner tiled;
    MergeOwner merge;
    SplitOwner split;
    LrcOwner lrc;
    std::int64_t max_row = 0;
};

namespace {

// A derived layout serves the matrix: free the plain col / val (keep_plain_csr).
void drop_plain(b200_matrix& A) {
    CsrDev& d = A.csr;
    if (!(d.tiled || d.lrc) || keep_plain_csr()) return;
    A.col.release();
    A.val.release();
    d.col = nullptr;
    d.val = nullptr;
}

CsrKernel matrix_kernel(const b200_matrix* A) {
    return choose_csr_kernel(A->csr, rt().kernel);
}

}  // namespace

extern "C" {

int b200_matrix_create_csr(b200_matrix** out, std::int64_t rows, const std::int64_t* row_ptr,
                           const std::int64_t* col_ind, const double* val) {
    return boundary("b200_matrix_create_csr", [&] {
        ensure_init();
        if (!out) throw Error(Errc::DataError, "out is NULL");
        if (rows < 0) throw Error(Errc::DataError, "rows < 0");
        auto A = std::make_unique<b200_matrix>();
        A->format = 0;
        A->device = rt().device;
        const std::int64_t nnz = row_ptr[rows];
        if (nnz < 0) throw Error(Errc::OutOfBounds, "row_ptr[rows] < 0");
        bool monotone = true, col32 = true;
        std::int64_t max_row = 0;
        upload_row_ptr(A->row_ptr, row_ptr, rows, nnz, &max_row, &monotone);
        const std::int64_t cols = upload_col_ind(A->col, col_ind, nnz, &col32);
        A->val.ensure(nnz * sizeof(double));
        host_in(val, nnz * sizeof(double));
        if (nnz > 0)
            B200_CUDA(cudaMemcpyAsync(A->val.ptr, val, nnz * sizeof(double), cudaMemcpyHostToDevice, rt().stream));
        B200_CUDA(cudaStreamSynchronize(rt().stream));
        CsrDev& d = A->csr;
        d.rows = rows;
        d.nnz = nnz;
        d.cols = cols;
        d.max_row = max_row;
        d.row_ptr = A->row_ptr.as<std::int64_t>();
        d.col = A->col.ptr;
        d.col32 = col32;
        d.val = A->val.as<double>();
        d.monotone = monotone;
        A->max_row = max_row;
        if (A->tiled.refresh(rows, row_ptr, col_ind, val, cols, monotone, max_row, rt().kernel)) d.tiled = &A->tiled.dev;
        if (!d.tiled && A->lrc.refresh(d, row_ptr, col_ind, rt().kernel))
            d.lrc = &A->lrc.dev;
        if (!d.tiled && !d.lrc && A->split.refresh(d, row_ptr, rt().kernel)) d.split = &A->split.dev;
        if (!d.tiled && !d.lrc && A->merge.refresh(d, row_ptr, rt().kernel)) d.merge = &A->merge.dev;
        drop_plain(*A);
        *out = A.release();
    });
}

int b200_matrix_create_jds(b200_matrix** out, std::int64_t rows, const std::int64_t* nzcnt,
                           const std::int64_t* perm, const double* val, const std::int64_t* jd_ptr,
                           const std::int64_t* col_ind) {
    return boundary("b200_matrix_create_jds", [&] {
        ensure_init();
        if (!out) throw Error(Errc::DataError, "out is NULL");
        if (rows < 0) throw Error(Errc::DataError, "rows < 0");
        Runtime& r = rt();
        auto A = std::make_unique<b200_matrix>();
        A->format = 1;
        A->device = r.device;
        std::int64_t max_nz = 0;
        for (std::int64_t i = 0; i < rows; ++i) max_nz = std::max(max_nz, nzcnt[i]);
        const std::int64_t njd = rows > 0 ? max_nz + 1 : 0;
        const std::int64_t nnz = njd > 0 ? jd_ptr[max_nz] : 0;
        if (nnz < 0) throw Error(Errc::OutOfBounds, "jd_ptr[max_nz] < 0");
        A->nzcnt.ensure(rows * 8);
        A->perm.ensure(rows * 8);
        A->inv_perm.ensure(rows * 8);
        A->jd_ptr.ensure(njd * 8);
        if (rows > 0) {
            host_in(nzcnt, rows * 8);
            host_in(perm, rows * 8);
            host_in(jd_ptr, njd * 8);
            B200_CUDA(cudaMemcpyAsync(A->nzcnt.ptr, nzcnt, rows * 8, cudaMemcpyHostToDevice, r.stream));
            B200_CUDA(cudaMemcpyAsync(A->perm.ptr, perm, rows * 8, cudaMemcpyHostToDevice, r.stream));
            B200_CUDA(cudaMemcpyAsync(A->jd_ptr.ptr, jd_ptr, njd * 8, cudaMemcpyHostToDevice, r.stream));
        }
        B200_CUDA(cudaMemsetAsync(r.flags.ptr, 0, 16, r.stream));
        launch_invert_perm(A->perm.as<std::int64_t>(), rows, A->inv_perm.as<std::int64_t>(), r.d_bad(), r.stream);
        int bad = 0;
        B200_CUDA(cudaMemcpyAsync(&bad, r.d_bad(), 4, cudaMemcpyDeviceToHost, r.stream));
        B200_CUDA(cudaStreamSynchronize(r.stream));
        if (bad & 1) throw Error(Errc::OutOfBounds, "perm entry outside [0, rows)");
        const bool bijective = (bad & 2) == 0;
        B200_CUDA(cudaMemsetAsync(r.flags.ptr, 0, 16, r.stream));
        launch_check_jds(A->nzcnt.as<std::int64_t>(), A->jd_ptr.as<std::int64_t>(), rows, njd, nnz, r.d_bad(),
                         r.stream);
        B200_CUDA(cudaMemcpyAsync(&bad, r.d_bad(), 4, cudaMemcpyDeviceToHost, r.stream));
        B200_CUDA(cudaStreamSynchronize(r.stream));
        if (bad) throw Error(Errc::OutOfBounds, "jd_ptr[k] + perm[i] outside [0, nnz)");
        bool col32 = true;
        const std::int64_t cols = upload_col_ind(A->col, col_ind, nnz, &col32);
        A->val.ensure(nnz * 8);
        host_in(val, nnz * 8);
        if (nnz > 0) B200_CUDA(cudaMemcpyAsync(A->val.ptr, val, nnz * 8, cudaMemcpyHostToDevice, r.stream));
        B200_CUDA(cudaStreamSynchronize(r.stream));
        JdsDev& d = A->jds;
        d.rows = rows;
        d.nnz = nnz;
        d.cols = cols;
        d.njd = njd;
        d.nzcnt = A->nzcnt.as<std::int64_t>();
        d.perm = A->perm.as<std::int64_t>();
        d.inv_perm = bijective ? A->inv_perm.as<std::int64_t>() : nullptr;
        d.jd_ptr = A->jd_ptr.as<std::int64_t>();
        d.col = A->col.ptr;
        d.col32 = col32;
        d.val = A->val.as<double>();
        d.seg = jds_segments(nzcnt, rows);
        A->max_row = max_nz;
        *out = A.release();
    });
}

void b200_matrix_free(b200_matrix* A) {
    if (!A) return;
    // Kernels launched on caller streams (the NULL stream included, which does
    // not order against the library's non-blocking stream) may still read these
    // buffers; the caching pool hands blocks out again on rt().stream, so wait
    // for the device before recycling them.
    device_quiesce();
    A->row_ptr.release();
    A->col.release();
    A->val.release();
    A->nzcnt.release();
    A->perm.release();
    A->inv_perm.release();
    A->jd_ptr.release();
    A->tiled.release();
    A->merge.release();
    A->split.release();
    A->lrc.release();
    delete A;
}

int b200_matrix_info_get(const b200_matrix* A, b200_matrix_info* info) {
    return boundary("b200_matrix_info_get", [&] {
        if (!A || !info) throw Error(Errc::DataError, "NULL argument");
        *info = b200_matrix_info{};
        info->format = A->format;
        info->max_row = A->max_row;
        if (A->format == 0) {
            info->rows = A->csr.rows;
            info->cols = A->csr.cols;
            info->nnz = A->csr.nnz;
            info->kernel = static_cast<int32_t>(matrix_kernel(A));
            // column index width the chosen kernel streams (tiled: 16-bit slab-local keys)
            info->col_bytes = info->kernel == static_cast<int32_t>(CsrKernel::Tiled)  ? 2
                              : info->kernel == static_cast<int32_t>(CsrKernel::Lane) ? 4
                              : (A->csr.col32 ? 4 : 8);
            info->lanes = csr_vector_width(A->csr);
        } else {
            info->rows = A->jds.rows;
            info->cols = A->jds.cols;
            info->nnz = A->jds.nnz;
            info->col_bytes = A->jds.col32 ? 4 : 8;
            info->kernel = jds_segmented(A->jds) ? 1 : 0;
            info->lanes = info->kernel == 1 ? A->jds.seg.g[0] : 1;
        }
        info->device_bytes = static_cast<std::int64_t>(A->row_ptr.bytes + A->col.bytes + A->val.bytes + A->nzcnt.bytes +
                                                       A->perm.bytes + A->inv_perm.bytes + A->jd_ptr.bytes) +
                             A->tiled.bytes + A->lrc.bytes;
    });
}

int b200_matrix_create_stencil27(b200_matrix** out, std::int64_t nx, double diag, double offdiag) {
    return boundary("b200_matrix_create_stencil27", [&] {
        ensure_init();
        if (!out) throw Error(Errc::DataError, "out is NULL");
        if (nx < 1) throw Error(Errc::DataError, "nx < 1");
        const std::int64_t n = nx * nx * nx;
        if (n - 1 > INT32_MAX) throw Error(Errc::DataError, "nx^3 exceeds int32 column indices");
        auto A = std::make_unique<b200_matrix>();
        A->format = 0;
        A->device = rt().device;
        gen_stencil27_device(nx, diag, offdiag, A->row_ptr, A->col, A->val, rt().stream);
        CsrDev& d = A->csr;
        d.rows = n;
        d.nnz = stencil27_nnz(nx);
        d.cols = n;
        d.max_row = std::min<std::int64_t>(27, n);
        d.row_ptr = A->row_ptr.as<std::int64_t>();
        d.col = A->col.ptr;
        d.col32 = true;
        d.val = A->val.as<double>();
        d.monotone = true;
        A->max_row = d.max_row;
        // the lane-range layout streams banded rows at ~0.9 of copy (the
        // row-parallel kernel ~0.75); built on the device from the generated CSR
        const CsrKernel pol = rt().kernel;
        if ((pol == CsrKernel::Auto && d.nnz >= (std::int64_t(16) << 20)) || pol == CsrKernel::Lane) {
            lrc_build_device(n, d.row_ptr, d.col, true, d.val, d.nnz, n, A->lrc, rt().stream);
            d.lrc = &A->lrc.dev;
        }
        drop_plain(*A);
        *out = A.release();
    });
}

int b200_matrix_create_stencil27_rows(b200_matrix** out, std::int64_t nx, std::int64_t r0, std::int64_t r1,
                                      double diag, double offdiag) {
    return boundary("b200_matrix_create_stencil27_rows", [&] {
        ensure_init();
        if (!out) throw Error(Errc::DataError, "out is NULL");
        const std::int64_t n = nx * nx * nx;
        if (nx < 1 || n - 1 > INT32_MAX) throw Error(Errc::DataError, "nx must give int32 column indices");
        if (r0 < 0 || r1 < r0 || r1 > n) throw Error(Errc::DataError, "row range outside [0, nx^3]");
        auto A = std::make_unique<b200_matrix>();
        A->format = 0;
        A->device = rt().device;
        gen_stencil27_rows_device(nx, r0, r1, diag, offdiag, A->row_ptr, A->col, A->val, rt().stream);
        CsrDev& d = A->csr;
        d.rows = r1 - r0;
        d.nnz = stencil27_prefix_nnz(nx, r1) - stencil27_prefix_nnz(nx, r0);
        d.cols = n;  // global columns: the block reads the full x
        d.max_row = d.rows ? std::min<std::int64_t>(27, n) : 0;
        d.row_ptr = A->row_ptr.as<std::int64_t>();
        d.col = A->col.ptr;
        d.col32 = true;
        d.val = A->val.as<double>();
        d.monotone = true;
        A->max_row = d.max_row;
        const CsrKernel pol = rt().kernel;
        if (d.rows && ((pol == CsrKernel::Auto && d.nnz >= (std::int64_t(16) << 20)) || pol == CsrKernel::Lane)) {
            lrc_build_device(d.rows, d.row_ptr, d.col, true, d.val, d.nnz, n, A->lrc, rt().stream);
            d.lrc = &A->lrc.dev;
        }
        drop_plain(*A);
        *out = A.release();
    });
}

// LILAC_B200_PAGERANK_FUSED=0: SpMV + update kernels (experiments)
static bool fused_pagerank() {
    static const bool on = [] {
        const char* e = std::getenv("LILAC_B200_PAGERANK_FUSED");
        return !(e && std::strcmp(e, "0") == 0);
    }();
    return on;
}

int b200_pagerank_device(const b200_matrix* A, double damping, int iters, double* x, double* work, void* stream) {
    return boundary("b200_pagerank_device", [&] {
        if (!A || A->format != 0) throw Error(Errc::DataError, "PageRank needs a CSR matrix");
        if (A->csr.rows != A->csr.cols && A->csr.cols > A->csr.rows)
            throw Error(Errc::DataError, "PageRank needs a square operator");
        cudaStream_t s = static_cast<cudaStream_t>(stream);
        // the lane-range layout folds the update into its row stores: the
        // iterate ping-pongs between x and work (one pass per step instead of
        // SpMV + update), copied back into x after an odd number of steps
        const bool fused = A->csr.lrc && iters > 0 && A->csr.lrc->units > 0 && fused_pagerank();
        double* cur = x;
        double* nxt = work;
        for (int it = 0; it < iters; ++it) {
            if (fused && launch_pagerank_lrc(*A->csr.lrc, A->csr.rows, cur, nxt, damping, s)) {
                std::swap(cur, nxt);
                continue;
            }
            if (cur != x) {  // (not reached: a layout either fuses every step or none)
                B200_CUDA(cudaMemcpyAsync(x, cur, sizeof(double) * static_cast<std::size_t>(A->csr.rows),
                                          cudaMemcpyDeviceToDevice, s));
                cur = x;
                nxt = work;
            }
            launch_spmv_csr(A->csr, x, work, rt().kernel, s);
            launch_pagerank_update(A->csr.rows, x, work, damping, s);
        }
        if (cur != x)
            B200_CUDA(cudaMemcpyAsync(x, cur, sizeof(double) * static_cast<std::size_t>(A->csr.rows),
                                      cudaMemcpyDeviceToDevice, s));
    });
}

int b200_pagerank_step_device(const b200_matrix* A, double damping, const double* x, double* y, void* stream) {
    return boundary("b200_pagerank_step_device", [&] {
        if (!A || A->format != 0) throw Error(Errc::DataError, "PageRank needs a CSR matrix");
        if (A->csr.rows != A->csr.cols && A->csr.cols > A->csr.rows)
            throw Error(Errc::DataError, "PageRank needs a square operator");
        if (x == y) throw Error(Errc::DataError, "PageRank step: y must not alias x");
        cudaStream_t s = static_cast<cudaStream_t>(stream);
        if (A->csr.lrc && fused_pagerank() && launch_pagerank_lrc(*A->csr.lrc, A->csr.rows, x, y, damping, s)) return;
        launch_spmv_csr(A->csr, x, y, rt().kernel, s);
        launch_pagerank_update(A->csr.rows, y, y, damping, s);  // elementwise in place
    });
}

int b200_spmv_device(const b200_matrix* A, const double* x, double* y, void* stream) {
    return boundary("b200_spmv_device", [&] {
        if (!A) throw Error(Errc::DataError, "NULL matrix");
        cudaStream_t s = static_cast<cudaStream_t>(stream);
        if (A->format == 0)
            launch_spmv_csr(A->csr, x, y, rt().kernel, s);
        else
            launch_spmv_jds(A->jds, x, y, s);
    });
}

int b200_dot_device(const double* a, const double* b, std::int64_t n, double* result, void* stream) {
    return boundary("b200_dot_device", [&] {
        ensure_init();
        Runtime& r = rt();
        cudaStream_t s = static_cast<cudaStream_t>(stream);
        if (r.exact_blas)
            launch_dot_exact(a, b, n, result, s);
        else
            launch_dot(a, b, n, result, r.partials.as<double>(), r.d_ticket(), s);
    });
}

int b200_gemm_device(std::int64_t n, std::int64_t m, std::int64_t p, const double* a, const double* b, double* c,
                     int exact, void* stream) {
    return boundary("b200_gemm_device", [&] {
        ensure_init();
        if (n < 0 || m < 0 || p < 0) throw Error(Errc::DataError, "negative gemm extent");
        launch_gemm(n, m, p, a, b, c, exact != 0, static_cast<cudaStream_t>(stream));
    });
}

int b200_axpy_device(std::int64_t n, double* y, double alpha, const double* x, void* stream) {
    return boundary("b200_axpy_device", [&] { launch_axpy(n, y, alpha, x, static_cast<cudaStream_t>(stream)); });
}

int b200_dbuf_alloc(B200Buf* b, std::size_t bytes) {
    return boundary("b200_dbuf_alloc", [&] {
        ensure_init();
        b->ptr = nullptr;
        b->bytes = bytes;
        B200_CUDA(cudaMalloc(&b->ptr, bytes + kPadBytes));
    });
}

int b200_dbuf_upload(B200Buf* b, const void* host, std::size_t bytes) {
    return boundary("b200_dbuf_upload", [&] {
        ensure_init();
        if (!b->ptr || b->bytes < bytes) {
            if (b->ptr) cudaFree(b->ptr);
            b->ptr = nullptr;
            B200_CUDA(cudaMalloc(&b->ptr, bytes + kPadBytes));
            b->bytes = bytes;
        }
        host_in(host, bytes);
        if (bytes) B200_CUDA(cudaMemcpy(b->ptr, host, bytes, cudaMemcpyHostToDevice));
    });
}

int b200_dbuf_download(void* host, const B200Buf* b, std::size_t bytes) {
    return boundary("b200_dbuf_download", [&] {
        // A DMA write into caller memory: any lazy write-back range under the
        // destination is superseded (its device bytes must never be filled over
        // the new ones), device mirrors of it are stale, and guards are dirtied.
        lilac::marshal::supersede_range(host, bytes);
        mirrors_forget(host, bytes);
        lilac::marshal::note_host_write(host, bytes);
        if (bytes) B200_CUDA(cudaMemcpy(host, b->ptr, bytes, cudaMemcpyDeviceToHost));
    });
}

void b200_dbuf_free(B200Buf* b) {
    if (b && b->ptr) cudaFree(b->ptr);
    if (b) {
        b->ptr = nullptr;
        b->bytes = 0;
    }
}

int b200_spmv_csr_dev(std::int64_t rows, std::int64_t nnz, std::int64_t cols, const void* row_ptr,
                      const void* col_ind, const void* val, const void* x, void* y) {
    return boundary("b200_spmv_csr_dev", [&] {
        ensure_init();
        CsrDev A;
        A.rows = rows;
        A.nnz = nnz;
        A.cols = cols;
        A.row_ptr = static_cast<const std::int64_t*>(row_ptr);
        A.col = col_ind;
        A.col32 = false;  // ABI width, as the spec marshals it
        A.val = static_cast<const double*>(val);
        launch_spmv_csr(A, static_cast<const double*>(x), static_cast<double*>(y), CsrKernel::Vector, rt().stream);
        B200_CUDA(cudaStreamSynchronize(rt().stream));
    });
}

}  // extern "C"

// exposed for cg.cpp
namespace b200 {
const CsrDev* matrix_csr(const b200_matrix* A) { return A && A->format == 0 ? &A->csr : nullptr; }
}  // namespace b200
