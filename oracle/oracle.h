/*
 * oracle.h — CPU restatement of the LiLAC harness path. TEST INFRASTRUCTURE ONLY.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
 * reference legs may load this library, and only as the checker or the timed
 * CPU baseline. The product path (paper_2001_07938_b200/) never links it.
 *
 * Parity status: PINNED. Every function below that restates reference
 * semantics is checked bit-for-bit against the tests/golden JSON fixtures, which were
 * produced by the reference itself (oracle/_ref, built from
 * /root/reference/proj/src by oracle/Makefile; see tests/golden/README.md).
 * The exceptions are marked "unpinned" (axpy: not a reference computation;
 * NPB makea/CG: external benchmark, pinned instead by NPB's official zeta).
 */
#ifndef LILAC_ORACLE_H
#define LILAC_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- reference computations (what_interp.cpp:87-108 via kernels.lilac) ---- */

/* spmv_csr, kernels.lilac:1-4: output[i] = dot(row_ptr[i] <= j < row_ptr[i+1]) val[j]*x[col_ind[j]].
 * Returns 0, or -1 on an index the reference would reject with OutOfBounds
 * (what_interp.cpp:52-53, 67-68); `nnz`/`ncols` are the array extents. */
int orc_spmv_csr(int64_t rows, double* output, const int64_t* row_ptr, const double* val,
                 const double* x, const int64_t* col_ind, int64_t nnz, int64_t ncols);

/* spmv_jds, kernels.lilac:9-12 (perm maps original row -> jagged position). */
int orc_spmv_jds(int64_t rows, double* output, const int64_t* nzcnt, const int64_t* perm,
                 const double* val, const int64_t* jd_ptr, const double* x,
                 const int64_t* col_ind, int64_t nnz, int64_t njd, int64_t ncols);

/* dotproduct, kernels.lilac:6-7; result[0] = sum_{i<length} a[i]*b[i] from +0.0. */
void orc_dot(double* result, int64_t length, const double* a, const double* b);
/* gemm, kernels.lilac:14-19: c[i*m+j] = sum_{k<p} a[i*p+k]*b[k*m+j] from +0.0, k ascending. */
void orc_gemm(int64_t n, int64_t m, double* c, int64_t p, const double* a, const double* b);

/* Unpinned CG companion (not expressible in LiLAC-What): y[i] = y[i] + alpha*x[i]. */
void orc_axpy(int64_t n, double* y, double alpha, const double* x);

/* Multi-threaded CSR SpMV (static row split, per-row order unchanged, so the
 * result is bit-identical to orc_spmv_csr for any thread count). */
void orc_spmv_csr_mt(int64_t rows, double* output, const int64_t* row_ptr, const double* val,
                     const double* x, const int64_t* col_ind, int nthreads);

/* Multi-threaded JDS SpMV (original rows split across threads, per-row k order
 * unchanged: bit-identical to orc_spmv_jds). No bounds checks. */
void orc_spmv_jds_mt(int64_t rows, double* output, const int64_t* nzcnt, const int64_t* perm,
                     const double* val, const int64_t* jd_ptr, const double* x, const int64_t* col_ind,
                     int nthreads);

/* ---- format encoders (tests/support/oracles.hpp:68-156) ---- */

/* csr_from_dense (oracles.hpp:68-84). Caller sizes val/col_ind for the
 * nonzero count (orc_count_nonzeros). row_ptr has rows+1 entries. */
int64_t orc_count_nonzeros(int64_t rows, int64_t cols, const double* a);
void orc_csr_from_dense(int64_t rows, int64_t cols, const double* a, double* val,
                        int64_t* col_ind, int64_t* row_ptr);

/* jds_from_csr: the jds_from_dense contract (oracles.hpp:109-144) applied to a
 * CSR matrix with ascending columns per row — rows stable-sorted by nonzero
 * count descending, perm[orig]=jagged, diagonals k = 0..max_nz-1.
 * jd_ptr needs max_nz+1 entries (orc_csr_max_row). */
int64_t orc_csr_max_row(int64_t rows, const int64_t* row_ptr);
void orc_jds_from_csr(int64_t rows, const int64_t* row_ptr, const double* csr_val,
                      const int64_t* csr_col, int64_t* perm, int64_t* nzcnt, int64_t* jd_ptr,
                      double* val, int64_t* col_ind);

/* ---- marshal change detection (marshal.cpp:108-116) ---- */
uint64_t orc_fnv1a(const void* data, size_t size);

/* ---- row partition for the sharded driver ----
 * bounds[g] = lower_bound(row_ptr, row_ptr[0] + ceil(g*nnz/k)) clamped to
 * [bounds[g-1], rows]; bounds[0]=0, bounds[k]=rows.  k+1 entries. */
void orc_partition_rows(int64_t rows, const int64_t* row_ptr, int k, int64_t* bounds);

/* ---- NPB CG (external benchmark, restated from the NPB 3.x specification) ---- */

/* NPB randlc: x <- a*x mod 2^46, returns x*2^-46. */
double orc_randlc(double* x, double a);

/* makea for (na, nonzer, shift), rcond = 0.1. First call with val==NULL to
 * get the nonzero count into *nnz_out (row_ptr still filled, na+1 entries);
 * then call again with val/col_ind sized to it. 0-based CSR, ascending
 * columns, duplicates summed in generation order. */
int orc_npb_makea(int64_t na, int nonzer, double shift, int64_t* row_ptr, int64_t* col_ind,
                  double* val, int64_t* nnz_out);

/* Full NPB CG benchmark loop (one untimed warm-up conj_grad, then niter
 * iterations of 25 CG steps) with the scalar restatement above. Returns zeta;
 * *rnorm_out receives the last residual norm. */
double orc_npb_cg(int64_t na, const int64_t* row_ptr, const int64_t* col_ind, const double* val,
                  int niter, double shift, double* rnorm_out);

/* One NPB outer iteration from the caller's x (updated in place to z/|z|):
 * conj_grad with its SpMV on `nthreads` threads (0 = all online CPUs), then
 * zeta = shift + 1/(x.z). Scratch z, p, q, r: n doubles each. The timed
 * native CPU baseline of bench.py. */
double orc_npb_outer(int64_t n, const int64_t* row_ptr, const int64_t* col_ind, const double* val, double* x,
                     double* z, double* p, double* q, double* r, double shift, int nthreads, double* rnorm_out);

#ifdef __cplusplus
}
#endif

#endif
