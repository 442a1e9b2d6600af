/*
 * lilac_b200.h — C ABI of the B200 backend for the LiLAC-How harness path.
 *
 * Shared library: paper_2001_07938_b200/liblilac_b200.so (sm_100a kernels +
 * C++ marshaling runtime). Plain C types only; all pointers are HOST pointers
 * unless the name says _device.
 *
 * Drop-in contract (reference, /root/reference/proj):
 *   - Every harness entry point has the signature harnessgen emits for its
 *     computation: `extern "C" void <HARNESS>(<params in infer_interface order>)`
 *     with kinds mapped ScalarInt -> int64_t, ArrayInt -> const int64_t*,
 *     ArrayFloatIn -> const double*, ArrayFloatOut -> double*
 *     (src/harnessgen.cpp:10-18, 86-92; src/what_parse.cpp:356-429).
 *     "All harness interfaces for the same WhatProgram share the signature"
 *     (SPEC.md:509), so linking this library instead of another harness
 *     library is sufficient.
 *   - No init/fini calls are required: the first call initialises the device
 *     and registers an atexit teardown that releases every marshal object
 *     (harnessgen.cpp:98-113; golden fixtures/gen/cusparse_spmv.gen.cpp:96-110).
 *   - Errors: the reference lets lilac::Error escape (marshal.hpp:172-179); a C
 *     caller sees std::terminate. Here every entry point catches at the
 *     boundary, records the message (b200_last_error) and, in the default
 *     error mode, prints `lilac-b200: <Code>: <message>` and aborts. In
 *     B200_ERRORS_RETURN mode the call returns with outputs untouched. There is
 *     never a CPU fallback.
 */
#ifndef LILAC_B200_H
#define LILAC_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ==========================================================================
 * 1. Harness entry points (drop-in for the reference's harness symbols)
 * ========================================================================== */

/* spmv_csr (fixtures/lilac/kernels.lilac:1-4; reference harness
 * interp.cpp:330-389 "lilac.spmv_csr"; generated shape cusparse_spmv.gen.cpp:93).
 * output[i] = sum_{row_ptr[i] <= j < row_ptr[i+1]} val[j] * x[col_ind[j]], i < rows.
 * Extents follow the reference spec's marshaling section (cusparse.lilac:52-61):
 * nnz = row_ptr[rows] (LastEntry), cols = 1 + max(col_ind[0..nnz)) (ReadableMax),
 * x[0..cols), output[0..rows). row_ptr/col_ind/val stay resident on the device
 * across calls while unchanged; only x and output move per call. */
void b200_spmv_csr(int64_t rows, double* output, const int64_t* row_ptr, const double* val,
                   const double* x, const int64_t* col_ind);

/* spmv_jds (kernels.lilac:9-12; "lilac.spmv_jds"):
 * output[i] = sum_{k < nzcnt[perm[i]]} val[jd_ptr[k]+perm[i]] * x[col_ind[jd_ptr[k]+perm[i]]].
 * Extents: max_nz = max(nzcnt), jd_ptr[0..max_nz], nnz = jd_ptr[max_nz],
 * cols = 1 + max(col_ind[0..nnz)). Bit-identical to the reference. */
void b200_spmv_jds(int64_t rows, double* output, const int64_t* nzcnt, const int64_t* perm,
                   const double* val, const int64_t* jd_ptr, const double* x,
                   const int64_t* col_ind);

/* dotproduct (kernels.lilac:6-7; "lilac.dotproduct"; C shape pinned by
 * test_harnessgen.cpp:107-108): result[0] = sum_{i<length} a[i]*b[i]. */
void b200_dot(double* result, int64_t length, const double* a, const double* b);

/* CG companions the reference cannot express in LiLAC-What (
 * extension kinds, same conventions):
 *   b200_axpy: y[i] = y[i] + alpha * x[i]
 *   b200_xpay: y[i] = x[i] + beta * y[i]      (NPB CG's p = r + beta*p)  */
/* gemm (kernels.lilac:14-19; "lilac.gemm"; infer_interface order n, m, c, p,
 * a, b): c[i*m + j] = sum_{k<p} a[i*p + k] * b[k*m + j], row-major f64.
 * b200_set_exact_blas(1): one thread per output in the reference's k order
 * (bit-identical); else the FP64 tensor-core (DMMA) kernel (tolerance). */
void b200_gemm(int64_t n, int64_t m, double* c, int64_t p, const double* a, const double* b);
void b200_axpy(int64_t n, double* y, double alpha, const double* x);
void b200_xpay(int64_t n, double* y, double beta, const double* x);

/* ==========================================================================
 * 2. Runtime control
 * ========================================================================== */

#define B200_ERRORS_ABORT 0
#define B200_ERRORS_RETURN 1

/* Optional explicit init on a device (default: LILAC_B200_DEVICE or the current
 * CUDA device). Returns 0 or -1 (see b200_last_error). */
int b200_init(int device);
/* Release every marshal object and device buffer now (also runs at exit). */
void b200_shutdown(void);
void b200_set_error_mode(int mode);
const char* b200_last_error(void);
/* Last error code name ("OutOfBounds", "HookFailure", "DataError",
 * "DeviceError", ...) or "" when the last call succeeded. */
const char* b200_last_error_code(void);
/* CSR kernel policy, applied at the next matrix upload: "auto" (tiled for
 * poor x locality, split for skewed rows, else vector) | "vector" | "tiled" |
 * "split" | "merge" | "exact" (bit-identical to the reference). Also
 * LILAC_B200_KERNEL.
 * Returns 0 or -1. */
int b200_set_kernel(const char* name);
/* Change-detection strategy for harness objects created afterwards:
 * "hybrid" (default) | "pageprotect" | "checksum" | "naive" (LILAC_MARSHAL_STRATEGY). */
int b200_set_strategy(const char* name);
/* 1 = dot/axpy also use the reference's sequential order (bit-exact). */
void b200_set_exact_blas(int on);
/* Output write-back mode. "eager" (default; the reference's
 * behaviour, gen.cpp:112-118): every OUTPUT binding is copied device->host
 * before the call returns. "lazy": a page-aligned output of >= 8 KiB stays on
 * the device; its host pages are mapped PROT_NONE and filled on first CPU
 * touch (page fault) or by b200_host_sync, and a later harness input over the
 * same bytes is served device-to-device. The call returns without a host
 * sync. Caveat: DMA and system calls do not fault — call b200_host_sync
 * before handing such a buffer to another library or to read()/write().
 * Also LILAC_B200_WRITEBACK=lazy. */
int b200_set_writeback(const char* mode);
/* Per-call profiling (host phase timers, kernel time via CUDA events in the
 * harness stats). Off by default: it costs clock reads and two event records
 * per call. Also LILAC_B200_PROFILE=1. */
void b200_set_profiling(int on);
/* Materialise lazy write-back bytes in [host, host+bytes) (NULL: all). */
int b200_host_sync(const void* host, size_t bytes);
/* A write that does not fault is about to land in [host, host+bytes) — a
 * system call (read(), recv(), fread() into the buffer) or another library's
 * DMA — into an array the harness has seen: lazy bytes there are filled, the
 * change-detection guards over it are lifted (a guarded page would make the
 * system call fail with EFAULT) and its regions are marked changed, so the
 * next call re-marshals them; device mirrors of the range are dropped. */
int b200_host_will_write(void* host, size_t bytes);
/* The caller is about to free (or hand to an allocator) [host, host+bytes):
 * drop every binding, device mirror, page guard and lazy range over it,
 * without filling (NULL: everything). Guards and lazy pages must not outlive
 * the memory they describe: a recycled buffer would otherwise be served stale
 * device bytes or receive an old lazy fill. Call b200_host_sync first to
 * keep the lazy bytes. */
int b200_host_forget(const void* host, size_t bytes);
/* Lazy write-back counters: ranges deferred, filled on a page fault, filled
 * explicitly (DMA reads, b200_host_sync, partial overwrites), cancelled by a
 * covering write-back, bytes deferred, bytes materialised. */
int b200_lazy_counters(int64_t* ranges, int64_t* fault_fills, int64_t* explicit_fills, int64_t* cancelled,
                       int64_t* bytes_deferred, int64_t* bytes_filled);
/* Library and build identification, e.g. "lilac-b200 0.1 sm_100a". */
const char* b200_version(void);

/* ==========================================================================
 * 3. Counters (MarshalCounters, reference marshal.hpp:62-66, plus transfers)
 * ========================================================================== */

typedef struct {
    char region[64];        /* "<harness>.<param>", e.g. "b200_spmv_csr.val" */
    int64_t n_construct;
    int64_t n_update;
    int64_t n_destruct;
    int64_t bytes_h2d;      /* host->device bytes moved by update hooks */
    int64_t bytes_d2h;      /* device->host bytes moved by write-backs */
    int64_t bytes_d2d;      /* bytes served from a device mirror instead of the host */
    int32_t strategy;       /* 0 pageprotect, 1 checksum, 2 exact, 3 naive, 4 hybrid */
    int32_t fell_back;      /* PageProtect demoted to Checksum */
    int32_t streaming;      /* adaptive: rewritten every call, no longer guarded */
    int32_t constructed;
} b200_region_stats;

typedef struct {
    char harness[32];
    int64_t calls;
    double t_total_ms;      /* wall time inside the entry point */
    double t_poll_ms;       /* change detection + uploads (acquire phase) */
    double t_kernel_ms;     /* device time of the compute kernels (CUDA events) */
    double t_writeback_ms;  /* output transfer */
    int64_t bytes_h2d;
    int64_t bytes_d2h;
    int64_t bytes_d2d;      /* inputs served from device mirrors (no host transfer) */
} b200_harness_stats;

/* Copies up to `cap` region rows; returns the number of regions. */
int b200_region_stats_get(b200_region_stats* out, int cap);
int b200_harness_stats_get(b200_harness_stats* out, int cap);
void b200_stats_reset(void);
/* Change-detection cost counters since process start: SIGSEGV traps taken,
 * mprotect calls, bytes hashed; and device bytes currently held as mirrors. */
int b200_marshal_counters(int64_t* faults, int64_t* mprotects, int64_t* hash_bytes, int64_t* mirror_bytes);
/* Guarded caller regions found in DMA-reachable host memory (CUDA-pinned,
 * registered or managed). Page guards see CPU stores only: if another library
 * writes such an array by DMA or from a kernel, the resident copy would go
 * stale. Either call b200_host_forget on it after such a write, or run with
 * LILAC_B200_PINNED=always (those regions are then re-marshaled every call). */
int64_t b200_dma_visible_regions(void);
/* Host-side phase accumulators (ns, counts), collected while profiling is on
 * (b200_set_profiling): mirror fetch, mirror poll, D2D, H2D, D2H+sync, mirror
 * publish, publish guard, acquire (axpy/xpay inputs), launch, binding pick,
 * acquire_out, buffer hand-over, cudaMalloc (count only). Returns the number
 * of phases. */
int b200_host_profile(int64_t* ns, int64_t* counts, int cap);

/* ==========================================================================
 * 4. Resident device API (the harness internals, for drivers and benchmarks)
 * ========================================================================== */

typedef struct b200_matrix b200_matrix;  /* resident CSR or JDS matrix */

typedef struct {
    int64_t rows, cols, nnz, max_row;
    int32_t format;        /* 0 CSR, 1 JDS */
    int32_t col_bytes;     /* column index width the kernel streams: 8, 4 (narrowed) or 2 (tiled keys) */
    int32_t kernel;        /* CSR kernel chosen: 1 vector, 2 merge, 3 exact, 4 tiled, 5 split, 6 lane-range;
                              JDS: 0 thread per jagged row, 1 lane-segmented (k_jds_seg) */
    int32_t lanes;         /* CSR vector kernel lanes per row; JDS segmented: most lanes per row */
    int64_t device_bytes;  /* resident bytes */
} b200_matrix_info;

/* Upload host CSR / JDS arrays (same meaning and extents as the harness
 * entries). Returns 0 or -1. */
int b200_matrix_create_csr(b200_matrix** out, int64_t rows, const int64_t* row_ptr,
                           const int64_t* col_ind, const double* val);
int b200_matrix_create_jds(b200_matrix** out, int64_t rows, const int64_t* nzcnt,
                           const int64_t* perm, const double* val, const int64_t* jd_ptr,
                           const int64_t* col_ind);
void b200_matrix_free(b200_matrix* A);
int b200_matrix_info_get(const b200_matrix* A, b200_matrix_info* info);
/* y_device = A x_device on `stream` (cudaStream_t, may be NULL = default). */
int b200_spmv_device(const b200_matrix* A, const double* x_device, double* y_device, void* stream);
/* result_device[0] = a.b, deterministic (fixed partition + fixed-order sums). */
int b200_dot_device(const double* a_device, const double* b_device, int64_t n,
                    double* result_device, void* stream);
int b200_axpy_device(int64_t n, double* y_device, double alpha, const double* x_device, void* stream);
/* c = a b on device buffers (row-major: a n x p, b p x m, c n x m; the
 * b200_gemm computation). exact = 1: the reference's k order, bit-identical;
 * 0: the FP64 tensor-core (DMMA) kernel, within the north-star tolerance. */
int b200_gemm_device(int64_t n, int64_t m, int64_t p, const double* a_device, const double* b_device,
                     double* c_device, int exact, void* stream);
/* The 27-point stencil operator on an nx^3 grid (SURVEY §8(d) input 5),
 * generated directly in HBM: rows in lexicographic (i, j, k) order, each
 * row's neighbours in increasing column order, `diag` on the diagonal and
 * `offdiag` elsewhere (26.1 / -1 gives the SPD operator of the config). nx^3
 * must fit int32 columns (nx <= 1290). */
int b200_matrix_create_stencil27(b200_matrix** out, int64_t nx, double diag, double offdiag);
/* Rows [r0, r1) of the same operator as a resident matrix of r1 - r0 rows
 * over the full nx^3 columns (one shard of the row-sharded config). */
int b200_matrix_create_stencil27_rows(b200_matrix** out, int64_t nx, int64_t r0, int64_t r1, double diag,
                                      double offdiag);
/* `iters` PageRank steps on device vectors (SURVEY §8(d) input 4):
 * work = A x; x = damping*work + (1-damping)/n. A is the column-stochastic
 * transposed adjacency; x holds the start vector (e.g. 1/n). */
int b200_pagerank_device(const b200_matrix* A, double damping, int iters, double* x_device, double* work_device,
                         void* stream);
/* One PageRank step y = damping*(A x) + (1-damping)/rows into another device
 * vector (y must not alias x). On the lane-range layout the update is folded
 * into the SpMV's row stores (one pass, the same bits as SpMV + update). */
int b200_pagerank_step_device(const b200_matrix* A, double damping, const double* x_device, double* y_device,
                              void* stream);

/* Device buffers for harness TUs generated from a LiLAC-How spec
 * (paper_2001_07938_b200/specs/b200.lilac, emitted by the reference's own
 * harnessgen::gen_all): the marshal classes' code blocks call these. */
typedef struct {
    void* ptr;
    size_t bytes;
} B200Buf;
int b200_dbuf_alloc(B200Buf* b, size_t bytes);
int b200_dbuf_upload(B200Buf* b, const void* host, size_t bytes);  /* (re)allocates, H2D */
int b200_dbuf_download(void* host, const B200Buf* b, size_t bytes);
void b200_dbuf_free(B200Buf* b);
/* y = A x on device arrays at the ABI widths (int64 row_ptr/col_ind, f64),
 * rows/nnz/cols as the spec's marshaling derives them; synchronises. */
int b200_spmv_csr_dev(int64_t rows, int64_t nnz, int64_t cols, const void* row_ptr, const void* col_ind,
                      const void* val, const void* x, void* y);

/* ==========================================================================
 * 5. NPB CG driver (device-resident solver over a resident CSR matrix)
 * ========================================================================== */

typedef struct b200_cg b200_cg;

int b200_cg_create(b200_cg** out, const b200_matrix* A);
void b200_cg_free(b200_cg* cg);
/* x = 1 (NPB's start vector). */
int b200_cg_reset(b200_cg* cg, void* stream);
/* One NPB outer iteration: conj_grad (cgitmax CG steps + residual), then
 * zeta = shift + 1/(x.z), x = z/|z|. Uses a captured CUDA graph per stream. */
int b200_cg_outer(b200_cg* cg, int cgitmax, double shift, void* stream);
/* One CG step (spmv+dot, z/r update + r.r, p update). */
int b200_cg_step(b200_cg* cg, void* stream);
/* Plain CG in steps (the stencil config): b200_cg_start sets x = b (device
 * array of n doubles; NULL keeps the current x), z = 0, r = p = b, rho = r.r;
 * each b200_cg_step advances one iteration; b200_cg_finish computes
 * rnorm = |b - A z|. b200_cg_scalars copies rho and rnorm to the host on
 * `stream` (synchronises that stream). */
int b200_cg_start(b200_cg* cg, const double* b_device, void* stream);
int b200_cg_finish(b200_cg* cg, void* stream);
int b200_cg_scalars(b200_cg* cg, void* stream, double* rho, double* rnorm);
/* Copies zeta and the last residual norm to the host (synchronises). */
int b200_cg_result(b200_cg* cg, double* zeta, double* rnorm);
/* Plain CG on A z = b from z = 0: `iters` steps (the conj_grad recurrence),
 * then rnorm = |b - A z|. b_device / z_device: device arrays of n doubles
 * (z_device may be NULL). Synchronises. */
int b200_cg_solve(b200_cg* cg, const double* b_device, int iters, double* z_device, double* rnorm);
/* The whole NPB benchmark (1 untimed warm-up outer iteration + reset +
 * niter outer iterations). Returns 0 or -1; zeta/rnorm on the host. */
int b200_npb_cg(b200_cg* cg, int niter, double shift, double* zeta, double* rnorm);

/* ==========================================================================
 * 6. Workload synthesis (bench inputs; host arrays, caller-owned)
 * ========================================================================== */

/* NPB makea (rcond 0.1, randlc seed 314159265, multiplier 5^13), 0-based CSR,
 * ascending columns, duplicates summed in generation order. Call with
 * col_ind/val NULL to get *nnz (row_ptr filled), then again with storage. */
int b200_gen_npb(int64_t na, int nonzer, double shift, int64_t* row_ptr, int64_t* col_ind,
                 double* val, int64_t* nnz);

/* Graph500 Kronecker graph (2^scale vertices, edgefactor * 2^scale edges,
 * quadrant probabilities a/b/c, counter-based hashed uniforms from `seed`,
 * vertex labels permuted) as the PageRank operator: CSR of the transposed,
 * column-stochastic adjacency (row = dst, ascending src, duplicate edges kept,
 * val = 1/outdeg(src)). row_ptr: 2^scale + 1; col_ind / val: edgefactor *
 * 2^scale entries. Host threads. */
int b200_gen_kronecker(int scale, int edgefactor, uint64_t seed, double a, double b, double c, int64_t* row_ptr,
                       int64_t* col_ind, double* val);

/* ==========================================================================
 * 7. Row sharding (multi-GPU driver)
 * ========================================================================== */

/* nnz-balanced contiguous row ranges: bounds[g] = lower_bound(row_ptr,
 * row_ptr[0] + ceil(g*nnz/k)), clamped monotone; bounds[0]=0, bounds[k]=rows. */
void b200_partition_rows(int64_t rows, const int64_t* row_ptr, int k, int64_t* bounds);

/* Column footprint of a row block: [min col, max col + 1) of its nonzeros
 * (0, 0 when empty): the replica entries the block's SpMV reads. */
void b200_shard_footprint(int64_t rows, const int64_t* row_ptr, const int64_t* col_ind, int64_t* fmin,
                          int64_t* fmax);
/* The exchange plan: out[(s*world + r)*2 + {0,1}] = the slice-relative range
 * [lo, hi) of shard s (rows [bounds[s], bounds[s+1])) that rank r reads
 * (its footprint [fmin[r], fmax[r]) intersected with the shard). The peer
 * exchange pushes exactly these ranges. Host only. */
void b200_dist_send_ranges(int world, const int64_t* bounds, const int64_t* fmin, const int64_t* fmax,
                           int64_t* out);

/* Row-sharded NPB CG: each shard owns rows [bounds[g],
 * bounds[g+1]), keeps them resident, and all-gathers p every CG step (NCCL
 * over NVLink; grouped broadcasts for the variable slice sizes); the two dot
 * products are gathered in rank order and summed identically on every shard. */
typedef struct b200_dist_cg b200_dist_cg;

/* NCCL unique id (128 bytes) for b200_dist_cg_create_nccl; create on rank 0
 * and share it (e.g. torch.distributed broadcast). */
int b200_dist_nccl_id(void* id128);
/* One shard per process: this process is `rank` of `world` and owns rows
 * [bounds[rank], bounds[rank+1]); row_ptr has (rows+1) entries for those rows
 * with offsets into col_ind/val (global column indices). */
int b200_dist_cg_create_nccl(b200_dist_cg** out, int rank, int world, const void* nccl_id, int64_t n,
                             const int64_t* bounds, const int64_t* row_ptr, const int64_t* col_ind,
                             const double* val);
/* k shards on this process's GPU exchanging by device copies: the same
 * sharded algorithm, for single-GPU verification. Full CSR on input. */
int b200_dist_cg_create_local(b200_dist_cg** out, int k, int64_t n, const int64_t* row_ptr,
                              const int64_t* col_ind, const double* val);
/* The 27-point stencil (SURVEY §8(d) input 5) row-sharded: every shard's rows
 * are generated in its own HBM (nnz-balanced bounds, b200_dist_cg_bounds),
 * column footprint = its rows' neighbours, so the p exchange moves a halo of
 * about nx^2 rows per neighbour instead of the whole vector. One shard per
 * process (NCCL / peer memory) or k local shards on one GPU. */
int b200_dist_cg_create_stencil27_nccl(b200_dist_cg** out, int rank, int world, const void* nccl_id, int64_t nx,
                                       double diag, double offdiag);
int b200_dist_cg_create_stencil27_local(b200_dist_cg** out, int k, int64_t nx, double diag, double offdiag);
/* bounds[0..world] of the sharded driver's row partition. */
int b200_dist_cg_bounds(const b200_dist_cg* d, int64_t* bounds);
/* Plain sharded CG in steps: start_rowsum sets x = b = A 1 (the config's
 * right-hand side), z = 0, r = p = b; step = one CG iteration (SpMV + dots +
 * updates + the p exchange); finish = |b - A z| (gathers z); scalars copies
 * rho and rnorm to the host on `stream`. */
int b200_dist_cg_start_rowsum(b200_dist_cg* d, void* stream);
/* Plain sharded CG from b = the shards' x (e.g. b200_dist_cg_load_x from
 * host memory): z = 0, r = p = b. */
int b200_dist_cg_start(b200_dist_cg* d, void* stream);
int b200_dist_cg_step(b200_dist_cg* d, void* stream);
int b200_dist_cg_finish(b200_dist_cg* d, void* stream);
int b200_dist_cg_scalars(b200_dist_cg* d, void* stream, double* rho, double* rnorm);
void b200_dist_cg_free(b200_dist_cg* d);
int b200_dist_cg_reset(b200_dist_cg* d, void* stream);
int b200_dist_cg_outer(b200_dist_cg* d, int cgitmax, double shift, void* stream);
int b200_dist_cg_result(b200_dist_cg* d, double* zeta, double* rnorm);
/* x of the shards held by this process (in shard order, i.e. its owned rows)
 * from host memory (pinned for an asynchronous copy) on `stream`. */
int b200_dist_cg_load_x(b200_dist_cg* d, const double* x_host, void* stream);
/* Peer-memory exchange (no collective library): each shard stores its scalar
 * partials and its p / z slice straight into every peer's buffers and raises
 * an epoch flag per sender; receivers wait on the flags (p2p.cu).
 *  - local shards (b200_dist_cg_create_local): b200_dist_cg_use_p2p_local;
 *  - one shard per process (b200_dist_cg_create_nccl): b200_dist_cg_p2p_export
 *    writes this rank's record (208 bytes: three CUDA IPC handles and its
 *    column footprint), the caller all-gathers them (rank-major) and passes
 *    all to b200_dist_cg_p2p_attach.
 * A shard pushes to each peer only the part of its slice inside the peer's
 * column footprint (all of it for NPB; a halo for banded / stencil rows).
 * A wait without progress for 5 s fails the next result call (DeviceError). */
int b200_dist_cg_use_p2p_local(b200_dist_cg* d);
int b200_dist_cg_p2p_export(b200_dist_cg* d, void* out208);
int b200_dist_cg_p2p_attach(b200_dist_cg* d, const void* handles);
/* 0 local device copies, 1 NCCL, 2 peer memory. */
int b200_dist_cg_transport(const b200_dist_cg* d);
/* With the peer-memory exchange and the tiled layout on every shard, the CG
 * steps of an outer iteration run in one persistent kernel per process
 * (k_cg_tiled_dist: SpMV, partial publish, flag waits and the p push inside
 * it; local shards share one cooperative grid). on = 0 keeps the per-step
 * kernels (default on; LILAC_B200_DIST_FUSED=0 turns it off process-wide).
 * b200_dist_cg_fused: 1 if the last outer iteration ran the fused kernel. */
int b200_dist_cg_set_fused(b200_dist_cg* d, int on);
int b200_dist_cg_fused(const b200_dist_cg* d);
int b200_dist_npb(b200_dist_cg* d, int niter, double shift, double* zeta, double* rnorm);
int b200_dist_cg_info(const b200_dist_cg* d, int shard, int64_t* row0, int64_t* rows, int64_t* nnz,
                      int32_t* tiled);

#ifdef __cplusplus
}
#endif

#endif /* LILAC_B200_H */
