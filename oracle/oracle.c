/*
 * oracle.c — CPU restatement of the LiLAC harness path. TEST INFRASTRUCTURE ONLY
 * (see oracle.h for who may call it). Compiled with -O2 -ffp-contract=off so
 * every `acc += a*b` is a separate IEEE multiply and add, as in the reference
 * build (g++ x86-64 default, no FMA contraction).
 */
#include "oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

#include <pthread.h>
#include <unistd.h>

/* ------------------------------------------------------------------------ */
/* Reference computations                                                    */
/* ------------------------------------------------------------------------ */

/* Restates Eval::run_forall/run_dot (what_interp.cpp:72-108) for the
 * spmv_csr program (kernels.lilac:1-4): lexicographic forall over i, a dot
 * over j accumulating from exact +0.0 left to right, then one store to
 * output[i]. Bounds checks mirror the OutOfBounds throws at
 * what_interp.cpp:52-53 (int arrays) and :67-68 (float arrays). */
int orc_spmv_csr(int64_t rows, double* output, const int64_t* row_ptr, const double* val,
                 const double* x, const int64_t* col_ind, int64_t nnz, int64_t ncols) {
    for (int64_t i = 0; i < rows; ++i) {
        int64_t lo = row_ptr[i], hi = row_ptr[i + 1];
        double acc = 0.0;
        for (int64_t j = lo; j < hi; ++j) {
            if (j < 0 || j >= nnz) return -1;
            int64_t c = col_ind[j];
            if (c < 0 || c >= ncols) return -1;
            acc += val[j] * x[c];
        }
        output[i] = acc;
    }
    return 0;
}

/* spmv_jds (kernels.lilac:9-12): the dot range is [0, nzcnt[perm[i]]), the
 * element address is jd_ptr[k] + perm[i] (what_interp.cpp:87-108 with the
 * wrap_add of :9-11 — irrelevant for valid data). */
int orc_spmv_jds(int64_t rows, double* output, const int64_t* nzcnt, const int64_t* perm,
                 const double* val, const int64_t* jd_ptr, const double* x,
                 const int64_t* col_ind, int64_t nnz, int64_t njd, int64_t ncols) {
    for (int64_t i = 0; i < rows; ++i) {
        int64_t p = perm[i];
        if (p < 0 || p >= rows) return -1;
        int64_t len = nzcnt[p];
        double acc = 0.0;
        for (int64_t k = 0; k < len; ++k) {
            if (k >= njd) return -1;
            int64_t off = jd_ptr[k] + p;
            if (off < 0 || off >= nnz) return -1;
            int64_t c = col_ind[off];
            if (c < 0 || c >= ncols) return -1;
            acc += val[off] * x[c];
        }
        output[i] = acc;
    }
    return 0;
}

/* dotproduct (kernels.lilac:6-7); scalar-result protocol interp.cpp:335-346:
 * the result slot starts as a synthesized {0.0} and receives acc. */
void orc_dot(double* result, int64_t length, const double* a, const double* b) {
    double acc = 0.0;
    for (int64_t i = 0; i < length; ++i) acc += a[i] * b[i];
    result[0] = acc;
}

void orc_axpy(int64_t n, double* y, double alpha, const double* x) {
    for (int64_t i = 0; i < n; ++i) y[i] = y[i] + alpha * x[i];
}

typedef struct {
    int64_t lo, hi;
    double* output;
    const int64_t* row_ptr;
    const double* val;
    const double* x;
    const int64_t* col_ind;
} csr_slice;

static void* csr_slice_run(void* arg) {
    const csr_slice* s = (const csr_slice*)arg;
    for (int64_t i = s->lo; i < s->hi; ++i) {
        double acc = 0.0;
        for (int64_t j = s->row_ptr[i]; j < s->row_ptr[i + 1]; ++j)
            acc += s->val[j] * s->x[s->col_ind[j]];
        s->output[i] = acc;
    }
    return NULL;
}

void orc_spmv_csr_mt(int64_t rows, double* output, const int64_t* row_ptr, const double* val,
                     const double* x, const int64_t* col_ind, int nthreads) {
    if (nthreads <= 0) nthreads = (int)sysconf(_SC_NPROCESSORS_ONLN);
    if (nthreads > 256) nthreads = 256;
    if (nthreads <= 1 || rows < 4096) {
        csr_slice s = {0, rows, output, row_ptr, val, x, col_ind};
        csr_slice_run(&s);
        return;
    }
    pthread_t th[256];
    csr_slice sl[256];
    for (int t = 0; t < nthreads; ++t) {
        sl[t] = (csr_slice){rows * t / nthreads, rows * (t + 1) / nthreads, output, row_ptr, val, x, col_ind};
        pthread_create(&th[t], NULL, csr_slice_run, &sl[t]);
    }
    for (int t = 0; t < nthreads; ++t) pthread_join(th[t], NULL);
}

/* Multi-threaded JDS SpMV: original rows split statically across threads,
 * each row in the reference's k order (bit-identical to orc_spmv_jds; no
 * bounds checks: the caller validated the arrays with orc_spmv_jds). */
typedef struct {
    int64_t lo, hi;
    double* output;
    const int64_t *nzcnt, *perm, *jd_ptr, *col_ind;
    const double *val, *x;
} jds_slice;

static void* jds_slice_run(void* arg) {
    const jds_slice* s = (const jds_slice*)arg;
    for (int64_t i = s->lo; i < s->hi; ++i) {
        const int64_t p = s->perm[i], len = s->nzcnt[p];
        double acc = 0.0;
        for (int64_t k = 0; k < len; ++k) {
            const int64_t off = s->jd_ptr[k] + p;
            acc += s->val[off] * s->x[s->col_ind[off]];
        }
        s->output[i] = acc;
    }
    return NULL;
}

void orc_spmv_jds_mt(int64_t rows, double* output, const int64_t* nzcnt, const int64_t* perm,
                     const double* val, const int64_t* jd_ptr, const double* x, const int64_t* col_ind,
                     int nthreads) {
    if (nthreads <= 0) nthreads = (int)sysconf(_SC_NPROCESSORS_ONLN);
    if (nthreads > 256) nthreads = 256;
    if (nthreads <= 1 || rows < 4096) {
        jds_slice s = {0, rows, output, nzcnt, perm, jd_ptr, col_ind, val, x};
        jds_slice_run(&s);
        return;
    }
    pthread_t th[256];
    jds_slice sl[256];
    for (int t = 0; t < nthreads; ++t) {
        sl[t] = (jds_slice){rows * t / nthreads, rows * (t + 1) / nthreads, output, nzcnt, perm, jd_ptr, col_ind,
                            val, x};
        pthread_create(&th[t], NULL, jds_slice_run, &sl[t]);
    }
    for (int t = 0; t < nthreads; ++t) pthread_join(th[t], NULL);
}

/* ------------------------------------------------------------------------ */
/* Encoders                                                                  */
/* ------------------------------------------------------------------------ */

int64_t orc_count_nonzeros(int64_t rows, int64_t cols, const double* a) {
    int64_t n = 0;
    for (int64_t i = 0; i < rows * cols; ++i) n += a[i] != 0.0;
    return n;
}

/* csr_from_dense, oracles.hpp:68-84: row-major scan, v != 0.0 kept. */
void orc_csr_from_dense(int64_t rows, int64_t cols, const double* a, double* val,
                        int64_t* col_ind, int64_t* row_ptr) {
    int64_t n = 0;
    row_ptr[0] = 0;
    for (int64_t i = 0; i < rows; ++i) {
        for (int64_t k = 0; k < cols; ++k) {
            double v = a[i * cols + k];
            if (v != 0.0) {
                val[n] = v;
                col_ind[n] = k;
                ++n;
            }
        }
        row_ptr[i + 1] = n;
    }
}

int64_t orc_csr_max_row(int64_t rows, const int64_t* row_ptr) {
    int64_t m = 0;
    for (int64_t i = 0; i < rows; ++i)
        if (row_ptr[i + 1] - row_ptr[i] > m) m = row_ptr[i + 1] - row_ptr[i];
    return m;
}

/* jds_from_dense, oracles.hpp:109-144, fed from CSR (same nonzero order per
 * row, since csr_from_dense and jds_from_dense both scan columns ascending).
 * std::stable_sort by descending count == counting sort by count, iterating
 * counts high to low and rows in original order inside a count. */
void orc_jds_from_csr(int64_t rows, const int64_t* row_ptr, const double* csr_val,
                      const int64_t* csr_col, int64_t* perm, int64_t* nzcnt, int64_t* jd_ptr,
                      double* val, int64_t* col_ind) {
    int64_t max_nz = orc_csr_max_row(rows, row_ptr);
    int64_t* order = (int64_t*)malloc(sizeof(int64_t) * (size_t)(rows > 0 ? rows : 1));
    int64_t j = 0;
    for (int64_t c = max_nz; c >= 0; --c)
        for (int64_t i = 0; i < rows; ++i)
            if (row_ptr[i + 1] - row_ptr[i] == c) order[j++] = i;
    for (j = 0; j < rows; ++j) {
        perm[order[j]] = j;
        nzcnt[j] = row_ptr[order[j] + 1] - row_ptr[order[j]];
    }
    int64_t n = 0;
    jd_ptr[0] = 0;
    for (int64_t k = 0; k < max_nz; ++k) {
        for (j = 0; j < rows && nzcnt[j] > k; ++j) {
            int64_t src = row_ptr[order[j]] + k;
            val[n] = csr_val[src];
            col_ind[n] = csr_col[src];
            ++n;
        }
        jd_ptr[k + 1] = n;
    }
    free(order);
}

/* ------------------------------------------------------------------------ */
/* Marshal checksum                                                          */
/* ------------------------------------------------------------------------ */

/* marshal.cpp:108-116 */
uint64_t orc_fnv1a(const void* data, size_t size) {
    const unsigned char* p = (const unsigned char*)data;
    uint64_t h = 14695981039346656037ULL;
    for (size_t i = 0; i < size; ++i) {
        h ^= p[i];
        h *= 1099511628211ULL;
    }
    return h;
}

/* ------------------------------------------------------------------------ */
/* Row partition                                                             */
/* ------------------------------------------------------------------------ */

static int64_t lower_bound_i64(const int64_t* a, int64_t n, int64_t v) {
    int64_t lo = 0, hi = n;
    while (lo < hi) {
        int64_t mid = lo + (hi - lo) / 2;
        if (a[mid] < v)
            lo = mid + 1;
        else
            hi = mid;
    }
    return lo;
}

void orc_partition_rows(int64_t rows, const int64_t* row_ptr, int k, int64_t* bounds) {
    int64_t base = rows > 0 ? row_ptr[0] : 0;
    int64_t nnz = rows > 0 ? row_ptr[rows] - base : 0;
    bounds[0] = 0;
    for (int g = 1; g < k; ++g) {
        int64_t target = base + (nnz * g + k - 1) / k;
        int64_t r = rows > 0 ? lower_bound_i64(row_ptr, rows + 1, target) : 0;
        if (r > rows) r = rows;
        if (r < bounds[g - 1]) r = bounds[g - 1];
        bounds[g] = r;
    }
    bounds[k] = rows;
}

/* ------------------------------------------------------------------------ */
/* NPB CG (NPB 3.x cg: randlc, sprnvc, vecset, makea, sparse, conj_grad)      */
/* ------------------------------------------------------------------------ */

double orc_randlc(double* x, double a) {
    const double r23 = 1.1920928955078125e-07, r46 = r23 * r23;
    const double t23 = 8.388608e+06, t46 = t23 * t23;
    double t1, t2, t3, t4, a1, a2, x1, x2, z;
    t1 = r23 * a;
    a1 = (double)(int)t1;
    a2 = a - t23 * a1;
    t1 = r23 * (*x);
    x1 = (double)(int)t1;
    x2 = *x - t23 * x1;
    t1 = a1 * x2 + a2 * x1;
    t2 = (double)(int)(r23 * t1);
    z = t1 - t23 * t2;
    t3 = t23 * z + a2 * x2;
    t4 = (double)(int)(r46 * t3);
    *x = t3 - t46 * t4;
    return r46 * (*x);
}

typedef struct {
    double tran, amult;
} npb_rng;

/* sprnvc: nz distinct random positions in [1, n] with random values. */
static void npb_sprnvc(npb_rng* g, int64_t n, int nz, int64_t nn1, double* v, int64_t* iv) {
    int nzv = 0;
    while (nzv < nz) {
        double vecelt = orc_randlc(&g->tran, g->amult);
        double vecloc = orc_randlc(&g->tran, g->amult);
        int64_t i = (int64_t)(nn1 * vecloc) + 1; /* icnvrt */
        if (i > n) continue;
        int was_gen = 0;
        for (int ii = 0; ii < nzv; ++ii)
            if (iv[ii] == i) {
                was_gen = 1;
                break;
            }
        if (was_gen) continue;
        v[nzv] = vecelt;
        iv[nzv] = i;
        ++nzv;
    }
}

/* vecset: set v at position i to val, appending if absent. */
static void npb_vecset(double* v, int64_t* iv, int* nzv, int64_t i, double val) {
    int set = 0;
    for (int k = 0; k < *nzv; ++k)
        if (iv[k] == i) {
            v[k] = val;
            set = 1;
        }
    if (!set) {
        v[*nzv] = val;
        iv[*nzv] = i;
        *nzv += 1;
    }
}

int orc_npb_makea(int64_t n, int nonzer, double shift, int64_t* row_ptr, int64_t* col_ind,
                  double* val, int64_t* nnz_out) {
    const double rcond = 0.1;
    const int w = nonzer + 1;
    npb_rng g = {314159265.0, 1220703125.0};
    (void)orc_randlc(&g.tran, g.amult); /* zeta = randlc(&tran, amult) in main */

    int* arow = (int*)malloc(sizeof(int) * (size_t)n);
    int64_t* acol = (int64_t*)malloc(sizeof(int64_t) * (size_t)n * (size_t)w);
    double* aelt = (double*)malloc(sizeof(double) * (size_t)n * (size_t)w);
    int64_t nn1 = 1;
    do {
        nn1 *= 2;
    } while (nn1 < n);

    double vc[64];
    int64_t ivc[64];
    for (int64_t iouter = 0; iouter < n; ++iouter) {
        int nzv = nonzer;
        npb_sprnvc(&g, n, nzv, nn1, vc, ivc);
        npb_vecset(vc, ivc, &nzv, iouter + 1, 0.5);
        arow[iouter] = nzv;
        for (int e = 0; e < nzv; ++e) {
            acol[iouter * w + e] = ivc[e] - 1;
            aelt[iouter * w + e] = vc[e];
        }
    }

    /* sparse(): count triples per row, then insert with summing of duplicates */
    int64_t* rowstr = (int64_t*)calloc((size_t)n + 1, sizeof(int64_t));
    for (int64_t i = 0; i < n; ++i)
        for (int e = 0; e < arow[i]; ++e) rowstr[acol[i * w + e] + 1] += arow[i];
    for (int64_t j = 1; j <= n; ++j) rowstr[j] += rowstr[j - 1];
    int64_t cap = rowstr[n];
    double* a = (double*)malloc(sizeof(double) * (size_t)(cap > 0 ? cap : 1));
    int64_t* colidx = (int64_t*)malloc(sizeof(int64_t) * (size_t)(cap > 0 ? cap : 1));
    int64_t* nzloc = (int64_t*)calloc((size_t)n, sizeof(int64_t));
    for (int64_t k = 0; k < cap; ++k) {
        a[k] = 0.0;
        colidx[k] = -1;
    }
    double size = 1.0;
    double ratio = pow(rcond, 1.0 / (double)n);
    for (int64_t i = 0; i < n; ++i) {
        for (int nza = 0; nza < arow[i]; ++nza) {
            int64_t j = acol[i * w + nza];
            double scale = size * aelt[i * w + nza];
            for (int nzrow = 0; nzrow < arow[i]; ++nzrow) {
                int64_t jcol = acol[i * w + nzrow];
                double va = aelt[i * w + nzrow] * scale;
                if (jcol == j && j == i) va = va + rcond - shift;
                int64_t k;
                int found = 0;
                for (k = rowstr[j]; k < rowstr[j + 1]; ++k) {
                    if (colidx[k] > jcol) {
                        for (int64_t kk = rowstr[j + 1] - 2; kk >= k; --kk)
                            if (colidx[kk] > -1) {
                                a[kk + 1] = a[kk];
                                colidx[kk + 1] = colidx[kk];
                            }
                        colidx[k] = jcol;
                        a[k] = 0.0;
                        found = 1;
                        break;
                    } else if (colidx[k] == -1) {
                        colidx[k] = jcol;
                        found = 1;
                        break;
                    } else if (colidx[k] == jcol) {
                        nzloc[j] += 1;
                        found = 1;
                        break;
                    }
                }
                if (!found) {
                    free(arow); free(acol); free(aelt); free(rowstr); free(a); free(colidx); free(nzloc);
                    return -1;
                }
                a[k] = a[k] + va;
            }
        }
        size = size * ratio;
    }
    for (int64_t j = 1; j < n; ++j) nzloc[j] += nzloc[j - 1];
    /* compaction into the caller's arrays */
    row_ptr[0] = 0;
    for (int64_t j = 0; j < n; ++j) row_ptr[j + 1] = rowstr[j + 1] - nzloc[j];
    *nnz_out = row_ptr[n];
    if (val && col_ind) {
        for (int64_t j = 0; j < n; ++j) {
            int64_t src = rowstr[j];
            for (int64_t k = row_ptr[j]; k < row_ptr[j + 1]; ++k, ++src) {
                val[k] = a[src];
                col_ind[k] = colidx[src];
            }
        }
    }
    free(arow); free(acol); free(aelt); free(rowstr); free(a); free(colidx); free(nzloc);
    return 0;
}

static double npb_conj_grad(int64_t n, const int64_t* rowstr, const int64_t* colidx,
                            const double* a, const double* x, double* z, double* p, double* q,
                            double* r) {
    const int cgitmax = 25;
    double rho = 0.0, d, alpha, beta, rho0, sum;
    for (int64_t j = 0; j < n; ++j) {
        q[j] = 0.0;
        z[j] = 0.0;
        r[j] = x[j];
        p[j] = r[j];
    }
    for (int64_t j = 0; j < n; ++j) rho = rho + r[j] * r[j];
    for (int cgit = 1; cgit <= cgitmax; ++cgit) {
        orc_spmv_csr_mt(n, q, rowstr, a, p, colidx, 0);
        d = 0.0;
        for (int64_t j = 0; j < n; ++j) d = d + p[j] * q[j];
        alpha = rho / d;
        rho0 = rho;
        rho = 0.0;
        for (int64_t j = 0; j < n; ++j) {
            z[j] = z[j] + alpha * p[j];
            r[j] = r[j] - alpha * q[j];
        }
        for (int64_t j = 0; j < n; ++j) rho = rho + r[j] * r[j];
        beta = rho / rho0;
        for (int64_t j = 0; j < n; ++j) p[j] = r[j] + beta * p[j];
    }
    orc_spmv_csr_mt(n, r, rowstr, a, z, colidx, 0);
    sum = 0.0;
    for (int64_t j = 0; j < n; ++j) {
        d = x[j] - r[j];
        sum = sum + d * d;
    }
    return sqrt(sum);
}

/* One NPB outer iteration from the caller's x (NPB 3.x cg main loop body):
 * conj_grad with the SpMV on `nthreads` threads (bit-identical for any count),
 * then zeta = shift + 1/(x.z), x = z/|z|. Returns zeta; *rnorm_out = |x - A z|.
 * Scratch: z, p, q, r of n doubles. */
static double npb_conj_grad_t(int64_t n, const int64_t* rowstr, const int64_t* colidx, const double* a,
                              const double* x, double* z, double* p, double* q, double* r, int nthreads) {
    const int cgitmax = 25;
    double rho = 0.0, d, alpha, beta, rho0, sum;
    for (int64_t j = 0; j < n; ++j) {
        q[j] = 0.0;
        z[j] = 0.0;
        r[j] = x[j];
        p[j] = r[j];
    }
    for (int64_t j = 0; j < n; ++j) rho = rho + r[j] * r[j];
    for (int cgit = 1; cgit <= cgitmax; ++cgit) {
        orc_spmv_csr_mt(n, q, rowstr, a, p, colidx, nthreads);
        d = 0.0;
        for (int64_t j = 0; j < n; ++j) d = d + p[j] * q[j];
        alpha = rho / d;
        rho0 = rho;
        rho = 0.0;
        for (int64_t j = 0; j < n; ++j) {
            z[j] = z[j] + alpha * p[j];
            r[j] = r[j] - alpha * q[j];
        }
        for (int64_t j = 0; j < n; ++j) rho = rho + r[j] * r[j];
        beta = rho / rho0;
        for (int64_t j = 0; j < n; ++j) p[j] = r[j] + beta * p[j];
    }
    orc_spmv_csr_mt(n, r, rowstr, a, z, colidx, nthreads);
    sum = 0.0;
    for (int64_t j = 0; j < n; ++j) {
        d = x[j] - r[j];
        sum = sum + d * d;
    }
    return sqrt(sum);
}

double orc_npb_outer(int64_t n, const int64_t* row_ptr, const int64_t* col_ind, const double* val, double* x,
                     double* z, double* p, double* q, double* r, double shift, int nthreads, double* rnorm_out) {
    const double rnorm = npb_conj_grad_t(n, row_ptr, col_ind, val, x, z, p, q, r, nthreads);
    double t1 = 0.0, t2 = 0.0;
    for (int64_t j = 0; j < n; ++j) {
        t1 = t1 + x[j] * z[j];
        t2 = t2 + z[j] * z[j];
    }
    t2 = 1.0 / sqrt(t2);
    for (int64_t j = 0; j < n; ++j) x[j] = t2 * z[j];
    if (rnorm_out) *rnorm_out = rnorm;
    return shift + 1.0 / t1;
}

double orc_npb_cg(int64_t n, const int64_t* row_ptr, const int64_t* col_ind, const double* val,
                  int niter, double shift, double* rnorm_out) {
    double* x = (double*)malloc(sizeof(double) * (size_t)n);
    double* z = (double*)malloc(sizeof(double) * (size_t)n);
    double* p = (double*)malloc(sizeof(double) * (size_t)n);
    double* q = (double*)malloc(sizeof(double) * (size_t)n);
    double* r = (double*)malloc(sizeof(double) * (size_t)n);
    double zeta = 0.0, rnorm = 0.0;
    for (int64_t j = 0; j < n; ++j) x[j] = 1.0;
    for (int it = 0; it <= niter; ++it) {
        /* it == 0 is NPB's untimed warm-up iteration, after which x is reset */
        rnorm = npb_conj_grad(n, row_ptr, col_ind, val, x, z, p, q, r);
        double t1 = 0.0, t2 = 0.0;
        for (int64_t j = 0; j < n; ++j) {
            t1 = t1 + x[j] * z[j];
            t2 = t2 + z[j] * z[j];
        }
        t2 = 1.0 / sqrt(t2);
        if (it > 0) zeta = shift + 1.0 / t1;
        for (int64_t j = 0; j < n; ++j) x[j] = t2 * z[j];
        if (it == 0)
            for (int64_t j = 0; j < n; ++j) x[j] = 1.0;
    }
    free(x); free(z); free(p); free(q); free(r);
    if (rnorm_out) *rnorm_out = rnorm;
    return zeta;
}

/* gemm (kernels.lilac:14-19) in what_interp.cpp's order: forall i, forall j,
 * acc = +0.0, k ascending, separate mul and add (-ffp-contract=off). */
void orc_gemm(int64_t n, int64_t m, double* c, int64_t p, const double* a, const double* b) {
    for (int64_t i = 0; i < n; ++i)
        for (int64_t j = 0; j < m; ++j) {
            double acc = 0.0;
            for (int64_t k = 0; k < p; ++k) acc += a[i * p + k] * b[k * m + j];
            c[i * m + j] = acc;
        }
}
