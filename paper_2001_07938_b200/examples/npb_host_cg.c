/* npb_host_cg.c — the LiLAC usage model in C: NPB CG's conj_grad as a
 * compiled host program whose SpMV, dot-product and axpy loops were replaced
 * by calls to the harness entry points (include/lilac_b200.h §1), i.e. what a
 * program rewritten by LiLAC and linked against liblilac_b200.so executes.
 * The vectors live in the caller's host memory; the harness runtime decides
 * what crosses the bus (resident matrix, device mirrors, lazy write-back).
 *
 * Built by paper_2001_07938_b200/build.py into libnpb_host_cg.so; bench.py
 * times it for the e2e leg (no interpreter between the calls). */
#include <math.h>
#include <stdint.h>
#include <string.h>

#include "lilac_b200.h"

enum { kCgItMax = 25 };

/* One NPB outer iteration (NPB 3.x cg main loop body): conj_grad from x,
 * then zeta = shift + 1/(x.z), x = z / |z|. Returns zeta; *rnorm_out = |x - A z|. */
double npb_host_cg_outer(int64_t n, const int64_t* row_ptr, const double* val, const int64_t* col_ind, double* x,
                         double* z, double* r, double* p, double* q, double* res, double shift, double* rnorm_out) {
    double rho, rho0, d, alpha, beta;
    memset(z, 0, sizeof(double) * (size_t)n);
    memset(q, 0, sizeof(double) * (size_t)n);
    memcpy(r, x, sizeof(double) * (size_t)n);
    memcpy(p, r, sizeof(double) * (size_t)n);
    b200_dot(&rho, n, r, r);
    for (int it = 0; it < kCgItMax; ++it) {
        b200_spmv_csr(n, q, row_ptr, val, p, col_ind);  /* q = A p */
        b200_dot(&d, n, p, q);
        alpha = rho / d;
        rho0 = rho;
        b200_axpy(n, z, alpha, p);   /* z = z + alpha p */
        b200_axpy(n, r, -alpha, q);  /* r = r - alpha q */
        b200_dot(&rho, n, r, r);
        beta = rho / rho0;
        b200_xpay(n, p, beta, r);    /* p = r + beta p */
    }
    b200_spmv_csr(n, r, row_ptr, val, z, col_ind); /* r = A z */
    for (int64_t i = 0; i < n; ++i) res[i] = x[i] - r[i];
    double rr, t1, zz;
    b200_dot(&rr, n, res, res);
    b200_dot(&t1, n, x, z);
    b200_dot(&zz, n, z, z);
    const double t2 = 1.0 / sqrt(zz);
    for (int64_t i = 0; i < n; ++i) x[i] = t2 * z[i];
    if (rnorm_out) *rnorm_out = sqrt(rr);
    return shift + 1.0 / t1;
}
