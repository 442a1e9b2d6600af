// cg.cu — device kernels of the NPB CG driver (conj_grad, NPB 3.x cg).
//
// One CG step = 3 kernels:
//   spmv_dot   q = A p, d = p.q; alpha = rho/d           (kernels.cu, fused)
//   update_zr  z += alpha p, r -= alpha q, rho' = r.r;  beta = rho'/rho
//   update_p   p = r + beta p
// Scalars never leave the device (CgScalars); reductions are deterministic
// (fixed grid, fixed per-thread order, fixed trees, last-CTA finalisation).
// Elementwise updates use explicitly rounded mul/add so each element matches
// the scalar NPB loop bit for bit; only the dot products reassociate.

#include "b200.hpp"
#include "cg_fin.cuh"
#include "p2p.hpp"

#include <algorithm>

namespace b200 {

namespace {

constexpr int kThreads = 256;

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

__device__ __forceinline__ double block_sum(double v) {
    __shared__ double sh[kThreads / 32];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    v = warp_sum(v);
    __syncthreads();
    if (lane == 0) sh[w] = v;
    __syncthreads();
    if (w == 0) v = warp_sum(lane < kThreads / 32 ? sh[lane] : 0.0);
    return v;
}

// Writes this CTA's partials (NV values) and, in the last CTA to arrive, sums
// each partial array in CTA order; totals valid in thread 0 of that CTA.
template <int NV>
__device__ bool finish(const double (&v)[NV], double* partials, unsigned int* ticket, double (&tot)[NV]) {
    __shared__ bool last;
    double s[NV];
#pragma unroll
    for (int k = 0; k < NV; ++k) s[k] = block_sum(v[k]);
    if (threadIdx.x == 0) {
#pragma unroll
        for (int k = 0; k < NV; ++k) partials[k * kMaxParts + blockIdx.x] = s[k];
    }
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) last = atomicAdd(ticket, 1u) == gridDim.x - 1;
    __syncthreads();
    if (!last) return false;
    __threadfence();
#pragma unroll
    for (int k = 0; k < NV; ++k) {
        double a = 0.0;
        for (unsigned i = threadIdx.x; i < gridDim.x; i += kThreads) a += __ldcg(partials + k * kMaxParts + i);
        tot[k] = block_sum(a);
    }
    if (threadIdx.x == 0) *ticket = 0u;
    return true;
}

#define GRID_STRIDE(i, n)                                                                   \
    for (std::int64_t i = static_cast<std::int64_t>(blockIdx.x) * kThreads + threadIdx.x; i < (n); \
         i += static_cast<std::int64_t>(gridDim.x) * kThreads)

__global__ void __launch_bounds__(kThreads) k_cg_init(CgVectors v) {
    double rr = 0.0;
    GRID_STRIDE(i, v.n) {
        const double xi = v.x[i];
        v.q[i] = 0.0;
        v.z[i] = 0.0;
        v.r[i] = xi;
        v.p[i] = xi;
        rr += xi * xi;
    }
    double part[1] = {rr}, tot[1];
    if (finish<1>(part, v.partials, &v.sc->ticket[1], tot) && threadIdx.x == 0) {
        if (v.sc->nranks > 1)
            p2p_publish(v.sc, tot, 1);
        else
            v.sc->rho = tot[0];
    }
}

__global__ void __launch_bounds__(kThreads) k_cg_update_zr(CgVectors v) {
    pdl_trigger();
    pdl_wait();
    const double alpha = v.sc->alpha;
    double rr = 0.0;
    GRID_STRIDE(i, v.n) {
        const double zi = __dadd_rn(v.z[i], __dmul_rn(alpha, v.p[i]));
        const double ri = __dsub_rn(v.r[i], __dmul_rn(alpha, v.q[i]));
        v.z[i] = zi;
        v.r[i] = ri;
        rr += ri * ri;
    }
    double part[1] = {rr}, tot[1];
    if (finish<1>(part, v.partials, &v.sc->ticket[1], tot) && threadIdx.x == 0) {
        if (v.sc->nranks > 1) {
            p2p_publish(v.sc, tot, 1);
        } else {
            v.sc->rho = tot[0];
            v.sc->beta = tot[0] / v.sc->rho0;
        }
    }
}

__global__ void __launch_bounds__(kThreads) k_cg_update_p(CgVectors v) {
    pdl_trigger();
    pdl_wait();
    const double beta = v.sc->beta;
    GRID_STRIDE(i, v.n) v.p[i] = __dadd_rn(v.r[i], __dmul_rn(beta, v.p[i]));
}

__global__ void __launch_bounds__(kThreads) k_cg_resid(CgVectors v) {
    double s = 0.0;
    GRID_STRIDE(i, v.n) {
        const double d = __dsub_rn(v.x[i], v.r[i]);
        s += d * d;
    }
    double part[1] = {s}, tot[1];
    if (finish<1>(part, v.partials, &v.sc->ticket[2], tot) && threadIdx.x == 0) {
        if (v.sc->nranks > 1)
            p2p_publish(v.sc, tot, 1);
        else
            v.sc->rnorm = sqrt(tot[0]);
    }
}

__global__ void __launch_bounds__(kThreads) k_cg_norms(CgVectors v, double shift) {
    double a = 0.0, b = 0.0;
    GRID_STRIDE(i, v.n) {
        const double zi = v.z[i];
        a += v.x[i] * zi;
        b += zi * zi;
    }
    double part[2] = {a, b}, tot[2];
    if (finish<2>(part, v.partials, &v.sc->ticket[3], tot) && threadIdx.x == 0) {
        if (v.sc->nranks > 1) {
            p2p_publish(v.sc, tot, 2);
        } else {
            v.sc->t1 = tot[0];
            v.sc->t2 = 1.0 / sqrt(tot[1]);
            v.sc->zeta = shift + 1.0 / tot[0];
        }
    }
}

// p.q after a merge-path SpMV (same scalar protocol as the fused kernels).
__global__ void __launch_bounds__(kThreads) k_cg_dot_scalars(const double* __restrict__ p,
                                                              const double* __restrict__ q, std::int64_t n,
                                                              double* partials, unsigned int* ticket, CgScalars* sc) {
    double a = 0.0;
    GRID_STRIDE(i, n) a += p[i] * q[i];
    double part[1] = {a}, tot[1];
    if (finish<1>(part, partials, ticket, tot) && threadIdx.x == 0) {
        if (sc->nranks > 1) {
            p2p_publish(sc, tot, 1);
        } else {
            sc->d = tot[0];
            sc->rho0 = sc->rho;
            sc->alpha = sc->rho / tot[0];
        }
    }
}

// Sharded finalisation: sum the shards' partials in rank order (deterministic).
__global__ void k_cg_fin(int what, CgScalars* sc, const double* __restrict__ g, int nranks, double shift) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    cg_fin_apply(what, sc, g, nranks, shift);
}

__global__ void __launch_bounds__(kThreads) k_cg_scale_x(CgVectors v) {
    const double t2 = v.sc->t2;
    GRID_STRIDE(i, v.n) v.x[i] = __dmul_rn(t2, v.z[i]);
}

__global__ void k_cg_fill(double* x, std::int64_t n, double val) {
    GRID_STRIDE(i, n) x[i] = val;
}

// Two elements per thread: the CG vectors are L2-resident between steps, so
// these kernels are latency-bound — all of a thread's loads should be in
// flight at once rather than walked in a grid-stride loop.
// Large vectors (the stencil's 74M rows): one full wave of 8 CTAs per SM
// walking grid-stride (2048 CTAs were 1.7 waves, the second 73% full).
unsigned vec_grid(const CgVectors& v) {
    std::int64_t g = (v.n + kThreads * 2 - 1) / (kThreads * 2);
    return static_cast<unsigned>(std::max<std::int64_t>(1, std::min<std::int64_t>(g, 148 * 8)));
}

}  // namespace

void cg_launch_init(const CgVectors& v, cudaStream_t s) {
    k_cg_init<<<vec_grid(v), kThreads, 0, s>>>(v);
    B200_CUDA(cudaGetLastError());
}

void launch_cg_dot_scalars(const double* p, const double* q, std::int64_t n, double* partials, unsigned int* ticket,
                           CgScalars* sc, cudaStream_t s) {
    std::int64_t g = (n + kThreads * 4 - 1) / (kThreads * 4);
    g = std::max<std::int64_t>(1, std::min<std::int64_t>(g, std::min(kMaxParts, 148 * 8)));
    k_cg_dot_scalars<<<static_cast<unsigned>(g), kThreads, 0, s>>>(p, q, n, partials, ticket, sc);
    B200_CUDA(cudaGetLastError());
}

void cg_launch_fin(CgFin what, CgScalars* sc, const double* gathered, int nranks, double shift, cudaStream_t s) {
    k_cg_fin<<<1, 32, 0, s>>>(static_cast<int>(what), sc, gathered, nranks, shift);
    B200_CUDA(cudaGetLastError());
}

void cg_launch_spmv_dot(const CsrDev& A, const CgVectors& v, cudaStream_t s) {
    launch_spmv_csr_dot(A, v.p_full, v.q, v.partials, &v.sc->ticket[0], v.sc, s, v.row0);
}

void cg_launch_update_zr(const CgVectors& v, cudaStream_t s) {
    launch_pdl(k_cg_update_zr, dim3(vec_grid(v)), dim3(kThreads), 0, s, v);
}

void cg_launch_update_p(const CgVectors& v, cudaStream_t s) {
    launch_pdl(k_cg_update_p, dim3(vec_grid(v)), dim3(kThreads), 0, s, v);
}

void cg_launch_norms(const CgVectors& v, double shift, cudaStream_t s) {
    k_cg_norms<<<vec_grid(v), kThreads, 0, s>>>(v, shift);
    B200_CUDA(cudaGetLastError());
}

void cg_launch_scale_x(const CgVectors& v, cudaStream_t s) {
    k_cg_scale_x<<<vec_grid(v), kThreads, 0, s>>>(v);
    B200_CUDA(cudaGetLastError());
}

void cg_launch_resid_partial(const CgVectors& v, cudaStream_t s) {
    k_cg_resid<<<vec_grid(v), kThreads, 0, s>>>(v);
    B200_CUDA(cudaGetLastError());
}

void cg_launch_iteration(const CsrDev& A, const CgVectors& v, cudaStream_t s) {
    cg_launch_spmv_dot(A, v, s);
    cg_launch_update_zr(v, s);
    cg_launch_update_p(v, s);
}

void cg_launch_iterations(const CsrDev& A, const CgVectors& v, int steps, cudaStream_t s) {
    if (A.tiled && launch_cg_tiled(*A.tiled, v, steps, s)) return;
    for (int it = 0; it < steps; ++it) cg_launch_iteration(A, v, s);
}

void cg_launch_residual(const CsrDev& A, const CgVectors& v, cudaStream_t s) {
    launch_spmv_csr(A, v.z_full, v.r, CsrKernel::Auto, s);
    k_cg_resid<<<vec_grid(v), kThreads, 0, s>>>(v);
    B200_CUDA(cudaGetLastError());
}

void cg_launch_outer_update(const CgVectors& v, double shift, cudaStream_t s) {
    k_cg_norms<<<vec_grid(v), kThreads, 0, s>>>(v, shift);
    k_cg_scale_x<<<vec_grid(v), kThreads, 0, s>>>(v);
    B200_CUDA(cudaGetLastError());
}

void cg_launch_reset_x(const CgVectors& v, cudaStream_t s) {
    k_cg_fill<<<vec_grid(v), kThreads, 0, s>>>(v.x, v.n, 1.0);
    B200_CUDA(cudaGetLastError());
}

}  // namespace b200
