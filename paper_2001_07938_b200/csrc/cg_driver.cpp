// cg_driver.cpp — NPB CG benchmark driver over a resident CSR matrix
// (section 5 of include/lilac_b200.h). Restates NPB 3.x cg's main loop and
// conj_grad (cgitmax = 25) on the device; one outer iteration is captured
// once as a CUDA graph and replayed, so the host issues one launch per NPB
// iteration instead of ~80.

#include "lilac_b200.h"
#include "runtime.hpp"

#include <memory>

using namespace b200;

namespace b200 {
const CsrDev* matrix_csr(const b200_matrix* A);
}

struct b200_cg {
    CsrDev A;
    DevBuf x, z, p, q, r, partials, scalars;
    CgVectors v{};
    cudaGraphExec_t graph = nullptr;
    int graph_cgitmax = -1;
    double graph_shift = 0.0;
};

namespace {

cudaStream_t pick(void* stream) {
    return stream ? static_cast<cudaStream_t>(stream) : rt().stream;
}

void record_outer(b200_cg* cg, int cgitmax, double shift, cudaStream_t s) {
    cg_launch_init(cg->v, s);
    cg_launch_iterations(cg->A, cg->v, cgitmax, s);
    cg_launch_residual(cg->A, cg->v, s);
    cg_launch_outer_update(cg->v, shift, s);
}

void build_graph(b200_cg* cg, int cgitmax, double shift, cudaStream_t s) {
    if (cg->graph && cg->graph_cgitmax == cgitmax && cg->graph_shift == shift) return;
    if (cg->graph) {
        cudaGraphExecDestroy(cg->graph);
        cg->graph = nullptr;
    }
    cudaGraph_t g = nullptr;
    B200_CUDA(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
    try {
        record_outer(cg, cgitmax, shift, s);
    } catch (...) {
        cudaStreamEndCapture(s, &g);
        if (g) cudaGraphDestroy(g);
        throw;
    }
    B200_CUDA(cudaStreamEndCapture(s, &g));
    cudaError_t e = cudaGraphInstantiate(&cg->graph, g, 0);
    cudaGraphDestroy(g);
    if (e != cudaSuccess) throw_cuda(e, "cudaGraphInstantiate", __FILE__, __LINE__);
    cg->graph_cgitmax = cgitmax;
    cg->graph_shift = shift;
}

}  // namespace

extern "C" {

int b200_cg_create(b200_cg** out, const b200_matrix* Am) {
    return boundary("b200_cg_create", [&] {
        ensure_init();
        const CsrDev* A = matrix_csr(Am);
        if (!A) throw Error(Errc::DataError, "CG needs a CSR matrix");
        if (A->cols > A->rows) throw Error(Errc::DataError, "CG needs a square matrix (cols <= rows)");
        auto cg = std::make_unique<b200_cg>();
        cg->A = *A;
        const std::size_t bytes = sizeof(double) * static_cast<std::size_t>(A->rows);
        for (DevBuf* b : {&cg->x, &cg->z, &cg->p, &cg->q, &cg->r}) b->ensure(bytes);
        cg->partials.ensure(sizeof(double) * kMaxParts * 4);
        cg->scalars.ensure(sizeof(CgScalars));
        B200_CUDA(cudaMemsetAsync(cg->scalars.ptr, 0, sizeof(CgScalars), rt().stream));
        cg->v.n = A->rows;
        cg->v.x = cg->x.as<double>();
        cg->v.z = cg->z.as<double>();
        cg->v.p = cg->p.as<double>();
        cg->v.q = cg->q.as<double>();
        cg->v.r = cg->r.as<double>();
        cg->v.p_full = cg->v.p;
        cg->v.z_full = cg->v.z;
        cg->v.row0 = 0;
        cg->v.partials = cg->partials.as<double>();
        cg->v.sc = cg->scalars.as<CgScalars>();
        cg_launch_reset_x(cg->v, rt().stream);
        B200_CUDA(cudaStreamSynchronize(rt().stream));
        *out = cg.release();
    });
}

void b200_cg_free(b200_cg* cg) {
    if (!cg) return;
    device_quiesce();  // caller-stream work may still use the buffers (see b200_matrix_free)
    if (cg->graph) cudaGraphExecDestroy(cg->graph);
    for (DevBuf* b : {&cg->x, &cg->z, &cg->p, &cg->q, &cg->r, &cg->partials, &cg->scalars}) b->release();
    delete cg;
}

int b200_cg_reset(b200_cg* cg, void* stream) {
    return boundary("b200_cg_reset", [&] { cg_launch_reset_x(cg->v, pick(stream)); });
}

int b200_cg_outer(b200_cg* cg, int cgitmax, double shift, void* stream) {
    return boundary("b200_cg_outer", [&] {
        cudaStream_t s = pick(stream);
        build_graph(cg, cgitmax, shift, s);
        B200_CUDA(cudaGraphLaunch(cg->graph, s));
    });
}

int b200_cg_step(b200_cg* cg, void* stream) {
    return boundary("b200_cg_step", [&] { cg_launch_iteration(cg->A, cg->v, pick(stream)); });
}

int b200_cg_start(b200_cg* cg, const double* b_device, void* stream) {
    return boundary("b200_cg_start", [&] {
        cudaStream_t s = pick(stream);
        const std::size_t bytes = sizeof(double) * static_cast<std::size_t>(cg->v.n);
        if (b_device && bytes) B200_CUDA(cudaMemcpyAsync(cg->v.x, b_device, bytes, cudaMemcpyDeviceToDevice, s));
        cg_launch_init(cg->v, s);  // z = 0, r = p = b, rho = r.r
    });
}

int b200_cg_finish(b200_cg* cg, void* stream) {
    return boundary("b200_cg_finish", [&] { cg_launch_residual(cg->A, cg->v, pick(stream)); });
}

int b200_cg_scalars(b200_cg* cg, void* stream, double* rho, double* rnorm) {
    return boundary("b200_cg_scalars", [&] {
        cudaStream_t s = pick(stream);
        CgScalars sc;
        B200_CUDA(cudaMemcpyAsync(&sc, cg->v.sc, sizeof sc, cudaMemcpyDeviceToHost, s));
        B200_CUDA(cudaStreamSynchronize(s));
        if (rho) *rho = sc.rho;
        if (rnorm) *rnorm = sc.rnorm;
    });
}

int b200_cg_result(b200_cg* cg, double* zeta, double* rnorm) {
    return boundary("b200_cg_result", [&] {
        CgScalars sc;
        B200_CUDA(cudaDeviceSynchronize());
        B200_CUDA(cudaMemcpy(&sc, cg->v.sc, sizeof sc, cudaMemcpyDeviceToHost));
        if (zeta) *zeta = sc.zeta;
        if (rnorm) *rnorm = sc.rnorm;
    });
}

int b200_cg_solve(b200_cg* cg, const double* b, int iters, double* z_out, double* rnorm) {
    return boundary("b200_cg_solve", [&] {
        if (iters < 0) throw Error(Errc::DataError, "iters < 0");
        cudaStream_t s = rt().stream;
        const std::size_t bytes = sizeof(double) * static_cast<std::size_t>(cg->v.n);
        if (bytes) B200_CUDA(cudaMemcpyAsync(cg->v.x, b, bytes, cudaMemcpyDeviceToDevice, s));
        cg_launch_init(cg->v, s);  // z = 0, r = p = b
        cg_launch_iterations(cg->A, cg->v, iters, s);
        cg_launch_residual(cg->A, cg->v, s);  // |b - A z|
        if (z_out && bytes) B200_CUDA(cudaMemcpyAsync(z_out, cg->v.z, bytes, cudaMemcpyDeviceToDevice, s));
        B200_CUDA(cudaStreamSynchronize(s));
        CgScalars sc;
        B200_CUDA(cudaMemcpy(&sc, cg->v.sc, sizeof sc, cudaMemcpyDeviceToHost));
        if (rnorm) *rnorm = sc.rnorm;
    });
}

int b200_npb_cg(b200_cg* cg, int niter, double shift, double* zeta, double* rnorm) {
    return boundary("b200_npb_cg", [&] {
        cudaStream_t s = rt().stream;
        cg_launch_reset_x(cg->v, s);
        build_graph(cg, 25, shift, s);
        B200_CUDA(cudaGraphLaunch(cg->graph, s));  // NPB's untimed warm-up iteration
        cg_launch_reset_x(cg->v, s);
        for (int it = 0; it < niter; ++it) B200_CUDA(cudaGraphLaunch(cg->graph, s));
        B200_CUDA(cudaStreamSynchronize(s));
        CgScalars sc;
        B200_CUDA(cudaMemcpy(&sc, cg->v.sc, sizeof sc, cudaMemcpyDeviceToHost));
        if (zeta) *zeta = sc.zeta;
        if (rnorm) *rnorm = sc.rnorm;
    });
}

}  // extern "C"
