// gemm.cu — the dense `gemm` computation of the reference's kernels.lilac
// (fixtures/lilac/kernels.lilac:14-19):
//   c[i*m + j] = dot (0 <= k < p) a[i*p + k] * b[k*m + j]   (row-major, f64)
// Two paths: the exact kernel (one thread per output, k in the reference
// order, separate mul and add: bit-identical to what_interp.cpp) and the fast
// path, cuBLAS DGEMM (a plain library GEMM; f64 has no tcgen05 kind), loaded
// with dlopen so the library does not depend on cuBLAS unless it is used.

#include "b200.hpp"

#include <dlfcn.h>

#include <mutex>

namespace b200 {

namespace {

constexpr int kTile = 16;

__global__ void k_gemm_exact(std::int64_t n, std::int64_t m, std::int64_t p, const double* __restrict__ a,
                             const double* __restrict__ b, double* __restrict__ c) {
    const std::int64_t j = static_cast<std::int64_t>(blockIdx.x) * kTile + threadIdx.x;
    const std::int64_t i = static_cast<std::int64_t>(blockIdx.y) * kTile + threadIdx.y;
    if (i >= n || j >= m) return;
    double acc = 0.0;
    for (std::int64_t k = 0; k < p; ++k) acc = __dadd_rn(acc, __dmul_rn(a[i * p + k], b[k * m + j]));
    c[i * m + j] = acc;
}

// cuBLAS entry points used (cublas_v2.h), resolved at first use.
using cublasHandle = void*;
struct CublasApi {
    void* lib = nullptr;
    int (*Create)(cublasHandle*) = nullptr;
    int (*SetStream)(cublasHandle, cudaStream_t) = nullptr;
    int (*Dgemm)(cublasHandle, int, int, int, int, int, const double*, const double*, int, const double*, int,
                 const double*, double*, int) = nullptr;
    cublasHandle handle = nullptr;
};

CublasApi& cublas() {
    static CublasApi api;
    static std::once_flag once;
    std::call_once(once, [] {
        for (const char* name : {"libcublas.so.12", "libcublas.so"}) {
            api.lib = dlopen(name, RTLD_NOW | RTLD_GLOBAL);
            if (api.lib) break;
        }
        if (!api.lib) return;
        api.Create = reinterpret_cast<decltype(api.Create)>(dlsym(api.lib, "cublasCreate_v2"));
        api.SetStream = reinterpret_cast<decltype(api.SetStream)>(dlsym(api.lib, "cublasSetStream_v2"));
        api.Dgemm = reinterpret_cast<decltype(api.Dgemm)>(dlsym(api.lib, "cublasDgemm_v2"));
        if (api.Create && api.Create(&api.handle) != 0) api.handle = nullptr;
    });
    if (!api.handle || !api.SetStream || !api.Dgemm)
        throw Error(Errc::DeviceError, "cuBLAS (libcublas.so.12) is not loadable: the fast gemm path needs it "
                                       "(b200_set_exact_blas(1) selects the exact kernel)");
    return api;
}

}  // namespace

void launch_gemm(std::int64_t n, std::int64_t m, std::int64_t p, const double* a, const double* b, double* c,
                 bool exact, cudaStream_t s) {
    if (n <= 0 || m <= 0) return;
    if (exact || p == 0) {
        const dim3 blk(kTile, kTile);
        const dim3 grd(static_cast<unsigned>((m + kTile - 1) / kTile), static_cast<unsigned>((n + kTile - 1) / kTile));
        k_gemm_exact<<<grd, blk, 0, s>>>(n, m, p, a, b, c);
        B200_CUDA(cudaGetLastError());
        return;
    }
    if (n > INT32_MAX || m > INT32_MAX || p > INT32_MAX) throw Error(Errc::DataError, "gemm extent exceeds int32");
    CublasApi& api = cublas();
    if (api.SetStream(api.handle, s) != 0) throw Error(Errc::DeviceError, "cublasSetStream failed");
    // row-major C = A B is column-major C^T = B^T A^T: (m x p)(p x n)
    const double one = 1.0, zero = 0.0;
    const int rc = api.Dgemm(api.handle, 0 /*N*/, 0 /*N*/, static_cast<int>(m), static_cast<int>(n),
                             static_cast<int>(p), &one, b, static_cast<int>(m), a, static_cast<int>(p), &zero, c,
                             static_cast<int>(m));
    if (rc != 0) throw Error(Errc::DeviceError, "cublasDgemm failed (status " + std::to_string(rc) + ")");
}

}  // namespace b200
