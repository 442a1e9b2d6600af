// gemm.cu — the dense `gemm` computation of the reference's kernels.lilac
// (fixtures/lilac/kernels.lilac:14-19):
//   c[i*m + j] = dot (0 <= k < p) a[i*p + k] * b[k*m + j]   (row-major, f64)
// Two kernels: the exact one (one thread per output, k in the reference
// order, separate mul and add: bit-identical to what_interp.cpp) and the fast
// one on the FP64 tensor-core path (DMMA, mma.sync m8n8k4 f64 — f64 has no
// tcgen05 kind): 64 x 64 output tiles per CTA of 4 warps (32 x 32 each, 16
// accumulator tiles), 16-deep k slices staged in padded shared memory with
// the next slice's loads in flight in registers. Sums reassociate across k
// slices: within the north-star tolerance, not bit-exact.

#include "b200.hpp"

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

constexpr int kBM = 64, kBN = 64, kBK = 16;
constexpr int kGemmThreads = 128;  // 4 warps, 2 x 2 over the 64 x 64 tile
constexpr int kAStride = kBK + 1;  // padded rows: the 8 rows of an A fragment hit distinct banks
constexpr int kBStride = kBN + 4;

__device__ __forceinline__ void dmma(double (&d)[2], double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
                 : "+d"(d[0]), "+d"(d[1])
                 : "d"(a), "d"(b));
}

__global__ void __launch_bounds__(kGemmThreads) k_gemm_dmma(int n, int m, int p, const double* __restrict__ a,
                                                            const double* __restrict__ b, double* __restrict__ c) {
    __shared__ double As[kBM * kAStride];
    __shared__ double Bs[kBK * kBStride];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int wr = warp >> 1, wc = warp & 1;  // this warp's 32 x 32 quadrant
    const int i0 = blockIdx.y * kBM, j0 = blockIdx.x * kBN;
    const int g = lane >> 2, q = lane & 3;  // fragment coordinates (groupID, thread in group)
    double acc[4][4][2];
#pragma unroll
    for (int ti = 0; ti < 4; ++ti)
#pragma unroll
        for (int tj = 0; tj < 4; ++tj) acc[ti][tj][0] = acc[ti][tj][1] = 0.0;
    // each thread moves 8 elements of A (64 x 16) and 8 of B (16 x 64) per k slice
    double ra[8], rb[8];
    auto load = [&](int k0) {
#pragma unroll
        for (int e = 0; e < 8; ++e) {
            const int ia = e * kGemmThreads + tid;  // A: row ia / 16, col ia % 16
            const int r = ia / kBK, kk = ia % kBK;
            ra[e] = (i0 + r < n && k0 + kk < p) ? __ldg(a + static_cast<std::int64_t>(i0 + r) * p + k0 + kk) : 0.0;
            const int kb = ia / kBN, cc = ia % kBN;  // B: row ia / 64, col ia % 64
            rb[e] = (k0 + kb < p && j0 + cc < m) ? __ldg(b + static_cast<std::int64_t>(k0 + kb) * m + j0 + cc) : 0.0;
        }
    };
    auto store = [&]() {
#pragma unroll
        for (int e = 0; e < 8; ++e) {
            const int ia = e * kGemmThreads + tid;
            As[(ia / kBK) * kAStride + ia % kBK] = ra[e];
            Bs[(ia / kBN) * kBStride + ia % kBN] = rb[e];
        }
    };
    load(0);
    for (int k0 = 0; k0 < p; k0 += kBK) {
        __syncthreads();  // the previous slice's fragments are consumed
        store();
        __syncthreads();
        if (k0 + kBK < p) load(k0 + kBK);  // in flight during this slice's MMAs
#pragma unroll
        for (int kk = 0; kk < kBK; kk += 4) {
            double fa[4], fb[4];
#pragma unroll
            for (int t = 0; t < 4; ++t) {
                fa[t] = As[(wr * 32 + t * 8 + g) * kAStride + kk + q];  // A[row g][k q]
                fb[t] = Bs[(kk + q) * kBStride + wc * 32 + t * 8 + g];  // B[k q][col g]
            }
#pragma unroll
            for (int ti = 0; ti < 4; ++ti)
#pragma unroll
                for (int tj = 0; tj < 4; ++tj) dmma(acc[ti][tj], fa[ti], fb[tj]);
        }
    }
    // D fragment: row g, columns 2q and 2q+1 of each 8 x 8 tile
#pragma unroll
    for (int ti = 0; ti < 4; ++ti) {
        const int i = i0 + wr * 32 + ti * 8 + g;
        if (i >= n) continue;
#pragma unroll
        for (int tj = 0; tj < 4; ++tj) {
            const int j = j0 + wc * 32 + tj * 8 + 2 * q;
            if (j < m) c[static_cast<std::int64_t>(i) * m + j] = acc[ti][tj][0];
            if (j + 1 < m) c[static_cast<std::int64_t>(i) * m + j + 1] = acc[ti][tj][1];
        }
    }
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
    const dim3 grd(static_cast<unsigned>((m + kBN - 1) / kBN), static_cast<unsigned>((n + kBM - 1) / kBM));
    k_gemm_dmma<<<grd, kGemmThreads, 0, s>>>(static_cast<int>(n), static_cast<int>(m), static_cast<int>(p), a, b, c);
    B200_CUDA(cudaGetLastError());
}

}  // namespace b200
