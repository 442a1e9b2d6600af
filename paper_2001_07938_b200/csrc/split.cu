// split.cu — CSR SpMV for skewed row lengths (power-law graphs): the vector
// kernel on the short rows, one warp per <= kSplitChunk-nonzero chunk of each
// long row, and a per-row sum of the chunk partials in chunk order.
//
// Why not only merge-path (merge.cu): on the Kronecker scale-22 operator the
// merge kernel is bound by shared-memory latency (per-thread binary searches
// and the sequential merge walk; ncu: short_scoreboard + mio_throttle stalls,
// 21% issue, profiles/r01_kron_merge.md) at 0.92 ms; here a short row costs
// what it costs in the vector kernel and a long row is spread over many warps.
// Deterministic: every sum is taken in a fixed order.

#include "b200.hpp"
#include "ldst.cuh"

#include <algorithm>

namespace b200 {

namespace {

constexpr int kThreads = 256;
constexpr int kSMs = 148;
constexpr int kChunkU = 8;  // loads in flight per lane

template <typename IdxT>
__global__ void __launch_bounds__(kThreads) k_csr_chunks(std::int64_t nchunks, const std::int64_t* __restrict__ lo_,
                                                         const std::int64_t* __restrict__ hi_,
                                                         const IdxT* __restrict__ col,
                                                         const double* __restrict__ val,
                                                         const double* __restrict__ x, double* __restrict__ part) {
    const int lane = threadIdx.x & 31;
    const std::int64_t warps = static_cast<std::int64_t>(gridDim.x) * (kThreads / 32);
    const std::uint64_t pstream = policy_evict_first(), pgather = policy_evict_last();
    for (std::int64_t c = (static_cast<std::int64_t>(blockIdx.x) * kThreads + threadIdx.x) / 32; c < nchunks;
         c += warps) {
        const std::int64_t lo = __ldg(lo_ + c), hi = __ldg(hi_ + c);
        double acc = 0.0;
        for (std::int64_t jb = lo + lane; jb < hi; jb += 32 * kChunkU) {
            std::int64_t cc[kChunkU];
            double vv[kChunkU];
#pragma unroll
            for (int u = 0; u < kChunkU; ++u) {
                const std::int64_t j = jb + 32 * u;
                cc[u] = j < hi ? ld_stream_idx(col + j, pstream) : 0;
                vv[u] = j < hi ? ld_stream_f64(val + j, pstream) : 0.0;
            }
#pragma unroll
            for (int u = 0; u < kChunkU; ++u) {
                const std::int64_t j = jb + 32 * u;
                if (j < hi) acc += vv[u] * ld_gather_f64(x + cc[u], pgather);
            }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
        if (lane == 0) part[c] = acc;
    }
}

__global__ void k_split_fix(std::int64_t nlong, const std::int64_t* __restrict__ rows,
                            const std::int64_t* __restrict__ first, const double* __restrict__ part,
                            double* __restrict__ y) {
    const std::int64_t i = static_cast<std::int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= nlong) return;
    double s = 0.0;
    for (std::int64_t c = first[i]; c < first[i + 1]; ++c) s += part[c];
    y[rows[i]] = s;
}

}  // namespace

void launch_spmv_split(const CsrDev& A, const double* x, double* y, cudaStream_t s) {
    const SplitDev& P = *A.split;
    if (A.rows <= 0) return;
    launch_csr_vector_short(A, x, y, P.short_max, s);
    if (P.nchunks > 0) {
        const unsigned g = static_cast<unsigned>(
            std::min<std::int64_t>((P.nchunks + kThreads / 32 - 1) / (kThreads / 32), kSMs * 16));
        if (A.col32)
            k_csr_chunks<std::int32_t><<<g, kThreads, 0, s>>>(P.nchunks, P.chunk_lo, P.chunk_hi,
                                                              static_cast<const std::int32_t*>(A.col), A.val, x,
                                                              P.partial);
        else
            k_csr_chunks<std::int64_t><<<g, kThreads, 0, s>>>(P.nchunks, P.chunk_lo, P.chunk_hi,
                                                              static_cast<const std::int64_t*>(A.col), A.val, x,
                                                              P.partial);
        k_split_fix<<<static_cast<unsigned>((P.nlong + 255) / 256), 256, 0, s>>>(P.nlong, P.long_rows, P.long_first,
                                                                                  P.partial, y);
    }
    B200_CUDA(cudaGetLastError());
}

}  // namespace b200
