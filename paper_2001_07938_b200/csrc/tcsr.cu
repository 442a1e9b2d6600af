// tcsr.cu — tiled CSR SpMV for matrices whose x gathers have no locality.
//
// Why: with random columns (NPB CG) the plain vector kernel is bound by the
// L1TEX pipe, not HBM — every warp-wide x gather touches ~32 distinct sectors
// (32 wavefronts), ncu: l1tex 88.7% busy at 45% of HBM peak (profiles/). Here
// x is staged in shared memory one column slab at a time (cp.async.bulk into a
// double buffer, completion on an mbarrier), so a gather costs a few bank
// cycles instead of 32 L1 wavefronts, while val/key stream from HBM with
// fully coalesced 16-byte loads.
//
// One CTA (32 warps) per tile; warp w owns a contiguous row range of the tile.
// For each slab the warp streams its contiguous (slab, warp) run two nonzeros
// per lane, gathers x from smem, and reduces by row with a shuffle-based
// segmented scan; row partials accumulate in a shared y buffer (rows are owned
// by one warp: no atomics, deterministic order). y is written once per tile.

#include "b200.hpp"

#include <algorithm>

namespace b200 {

namespace {

constexpr unsigned kFull = 0xffffffffu;
constexpr unsigned kSent = 0xffffu;  // sentinel tile-local row (> kMaxTileRows)
constexpr std::size_t kTileSmem = sizeof(double) * (2 * kSlabW + kMaxTileRows);

__device__ __forceinline__ std::uint32_t smem_addr(const void* p) {
    return static_cast<std::uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(std::uint64_t* b, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(b)), "r"(count) : "memory");
}

__device__ __forceinline__ void mbar_arrive_tx(std::uint64_t* b, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(b)), "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ void mbar_wait(std::uint64_t* b, unsigned parity) {
    asm volatile(
        "{\n\t.reg .pred P1;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
        "@P1 bra DONE_%=;\n\t"
        "bra WAIT_%=;\n"
        "DONE_%=:\n\t}" ::"r"(smem_addr(b)),
        "r"(parity)
        : "memory");
}

__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, std::uint64_t* b) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_addr(dst)),
                 "l"(src), "r"(bytes), "r"(smem_addr(b))
                 : "memory");
}

__device__ __forceinline__ double2 ld_stream_f64x2(const double* p) {
    double2 r;
    asm("ld.global.nc.L1::no_allocate.v2.f64 {%0, %1}, [%2];" : "=d"(r.x), "=d"(r.y) : "l"(p));
    return r;
}

__device__ __forceinline__ uint2 ld_stream_u32x2(const std::uint32_t* p) {
    uint2 r;
    asm("ld.global.nc.L1::no_allocate.v2.u32 {%0, %1}, [%2];" : "=r"(r.x), "=r"(r.y) : "l"(p));
    return r;
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
    return v;
}

// Thread 0: start the copy of slab k of x into buffer `buf`. The even part
// goes through the bulk-copy engine (16-byte granules); an odd last column is
// stored by thread 0 itself and becomes visible at the next __syncthreads.
__device__ __forceinline__ void issue_slab(const TcsrDev& T, const double* __restrict__ x, double* xs, int k,
                                           std::uint64_t* mbar) {
    const std::int64_t c0 = static_cast<std::int64_t>(k) * kSlabW;
    const long long rem = static_cast<long long>(T.cols - c0);
    const int len = static_cast<int>(rem < kSlabW ? rem : kSlabW);
    const int even = len & ~1;
    mbar_arrive_tx(mbar, static_cast<unsigned>(even) * 8u);
    if (even) bulk_g2s(xs, x + c0, static_cast<unsigned>(even) * 8u, mbar);
    if (len & 1) xs[even] = x[c0 + even];
}

// One 64-nonzero piece: lane holds nonzeros (k0,p0), (k1,p1) with row keys
// non-decreasing across lanes. Adds every row's piece-sum into yp[row].
__device__ __forceinline__ void reduce_piece(unsigned k0, double p0, unsigned k1, double p1, int lane,
                                             double* yp) {
    const bool split = k0 != k1;
    double s = split ? p1 : p0 + p1;
    const unsigned pk = __shfl_up_sync(kFull, k1, 1);
    const bool head = lane == 0 || pk != k1;
    const unsigned hm = __ballot_sync(kFull, head);
    const int seg = 31 - __clz(hm & (kFull >> (31 - lane)));
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const double t = __shfl_up_sync(kFull, s, d);
        if (lane - d >= seg) s += t;
    }
    const double ps = __shfl_up_sync(kFull, s, 1);
    const unsigned nk0 = __shfl_down_sync(kFull, k0, 1);
    if (split && k0 != kSent) yp[k0] += (lane > 0 && pk == k0) ? p0 + ps : p0;
    if ((lane == 31 || nk0 != k1) && k1 != kSent) yp[k1] += s;
}

template <bool DOT>
__global__ void __launch_bounds__(kTileThreads, 1)
    k_spmv_tiled(TcsrDev T, const double* __restrict__ x, double* __restrict__ y, double* partials,
                 unsigned int* ticket, CgScalars* sc) {
    extern __shared__ __align__(128) double smem[];
    double* xs = smem;                   // [2][kSlabW]
    double* yp = smem + 2 * kSlabW;      // [kMaxTileRows]
    __shared__ __align__(8) std::uint64_t mbar[2];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;

    if (tid == 0) {
        mbar_init(&mbar[0], 1);
        mbar_init(&mbar[1], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    unsigned phase0 = 0, phase1 = 0;
    double pq = 0.0;

    for (std::int64_t t = blockIdx.x; t < T.ntiles; t += gridDim.x) {
        const std::int64_t row0 = T.tile_row0[t];
        const int nrows = static_cast<int>(T.tile_row0[t + 1] - row0);
        const std::int64_t base = T.tile_base[t];
        const std::int32_t* wo = T.woff + t * (static_cast<std::int64_t>(T.nslabs) * kTileWarps + 1);
        for (int r = tid; r < nrows; r += kTileThreads) yp[r] = 0.0;
        if (tid == 0 && T.nslabs > 0) {
            issue_slab(T, x, xs, 0, &mbar[0]);
            if (T.nslabs > 1) issue_slab(T, x, xs + kSlabW, 1, &mbar[1]);
        }
        __syncthreads();
        for (int k = 0; k < T.nslabs; ++k) {
            const int buf = k & 1;
            if (buf == 0) {
                mbar_wait(&mbar[0], phase0);
                phase0 ^= 1;
            } else {
                mbar_wait(&mbar[1], phase1);
                phase1 ^= 1;
            }
            const double* xb = xs + buf * kSlabW;
            const std::int64_t lo = base + wo[k * kTileWarps + warp];
            const std::int64_t hi = base + wo[k * kTileWarps + warp + 1];
            for (std::int64_t c = lo & ~std::int64_t(1); c < hi; c += 128) {
                double2 v[2];
                uint2 kk[2];
#pragma unroll
                for (int u = 0; u < 2; ++u) {
                    const std::int64_t j = c + 64 * u + 2 * lane;
                    if (j < hi) {
                        v[u] = ld_stream_f64x2(T.val + j);
                        kk[u] = ld_stream_u32x2(T.key + j);
                    } else {
                        v[u] = make_double2(0.0, 0.0);
                        kk[u] = make_uint2(kSent << 16, kSent << 16);
                    }
                }
#pragma unroll
                for (int u = 0; u < 2; ++u) {
                    const std::int64_t j = c + 64 * u + 2 * lane;
                    unsigned k0 = kk[u].x >> 16, k1 = kk[u].y >> 16;
                    double p0 = 0.0, p1 = 0.0;
                    if (j + 1 >= hi) k1 = kSent;          // second element past the run
                    if (j < lo) k0 = k1;                  // first element before the run
                    else if (k0 != kSent) p0 = v[u].x * xb[kk[u].x & 0xffffu];
                    if (k1 != kSent) p1 = v[u].y * xb[kk[u].y & 0xffffu];
                    reduce_piece(k0, p0, k1, p1, lane, yp);
                }
            }
            __syncthreads();  // every warp is done with xs[buf]
            if (tid == 0 && k + 2 < T.nslabs) issue_slab(T, x, xs + buf * kSlabW, k + 2, &mbar[buf]);
        }
        for (int r = tid; r < nrows; r += kTileThreads) {
            const double v = yp[r];
            y[row0 + r] = v;
            if (DOT) pq += v * __ldg(x + row0 + r);
        }
        __syncthreads();  // yp reused by the next tile
    }

    if (DOT) {
        __shared__ double red[kTileWarps];
        __shared__ bool last;
        double s = warp_sum(pq);
        if (lane == 0) red[warp] = s;
        __syncthreads();
        if (warp == 0) {
            s = warp_sum(red[lane]);
            if (lane == 0) partials[blockIdx.x] = s;
        }
        __threadfence();
        __syncthreads();
        if (tid == 0) last = atomicAdd(ticket, 1u) == gridDim.x - 1;
        __syncthreads();
        if (last) {
            __threadfence();
            double a = 0.0;
            for (unsigned i = tid; i < gridDim.x; i += kTileThreads) a += __ldcg(partials + i);
            a = warp_sum(a);
            __syncthreads();
            if (lane == 0) red[warp] = a;
            __syncthreads();
            if (warp == 0) {
                a = warp_sum(red[lane]);
                if (lane == 0) {
                    sc->d = a;
                    sc->rho0 = sc->rho;
                    sc->alpha = sc->rho / a;
                    *ticket = 0u;
                }
            }
        }
    }
}

int g_sms = 0;

}  // namespace

void launch_spmv_tiled(const TcsrDev& T, std::int64_t rows, const double* x, double* y, double* partials,
                       unsigned int* ticket, CgScalars* sc, cudaStream_t s) {
    static bool configured = false;
    if (!configured) {
        B200_CUDA(cudaFuncSetAttribute(k_spmv_tiled<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(kTileSmem)));
        B200_CUDA(cudaFuncSetAttribute(k_spmv_tiled<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(kTileSmem)));
        int dev = 0;
        B200_CUDA(cudaGetDevice(&dev));
        B200_CUDA(cudaDeviceGetAttribute(&g_sms, cudaDevAttrMultiProcessorCount, dev));
        configured = true;
    }
    if (rows <= 0 || T.ntiles <= 0) return;
    const unsigned grid = static_cast<unsigned>(std::min<std::int64_t>(T.ntiles, g_sms));
    if (partials) {
        const unsigned g = std::min<unsigned>(grid, kMaxParts);
        k_spmv_tiled<true><<<g, kTileThreads, kTileSmem, s>>>(T, x, y, partials, ticket, sc);
    } else {
        k_spmv_tiled<false><<<grid, kTileThreads, kTileSmem, s>>>(T, x, y, nullptr, nullptr, nullptr);
    }
    B200_CUDA(cudaGetLastError());
}

}  // namespace b200
