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
#include <cstdlib>

namespace b200 {

namespace {

constexpr unsigned kFull = 0xffffffffu;
constexpr unsigned kSent = 0xffffu;  // sentinel tile-local row (> kMaxTileRows)
constexpr std::size_t kTileSmem = sizeof(double) * (2 * kSlabW + kMaxTileRows);
#ifndef B200_TILED_PREFETCH
#define B200_TILED_PREFETCH 1
#endif
constexpr int kPrefetch = B200_TILED_PREFETCH;  // chunks in flight beyond the one being reduced

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

// 256-bit load (sm_100): one instruction moves a lane's 32 contiguous bytes,
// so a warp instruction covers 1 KB with every sector fully used.
__device__ __forceinline__ void ld_stream_f64x4(const double* p, double2& a, double2& b) {
    asm("ld.global.nc.L1::no_allocate.v4.f64 {%0, %1, %2, %3}, [%4];"
        : "=d"(a.x), "=d"(a.y), "=d"(b.x), "=d"(b.y)
        : "l"(p));
}

__device__ __forceinline__ uint4 ld_stream_u32x4(const std::uint32_t* p) {
    uint4 r;
    asm("ld.global.nc.L1::no_allocate.v4.u32 {%0, %1, %2, %3}, [%4];"
        : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
        : "l"(p));
    return r;
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
    return v;
}

__device__ __forceinline__ int slab_len(const TcsrDev& T, int k) {
    const long long rem = static_cast<long long>(T.cols - static_cast<std::int64_t>(k) * kSlabW);
    return static_cast<int>(rem < kSlabW ? rem : kSlabW);
}

// Start the copy of slab k of x into `xs` through the bulk-copy engine
// (16-byte granules). An odd last column is stored by this thread before its
// arrive (release) on the slab's mbarrier, so every consumer's wait (acquire)
// sees it together with the bulk bytes. x is never read past cols.
__device__ __forceinline__ void issue_slab(const TcsrDev& T, const double* __restrict__ x, double* xs, int k,
                                           std::uint64_t* mbar) {
    const int len = slab_len(T, k);
    const int even = len & ~1;
    const double* src = x + static_cast<std::int64_t>(k) * kSlabW;
    if (len & 1) xs[even] = src[even];
    mbar_arrive_tx(mbar, static_cast<unsigned>(even) * 8u);
    if (even) bulk_g2s(xs, src, static_cast<unsigned>(even) * 8u, mbar);
}

__device__ __forceinline__ double lds_f64(std::uint32_t addr) {
    double v;
    asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(addr));
    return v;
}

__device__ __forceinline__ void sts_add_f64(std::uint32_t addr, double v) {
    double o;
    asm volatile("ld.shared.f64 %0, [%1];" : "=d"(o) : "r"(addr));
    asm volatile("st.shared.f64 [%0], %1;" ::"r"(addr), "d"(o + v));
}

struct Chunk {
    double2 v0, v1;
    uint4 k;
};

// A lane's four consecutive nonzeros of a (slab, warp) run, tile-relative
// index j (predicated on j < hi; over-reads stay inside the padded arrays).
__device__ __forceinline__ Chunk load_chunk(const double* vb, const std::uint32_t* kb, int j, int hi) {
    Chunk c;
    if (j < hi) {
        ld_stream_f64x4(vb + j, c.v0, c.v1);
        c.k = ld_stream_u32x4(kb + j);
    } else {
        c.v0 = c.v1 = make_double2(0.0, 0.0);
        c.k = make_uint4(0, 0, 0, 0);
    }
    return c;
}

// One 128-nonzero piece, after the lane-local pass: lane holds its head run
// (k0, p0) and tail run (k1, p1) (k0 == k1: a single run, value p1). Row keys
// are non-decreasing across lanes. Adds every row's piece-sum into yp[row]
// (rows are owned by this warp).
__device__ __forceinline__ void reduce_piece(unsigned k0, double p0, unsigned k1, double p1, int lane,
                                             std::uint32_t yp_s) {
    const bool split = k0 != k1;
    double s = p1;
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
    if (split && k0 != kSent) sts_add_f64(yp_s + 8u * k0, (lane > 0 && pk == k0) ? p0 + ps : p0);
    if ((lane == 31 || nk0 != k1) && k1 != kSent) sts_add_f64(yp_s + 8u * k1, s);
}

// Lane-local pass over 4 consecutive nonzeros (keys non-decreasing): rows
// strictly inside the lane are exclusive to it and flushed here; the head and
// tail runs go to the warp-level reduce_piece.
__device__ __forceinline__ void lane_runs(const unsigned (&key)[4], const double (&p)[4], int lane,
                                          std::uint32_t yp_s) {
    double acc = p[0], head = 0.0;
    unsigned rk = key[0];
#pragma unroll
    for (int e = 1; e < 4; ++e) {
        if (key[e] == rk) {
            acc += p[e];
        } else {
            if (rk == key[0])
                head = acc;
            else if (rk != kSent)
                sts_add_f64(yp_s + 8u * rk, acc);
            rk = key[e];
            acc = p[e];
        }
    }
    reduce_piece(key[0], head, rk, acc, lane, yp_s);
}

// Processes a (slab, warp) run [lo, hi) (tile-relative) against the slab in
// shared memory at xb_s. Interior chunks take an unmasked fast path; the first
// and last chunk of a run mask elements outside [lo, hi).
template <int PF, int MODE>
__device__ __forceinline__ void process_run(const double* vb, const std::uint32_t* kb, int mis, int lo, int hi,
                                            std::uint32_t xb_s, std::uint32_t yp_s, int lane) {
    // 32-byte alignment is absolute: `mis` = tile base mod 4
    const int c0 = ((lo + mis) & ~3) - mis;
    Chunk q[PF + 1];
#pragma unroll
    for (int i = 0; i < PF; ++i) q[i] = load_chunk(vb, kb, c0 + 128 * i + 4 * lane, hi);
    for (int c = c0; c < hi; c += 128) {
        q[PF] = load_chunk(vb, kb, c + 128 * PF + 4 * lane, hi);  // prefetch PF chunks ahead
        const Chunk cur = q[0];
#pragma unroll
        for (int i = 0; i < PF; ++i) q[i] = q[i + 1];
        const double ev[4] = {cur.v0.x, cur.v0.y, cur.v1.x, cur.v1.y};
        const unsigned kw[4] = {cur.k.x, cur.k.y, cur.k.z, cur.k.w};
        unsigned key[4];
        double p[4];
        if (c >= lo && c + 128 <= hi) {  // warp-uniform: every element valid
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const double xv = (MODE == 1 || MODE == 3) ? 1.0 : lds_f64(xb_s + 8u * (kw[e] & 0xffffu));
                key[e] = kw[e] >> 16;
                p[e] = ev[e] * xv;
            }
        } else {
            const int j = c + 4 * lane;
            const int front = lo - j, back = hi - j;  // element e valid iff front <= e < back
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const double xv = (MODE == 1 || MODE == 3) ? 1.0 : lds_f64(xb_s + 8u * (kw[e] & 0xffffu));
                key[e] = e < back ? kw[e] >> 16 : kSent;
                p[e] = (e >= front && e < back) ? ev[e] * xv : 0.0;
            }
            // leading elements before lo (first chunk, lane 0) take the next key
#pragma unroll
            for (int e = 2; e >= 0; --e)
                if (e < front) key[e] = key[e + 1];
        }
        if (MODE >= 2) {
            if (p[0] == 12345.678) sts_add_f64(yp_s, p[1]);  // probe: no reduction
        } else {
            lane_runs(key, p, lane, yp_s);
        }
    }
}

template <bool DOT, int PF, int MODE = 0>
__global__ void __launch_bounds__(kTileThreads, 1)
    k_spmv_tiled(TcsrDev T, const double* __restrict__ x, double* __restrict__ y, double* partials,
                 unsigned int* ticket, CgScalars* sc) {
    extern __shared__ __align__(128) double smem[];
    double* xs = smem;               // [2][kSlabW]
    double* yp = smem + 2 * kSlabW;  // [kMaxTileRows]
    __shared__ __align__(8) std::uint64_t mbar[2];
    __shared__ unsigned released[2];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const std::uint32_t xs_s = smem_addr(xs), yp_s = smem_addr(yp);

    if (tid == 0) {
        released[0] = released[1] = 0;
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
        const double* vb = T.val + base;
        const std::uint32_t* kb = T.key + base;
        const std::int32_t* wo = T.woff + t * (static_cast<std::int64_t>(T.nslabs) * kTileWarps + 1);
        for (int r = tid; r < nrows; r += kTileThreads) yp[r] = 0.0;
        if (tid == 0 && T.nslabs > 0 && MODE < 5) {
            issue_slab(T, x, xs, 0, &mbar[0]);
            if (T.nslabs > 1) issue_slab(T, x, xs + kSlabW, 1, &mbar[1]);
        }
        __syncthreads();
        // Free-running slabs: a warp moves on as soon as the next slab has
        // landed; the last warp to release a buffer refills it (no CTA barrier).
        for (int k = 0; k < T.nslabs; ++k) {
            const int buf = k & 1;
            if (MODE >= 5) {
            } else if (buf == 0) {
                mbar_wait(&mbar[0], phase0);
                phase0 ^= 1;
            } else {
                mbar_wait(&mbar[1], phase1);
                phase1 ^= 1;
            }
            process_run<PF, MODE == 5 ? 3 : (MODE == 6 ? 0 : MODE)>(
                vb, kb, static_cast<int>(base & 3), wo[k * kTileWarps + warp], wo[k * kTileWarps + warp + 1],
                xs_s + 8u * static_cast<unsigned>(buf * kSlabW), yp_s, lane);
            __syncwarp();
            if (lane == 0) {
                __threadfence_block();
                if (atomicAdd(&released[buf], 1u) == kTileWarps - 1) {
                    released[buf] = 0;
                    if (k + 2 < T.nslabs && MODE < 5) issue_slab(T, x, xs + buf * kSlabW, k + 2, &mbar[buf]);
                }
            }
        }
        __syncthreads();  // every row of the tile is complete
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

template <int MODE, int PF>
void launch_probe(const TcsrDev& T, const double* x, double* y, unsigned grid, cudaStream_t s) {
    static bool configured = false;
    if (!configured) {
        B200_CUDA(cudaFuncSetAttribute(k_spmv_tiled<false, PF, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(kTileSmem)));
        configured = true;
    }
    k_spmv_tiled<false, PF, MODE><<<grid, kTileThreads, kTileSmem, s>>>(T, x, y, nullptr, nullptr, nullptr);
}

template <int PF>
void launch_pf(const TcsrDev& T, const double* x, double* y, double* partials, unsigned int* ticket, CgScalars* sc,
               unsigned grid, cudaStream_t s) {
    static bool configured = false;
    if (!configured) {
        B200_CUDA(cudaFuncSetAttribute(k_spmv_tiled<false, PF>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(kTileSmem)));
        B200_CUDA(cudaFuncSetAttribute(k_spmv_tiled<true, PF>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(kTileSmem)));
        configured = true;
    }
    if (partials)
        k_spmv_tiled<true, PF><<<std::min<unsigned>(grid, kMaxParts), kTileThreads, kTileSmem, s>>>(T, x, y, partials,
                                                                                                   ticket, sc);
    else
        k_spmv_tiled<false, PF><<<grid, kTileThreads, kTileSmem, s>>>(T, x, y, nullptr, nullptr, nullptr);
}

void launch_spmv_tiled(const TcsrDev& T, std::int64_t rows, const double* x, double* y, double* partials,
                       unsigned int* ticket, CgScalars* sc, cudaStream_t s) {
    static int pf = -1;
    if (pf < 0) {
        int dev = 0;
        B200_CUDA(cudaGetDevice(&dev));
        B200_CUDA(cudaDeviceGetAttribute(&g_sms, cudaDevAttrMultiProcessorCount, dev));
        const char* e = std::getenv("LILAC_B200_TILED_PF");
        pf = (e && *e) ? std::atoi(e) : kPrefetch;
    }
    if (rows <= 0 || T.ntiles <= 0) return;
    const unsigned grid = static_cast<unsigned>(std::min<std::int64_t>(T.ntiles, g_sms));
    static int mode = -1;
    if (mode < 0) {
        const char* e = std::getenv("LILAC_B200_TILED_PROBE");  // timing probes only: wrong results
        mode = (e && *e) ? std::atoi(e) : 0;
    }
    if (mode == 1 && !partials) launch_probe<1, 1>(T, x, y, grid, s);
    else if (mode == 2 && !partials) launch_probe<2, 1>(T, x, y, grid, s);
    else if (mode == 3 && !partials) launch_probe<3, 1>(T, x, y, grid, s);
    else if (mode == 4 && !partials) launch_probe<3, 2>(T, x, y, grid, s);
    else if (mode == 5 && !partials) launch_probe<5, 1>(T, x, y, grid, s);
    else if (mode == 6 && !partials) launch_probe<6, 1>(T, x, y, grid, s);
    else if (pf >= 2)
        launch_pf<2>(T, x, y, partials, ticket, sc, grid, s);
    else
        launch_pf<1>(T, x, y, partials, ticket, sc, grid, s);
    B200_CUDA(cudaGetLastError());
}

}  // namespace b200
