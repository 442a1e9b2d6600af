// tcsr.cu — tiled CSR SpMV for matrices whose x gathers have no locality.
//
// Why: with random columns (NPB CG) the plain vector kernel is bound by the
// L1TEX pipe, not HBM — every warp-wide x gather touches ~32 distinct sectors
// (32 wavefronts), ncu: l1tex 88.7% busy at 45% of HBM peak (profiles/). Here
// x is staged in shared memory one column slab at a time (cp.async.bulk into a
// double buffer, completion on an mbarrier), so a gather costs a few bank
// cycles instead of 32 L1 wavefronts, while val/key stream from HBM with
// fully coalesced 256-bit loads.
//
// One CTA (32 warps) per tile; warp w owns a contiguous row range of the tile.
// For each slab the warp streams its (slab, warp) run: each lane walks its own
// contiguous range of the run (layout in b200.hpp) chunk by chunk, gathers x
// from smem and sums rows in registers, flushing a row that began and ended
// inside the lane straight into a shared y buffer; the rows crossing lane
// boundaries are combined once per run by a shuffle-based segmented scan.
// Rows are owned by one warp: no atomics, deterministic order. y is written
// once per tile.

#include "b200.hpp"
#include "p2p.hpp"

#include <algorithm>
#include <cstdlib>

namespace b200 {

namespace {

constexpr unsigned kFull = 0xffffffffu;
#ifndef LILAC_PF_AHEAD
#define LILAC_PF_AHEAD 1
#endif
constexpr int kPfAhead = LILAC_PF_AHEAD;
constexpr std::size_t kTileSmem = sizeof(double) * (2 * kSlabStride + kMaxTileRows);

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

// x slabs are re-read by every tile: keep them in L2 (evict_last)
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, std::uint64_t* b) {
    std::uint64_t pol;
    asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
            smem_addr(dst)),
        "l"(src), "r"(bytes), "r"(smem_addr(b)), "l"(pol)
        : "memory");
}

// 256-bit load (sm_100): one instruction moves a lane's 32 contiguous bytes,
// so a warp instruction covers 1 KB with every sector fully used. The matrix
// is read once: L2 evict_first once consumed, so it does not push out x or the
// runs prefetched for the next slab.
__device__ __forceinline__ void ld_stream_f64x4(const double* p, double2& a, double2& b, std::uint64_t pol) {
    asm("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.f64 {%0, %1, %2, %3}, [%4], %5;"
        : "=d"(a.x), "=d"(a.y), "=d"(b.x), "=d"(b.y)
        : "l"(p), "l"(pol));
}

__device__ __forceinline__ uint2 ld_stream_u16x4(const std::uint16_t* p, std::uint64_t pol) {
    uint2 r;
    asm("ld.global.nc.L1::no_allocate.L2::cache_hint.v2.u32 {%0, %1}, [%2], %3;"
        : "=r"(r.x), "=r"(r.y)
        : "l"(p), "l"(pol));
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

// Asynchronous L2 prefetch of [p, p+bytes) by the bulk-copy engine: no
// registers, no completion tracking. Range widened to 16-byte granules.
__device__ __forceinline__ void prefetch_l2(const void* p, std::size_t bytes) {
    const std::uintptr_t a = reinterpret_cast<std::uintptr_t>(p) & ~std::uintptr_t(15);
    const std::uintptr_t e = (reinterpret_cast<std::uintptr_t>(p) + bytes + 15) & ~std::uintptr_t(15);
    if (e > a)
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(a), "r"(static_cast<unsigned>(e - a))
                     : "memory");
}

// Prefetch a (slab, warp) run's val and key bytes into L2.
__device__ __forceinline__ void prefetch_run(const double* vb, const std::uint16_t* kb, int lo, int hi) {
    if (hi > lo) {
        prefetch_l2(vb + lo, static_cast<std::size_t>(hi - lo) * 8);
        prefetch_l2(kb + lo, static_cast<std::size_t>(hi - lo) * 2);
    }
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


// One chunk of a lane's range: 4 nonzeros, one 256-bit val load and one
// 64-bit key load (4 x 16-bit keys), both aligned (chunks are 32 B).
struct Chunk {
    double2 v0, v1;
    uint2 k;
};

__device__ __forceinline__ void load_chunk(Chunk& c, const double* vb, const std::uint16_t* kb, unsigned e,
                                           std::uint64_t pol) {
    ld_stream_f64x4(vb + e, c.v0, c.v1, pol);
    c.k = ld_stream_u16x4(kb + e, pol);
}

// A lane's walk state over its range: the row being summed, its partial
// sum, and the head run (the lane's first row, which may have begun in an
// earlier lane) once a later row starts.
struct Walk {
    unsigned row;
    double acc, head;
    bool in_head;
};

template <int MODE>
__device__ __forceinline__ void walk_one(Walk& w, double v, unsigned key, std::uint32_t xb_s, std::uint32_t yp_s) {
    const double p = (MODE == 1 || MODE == 3) ? v : v * lds_f64(xb_s + 8u * (key & kKeyColMask));
    if (MODE >= 2) {
        w.acc += p;
        return;
    }
    // a new row: the previous one is complete (branch-free; the flush of a
    // row that began and ended in this lane is predicated, exclusive)
    const bool st = (key & kKeyStart) != 0u;
    if (st && !w.in_head) sts_add_f64(yp_s + 8u * w.row, w.acc);
    w.head = st && w.in_head ? w.acc : w.head;
    w.in_head = w.in_head && !st;
    w.row += st ? 1u : 0u;
    w.acc = (st ? 0.0 : w.acc) + p;
}

template <int MODE>
__device__ __forceinline__ void walk_chunk(Walk& w, const Chunk& c, std::uint32_t xb_s, std::uint32_t yp_s) {
    walk_one<MODE>(w, c.v0.x, c.k.x & 0xffffu, xb_s, yp_s);
    walk_one<MODE>(w, c.v0.y, c.k.x >> 16, xb_s, yp_s);
    walk_one<MODE>(w, c.v1.x, c.k.y & 0xffffu, xb_s, yp_s);
    walk_one<MODE>(w, c.v1.y, c.k.y >> 16, xb_s, yp_s);
}

// Combines the lanes' boundary rows once per run: lane l holds its head run
// (k0, p0, only when split) and its tail run (k1, p1); rows are
// non-decreasing across lanes. Adds each row's sum into yp[row] (rows are
// owned by this warp: no atomics, fixed order). `cont`: the lane's first row
// began in an earlier lane; inactive lanes (no chunks) are segment heads that
// store nothing.
__device__ __forceinline__ void reduce_lanes(unsigned k0, double p0, unsigned k1, double p1, bool split, bool cont,
                                             bool active, int lane, std::uint32_t yp_s) {
    double s = p1;
    const bool head = lane == 0 || split || !cont || !active;
    const unsigned hm = __ballot_sync(kFull, head);
    const int seg = 31 - __clz(hm & (kFull >> (31 - lane)));
    const int maxspan = static_cast<int>(__reduce_max_sync(kFull, static_cast<unsigned>(lane - seg + 1)));
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        if (d >= maxspan) break;
        const double t = __shfl_up_sync(kFull, s, d);
        if (lane - d >= seg) s += t;
    }
    // two ordered store passes over distinct rows: (1) every segment's sum at
    // its last lane; (2) the head run of every split lane (a row running from
    // lane i-1's tail into lane i's head gets both)
    if (active && (lane == 31 || ((hm >> (lane + 1)) & 1u))) sts_add_f64(yp_s + 8u * k1, s);
    __syncwarp();
    if (active && split) sts_add_f64(yp_s + 8u * k0, p0);
}

// Processes a (slab, warp) run [lo, hi) (tile-relative, multiples of kChunk)
// with lane descriptor `ld` against the slab in shared memory at xb_s. The
// run's bytes were prefetched into L2 one slab ahead; the next chunk is
// loaded while the current one is walked.
template <int MODE>
__device__ __forceinline__ void process_run(const double* vb, const std::uint16_t* kb, int lo, int hi, unsigned ld,
                                            std::uint32_t xb_s, std::uint32_t yp_s, int lane) {
    std::uint64_t pol;
    asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    const int C = (hi - lo) / kChunk, m = C >> 5, r = C & 31;
    const int cnt = m + (lane < r ? 1 : 0), iters = m + (r > 0 ? 1 : 0);
    const unsigned e0 = static_cast<unsigned>(lo + kChunk * lane);  // chunk i at e0 + 128 i
    Walk w{ld & 0x7fffu, 0.0, 0.0, true};
    Chunk ca, cb;
    if (cnt > 0) load_chunk(ca, vb, kb, e0, pol);
    for (int i = 0; i < iters; i += 2) {
        if (cnt > i + 1) load_chunk(cb, vb, kb, e0 + 128u * (i + 1), pol);
        if (cnt > i) walk_chunk<MODE>(w, ca, xb_s, yp_s);
        if (i + 1 >= iters) break;
        if (cnt > i + 2) load_chunk(ca, vb, kb, e0 + 128u * (i + 2), pol);
        if (cnt > i + 1) walk_chunk<MODE>(w, cb, xb_s, yp_s);
    }
    if (MODE >= 2) {  // probe: no row sums
        if (w.acc == 12345.678) sts_add_f64(yp_s, w.acc);
        return;
    }
    reduce_lanes(ld & 0x7fffu, w.head, w.row, w.acc, !w.in_head, (ld & kLaneCont) != 0u, cnt > 0, lane, yp_s);
}

template <bool DOT, int MODE = 0>
__global__ void __launch_bounds__(kTileThreads, 1)
    k_spmv_tiled(TcsrDev T, const double* __restrict__ x, double* __restrict__ y, double* partials,
                 unsigned int* ticket, CgScalars* sc, std::int64_t dot_off) {
    extern __shared__ __align__(128) double smem[];
    double* xs = smem;                    // [2][kSlabStride]: slab + zero cell
    double* yp = smem + 2 * kSlabStride;  // [kMaxTileRows]
    __shared__ __align__(8) std::uint64_t mbar[2];
    __shared__ unsigned released[2];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const std::uint32_t xs_s = smem_addr(xs), yp_s = smem_addr(yp);

    if (tid == 0) {
        released[0] = released[1] = 0;
        xs[kSlabW] = xs[kSlabStride + kSlabW] = 0.0;  // padding entries read these
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
        const std::uint16_t* kb = T.key + base;
        const std::int32_t* wo = T.woff + t * (static_cast<std::int64_t>(T.nslabs) * kTileWarps + 1);
        const std::uint16_t* lr = T.lrow + t * (static_cast<std::int64_t>(T.nslabs) * kTileWarps) * 32 + lane;
        for (int r = tid; r < nrows; r += kTileThreads) yp[r] = 0.0;
        if (lane == 0)  // runs stream into L2 kPfAhead slabs ahead of their use
            for (int k = 0; k < kPfAhead && k < T.nslabs; ++k)
                prefetch_run(vb, kb, wo[k * kTileWarps + warp], wo[k * kTileWarps + warp + 1]);
        // lane descriptors are loaded one run ahead (registers)
        unsigned dnext = T.nslabs > 0 ? __ldg(lr + warp * 32) : 0u;
        if (tid == 0 && T.nslabs > 0 && MODE < 5) {
            issue_slab(T, x, xs, 0, &mbar[0]);
            if (T.nslabs > 1) issue_slab(T, x, xs + kSlabStride, 1, &mbar[1]);
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
            const unsigned dcur = dnext;
            if (k + 1 < T.nslabs) {
                if (lane == 0 && k + kPfAhead < T.nslabs)
                    prefetch_run(vb, kb, wo[(k + kPfAhead) * kTileWarps + warp],
                                 wo[(k + kPfAhead) * kTileWarps + warp + 1]);
                dnext = __ldg(lr + ((k + 1) * kTileWarps + warp) * 32);
            }
            process_run<MODE == 5 ? 3 : (MODE == 6 ? 0 : MODE)>(
                vb, kb, wo[k * kTileWarps + warp], wo[k * kTileWarps + warp + 1], dcur,
                xs_s + 8u * static_cast<unsigned>(buf * kSlabStride), yp_s, lane);
            __syncwarp();
            if (lane == 0) {
                __threadfence_block();
                if (atomicAdd(&released[buf], 1u) == kTileWarps - 1) {
                    released[buf] = 0;
                    if (k + 2 < T.nslabs && MODE < 5) issue_slab(T, x, xs + buf * kSlabStride, k + 2, &mbar[buf]);
                }
            }
        }
        __syncthreads();  // every row of the tile is complete
        for (int r = tid; r < nrows; r += kTileThreads) {
            const double v = yp[r];
            y[row0 + r] = v;
            if (DOT) pq += v * __ldg(x + dot_off + row0 + r);
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
                    if (sc->nranks > 1) {
                        p2p_publish(sc, &a, 1);  // the shard's partial; alpha after the exchange
                    } else {
                        sc->d = a;
                        sc->rho0 = sc->rho;
                        sc->alpha = sc->rho / a;
                    }
                    *ticket = 0u;
                }
            }
        }
    }
}

int g_sms = 0;

}  // namespace

template <int MODE>
void launch_variant(const TcsrDev& T, const double* x, double* y, double* partials, unsigned int* ticket,
                    CgScalars* sc, unsigned grid, cudaStream_t s, std::int64_t dot_off) {
    static bool configured = false;
    if (!configured) {
        B200_CUDA(cudaFuncSetAttribute(k_spmv_tiled<false, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(kTileSmem)));
        B200_CUDA(cudaFuncSetAttribute(k_spmv_tiled<true, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(kTileSmem)));
        configured = true;
    }
    if (partials)
        k_spmv_tiled<true, MODE><<<std::min<unsigned>(grid, kMaxParts), kTileThreads, kTileSmem, s>>>(
            T, x, y, partials, ticket, sc, dot_off);
    else
        k_spmv_tiled<false, MODE><<<grid, kTileThreads, kTileSmem, s>>>(T, x, y, nullptr, nullptr, nullptr, 0);
}

void launch_spmv_tiled(const TcsrDev& T, std::int64_t rows, const double* x, double* y, double* partials,
                       unsigned int* ticket, CgScalars* sc, cudaStream_t s, std::int64_t dot_off) {
    static int mode = -1;
    if (mode < 0) {
        int dev = 0;
        B200_CUDA(cudaGetDevice(&dev));
        B200_CUDA(cudaDeviceGetAttribute(&g_sms, cudaDevAttrMultiProcessorCount, dev));
        const char* m = std::getenv("LILAC_B200_TILED_PROBE");  // timing probes only: wrong results
        mode = (m && *m) ? std::atoi(m) : 0;
    }
    if (rows <= 0 || T.ntiles <= 0) return;
    const unsigned grid = static_cast<unsigned>(std::min<std::int64_t>(T.ntiles, g_sms));
    switch (partials ? 0 : mode) {  // probes never on the fused CG path
    case 1: launch_variant<1>(T, x, y, partials, ticket, sc, grid, s, dot_off); break;
    case 2: launch_variant<2>(T, x, y, partials, ticket, sc, grid, s, dot_off); break;
    case 5: launch_variant<5>(T, x, y, partials, ticket, sc, grid, s, dot_off); break;
    case 6: launch_variant<6>(T, x, y, partials, ticket, sc, grid, s, dot_off); break;
    default: launch_variant<0>(T, x, y, partials, ticket, sc, grid, s, dot_off); break;
    }
    B200_CUDA(cudaGetLastError());
}

}  // namespace b200
