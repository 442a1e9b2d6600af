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
#include "p2p.hpp"

#include <algorithm>
#include <cstdlib>

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

__device__ __forceinline__ uint4 ld_stream_u32x4(const std::uint32_t* p, std::uint64_t pol) {
    uint4 r;
    asm("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.u32 {%0, %1, %2, %3}, [%4], %5;"
        : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
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
__device__ __forceinline__ void prefetch_run(const double* vb, const std::uint32_t* kb, int lo, int hi) {
    if (hi > lo) {
        prefetch_l2(vb + lo, static_cast<std::size_t>(hi - lo) * 8);
        prefetch_l2(kb + lo, static_cast<std::size_t>(hi - lo) * 4);
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


// A lane's four consecutive nonzeros of a (slab, warp) run: one 256-bit val
// load and one 128-bit key load, both 32/16-byte aligned (runs start on
// kRunAlign boundaries). Lanes past the run end get zeros (and sentinel keys).
struct Chunk {
    double2 v0, v1;
    uint4 k;
};

__device__ __forceinline__ void load_chunk(Chunk& c, const double* vb, const std::uint32_t* kb, int j, int hi,
                                           std::uint64_t pol) {
    if (j < hi) {
        ld_stream_f64x4(vb + j, c.v0, c.v1, pol);
        c.k = ld_stream_u32x4(kb + j, pol);
    } else {
        c.v0 = c.v1 = make_double2(0.0, 0.0);
        c.k = make_uint4(kPadKey, kPadKey, kPadKey, kPadKey);
    }
}

// One 128-nonzero piece after the lane-local pass: lane holds its head run
// (k0, p0) and tail run (k1, p1) (k0 == k1: a single run, value p1). Row keys
// are non-decreasing across lanes. Adds every row's piece-sum into yp[row]
// (rows are owned by this warp: no atomics, fixed order).
// `cont`: the lane's first element continues the row of the element before it
// (a layout bit, kKeyCont), so a non-split lane starts a segment iff !cont.
__device__ __forceinline__ void reduce_piece(unsigned k0, double p0, unsigned k1, double p1, bool cont, int lane,
                                             std::uint32_t yp_s) {
    const bool split = k0 != k1;
    double s = p1;
    const bool head = lane == 0 || split || !cont;
    const unsigned hm = __ballot_sync(kFull, head);
    const int seg = 31 - __clz(hm & (kFull >> (31 - lane)));
    // only as many doubling steps as the longest row segment of the piece
    // needs (NPB: rows span ~5 lanes, so usually 3 of the 5; each f64 step
    // is two SHFLs + a DADD)
    const int maxspan = static_cast<int>(__reduce_max_sync(kFull, static_cast<unsigned>(lane - seg + 1)));
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        if (d >= maxspan) break;
        const double t = __shfl_up_sync(kFull, s, d);
        if (lane - d >= seg) s += t;
    }
    // Two store passes, each touching distinct rows: (1) every segment's sum
    // at its last lane (the next lane starts a segment); (2) the head run of
    // every split lane. A row continuing from lane i-1's tail into lane i's
    // head gets both; the passes are ordered, so no shuffle of the scan value
    // into the split lane is needed.
    if ((lane == 31 || ((hm >> (lane + 1)) & 1u)) && k1 != kSent) sts_add_f64(yp_s + 8u * k1, s);
    __syncwarp();
    if (split && k0 != kSent) sts_add_f64(yp_s + 8u * k0, p0);
}

// Processes a (slab, warp) run [lo, hi) (tile-relative, both multiples of
// kRunAlign) against the slab in shared memory at xb_s. The run's bytes were
// prefetched into L2 one slab ahead, so these loads are L2 hits; the next
// chunk is loaded into registers while this one is reduced.
template <int MODE>
__device__ __forceinline__ void process_run(const double* vb, const std::uint32_t* kb, int lo, int hi,
                                            std::uint32_t xb_s, std::uint32_t yp_s, int lane) {
    std::uint64_t pol;
    asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    Chunk cur, nxt;
    load_chunk(cur, vb, kb, lo + 4 * lane, hi, pol);
    for (int c = lo; c < hi; c += 128) {
        load_chunk(nxt, vb, kb, c + 128 + 4 * lane, hi, pol);
        const unsigned k0 = cur.k.x >> 16, k1 = cur.k.y >> 16, k2 = cur.k.z >> 16, k3 = cur.k.w >> 16;
        double p0, p1, p2, p3;
        if (MODE == 1 || MODE == 3) {  // probe: no gather
            p0 = cur.v0.x, p1 = cur.v0.y, p2 = cur.v1.x, p3 = cur.v1.y;
        } else {
            p0 = cur.v0.x * lds_f64(xb_s + 8u * (cur.k.x & kKeyColMask));
            p1 = cur.v0.y * lds_f64(xb_s + 8u * (cur.k.y & kKeyColMask));
            p2 = cur.v1.x * lds_f64(xb_s + 8u * (cur.k.z & kKeyColMask));
            p3 = cur.v1.y * lds_f64(xb_s + 8u * (cur.k.w & kKeyColMask));
        }
        if (MODE >= 2) {
            if (p0 == 12345.678) sts_add_f64(yp_s, p1 + p2 + p3);  // probe: no reduction
        } else {
            // lane-local pass, branch-free for the common case (keys sorted):
            // tail run = elements equal to k3, head run = elements equal to k0
            double tail = p3;
            tail += k2 == k3 ? p2 : 0.0;
            tail += k1 == k3 ? p1 : 0.0;
            tail += k0 == k3 ? p0 : 0.0;
            double head = p0;
            head += k1 == k0 ? p1 : 0.0;
            head += k2 == k0 ? p2 : 0.0;
            // rows strictly inside the lane (a row with <= 2 nonzeros in this
            // slab) are exclusive to it: flushed here, rarely taken
            const bool in1 = k1 != k0 && k1 != k3, in2 = k2 != k0 && k2 != k3;
            if (in1 | in2) {
                if (in1) sts_add_f64(yp_s + 8u * k1, k2 == k1 ? p1 + p2 : p1);
                if (in2 && k2 != k1) sts_add_f64(yp_s + 8u * k2, p2);
            }
            reduce_piece(k0, head, k3, tail, (cur.k.x & kKeyCont) != 0u, lane, yp_s);
        }
        cur = nxt;
    }
}

template <bool DOT, int MODE = 0>
__global__ void __launch_bounds__(kTileThreads, 1)
    k_spmv_tiled(TcsrDev T, const double* __restrict__ x, double* __restrict__ y, double* partials,
                 unsigned int* ticket, CgScalars* sc, std::int64_t dot_off) {
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
        if (lane == 0 && T.nslabs > 0) prefetch_run(vb, kb, wo[warp], wo[warp + 1]);
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
            if (lane == 0 && k + 1 < T.nslabs)  // next slab's run streams into L2 meanwhile
                prefetch_run(vb, kb, wo[(k + 1) * kTileWarps + warp], wo[(k + 1) * kTileWarps + warp + 1]);
            process_run<MODE == 5 ? 3 : (MODE == 6 ? 0 : MODE)>(
                vb, kb, wo[k * kTileWarps + warp], wo[k * kTileWarps + warp + 1],
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
