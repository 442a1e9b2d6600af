// lrcsr.cu — lane-range CSR SpMV (layout in b200.hpp, builder in
// lrcsr_build.cpp) for matrices whose x gathers go to global memory.
//
// Why: on a skewed graph (Kronecker scale 22: half the rows empty, one row of
// 160k nonzeros, x = 33.5 MB) a row-parallel kernel waits on row_ptr -> col ->
// x dependence chains and on its longest rows, and every random 8-byte gather
// is one L1TEX wavefront (~1 per cycle per SM: the floor of any global-gather
// kernel). Here every warp streams fixed-size units of nonzeros with 256-bit
// loads (no row_ptr on the path), each lane walks its own contiguous range
// summing rows in registers, and the gathers of the most frequent columns —
// a large share of a power-law graph's nonzeros — come from a shared-memory
// copy of their x values instead of the L1TEX queue.
//
// Per call: (1) k_lrc_gather_hot packs x[hot_cols] into x_hot (+ a zero
// cell); (2) k_spmv_lrc: one CTA of 32 warps per SM bulk-copies x_hot into
// shared memory, then each warp takes units round-robin; rows complete inside
// a unit are stored directly, the open rows at the unit's ends go to its
// carry; (3) k_lrc_fixup sums every row that crossed units, in unit order.
// All sums are in a fixed order: deterministic run to run.

#include "b200.hpp"
#include "ldst.cuh"

#include <algorithm>

namespace b200 {

namespace {

constexpr unsigned kFull = 0xffffffffu;
constexpr int kLrcThreads = 1024;
constexpr int kLrcWarps = kLrcThreads / 32;

__device__ __forceinline__ std::uint32_t smem_u32(const void* p) {
    return static_cast<std::uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void ld_f64x4(const double* p, double (&v)[4], std::uint64_t pol) {
    asm("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.f64 {%0, %1, %2, %3}, [%4], %5;"
        : "=d"(v[0]), "=d"(v[1]), "=d"(v[2]), "=d"(v[3])
        : "l"(p), "l"(pol));
}

__device__ __forceinline__ void ld_u32x4(const std::uint32_t* p, std::uint32_t (&c)[4], std::uint64_t pol) {
    asm("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.u32 {%0, %1, %2, %3}, [%4], %5;"
        : "=r"(c[0]), "=r"(c[1]), "=r"(c[2]), "=r"(c[3])
        : "l"(p), "l"(pol));
}

struct LChunk {
    double v[4];
    std::uint32_t c[4];
};

__device__ __forceinline__ void load_lchunk(LChunk& k, const LrcDev& L, std::int64_t e, std::uint64_t pol) {
    ld_f64x4(L.val + e, k.v, pol);
    ld_u32x4(L.col + e, k.c, pol);
}

// x for one nonzero: the shared-memory slot of a hot column, else global
template <bool HOT>
__device__ __forceinline__ double gather_x(std::uint32_t c, const double* __restrict__ x, std::uint32_t xs_s,
                                           std::uint64_t pol) {
    const std::uint32_t idx = c & kLrcColMask;
    if (HOT && (c & kLrcHot)) {
        double v;
        asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(xs_s + 8u * idx));
        return v;
    }
    return ld_gather_f64(x + idx, pol);
}

template <bool RMAP>
__device__ __forceinline__ std::int64_t out_row(const LrcDev& L, std::uint32_t r) {
    return RMAP ? static_cast<std::int64_t>(__ldg(L.rmap + r)) : static_cast<std::int64_t>(r);
}

// A lane's walk over its range: the compact row being summed and its partial,
// the head partial (the lane's first row, begun before the lane) once closed.
struct LWalk {
    std::uint32_t row;
    double acc, head;
    bool in_head;
};

template <bool RMAP>
__device__ __forceinline__ void lwalk_one(LWalk& w, double v, double xv, std::uint32_t c, const LrcDev& L,
                                          double* __restrict__ y) {
    const bool st = (c & kLrcStart) != 0u;
    // a row that began and ended inside this lane is complete: store it
    if (st && !w.in_head) y[out_row<RMAP>(L, w.row)] = w.acc;
    w.head = st && w.in_head ? w.acc : w.head;
    w.in_head = w.in_head && !st;
    w.row += st ? 1u : 0u;
    w.acc = fma(v, xv, st ? 0.0 : w.acc);
}

template <bool HOT, bool RMAP>
__global__ void __launch_bounds__(kLrcThreads, 1)
    k_spmv_lrc(LrcDev L, const double* __restrict__ x, double* __restrict__ y) {
    extern __shared__ __align__(128) double xs[];
    __shared__ __align__(8) std::uint64_t mbar;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const std::uint32_t xs_s = smem_u32(xs);
    const std::uint64_t pol = policy_evict_first(), gpol = policy_evict_last();
    const std::int64_t stride = static_cast<std::int64_t>(gridDim.x) * kLrcWarps;
    std::int64_t u = static_cast<std::int64_t>(blockIdx.x) * kLrcWarps + warp;
    LChunk ca, cb;
    if (u < L.units) {  // the matrix does not depend on the preceding kernels
        const std::int64_t e0 = u * kLrcUnit + 4 * lane;
        load_lchunk(ca, L, e0, pol);
        load_lchunk(cb, L, e0 + 128, pol);
    }
    if (HOT) {
        if (threadIdx.x == 0) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&mbar)) : "memory");
            asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        }
        __syncthreads();
        pdl_wait();  // x_hot is written by the preceding gather kernel
        if (threadIdx.x == 0) {
            const unsigned bytes = static_cast<unsigned>(L.hot + 2) / 2u * 16u;  // 16-byte granules
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&mbar)), "r"(bytes)
                         : "memory");
            asm volatile(
                "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(xs_s),
                "l"(L.x_hot), "r"(bytes), "r"(smem_u32(&mbar))
                : "memory");
        }
    }
    bool waited = !HOT;
    for (; u < L.units; u += stride) {
        const std::uint32_t d = __ldg(L.desc + u * 32 + lane);
        const bool cont = (d & kLrcCont) != 0u;
        LWalk w{(d & ~kLrcCont) - (cont ? 0u : 1u), 0.0, 0.0, true};
        const std::int64_t e0 = u * kLrcUnit + 4 * lane;  // chunk i at e0 + 128 i
        if (!waited) {
            asm volatile(
                "{\n\t.reg .pred P1;\n"
                "LRC_WAIT_%=:\n\t"
                "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n\t"
                "@P1 bra LRC_DONE_%=;\n\t"
                "bra LRC_WAIT_%=;\n"
                "LRC_DONE_%=:\n\t}" ::"r"(smem_u32(&mbar))
                : "memory");
            waited = true;
        }
        // chunks i+1 and i+2 stream in while chunk i's gathers are in flight
#pragma unroll
        for (int i = 0; i < kLrcChunks; ++i) {
            double xa[4];
#pragma unroll
            for (int s = 0; s < 4; ++s) xa[s] = gather_x<HOT>(ca.c[s], x, xs_s, gpol);
            LChunk na;
            if (i + 2 < kLrcChunks) load_lchunk(na, L, e0 + 128 * (i + 2), pol);
#pragma unroll
            for (int s = 0; s < 4; ++s) lwalk_one<RMAP>(w, ca.v[s], xa[s], ca.c[s], L, y);
            ca = cb;
            if (i + 2 < kLrcChunks) cb = na;
        }
        // the next unit's first two chunks stream in during this reduction
        if (u + stride < L.units) {
            const std::int64_t n0 = (u + stride) * kLrcUnit + 4 * lane;
            load_lchunk(ca, L, n0, pol);
            load_lchunk(cb, L, n0 + 128, pol);
        }
        // ---- combine the lanes' open rows -------------------------------------
        const bool split = !w.in_head;  // a row began inside this lane
        const unsigned sm = __ballot_sync(kFull, split);
        const unsigned hm = sm | 1u;    // segment heads: split lanes and lane 0
        const int seg = 31 - __clz(hm & (kFull >> (31 - lane)));
        double S = w.acc;  // inclusive segmented scan of the lanes' tail partials
        const int maxspan = static_cast<int>(__reduce_max_sync(kFull, static_cast<unsigned>(lane - seg + 1)));
#pragma unroll
        for (int dd = 1; dd < 32; dd <<= 1) {
            if (dd >= maxspan) break;
            const double t = __shfl_up_sync(kFull, S, dd);
            if (lane - dd >= seg) S += t;
        }
        const double Sprev = __shfl_up_sync(kFull, S, 1);
        const std::uint32_t rprev = __shfl_up_sync(kFull, w.row, 1);
        const int segprev = __shfl_up_sync(kFull, seg, 1);
        // a split lane b > 0 closes the row open at lane b-1: complete if that
        // row's segment began with a row start inside this unit
        const bool closes = lane > 0 && split;
        const bool fresh = ((sm >> segprev) & 1u) != 0u;
        const double tot = Sprev + w.head;  // w.head is 0 for a lane whose first nonzero starts a row
        if (closes && fresh) y[out_row<RMAP>(L, rprev)] = tot;
        // carries: the row open at the unit's start (lane 0 continues it)
        const bool cont0 = __shfl_sync(kFull, static_cast<int>(cont), 0) != 0;
        const int b = sm ? __ffs(static_cast<int>(sm & ~1u)) - 1 : -1;  // first split lane > 0
        const double head0 = __shfl_sync(kFull, w.head, 0);
        const double totb = __shfl_sync(kFull, tot, b < 0 ? 0 : b);
        const std::uint32_t rowb = __shfl_sync(kFull, rprev, b < 0 ? 0 : b);
        const double S31 = __shfl_sync(kFull, S, 31);
        const std::uint32_t row31 = __shfl_sync(kFull, w.row, 31);
        const int seg31 = __shfl_sync(kFull, seg, 31);
        if (lane == 0) {
            LrcCarry c;
            c.pad = 0;
            c.split = sm != 0u;
            c.head_row = -1;
            c.head_val = 0.0;
            if (cont0) {
                const std::uint32_t first = d & ~kLrcCont;
                if (sm & 1u) {  // lane 0 itself closes it
                    c.head_row = static_cast<std::int32_t>(first);
                    c.head_val = w.head;
                } else if (b >= 0) {  // closed at the first split lane
                    c.head_row = static_cast<std::int32_t>(rowb);
                    c.head_val = totb;
                } else {  // no row begins in this unit: it is all one row's
                    c.head_row = static_cast<std::int32_t>(first);
                    c.head_val = S31;
                }
            }
            // the row open at the unit's end, if it began in this unit
            const bool tail = ((sm >> seg31) & 1u) != 0u;
            c.tail_row = tail ? static_cast<std::int32_t>(row31) : -1;
            c.tail_val = tail ? S31 : 0.0;
            L.carry[u] = c;
        }
    }
}

// x_hot[i] = x[hot_cols[i]], x_hot[hot] = 0 (the padding entries' cell).
__global__ void k_lrc_gather_hot(const std::int32_t* __restrict__ cols, int hot, const double* __restrict__ x,
                                 double* __restrict__ out) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < hot) out[i] = __ldg(x + cols[i]);
    if (i == hot) out[i] = 0.0;
    pdl_trigger();
}

// Rows that crossed units: the unit where a row began walks forward over the
// units it continues into, summing in unit order.
template <bool RMAP>
__global__ void k_lrc_fixup(LrcDev L, double* __restrict__ y) {
    pdl_wait();
    const std::int64_t stride = static_cast<std::int64_t>(gridDim.x) * blockDim.x;
    for (std::int64_t u = static_cast<std::int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; u < L.units;
         u += stride) {
        const LrcCarry c = L.carry[u];
        if (c.tail_row < 0) continue;
        double tot = c.tail_val;
        for (std::int64_t v = u + 1; v < L.units; ++v) {
            const int hr = __ldcg(&L.carry[v].head_row);
            if (hr != c.tail_row) break;
            tot += __ldcg(&L.carry[v].head_val);
            if (__ldcg(&L.carry[v].split)) break;
        }
        y[out_row<RMAP>(L, static_cast<std::uint32_t>(c.tail_row))] = tot;
    }
}

int g_lrc_sms = 0;

template <bool HOT, bool RMAP>
void lrc_launch(const LrcDev& L, const double* x, double* y, cudaStream_t s) {
    static bool attr = false;
    const std::size_t smem = HOT ? sizeof(double) * static_cast<std::size_t>(kLrcHotMax + 2) : 0;
    if (!attr) {
        B200_CUDA(cudaFuncSetAttribute(k_spmv_lrc<HOT, RMAP>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(smem)));
        attr = true;
    }
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(static_cast<unsigned>(std::min<std::int64_t>(g_lrc_sms, (L.units + kLrcWarps - 1) / kLrcWarps)));
    cfg.blockDim = dim3(kLrcThreads);
    cfg.dynamicSmemBytes = HOT ? sizeof(double) * static_cast<std::size_t>(L.hot + 2) : 0;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = HOT ? 1 : 0;
    B200_CUDA(cudaLaunchKernelEx(&cfg, k_spmv_lrc<HOT, RMAP>, L, x, y));
    cudaLaunchConfig_t fc{};
    const std::int64_t fb = std::min<std::int64_t>((L.units + 255) / 256, 148 * 8);
    fc.gridDim = dim3(static_cast<unsigned>(std::max<std::int64_t>(fb, 1)));
    fc.blockDim = dim3(256);
    fc.stream = s;
    fc.attrs = at;
    fc.numAttrs = 0;  // the carries are complete only when every unit is: plain stream order
    B200_CUDA(cudaLaunchKernelEx(&fc, k_lrc_fixup<RMAP>, L, y));
}

}  // namespace

void launch_spmv_lrc(const LrcDev& L, std::int64_t rows, const double* x, double* y, cudaStream_t s) {
    if (rows <= 0) return;
    if (!g_lrc_sms) {
        int dev = 0;
        B200_CUDA(cudaGetDevice(&dev));
        B200_CUDA(cudaDeviceGetAttribute(&g_lrc_sms, cudaDevAttrMultiProcessorCount, dev));
    }
    if (L.has_empty) B200_CUDA(cudaMemsetAsync(y, 0, sizeof(double) * static_cast<std::size_t>(rows), s));
    if (L.units == 0) return;
    // always through the shared-memory cell path: padding entries read its
    // zero cell (never an Inf or NaN of x), whether or not columns are hot
    k_lrc_gather_hot<<<(L.hot + 1 + 255) / 256, 256, 0, s>>>(L.hot_cols, L.hot, x, L.x_hot);
    B200_CUDA(cudaGetLastError());
    if (L.rmap)
        lrc_launch<true, true>(L, x, y, s);
    else
        lrc_launch<true, false>(L, x, y, s);
    B200_CUDA(cudaGetLastError());
}

}  // namespace b200
