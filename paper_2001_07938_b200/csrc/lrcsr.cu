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
#include "tcsr.hpp"

#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>

#include <algorithm>
#include <cstdlib>

namespace b200 {

namespace {

constexpr unsigned kFull = 0xffffffffu;
#ifndef LILAC_LRC_THREADS
#define LILAC_LRC_THREADS 1024
#endif
constexpr int kLrcThreads = LILAC_LRC_THREADS;
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

// The value a finished row stores: the SpMV's sum, or with PR the PageRank
// update d * sum + (1 - d) / n applied in the same store (exactly
// k_pagerank_update's operations: the same bits as SpMV + update).
template <bool PR>
__device__ __forceinline__ double row_out(double v, double d, double tele) {
    return PR ? __dadd_rn(__dmul_rn(d, v), tele) : v;
}

// A lane's walk over its range: the compact row being summed and its partial,
// the head partial (the lane's first row, begun before the lane) once closed.
struct LWalk {
    std::uint32_t row;
    double acc, head;
    bool in_head;
};

template <bool RMAP, bool PR>
__device__ __forceinline__ void lwalk_one(LWalk& w, double v, double xv, std::uint32_t c, const LrcDev& L,
                                          double* __restrict__ y, double d, double tele) {
    const bool st = (c & kLrcStart) != 0u;
    // a row that began and ended inside this lane is complete: store it
    if (st && !w.in_head) y[out_row<RMAP>(L, w.row)] = row_out<PR>(w.acc, d, tele);
    w.head = st && w.in_head ? w.acc : w.head;
    w.in_head = w.in_head && !st;
    w.row += st ? 1u : 0u;
    w.acc = fma(v, xv, st ? 0.0 : w.acc);
}

template <bool HOT, bool RMAP, bool PR>
__global__ void __launch_bounds__(kLrcThreads, 1)
    k_spmv_lrc(LrcDev L, const double* __restrict__ x, double* __restrict__ y, double pr_d, double pr_tele) {
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
    pdl_trigger();  // the fix-up may launch now; its griddepcontrol.wait covers this grid
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
            for (int s = 0; s < 4; ++s) lwalk_one<RMAP, PR>(w, ca.v[s], xa[s], ca.c[s], L, y, pr_d, pr_tele);
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
        if (closes && fresh) y[out_row<RMAP>(L, rprev)] = row_out<PR>(tot, pr_d, pr_tele);
        // carries: the row open at the unit's start (lane 0 continues it)
        const bool cont0 = __shfl_sync(kFull, static_cast<int>(cont), 0) != 0;
        const int b = sm ? __ffs(static_cast<int>(sm & ~1u)) - 1 : -1;  // first split lane > 0
        const double head0 = __shfl_sync(kFull, w.head, 0);
        const double totb = __shfl_sync(kFull, tot, b < 0 ? 0 : b);
        const double S31 = __shfl_sync(kFull, S, 31);
        if (lane == 0) {
            LrcCarry c;
            // the row open at the unit's start (lane 0 continues it): closed by
            // lane 0 itself, at the first split lane, or never (all one row)
            c.head_val = !cont0 ? 0.0 : (sm & 1u) ? w.head : (b >= 0 ? totb : S31);
            c.tail_val = S31;  // the row open at the unit's end (used when it began here)
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

// Rows that crossed units (the structural plan): a short crossing is summed
// by one thread in unit order, a long one by a warp (lanes stride the units,
// then a fixed shuffle tree). Empty rows (never in the stream) are zeroed here.
template <bool RMAP, bool PR>
__global__ void k_lrc_fixup(LrcDev L, double* __restrict__ y, double pr_d, double pr_tele) {
    const std::int64_t tid = static_cast<std::int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    const std::int64_t stride = static_cast<std::int64_t>(gridDim.x) * blockDim.x;
    for (std::int64_t i = tid; i < L.nempty; i += stride) y[__ldg(L.empty + i)] = row_out<PR>(0.0, pr_d, pr_tele);
    pdl_wait();  // every unit's carry is written
    for (std::int64_t i = tid; i < L.nfix_short; i += stride) {
        const LrcFix f = L.fix[i];
        double tot = __ldcg(&L.carry[f.u].tail_val);
        for (int v = f.u + 1; v <= f.e; ++v) tot += __ldcg(&L.carry[v].head_val);
        y[out_row<RMAP>(L, static_cast<std::uint32_t>(f.row))] = row_out<PR>(tot, pr_d, pr_tele);
    }
    const int lane = threadIdx.x & 31;
    for (std::int64_t i = tid >> 5; i < L.nfix_long; i += stride >> 5) {
        const LrcFix f = L.fix[L.nfix_short + i];
        double part = 0.0;
        for (int v = f.u + 1 + lane; v <= f.e; v += 32) part += __ldcg(&L.carry[v].head_val);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) part += __shfl_xor_sync(kFull, part, o);
        if (lane == 0)
            y[out_row<RMAP>(L, static_cast<std::uint32_t>(f.row))] =
                row_out<PR>(__ldcg(&L.carry[f.u].tail_val) + part, pr_d, pr_tele);
    }
}

int g_lrc_sms = 0;

template <bool HOT, bool RMAP, bool PR = false>
void lrc_launch(const LrcDev& L, const double* x, double* y, cudaStream_t s, double pr_d = 0.0,
                double pr_tele = 0.0) {
    static std::uint64_t attr = 0;
    const std::size_t smem = HOT ? sizeof(double) * static_cast<std::size_t>(kLrcHotMax + 2) : 0;
    if (first_on_device(attr))
        B200_CUDA(cudaFuncSetAttribute(k_spmv_lrc<HOT, RMAP, PR>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(smem)));
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
    B200_CUDA(cudaLaunchKernelEx(&cfg, k_spmv_lrc<HOT, RMAP, PR>, L, x, y, pr_d, pr_tele));
    cudaLaunchConfig_t fc{};
    const std::int64_t work = std::max({L.nfix_short, 32 * L.nfix_long, L.nempty});
    const std::int64_t fb = std::min<std::int64_t>((work + 255) / 256, 148 * 8);
    fc.gridDim = dim3(static_cast<unsigned>(std::max<std::int64_t>(fb, 1)));
    fc.blockDim = dim3(256);
    fc.stream = s;
    fc.attrs = at;
    fc.numAttrs = 1;  // launched early; zeroes the empty rows, then waits for every carry
    B200_CUDA(cudaLaunchKernelEx(&fc, k_lrc_fixup<RMAP, PR>, L, y, pr_d, pr_tele));
}

}  // namespace

// ---- device-side builder (a resident CSR: the device-generated stencil, the
// harness's uploaded arrays) --------------------------------------------------

namespace {

constexpr int kBT = 256;

unsigned bgrid(std::int64_t n) {
    return static_cast<unsigned>(std::max<std::int64_t>(1, std::min<std::int64_t>((n + kBT - 1) / kBT, 148 * 64)));
}

#define GS_LOOP(i, n)                                                                                        \
    for (std::int64_t i = static_cast<std::int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < (n);        \
         i += static_cast<std::int64_t>(gridDim.x) * blockDim.x)

__device__ __forceinline__ std::int64_t lrc_pos_d(std::int64_t e) {
    const std::int64_t u = e / kLrcUnit, w = e % kLrcUnit;
    const std::int64_t l = w / kLrcLaneNnz, k = w % kLrcLaneNnz;
    return u * kLrcUnit + (32 * (k / 4) + l) * 4 + (k % 4);
}

template <typename IdxT>
__global__ void k_lrc_freq(const IdxT* __restrict__ col, std::int64_t nnz, unsigned* __restrict__ freq) {
    GS_LOOP(j, nnz) atomicAdd(freq + col[j], 1u);
}

__global__ void k_lrc_iota(std::int32_t* __restrict__ v, std::int64_t n) {
    GS_LOOP(i, n) v[i] = static_cast<std::int32_t>(i);
}

// slots for the chosen hot columns (sorted ascending by column)
__global__ void k_lrc_slots(const std::int32_t* __restrict__ hot_cols, int hot, std::int32_t* __restrict__ slot) {
    GS_LOOP(i, hot) slot[hot_cols[i]] = static_cast<std::int32_t>(i);
}

template <typename IdxT>
__global__ void k_lrc_scatter(const IdxT* __restrict__ col, const double* __restrict__ val, std::int64_t nnz,
                              std::int64_t total, const std::int32_t* __restrict__ slot, int hot,
                              double* __restrict__ oval, std::uint32_t* __restrict__ ocol) {
    GS_LOOP(e, total) {
        const std::int64_t p = lrc_pos_d(e);
        if (e < nnz) {
            const std::int64_t c = static_cast<std::int64_t>(col[e]);
            const std::int32_t sl = slot ? slot[c] : -1;
            oval[p] = val[e];
            ocol[p] = sl >= 0 ? (kLrcHot | static_cast<std::uint32_t>(sl)) : static_cast<std::uint32_t>(c);
        } else {  // padding: value 0 times the zero cell
            oval[p] = 0.0;
            ocol[p] = kLrcHot | static_cast<std::uint32_t>(hot);
        }
    }
}

// row starts, nonempty flags (for the compaction scan)
__global__ void k_lrc_rows(const std::int64_t* __restrict__ rp, std::int64_t rows, std::uint32_t* __restrict__ ocol,
                           std::int32_t* __restrict__ nonempty) {
    GS_LOOP(r, rows) {
        const std::int64_t a = rp[r] - rp[0], b = rp[r + 1] - rp[0];
        nonempty[r] = b > a ? 1 : 0;
        if (b > a) ocol[lrc_pos_d(a)] |= kLrcStart;
    }
}

__global__ void k_lrc_rmap(const std::int32_t* __restrict__ comp, const std::int32_t* __restrict__ nonempty,
                           std::int64_t rows, std::int32_t* __restrict__ rmap, std::int32_t* __restrict__ empty) {
    GS_LOOP(r, rows) {
        if (nonempty[r])
            rmap[comp[r]] = static_cast<std::int32_t>(r);
        else
            empty[r - comp[r]] = static_cast<std::int32_t>(r);
    }
}

__global__ void k_lrc_desc(const std::int64_t* __restrict__ rp, std::int64_t rows, std::int64_t nnz,
                           std::int64_t units, const std::int32_t* __restrict__ comp, std::uint32_t last,
                           std::uint32_t* __restrict__ desc) {
    GS_LOOP(q, units * 32) {
        const std::int64_t e0 = (q / 32) * kLrcUnit + (q % 32) * kLrcLaneNnz;
        if (e0 >= nnz) {
            desc[q] = last | kLrcCont;
            continue;
        }
        const std::int64_t t = rp[0] + e0;
        std::int64_t lo = 0, hi = rows + 1;  // first index with rp[idx] > t
        while (lo < hi) {
            const std::int64_t mid = (lo + hi) >> 1;
            if (rp[mid] <= t)
                lo = mid + 1;
            else
                hi = mid;
        }
        const std::int64_t r = lo - 1;
        const std::uint32_t cr = comp ? static_cast<std::uint32_t>(comp[r]) : static_cast<std::uint32_t>(r);
        desc[q] = cr | (rp[r] == t ? 0u : kLrcCont);
    }
}

// The crossing-row plan: for each unit, the row holding its last nonzero,
// when that row began inside the unit (else an earlier unit owns it).
__global__ void k_lrc_plan(const std::int64_t* __restrict__ rp, std::int64_t rows, std::int64_t nnz,
                           std::int64_t units, const std::int32_t* __restrict__ comp, LrcFix* __restrict__ fix_short,
                           LrcFix* __restrict__ fix_long, unsigned long long* __restrict__ counts) {
    GS_LOOP(u, units) {
        const std::int64_t last = std::min<std::int64_t>((u + 1) * kLrcUnit, nnz) - 1;
        const std::int64_t t = rp[0] + last;
        std::int64_t lo = 0, hi = rows + 1;  // first index with rp[idx] > t
        while (lo < hi) {
            const std::int64_t mid = (lo + hi) >> 1;
            if (rp[mid] <= t)
                lo = mid + 1;
            else
                hi = mid;
        }
        const std::int64_t r = lo - 1;
        if (rp[r] - rp[0] < u * kLrcUnit) continue;  // began in an earlier unit
        LrcFix f;
        f.u = static_cast<std::int32_t>(u);
        f.e = static_cast<std::int32_t>((rp[r + 1] - rp[0] - 1) / kLrcUnit);
        f.row = comp ? comp[r] : static_cast<std::int32_t>(r);
        f.pad = 0;
        if (f.e - f.u <= kLrcFixShort)
            fix_short[atomicAdd(&counts[0], 1ull)] = f;
        else
            fix_long[atomicAdd(&counts[1], 1ull)] = f;
    }
}

}  // namespace

int lrc_hot_cap() {
    const char* e = std::getenv("LILAC_B200_LRC_HOT");
    // measured on Kronecker scale 22: 0 -> 351 us, 4096 -> 319, 12288 -> 294,
    // 16384 -> 294, 27647 -> 513 (the cache then leaves L1 too small for the
    // remaining global gathers)
    return e && *e ? static_cast<int>(std::min<long>(std::atol(e), kLrcHotMax)) : 12288;
}

void lrc_build_device(std::int64_t rows, const std::int64_t* rp, const void* col, bool col32, const double* val,
                      std::int64_t nnz, std::int64_t cols, LrcOwner& o, cudaStream_t s) {
    o.release();
    const std::int64_t units = (nnz + kLrcUnit - 1) / kLrcUnit, total = units * kLrcUnit;
    // ---- hot set: column frequencies, top `cap` by (count desc, column asc) ----
    const int cap = lrc_hot_cap();
    int hot = 0;
    std::int64_t covered = 0;
    DevBuf slot;
    if (cap > 0 && cols > 0 && nnz > 0) {
        DevBuf freq, keys_out, cols_in, cols_out, tmp;
        freq.ensure(sizeof(unsigned) * cols, false);
        B200_CUDA(cudaMemsetAsync(freq.ptr, 0, sizeof(unsigned) * cols, s));
        if (col32)
            k_lrc_freq<<<bgrid(nnz), kBT, 0, s>>>(static_cast<const std::int32_t*>(col), nnz, freq.as<unsigned>());
        else
            k_lrc_freq<<<bgrid(nnz), kBT, 0, s>>>(static_cast<const std::int64_t*>(col), nnz, freq.as<unsigned>());
        cols_in.ensure(sizeof(std::int32_t) * cols, false);
        k_lrc_iota<<<bgrid(cols), kBT, 0, s>>>(cols_in.as<std::int32_t>(), cols);
        keys_out.ensure(sizeof(unsigned) * cols, false);
        cols_out.ensure(sizeof(std::int32_t) * cols, false);
        std::size_t tb = 0;
        B200_CUDA(cub::DeviceRadixSort::SortPairsDescending(nullptr, tb, freq.as<unsigned>(), keys_out.as<unsigned>(),
                                                            cols_in.as<std::int32_t>(), cols_out.as<std::int32_t>(),
                                                            static_cast<int>(cols), 0, 32, s));
        tmp.ensure(tb, false);
        B200_CUDA(cub::DeviceRadixSort::SortPairsDescending(tmp.ptr, tb, freq.as<unsigned>(), keys_out.as<unsigned>(),
                                                            cols_in.as<std::int32_t>(), cols_out.as<std::int32_t>(),
                                                            static_cast<int>(cols), 0, 32, s));
        const int want = static_cast<int>(std::min<std::int64_t>(cap, cols));
        std::vector<unsigned> cnt(static_cast<std::size_t>(want));
        std::vector<std::int32_t> hc(static_cast<std::size_t>(want));
        B200_CUDA(cudaMemcpyAsync(cnt.data(), keys_out.ptr, sizeof(unsigned) * want, cudaMemcpyDeviceToHost, s));
        B200_CUDA(cudaMemcpyAsync(hc.data(), cols_out.ptr, sizeof(std::int32_t) * want, cudaMemcpyDeviceToHost, s));
        B200_CUDA(cudaStreamSynchronize(s));
        int k = 0;
        while (k < want && cnt[k] >= 2) covered += cnt[k++];
        if (static_cast<double>(covered) >= 0.05 * static_cast<double>(nnz)) {
            hot = k;
            hc.resize(static_cast<std::size_t>(hot));
            std::sort(hc.begin(), hc.end());
            o.hot_cols.ensure(sizeof(std::int32_t) * std::max(hot, 1));
            B200_CUDA(cudaMemcpyAsync(o.hot_cols.ptr, hc.data(), sizeof(std::int32_t) * hot, cudaMemcpyHostToDevice, s));
            slot.ensure(sizeof(std::int32_t) * cols, false);
            B200_CUDA(cudaMemsetAsync(slot.ptr, 0xff, sizeof(std::int32_t) * cols, s));
            k_lrc_slots<<<bgrid(hot), kBT, 0, s>>>(o.hot_cols.as<std::int32_t>(), hot, slot.as<std::int32_t>());
        } else {
            covered = 0;
        }
        B200_CUDA(cudaStreamSynchronize(s));
        for (DevBuf* b : {&freq, &keys_out, &cols_in, &cols_out, &tmp}) b->release();
    }
    if (!o.hot_cols.ptr) o.hot_cols.ensure(16);
    // ---- nonzeros ---------------------------------------------------------------
    o.val.ensure(sizeof(double) * std::max<std::int64_t>(total, 2), false);
    o.col.ensure(sizeof(std::uint32_t) * std::max<std::int64_t>(total, 4), false);
    if (col32)
        k_lrc_scatter<<<bgrid(total), kBT, 0, s>>>(static_cast<const std::int32_t*>(col) , val, nnz, total,
                                                   hot ? slot.as<std::int32_t>() : nullptr, hot, o.val.as<double>(),
                                                   o.col.as<std::uint32_t>());
    else
        k_lrc_scatter<<<bgrid(total), kBT, 0, s>>>(static_cast<const std::int64_t*>(col), val, nnz, total,
                                                   hot ? slot.as<std::int32_t>() : nullptr, hot, o.val.as<double>(),
                                                   o.col.as<std::uint32_t>());
    // ---- rows: starts, compaction ---------------------------------------------------
    DevBuf nonempty, comp;
    nonempty.ensure(sizeof(std::int32_t) * (rows + 1), false);
    comp.ensure(sizeof(std::int32_t) * (rows + 1), false);
    k_lrc_rows<<<bgrid(rows), kBT, 0, s>>>(rp, rows, o.col.as<std::uint32_t>(), nonempty.as<std::int32_t>());
    B200_CUDA(cudaMemsetAsync(nonempty.as<std::int32_t>() + rows, 0, sizeof(std::int32_t), s));
    {
        std::size_t tb = 0;
        B200_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tb, nonempty.as<std::int32_t>(), comp.as<std::int32_t>(),
                                                rows + 1, s));
        DevBuf tmp;
        tmp.ensure(tb, false);
        B200_CUDA(cub::DeviceScan::ExclusiveSum(tmp.ptr, tb, nonempty.as<std::int32_t>(), comp.as<std::int32_t>(),
                                                rows + 1, s));
        B200_CUDA(cudaStreamSynchronize(s));
        tmp.release();
    }
    std::int32_t rows_c = 0;
    B200_CUDA(cudaMemcpy(&rows_c, comp.as<std::int32_t>() + rows, sizeof rows_c, cudaMemcpyDeviceToHost));
    const bool has_empty = rows_c != rows;
    if (has_empty) {
        o.rmap.ensure(sizeof(std::int32_t) * std::max<std::int64_t>(rows_c, 1));
        o.empty.ensure(sizeof(std::int32_t) * std::max<std::int64_t>(rows - rows_c, 1));
        k_lrc_rmap<<<bgrid(rows), kBT, 0, s>>>(comp.as<std::int32_t>(), nonempty.as<std::int32_t>(), rows,
                                               o.rmap.as<std::int32_t>(), o.empty.as<std::int32_t>());
    }
    o.desc.ensure(sizeof(std::uint32_t) * std::max<std::int64_t>(units * 32, 4), false);
    k_lrc_desc<<<bgrid(units * 32), kBT, 0, s>>>(rp, rows, nnz, units, has_empty ? comp.as<std::int32_t>() : nullptr,
                                                 static_cast<std::uint32_t>(std::max(rows_c - 1, 0)),
                                                 o.desc.as<std::uint32_t>());
    B200_CUDA(cudaGetLastError());
    // crossing-row plan (short crossings first, then long ones)
    std::int64_t nshort = 0, nlong = 0;
    {
        DevBuf fs, fl, cnt;
        fs.ensure(sizeof(LrcFix) * std::max<std::int64_t>(units, 1), false);
        fl.ensure(sizeof(LrcFix) * std::max<std::int64_t>(units, 1), false);
        cnt.ensure(16, false);
        B200_CUDA(cudaMemsetAsync(cnt.ptr, 0, 16, s));
        k_lrc_plan<<<bgrid(units), kBT, 0, s>>>(rp, rows, nnz, units, has_empty ? comp.as<std::int32_t>() : nullptr,
                                                fs.as<LrcFix>(), fl.as<LrcFix>(), cnt.as<unsigned long long>());
        unsigned long long c[2] = {0, 0};
        B200_CUDA(cudaMemcpyAsync(c, cnt.ptr, 16, cudaMemcpyDeviceToHost, s));
        B200_CUDA(cudaStreamSynchronize(s));
        nshort = static_cast<std::int64_t>(c[0]);
        nlong = static_cast<std::int64_t>(c[1]);
        o.fix.ensure(sizeof(LrcFix) * std::max<std::int64_t>(nshort + nlong, 1));
        if (nshort)
            B200_CUDA(cudaMemcpyAsync(o.fix.ptr, fs.ptr, sizeof(LrcFix) * nshort, cudaMemcpyDeviceToDevice, s));
        if (nlong)
            B200_CUDA(cudaMemcpyAsync(o.fix.as<LrcFix>() + nshort, fl.ptr, sizeof(LrcFix) * nlong,
                                      cudaMemcpyDeviceToDevice, s));
        B200_CUDA(cudaStreamSynchronize(s));
        for (DevBuf* b : {&fs, &fl, &cnt}) b->release();
    }
    o.x_hot.ensure(sizeof(double) * static_cast<std::size_t>(hot + 2));
    B200_CUDA(cudaMemsetAsync(o.x_hot.ptr, 0, sizeof(double) * static_cast<std::size_t>(hot + 2), s));
    o.carry.ensure(sizeof(LrcCarry) * static_cast<std::size_t>(std::max<std::int64_t>(units, 1)));
    B200_CUDA(cudaStreamSynchronize(s));
    for (DevBuf* b : {&slot, &nonempty, &comp}) b->release();
    LrcDev& d = o.dev;
    d = LrcDev{};
    d.units = units;
    d.nnz = nnz;
    d.rows_c = rows_c;
    d.hot = hot;
    d.has_empty = has_empty;
    d.val = o.val.as<double>();
    d.col = o.col.as<std::uint32_t>();
    d.desc = o.desc.as<std::uint32_t>();
    d.rmap = has_empty ? o.rmap.as<std::int32_t>() : nullptr;
    d.empty = has_empty ? o.empty.as<std::int32_t>() : nullptr;
    d.nempty = rows - rows_c;
    d.hot_cols = o.hot_cols.as<std::int32_t>();
    d.x_hot = o.x_hot.as<double>();
    d.carry = o.carry.as<LrcCarry>();
    d.fix = o.fix.as<LrcFix>();
    d.nfix_short = nshort;
    d.nfix_long = nlong;
    o.hot_covered = covered;
    o.bytes = total * 12 + units * 32 * 4 + (has_empty ? rows * 4 : 0);
    o.valid = true;
}

void launch_spmv_lrc(const LrcDev& L, std::int64_t rows, const double* x, double* y, cudaStream_t s) {
    if (rows <= 0) return;
    if (!g_lrc_sms) {
        int dev = 0;
        B200_CUDA(cudaGetDevice(&dev));
        B200_CUDA(cudaDeviceGetAttribute(&g_lrc_sms, cudaDevAttrMultiProcessorCount, dev));
    }
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

bool launch_pagerank_lrc(const LrcDev& L, std::int64_t rows, const double* x, double* y, double d, cudaStream_t s) {
    if (rows <= 0 || L.units == 0) return false;  // nothing streamed: the caller's SpMV + update
    if (!g_lrc_sms) {
        int dev = 0;
        B200_CUDA(cudaGetDevice(&dev));
        B200_CUDA(cudaDeviceGetAttribute(&g_lrc_sms, cudaDevAttrMultiProcessorCount, dev));
    }
    const double tele = (1.0 - d) / static_cast<double>(rows);
    k_lrc_gather_hot<<<(L.hot + 1 + 255) / 256, 256, 0, s>>>(L.hot_cols, L.hot, x, L.x_hot);
    B200_CUDA(cudaGetLastError());
    if (L.rmap)
        lrc_launch<true, true, true>(L, x, y, s, d, tele);
    else
        lrc_launch<true, false, true>(L, x, y, s, d, tele);
    B200_CUDA(cudaGetLastError());
    return true;
}

}  // namespace b200
