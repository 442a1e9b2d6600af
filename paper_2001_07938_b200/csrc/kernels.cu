// kernels.cu — sm_100a kernels for the LiLAC harness path.
//
// Semantics restated from the reference interpreter (what_interp.cpp:87-108,
// kernels.lilac:1-12): one output element per row, accumulated from +0.0.
//  * csr_vector: S lanes per row, 16-byte streaming loads of val/col (L1
//    no-allocate), read-only gathers of x, shuffle reduction. Reassociates:
//    within the north-star tolerance, not bit-exact.
//  * csr_exact: one thread per row, left-to-right __dadd_rn(acc, __dmul_rn(.))
//    — bit-identical to the reference harness.
//  * jds: one thread per jagged row, coalesced val[jd_ptr[k]+j]; its per-row
//    order equals the reference's k order, so it is bit-exact too.
// SpMV is a streaming gather, not a dense contraction: no tensor cores.

#include "b200.hpp"
#include "p2p.hpp"

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <cmath>

namespace b200 {

namespace {

constexpr int kThreads = 256;
constexpr int kSMs = 148;
#ifndef LILAC_JDS_U
#define LILAC_JDS_U 20  // Parboil shape: 8 -> 17.1 us, 16 -> 16.4, 20-28 -> 14.35
#endif
constexpr int kJdsU = LILAC_JDS_U;  // JDS diagonals in flight per thread

// ---- load helpers -----------------------------------------------------------

__device__ __forceinline__ double2 ld_stream(const double* p) {
    double2 r;
    asm("ld.global.nc.L1::no_allocate.v2.f64 {%0, %1}, [%2];" : "=d"(r.x), "=d"(r.y) : "l"(p));
    return r;
}

// matrix streams: read once, L2 evict_first (keeps x and the rest resident)
__device__ __forceinline__ double2 ld_stream_ef(const double* p, std::uint64_t pol) {
    double2 r;
    asm("ld.global.nc.L1::no_allocate.L2::cache_hint.v2.f64 {%0, %1}, [%2], %3;"
        : "=d"(r.x), "=d"(r.y)
        : "l"(p), "l"(pol));
    return r;
}

struct Idx2 {
    long long a, b;
};

__device__ __forceinline__ Idx2 ld_stream_idx(const std::int32_t* p, std::uint64_t pol) {
    int a, b;
    asm("ld.global.nc.L1::no_allocate.L2::cache_hint.v2.s32 {%0, %1}, [%2], %3;" : "=r"(a), "=r"(b) : "l"(p), "l"(pol));
    return {a, b};
}

__device__ __forceinline__ Idx2 ld_stream_idx(const std::int64_t* p, std::uint64_t pol) {
    long long a, b;
    asm("ld.global.nc.L1::no_allocate.L2::cache_hint.v2.s64 {%0, %1}, [%2], %3;" : "=l"(a), "=l"(b) : "l"(p), "l"(pol));
    return {a, b};
}

__device__ __forceinline__ std::uint64_t make_evict_first() {
    std::uint64_t pol;
    asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}

__device__ __forceinline__ std::uint64_t make_evict_last() {
    std::uint64_t pol;
    asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}

__device__ __forceinline__ long long ld_stream_col(const std::int32_t* p, std::uint64_t pol) {
    int v;
    asm("ld.global.nc.L1::no_allocate.L2::cache_hint.s32 %0, [%1], %2;" : "=r"(v) : "l"(p), "l"(pol));
    return v;
}

__device__ __forceinline__ long long ld_stream_col(const std::int64_t* p, std::uint64_t pol) {
    long long v;
    asm("ld.global.nc.L1::no_allocate.L2::cache_hint.s64 %0, [%1], %2;" : "=l"(v) : "l"(p), "l"(pol));
    return v;
}

__device__ __forceinline__ double ld_stream_val(const double* p, std::uint64_t pol) {
    double v;
    asm("ld.global.nc.L1::no_allocate.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(p), "l"(pol));
    return v;
}

// x gathers: keep x in L2 (evict_last)
__device__ __forceinline__ double ld_gather(const double* p, std::uint64_t pol) {
    double v;
    asm("ld.global.nc.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(p), "l"(pol));
    return v;
}

__device__ __forceinline__ double warp_sum(double v, unsigned mask = 0xffffffffu) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(mask, v, o);
    return v;
}

// Block-wide sum with a fixed tree (deterministic). Result valid in thread 0.
__device__ __forceinline__ double block_sum(double v) {
    __shared__ double sh[kThreads / 32];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    v = warp_sum(v);
    __syncthreads();
    if (lane == 0) sh[w] = v;
    __syncthreads();
    if (w == 0) {
        v = lane < kThreads / 32 ? sh[lane] : 0.0;
        v = warp_sum(v);
    }
    return v;
}

// Last-CTA-done reduction of per-CTA partials in fixed order. Every CTA calls
// it after writing partials[blockIdx.x]; returns true in the CTA that must
// finish (its thread 0 then holds the total in *total).
__device__ __forceinline__ bool last_cta_sum(double* partials, unsigned int* ticket, double* total) {
    __shared__ bool last;
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) last = atomicAdd(ticket, 1u) == gridDim.x - 1;
    __syncthreads();
    if (!last) return false;
    __threadfence();
    double s = 0.0;
    for (unsigned i = threadIdx.x; i < gridDim.x; i += blockDim.x) s += __ldcg(partials + i);
    s = block_sum(s);
    if (threadIdx.x == 0) {
        *total = s;
        *ticket = 0u;
    }
    return true;
}

// ---- CSR vector kernel --------------------------------------------------------

// S lanes cooperate on a row; each lane consumes 2 consecutive nonzeros per
// step (one 16-byte val load, one 8/16-byte col load) and U steps are issued
// before any x gather is consumed. Row starts are rounded down to an even
// index so every vector load is aligned; the out-of-row elements are masked.
// One row's partial sum on one lane of an S-lane group: each lane consumes 2
// consecutive nonzeros per step (one 16-byte val load, one 8/16-byte col load)
// and U steps are issued before any x gather is consumed. The row start is
// rounded down to an even index so every vector load is aligned; the
// out-of-row elements are masked. The caller reduces over the group.
template <int S, int U, typename IdxT>
__device__ __forceinline__ double vector_row(std::int64_t start, std::int64_t end, int lane,
                                             const IdxT* __restrict__ col, const double* __restrict__ val,
                                             const double* __restrict__ x, std::uint64_t pol) {
    double acc = 0.0;
    for (std::int64_t jb = (start & ~std::int64_t(1)) + 2 * lane; jb < end; jb += 2 * S * U) {
        double2 v[U];
        Idx2 c[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const std::int64_t j = jb + 2 * S * u;
            if (j < end) {
                v[u] = ld_stream_ef(val + j, pol);
                c[u] = ld_stream_idx(col + j, pol);
            } else {
                v[u] = make_double2(0.0, 0.0);
                c[u] = {0, 0};
            }
        }
        double xa[U], xb[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const std::int64_t j = jb + 2 * S * u;
            xa[u] = (j < end && j >= start) ? __ldg(x + c[u].a) : 0.0;
            xb[u] = (j + 1 < end) ? __ldg(x + c[u].b) : 0.0;
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            acc += v[u].x * xa[u];
            acc += v[u].y * xb[u];
        }
    }
    return acc;
}

template <int S>
__device__ __forceinline__ unsigned group_mask() {
    return S == 32 ? 0xffffffffu : (((1u << S) - 1u) << ((threadIdx.x & 31) & ~(S - 1)));
}

// S lanes cooperate on a row (vector_row). Rows longer than max_len are left
// to the split plan's chunk path.
// Rows that fit one U=2 pass of the group (max row + 1 <= 4S: banded and
// stencil matrices), software-pipelined across the group's rows: the next
// row's row_ptr and val/col loads are issued before this row's x gathers are
// consumed, so two rows' streams are in flight per lane.
struct Pass {
    double2 v[2];
    Idx2 c[2];
};

template <int S, typename IdxT>
__device__ __forceinline__ void load_pass(Pass& p, std::int64_t start, std::int64_t end, int lane,
                                          const IdxT* __restrict__ col, const double* __restrict__ val,
                                          std::uint64_t pol) {
#pragma unroll
    for (int u = 0; u < 2; ++u) {
        const std::int64_t j = (start & ~std::int64_t(1)) + 2 * lane + 2 * S * u;
        if (j < end) {
            p.v[u] = ld_stream_ef(val + j, pol);
            p.c[u] = ld_stream_idx(col + j, pol);
        } else {
            p.v[u] = make_double2(0.0, 0.0);
            p.c[u] = {0, 0};
        }
    }
}

// Launch bounds for 5 CTAs per SM (48 registers, a 16-byte spill): 5.80 ->
// 5.37 ms on the N=420 stencil; at 6 (40 registers) the spills cost 7.1 ms.
template <int S, typename IdxT, bool DOT>
__global__ void __launch_bounds__(kThreads, 5) k_csr_vector_1p(std::int64_t rows,
                                                            const std::int64_t* __restrict__ row_ptr,
                                                            const IdxT* __restrict__ col,
                                                            const double* __restrict__ val,
                                                            const double* __restrict__ x,
                                                            double* __restrict__ y,
                                                            double* __restrict__ partials,
                                                            unsigned int* ticket, CgScalars* sc,
                                                            std::int64_t dot_off) {
    const int lane = threadIdx.x & (S - 1);
    const unsigned gmask = group_mask<S>();
    const std::int64_t groups = static_cast<std::int64_t>(gridDim.x) * (kThreads / S);
    const std::uint64_t pol = make_evict_first();
    double pq = 0.0;
    std::int64_t row = (static_cast<std::int64_t>(blockIdx.x) * kThreads + threadIdx.x) / S;
    std::int64_t start = 0, end = 0;
    Pass cur;
    if (row < rows) {
        start = __ldg(row_ptr + row);
        end = __ldg(row_ptr + row + 1);
        load_pass<S>(cur, start, end, lane, col, val, pol);
    }
    for (; row < rows; row += groups) {
        const std::int64_t nrow = row + groups;
        std::int64_t nstart = 0, nend = 0;
        if (nrow < rows) {
            nstart = __ldg(row_ptr + nrow);
            nend = __ldg(row_ptr + nrow + 1);
        }
        double xa[2], xb[2];
#pragma unroll
        for (int u = 0; u < 2; ++u) {
            const std::int64_t j = (start & ~std::int64_t(1)) + 2 * lane + 2 * S * u;
            xa[u] = (j < end && j >= start) ? __ldg(x + cur.c[u].a) : 0.0;
            xb[u] = (j + 1 < end) ? __ldg(x + cur.c[u].b) : 0.0;
        }
        Pass nxt;
        if (nrow < rows) load_pass<S>(nxt, nstart, nend, lane, col, val, pol);
        double acc = 0.0;
#pragma unroll
        for (int u = 0; u < 2; ++u) {
            acc += cur.v[u].x * xa[u];
            acc += cur.v[u].y * xb[u];
        }
#pragma unroll
        for (int o = S / 2; o > 0; o >>= 1) acc += __shfl_xor_sync(gmask, acc, o);
        if (lane == 0) {
            y[row] = acc;
            if (DOT) pq += acc * __ldg(x + dot_off + row);
        }
        cur = nxt;
        start = nstart;
        end = nend;
    }
    if (DOT) {
        double s = block_sum(pq);
        if (threadIdx.x == 0) partials[blockIdx.x] = s;
        double total;
        if (last_cta_sum(partials, ticket, &total) && threadIdx.x == 0) {
            if (sc->nranks > 1) {
                p2p_publish(sc, &total, 1);
            } else {
                sc->d = total;
                sc->rho0 = sc->rho;
                sc->alpha = sc->rho / total;
            }
        }
    }
}

template <int S, int U, typename IdxT, bool DOT>
__global__ void __launch_bounds__(kThreads) k_csr_vector(std::int64_t rows,
                                                         const std::int64_t* __restrict__ row_ptr,
                                                         const IdxT* __restrict__ col,
                                                         const double* __restrict__ val,
                                                         const double* __restrict__ x,
                                                         double* __restrict__ y,
                                                         double* __restrict__ partials,
                                                         unsigned int* ticket, CgScalars* sc,
                                                         std::int64_t dot_off, std::int64_t max_len) {
    const int lane = threadIdx.x & (S - 1);
    const unsigned gmask = group_mask<S>();
    const std::int64_t groups = static_cast<std::int64_t>(gridDim.x) * (kThreads / S);
    const std::uint64_t pol = make_evict_first();
    double pq = 0.0;
    for (std::int64_t row = (static_cast<std::int64_t>(blockIdx.x) * kThreads + threadIdx.x) / S;
         row < rows; row += groups) {
        const std::int64_t start = __ldg(row_ptr + row), end = __ldg(row_ptr + row + 1);
        if (end - start > max_len) continue;  // a long row of the split plan: chunked elsewhere
        double acc = vector_row<S, U>(start, end, lane, col, val, x, pol);
#pragma unroll
        for (int o = S / 2; o > 0; o >>= 1) acc += __shfl_xor_sync(gmask, acc, o);
        if (lane == 0) {
            y[row] = acc;
            if (DOT) pq += acc * __ldg(x + dot_off + row);
        }
    }
    if (DOT) {
        double s = block_sum(pq);
        if (threadIdx.x == 0) partials[blockIdx.x] = s;
        double total;
        if (last_cta_sum(partials, ticket, &total) && threadIdx.x == 0) {
            if (sc->nranks > 1) {
                p2p_publish(sc, &total, 1);  // the shard's partial; alpha after the exchange
            } else {
                sc->d = total;
                sc->rho0 = sc->rho;
                sc->alpha = sc->rho / total;
            }
        }
    }
}

// ---- split kernel (skewed rows) -------------------------------------------------
//
// One launch; warps pull work units from a global counter: first the chunks of
// the long rows (<= kSplitChunk nonzeros each, 8 loads in flight per lane),
// then blocks of short rows walked as the vector kernel does. The warp that
// completes a long row's last chunk sums the row's partials in chunk order
// (deterministic) and stores y. Why not merge-path alone: on the Kronecker
// scale-22 operator it is bound by shared-memory latency (binary searches, the
// sequential merge walk) at 0.92 ms.
#ifndef LILAC_SPLIT_MINB
#define LILAC_SPLIT_MINB 6
#endif
constexpr int kChunkU = 8;
constexpr int kShortPasses = 8;  // short-row unit: 8 passes of the warp's 32/S row groups

template <int S, typename IdxT>
__global__ void __launch_bounds__(kThreads, LILAC_SPLIT_MINB) k_csr_split(std::int64_t rows, const std::int64_t* __restrict__ row_ptr,
                                                        const IdxT* __restrict__ col,
                                                        const double* __restrict__ val,
                                                        const double* __restrict__ x, double* __restrict__ y,
                                                        SplitDev P, unsigned long long* work) {
    constexpr std::int64_t kRowsPerUnit = kShortPasses * (32 / S);
    const int lane = threadIdx.x & 31;
    const std::uint64_t pol = make_evict_first(), pgather = make_evict_last();
    const std::int64_t short_units = (rows + kRowsPerUnit - 1) / kRowsPerUnit;
    for (;;) {
        std::int64_t u = 0;
        if (lane == 0) u = static_cast<std::int64_t>(atomicAdd(work, 1ull));
        u = __shfl_sync(0xffffffffu, u, 0);
        if (u >= P.nchunks + short_units) return;
        if (u >= P.nchunks) {  // a block of short rows
            const std::int64_t r0 = (u - P.nchunks) * kRowsPerUnit;
            const int glane = lane & (S - 1);
            const unsigned gmask = group_mask<S>();
            for (std::int64_t row = r0 + lane / S; row < r0 + kRowsPerUnit && row < rows; row += 32 / S) {
                const std::int64_t start = __ldg(row_ptr + row), end = __ldg(row_ptr + row + 1);
                if (end - start > P.short_max) continue;
                double acc = vector_row<S, 2>(start, end, glane, col, val, x, pol);
#pragma unroll
                for (int o = S / 2; o > 0; o >>= 1) acc += __shfl_xor_sync(gmask, acc, o);
                if (glane == 0) y[row] = acc;
            }
            continue;
        }
        const std::int64_t lo = __ldg(P.chunk_lo + u), hi = __ldg(P.chunk_hi + u);
        double acc = 0.0;
        for (std::int64_t jb = lo + lane; jb < hi; jb += 32 * kChunkU) {
            long long cc[kChunkU];
            double vv[kChunkU];
#pragma unroll
            for (int k = 0; k < kChunkU; ++k) {
                const std::int64_t j = jb + 32 * k;
                cc[k] = j < hi ? ld_stream_col(col + j, pol) : 0;
                vv[k] = j < hi ? ld_stream_val(val + j, pol) : 0.0;
            }
#pragma unroll
            for (int k = 0; k < kChunkU; ++k)
                if (jb + 32 * k < hi) acc += vv[k] * ld_gather(x + cc[k], pgather);
        }
        acc = warp_sum(acc);
        if (lane == 0) {
            const std::int64_t i = __ldg(P.chunk_row + u);
            const std::int64_t f0 = __ldg(P.long_first + i), f1 = __ldg(P.long_first + i + 1);
            if (f1 - f0 == 1) {
                y[__ldg(P.long_rows + i)] = acc;
            } else {
                P.partial[u] = acc;
                __threadfence();
                if (atomicAdd(P.done + i, 1u) == static_cast<unsigned>(f1 - f0 - 1)) {
                    __threadfence();
                    double sum = 0.0;
                    for (std::int64_t k = f0; k < f1; ++k) sum += __ldcg(P.partial + k);
                    y[__ldg(P.long_rows + i)] = sum;
                    P.done[i] = 0u;  // ready for the next call
                }
            }
        }
        __syncwarp();
    }
}

// ---- exact kernels ------------------------------------------------------------

template <typename IdxT>
__global__ void __launch_bounds__(kThreads) k_csr_exact(std::int64_t rows,
                                                        const std::int64_t* __restrict__ row_ptr,
                                                        const IdxT* __restrict__ col,
                                                        const double* __restrict__ val,
                                                        const double* __restrict__ x,
                                                        double* __restrict__ y) {
    const std::int64_t stride = static_cast<std::int64_t>(gridDim.x) * kThreads;
    for (std::int64_t row = static_cast<std::int64_t>(blockIdx.x) * kThreads + threadIdx.x; row < rows;
         row += stride) {
        const std::int64_t start = row_ptr[row], end = row_ptr[row + 1];
        double acc = 0.0;
        for (std::int64_t j = start; j < end; ++j)
            acc = __dadd_rn(acc, __dmul_rn(__ldg(val + j), __ldg(x + static_cast<std::int64_t>(col[j]))));
        y[row] = acc;
    }
}

// JDS, thread per jagged row j (coalesced over j); y scattered through inv_perm.
#if LILAC_CTA_TRACE
__device__ unsigned long long g_jds_trace[3 * 4096];  // per block: SM, entry, exit (tools/jds_trace.py)
#endif
template <typename IdxT>
__global__ void __launch_bounds__(kThreads) k_jds(std::int64_t rows, const std::int64_t* __restrict__ nzcnt,
                                                  const std::int64_t* __restrict__ inv_perm,
                                                  const std::int64_t* __restrict__ jd_ptr,
                                                  const IdxT* __restrict__ col,
                                                  const double* __restrict__ val,
                                                  const double* __restrict__ x, double* __restrict__ y) {
#if LILAC_CTA_TRACE
    unsigned long long t_in;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t_in));
#endif
    const std::int64_t stride = static_cast<std::int64_t>(gridDim.x) * kThreads;
    for (std::int64_t j = static_cast<std::int64_t>(blockIdx.x) * kThreads + threadIdx.x; j < rows; j += stride) {
        const std::int64_t len = __ldg(nzcnt + j);
        double acc = 0.0;
        std::int64_t k = 0;
        // kJdsU diagonals in flight: all val/col loads of the group, then all x
        // gathers, then the sums in the reference k order (two memory round
        // trips per group; the longest jagged rows set the kernel time)
        for (; k + kJdsU <= len; k += kJdsU) {
            double v[kJdsU], xv[kJdsU];
            long long c[kJdsU];
#pragma unroll
            for (int u = 0; u < kJdsU; ++u) {
                const std::int64_t off = __ldg(jd_ptr + k + u) + j;
                asm("ld.global.nc.L1::no_allocate.f64 %0, [%1];" : "=d"(v[u]) : "l"(val + off));
                c[u] = static_cast<long long>(__ldg(col + off));
            }
#pragma unroll
            for (int u = 0; u < kJdsU; ++u) xv[u] = __ldg(x + c[u]);
#pragma unroll
            for (int u = 0; u < kJdsU; ++u) acc = __dadd_rn(acc, __dmul_rn(v[u], xv[u]));
        }
        if (k < len) {  // the last < kJdsU diagonals: one masked group, all loads in flight
            const std::int64_t rem = len - k;
            double v[kJdsU], xv[kJdsU];
            long long c[kJdsU];
#pragma unroll
            for (int u = 0; u < kJdsU; ++u) {
                v[u] = 0.0;
                c[u] = 0;
                if (u < rem) {
                    const std::int64_t off = __ldg(jd_ptr + k + u) + j;
                    asm("ld.global.nc.L1::no_allocate.f64 %0, [%1];" : "=d"(v[u]) : "l"(val + off));
                    c[u] = static_cast<long long>(__ldg(col + off));
                }
            }
#pragma unroll
            for (int u = 0; u < kJdsU; ++u) xv[u] = u < rem ? __ldg(x + c[u]) : 0.0;
#pragma unroll
            for (int u = 0; u < kJdsU; ++u)
                if (u < rem) acc = __dadd_rn(acc, __dmul_rn(v[u], xv[u]));
        }
        y[__ldg(inv_perm + j)] = acc;
    }
#if LILAC_CTA_TRACE
    __syncthreads();
    if (threadIdx.x == 0 && blockIdx.x < 4096) {
        unsigned long long t_out;
        unsigned smid;
        asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t_out));
        asm volatile("mov.u32 %0, %smid;" : "=r"(smid));
        g_jds_trace[3 * blockIdx.x] = smid;
        g_jds_trace[3 * blockIdx.x + 1] = t_in;
        g_jds_trace[3 * blockIdx.x + 2] = t_out;
    }
#endif
}

// Segmented JDS (JdsSeg in b200.hpp): every lane loads the val/col of its
// (at most kJdsSegD) diagonals and gathers x at once, so a row's memory chain
// is two trips whatever its length; the products are then summed in k order,
// the running sum passed from lane to lane of the row's group by shuffles
// (__dmul_rn / __dadd_rn, as the reference: bit-identical). Small register
// footprint: the grid is about one wave on the Parboil shape.
#ifndef LILAC_JDS_SEG_BLOCKS
#define LILAC_JDS_SEG_BLOCKS 6
#endif
template <typename IdxT>
__global__ void __launch_bounds__(kThreads, LILAC_JDS_SEG_BLOCKS)
    k_jds_seg(const std::int64_t* __restrict__ nzcnt, const std::int64_t* __restrict__ inv_perm,
              const std::int64_t* __restrict__ jd_ptr, const IdxT* __restrict__ col, const double* __restrict__ val,
              const double* __restrict__ x, double* __restrict__ y, const JdsSeg sg) {
#if LILAC_CTA_TRACE
    unsigned long long t_in;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t_in));
    if (threadIdx.x == 0 && blockIdx.x < 4096) g_jds_trace[3 * blockIdx.x + 1] = t_in;
#endif
    const std::int64_t gw = (static_cast<std::int64_t>(blockIdx.x) * kThreads + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (gw >= sg.warp0[sg.nzones]) return;  // warp-uniform
    int z = 0;
    while (z + 1 < sg.nzones && gw >= sg.warp0[z + 1]) ++z;
    const int G = sg.g[z], rpw = 32 / G;
    const int r = lane / G, seg = lane - r * G;
    const std::int64_t j = sg.row0[z] + (gw - sg.warp0[z]) * rpw + r;
    const bool active = r < rpw && j < sg.row0[z + 1];
    const std::int64_t k0 = static_cast<std::int64_t>(seg) * kJdsSegD;
    // the output slot is loaded with nzcnt, not after the sum (cold L2:
    // 17.4 -> 16.9 us). Loading the diagonal starts early as well was slower
    // (12.3 -> 13.7 us warm: ten more loads per lane).
    const std::int64_t ip = active && seg == 0 ? __ldg(inv_perm + j) : 0;
    const std::int64_t len = active ? __ldg(nzcnt + j) : 0;
    const int cnt = static_cast<int>(len - k0 < 0 ? 0 : (len - k0 > kJdsSegD ? kJdsSegD : len - k0));
    double v[kJdsSegD];
    long long c[kJdsSegD];
#pragma unroll
    for (int u = 0; u < kJdsSegD; ++u) {
        v[u] = 0.0;
        c[u] = 0;
        if (u < cnt) {
            const std::int64_t off = __ldg(jd_ptr + k0 + u) + j;
            asm("ld.global.nc.L1::no_allocate.f64 %0, [%1];" : "=d"(v[u]) : "l"(val + off));
            c[u] = static_cast<long long>(__ldg(col + off));
        }
    }
#pragma unroll
    for (int u = 0; u < kJdsSegD; ++u)
        if (u < cnt) v[u] = __dmul_rn(v[u], __ldg(x + c[u]));
    // the row's running sum, segment by segment in k order
    double acc = 0.0;
    const int base = r * G;
    for (int s = 0; s < G; ++s) {
        if (seg == s) {
#pragma unroll
            for (int u = 0; u < kJdsSegD; ++u)
                if (u < cnt) acc = __dadd_rn(acc, v[u]);
        }
        const int src = base + s;
        acc = __shfl_sync(0xffffffffu, acc, src < 32 ? src : lane);
    }
    if (active && seg == 0) y[ip] = acc;
#if LILAC_CTA_TRACE
    __syncwarp();
    if (lane == 0 && blockIdx.x < 4096) {  // the block's last warp to finish wins
        unsigned long long t_out;
        unsigned smid;
        asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t_out));
        asm volatile("mov.u32 %0, %smid;" : "=r"(smid));
        g_jds_trace[3 * blockIdx.x] = smid;
        atomicMax(&g_jds_trace[3 * blockIdx.x + 2], t_out);
    }
#endif
}

// JDS when perm is not a bijection: thread per original row (uncoalesced,
// still the reference's semantics and order).
template <typename IdxT>
__global__ void __launch_bounds__(kThreads) k_jds_rowwise(std::int64_t rows,
                                                          const std::int64_t* __restrict__ nzcnt,
                                                          const std::int64_t* __restrict__ perm,
                                                          const std::int64_t* __restrict__ jd_ptr,
                                                          const IdxT* __restrict__ col,
                                                          const double* __restrict__ val,
                                                          const double* __restrict__ x,
                                                          double* __restrict__ y) {
    const std::int64_t stride = static_cast<std::int64_t>(gridDim.x) * kThreads;
    for (std::int64_t i = static_cast<std::int64_t>(blockIdx.x) * kThreads + threadIdx.x; i < rows; i += stride) {
        const std::int64_t p = perm[i];
        const std::int64_t len = nzcnt[p];
        double acc = 0.0;
        for (std::int64_t k = 0; k < len; ++k) {
            const std::int64_t off = jd_ptr[k] + p;
            acc = __dadd_rn(acc, __dmul_rn(val[off], x[static_cast<std::int64_t>(col[off])]));
        }
        y[i] = acc;
    }
}

// ---- validation / narrowing ----------------------------------------------------

__global__ void k_scan_cols(const std::int64_t* __restrict__ col64, std::int64_t nnz,
                            std::int32_t* __restrict__ col32, unsigned long long* d_max, int* d_bad) {
    const std::int64_t stride = static_cast<std::int64_t>(gridDim.x) * blockDim.x;
    long long m = -1;
    int bad = 0;
    for (std::int64_t i = static_cast<std::int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < nnz; i += stride) {
        const long long c = col64[i];
        bad |= c < 0;
        m = c > m ? c : m;
        if (col32) col32[i] = static_cast<std::int32_t>(c);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        long long om = __shfl_xor_sync(0xffffffffu, m, o);
        m = om > m ? om : m;
        bad |= __shfl_xor_sync(0xffffffffu, bad, o);
    }
    if ((threadIdx.x & 31) == 0) {
        if (m >= 0) atomicMax(d_max, static_cast<unsigned long long>(m) + 1ull);
        if (bad) atomicOr(d_bad, 1);
    }
}

__global__ void k_check_row_ptr(const std::int64_t* __restrict__ rp, std::int64_t rows, std::int64_t nnz,
                                unsigned long long* d_max, int* d_bad) {
    const std::int64_t stride = static_cast<std::int64_t>(gridDim.x) * blockDim.x;
    long long m = 0;
    int bad = 0;
    for (std::int64_t i = static_cast<std::int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < rows; i += stride) {
        const long long a = rp[i], b = rp[i + 1];
        if (b > a) {
            bad |= (a < 0 || b > nnz) ? 1 : 0;
            m = (b - a) > m ? (b - a) : m;
        } else if (b < a) {
            bad |= 2;  // non-monotone: legal (empty row), but rules out merge kernels
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        long long om = __shfl_xor_sync(0xffffffffu, m, o);
        m = om > m ? om : m;
        bad |= __shfl_xor_sync(0xffffffffu, bad, o);
    }
    if ((threadIdx.x & 31) == 0) {
        atomicMax(d_max, static_cast<unsigned long long>(m));
        if (bad) atomicOr(d_bad, bad);
    }
}

__global__ void k_fill_i64(std::int64_t* p, std::int64_t n, std::int64_t v) {
    const std::int64_t stride = static_cast<std::int64_t>(gridDim.x) * blockDim.x;
    for (std::int64_t i = static_cast<std::int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride)
        p[i] = v;
}

__global__ void k_invert_perm(const std::int64_t* __restrict__ perm, std::int64_t rows, std::int64_t* inv, int* d_bad) {
    const std::int64_t stride = static_cast<std::int64_t>(gridDim.x) * blockDim.x;
    for (std::int64_t i = static_cast<std::int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < rows; i += stride) {
        const long long p = perm[i];
        if (p < 0 || p >= rows) {
            atomicOr(d_bad, 1);  // out of range: the reference throws OutOfBounds
            continue;
        }
        unsigned long long prev = atomicExch(reinterpret_cast<unsigned long long*>(inv + p),
                                             static_cast<unsigned long long>(i));
        if (static_cast<long long>(prev) != -1) atomicOr(d_bad, 2);  // not a bijection
    }
}

__global__ void k_check_jds(const std::int64_t* __restrict__ nzcnt, const std::int64_t* __restrict__ jd_ptr,
                            std::int64_t rows, std::int64_t njd, std::int64_t nnz, int* d_bad) {
    const std::int64_t stride = static_cast<std::int64_t>(gridDim.x) * blockDim.x;
    for (std::int64_t p = static_cast<std::int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; p < rows; p += stride) {
        const long long len = nzcnt[p];
        if (len <= 0) continue;
        if (len > njd) {
            atomicOr(d_bad, 1);
            continue;
        }
        for (long long k = 0; k < len; ++k) {
            const long long off = jd_ptr[k] + p;
            if (off < 0 || off >= nnz) {
                atomicOr(d_bad, 1);
                break;
            }
        }
    }
}

// ---- BLAS-1 --------------------------------------------------------------------

// Deterministic dot: CTA b owns a fixed contiguous slice, threads stride it
// with 16-byte loads, fixed-tree block sum, last CTA sums the partials in order.
// Publishes a scalar result to host-mapped memory: value, system fence, then
// the call's sequence number (the host spins on it instead of a D2H + sync).
__device__ __forceinline__ void post_host(double v, HostSlot slot) {
    if (!slot.value) return;
    *reinterpret_cast<volatile double*>(slot.value) = v;
    __threadfence_system();
    *reinterpret_cast<volatile unsigned*>(slot.flag) = slot.seq;
}

__global__ void __launch_bounds__(kThreads) k_dot(const double* __restrict__ a, const double* __restrict__ b,
                                                  std::int64_t n, double* result, double* partials,
                                                  unsigned int* ticket, HostSlot slot) {
    const std::int64_t per = (n + gridDim.x - 1) / gridDim.x;
    const std::int64_t lo = min(n, per * blockIdx.x), hi = min(n, lo + per);
    double s = 0.0;
    // vector part: 16-byte pairs. a and b may be any 8-byte-aligned views
    // (a sub-range of a mirror, a torch slice): pair boundaries follow a's
    // address parity, and when b's parity differs the slice is walked scalar.
    const unsigned pa = static_cast<unsigned>(reinterpret_cast<std::uintptr_t>(a) >> 3) & 1u;
    const unsigned pb = static_cast<unsigned>(reinterpret_cast<std::uintptr_t>(b) >> 3) & 1u;
    std::int64_t vlo = lo + ((lo + pa) & 1), vhi = hi - ((hi + pa) & 1);
    if (pa != pb || vlo > vhi) vlo = vhi = lo;
    for (std::int64_t i = lo + threadIdx.x; i < vlo; i += kThreads) s += a[i] * b[i];
    for (std::int64_t i = vlo + 2 * threadIdx.x; i < vhi; i += 2 * kThreads) {
        const double2 x = ld_stream(a + i), y = ld_stream(b + i);
        s += x.x * y.x;
        s += x.y * y.y;
    }
    for (std::int64_t i = max(vhi, vlo) + threadIdx.x; i < hi; i += kThreads) s += a[i] * b[i];
    s = block_sum(s);
    if (threadIdx.x == 0) partials[blockIdx.x] = s;
    double total;
    if (last_cta_sum(partials, ticket, &total) && threadIdx.x == 0) {
        *result = total;
        post_host(total, slot);
    }
}

// Reference order, one thread: bit-identical to what_interp.cpp:97-101.
__global__ void k_dot_exact(const double* a, const double* b, std::int64_t n, double* result, HostSlot slot) {
    if (blockIdx.x != 0 || threadIdx.x != 0) return;
    double acc = 0.0;
    for (std::int64_t i = 0; i < n; ++i) acc = __dadd_rn(acc, __dmul_rn(a[i], b[i]));
    *result = acc;
    post_host(acc, slot);
}

// out = y + alpha*x (axpy) or out = x + beta*y (xpay); out may alias y (each
// element is read before it is written by the same thread).
template <bool XPAY>
__global__ void k_vec2(std::int64_t n, double* out, const double* y, double s, const double* __restrict__ x) {
    const std::int64_t stride = static_cast<std::int64_t>(gridDim.x) * blockDim.x;
    for (std::int64_t i = static_cast<std::int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride)
        out[i] = XPAY ? __dadd_rn(x[i], __dmul_rn(s, y[i])) : __dadd_rn(y[i], __dmul_rn(s, x[i]));
}

unsigned grid_for(std::int64_t threads, unsigned cap = kSMs * 16) {
    std::int64_t b = (threads + kThreads - 1) / kThreads;
    return static_cast<unsigned>(std::max<std::int64_t>(1, std::min<std::int64_t>(b, cap)));
}

#ifndef LILAC_VEC_U
#define LILAC_VEC_U 2
#endif

template <int S, typename IdxT, bool DOT>
void vector_launch(const CsrDev& A, const double* x, double* y, double* partials, unsigned* ticket,
                   CgScalars* sc, unsigned grid, cudaStream_t s, std::int64_t dot_off, std::int64_t max_len) {
    static const int onepass = [] {  // LILAC_B200_VEC_1P: 0 off, 1 whenever rows fit, else by size
        const char* e = std::getenv("LILAC_B200_VEC_1P");
        return (e && *e) ? std::atoi(e) : 2;
    }();
    // measured on the 27-point stencil: the plain kernel (2048 threads per SM)
    // wins while the matrix is small (N=256, 3.6e8 nonzeros: 0.73 vs 0.67 of
    // copy) and degrades as the footprint grows (TLB reach: N=420, 2.0e9
    // nonzeros: 0.625); the pipelined one (1024 threads, two rows in flight)
    // holds 0.68 at every size; the crossover is near 8 GB of matrix
    const std::int64_t mbytes = A.nnz * (A.col32 ? 12 : 16);
    if (onepass && A.max_row + 1 <= 4 * S && max_len >= A.max_row &&
        (onepass == 1 || mbytes > (std::int64_t(8) << 30))) {
        k_csr_vector_1p<S, IdxT, DOT><<<grid, kThreads, 0, s>>>(A.rows, A.row_ptr, static_cast<const IdxT*>(A.col),
                                                                A.val, x, y, partials, ticket, sc, dot_off);
        return;
    }
    k_csr_vector<S, LILAC_VEC_U, IdxT, DOT><<<grid, kThreads, 0, s>>>(A.rows, A.row_ptr, static_cast<const IdxT*>(A.col),
                                                            A.val, x, y, partials, ticket, sc, dot_off, max_len);
}

template <typename IdxT, bool DOT>
void vector_dispatch(const CsrDev& A, int S, const double* x, double* y, double* partials, unsigned* ticket,
                     CgScalars* sc, unsigned grid, cudaStream_t s, std::int64_t dot_off = 0,
                     std::int64_t max_len = INT64_MAX) {
    switch (S) {
    case 2: vector_launch<2, IdxT, DOT>(A, x, y, partials, ticket, sc, grid, s, dot_off, max_len); break;
    case 4: vector_launch<4, IdxT, DOT>(A, x, y, partials, ticket, sc, grid, s, dot_off, max_len); break;
    case 8: vector_launch<8, IdxT, DOT>(A, x, y, partials, ticket, sc, grid, s, dot_off, max_len); break;
    case 16: vector_launch<16, IdxT, DOT>(A, x, y, partials, ticket, sc, grid, s, dot_off, max_len); break;
    default: vector_launch<32, IdxT, DOT>(A, x, y, partials, ticket, sc, grid, s, dot_off, max_len); break;
    }
}

}  // namespace

// ---- host launchers ------------------------------------------------------------------

const char* csr_kernel_name(CsrKernel k) {
    switch (k) {
    case CsrKernel::Auto: return "auto";
    case CsrKernel::Vector: return "vector";
    case CsrKernel::Merge: return "merge";
    case CsrKernel::Exact: return "exact";
    case CsrKernel::Tiled: return "tiled";
    case CsrKernel::Split: return "split";
    case CsrKernel::Lane: return "lane";
    }
    return "?";
}

CsrKernel parse_csr_kernel(const std::string& s) {
    if (s.empty() || s == "auto") return CsrKernel::Auto;
    if (s == "vector") return CsrKernel::Vector;
    if (s == "merge") return CsrKernel::Merge;
    if (s == "split") return CsrKernel::Split;
    if (s == "exact") return CsrKernel::Exact;
    if (s == "tiled") return CsrKernel::Tiled;
    if (s == "lane") return CsrKernel::Lane;
    throw Error(Errc::DataError, "unknown CSR kernel '" + s + "' (auto, vector, tiled, split, merge, lane, exact)");
}

int csr_vector_width(const CsrDev& A) {
    const double mean = A.rows > 0 ? static_cast<double>(A.nnz) / static_cast<double>(A.rows) : 0.0;
    // lanes so that one U=2 step (4*S nonzeros) covers roughly a mean row
    int S = 2;
    while (S < 32 && 4.0 * S < mean) S *= 2;
    return S;
}

CsrKernel choose_csr_kernel(const CsrDev& A, CsrKernel requested) {
    // the plain arrays were dropped once a derived layout was built (keep_plain_csr)
    if (!A.val && A.tiled) return CsrKernel::Tiled;
    if (!A.val && A.lrc) return CsrKernel::Lane;
    if (requested == CsrKernel::Exact) return CsrKernel::Exact;
    if (requested == CsrKernel::Vector) return CsrKernel::Vector;
    if (requested == CsrKernel::Merge) return A.merge ? CsrKernel::Merge : CsrKernel::Vector;
    if (requested == CsrKernel::Split) return A.split ? CsrKernel::Split : CsrKernel::Vector;
    if (requested == CsrKernel::Tiled) return A.tiled ? CsrKernel::Tiled : CsrKernel::Vector;
    if (requested == CsrKernel::Lane) return A.lrc ? CsrKernel::Lane : CsrKernel::Vector;
    // Auto: the derived layouts exist only when they were judged to pay at
    // upload (tcsr_wanted / merge_wanted)
    if (A.tiled) return CsrKernel::Tiled;
    if (A.lrc) return CsrKernel::Lane;
    if (A.split) return CsrKernel::Split;
    if (A.merge) return CsrKernel::Merge;
    return CsrKernel::Vector;
}

static unsigned vector_grid(const CsrDev& A, int S) {
    return grid_for(A.rows * static_cast<std::int64_t>(S), kSMs * 8 * 4);
}

template <int S, typename IdxT>
void split_launch(const CsrDev& A, const double* x, double* y, cudaStream_t s) {
    const SplitDev& P = *A.split;
    static unsigned per_sm = 0;
    if (!per_sm) {
        int b = 0;
        B200_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, k_csr_split<S, IdxT>, kThreads, 0));
        per_sm = static_cast<unsigned>(std::max(b, 1));
    }
    // one resident wave of warps pulling work units; the counter restarts per call
    B200_CUDA(cudaMemsetAsync(P.work, 0, sizeof(unsigned long long), s));
    k_csr_split<S, IdxT><<<kSMs * per_sm, kThreads, 0, s>>>(A.rows, A.row_ptr, static_cast<const IdxT*>(A.col),
                                                            A.val, x, y, P, P.work);
}

template <typename IdxT>
void split_dispatch(const CsrDev& A, int S, const double* x, double* y, cudaStream_t s) {
    switch (S) {
    case 2: split_launch<2, IdxT>(A, x, y, s); break;
    case 4: split_launch<4, IdxT>(A, x, y, s); break;
    case 8: split_launch<8, IdxT>(A, x, y, s); break;
    case 16: split_launch<16, IdxT>(A, x, y, s); break;
    default: split_launch<32, IdxT>(A, x, y, s); break;
    }
}

void launch_spmv_split(const CsrDev& A, const double* x, double* y, cudaStream_t s) {
    if (A.rows <= 0) return;
    const int S = csr_vector_width(A);
    if (A.col32)
        split_dispatch<std::int32_t>(A, S, x, y, s);
    else
        split_dispatch<std::int64_t>(A, S, x, y, s);
    B200_CUDA(cudaGetLastError());
}

void launch_spmv_csr(const CsrDev& A, const double* x, double* y, CsrKernel k, cudaStream_t s) {
    if (A.rows <= 0) return;
    k = choose_csr_kernel(A, k);
    if (k == CsrKernel::Tiled) {
        launch_spmv_tiled(*A.tiled, A.rows, x, y, nullptr, nullptr, nullptr, s);
        return;
    }
    if (k == CsrKernel::Merge) {
        launch_spmv_merge(A, x, y, s);
        return;
    }
    if (k == CsrKernel::Split) {
        launch_spmv_split(A, x, y, s);
        return;
    }
    if (k == CsrKernel::Lane) {
        launch_spmv_lrc(*A.lrc, A.rows, x, y, s);
        return;
    }
    if (k == CsrKernel::Exact) {
        unsigned g = grid_for(A.rows);
        if (A.col32)
            k_csr_exact<std::int32_t><<<g, kThreads, 0, s>>>(A.rows, A.row_ptr, static_cast<const std::int32_t*>(A.col), A.val, x, y);
        else
            k_csr_exact<std::int64_t><<<g, kThreads, 0, s>>>(A.rows, A.row_ptr, static_cast<const std::int64_t*>(A.col), A.val, x, y);
    } else {
        const int S = csr_vector_width(A);
        const unsigned g = vector_grid(A, S);
        if (A.col32)
            vector_dispatch<std::int32_t, false>(A, S, x, y, nullptr, nullptr, nullptr, g, s);
        else
            vector_dispatch<std::int64_t, false>(A, S, x, y, nullptr, nullptr, nullptr, g, s);
    }
    B200_CUDA(cudaGetLastError());
}

void launch_spmv_csr_dot(const CsrDev& A, const double* p, double* q, double* partials, unsigned* ticket,
                         CgScalars* sc, cudaStream_t s, std::int64_t dot_off) {
    if (A.tiled) {
        launch_spmv_tiled(*A.tiled, A.rows, p, q, partials, ticket, sc, s, dot_off);
        return;
    }
    if (A.lrc || A.split || A.merge) {  // rows finish only after the fix-up: dot in its own pass
        if (A.lrc)
            launch_spmv_lrc(*A.lrc, A.rows, p, q, s);
        else if (A.split)
            launch_spmv_split(A, p, q, s);
        else
            launch_spmv_merge(A, p, q, s);
        launch_cg_dot_scalars(p + dot_off, q, A.rows, partials, ticket, sc, s);
        return;
    }
    const int S = csr_vector_width(A);
    const unsigned g = std::min<unsigned>(vector_grid(A, S), kMaxParts);
    if (A.col32)
        vector_dispatch<std::int32_t, true>(A, S, p, q, partials, ticket, sc, g, s, dot_off);
    else
        vector_dispatch<std::int64_t, true>(A, S, p, q, partials, ticket, sc, g, s, dot_off);
    B200_CUDA(cudaGetLastError());
}

JdsSeg jds_segments(const std::int64_t* nz, std::int64_t rows) {
    JdsSeg sg;
    if (rows <= 0) return sg;
    for (std::int64_t j = 1; j < rows; ++j)
        if (nz[j] > nz[j - 1]) return sg;  // not length-sorted
    if (nz[0] > static_cast<std::int64_t>(32) * kJdsSegD || nz[rows - 1] < 0) return sg;
    auto groups = [](std::int64_t L) { return L <= kJdsSegD ? 1 : static_cast<int>((L + kJdsSegD - 1) / kJdsSegD); };
    std::int64_t j = 0, w = 0;
    int z = 0;
    while (j < rows) {
        const int G = groups(nz[j]);
        // first row of a smaller group count: nz[row] <= kJdsSegD * (G - 1)
        std::int64_t lo = j, hi = rows;
        const std::int64_t lim = static_cast<std::int64_t>(kJdsSegD) * (G - 1);
        while (lo < hi) {
            const std::int64_t mid = lo + (hi - lo) / 2;
            if (G > 1 && nz[mid] <= lim) hi = mid; else lo = mid + 1;
        }
        const std::int64_t end = G > 1 ? lo : rows;
        const int rpw = 32 / G;
        sg.g[z] = G;
        sg.row0[z] = j;
        sg.warp0[z] = w;
        w += (end - j + rpw - 1) / rpw;
        ++z;
        j = end;
    }
    sg.row0[z] = rows;
    sg.warp0[z] = w;
    sg.nzones = z;
    return sg;
}

bool jds_segmented(const JdsDev& A) {
    static const bool seg_off = [] {
        const char* e = std::getenv("LILAC_B200_JDS");
        return e && std::strcmp(e, "rowthread") == 0;  // experiments: the thread-per-row kernel
    }();
    return A.inv_perm && A.seg.nzones > 0 && !seg_off;
}

void launch_spmv_jds(const JdsDev& A, const double* x, double* y, cudaStream_t s) {
    if (A.rows <= 0) return;
    if (jds_segmented(A)) {
        const std::int64_t threads = A.seg.warp0[A.seg.nzones] * 32;
        const unsigned gs = static_cast<unsigned>((threads + kThreads - 1) / kThreads);
        if (A.col32)
            k_jds_seg<std::int32_t><<<gs, kThreads, 0, s>>>(A.nzcnt, A.inv_perm, A.jd_ptr,
                                                            static_cast<const std::int32_t*>(A.col), A.val, x, y,
                                                            A.seg);
        else
            k_jds_seg<std::int64_t><<<gs, kThreads, 0, s>>>(A.nzcnt, A.inv_perm, A.jd_ptr,
                                                            static_cast<const std::int64_t*>(A.col), A.val, x, y,
                                                            A.seg);
        B200_CUDA(cudaGetLastError());
        return;
    }
    const unsigned g = grid_for(A.rows);
    if (A.inv_perm) {
        if (A.col32)
            k_jds<std::int32_t><<<g, kThreads, 0, s>>>(A.rows, A.nzcnt, A.inv_perm, A.jd_ptr,
                                                       static_cast<const std::int32_t*>(A.col), A.val, x, y);
        else
            k_jds<std::int64_t><<<g, kThreads, 0, s>>>(A.rows, A.nzcnt, A.inv_perm, A.jd_ptr,
                                                       static_cast<const std::int64_t*>(A.col), A.val, x, y);
    } else {
        if (A.col32)
            k_jds_rowwise<std::int32_t><<<g, kThreads, 0, s>>>(A.rows, A.nzcnt, A.perm, A.jd_ptr,
                                                               static_cast<const std::int32_t*>(A.col), A.val, x, y);
        else
            k_jds_rowwise<std::int64_t><<<g, kThreads, 0, s>>>(A.rows, A.nzcnt, A.perm, A.jd_ptr,
                                                               static_cast<const std::int64_t*>(A.col), A.val, x, y);
    }
    B200_CUDA(cudaGetLastError());
}

void launch_scan_cols(const std::int64_t* col64, std::int64_t nnz, std::int32_t* col32, unsigned long long* d_max,
                      int* d_bad, cudaStream_t s) {
    if (nnz <= 0) return;
    k_scan_cols<<<grid_for(nnz, kSMs * 8), kThreads, 0, s>>>(col64, nnz, col32, d_max, d_bad);
    B200_CUDA(cudaGetLastError());
}

void launch_check_row_ptr(const std::int64_t* row_ptr, std::int64_t rows, std::int64_t nnz,
                          unsigned long long* d_max, int* d_bad, cudaStream_t s) {
    if (rows <= 0) return;
    k_check_row_ptr<<<grid_for(rows, kSMs * 8), kThreads, 0, s>>>(row_ptr, rows, nnz, d_max, d_bad);
    B200_CUDA(cudaGetLastError());
}

void launch_invert_perm(const std::int64_t* perm, std::int64_t rows, std::int64_t* inv, int* d_bad, cudaStream_t s) {
    if (rows <= 0) return;
    k_fill_i64<<<grid_for(rows, kSMs * 8), kThreads, 0, s>>>(inv, rows, -1);
    k_invert_perm<<<grid_for(rows, kSMs * 8), kThreads, 0, s>>>(perm, rows, inv, d_bad);
    B200_CUDA(cudaGetLastError());
}

void launch_check_jds(const std::int64_t* nzcnt, const std::int64_t* jd_ptr, std::int64_t rows, std::int64_t njd,
                      std::int64_t nnz, int* d_bad, cudaStream_t s) {
    if (rows <= 0) return;
    k_check_jds<<<grid_for(rows, kSMs * 8), kThreads, 0, s>>>(nzcnt, jd_ptr, rows, njd, nnz, d_bad);
    B200_CUDA(cudaGetLastError());
}

int dot_parts_for(std::int64_t n) {
    // ~4K elements per CTA at minimum; at most 8 CTAs per SM
    std::int64_t g = (n + 4095) / 4096;
    return static_cast<int>(std::max<std::int64_t>(1, std::min<std::int64_t>(g, kSMs * 8)));
}

void launch_dot(const double* a, const double* b, std::int64_t n, double* result, double* partials,
                unsigned int* ticket, cudaStream_t s, HostSlot slot) {
    k_dot<<<dot_parts_for(n), kThreads, 0, s>>>(a, b, n, result, partials, ticket, slot);
    B200_CUDA(cudaGetLastError());
}

void launch_dot_exact(const double* a, const double* b, std::int64_t n, double* result, cudaStream_t s,
                      HostSlot slot) {
    k_dot_exact<<<1, 32, 0, s>>>(a, b, n, result, slot);
    B200_CUDA(cudaGetLastError());
}

void launch_axpy(std::int64_t n, double* y, double alpha, const double* x, cudaStream_t s) {
    launch_axpy_to(n, y, y, alpha, x, s);
}

void launch_xpay(std::int64_t n, double* y, double beta, const double* x, cudaStream_t s) {
    launch_xpay_to(n, y, y, beta, x, s);
}

void launch_axpy_to(std::int64_t n, double* out, const double* y, double alpha, const double* x, cudaStream_t s) {
    if (n <= 0) return;
    k_vec2<false><<<grid_for(n, kSMs * 8), kThreads, 0, s>>>(n, out, y, alpha, x);
    B200_CUDA(cudaGetLastError());
}

void launch_xpay_to(std::int64_t n, double* out, const double* y, double beta, const double* x, cudaStream_t s) {
    if (n <= 0) return;
    k_vec2<true><<<grid_for(n, kSMs * 8), kThreads, 0, s>>>(n, out, y, beta, x);
    B200_CUDA(cudaGetLastError());
}

#if LILAC_CTA_TRACE
extern "C" int b200_debug_jds_trace(unsigned long long* out, int n) {
    return cudaMemcpyFromSymbol(out, g_jds_trace, sizeof(unsigned long long) * std::min(n, 3 * 4096)) == cudaSuccess
               ? 0
               : 1;
}
#endif

}  // namespace b200
